"""Slab domain decomposition of one large scene (BASELINE config 5).

The global grid is cut along x into windows owned by ranks (one GPU each).
A particle belongs to the window that owns its base cell.  Each window's
device context covers its owned x-range plus ``ghost_bricks`` 4-node brick
layers on either side (mpm_set_slab); per substep:

  1. particle stage (G2P(n) + F/stress + P2G(n+1)) into the local grid;
  2. halo reduction: touched ghost bricks are packed sparsely (global brick
     id + 64 nodes of momentum/mass) and sent to the owning neighbour, which
     adds them into its bricks (mpm_halo_pack / mpm_halo_unpack_add);
  3. grid op on the window (walls and tools in global coordinates);
  4. velocity halo: the owner returns the velocities of exactly the bricks it
     received, which overwrite the sender's ghost bricks;
and at the end of each re-binning stretch particles whose base cell left the
owned range migrate to the neighbour (mpm_extract_migrants /
mpm_append_particles) before the next re-binning.  Ghost layers must cover the
drift of one stretch (SimParams.rebin_interval substeps).

Exchanges go through an ``Exchange`` object: ``LocalExchange`` copies device
buffers between windows living in one process (single-GPU emulation and
tests), ``TorchExchange`` uses torch.distributed point-to-point send/recv
(NCCL over NVLink between GPUs; gloo on CPU for protocol tests).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib, core
from .errors import ParameterError

NF = 26          # particle float fields (csrc/common.cuh)
ROWS = NF + 2    # + material id + particle id


def balanced_partition(base_x, res_x: int, ranks: int) -> list[tuple[int, int]]:
    """Owned base-cell x ranges [lo, hi) (multiples of 4 nodes) holding about
    the same number of particles each: cuts at the particle-count quantiles of
    the 4-node brick columns, every window at least one column wide.  Raises
    ParameterError when fewer brick columns hold particles than there are
    ranks (some window would start empty)."""
    bricks = res_x // 4
    if ranks < 1 or bricks < ranks:
        raise ParameterError("too many slabs for the grid")
    col = np.clip(np.asarray(base_x, dtype=np.int64) // 4, 0, bricks - 1)
    hist = np.bincount(col, minlength=bricks).astype(np.float64)
    if np.count_nonzero(hist) < ranks:
        raise ParameterError(f"only {np.count_nonzero(hist)} occupied 4-node x columns for {ranks} slabs")
    cum = np.cumsum(hist)
    total = cum[-1]
    cuts, lo = [], 0
    for r in range(1, ranks):
        # first column boundary whose cumulative count reaches r/ranks of the total,
        # leaving at least one column and one occupied column for every later rank
        c = int(np.searchsorted(cum, total * r / ranks, side="left")) + 1
        c = max(c, lo + 1)
        while c < bricks and cum[c - 1] - (cum[lo - 1] if lo else 0.0) == 0:
            c += 1  # this window must hold particles
        c = min(c, bricks - (ranks - r))
        while np.count_nonzero(hist[c:]) < ranks - r:
            c -= 1
        cuts.append(c)
        lo = c
    edges = [0] + cuts + [bricks]
    return [(4 * a, 4 * b) for a, b in zip(edges, edges[1:])]


def partition(res_x: int, ranks: int, weights=None) -> list[tuple[int, int]]:
    """Owned base-cell x ranges [lo, hi) per rank, multiples of 4 nodes."""
    bricks = res_x // 4
    if ranks < 1 or bricks < ranks:
        raise ParameterError("too many slabs for the grid")
    w = np.ones(ranks) if weights is None else np.asarray(weights, dtype=np.float64)
    cuts = np.round(np.cumsum(w) / w.sum() * bricks).astype(int)
    lo = 0
    out = []
    for r in range(ranks):
        hi = int(cuts[r]) if r < ranks - 1 else bricks
        hi = max(hi, lo + 1)
        out.append((4 * lo, 4 * hi))
        lo = hi
    return out


class SlabWindow:
    """One rank's window: a SimState over the local grid + slab configuration."""

    def __init__(self, grid: core.Grid, own: tuple[int, int], x, v, F, C, mass, vol0, mat, ids,
                 ghost_bricks: int = 2, device: int | None = None, capacity: int | None = None):
        self.global_grid = grid
        self.own = own
        g = 4 * ghost_bricks
        nx, ny, nz = grid.resolution
        self.offset = max(0, own[0] - g)
        end = min(nx, own[1] + g)
        res = (end - self.offset, ny, nz)
        dx = grid.dx
        local = core.Grid(res, (res[0] * dx, ny * dx, nz * dx))
        xl = np.array(x, dtype=np.float64, copy=True)
        xl[:, 0] -= self.offset * dx
        self.state = core.SimState(local, xl, v, F, C, mass, vol0, mat, device=device)
        self.ids = np.asarray(ids, dtype=np.int32)
        self.ghost_bricks = ghost_bricks
        self.capacity = capacity
        self._configured = False

    def configure(self, materials, params, colliders=None, rows=None):
        st = self.state
        theta = core._theta(st, params) if colliders else None
        ctx = st._prepare(materials, params, theta)
        if not self._configured:
            L = _lib.lib()
            gres = (ctypes.c_int * 3)(*self.global_grid.resolution)
            off = (ctypes.c_int * 3)(self.offset, 0, 0)
            ctx.call("mpm_set_slab", gres, off, self.ghost_bricks)
            if self.capacity:
                ctx.call("mpm_reserve", ctypes.c_int64(int(self.capacity)))
            # the device keeps global particle ids in its original-index slots;
            # from here on the window is read through download(), not SimState fields
            ctx.call("mpm_set_ids", _lib.ptr(self.ids, _lib._I32))
            st._slab_window = True
            self._configured = True
        if colliders:
            st._packed_colliders(colliders, params)
            st._upload_colliders()
            st._upload_pose_rows(*rows)
        return ctx

    def buffers(self, side):
        ctx = self.state._ctx
        si, sd, ri, rd = (_lib._VP() for _ in range(4))
        cap = ctypes.c_int64()
        ctx.call("mpm_halo_buffers", side, ctypes.byref(si), ctypes.byref(sd), ctypes.byref(ri),
                 ctypes.byref(rd), ctypes.byref(cap))
        return si.value, sd.value, ri.value, rd.value, cap.value

    def download(self):
        """(ids, x global, v, F, C) of the particles currently owned, device order."""
        ctx = self.state._ctx
        n = int(_lib.lib().mpm_particle_count(ctx.h))
        ids = np.empty(n, np.int32)
        x, v = np.empty((n, 3)), np.empty((n, 3))
        F, C = np.empty((n, 3, 3)), np.empty((n, 3, 3))
        ctx.call("mpm_download_rows", _lib.ptr(ids, _lib._I32), _lib.ptr(x), _lib.ptr(v), _lib.ptr(F),
                 _lib.ptr(C))
        return ids, x, v, F, C


class LocalExchange:
    """All windows in this process (one GPU): exchanges are device copies."""

    def __init__(self, windows):
        self.w = windows

    def halo(self, counts, phase):
        """counts[r][side] records packed by window r toward `side`; phase 'mass'
        delivers window r's side-1 records to r+1's side-0 receive buffers (and
        side-0 to r-1's side-1), 'vel' replies in the opposite direction."""
        L = _lib.lib()
        recv = [[0, 0] for _ in self.w]
        for r, win in enumerate(self.w):
            for side, nb in ((0, r - 1), (1, r + 1)):
                if nb < 0 or nb >= len(self.w):
                    continue
                m = counts[r][side]
                si, sd, _, _, _ = win.buffers(side)
                _, _, ri, rd, _ = self.w[nb].buffers(1 - side)
                if phase == "mass":
                    L.mpm_device_copy(ri, si, 4 * m)
                L.mpm_device_copy(rd, sd, 16 * 64 * m)
                recv[nb][1 - side] = m
        return recv

    def migrate(self, outgoing):
        """outgoing[r] = {side: (ptr, m)} (packed ROWS x m blocks) -> appended
        to the neighbours."""
        for r, out in enumerate(outgoing):
            for side, (ptr, m) in out.items():
                nb = r - 1 if side == 0 else r + 1
                if m == 0 or nb < 0 or nb >= len(self.w):
                    continue
                self.w[nb].state._ctx.call("mpm_append_particles", ptr, ctypes.c_int64(m),
                                           ctypes.c_int64(m), self.w[r].offset)


class TorchExchange:
    """torch.distributed point-to-point between neighbouring ranks (one window
    per rank): NCCL on the device tensors; with the gloo backend (CPU-only
    point-to-point) the tensors are staged through host memory, which lets
    the multi-process path run as several processes on one GPU in tests."""

    def __init__(self, window, rank, world, device="cuda", host_staging=None):
        import torch.distributed as dist
        self.win, self.rank, self.world, self.device = window, rank, world, device
        self.host_staging = (dist.get_backend() == "gloo") if host_staging is None else bool(host_staging)

    def _sendrecv(self, send: dict, recv_shapes: dict, dtype):
        import torch
        import torch.distributed as dist
        ops, out = [], {}
        where = "cpu" if self.host_staging else self.device
        for nb, t in send.items():
            ops.append(dist.P2POp(dist.isend, t.to(where) if self.host_staging else t, nb))
        for nb, shape in recv_shapes.items():
            out[nb] = torch.empty(shape, dtype=dtype, device=where)
            ops.append(dist.P2POp(dist.irecv, out[nb], nb))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        if self.host_staging:
            out = {nb: t.to(self.device) for nb, t in out.items()}
        return out

    def counts(self, mine: dict):
        """Exchange int64 counts with the neighbours: {nb: count} -> {nb: count}."""
        import torch
        send = {nb: torch.tensor([c], dtype=torch.int64, device=self.device) for nb, c in mine.items()}
        got = self._sendrecv(send, {nb: (1,) for nb in mine}, torch.int64)
        return {nb: int(t.item()) for nb, t in got.items()}

    def payload(self, mine: dict, recv_counts: dict, width: int, dtype):
        """Exchange per-neighbour tensors of shape (count, width)."""
        return self._sendrecv(mine, {nb: (recv_counts[nb], width) for nb in recv_counts}, dtype)


class IpcExchange:
    """Peer-memory halo exchange between neighbouring ranks: each window maps
    its neighbours' receive buffers (CUDA IPC; NVLink P2P between GPUs) and
    the pack kernels write straight into them (mpm_ipc_halo); the streams are
    ordered by counters in device memory (stream wait / write-value
    operations), so a substep has no host barrier (interprocess events plus
    two host barriers per substep remain as the fallback).  Migration at
    re-binning and the one-time handle exchange go through torch.distributed."""

    def __init__(self, window, rank, world, device="cuda"):
        self.host = TorchExchange(window, rank, world, device)
        self.win, self.rank, self.world, self.device = window, rank, world, device
        self.sides = None
        self.device_ordered = False

    def connect(self, ctx):
        """Export our buffers / events, map the neighbours' (collective: every
        rank calls it once, when its window's context exists)."""
        import torch.distributed as dist
        if self.sides is not None:
            return
        L = _lib.lib()
        size = int(L.mpm_ipc_blob_size())
        blobs = {}
        for side in (0, 1):
            buf = ctypes.create_string_buffer(size)
            ctx.call("mpm_ipc_export", side, buf)
            blobs[side] = buf.raw
        every = [None] * self.world
        dist.all_gather_object(every, blobs)
        self.sides = 0
        for side, nb in _neighbours(self.rank, self.world).items():
            ctx.call("mpm_ipc_import", side, every[nb][1 - side])
            self.sides |= 1 << side
        mode = ctypes.c_int(0)
        ctx.call("mpm_ipc_mode", ctypes.byref(mode))
        # every rank must agree (a mixed pair would deadlock)
        modes = [None] * self.world
        dist.all_gather_object(modes, int(mode.value))
        self.device_ordered = all(m == 1 for m in modes)
        dist.barrier()

    def counts(self, mine):
        return self.host.counts(mine)

    def _sendrecv(self, send, recv_shapes, dtype):
        return self.host._sendrecv(send, recv_shapes, dtype)

    def halo(self, ctx, phase):
        ctx.call("mpm_ipc_halo", phase, self.sides)


def step_local(windows, exchange: LocalExchange, materials, params, colliders=None, pose_rows=None):
    """One frame (params.substeps_per_frame substeps) of every window in this process."""
    nsub = params.substeps_per_frame
    L = int(params.rebin_interval)
    inverted = 0
    for win in windows:
        win.configure(materials, params, colliders, pose_rows)
    s = 0
    while s < nsub:
        span = min(L, nsub - s)
        for win in windows:
            win.state._ctx.call("mpm_stage_begin", nsub, int(bool(colliders)))
        for t in range(span):
            sub = s + t
            for win in windows:
                win.state._ctx.call("mpm_stage_particles", int(t == 0))
            counts = []
            for win in windows:
                c = []
                for side in (0, 1):
                    n = ctypes.c_int64()
                    win.state._ctx.call("mpm_halo_pack", side, ctypes.byref(n))
                    c.append(n.value)
                counts.append(c)
            recv = exchange.halo(counts, "mass")
            for r, win in enumerate(windows):
                for side in (0, 1):
                    win.state._ctx.call("mpm_halo_unpack_add", side, ctypes.c_int64(recv[r][side]))
            for win in windows:
                win.state._ctx.call("mpm_stage_grid", sub, int(sub != nsub - 1))
            vcounts = []
            for win in windows:
                c = []
                for side in (0, 1):
                    n = ctypes.c_int64()
                    win.state._ctx.call("mpm_halo_pack_vel", side, ctypes.byref(n))
                    c.append(n.value)
                vcounts.append(c)
            # velocity replies travel back toward the sender of each brick
            vrecv = exchange.halo(vcounts, "vel")
            for r, win in enumerate(windows):
                for side in (0, 1):
                    win.state._ctx.call("mpm_halo_unpack_vel", side, ctypes.c_int64(vrecv[r][side]))
        for win in windows:
            inv = ctypes.c_int64()
            win.state._ctx.call("mpm_stage_end", ctypes.byref(inv))
            inverted += inv.value
        outgoing = []
        for win in windows:
            nlo, nhi, plo, phi, cap = (ctypes.c_int64(), ctypes.c_int64(), _lib._VP(), _lib._VP(),
                                       ctypes.c_int64())
            win.state._ctx.call("mpm_extract_migrants", win.own[0], win.own[1], ctypes.byref(nlo),
                                ctypes.byref(nhi), ctypes.byref(plo), ctypes.byref(phi), ctypes.byref(cap))
            outgoing.append({0: (plo.value, nlo.value), 1: (phi.value, nhi.value)})
        exchange.migrate(outgoing)
        s += span
    return inverted


class PeerExchange(LocalExchange):
    """All windows in this process, exchanged through peer memory: the halo
    pack kernels write straight into the neighbour window's receive buffers
    (mpm_peer_connect + mpm_ipc_halo, the same kernels as IpcExchange between
    processes) and the windows' streams are ordered by events recorded and
    waited in host issue order, so a substep issues no host synchronisation
    at all."""

    def __init__(self, windows):
        from concurrent.futures import ThreadPoolExecutor
        super().__init__(windows)
        self.sides = []
        self.connected = False
        self.pool = ThreadPoolExecutor(max_workers=len(windows))

    def connect(self):
        if self.connected:
            return
        L = _lib.lib()
        n = len(self.w)
        for r in range(n - 1):
            h = self.w[r].state._ctx.h
            _lib.check(L.mpm_peer_connect(h, 1, self.w[r + 1].state._ctx.h), h, "mpm_peer_connect")
        self.sides = [(1 if r > 0 else 0) | (2 if r < n - 1 else 0) for r in range(n)]
        self.connected = True


def step_local_peer(windows, exchange: PeerExchange, materials, params, colliders=None, pose_rows=None):
    """One frame of every window in this process with peer-memory halos:
    per substep every window's particle stage, halo phases and grid op are
    enqueued on its own stream without host synchronisation; the host syncs
    once per re-binning stretch (inverted count + migration).  Returns the
    frame's inverted-element count summed over windows."""
    nsub = params.substeps_per_frame
    L = int(params.rebin_interval)
    inverted = 0
    for win in windows:
        win.configure(materials, params, colliders, pose_rows)
    exchange.connect()
    ctxs = [win.state._ctx for win in windows]
    sides = exchange.sides
    s = 0
    while s < nsub:
        span = min(L, nsub - s)
        for c in ctxs:
            c.call("mpm_stage_begin", nsub, int(bool(colliders)))
        for t in range(span):
            sub = s + t
            for c in ctxs:
                c.call("mpm_stage_particles", int(t == 0))
            # each halo phase is issued for every window before the next phase
            # (the event waits of a phase follow the neighbours' records)
            for phase in (0, 1, None, 2, 3):
                for r, c in enumerate(ctxs):
                    if phase is None:
                        c.call("mpm_stage_grid", sub, int(sub != nsub - 1))
                    elif sides[r]:
                        c.call("mpm_ipc_halo", phase, sides[r])
        # stretch end, one host thread per window (the ctypes calls release the
        # GIL): each window's final G2P, inverted count and migrant extraction
        # synchronise only that window's stream, concurrently with the others
        outgoing = list(exchange.pool.map(_stretch_end, windows))
        inverted += sum(o[0] for o in outgoing)
        exchange.migrate([o[1] for o in outgoing])
        s += span
    return inverted


def _stretch_end(win):
    c = win.state._ctx
    inv = ctypes.c_int64()
    c.call("mpm_stage_end", ctypes.byref(inv))
    nlo, nhi, plo, phi, cap = (ctypes.c_int64(), ctypes.c_int64(), _lib._VP(), _lib._VP(), ctypes.c_int64())
    c.call("mpm_extract_migrants", win.own[0], win.own[1], ctypes.byref(nlo), ctypes.byref(nhi),
           ctypes.byref(plo), ctypes.byref(phi), ctypes.byref(cap))
    return inv.value, {0: (plo.value, nlo.value), 1: (phi.value, nhi.value)}


def gather(windows, n_total: int):
    """Global x, v, F, C (particle-id order) from all windows of this process."""
    x, v = np.full((n_total, 3), np.nan), np.full((n_total, 3), np.nan)
    F, C = np.full((n_total, 3, 3), np.nan), np.full((n_total, 3, 3), np.nan)
    for win in windows:
        ids, xw, vw, Fw, Cw = win.download()
        x[ids], v[ids], F[ids], C[ids] = xw, vw, Fw, Cw
    return x, v, F, C


def split_state(grid: core.Grid, x, v, F, C, mass, vol0, mat, ranks: int, ghost_bricks: int = 2,
                device: int | None = None, capacity_factor: float = 1.5):
    """Cut a global particle set into slab windows (base-cell ownership)."""
    dx = grid.dx
    base = np.floor(np.asarray(x)[:, 0] / dx - 0.5).astype(np.int64)
    # windows of equal particle count (a scene that does not span the domain
    # would otherwise leave the outer windows empty)
    parts = balanced_partition(base, grid.resolution[0], ranks)
    wins = []
    ids = np.arange(len(x), dtype=np.int32)
    for own in parts:
        sel = (base >= own[0]) & (base < own[1])
        if not sel.any():
            raise ParameterError(f"slab window {own} would start without particles")
        cap = int(max(16, capacity_factor * sel.sum() + 1024))
        wins.append(SlabWindow(grid, own, x[sel], v[sel], F[sel], C[sel], mass[sel], vol0[sel], mat[sel],
                               ids[sel], ghost_bricks=ghost_bricks, device=device, capacity=cap))
    return wins


def rank_window(grid: core.Grid, positions, rest_volume: float, density: float, ranks: int, rank: int,
                ghost_bricks: int = 2, device: int | None = None, capacity_factor: float = 1.5) -> SlabWindow:
    """This rank's window of a fresh scene (F = I, v = C = 0, one material),
    built from the global positions without materialising the global
    v / F / C arrays (a 64 M-particle scene on every rank of a node would
    otherwise hold 14 GB of host state per rank).  Same cuts as split_state."""
    x = np.asarray(positions)
    base = np.floor(x[:, 0] / grid.dx - 0.5).astype(np.int64)
    own = balanced_partition(base, grid.resolution[0], ranks)[rank]
    sel = np.nonzero((base >= own[0]) & (base < own[1]))[0]
    n = len(sel)
    cap = int(max(16, capacity_factor * n + 1024))
    vol = np.full(n, rest_volume)
    return SlabWindow(grid, own, x[sel], np.zeros((n, 3)), np.broadcast_to(np.eye(3), (n, 3, 3)),
                      np.zeros((n, 3, 3)), density * vol, vol, np.zeros(n, np.int32), sel.astype(np.int32),
                      ghost_bricks=ghost_bricks, device=device, capacity=cap)


# ---------------------------------------------------------------------------
# one window per rank (torchrun): exchanges over torch.distributed
# ---------------------------------------------------------------------------

def _dev_tensor(nbytes_or_shape, dtype, device):
    import torch
    return torch.empty(nbytes_or_shape, dtype=dtype, device=device)


def _neighbours(rank, world):
    return {side: nb for side, nb in ((0, rank - 1), (1, rank + 1)) if 0 <= nb < world}


def _halo_exchange(win: SlabWindow, ex: TorchExchange, counts: dict, with_ids: bool):
    """Send our packed side buffers to the neighbours, receive theirs into our
    receive buffers.  counts: {side: records}.  Returns {side: records received}."""
    import torch
    L = _lib.lib()
    nbs = _neighbours(ex.rank, ex.world)
    got = ex.counts({nb: counts[side] for side, nb in nbs.items()})
    recv = {}
    for name, width, dtype, elem in ((("ids", 1, torch.int32, 4),) if with_ids else ()) + (("data", 256, torch.float32, 4),):
        send = {}
        for side, nb in nbs.items():
            si, sd, _, _, _ = win.buffers(side)
            t = _dev_tensor((counts[side], width), dtype, ex.device)
            L.mpm_device_copy(t.data_ptr(), si if name == "ids" else sd, counts[side] * width * elem)
            send[nb] = t
        out = ex.payload(send, got, width, dtype)
        for side, nb in nbs.items():
            _, _, ri, rd, _ = win.buffers(side)
            n = got[nb]
            L.mpm_device_copy(ri if name == "ids" else rd, out[nb].data_ptr(), n * width * elem)
            recv[side] = n
        torch.cuda.synchronize()
    return {side: recv.get(side, 0) for side in (0, 1)}


def step_distributed(win: SlabWindow, ex, materials, params, colliders=None, pose_rows=None):
    """One frame for this rank's window; halos travel through the exchange
    (TorchExchange: torch.distributed point-to-point; IpcExchange: the pack
    kernels write into the neighbours' mapped buffers), migrants over
    torch.distributed."""
    import torch
    L = _lib.lib()
    ctx = win.configure(materials, params, colliders, pose_rows)
    if isinstance(ex, IpcExchange):
        ex.connect(ctx)
    nsub = params.substeps_per_frame
    span_max = int(params.rebin_interval)
    inverted = 0
    s = 0
    while s < nsub:
        span = min(span_max, nsub - s)
        ctx.call("mpm_stage_begin", nsub, int(bool(colliders)))
        for t in range(span):
            sub = s + t
            ctx.call("mpm_stage_particles", int(t == 0))
            if isinstance(ex, IpcExchange):
                import torch.distributed as dist
                ex.halo(ctx, 0)
                if not ex.device_ordered:
                    dist.barrier()  # event fallback: records before the matching waits
                ex.halo(ctx, 1)
                ctx.call("mpm_stage_grid", sub, int(sub != nsub - 1))
                ex.halo(ctx, 2)
                if not ex.device_ordered:
                    dist.barrier()
                ex.halo(ctx, 3)
                continue
            counts = {}
            for side in (0, 1):
                n = ctypes.c_int64()
                ctx.call("mpm_halo_pack", side, ctypes.byref(n))
                counts[side] = n.value
            recv = _halo_exchange(win, ex, counts, with_ids=True)
            for side in (0, 1):
                ctx.call("mpm_halo_unpack_add", side, ctypes.c_int64(recv[side]))
            ctx.call("mpm_stage_grid", sub, int(sub != nsub - 1))
            vcounts = {}
            for side in (0, 1):
                n = ctypes.c_int64()
                ctx.call("mpm_halo_pack_vel", side, ctypes.byref(n))
                vcounts[side] = n.value
            vrecv = _halo_exchange(win, ex, vcounts, with_ids=False)
            for side in (0, 1):
                ctx.call("mpm_halo_unpack_vel", side, ctypes.c_int64(vrecv[side]))
        inv = ctypes.c_int64()
        ctx.call("mpm_stage_end", ctypes.byref(inv))
        inverted += inv.value
        # migration
        nlo, nhi, plo, phi, cap = (ctypes.c_int64(), ctypes.c_int64(), _lib._VP(), _lib._VP(), ctypes.c_int64())
        ctx.call("mpm_extract_migrants", win.own[0], win.own[1], ctypes.byref(nlo), ctypes.byref(nhi),
                 ctypes.byref(plo), ctypes.byref(phi), ctypes.byref(cap))
        nbs = _neighbours(ex.rank, ex.world)
        mine = {0: (plo.value, nlo.value), 1: (phi.value, nhi.value)}
        got = ex.counts({nb: mine[side][1] for side, nb in nbs.items()})
        send = {}
        for side, nb in nbs.items():
            ptr, m = mine[side]
            t = _dev_tensor((ROWS, m), torch.float32, ex.device)
            L.mpm_device_copy(t.data_ptr(), ptr, 4 * ROWS * m)  # packed ROWS x m block: one copy
            send[nb] = t
        ops_out = ex._sendrecv({nb: t.reshape(-1) for nb, t in send.items()},
                               {nb: (ROWS * got[nb],) for nb in got}, torch.float32)
        torch.cuda.synchronize()
        offsets = getattr(ex, "_nb_offsets", None)
        if offsets is None:  # window offsets are fixed: exchanged once
            offsets = ex._nb_offsets = ex.counts({nb: win.offset for nb in nbs.values()})
        for nb, t in ops_out.items():
            m = got[nb]
            if m:
                ctx.call("mpm_append_particles", _lib._VP(t.data_ptr()), ctypes.c_int64(m), ctypes.c_int64(m),
                         offsets[nb])
        torch.cuda.synchronize()
        s += span
    # the frame's inverted-element count and NaN flag over all windows (the
    # reference's StepReport.inverted_particles is global, core.py:316-320):
    # one all-reduce per frame
    import torch.distributed as dist
    flag = ctypes.c_int(0)
    ctx.call("mpm_has_nan", ctypes.byref(flag))
    red = torch.tensor([inverted, int(flag.value != 0)], dtype=torch.int64, device=ex.device)
    dist.all_reduce(red)
    win.last_nan = bool(red[1].item())
    return int(red[0].item())
