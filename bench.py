"""Benchmark: MLS-MPM Neo-Hookean substep throughput on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c3] [--particles P] [--no-cpu-baseline]

Workload (N=1): BASELINE config 3 -- a 1 M-particle Neo-Hookean slab on a
256^3 grid pressed 3 cm deep by a box tool moving down at 0.5 m/s, then held
(SimParams defaults:
dt 5e-4, 25 substeps per step, theta 0.5 dx, Coulomb mu 0.4).  One "step" is
one ``softmpm.step`` frame = 25 substeps.  Metric: particle-substeps/s.

* value     device-resident frames timed with CUDA events on the context
            stream (pose table built on the host and uploaded per frame, as
            ``step`` does); L2 is flushed (512 MiB memset) between frames.
* e2e       same frames through the C-ABI with HOST fp64 buffers: upload of
            x/v/F/C from pinned memory + 25 substeps + download of x/v/F/C,
            wall clock with the copies inside the timed region.
* roofline  dominant kernel of the substep (g2p_stress_kernel or
            p2g_tile_kernel; one launch = one substep of every particle);
            achieved = 200 B x particles / mean launch time,
            peak = MEASURED_PEAKS.json hbm_gbs; substep_frac uses the whole
            substep time instead.
* cpu_baseline  the CPU oracle O1 (oracle/, C restatement of the reference's
            numba kernels, OpenMP over all host cores) on a bounded sample of
            the same scene.
* --impl reference  times that CPU path alone on this config (the driver's
            reference arm); rank 0 only under torchrun.
N>1 (torchrun): every rank runs its own replica scene on its own GPU (batched
independent environments, BASELINE config 4 style; no data-path
collective) -> "scaling": "weak"; time = max over ranks.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "particle-substeps/sec (MLS-MPM, Neo-Hookean)"
UNIT = "particle-substeps/s"
NOMINAL_HBM_GBS = 8000.0  # B200 datasheet HBM3e bandwidth (report beside the measured peak)
GRID_BYTES_PER_NODE = 56   # SURVEY 8d grid term per active node
BYTES_PER_PARTICLE_SUBSTEP = 200  # fp32 x,v,F,C read+written once + mass,vol0


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def _ncu_traffic(kernel_prefix: str, config: str):
    """DRAM bytes per launch of the dominant kernel from the newest committed
    `ncu --set full` summary OF THIS CONFIG (profiles/rNN_ncu_<kernel>_<config>.json,
    written by tools/ncu_summary.py from a capture of this bench), or None --
    a capture of another configuration is never borrowed."""
    import glob
    best = None
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", f"r*_ncu_*_{config}.json"))):
        try:
            with open(path) as f:
                d = json.load(f)
        except Exception:
            continue
        for rec in d if isinstance(d, list) else [d]:
            if kernel_prefix in str(rec.get("kernel", "")) and rec.get("dram_bytes"):
                best = (rec["dram_bytes"], os.path.relpath(path, ROOT), rec.get("dram_bytes_warm"))
    return best


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0:  # sampler running before timing starts
                time.sleep(0.01)
            self.skip = len(self.lines)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        lines = self.lines[getattr(self, "skip", 0):] or self.lines[-1:]
        for ln in lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[2:6]):
                if val.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def build_scene(config: str, particles: int | None, seed: int):
    from paper_2402_01181_b200 import scenes
    if config == "c4":  # CPU legs: one environment (environments run sequentially on the CPU)
        b, mats, params, fns = scenes.c4_envs(count=particles or 30_000, env_ids=[seed - 1])
        st = b.state
        return st, mats, params, [c for c in b.colliders[0]], fns[0]
    kw = {"seed": seed}
    if particles:
        kw["count"] = particles
    return scenes.BUILDERS[config](**kw)


def pose_rows(st, cols, params, pose_fn, t0):
    """Per-substep pose table exactly as core.step builds it."""
    from paper_2402_01181_b200.core import pose_table
    return list(pose_table(st, cols, params, pose_fn, t0))


def cpu_oracle_rate(config, particles, seed, substeps, threads):
    """O1 (fp64 CPU restatement of the reference kernels) particle-substeps/s."""
    from oracle import oracle as O
    import paper_2402_01181_b200 as sm
    st, mats, params, cols, pose_fn = build_scene(config, particles, seed)
    O.set_threads(threads)
    g = st.grid
    op = O.OracleParams(res=g.resolution, dx=g.dx, theta=0.5 * g.dx, chunks=8)
    osim = O.OracleSim(op, st.x, st.v, st.F, st.C, st.mass, st.vol0, st.material_id, mats[0].mu,
                       mats[0].lam)
    t = 0.0
    times = []
    for i in range(substeps + 1):
        t0 = time.perf_counter()
        if cols:
            pose_fn(cols, t)
        osim.substep(sm.pack_colliders(cols) if cols else None)
        times.append(time.perf_counter() - t0)
        t += params.dt
    n = st.particle_count
    dt_med = float(np.median(times[1:]))
    return n / dt_med, times[1:], n


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def _import_reference():
    """The unmodified reference package (softmpm, numba) installed by
    tools/install_reference.sh into baseline/_ref, or None.  Its off-path
    scikit-image import is stubbed; numba's cache goes to /tmp."""
    if not os.path.isdir(os.path.join(REF_DIR, "softmpm")):
        return None
    import types
    if "skimage" not in sys.modules:
        sk = types.ModuleType("skimage")
        sk.measure = types.ModuleType("skimage.measure")
        sys.modules["skimage"], sys.modules["skimage.measure"] = sk, sk.measure
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/softmpm_numba_cache")
    if REF_DIR not in sys.path:
        sys.path.append(REF_DIR)
    try:
        import softmpm
        return softmpm
    except Exception:
        return None


def numba_reference_rate(config, particles, seed, substeps, threads, warmup=1):
    """The reference's own CPU path -- softmpm.core.substep (numba kernels,
    kernels.py:161-534) with the per-substep pose_fn, as core.step runs it --
    on the same scene (positions, tool path), numba threads = `threads`.
    Returns (particle-substeps/s, per-substep seconds, n) or None."""
    ref = _import_reference()
    if ref is None:
        return None
    import numba
    numba.set_num_threads(max(1, min(threads, numba.config.NUMBA_NUM_THREADS)))
    st, mats, params, cols, pose_fn = build_scene(config, particles, seed)
    g = st.grid
    rst = ref.SimState(grid=ref.Grid(resolution=g.resolution, extent=g.extent), x=st.x.copy(), v=st.v.copy(),
                       F=st.F.copy(), C=st.C.copy(), mass=st.mass.copy(), vol0=st.vol0.copy(),
                       material_id=st.material_id.copy())
    rmats = [ref.Material(m.young_modulus, m.poisson_ratio, m.density) for m in mats]
    rparams = ref.SimParams(dt=params.dt)
    rcols = [ref.RigidCollider(id=c.id, shape=ref.Box(np.asarray(c.shape.half_extents)),
                               friction_mu=c.friction_mu) for c in cols]
    t = 0.0
    times = []
    for i in range(warmup + substeps):
        t0 = time.perf_counter()
        if rcols:
            pose_fn(rcols, t)
        ref.core.substep(rst, rmats, rparams, rcols)
        if i >= warmup:
            times.append(time.perf_counter() - t0)
        t += params.dt
    n = st.particle_count
    return n / float(np.median(times)), times, n


def scene_workload(config, n, res, ncols):
    return (f"{config}: {n} particles/GPU, {res}^3 grid, {ncols} tool(s)"
            + (" pressing 3 cm at 0.5 m/s then holding" if config == "c3" else "")
            + (" (settling under gravity, dt 1e-4, re-binned once per step)" if config == "c5" else "")
            + ", 25 substeps per step")


def run_reference(args, rank, world):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    if args.config in ("c1", "c3") and _import_reference() is not None:
        return run_reference_numba(args, world, threads)
    from oracle import oracle as O
    O.set_threads(threads)
    import paper_2402_01181_b200 as sm
    st, mats, params, cols, pose_fn = build_scene(args.config, args.particles, 1)
    g = st.grid
    op = O.OracleParams(res=g.resolution, dx=g.dx, theta=0.5 * g.dx, chunks=8)
    osim = O.OracleSim(op, st.x, st.v, st.F, st.C, st.mass, st.vol0, st.material_id, mats[0].mu,
                       mats[0].lam)
    n = st.particle_count
    t = 0.0
    per = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        if cols:
            pose_fn(cols, t)
        osim.substep(sm.pack_colliders(cols) if cols else None)
        el = time.perf_counter() - t0
        t += params.dt
        if i >= args.warmup:
            per.append(el)
    tot = sum(per)
    value = n * len(per) / tot
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * tot / len(per),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": scene_workload(args.config, n, g.resolution[0], len(cols)),
                   "particles_per_gpu": n, "grid": list(g.resolution),
                   "substeps_per_step": params.substeps_per_frame,
                   "parallelism": f"CPU, {threads} threads (each timed step is one substep of the frame)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"each step = 1 substep of the full {args.config} scene "
                                   f"(O1 fp64 C restatement of kernels.py, 8 chunks, OpenMP)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def run_reference_numba(args, world, threads):
    """Reference arm on the reference's own code: softmpm.core.substep (numba,
    all host threads) from baseline/_ref, one substep of the full scene per
    timed step (JIT compile inside the warm-up steps)."""
    rate, times, n = numba_reference_rate(args.config, args.particles, 1, args.steps, threads,
                                          warmup=max(1, args.warmup))
    st, _, params, cols, _ = build_scene(args.config, args.particles, 1)
    g = st.grid
    tot = float(sum(times))
    value = n * len(times) / tot
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * tot / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": scene_workload(args.config, n, g.resolution[0], len(cols)),
                   "particles_per_gpu": n, "grid": list(g.resolution),
                   "substeps_per_step": params.substeps_per_frame,
                   "parallelism": f"CPU, {threads} numba threads (each timed step is one substep of the frame)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"each step = 1 substep of the full {args.config} scene: the unmodified "
                                   f"reference softmpm.core.substep (numba, baseline/_ref) with its pose_fn"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def run_ours(args, rank, world, local_rank):
    import paper_2402_01181_b200 as sm
    from paper_2402_01181_b200 import _lib
    import torch

    torch.cuda.set_device(local_rank)
    dist = world > 1
    if dist:
        import torch.distributed as tdist
    if args.config == "c5" and world > 1:
        return run_slab(args, rank, world, local_rank)
    if args.config == "c4":
        from paper_2402_01181_b200 import scenes
        from paper_2402_01181_b200.batch import shard
        env_ids = list(shard(args.envs, world, rank))
        batch, mats, params, _ = scenes.c4_envs(count=args.particles or 30_000, env_ids=env_ids)
        st = batch.state
        st.device = local_rank
        cols = batch._proxies
        nsub = params.substeps_per_frame
        traj = scenes.c4_trajectory()

        def c4_poses(t0):
            E = batch.n_envs
            R = np.broadcast_to(np.eye(3), (nsub, E, 1, 3, 3)).copy()
            T = np.zeros((nsub, E, 1, 3))
            lv = np.zeros((nsub, E, 1, 3))
            t = t0
            for s in range(nsub):  # every environment follows the same tool path
                poses, _ = sm.pose_at(traj, t)
                T[s, :, 0] = poses[0][0]
                lv[s, :, 0] = poses[0][2]
                t += params.dt
            return {"R": R, "T": T, "lv": lv}

        def rows_for(t0):
            return batch.pose_rows(c4_poses(t0))

        def warm():
            batch.step(mats, params, poses=c4_poses(batch.time))

        workload = (f"c4: {batch.n_envs} environments/GPU x {args.particles or 30_000} particles "
                    f"(64^3 each, tiles {batch.tiles}), box tool each, 25 substeps per step")
    else:
        st, mats, params, cols, pose_fn = build_scene(args.config, args.particles, 1 + rank)
        st.device = local_rank
        batch = None

        def rows_for(t0):
            return pose_rows(st, cols, params, pose_fn, t0)

        def warm():
            sm.step(st, mats, params, cols, pose_fn)

        workload = scene_workload(args.config, st.particle_count, st.grid.resolution[0], len(cols))
    if args.config == "c5":
        # scenes.c5 re-bins every 5 substeps: across slab ranks the ghost
        # layers must cover one stretch's drift (slab.py).  One GPU holding the
        # whole volume has no such bound -- the tile margins absorb the drift
        # and off-tile particles take the exact global path -- so it re-bins
        # once per frame like the other configs.
        params.rebin_interval = params.substeps_per_frame
    if args.rebin:
        params.rebin_interval = args.rebin
    n = st.particle_count
    nsub = params.substeps_per_frame
    L = _lib.lib()

    # warm-up through the public API (creates the context, uploads, captures graphs)
    for _ in range(args.warmup):
        warm()
    ctx = st._ctx
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=f"cuda:{local_rank}")

    def frame(rows=None):
        t0 = batch.time if batch is not None else st.time
        if cols:
            st._upload_pose_rows(*(rows if rows is not None else rows_for(t0)))
        inv = ctypes.c_int64(0)
        ms = ctypes.c_double(0.0)
        ctx.call("mpm_substeps", nsub, int(bool(cols)), ctypes.byref(inv), ctypes.byref(ms))
        for _ in range(nsub):
            if batch is not None:
                batch.time += params.dt
            else:
                st.time += params.dt
        st._device_wrote(("x", "v", "F", "C"))
        return ms.value

    # ---- device-resident timed region ------------------------------------
    # (no per-kernel event nodes here: they cost ~15% of a frame; the kernel
    # breakdown comes from a second pass below)
    L.mpm_set_timing(ctx.h, 0)
    launches0 = ctx.launches
    dev_ms = 0.0
    if dist:
        tdist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        wall0 = time.perf_counter()
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            dev_ms += frame()
        torch.cuda.synchronize()
        wall = time.perf_counter() - wall0
    if dist:
        tdist.barrier()
    launches = ctx.launches - launches0
    # ---- kernel breakdown: same frames with a CUDA event pair around every
    # kernel (event-record nodes inside the graph, on the launching stream)
    prof_steps = min(args.steps, 10)
    L.mpm_set_timing(ctx.h, 1)
    flush.zero_()
    frame()  # captures the timing variant of the graph
    L.mpm_set_timing(ctx.h, 1)  # reset the accumulators
    prof_ms = 0.0
    torch.cuda.synchronize()
    for _ in range(prof_steps):
        flush.zero_()
        torch.cuda.synchronize()
        prof_ms += frame()
    torch.cuda.synchronize()
    tbuf = (ctypes.c_double * 16)()
    L.mpm_get_timing(ctx.h, tbuf)
    L.mpm_set_timing(ctx.h, 0)
    a_ms, a_n = tbuf[0], max(tbuf[1], 1.0)
    grid_ms, grid_n = tbuf[2], max(tbuf[3], 1.0)
    rebin_ms, g2p_ms = tbuf[4], tbuf[6]
    b_ms, b_n = tbuf[10], max(tbuf[11], 1.0)
    f_ms, f_n = tbuf[12], max(tbuf[13], 1.0)
    m_ms, m_n = tbuf[14], max(tbuf[15], 1.0)
    # dominant kernel (largest share of the timed region) for the roofline line;
    # n = launches, or substeps for the cooperative substeps_kernel
    dom, fused_ms, fused_n = max(
        [("substeps_kernel (cooperative, per substep: fused G2P+advect+F update+stress+P2G phase, "
          "grid barrier, grid-op phase; time per substep)", m_ms, m_n),
         ("fused_kernel (G2P+advect+F update+stress+P2G, 1 launch = 1 substep)", f_ms, f_n),
         ("g2p_stress_kernel (G2P+advect+F update+stress, 1 launch = 1 substep)", a_ms, a_n),
         ("p2g_tile_kernel (P2G scatter, 1 launch = 1 substep)", b_ms, b_n)], key=lambda t: t[1])
    t_dev = dev_ms / 1000.0
    if dist:
        tt = torch.tensor([t_dev], device=f"cuda:{local_rank}", dtype=torch.float64)
        tdist.all_reduce(tt, op=tdist.ReduceOp.MAX)
        t_dev = float(tt.item())
    total_units = n * world * nsub * args.steps
    value = total_units / t_dev

    # ---- e2e through the C-ABI with host buffers ---------------------------
    e2e_steps = max(2, args.steps // 2)
    host = {}
    sizes = {"x": 3, "v": 3, "F": 9, "C": 9}
    ptrs = []
    for k, w in sizes.items():
        nbytes = n * w * 8
        p = L.mpm_host_alloc(nbytes)
        if not p:
            host[k] = np.empty(n * w)
        else:
            ptrs.append(p)
            host[k] = np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(ctypes.c_double)),
                                            shape=(n * w,))
    ctx.call("mpm_download_particles", ctypes.c_uint32(15), *[_lib.ptr(host[k]) for k in sizes])
    h2d = d2h = n * 24 * 8
    if dist:
        tdist.barrier()
    torch.cuda.synchronize()
    e0 = time.perf_counter()
    import threading
    for _ in range(e2e_steps):
        # as core.step does: the field upload on a worker thread (the copy
        # releases the GIL) while this thread builds the frame's pose table
        up = threading.Thread(target=ctx.call, args=("mpm_upload_fields", ctypes.c_uint32(15),
                                                     *[_lib.ptr(host[k]) for k in sizes]))
        up.start()
        rows = rows_for(batch.time if batch is not None else st.time) if cols else None
        up.join()
        frame(rows)
        ctx.call("mpm_download_particles", ctypes.c_uint32(15), *[_lib.ptr(host[k]) for k in sizes])
    torch.cuda.synchronize()
    t_e2e = time.perf_counter() - e0
    if dist:
        tt = torch.tensor([t_e2e], device=f"cuda:{local_rank}", dtype=torch.float64)
        tdist.all_reduce(tt, op=tdist.ReduceOp.MAX)
        t_e2e = float(tt.item())
    e2e_value = n * world * nsub * e2e_steps / t_e2e
    for p in ptrs:
        L.mpm_host_free(p)
    assert not st.has_nan(), "simulation produced NaN"

    if rank != 0:
        return None
    peak, peak_src = _peaks()
    traffic = _ncu_traffic(dom.split(" ")[0], args.config)
    avg_fused_s = fused_ms / fused_n / 1000.0
    achieved = BYTES_PER_PARTICLE_SUBSTEP * n / avg_fused_s / 1e9
    substep_s = t_dev / (args.steps * nsub)
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000.0 * t_dev / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp32",
        "data": "synthetic",
        "config": {"workload": workload, "particles_per_gpu": n, "grid": list(st.grid.resolution),
                   "substeps_per_step": nsub, "parallelism": (f"environment shards x{world}" if args.config == "c4" else f"replicas x{world}"),
                   "l2": "flushed between steps (512 MiB memset)",
                   "wall_s_timed": wall},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic[0] if traffic else None,
                     "traffic_source": (f"dram__bytes_read.sum + dram__bytes_write.sum per launch, "
                                        f"{traffic[1]} (cold-cache ncu replay)") if traffic else None,
                     "traffic_warm": traffic[2] if traffic else None,
                     "kernel": dom,
                     "bytes_per_launch": BYTES_PER_PARTICLE_SUBSTEP * n,
                     "mean_launch_ms": 1000.0 * avg_fused_s, "peak_source": peak_src,
                     "substep_frac": (BYTES_PER_PARTICLE_SUBSTEP * n / substep_s / 1e9) / peak,
                     "peak_nominal": NOMINAL_HBM_GBS, "frac_nominal": achieved / NOMINAL_HBM_GBS,
                     "grid_bytes_per_launch": GRID_BYTES_PER_NODE * 64 * tbuf[8],
                     "grid_bytes_note": "SURVEY 8d grid term, 56 B x nodes of the active bricks "
                                        "(brick-granular: includes massless nodes of active bricks)",
                     "share_of_step": fused_ms / max(prof_ms, 1e-9),
                     "timing": f"mean_launch_ms from a {prof_steps}-frame pass with per-kernel CUDA events "
                               "(value/ms_per_step from the pass without them)"},
        "kernel_ms": {"substeps_kernel_per_substep": m_ms / m_n, "substeps_kernel_substeps": tbuf[15],
                      "fused_mean": f_ms / f_n, "fused_launches": tbuf[13],
                      "g2p_stress_mean": a_ms / a_n, "p2g_tile_mean": b_ms / b_n,
                      "grid_op_mean": grid_ms / grid_n,
                      "rebin_total": rebin_ms, "g2p_total": g2p_ms, "device_total": prof_ms,
                      "frames": prof_steps,
                      "active_bricks": tbuf[8], "work_items": tbuf[9]},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "steps": e2e_steps},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if world == 1 and not args.no_cpu_baseline and args.config != "c5":
        threads = os.cpu_count() or 1
        rate, times, nn = cpu_oracle_rate(args.config, args.particles, 1, args.cpu_substeps, threads)
        rate1, times1, _ = cpu_oracle_rate(args.config, args.particles, 1, 1, 1)
        env_note = (" (one environment: the CPU runs environments one after another, so its "
                    "particle-substeps/s is the batch's)") if args.config == "c4" else ""
        out["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
                               "sample": f"{args.cpu_substeps} substeps (after 1 warm-up) of the "
                                         f"same {args.config} scene, {nn} particles{env_note}, O1 fp64 C "
                                         f"restatement of kernels.py, 8 chunks, OpenMP",
                               "substep_s": times,
                               "value_1thread": rate1, "substep_s_1thread": times1}
        if args.config in ("c1", "c3"):  # box tools / none (the C2 SDF jaws stay on the port)
            try:
                r = numba_reference_rate(args.config, args.particles, 1, args.cpu_substeps, threads)
            except Exception as e:  # the port above stays the baseline
                r = None
                out["cpu_baseline"]["reference_numba_error"] = str(e)[:200]
            if r is not None:
                out["cpu_baseline"]["reference_numba"] = {
                    "value": r[0], "unit": UNIT, "cores": threads, "kind": "reference",
                    "substep_s": r[1],
                    "sample": f"{args.cpu_substeps} substeps (after 1 warm-up incl. JIT) of the same scene through "
                              f"the unmodified reference softmpm.core.substep (numba, baseline/_ref)"}
    return out


def run_slab(args, rank, world, local_rank, particles=None):
    """Config 5 across ranks: this rank's x-slab window of the 64 M-particle
    volume (slab.rank_window: balanced cuts), halos through peer memory (IPC
    over NVLink; the pack kernels write into the neighbour's buffers, streams
    ordered by device counters) or NCCL, migration once per 5-substep stretch.
    Strong scaling: the scene is fixed, N GPUs share it.  Returns the JSON
    object on rank 0 (None elsewhere)."""
    import torch
    import torch.distributed as tdist
    from paper_2402_01181_b200 import scenes, slab
    from paper_2402_01181_b200.dist import max_over_ranks, sum_over_ranks
    count = particles or args.particles or 64_000_000
    g, spawn, mats, params = scenes.c5_spawn(count=count)
    win = slab.rank_window(g, spawn.positions, spawn.rest_volume_per_particle, mats[0].density, world, rank,
                           ghost_bricks=2, device=local_rank)
    del spawn
    if args.exchange == "ipc":
        ex = slab.IpcExchange(win, rank, world, device=f"cuda:{local_rank}")
    else:
        ex = slab.TorchExchange(win, rank, world, device=f"cuda:{local_rank}")
    for _ in range(args.warmup):
        slab.step_distributed(win, ex, mats, params)
    n_local = int(_lib_count(win))
    launches0 = win.state._ctx.launches
    tdist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        t0 = time.perf_counter()
        for _ in range(args.steps):
            slab.step_distributed(win, ex, mats, params)
        torch.cuda.synchronize()
        tdist.barrier()
        el_local = time.perf_counter() - t0
    el = max_over_ranks(el_local, f"cuda:{local_rank}")
    n_total = sum_over_ranks(n_local, f"cuda:{local_rank}")
    launches = sum_over_ranks(win.state._ctx.launches - launches0, f"cuda:{local_rank}")
    assert not getattr(win, "last_nan", False), "slab run produced NaN"
    if rank != 0:
        return None
    value = n_total * params.substeps_per_frame * args.steps / el
    peak, peak_src = _peaks()
    achieved = BYTES_PER_PARTICLE_SUBSTEP * value / world / 1e9
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000.0 * el / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
        "config": {"workload": f"c5: {int(n_total)} particles, {g.resolution[0]}^3 grid, x-slabs over "
                               f"{world} GPUs ({'peer-memory (IPC/NVLink) halo' if args.exchange == 'ipc' else 'NCCL halo'}"
                               f" + NCCL migration per 5-substep stretch, dt 1e-4), 25 substeps per step",
                   "particles_total": int(n_total), "grid": list(g.resolution),
                   "parallelism": f"slab x{world} (balanced x cuts)",
                   "timing": "wall clock between device-synchronised barriers around the timed frames "
                             "(migration syncs the host once per stretch), max over ranks"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": None, "peak_source": peak_src,
                     "kernel": "whole substep per GPU incl. halo exchange and migration (no per-kernel "
                               "timing on the slab path)"},
        "e2e": {"value": None, "unit": UNIT,
                "unavailable": "slab path keeps each window's particles on its device between frames; "
                               "per-rank host upload/readback is not part of this loop"},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }


def _lib_count(win):
    from paper_2402_01181_b200 import _lib
    return _lib.lib().mpm_particle_count(win.state._ctx.h)


def _respawn(args) -> int:
    """--gpus N > 1 without a launcher: re-run this command under torchrun
    (one rank per GPU, 127.0.0.1 rendezvous) and return its exit code."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--envs", type=int, default=1024, help="c4: environments over all ranks")
    ap.add_argument("--rebin", type=int, default=None, help="override SimParams.rebin_interval")
    ap.add_argument("--particles", type=int, default=None)
    ap.add_argument("--slab-particles", type=int, default=None,
                    help="N > 1: particles of the C5 slab block run beside the main line "
                         "(default 64 M; 4 M with SOFTMPM_BENCH_SHARED_GPU; 0 = skip)")
    ap.add_argument("--exchange", default="ipc", choices=["ipc", "nccl"],
                    help="c5 over ranks: halo through peer memory (pack kernels write into the neighbour's "
                         "IPC-mapped buffers) or NCCL send/recv")
    ap.add_argument("--cpu-substeps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3 if args.impl == "ours" else args.warmup)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(_respawn(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but the launcher started {world} ranks")
    # plumbing check only (never a measurement): SOFTMPM_BENCH_SHARED_GPU=1 lets
    # several ranks share the visible GPUs over gloo, to exercise the N > 1 path
    # (barriers, max over ranks, sharding, the slab block) on a one-GPU box
    shared = os.environ.get("SOFTMPM_BENCH_SHARED_GPU") == "1"
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as tdist
        if shared:
            local_rank = local_rank % max(torch.cuda.device_count(), 1)
        elif torch.cuda.device_count() < world:
            sys.exit(f"bench.py: {world} ranks but {torch.cuda.device_count()} visible GPUs "
                     "(SOFTMPM_BENCH_SHARED_GPU=1 for a plumbing run)")
        torch.cuda.set_device(local_rank)
        if shared:
            tdist.init_process_group("gloo")
        else:
            tdist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
    try:
        out = run_ours(args, rank, world, local_rank)
        if world > 1 and args.config != "c5":
            # the north star's multi-GPU split beside the replica line: C5's
            # 64 M-particle volume slab-decomposed over the same N GPUs
            sp = args.slab_particles if args.slab_particles is not None else (4_000_000 if shared else 64_000_000)
            if sp > 0:
                blk = run_slab(args, rank, world, local_rank, particles=sp)
                if rank == 0:
                    if shared:
                        blk["note"] = "ranks share one GPU (plumbing run, not a measurement)"
                    out["slab"] = blk
        if rank == 0 and out is not None:
            print(json.dumps(out), flush=True)
    finally:
        if world > 1:
            import torch.distributed as tdist
            tdist.destroy_process_group()


if __name__ == "__main__":
    main()
