// slab_halo.cuh -- slab decomposition: ghost-brick halo records, peer-memory exchange, migration (sm_100a).
// Part of the kernel set included by kernels.cuh (namespace mpm).
#pragma once

namespace mpm {

// ---------------------------------------------------------------------------
// slab decomposition (config 5): sparse ghost-brick exchange + migration
// ---------------------------------------------------------------------------

// Pack the active bricks of one ghost slab (side 0: local x-bricks [0, gb),
// side 1: [nb0 - gb, nb0)) as records {global brick id, 64 x float4 gm}.
// rec_ids/rec_data: capacity-sized buffers; *count receives the record count.
__global__ void halo_pack_kernel(Params p, int side, int gb, int* rec_ids, float4* rec_data, int* count) {
  const int nitems = *p.active_count;
  const int lane = threadIdx.x & 31;
  for (int it = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); it < nitems;
       it += gridDim.x * (blockDim.x >> 5)) {
    const int b = p.active_list[it];
    const int bi = b / (p.nb[1] * p.nb[2]);
    const bool ghost = side == 0 ? bi < gb : bi >= p.nb[0] - gb;
    if (!ghost) continue;
    int slot = 0;
    if (lane == 0) slot = atomicAdd(count, 1);
    slot = __shfl_sync(0xffffffffu, slot, 0);
    if (lane == 0) {
      const int rem = b - bi * (p.nb[1] * p.nb[2]);
      rec_ids[slot] = (bi + (p.goff[0] >> BRICK_SHIFT)) * (p.nb[1] * p.nb[2]) + rem;  // global brick id
    }
    rec_data[(long long)slot * 64 + lane] = p.gm[((long long)b << 6) + lane];
    rec_data[(long long)slot * 64 + lane + 32] = p.gm[((long long)b << 6) + lane + 32];
  }
}

// Add received ghost records into the owned bricks (global -> local brick id)
// and mark them active; remembers the local ids for the velocity reply.
__global__ void halo_unpack_add_kernel(Params p, const int* rec_ids, const float4* rec_data, int n, int* local_ids) {
  const int lane = threadIdx.x & 31;
  const int per_slab = p.nb[1] * p.nb[2];
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += gridDim.x * (blockDim.x >> 5)) {
    const int gbid = rec_ids[r];
    const int b = gbid - (p.goff[0] >> BRICK_SHIFT) * per_slab;
    if (lane == 0) local_ids[r] = b;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const long long idx = ((long long)b << 6) + lane + 32 * h;
      const float4 a = rec_data[(long long)r * 64 + lane + 32 * h];
      float4 g = p.gm[idx];
      g.x += a.x;
      g.y += a.y;
      g.z += a.z;
      g.w += a.w;
      p.gm[idx] = g;
    }
    if (lane == 0) mark_brick(p, (long long)b << 6);
  }
}

// Velocity reply: gv of the bricks received from a side, in receive order.
__global__ void halo_pack_vel_kernel(Params p, const int* local_ids, int n, float4* rec_data) {
  const int lane = threadIdx.x & 31;
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += gridDim.x * (blockDim.x >> 5)) {
    const long long b = local_ids[r];
    rec_data[(long long)r * 64 + lane] = p.gv[(b << 6) + lane];
    rec_data[(long long)r * 64 + lane + 32] = p.gv[(b << 6) + lane + 32];
  }
}

// Write the owner's velocities into our ghost bricks (ids = our packed global ids).
__global__ void halo_unpack_vel_kernel(Params p, const int* rec_ids, const float4* rec_data, int n) {
  const int lane = threadIdx.x & 31;
  const int per_slab = p.nb[1] * p.nb[2];
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += gridDim.x * (blockDim.x >> 5)) {
    const long long b = rec_ids[r] - (p.goff[0] >> BRICK_SHIFT) * per_slab;
    p.gv[(b << 6) + lane] = rec_data[(long long)r * 64 + lane];
    p.gv[(b << 6) + lane + 32] = rec_data[(long long)r * 64 + lane + 32];
  }
}

// ---- peer-memory halo exchange (CUDA IPC / NVLink P2P) ------------------
// The pack kernels write straight into the NEIGHBOUR's receive buffers
// (mapped with cudaIpcOpenMemHandle; P2P stores and atomics over NVLink
// between GPUs), so packing and the transfer are one kernel; record counts
// live on the device and never visit the host.

// Ghost bricks of one side -> the neighbour's receive buffers; slot from the
// neighbour's counter, the global ids also kept locally for the velocity reply.
__global__ void ipc_pack_kernel(Params p, int side, int gb, int* peer_ids, float4* peer_data, int* peer_count,
                                int* my_ids, int* my_sent) {
  const int nitems = *p.active_count;
  const int lane = threadIdx.x & 31;
  for (int it = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); it < nitems;
       it += gridDim.x * (blockDim.x >> 5)) {
    const int b = p.active_list[it];
    const int bi = b / (p.nb[1] * p.nb[2]);
    const bool ghost = side == 0 ? bi < gb : bi >= p.nb[0] - gb;
    if (!ghost) continue;
    int slot = 0;
    if (lane == 0) slot = atomicAdd(peer_count, 1);
    slot = __shfl_sync(0xffffffffu, slot, 0);
    if (lane == 0) {
      const int rem = b - bi * (p.nb[1] * p.nb[2]);
      const int gbid = (bi + (p.goff[0] >> BRICK_SHIFT)) * (p.nb[1] * p.nb[2]) + rem;
      peer_ids[slot] = gbid;
      my_ids[slot] = gbid;
      atomicMax(my_sent, slot + 1);
    }
    peer_data[(long long)slot * 64 + lane] = p.gm[((long long)b << 6) + lane];
    peer_data[(long long)slot * 64 + lane + 32] = p.gm[((long long)b << 6) + lane + 32];
  }
}

__global__ void ipc_unpack_add_kernel(Params p, const int* rec_ids, const float4* rec_data, const int* count,
                                      int* local_ids) {
  const int n = *count;
  const int lane = threadIdx.x & 31;
  const int per_slab = p.nb[1] * p.nb[2];
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += gridDim.x * (blockDim.x >> 5)) {
    const int b = rec_ids[r] - (p.goff[0] >> BRICK_SHIFT) * per_slab;
    if (lane == 0) local_ids[r] = b;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const long long idx = ((long long)b << 6) + lane + 32 * h;
      const float4 a = rec_data[(long long)r * 64 + lane + 32 * h];
      float4 g = p.gm[idx];
      g.x += a.x;
      g.y += a.y;
      g.z += a.z;
      g.w += a.w;
      p.gm[idx] = g;
    }
    if (lane == 0) mark_brick(p, (long long)b << 6);
  }
}

// Velocity reply straight into the neighbour's velocity receive buffer.
__global__ void ipc_pack_vel_kernel(Params p, const int* local_ids, const int* n_recv, float4* peer_vdata) {
  const int n = *n_recv;
  const int lane = threadIdx.x & 31;
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += gridDim.x * (blockDim.x >> 5)) {
    const long long b = local_ids[r];
    peer_vdata[(long long)r * 64 + lane] = p.gv[(b << 6) + lane];
    peer_vdata[(long long)r * 64 + lane + 32] = p.gv[(b << 6) + lane + 32];
  }
}

__global__ void ipc_unpack_vel_kernel(Params p, const int* my_ids, const int* my_sent, const float4* vdata) {
  const int n = *my_sent;
  const int lane = threadIdx.x & 31;
  const int per_slab = p.nb[1] * p.nb[2];
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += gridDim.x * (blockDim.x >> 5)) {
    const long long b = my_ids[r] - (p.goff[0] >> BRICK_SHIFT) * per_slab;
    p.gv[(b << 6) + lane] = vdata[(long long)r * 64 + lane];
    p.gv[(b << 6) + lane + 32] = vdata[(long long)r * 64 + lane + 32];
  }
}

// Migration: flag = 0 keep, 1 leaves to the low neighbour, 2 to the high one
// (global base cell x outside [own_lo, own_hi)).
__global__ void migrant_flag_kernel(Params p, int own_lo, int own_hi, int* flag) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= p.n) return;
  const float g = (ldf(p, FX, i) + p.goffx[0]) * p.inv_dx;
  const int b = (int)floorf(g - 0.5f);
  flag[i] = b < own_lo ? 1 : (b >= own_hi ? 2 : 0);
}

// Migrant rows (flag 1: low neighbour, 2: high neighbour) packed per side:
// field q of row d at out[q * m + d], m = that side's migrant count (one
// contiguous ROWS x m block per neighbour), d = the migrant's rank among its
// side's migrants (exclusive scan).  The kept particles stay where they are:
// their slots and the migrants' holes are compacted by the next re-binning
// (bin_key_kernel skips flagged slots), so a stretch permutes the particle
// state once, not twice.
__global__ void migrant_rows_kernel(Params p, const int* flag, const int* pos_lo, const int* pos_hi, float* out_lo,
                                    float* out_hi, long long m_lo, long long m_hi) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= p.n) return;
  const int f = flag[i];
  if (f == 0) return;
  float* out = f == 1 ? out_lo : out_hi;
  const long long d = f == 1 ? pos_lo[i] : pos_hi[i];
  const long long out_cap = f == 1 ? m_lo : m_hi;
#pragma unroll
  for (int q = 0; q < NF; ++q) out[q * out_cap + d] = ldf(p, q, i);
  out[NF * out_cap + d] = __int_as_float(p.mat[i]);
  out[(NF + 1) * out_cap + d] = __int_as_float(p.orig[i]);
}

__global__ void flag_class_kernel(const int* flag, int cls, int* out, long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) out[i] = flag[i] == cls;
}

// Append m migrant rows (row layout of migrant_scatter_kernel) at slot n0,
// shifting x by dxs (source window offset - ours, in metres).
__global__ void append_rows_kernel(Params p, const float* rows, long long m, long long rows_cap, long long n0,
                                   float dxs) {
  const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (r >= m) return;
  const long long d = n0 + r;
#pragma unroll
  for (int q = 0; q < NF; ++q) {
    float v = rows[q * rows_cap + r];
    if (q == FX) v += dxs;
    p.P[q * p.cap + d] = v;
  }
  p.mat[d] = __float_as_int(rows[NF * rows_cap + r]);
  p.orig[d] = __float_as_int(rows[(NF + 1) * rows_cap + r]);
}

__global__ void set_ids_kernel(Params p, const int* ids) {
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s < p.n) p.orig[s] = ids[p.orig[s]];
}

// x (global), v, F, C in device order (slab windows: rows are identified by id).
__global__ void download_rows_kernel(Params p, double* x, double* v, double* F, double* C) {
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s >= p.n) return;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    x[3 * s + a] = (double)ldf(p, FX + a, s) + (double)p.goffx[a];
    v[3 * s + a] = ldf(p, FV + a, s);
  }
#pragma unroll
  for (int q = 0; q < 9; ++q) {
    F[9 * s + q] = ldf(p, FF + q, s);
    C[9 * s + q] = ldf(p, FC + q, s);
  }
}

__global__ void download_ids_kernel(Params p, int* ids, double* x) {
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s >= p.n) return;
  ids[s] = p.orig[s];
#pragma unroll
  for (int a = 0; a < 3; ++a) x[3 * s + a] = (double)ldf(p, FX + a, s) + (double)p.goffx[a];
}

}  // namespace mpm
