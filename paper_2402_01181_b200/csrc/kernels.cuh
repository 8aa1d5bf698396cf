// kernels.cuh -- the B200 MLS-MPM substep kernels (sm_100a).
//
// Fast path, per substep:
//   fused_kernel<G2P,P2G>  one CTA per particle-bin work item: G2P gather from
//                          gv (L1/L2-resident blocked grid) -> advect ->
//                          F update -> Neo-Hookean stress -> P2G scatter into a
//                          shared-memory tile covering the bin + halo, flushed
//                          once per work item with REDG.F32x4 into gm.
//   grid_op_kernel         active bricks only: momentum -> velocity, gravity,
//                          lazy collider distance + contact, domain boundary;
//                          clears gm for the next P2G.
//   g2p_kernel             final G2P of a frame (writes v, C, x).
// Deterministic path: cell-sorted permutation + det_payload_kernel +
// det_gather_kernel (node-owner gather, fixed order, no atomics).
#pragma once
#include "collide.cuh"
#include "common.cuh"

namespace mpm {

__device__ __forceinline__ void mark_brick(const Params& p, long long idx) {
  int b = (int)(idx >> 6);
  if (*((volatile int*)p.brick_flag + b) == 0) {
    if (atomicExch(&p.brick_flag[b], 1) == 0) {
      int s = atomicAdd(p.active_count, 1);
      p.active_list[s] = b;
    }
  }
}

__device__ __forceinline__ void warp_count_add(unsigned long long* dst, unsigned v) {
  unsigned s = __reduce_add_sync(0xffffffffu, v);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(dst, (unsigned long long)s);
}

// Per-axis node offsets into the blocked layout for a 3-node stencil.
__device__ __forceinline__ void axis_offsets(int b, int stride_brick, int stride_local, int o[3]) {
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    int c = b + q;
    o[q] = (c >> BRICK_SHIFT) * stride_brick + (c & 3) * stride_local;
  }
}

// G2P gather at x (kernels.py:451-516): v = sum w g, C = 4/dx^2 sum w g dp^T.
__device__ __forceinline__ void g2p_gather(const Params& p, const float x[3], float v[3],
                                           float C[9]) {
  int b[3];
  float f[3], w[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a) stencil(x[a], p.inv_dx, p.res[a], b[a], f[a], w[a]);
  int ox[3], oy[3], oz[3];
  axis_offsets(b[0], p.nb[1] * p.nb[2] * 64, 16, ox);
  axis_offsets(b[1], p.nb[2] * 64, 4, oy);
  axis_offsets(b[2], 64, 1, oz);
  float S[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) S[q] = 0.f;
  v[0] = v[1] = v[2] = 0.f;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    float di = (float)i - f[0];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      float wij = w[0][i] * w[1][j];
      float dj = (float)j - f[1];
      int oij = ox[i] + oy[j];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        float wt = wij * w[2][k];
        float dk = (float)k - f[2];
        float4 g = __ldg(p.gv + (oij + oz[k]));
        float wg[3] = {wt * g.x, wt * g.y, wt * g.z};
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          v[a] += wg[a];
          S[3 * a] += wg[a] * di;
          S[3 * a + 1] += wg[a] * dj;
          S[3 * a + 2] += wg[a] * dk;
        }
      }
    }
  }
  float cc = 4.0f * p.inv_dx;  // coef * dx = 4/dx
#pragma unroll
  for (int q = 0; q < 9; ++q) C[q] = S[q] * cc;
}

__device__ __forceinline__ void advect(const Params& p, float x[3], const float v[3]) {
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    float q = x[a] + p.dt * v[a];
    q = q < p.lo ? p.lo : q;
    q = q > p.hi[a] ? p.hi[a] : q;
    x[a] = q;
  }
}

// Scatter one particle's (momentum, mass) stencil.  TILE_MODE: into the smem
// tile with origin `org`; else straight into gm with REDG.F32x4.
template <bool TILE_MODE>
__device__ __forceinline__ void p2g_scatter(const Params& p, float* tile, const int org[3],
                                            const int b[3], const float f[3], const float w[3][3],
                                            float m, const float mv[3], const float A[9]) {
  float ax[3][3], ay[3][3], az[3][3];  // A[:,axis] * dp(axis, offset)
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    float d0 = ((float)q - f[0]) * p.dx, d1 = ((float)q - f[1]) * p.dx, d2 = ((float)q - f[2]) * p.dx;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      ax[q][r] = A[3 * r] * d0;
      ay[q][r] = A[3 * r + 1] * d1;
      az[q][r] = A[3 * r + 2] * d2;
    }
  }
  int ox[3], oy[3], oz[3];
  if (TILE_MODE) {
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      ox[q] = (b[0] - org[0] + q) * TILE * TILE;
      oy[q] = (b[1] - org[1] + q) * TILE;
      oz[q] = (b[2] - org[2] + q);
    }
  } else {
    axis_offsets(b[0], p.nb[1] * p.nb[2] * 64, 16, ox);
    axis_offsets(b[1], p.nb[2] * 64, 4, oy);
    axis_offsets(b[2], 64, 1, oz);
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      float wij = w[0][i] * w[1][j];
      float bij[3];
#pragma unroll
      for (int r = 0; r < 3; ++r) bij[r] = mv[r] + ax[i][r] + ay[j][r];
      int oij = ox[i] + oy[j];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        float wt = wij * w[2][k];
        int idx = oij + oz[k];
        float4 c = make_float4(wt * (bij[0] + az[k][0]), wt * (bij[1] + az[k][1]),
                               wt * (bij[2] + az[k][2]), wt * m);
        if (TILE_MODE) {
          float* t = tile + 4 * idx;
          atomicAdd(t, c.x);
          atomicAdd(t + 1, c.y);
          atomicAdd(t + 2, c.z);
          atomicAdd(t + 3, c.w);
        } else {
          atomicAdd(p.gm + idx, c);
          mark_brick(p, idx);
        }
      }
    }
  }
}

template <bool G2P, bool P2G>
__global__ void __launch_bounds__(256) fused_kernel(Params p) {
  extern __shared__ float4 tile4[];
  float* tile = reinterpret_cast<float*>(tile4);
  const int nwork = *p.nwork;
  unsigned inverted = 0;
  for (int wi = blockIdx.x; wi < nwork; wi += gridDim.x) {
    const int4 item = p.work[wi];
    int bin = item.x;
    int bz = bin % p.nbin[2];
    int by = (bin / p.nbin[2]) % p.nbin[1];
    int bx = bin / (p.nbin[1] * p.nbin[2]);
    const int org[3] = {bx * BIN - MARGIN, by * BIN - MARGIN, bz * BIN - MARGIN};
    if (P2G) {
      for (int t = threadIdx.x; t < TILE_NODES; t += blockDim.x) tile4[t] = make_float4(0.f, 0.f, 0.f, 0.f);
      __syncthreads();
    }
    for (int i = item.y + threadIdx.x; i < item.z; i += blockDim.x) {
      float x[3] = {ldf(p, FX, i), ldf(p, FX + 1, i), ldf(p, FX + 2, i)};
      float v[3], C[9];
      if (G2P) {
        g2p_gather(p, x, v, C);
        advect(p, x, v);
#pragma unroll
        for (int a = 0; a < 3; ++a) stf(p, FX + a, i, x[a]);
        if (!P2G) {
#pragma unroll
          for (int a = 0; a < 3; ++a) stf(p, FV + a, i, v[a]);
#pragma unroll
          for (int q = 0; q < 9; ++q) stf(p, FC + q, i, C[q]);
        }
      } else {
#pragma unroll
        for (int a = 0; a < 3; ++a) v[a] = ldf(p, FV + a, i);
#pragma unroll
        for (int q = 0; q < 9; ++q) C[q] = ldf(p, FC + q, i);
      }
      if (P2G) {
        float F[9], A[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) F[q] = ldf(p, FF + q, i);
        float m = ldf(p, FMASS, i), vol = ldf(p, FVOL, i);
        int mid = p.mat[i];
        float det = affine_update<false>(F, C, m, vol, __ldg(p.mu + mid), __ldg(p.lam + mid), p.dt,
                                         p.stress_coef, p.stress_form, A);
        inverted += det <= 0.0f;
#pragma unroll
        for (int q = 0; q < 9; ++q) stf(p, FF + q, i, F[q]);
        int b[3];
        float f[3], w[3][3];
#pragma unroll
        for (int a = 0; a < 3; ++a) stencil(x[a], p.inv_dx, p.res[a], b[a], f[a], w[a]);
        float mv[3] = {m * v[0], m * v[1], m * v[2]};
        bool inside = true;
#pragma unroll
        for (int a = 0; a < 3; ++a) inside &= (b[a] - org[a] >= 0) && (b[a] - org[a] <= TILE - 3);
        if (inside)
          p2g_scatter<true>(p, tile, org, b, f, w, m, mv, A);
        else
          p2g_scatter<false>(p, tile, org, b, f, w, m, mv, A);
      }
    }
    if (P2G) {
      __syncthreads();
      for (int t = threadIdx.x; t < TILE_NODES; t += blockDim.x) {
        float4 a = tile4[t];
        if (a.x == 0.f && a.y == 0.f && a.z == 0.f && a.w == 0.f) continue;
        int tz = t % TILE, ty = (t / TILE) % TILE, tx = t / (TILE * TILE);
        int gi = org[0] + tx, gj = org[1] + ty, gk = org[2] + tz;
        if (gi < 0 || gj < 0 || gk < 0 || gi >= p.res[0] || gj >= p.res[1] || gk >= p.res[2]) continue;
        long long idx = node_index(gi, gj, gk, p.nb[1], p.nb[2]);
        atomicAdd(p.gm + idx, a);
        mark_brick(p, idx);
      }
      __syncthreads();
    }
  }
  if (P2G) warp_count_add(p.inverted, inverted);
}

// Final G2P of a frame / stage g2p_advect: thread per particle.
__global__ void __launch_bounds__(256) g2p_kernel(Params p) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= p.n) return;
  float x[3] = {ldf(p, FX, i), ldf(p, FX + 1, i), ldf(p, FX + 2, i)};
  float v[3], C[9];
  g2p_gather(p, x, v, C);
  advect(p, x, v);
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    stf(p, FX + a, i, x[a]);
    stf(p, FV + a, i, v[a]);
  }
#pragma unroll
  for (int q = 0; q < 9; ++q) stf(p, FC + q, i, C[q]);
}

// Grid op (kernels.py:347-436) over active bricks (or all bricks when DENSE).
// 64 threads per brick.  Zero-mass nodes pass momentum through unchanged
// (kernels.py:364-365).  When `clear`, gm is zeroed for the next P2G.
template <bool DENSE>
__global__ void __launch_bounds__(256) grid_op_kernel(Params p, Colliders cs, int clear) {
  const long long nitems = DENSE ? (long long)p.nb[0] * p.nb[1] * p.nb[2] : (long long)*p.active_count;
  const int lane = threadIdx.x & 63;
  const int li = lane >> 4, lj = (lane >> 2) & 3, lk = lane & 3;
  const double cap = 2.0 * cs.theta;
  for (long long it = (long long)blockIdx.x * (blockDim.x >> 6) + (threadIdx.x >> 6); it < nitems;
       it += (long long)gridDim.x * (blockDim.x >> 6)) {
    long long b = DENSE ? it : (long long)p.active_list[it];
    int bi, bj, bk;
    brick_coords(b, p.nb, bi, bj, bk);
    int gi = bi * 4 + li, gj = bj * 4 + lj, gk = bk * 4 + lk;
    long long idx = (b << 6) | lane;
    float4 a = p.gm[idx];
    float4 out = a;
    if (a.w > 0.0f && gi < p.res[0] && gj < p.res[1] && gk < p.res[2]) {
      float inv_m = 1.0f / a.w;
      float v0 = a.x * inv_m + p.dt * p.gravity[0];
      float v1 = a.y * inv_m + p.dt * p.gravity[1];
      float v2 = a.z * inv_m + p.dt * p.gravity[2];
      if (cs.theta >= 0.0 && cs.count > 0) {
        double wx = (double)gi * p.dx64, wy = (double)gj * p.dx64, wz = (double)gk * p.dx64;
        double best;
        int ci = nearest_collider(cs, wx, wy, wz, cap, best);
        if (best < cs.theta && ci >= 0) {
          double vv[3] = {v0, v1, v2};
          resolve_contact(cs, ci, wx, wy, wz, vv);
          v0 = (float)vv[0];
          v1 = (float)vv[1];
          v2 = (float)vv[2];
        }
      }
      const int bw = p.bwidth;
      if (p.stick) {
        if (gi < bw || gi >= p.res[0] - bw || gj < bw || gj >= p.res[1] - bw || gk < bw ||
            gk >= p.res[2] - bw)
          v0 = v1 = v2 = 0.0f;
      } else {
        if (gi < bw && v0 < 0.0f) v0 = 0.0f;
        if (gi >= p.res[0] - bw && v0 > 0.0f) v0 = 0.0f;
        if (gj < bw && v1 < 0.0f) v1 = 0.0f;
        if (gj >= p.res[1] - bw && v1 > 0.0f) v1 = 0.0f;
        if (gk < bw && v2 < 0.0f) v2 = 0.0f;
        if (gk >= p.res[2] - bw && v2 > 0.0f) v2 = 0.0f;
      }
      out = make_float4(v0, v1, v2, a.w);
    }
    p.gv[idx] = out;
    if (clear) p.gm[idx] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (lane == 0) p.brick_flag[b] = 0;
  }
}

// Zero gm on the bricks of the active list (after a non-clearing grid op).
__global__ void clear_active_kernel(Params p) {
  const long long nitems = *p.active_count;
  for (long long it = (long long)blockIdx.x * (blockDim.x >> 6) + (threadIdx.x >> 6); it < nitems;
       it += (long long)gridDim.x * (blockDim.x >> 6)) {
    long long b = p.active_list[it];
    p.gm[(b << 6) | (threadIdx.x & 63)] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

__global__ void reset_counter_kernel(int* c, int* c2) {
  *c = 0;
  if (c2) *c2 = 0;
}

// ---------------------------------------------------------------------------
// binning (counting sort by 8^3-cell bin)
// ---------------------------------------------------------------------------

__global__ void bin_key_kernel(Params p, int* key, int* rank, int* bin_count) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= p.n) return;
  int c[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    float g = ldf(p, FX + a, i) * p.inv_dx;
    int bb = (int)floorf(g - 0.5f);
    c[a] = max(0, min(bb, p.res[a] - 3)) >> BIN_SHIFT;
  }
  int k = (c[0] * p.nbin[1] + c[1]) * p.nbin[2] + c[2];
  key[i] = k;
  rank[i] = atomicAdd(bin_count + k, 1);
}

__global__ void permute_kernel(const float* __restrict__ src, const int* __restrict__ src_mat,
                               const int* __restrict__ src_orig, float* __restrict__ dst,
                               int* __restrict__ dst_mat, int* __restrict__ dst_orig,
                               const int* __restrict__ key, const int* __restrict__ rank,
                               const int* __restrict__ start, long long n, long long cap) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  long long d = (long long)start[key[i]] + rank[i];
#pragma unroll
  for (int f = 0; f < NF; ++f) dst[f * cap + d] = src[f * cap + i];
  dst_mat[d] = src_mat[i];
  dst_orig[d] = src_orig[i];
}

__global__ void make_work_kernel(const int* bin_count, const int* bin_start, int nbins, int4* work,
                                 int* nwork) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nbins) return;
  int c = bin_count[b];
  if (!c) return;
  int items = (c + CHUNK - 1) / CHUNK;
  int base = atomicAdd(nwork, items);
  int s = bin_start[b];
  for (int t = 0; t < items; ++t)
    work[base + t] = make_int4(b, s + t * CHUNK, min(s + (t + 1) * CHUNK, s + c), 0);
}

// ---------------------------------------------------------------------------
// exclusive scan (3-phase; 512 threads x 8 items per block)
// ---------------------------------------------------------------------------
constexpr int SCAN_THREADS = 512, SCAN_ITEMS = 8, SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

__global__ void __launch_bounds__(SCAN_THREADS) scan_tile_kernel(const int* in, int* out, int* sums,
                                                                 long long n) {
  __shared__ int warp_tot[SCAN_THREADS / 32];
  long long base = (long long)blockIdx.x * SCAN_TILE + (long long)threadIdx.x * SCAN_ITEMS;
  int v[SCAN_ITEMS];
  int run = 0;
#pragma unroll
  for (int q = 0; q < SCAN_ITEMS; ++q) {
    v[q] = base + q < n ? in[base + q] : 0;
    int t = v[q];
    v[q] = run;
    run += t;
  }
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int incl = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) warp_tot[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    int t = lane < SCAN_THREADS / 32 ? warp_tot[lane] : 0;
    int ti = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, ti, o);
      if (lane >= o) ti += y;
    }
    if (lane < SCAN_THREADS / 32) warp_tot[lane] = ti - t;
    if (lane == SCAN_THREADS / 32 - 1 && sums) sums[blockIdx.x] = ti;
  }
  __syncthreads();
  int off = warp_tot[wid] + incl - run;
#pragma unroll
  for (int q = 0; q < SCAN_ITEMS; ++q)
    if (base + q < n) out[base + q] = v[q] + off;
}

__global__ void scan_add_kernel(int* out, const int* offs, long long n) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) out[i] += offs[i / SCAN_TILE];
}

// ---------------------------------------------------------------------------
// deterministic mode: cell-sorted permutation + node-owner gather
// ---------------------------------------------------------------------------

__global__ void cell_key_kernel(Params p, int* key, int* rank, int* cell_count) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= p.n) return;
  int c[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    float g = __fmul_rn(ldf(p, FX + a, i), p.inv_dx);
    int bb = (int)floorf(__fsub_rn(g, 0.5f));
    c[a] = max(0, min(bb, p.res[a] - 3));
  }
  int k = (c[0] * p.res[1] + c[1]) * p.res[2] + c[2];
  key[i] = k;
  rank[i] = atomicAdd(cell_count + k, 1);
}

__global__ void cell_fill_kernel(const int* key, const int* rank, const int* start, int* perm,
                                 long long n) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) perm[start[key[i]] + rank[i]] = (int)i;
}

// Order each cell's slots by original particle index (insertion sort; cells
// hold a handful of particles).
__global__ void cell_sort_kernel(const int* cell_count, const int* start, int* perm, const int* orig,
                                 long long ncells) {
  long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= ncells) return;
  int cnt = cell_count[c];
  if (cnt < 2) return;
  int* s = perm + start[c];
  for (int a = 1; a < cnt; ++a) {
    int v = s[a], key = orig[v];
    int b = a - 1;
    while (b >= 0 && orig[s[b]] > key) {
      s[b + 1] = s[b];
      --b;
    }
    s[b + 1] = v;
  }
}

// payload = (A 9, m v 3) per slot; F advanced in place (exact rounding).
__global__ void det_payload_kernel(Params p, float* payload) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  unsigned inv = 0;
  if (i < p.n) {
    float F[9], C[9], A[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) {
      F[q] = ldf(p, FF + q, i);
      C[q] = ldf(p, FC + q, i);
    }
    float m = ldf(p, FMASS, i), vol = ldf(p, FVOL, i);
    int mid = p.mat[i];
    float det = affine_update<true>(F, C, m, vol, p.mu[mid], p.lam[mid], p.dt, p.stress_coef,
                                    p.stress_form, A);
    inv = det <= 0.0f;
#pragma unroll
    for (int q = 0; q < 9; ++q) {
      stf(p, FF + q, i, F[q]);
      payload[q * p.cap + i] = A[q];
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) payload[(9 + a) * p.cap + i] = __fmul_rn(m, ldf(p, FV + a, i));
  }
  warp_count_add(p.inverted, inv);
}

// Node-owner gather: node (i,j,k) sums its 27 source cells in ascending cell
// key (offsets 2..0 per axis), particles in ascending original index, from
// 0.0f with separately rounded ops -- the order of oracle orc32_p2g_sorted.
__global__ void __launch_bounds__(256) det_gather_kernel(Params p, const float* payload,
                                                         const int* cell_count, const int* start,
                                                         const int* perm) {
  long long node = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long nn = (long long)p.res[0] * p.res[1] * p.res[2];
  if (node >= nn) return;
  int gk = (int)(node % p.res[2]);
  int gj = (int)((node / p.res[2]) % p.res[1]);
  int gi = (int)(node / ((long long)p.res[1] * p.res[2]));
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int oi = 2; oi >= 0; --oi) {
    int ci = gi - oi;
    if (ci < 0 || ci > p.res[0] - 3) continue;
    for (int oj = 2; oj >= 0; --oj) {
      int cj = gj - oj;
      if (cj < 0 || cj > p.res[1] - 3) continue;
      for (int ok = 2; ok >= 0; --ok) {
        int ck = gk - ok;
        if (ck < 0 || ck > p.res[2] - 3) continue;
        long long cell = ((long long)ci * p.res[1] + cj) * p.res[2] + ck;
        int s0 = start[cell], s1 = s0 + cell_count[cell];
        for (int s = s0; s < s1; ++s) {
          int q = perm[s];
          int b[3];
          float f[3], w[3][3];
#pragma unroll
          for (int a = 0; a < 3; ++a) stencil_rn(ldf(p, FX + a, q), p.inv_dx, p.res[a], b[a], f[a], w[a]);
          float wt = __fmul_rn(__fmul_rn(w[0][oi], w[1][oj]), w[2][ok]);
          float dp[3] = {__fmul_rn(__fsub_rn((float)oi, f[0]), p.dx),
                         __fmul_rn(__fsub_rn((float)oj, f[1]), p.dx),
                         __fmul_rn(__fsub_rn((float)ok, f[2]), p.dx)};
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            float t = __fadd_rn(payload[(9 + a) * p.cap + q], __fmul_rn(payload[(3 * a) * p.cap + q], dp[0]));
            t = __fadd_rn(t, __fmul_rn(payload[(3 * a + 1) * p.cap + q], dp[1]));
            t = __fadd_rn(t, __fmul_rn(payload[(3 * a + 2) * p.cap + q], dp[2]));
            acc[a] = __fadd_rn(acc[a], __fmul_rn(wt, t));
          }
          acc[3] = __fadd_rn(acc[3], __fmul_rn(wt, ldf(p, FMASS, q)));
        }
      }
    }
  }
  p.gm[node_index(gi, gj, gk, p.nb[1], p.nb[2])] = make_float4(acc[0], acc[1], acc[2], acc[3]);
}

// ---------------------------------------------------------------------------
// host <-> device conversions (fp64 AoS in caller order <-> fp32 SoA slots)
// ---------------------------------------------------------------------------

// staging layout per particle: x 3, v 3, F 9, C 9 doubles (AoS, caller order)
__global__ void upload_fields_kernel(Params p, const double* __restrict__ x, const double* __restrict__ v,
                                     const double* __restrict__ F, const double* __restrict__ C,
                                     unsigned mask) {
  long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s >= p.n) return;
  long long o = p.orig[s];
  if (mask & 1u)
    for (int a = 0; a < 3; ++a) stf(p, FX + a, s, (float)x[3 * o + a]);
  if (mask & 2u)
    for (int a = 0; a < 3; ++a) stf(p, FV + a, s, (float)v[3 * o + a]);
  if (mask & 4u)
    for (int q = 0; q < 9; ++q) stf(p, FF + q, s, (float)F[9 * o + q]);
  if (mask & 8u)
    for (int q = 0; q < 9; ++q) stf(p, FC + q, s, (float)C[9 * o + q]);
}

__global__ void download_fields_kernel(Params p, double* __restrict__ x, double* __restrict__ v,
                                       double* __restrict__ F, double* __restrict__ C, unsigned mask) {
  long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s >= p.n) return;
  long long o = p.orig[s];
  if (mask & 1u)
    for (int a = 0; a < 3; ++a) x[3 * o + a] = ldf(p, FX + a, s);
  if (mask & 2u)
    for (int a = 0; a < 3; ++a) v[3 * o + a] = ldf(p, FV + a, s);
  if (mask & 4u)
    for (int q = 0; q < 9; ++q) F[9 * o + q] = ldf(p, FF + q, s);
  if (mask & 8u)
    for (int q = 0; q < 9; ++q) C[9 * o + q] = ldf(p, FC + q, s);
}

__global__ void upload_static_kernel(Params p, const double* mass, const double* vol, const int* mat) {
  long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s >= p.n) return;
  stf(p, FMASS, s, (float)mass[s]);
  stf(p, FVOL, s, (float)vol[s]);
  p.mat[s] = mat[s];
  p.orig[s] = (int)s;
}

// grid: C-order fp64 (nx,ny,nz,3)+(nx,ny,nz) <-> blocked float4
__global__ void upload_grid_kernel(Params p, float4* dst, const double* mv, const double* m) {
  long long node = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long nn = (long long)p.res[0] * p.res[1] * p.res[2];
  if (node >= nn) return;
  int gk = (int)(node % p.res[2]);
  int gj = (int)((node / p.res[2]) % p.res[1]);
  int gi = (int)(node / ((long long)p.res[1] * p.res[2]));
  dst[node_index(gi, gj, gk, p.nb[1], p.nb[2])] =
      make_float4((float)mv[3 * node], (float)mv[3 * node + 1], (float)mv[3 * node + 2],
                  m ? (float)m[node] : 0.0f);
}

// phase 0: grid_mv = gm.xyz (after p2g); phase 1: velocity view (after
// grid_update): massive nodes -> gv, others -> gm.xyz (momentum, untouched
// by the reference's grid_update).
__global__ void download_grid_kernel(Params p, int phase, double* mv, double* m) {
  long long node = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long nn = (long long)p.res[0] * p.res[1] * p.res[2];
  if (node >= nn) return;
  int gk = (int)(node % p.res[2]);
  int gj = (int)((node / p.res[2]) % p.res[1]);
  int gi = (int)(node / ((long long)p.res[1] * p.res[2]));
  long long idx = node_index(gi, gj, gk, p.nb[1], p.nb[2]);
  float4 a = p.gm[idx];
  float4 o = a;
  if (phase == 1) {
    float4 g = p.gv[idx];
    if (a.w > 0.0f || phase == 2) o = g;
  } else if (phase == 2) {
    o = p.gv[idx];
  }
  mv[3 * node] = o.x;
  mv[3 * node + 1] = o.y;
  mv[3 * node + 2] = o.z;
  if (m) m[node] = a.w;
}

__global__ void collision_field_kernel(Params p, Colliders cs, double cap, double* dist, int* obj) {
  long long node = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long nn = (long long)p.res[0] * p.res[1] * p.res[2];
  if (node >= nn) return;
  int gk = (int)(node % p.res[2]);
  int gj = (int)((node / p.res[2]) % p.res[1]);
  int gi = (int)(node / ((long long)p.res[1] * p.res[2]));
  double best;
  int id = nearest_collider(cs, (double)gi * p.dx64, (double)gj * p.dx64, (double)gk * p.dx64, cap, best);
  dist[node] = best;
  obj[node] = id;
}

__global__ void has_nan_kernel(Params p, int* flag) {
  long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s >= p.n) return;
  bool bad = false;
  for (int f = 0; f < FC; ++f) bad |= isnan(ldf(p, f, s));
  if (bad) *flag = 1;
}

}  // namespace mpm
