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
#include "mc_table.h"

#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace mpm {

// Programmatic dependent launch (the fused kernel and the grid op alternate
// within a substep stretch): a kernel launched with programmatic stream
// serialization may start while its predecessor drains; griddep_wait() blocks
// until the predecessor has completed and its writes are visible, and
// griddep_trigger() lets the successor's CTAs be scheduled.  Each kernel
// triggers only after its own wait, so at most two kernels overlap and the
// code before a wait may read anything produced two launches back.  Both are
// no-ops in a normal launch.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

#ifdef FUSED_PROFILE
__device__ unsigned long long g_fprof[6];
__device__ unsigned long long g_fcnt[4];  // particles, G2P off-tile, P2G fallback
__device__ unsigned long long g_gprof[8];  // grid op: sum / max CTA ns, CTAs, launches, sum of per-launch max, clearing launches, bricks
__device__ unsigned long long g_cprof[4];  // grid contact: warp calls, lanes, cycles, max cycles
__device__ unsigned long long g_gwin[4] = {~0ull, 0ull, 0ull, 0ull};
// inter-kernel bubbles: [0] last fused CTA end, [1] last grid-op CTA end, [2] fused min start,
// [3] fused CTAs done, [4] sum fused->grid gap ns, [5] count, [6] sum grid->fused gap ns, [7] count
__device__ unsigned long long g_bub[8] = {0ull, 0ull, ~0ull, 0ull, 0ull, 0ull, 0ull, 0ull};
__device__ unsigned long long g_fwin[4];  // fused: sum of windows, launches, sum of CTA durations, CTAs
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define FPROF_COUNT(k) atomicAdd(&g_fcnt[k], 1ull)
#else
#define FPROF_COUNT(k)
#endif

__device__ __forceinline__ void mark_brick(const Params& p, long long idx) {
  int b = (int)(idx >> 6);
  if (*((volatile int*)p.brick_flag + b) == 0) {
    if (atomicExch(&p.brick_flag[b], 1) == 0) {
      int s = atomicAdd(p.active_count, 1);
      p.active_list[s] = b;
    }
  }
}

// Mark the (up to 2x2x2) bricks of a 3^3 stencil with base cell b: all flag
// loads are issued before any is tested (one L2 round trip, not one per node).
__device__ __forceinline__ void mark_stencil_bricks(const Params& p, const int b[3]) {
  const int bx0 = b[0] >> BRICK_SHIFT, by0 = b[1] >> BRICK_SHIFT, bz0 = b[2] >> BRICK_SHIFT;
  const int dx = ((b[0] + 2) >> BRICK_SHIFT) - bx0, dy = ((b[1] + 2) >> BRICK_SHIFT) - by0,
            dz = ((b[2] + 2) >> BRICK_SHIFT) - bz0;
  int id[8], f[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    id[k] = ((bx0 + ((k >> 2) & dx)) * p.nb[1] + by0 + ((k >> 1) & dy)) * p.nb[2] + bz0 + (k & dz);
    f[k] = *((volatile int*)p.brick_flag + id[k]);
  }
#pragma unroll
  for (int k = 0; k < 8; ++k)
    if (f[k] == 0 && atomicExch(&p.brick_flag[id[k]], 1) == 0) p.active_list[atomicAdd(p.active_count, 1)] = id[k];
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

// Velocity sources for the G2P gather: the blocked global grid (through L1)
// or a shared-memory SoA tile of the work item's node box.
struct GlobalVel {
  const float4* gv;
  int sx, sy;  // brick strides (x: nb1*nb2*64, y: nb2*64)
  __device__ __forceinline__ void offsets(const int b[3], int ox[3], int oy[3], int oz[3]) const {
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      ox[q] = ((b[0] + q) >> BRICK_SHIFT) * sx + ((b[0] + q) & 3) * 16;
      oy[q] = ((b[1] + q) >> BRICK_SHIFT) * sy + ((b[1] + q) & 3) * 4;
      oz[q] = ((b[2] + q) >> BRICK_SHIFT) * 64 + ((b[2] + q) & 3);
    }
  }
  __device__ __forceinline__ float3 load(int idx) const {
    const float4 g = __ldg(gv + idx);
    return make_float3(g.x, g.y, g.z);
  }
  __device__ __forceinline__ void load2(int idx, f2p& xy, float& z) const {
    const float4 g = __ldg(gv + idx);
    xy = f2_pack(g.x, g.y);
    z = g.z;
  }
};

struct TileVel {
  const float* t;  // 3 x TILE_NODES floats: (vx, vy) pairs, then vz
  int org[3];
  int lo[3], hi[3];  // loaded base-cell box (tile coords); nodes [lo, hi + 2]
  __device__ __forceinline__ void offsets(const int b[3], int ox[3], int oy[3], int oz[3]) const {
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      ox[q] = (b[0] - org[0] + q) * TILE * TILE_Z;
      oy[q] = (b[1] - org[1] + q) * TILE_Z;
      oz[q] = (b[2] - org[2] + q);
    }
  }
  __device__ __forceinline__ float3 load(int idx) const {
    const float2 xy = reinterpret_cast<const float2*>(t)[idx];
    return make_float3(xy.x, xy.y, t[2 * TILE_NODES + idx]);
  }
  __device__ __forceinline__ void load2(int idx, f2p& xy, float& z) const {
    xy = reinterpret_cast<const f2p*>(t)[idx];
    z = t[2 * TILE_NODES + idx];
  }
};

// Packed twin of g2p_gather below: the (x, y) velocity components travel as
// one FFMA2 pair, z as scalar FFMA (186 fp issue slots per particle instead of
// 279).  Same sums in the same order per component.
template <class Src>
__device__ __forceinline__ void g2p_gather_pk(const Params& p, const Src& src, const int b[3], const float f[3],
                                              const float w[3][3], float v[3], float C[9]) {
  int ox[3], oy[3], oz[3];
  src.offsets(b, ox, oy, oz);
  float wd[3][3];  // w * (offset - f)
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int q = 0; q < 3; ++q) wd[a][q] = w[a][q] * ((float)q - f[a]);
  f2p v01 = 0, c001 = 0, c101 = 0, c201 = 0;
  float vz = 0.f, c0z = 0.f, c1z = 0.f, c2z = 0.f;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    f2p hv01 = 0, hj01 = 0, hk01 = 0;
    float hvz = 0.f, hjz = 0.f, hkz = 0.f;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      f2p gv01 = 0, gk01 = 0;
      float gvz = 0.f, gkz = 0.f;
      const int oij = ox[i] + oy[j];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        f2p g01;
        float gz;
        src.load2(oij + oz[k], g01, gz);
        if (k == 0) {
          gv01 = f2_mul(f2_bc(w[2][0]), g01);
          gk01 = f2_mul(f2_bc(wd[2][0]), g01);
          gvz = w[2][0] * gz;
          gkz = wd[2][0] * gz;
        } else {
          gv01 = f2_fma(f2_bc(w[2][k]), g01, gv01);
          gk01 = f2_fma(f2_bc(wd[2][k]), g01, gk01);
          gvz = fmaf(w[2][k], gz, gvz);
          gkz = fmaf(wd[2][k], gz, gkz);
        }
      }
      if (j == 0) {
        hv01 = f2_mul(f2_bc(w[1][0]), gv01);
        hj01 = f2_mul(f2_bc(wd[1][0]), gv01);
        hk01 = f2_mul(f2_bc(w[1][0]), gk01);
        hvz = w[1][0] * gvz;
        hjz = wd[1][0] * gvz;
        hkz = w[1][0] * gkz;
      } else {
        hv01 = f2_fma(f2_bc(w[1][j]), gv01, hv01);
        hj01 = f2_fma(f2_bc(wd[1][j]), gv01, hj01);
        hk01 = f2_fma(f2_bc(w[1][j]), gk01, hk01);
        hvz = fmaf(w[1][j], gvz, hvz);
        hjz = fmaf(wd[1][j], gvz, hjz);
        hkz = fmaf(w[1][j], gkz, hkz);
      }
    }
    if (i == 0) {
      v01 = f2_mul(f2_bc(w[0][0]), hv01);
      c001 = f2_mul(f2_bc(wd[0][0]), hv01);
      c101 = f2_mul(f2_bc(w[0][0]), hj01);
      c201 = f2_mul(f2_bc(w[0][0]), hk01);
      vz = w[0][0] * hvz;
      c0z = wd[0][0] * hvz;
      c1z = w[0][0] * hjz;
      c2z = w[0][0] * hkz;
    } else {
      v01 = f2_fma(f2_bc(w[0][i]), hv01, v01);
      c001 = f2_fma(f2_bc(wd[0][i]), hv01, c001);
      c101 = f2_fma(f2_bc(w[0][i]), hj01, c101);
      c201 = f2_fma(f2_bc(w[0][i]), hk01, c201);
      vz = fmaf(w[0][i], hvz, vz);
      c0z = fmaf(wd[0][i], hvz, c0z);
      c1z = fmaf(w[0][i], hjz, c1z);
      c2z = fmaf(w[0][i], hkz, c2z);
    }
  }
  const float cc = 4.0f * p.inv_dx;  // coef * dx = 4/dx
  const f2p cc2 = f2_bc(cc);
  c001 = f2_mul(cc2, c001);
  c101 = f2_mul(cc2, c101);
  c201 = f2_mul(cc2, c201);
  v[0] = f2_lo(v01);
  v[1] = f2_hi(v01);
  v[2] = vz;
  C[0] = f2_lo(c001);
  C[3] = f2_hi(c001);
  C[6] = c0z * cc;
  C[1] = f2_lo(c101);
  C[4] = f2_hi(c101);
  C[7] = c1z * cc;
  C[2] = f2_lo(c201);
  C[5] = f2_hi(c201);
  C[8] = c2z * cc;
}

// G2P gather (kernels.py:451-516): v = sum w g, C = 4/dx^2 sum w g dp^T,
// evaluated separably (k, then j, then i sums): 279 FMA instead of 432.
template <class Src>
__device__ __forceinline__ void g2p_gather(const Params& p, const Src& src, const int b[3],
                                           const float f[3], const float w[3][3], float v[3],
                                           float C[9]) {
  int ox[3], oy[3], oz[3];
  src.offsets(b, ox, oy, oz);
  float wd[3][3];  // w * (offset - f)
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int q = 0; q < 3; ++q) wd[a][q] = w[a][q] * ((float)q - f[a]);
  float c0[3] = {0.f, 0.f, 0.f}, c1[3] = {0.f, 0.f, 0.f}, c2[3] = {0.f, 0.f, 0.f};
  v[0] = v[1] = v[2] = 0.f;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    float hv[3] = {0.f, 0.f, 0.f}, hj[3] = {0.f, 0.f, 0.f}, hk[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      float gv[3] = {0.f, 0.f, 0.f}, gk[3] = {0.f, 0.f, 0.f};
      const int oij = ox[i] + oy[j];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const float3 g = src.load(oij + oz[k]);
        gv[0] += w[2][k] * g.x; gv[1] += w[2][k] * g.y; gv[2] += w[2][k] * g.z;
        gk[0] += wd[2][k] * g.x; gk[1] += wd[2][k] * g.y; gk[2] += wd[2][k] * g.z;
      }
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        hv[r] += w[1][j] * gv[r];
        hj[r] += wd[1][j] * gv[r];
        hk[r] += w[1][j] * gk[r];
      }
    }
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      v[r] += w[0][i] * hv[r];
      c0[r] += wd[0][i] * hv[r];
      c1[r] += w[0][i] * hj[r];
      c2[r] += w[0][i] * hk[r];
    }
  }
  const float cc = 4.0f * p.inv_dx;  // coef * dx = 4/dx
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    C[3 * r] = c0[r] * cc;
    C[3 * r + 1] = c1[r] * cc;
    C[3 * r + 2] = c2[r] * cc;
  }
}

__device__ __forceinline__ GlobalVel global_vel(const Params& p) {
  GlobalVel s;
  s.gv = p.gv;
  s.sx = p.nb[1] * p.nb[2] * 64;
  s.sy = p.nb[2] * 64;
  return s;
}

// G2P at x from the global grid (stage g2p_advect / final G2P of a frame).
__device__ __forceinline__ void g2p_gather(const Params& p, const float x[3], float v[3], float C[9]) {
  int b[3];
  float f[3], w[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a) stencil(x[a], p.inv_dx, p.res[a], b[a], f[a], w[a]);
  g2p_gather(p, global_vel(p), b, f, w, v, C);
}

// x += dt v, clamped to the margins of the particle's environment tile
// (core.py:51-56, kernels.py:517-534; one tile = the whole grid normally).
// SINGLE: one environment, no slab window (the common case, specialised at
// compile time: no tile-origin arithmetic per particle and axis).
template <bool SINGLE = false>
__device__ __forceinline__ void advect(const Params& p, float x[3], const float v[3]) {
  if constexpr (SINGLE) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      float q = x[a] + p.dt * v[a];
      q = q < p.lo ? p.lo : q;
      q = q > p.hi[a] ? p.hi[a] : q;
      x[a] = q;
    }
  } else {
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    // environment tile origin in window-local coordinates (the walls keep a
    // particle >= 1.5 cells inside its tile, so the reciprocal's rounding
    // cannot move it across a tile boundary)
    const float org =
        (p.env_res[a] == p.gres[a] ? 0.0f : floorf((x[a] + p.goffx[a]) * p.inv_env_ext[a]) * p.env_ext[a]) -
        p.goffx[a];
    float q = x[a] + p.dt * v[a];
    q = q < org + p.lo ? org + p.lo : q;
    q = q > org + p.hi[a] ? org + p.hi[a] : q;
    x[a] = q;
  }
  }
}

// Per-particle P2G payload, computed in pass 1 of the fused kernel and kept
// in registers across the tile's scale reduction.
struct Payload {
  int b[3];      // base cell of the (advected) position
  float f[3];    // fractional offset in cells
  float m;       // mass
  float mv[3];   // m v
  float A[9];    // m C + k P F^T (kernels.py:264-275)
};

constexpr float MAGIC = 12582912.0f;  // 1.5 * 2^23: FFMA -> round-to-nearest int in the low bits
constexpr int MAGIC_BITS = 0x4B400000;

__device__ __forceinline__ int fixq(float wt, float val) {
  return __float_as_int(fmaf(wt, val, MAGIC)) - MAGIC_BITS;
}

// Scatter one payload.  TILE_MODE: int32 fixed-point ATOMS.ADD into the smem
// tile (origin org, per-channel scale S); else float REDG.F32x4 into gm.
template <bool TILE_MODE>
__device__ __forceinline__ void p2g_scatter(const Params& p, int* tile, const int org[3],
                                            const Payload& q, const float S[4]) {
  float w[3][3];
  float dxs[3][3];  // (offset - f) * dx
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    float t0 = 1.5f - q.f[a], t1 = q.f[a] - 1.0f, t2 = q.f[a] - 0.5f;
    w[a][0] = 0.5f * (t0 * t0);
    w[a][1] = 0.75f - t1 * t1;
    w[a][2] = 0.5f * (t2 * t2);
#pragma unroll
    for (int o = 0; o < 3; ++o) dxs[a][o] = ((float)o - q.f[a]) * p.dx;
  }
  // scaled payload: channel r of (mv, m) in tile units
  const float sc[4] = {TILE_MODE ? S[0] : 1.f, TILE_MODE ? S[1] : 1.f, TILE_MODE ? S[2] : 1.f,
                       TILE_MODE ? S[3] : 1.f};
  float ax[3][3], ay[3][3], az[3][3];
#pragma unroll
  for (int o = 0; o < 3; ++o)
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      ax[o][r] = q.A[3 * r] * sc[r] * dxs[0][o];
      ay[o][r] = q.A[3 * r + 1] * sc[r] * dxs[1][o];
      az[o][r] = q.A[3 * r + 2] * sc[r] * dxs[2][o];
    }
  const float mvs[3] = {q.mv[0] * sc[0], q.mv[1] * sc[1], q.mv[2] * sc[2]};
  const float ms = q.m * sc[3];
  int ox[3], oy[3], oz[3];
  if (TILE_MODE) {
#pragma unroll
    for (int o = 0; o < 3; ++o) {
      ox[o] = (q.b[0] - org[0] + o) * TILE * TILE_Z;
      oy[o] = (q.b[1] - org[1] + o) * TILE_Z;
      oz[o] = (q.b[2] - org[2] + o);
    }
  } else {
    axis_offsets(q.b[0], p.nb[1] * p.nb[2] * 64, 16, ox);
    axis_offsets(q.b[1], p.nb[2] * 64, 4, oy);
    axis_offsets(q.b[2], 64, 1, oz);
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const float wij = w[0][i] * w[1][j];
      float bij[3];
#pragma unroll
      for (int r = 0; r < 3; ++r) bij[r] = mvs[r] + ax[i][r] + ay[j][r];
      const int oij = ox[i] + oy[j];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const float wt = wij * w[2][k];
        const int idx = oij + oz[k];
        if (TILE_MODE) {
          int* t = tile + idx;  // SoA channels: conflict-free banks for spread nodes
          atomicAdd(t, fixq(wt, bij[0] + az[k][0]));
          atomicAdd(t + TILE_NODES, fixq(wt, bij[1] + az[k][1]));
          atomicAdd(t + 2 * TILE_NODES, fixq(wt, bij[2] + az[k][2]));
          atomicAdd(t + 3 * TILE_NODES, fixq(wt, ms));
        } else {
          atomicAdd(p.gm + idx, make_float4(wt * (bij[0] + az[k][0]), wt * (bij[1] + az[k][1]),
                                            wt * (bij[2] + az[k][2]), wt * ms));
        }
      }
    }
  }
  if (!TILE_MODE) mark_stencil_bricks(p, q.b);
}

// Raw particle fields of one slot.
template <bool G2P>
struct PRaw {
  float x[3];
  float F[9];
  float m, vol;
  int mid;
  float v[G2P ? 1 : 3];
  float C[G2P ? 1 : 9];
};

template <bool G2P>
__device__ __forceinline__ void load_raw(const Params& p, long long i, PRaw<G2P>& r) {
#pragma unroll
  for (int a = 0; a < 3; ++a) r.x[a] = ldf(p, FX + a, i);
#pragma unroll
  for (int q = 0; q < 9; ++q) r.F[q] = ldf(p, FF + q, i);
  r.m = ldf(p, FMASS, i);
  r.vol = ldf(p, FVOL, i);
  r.mid = p.mat[i];
  if (!G2P) {
#pragma unroll
    for (int a = 0; a < 3; ++a) r.v[a] = ldf(p, FV + a, i);
#pragma unroll
    for (int q = 0; q < 9; ++q) r.C[q] = ldf(p, FC + q, i);
  }
}

// Stage-A work for one slot: (G2P + advect) or (v, C as loaded), then F update
// + stress -> payload.  STORE: write x and F back.  Returns det(F').
template <bool G2P, bool STORE = true, bool SINGLE = false>
__device__ __forceinline__ float compute_payload(const Params& p, long long i, PRaw<G2P>& r, Payload& q,
                                                 const TileVel* tv) {
  float v[3], C[9];
  if (G2P) {
    int b[3];
    float f[3], w[3][3];
    bool in_tile = tv != nullptr;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      stencil(r.x[a], p.inv_dx, p.res[a], b[a], f[a], w[a]);
      if (tv) in_tile &= (b[a] - tv->org[a] >= tv->lo[a]) && (b[a] - tv->org[a] <= tv->hi[a]);
    }
    if (in_tile) {
      g2p_gather_pk(p, *tv, b, f, w, v, C);
    } else {
      if (tv) FPROF_COUNT(1);
      g2p_gather(p, global_vel(p), b, f, w, v, C);
    }
    advect<SINGLE>(p, r.x, v);
    if (STORE) {
#pragma unroll
      for (int a = 0; a < 3; ++a) stf(p, FX + a, i, r.x[a]);
    }
  } else {
#pragma unroll
    for (int a = 0; a < 3; ++a) v[a] = r.v[a];
#pragma unroll
    for (int c = 0; c < 9; ++c) C[c] = r.C[c];
  }
  const float det = affine_update<false>(r.F, C, r.m, r.vol, __ldg(p.mu + r.mid), __ldg(p.lam + r.mid), p.dt,
                                         p.stress_coef, p.stress_form, q.A);
  if (STORE) {
#pragma unroll
    for (int c = 0; c < 9; ++c) stf(p, FF + c, i, r.F[c]);
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const float g = r.x[a] * p.inv_dx;
    int bb = (int)floorf(g - 0.5f);
    bb = max(0, min(bb, p.res[a] - 3));
    q.b[a] = bb;
    q.f[a] = g - (float)bb;
    q.mv[a] = r.m * v[a];
  }
  q.m = r.m;
  return det;
}

// Per-channel magnitude bound of a payload's node contributions / weight:
// |mv_r + (A dp)_r| <= |mv_r| + 1.5 dx sum_c |A_rc|, and m.
__device__ __forceinline__ void payload_bound(const Params& p, const Payload& q, float b[4]) {
  const float h = 1.5f * p.dx;
#pragma unroll
  for (int r = 0; r < 3; ++r)
    b[r] = fabsf(q.mv[r]) + h * (fabsf(q.A[3 * r]) + fabsf(q.A[3 * r + 1]) + fabsf(q.A[3 * r + 2]));
  b[3] = q.m;
}

// Fixed-point scale of one channel for a work item whose per-particle bound
// is B and whose densest cell held maxcnt particles at re-binning:
//   S = 2^floor(log2(min(2^22 / (W B), 2^31 / (K * 2 maxcnt * B)))),
// W = 0.4219 the largest 27-point weight, K = 1.75^3 = 5.36 the sum over the 27
// stencil offsets of each offset's largest weight.  Every contribution then
// fits the FFMA magic-number conversion (|c S| < 2^22), and a node sum --
// at most K * (particles per cell) * B -- stays inside int32 even if cells
// double their occupancy before the next re-binning.
//
// The occupancy assumption is enforced, not trusted: the scatter counts the
// particles of every base cell in shared memory (cell_limit) and a particle
// whose cell already holds the limit goes down the float REDG path instead,
// so no tile node sum can leave int32 whatever the compression.  fx_shift (a
// test hook, 0 in production) loosens the node-sum term of the scale by
// 2^fx_shift and divides the cell limit by the same factor: without the
// guard, dense cells would then wrap; with it the bound still holds
// (K x limit x B x S <= 2^31) and the guard fires on ordinary scenes.
__device__ __forceinline__ float channel_scale(float B, int maxcnt, int fx_shift = 0) {
  if (!(B > 0.f)) return 1.0f;
  const float lim = fminf(4194304.0f / 0.4219f,
                          exp2f(31.0f + (float)fx_shift) / (5.36f * 2.0f * (float)max(maxcnt, 1)));
  return exp2f(floorf(log2f(lim / B)));
}
__device__ __forceinline__ int cell_limit(int maxcnt, int fx_shift) { return (2 * max(maxcnt, 1)) >> fx_shift; }

// One (ty, tz) column of the velocity tile, nodes tx in [x0, x1] (<= TILE):
// loads issued in groups of 5 before their shared-memory stores.
__device__ __forceinline__ void load_vtile_column(const Params& p, float* vtile, int orgx, int x0, int x1,
                                                  int ty, int tz, long long yz, long long xstride) {
  constexpr int G = 5;
  for (int xs = x0; xs <= x1; xs += G) {
    float4 g[G];
#pragma unroll
    for (int u = 0; u < G; ++u) {
      const int gi = orgx + xs + u;
      if (xs + u <= x1) g[u] = __ldg(p.gv + (gi >> BRICK_SHIFT) * xstride + yz + ((gi & 3) << 4));
    }
#pragma unroll
    for (int u = 0; u < G; ++u) {
      if (xs + u <= x1) {
        const int t = ((xs + u) * TILE + ty) * TILE_Z + tz;
        reinterpret_cast<float2*>(vtile)[t] = make_float2(g[u].x, g[u].y);
        vtile[2 * TILE_NODES + t] = g[u].z;
      }
    }
  }
}

// Same column with LDGSTS (cp.async, 4-byte, L1-allocating): no registers and
// no stall at issue; completion is awaited (cp.async.wait_all) before the
// barrier that publishes the tile.
__device__ __forceinline__ void cp_async4(float* dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async8(float* dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ void load_vtile_column_async(const Params& p, float* vtile, int orgx, int x0, int x1,
                                                        int ty, int tz, long long yz, long long xstride) {
  for (int tx = x0; tx <= x1; ++tx) {
    const int gi = orgx + tx;
    const float* src = reinterpret_cast<const float*>(p.gv + (gi >> BRICK_SHIFT) * xstride + yz + ((gi & 3) << 4));
    const int t = (tx * TILE + ty) * TILE_Z + tz;
    cp_async8(vtile + 2 * t, src);
    cp_async4(vtile + 2 * TILE_NODES + t, src + 2);
  }
}

// Stage A of a substep: G2P(n) -> advect -> F update -> Neo-Hookean stress for
// every particle of a work item; writes x, F and the P2G payload (m v, A, m:
// NPAY floats SoA) and the item's exact per-channel bound (warp max ->
// atomicMax on the float bits; bounds are zeroed before the launch).  The G2P
// reads a double-buffered shared-memory SoA velocity tile covering the node
// box this item scattered to in the previous substep (x is unchanged in
// between), so each item costs one barrier.
// G2P=false: first substep of a stretch (v, C from memory).
template <bool G2P>
__global__ void __launch_bounds__(FUSED_THREADS, 3) g2p_stress_kernel(Params p, float* __restrict__ pay,
                                                                    float4* __restrict__ bounds,
                                                                    const int* __restrict__ item_box) {
  extern __shared__ float vtiles[];  // G2P: 2 x (3 x TILE_NODES) SoA velocity tiles
  const int nwork = *p.nwork;
  unsigned inverted = 0;
  int buf = 0;
  for (int wi = blockIdx.x; wi < nwork; wi += gridDim.x, buf ^= 1) {
    const int4 item = p.work[wi];
    TileVel tv;
    float* vtile = vtiles + buf * 3 * TILE_NODES;
    tv.t = vtile;
    if (G2P) {
      const int bin = item.x;
      int bx, by, bz;
      bin_coords(p, bin, bx, by, bz);
      tv.org[0] = bx * BIN - MARGIN;
      tv.org[1] = by * BIN - MARGIN;
      tv.org[2] = bz * BIN - MARGIN;
      const int pb = item_box[wi];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        tv.lo[a] = (pb >> (4 * a)) & 15;
        tv.hi[a] = (pb >> (12 + 4 * a)) & 15;
      }
      // 2-D mapping over the (y, z) node box, loop along x
      for (int c = threadIdx.x; c < 256; c += blockDim.x) {
        const int ty = tv.lo[1] + (c >> 4), tz = tv.lo[2] + (c & 15);
        const int gj = tv.org[1] + ty, gk = tv.org[2] + tz;
        if (tv.lo[0] <= tv.hi[0] && ty <= tv.hi[1] + 2 && tz <= tv.hi[2] + 2 && gj < p.res[1] && gk < p.res[2]) {
          const long long yz = ((long long)(gj >> BRICK_SHIFT) * p.nb[2] + (gk >> BRICK_SHIFT)) * 64 +
                               ((gj & 3) << 2) + (gk & 3);
          const long long xstride = (long long)p.nb[1] * p.nb[2] * 64;
          load_vtile_column(p, vtile, tv.org[0], tv.lo[0], tv.hi[0] + 2, ty, tz, yz, xstride);
        }
      }
      __syncthreads();
    }
    float mx[4] = {0.f, 0.f, 0.f, 0.f};
    for (long long i = (long long)item.y + threadIdx.x; i < item.z; i += blockDim.x) {
      PRaw<G2P> cur;
      load_raw<G2P>(p, i, cur);
      Payload q;
      const float det = compute_payload<G2P>(p, i, cur, q, G2P ? &tv : nullptr);
      inverted += det <= 0.0f;
      float b[4];
      payload_bound(p, q, b);
#pragma unroll
      for (int c = 0; c < 4; ++c) mx[c] = fmaxf(mx[c], b[c]);
#pragma unroll
      for (int r = 0; r < 3; ++r) pay[r * p.cap + i] = q.mv[r];
#pragma unroll
      for (int r = 0; r < 9; ++r) pay[(3 + r) * p.cap + i] = q.A[r];
      pay[12 * p.cap + i] = q.m;
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const unsigned u = __reduce_max_sync(0xffffffffu, __float_as_uint(mx[c]));
      if ((threadIdx.x & 31) == 0 && u) atomicMax(reinterpret_cast<unsigned*>(bounds + wi) + c, u);
    }
  }
  warp_count_add(p.inverted, inverted);
}

// Scatter one particle's payload into the int32 tile with lane-rotated
// channels: slot s of a lane adds channel (s + rot) & 3 at tile + off[s], so
// the 4 lanes of a quad hit 4 different channel planes at each step -- the
// common case of several lanes on the same cell does not collide on one word.
// Every channel has the uniform form wt * (b + A_row . dp) (mass: b = m, zero
// A row); sel4 picks the rotated row values.
__device__ __forceinline__ float sel4(bool r1, bool r2, float v0, float v1, float v2, float v3) {
  const float a = r1 ? v1 : v0;
  const float b = r1 ? v3 : v2;
  return r2 ? b : a;
}

__device__ __forceinline__ void tile_scatter_rot(int* tile, const int off[4], bool r1, bool r2, const float sc[4],
                                                 const Payload& q, const int lc[3], float dx) {
  const float chb[4] = {q.mv[0], q.mv[1], q.mv[2], q.m};
  float bs[4], as[4][3];
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    bs[s] = sel4(r1, r2, chb[s & 3], chb[(s + 1) & 3], chb[(s + 2) & 3], chb[(s + 3) & 3]) * sc[s];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const float ca[4] = {q.A[c], q.A[3 + c], q.A[6 + c], 0.0f};
      as[s][c] = sel4(r1, r2, ca[s & 3], ca[(s + 1) & 3], ca[(s + 2) & 3], ca[(s + 3) & 3]) * sc[s];
    }
  }
  float w[3][3], dxs[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const float t0 = 1.5f - q.f[a], t1 = q.f[a] - 1.0f, t2 = q.f[a] - 0.5f;
    w[a][0] = 0.5f * (t0 * t0);
    w[a][1] = 0.75f - t1 * t1;
    w[a][2] = 0.5f * (t2 * t2);
#pragma unroll
    for (int o = 0; o < 3; ++o) dxs[a][o] = ((float)o - q.f[a]) * dx;
  }
  const int base = (lc[0] * TILE + lc[1]) * TILE_Z + lc[2];
#pragma unroll
  for (int ii = 0; ii < 3; ++ii) {
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const float wij = w[0][ii] * w[1][j];
      float bij[4];
#pragma unroll
      for (int s = 0; s < 4; ++s) bij[s] = bs[s] + as[s][0] * dxs[0][ii] + as[s][1] * dxs[1][j];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const float wt = wij * w[2][k];
        int* t = tile + base + (ii * TILE + j) * TILE_Z + k;
#pragma unroll
        for (int s = 0; s < 4; ++s) atomicAdd(t + off[s], fixq(wt, bij[s] + as[s][2] * dxs[2][k]));
      }
    }
  }
}

// Rotate a 4-vector left by rot = r1 + 2 r2 (v'[s] = v[(s + rot) & 3]) in two
// select stages: 8 FSEL instead of 12 for the 4-way select per element.
__device__ __forceinline__ void rot4(bool r1, bool r2, float v[4]) {
  const float a0 = r2 ? v[2] : v[0], a1 = r2 ? v[3] : v[1], a2 = r2 ? v[0] : v[2], a3 = r2 ? v[1] : v[3];
  v[0] = r1 ? a1 : a0;
  v[1] = r1 ? a2 : a1;
  v[2] = r1 ? a3 : a2;
  v[3] = r1 ? a0 : a3;
}

// Packed P2G scatter of one particle into the int32 tile (the fused kernel's
// hot loop).  Channel c of node (i, j, k) receives
//   w0_i w1_j w2_k (b_c + A_c . dp) S_c
// = w2_k alpha_ij,c + (w2_k dz_k) beta_ij,c,
//   alpha_ij = w0_i w1_j (b + A_x dx_i + A_y dy_j) S,  beta_ij = w0_i w1_j A_z S,
// evaluated as FFMA2(w2_k, alpha, FFMA2(w2_k dz_k, beta, MAGIC)) over channel
// pairs: 2 FFMA2 + 2 (IADD + ATOMS) per node and channel pair, instead of 6
// scalar FFMA / FMUL + 2 (IADD + ATOMS).  Both products round onto the integer
// grid of the magic constant (<= 1 unit of 1/S per contribution; every partial
// term is bounded by the channel bound like the full term, so the magic range
// holds).  Slots are rotated by the particle's rank in its cell (rot): slot s
// carries channel (s + rot) & 3 at tile + off[s].
__device__ __forceinline__ void tile_scatter_pk(int* tile, const int off[4], bool r1, bool r2, const float S[4],
                                                const Payload& q, const int lc[3], float dx) {
  // channel values scaled, then rotated into slots
  float bs[4] = {q.mv[0] * S[0], q.mv[1] * S[1], q.mv[2] * S[2], q.m * S[3]};
  float ax[4] = {q.A[0] * S[0], q.A[3] * S[1], q.A[6] * S[2], 0.0f};
  float ay[4] = {q.A[1] * S[0], q.A[4] * S[1], q.A[7] * S[2], 0.0f};
  float az[4] = {q.A[2] * S[0], q.A[5] * S[1], q.A[8] * S[2], 0.0f};
  rot4(r1, r2, bs);
  rot4(r1, r2, ax);
  rot4(r1, r2, ay);
  rot4(r1, r2, az);
  float w[3][3], dxs[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const float t0 = 1.5f - q.f[a], t1 = q.f[a] - 1.0f, t2 = q.f[a] - 0.5f;
    w[a][0] = 0.5f * (t0 * t0);
    w[a][1] = 0.75f - t1 * t1;
    w[a][2] = 0.5f * (t2 * t2);
#pragma unroll
    for (int o = 0; o < 3; ++o) dxs[a][o] = ((float)o - q.f[a]) * dx;
  }
  float wdz[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) wdz[k] = w[2][k] * dxs[2][k];
  const f2p b01 = f2_pack(bs[0], bs[1]), b23 = f2_pack(bs[2], bs[3]);
  const f2p ax01 = f2_pack(ax[0], ax[1]), ax23 = f2_pack(ax[2], ax[3]);
  const f2p ay01 = f2_pack(ay[0], ay[1]), ay23 = f2_pack(ay[2], ay[3]);
  const f2p az01 = f2_pack(az[0], az[1]), az23 = f2_pack(az[2], az[3]);
  const f2p mm = f2_bc(MAGIC);
#ifdef EXP_SCATTER_NOCONF  // timing experiment: conflict-free (wrong) addresses
  int* t0 = tile + (threadIdx.x & 31) + off[0];
#else
  int* t0 = tile + ((lc[0] * TILE + lc[1]) * TILE_Z + lc[2]) + off[0];
#endif
  int* t1 = t0 - off[0] + off[1];
  int* t2 = t0 - off[0] + off[2];
  int* t3 = t0 - off[0] + off[3];
#pragma unroll
  for (int ii = 0; ii < 3; ++ii) {
    const f2p bx01 = f2_fma(f2_bc(dxs[0][ii]), ax01, b01);
    const f2p bx23 = f2_fma(f2_bc(dxs[0][ii]), ax23, b23);
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const f2p wij = f2_bc(w[0][ii] * w[1][j]);
      const f2p al01 = f2_mul(wij, f2_fma(f2_bc(dxs[1][j]), ay01, bx01));
      const f2p al23 = f2_mul(wij, f2_fma(f2_bc(dxs[1][j]), ay23, bx23));
      const f2p be01 = f2_mul(wij, az01);
      const f2p be23 = f2_mul(wij, az23);
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const f2p v01 = f2_fma(f2_bc(w[2][k]), al01, f2_fma(f2_bc(wdz[k]), be01, mm));
        const f2p v23 = f2_fma(f2_bc(w[2][k]), al23, f2_fma(f2_bc(wdz[k]), be23, mm));
        const int o = (ii * TILE + j) * TILE_Z + k;
#ifdef EXP_SCATTER_STS  // timing experiment: plain stores instead of atomics
        t0[o] = __float_as_int(f2_lo(v01)) - MAGIC_BITS;
        t1[o] = __float_as_int(f2_hi(v01)) - MAGIC_BITS;
        t2[o] = __float_as_int(f2_lo(v23)) - MAGIC_BITS;
        t3[o] = __float_as_int(f2_hi(v23)) - MAGIC_BITS;
#else
        atomicAdd(t0 + o, __float_as_int(f2_lo(v01)) - MAGIC_BITS);
        atomicAdd(t1 + o, __float_as_int(f2_hi(v01)) - MAGIC_BITS);
        atomicAdd(t2 + o, __float_as_int(f2_lo(v23)) - MAGIC_BITS);
        atomicAdd(t3 + o, __float_as_int(f2_hi(v23)) - MAGIC_BITS);
#endif
      }
    }
  }
}

// Flush an int32 fixed-point tile's node box [x0,x1]x[y0,y1]x[z0,z1] (tile
// coordinates) into gm: one REDG.F32x4 per non-empty node, the box re-zeroed,
// and every brick overlapping the box marked active.  The whole CTA shares the
// work as (x-segment of SEG nodes, y, z) units, z fastest so consecutive lanes
// hit consecutive float4s of a brick row; a segment's 4*SEG LDS are issued
// before any of its REDGs.  Box nodes are inside the grid by construction
// (bases are clamped to [0, res-3]), so there are no bounds checks.
template <int SEG>
__device__ __forceinline__ void flush_tile(const Params& p, int* tile, const int* org, int x0, int x1, int y0, int y1,
                                           int z0, int z1, const float inv[4], int* ccount) {
  if (x1 < x0 + 2) return;  // empty box (every particle fell back to gm)
  const int nx = x1 - x0 + 1, ny = y1 - y0 + 1, nz = z1 - z0 + 1;
  const int nyz = ny * nz, units = nyz * ((nx + SEG - 1) / SEG);
  const float rz = 1.0f / (float)nz, ryz = 1.0f / (float)nyz;  // exact quotients for u < 2^10
  const long long xstride = (long long)p.nb[1] * p.nb[2] * 64;
  for (int u = threadIdx.x; u < units; u += blockDim.x) {
    const int seg = (int)(((float)u + 0.5f) * ryz);
    const int r = u - seg * nyz;
    const int dy = (int)(((float)r + 0.5f) * rz);
    const int ty = y0 + dy, tz = z0 + r - dy * nz, xs = x0 + SEG * seg;
    const int gj = org[1] + ty, gk = org[2] + tz;
    const long long yz = ((long long)(gj >> BRICK_SHIFT) * p.nb[2] + (gk >> BRICK_SHIFT)) * 64 +
                         ((gj & 3) << 2) + (gk & 3);
    int4 a[SEG];
#pragma unroll
    for (int k = 0; k < SEG; ++k) {
      const int t = ((xs + k) * TILE + ty) * TILE_Z + tz;
      a[k] = xs + k <= x1 ? make_int4(tile[t], tile[TILE_NODES + t], tile[2 * TILE_NODES + t], tile[3 * TILE_NODES + t])
                          : make_int4(0, 0, 0, 0);
    }
#pragma unroll
    for (int k = 0; k < SEG; ++k) {
      if (xs + k > x1) continue;
      const int t = ((xs + k) * TILE + ty) * TILE_Z + tz;
      tile[t] = 0;
      tile[TILE_NODES + t] = 0;
      tile[2 * TILE_NODES + t] = 0;
      tile[3 * TILE_NODES + t] = 0;
      ccount[t] = 0;  // the box covers every counted cell (cells [x0, x1 - 2] ...)
    }
#pragma unroll
    for (int k = 0; k < SEG; ++k) {
#ifndef EXP_FREEZE
      if ((a[k].x | a[k].y | a[k].z | a[k].w) == 0) continue;
#endif
      const int gi = org[0] + xs + k;
      atomicAdd(p.gm + (gi >> BRICK_SHIFT) * xstride + yz + ((gi & 3) << 4),
                make_float4((float)a[k].x * inv[0], (float)a[k].y * inv[1], (float)a[k].z * inv[2],
                            (float)a[k].w * inv[3]));
    }
  }
  const int bx0 = (org[0] + x0) >> BRICK_SHIFT, by0 = (org[1] + y0) >> BRICK_SHIFT, bz0 = (org[2] + z0) >> BRICK_SHIFT;
  const int nbx = ((org[0] + x1) >> BRICK_SHIFT) - bx0 + 1, nby = ((org[1] + y1) >> BRICK_SHIFT) - by0 + 1,
            nbz = ((org[2] + z1) >> BRICK_SHIFT) - bz0 + 1;
  // brick (bx, by, bz) of unit t by float reciprocals (exact: t < 2^10)
  const float rbz = 1.0f / (float)nbz, rbyz = 1.0f / (float)(nby * nbz);
  for (int t = threadIdx.x; t < nbx * nby * nbz; t += blockDim.x) {
    const int bx = (int)(((float)t + 0.5f) * rbyz), r = t - bx * nby * nbz;
    const int by = (int)(((float)r + 0.5f) * rbz), bz = r - by * nbz;
    mark_brick(p, ((long long)((bx0 + bx) * p.nb[1] + by0 + by) * p.nb[2] + bz0 + bz) << 6);
  }
}

// Stage B: P2G of one work item (<= CHUNK particles, cell-sorted) into an int32
// fixed-point shared-memory tile (fp32 atomicAdd on shared memory is a CAS loop
// on sm_100a; int32 ATOMS.ADD is native).  Each channel's power-of-two scale
// comes from the item's exact bound (channel_scale: no contribution leaves the
// FFMA magic range and no node sum can leave int32).  Particles whose stencil
// leaves the tile go straight to gm with float REDG.F32x4.  The flush walks
// only the touched node box, rescales exactly, issues one REDG.F32x4 per
// non-empty node, re-zeroes the tile, marks the box's 4^3 bricks active
// (flush_tile) and records the box for the next
// substep's G2P tile.  Two barriers per item.
__global__ void __launch_bounds__(P2G_THREADS, P2G_MIN_BLOCKS) p2g_tile_kernel(Params p, const float* __restrict__ pay,
                                                                               const float4* __restrict__ bounds,
                                                                               int* __restrict__ item_box) {
  extern __shared__ int tile[];  // SoA: 4 x TILE_NODES int32 channels (mv x, y, z, m) + per-cell counts
  int* ccount = tile + 4 * TILE_NODES;
  __shared__ int boxes[2][6];  // double-buffered by item parity: reset one while the other is live
  __shared__ float scale_s[4];
  const int nwork = *p.nwork;
  unsigned guard = 0;
  for (int t = threadIdx.x; t < 5 * TILE_NODES; t += blockDim.x) tile[t] = 0;
  if (threadIdx.x < 12) boxes[threadIdx.x / 6][threadIdx.x % 6] = (threadIdx.x % 6) < 3 ? TILE : -1;
  const int rot = threadIdx.x & 3;
  const bool r1 = rot & 1, r2 = rot & 2;
  int off[4];
#pragma unroll
  for (int s = 0; s < 4; ++s) off[s] = ((s + rot) & 3) * TILE_NODES;
  int par = 0;
  for (int wi = blockIdx.x; wi < nwork; wi += gridDim.x, par ^= 1) {
    int* box = boxes[par];
    const int4 item = p.work[wi];
    const int bin = item.x;
    int bx, by, bz;
    bin_coords(p, bin, bx, by, bz);
    const int org[3] = {bx * BIN - MARGIN, by * BIN - MARGIN, bz * BIN - MARGIN};
    // previous item's box (its flush ended before the last barrier)
    if (threadIdx.x < 6) boxes[par ^ 1][threadIdx.x] = threadIdx.x < 3 ? TILE : -1;
    if (threadIdx.x < 4) {
      const float4 bd = bounds[wi];
      const int c = threadIdx.x;
      scale_s[c] = channel_scale(c == 0 ? bd.x : c == 1 ? bd.y : c == 2 ? bd.z : bd.w, item.w, p.fx_shift);
    }
    __syncthreads();
    const float S[4] = {scale_s[0], scale_s[1], scale_s[2], scale_s[3]};
    float sc[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) sc[s] = sel4(r1, r2, S[s & 3], S[(s + 1) & 3], S[(s + 2) & 3], S[(s + 3) & 3]);
    int lo_c[3] = {TILE, TILE, TILE}, hi_c[3] = {-1, -1, -1};
    for (long long i = (long long)item.y + threadIdx.x; i < item.z; i += blockDim.x) {
      Payload q;
      int lc[3];
      bool fits = true;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const float g = ldf(p, FX + a, i) * p.inv_dx;
        int bb = (int)floorf(g - 0.5f);
        bb = max(0, min(bb, p.res[a] - 3));
        q.b[a] = bb;
        q.f[a] = g - (float)bb;
        lc[a] = bb - org[a];
        fits &= (lc[a] >= 0) && (lc[a] <= TILE - 3);
        q.mv[a] = pay[a * p.cap + i];
      }
#pragma unroll
      for (int r = 0; r < 9; ++r) q.A[r] = pay[(3 + r) * p.cap + i];
      q.m = pay[12 * p.cap + i];
      if (fits) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          lo_c[a] = min(lo_c[a], lc[a]);
          hi_c[a] = max(hi_c[a], lc[a]);
        }
        // overflow guard: the cell's particle count against the item's limit
        fits = atomicAdd(&ccount[(lc[0] * TILE + lc[1]) * TILE_Z + lc[2]], 1) < cell_limit(item.w, p.fx_shift);
        guard += !fits;
      }
      if (fits) {
        tile_scatter_rot(tile, off, r1, r2, sc, q, lc, p.dx);
      } else {
        const float one[4] = {1.f, 1.f, 1.f, 1.f};
        p2g_scatter<false>(p, tile, org, q, one);
      }
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int l = __reduce_min_sync(0xffffffffu, lo_c[a]);
      const int h = __reduce_max_sync(0xffffffffu, hi_c[a]);
      if ((threadIdx.x & 31) == 0) {
        atomicMin(&box[a], l);
        atomicMax(&box[3 + a], h);
      }
    }
    __syncthreads();
    const int x0 = box[0], x1 = box[3] + 2, y0 = box[1], y1 = box[4] + 2, z0 = box[2], z1 = box[5] + 2;
    if (threadIdx.x == 0) {
      // empty box (all particles fell back to gm) encodes lo = 15 > hi
      item_box[wi] = x1 - 2 < x0 ? 0x00000FFF
                                 : (x0 | (y0 << 4) | (z0 << 8) | ((x1 - 2) << 12) | ((y1 - 2) << 16) | ((z1 - 2) << 20));
    }
    const float inv[4] = {1.0f / S[0], 1.0f / S[1], 1.0f / S[2], 1.0f / S[3]};
    flush_tile<2>(p, tile, org, x0, x1, y0, y1, z0, z1, inv, ccount);
    __syncthreads();
  }
  warp_count_add(p.stats, guard);
}

// Fused steady-state substep: G2P(n) -> advect -> F update -> stress -> P2G(n+1)
// in one pass per work item, with no payload round trip (the per-substep
// working set x, F, m, V0 + grid stays L2-resident).  The G2P reads the
// shared-memory velocity tile of the node box the item scattered to in the
// previous substep; the P2G scatters cell-rank-rotated channels into the int32
// fixed-point tile whose scales come from the item's bounds in the previous
// substep (x BOUND_SAFETY for momentum, exact for mass).  A particle that
// exceeds those bounds or leaves the tile is scattered with float REDG.F32x4
// into gm directly.  The item's exact new bounds (bounds_out, zeroed before
// the launch) and node box are recorded for the next substep.
constexpr float BOUND_SAFETY = 2.0f;

// Decode a work item: tile origin and the velocity-tile box (the base cells it
// scattered from in the previous substep, item_box).
__device__ __forceinline__ void fused_item_geometry(const Params& p, const int4 item, int packed_box, TileVel& tv) {
  const int bin = item.x;
  int bx, by, bz;
  bin_coords(p, bin, bx, by, bz);
  tv.org[0] = bx * BIN - MARGIN;
  tv.org[1] = by * BIN - MARGIN;
  tv.org[2] = bz * BIN - MARGIN;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    tv.lo[a] = (packed_box >> (4 * a)) & 15;
    tv.hi[a] = (packed_box >> (12 + 4 * a)) & 15;
  }
}

// Start the (asynchronous) fill of an item's velocity tile; the caller waits
// with cp_async_wait_all before the barrier that publishes it.
__device__ __forceinline__ void fused_item_vtile_issue(const Params& p, const TileVel& tv, float* vtile) {
  if (tv.lo[0] > tv.hi[0]) return;
  const long long xstride = (long long)p.nb[1] * p.nb[2] * 64;
  for (int c = threadIdx.x; c < 256; c += blockDim.x) {
    const int ty = tv.lo[1] + (c >> 4), tz = tv.lo[2] + (c & 15);
    const int gj = tv.org[1] + ty, gk = tv.org[2] + tz;
    if (ty <= tv.hi[1] + 2 && tz <= tv.hi[2] + 2 && gj < p.res[1] && gk < p.res[2]) {
      const long long yz = ((long long)(gj >> BRICK_SHIFT) * p.nb[2] + (gk >> BRICK_SHIFT)) * 64 +
                           ((gj & 3) << 2) + (gk & 3);
      load_vtile_column_async(p, vtile, tv.org[0], tv.lo[0], tv.hi[0] + 2, ty, tz, yz, xstride);
    }
  }
}

// An item's channel scales (threads 0..3).
__device__ __forceinline__ void fused_item_scales(const int4 item, const float4 bd, float* scale_slot, int fx_shift) {
  if (threadIdx.x < 4) {
    const int c = threadIdx.x;
    const float b = c == 0 ? bd.x * BOUND_SAFETY : c == 1 ? bd.y * BOUND_SAFETY : c == 2 ? bd.z * BOUND_SAFETY : bd.w;
    scale_slot[c] = channel_scale(b, item.w, fx_shift);
  }
}

#ifdef FUSED_PROFILE
__device__ __forceinline__ long long fprof_clock() {
  long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)::"memory");
  return t;
}
__device__ __forceinline__ long long fprof_clock_dep(int dep) {
  if (dep == 0x7fffffff) __trap();  // the branch waits for dep (a shared load behind the barrier)
  return fprof_clock();
}
#define FPROF_MARK(v) const long long v = fprof_clock()
#define FPROF_MARK_DEP(v, d) const long long v = fprof_clock_dep(d)
#else
#define FPROF_MARK(v)
#define FPROF_MARK_DEP(v, d)
#endif

// Fused steady-state kernel, two barriers per item: [B] after the scatter
// (tile complete) and [A] after the flush of this item overlapped with the
// velocity-tile load of the CTA's next item (disjoint shared-memory regions).
// The fused steady-state substep as a CTA-level phase (used by fused_kernel
// and, once per substep, by the cooperative substeps_kernel).  zero_tile:
// the int32 tile is cleared first (the flushes leave it clean afterwards).
template <bool SINGLE>
__device__ __forceinline__ void fused_phase(const Params& p, float4* __restrict__ bounds_in,
                                            float4* __restrict__ bounds_out, int* __restrict__ item_box,
                                            bool zero_tile, bool dep_wait = false) {
  extern __shared__ float smem[];
  float* vtile = smem;                                           // 3 x TILE_NODES
  int* tile = reinterpret_cast<int*>(smem + 3 * TILE_NODES);     // 4 x TILE_NODES
  int* ccount = tile + 4 * TILE_NODES;                           // per-cell counts (overflow guard)
  __shared__ int boxes[2][6];
  __shared__ float scale_s[2][4];
  __shared__ int4 nxt_item;
  __shared__ int nxt_box;
  __shared__ float4 nxt_bounds;
  __shared__ int nxt_wi;
  const int nwork = *p.nwork;
  if (zero_tile)
    for (int t = threadIdx.x; t < 5 * TILE_NODES; t += blockDim.x) tile[t] = 0;
  if (threadIdx.x < 12) boxes[threadIdx.x / 6][threadIdx.x % 6] = (threadIdx.x % 6) < 3 ? TILE : -1;
  unsigned inverted = 0, guard = 0;
  int par = 0;
  // dynamic scheduling over the size-sorted work list: the first gridDim.x
  // items are taken in launch order, later ones from the counter
  // (work list, item boxes and bounds come from launches before the grid op:
  // read before the dependency wait; grid velocities, gm, counters after it)
  if (blockIdx.x < nwork) {
    TileVel tv0;
    const int4 it0 = p.work[blockIdx.x];
    fused_item_geometry(p, it0, item_box[blockIdx.x], tv0);
    if (dep_wait) griddep_wait();
    fused_item_vtile_issue(p, tv0, vtile);
    fused_item_scales(it0, bounds_in[blockIdx.x], scale_s[0], p.fx_shift);
    cp_async_wait_all();
  } else if (dep_wait) {
    griddep_wait();
  }
  if (dep_wait) griddep_trigger();
  __syncthreads();  // [A] first velocity tile + scales ready
#ifdef FUSED_PROFILE
  unsigned long long pr[5] = {0, 0, 0, 0, 0};
  long long tA = fprof_clock();
#endif
  for (int wi = blockIdx.x; wi < nwork; par ^= 1) {
    int* box = boxes[par];
    const int4 item = p.work[wi];
    TileVel tv;
    tv.t = vtile;
    fused_item_geometry(p, item, item_box[wi], tv);
    if (threadIdx.x == 32) {  // next item (claimed now) and its descriptor, read after [B]
      const int nxt = gridDim.x + atomicAdd(p.work_next, 1);
      nxt_wi = nxt;
      if (nxt < nwork) {
        nxt_item = p.work[nxt];
        nxt_box = item_box[nxt];
        nxt_bounds = bounds_in[nxt];
      }
    }
    const int* org = tv.org;
    const float4 bd = bounds_in[wi];
    const float B[4] = {bd.x * BOUND_SAFETY, bd.y * BOUND_SAFETY, bd.z * BOUND_SAFETY, bd.w};
    // previous item's box buffer (its flush ended before the last [A])
    if (threadIdx.x < 6) boxes[par ^ 1][threadIdx.x] = threadIdx.x < 3 ? TILE : -1;
    const float S[4] = {scale_s[par][0], scale_s[par][1], scale_s[par][2], scale_s[par][3]};
    float mx[4] = {0.f, 0.f, 0.f, 0.f};
    int lo_c[3] = {TILE, TILE, TILE}, hi_c[3] = {-1, -1, -1};
    const int climit = cell_limit(item.w, p.fx_shift);
    for (long long i = (long long)item.y + threadIdx.x; i < item.z; i += blockDim.x) {
      PRaw<true> r;
      load_raw<true>(p, i, r);
      Payload q;
      const float det = compute_payload<true, true, SINGLE>(p, i, r, q, &tv);
      inverted += det <= 0.0f;
      float bnd[4];
      payload_bound(p, q, bnd);
      bool fits = true;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        mx[c] = fmaxf(mx[c], bnd[c]);
        fits &= bnd[c] <= B[c];
      }
#ifdef FUSED_PROFILE
      const bool bound_ok = fits;
#endif
      int lc[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        lc[a] = q.b[a] - org[a];
        fits &= (lc[a] >= 0) && (lc[a] <= TILE - 3);
      }
      FPROF_COUNT(0);
      if (fits) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          lo_c[a] = min(lo_c[a], lc[a]);
          hi_c[a] = max(hi_c[a], lc[a]);
        }
        // overflow guard: the cell's particle count against the item's limit
        fits = atomicAdd(&ccount[(lc[0] * TILE + lc[1]) * TILE_Z + lc[2]], 1) < climit;
        guard += !fits;
      }
      if (!fits) {
        FPROF_COUNT(2);
#ifdef FUSED_PROFILE
        if (!bound_ok) FPROF_COUNT(3);
#endif
        const float one[4] = {1.f, 1.f, 1.f, 1.f};
        p2g_scatter<false>(p, tile, org, q, one);
        continue;
      }
      {
        // rotate the channel order by the particle's rank among this round's
        // lanes in the same base cell: the first particle of every cell
        // writes channel s at step s, so different cells of a warp row spread
        // over consecutive banks and same-cell lanes over channel planes
        const unsigned grp = __match_any_sync(__activemask(), (lc[0] * TILE + lc[1]) * TILE + lc[2]);
        const int crot = __popc(grp & ((1u << (threadIdx.x & 31)) - 1u)) & 3;
        const bool c1 = crot & 1, c2 = crot & 2;
        int coff[4];
#pragma unroll
        for (int s2 = 0; s2 < 4; ++s2) coff[s2] = ((s2 + crot) & 3) * TILE_NODES;
#ifndef EXP_NO_SCATTER
        tile_scatter_pk(tile, coff, c1, c2, S, q, lc, p.dx);
#endif
      }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const unsigned u = __reduce_max_sync(0xffffffffu, __float_as_uint(mx[c]));
      if ((threadIdx.x & 31) == 0 && u) atomicMax(reinterpret_cast<unsigned*>(bounds_out + wi) + c, u);
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int l = __reduce_min_sync(0xffffffffu, lo_c[a]);
      const int h = __reduce_max_sync(0xffffffffu, hi_c[a]);
      if ((threadIdx.x & 31) == 0) {
        atomicMin(&box[a], l);
        atomicMax(&box[3 + a], h);
      }
    }
    FPROF_MARK(tb0);
    __syncthreads();  // [B] scatter complete; velocity tile free
    FPROF_MARK_DEP(tb1, *(volatile int*)&boxes[par][0]);
    const int x0 = box[0], x1 = box[3] + 2, y0 = box[1], y1 = box[4] + 2, z0 = box[2], z1 = box[5] + 2;
    if (threadIdx.x == 0) {
      item_box[wi] = x1 - 2 < x0 ? 0x00000FFF
                                 : (x0 | (y0 << 4) | (z0 << 8) | ((x1 - 2) << 12) | ((y1 - 2) << 16) | ((z1 - 2) << 20));
      bounds_in[wi] = make_float4(0.f, 0.f, 0.f, 0.f);  // consumed: zero for its next use as bounds_out
    }
    // the CTA's next item: velocity-tile copies issued before the flush so
    // their L2 latency hides under it
    const int wnext = nxt_wi;
    const bool has_next = wnext < nwork;
    int4 itn;
    if (has_next) {
      TileVel tn;
      itn = nxt_item;
      fused_item_geometry(p, itn, nxt_box, tn);
      fused_item_vtile_issue(p, tn, vtile);
    }
#ifdef EXP_FREEZE  // timing experiments: the flush adds zeros (particles stay put)
    const float inv[4] = {0.f, 0.f, 0.f, 0.f};
#else
    const float inv[4] = {1.0f / S[0], 1.0f / S[1], 1.0f / S[2], 1.0f / S[3]};
#endif
#ifndef MPM_FLUSH_SEG
#define MPM_FLUSH_SEG 4
#endif
    flush_tile<MPM_FLUSH_SEG>(p, tile, org, x0, x1, y0, y1, z0, z1, inv, ccount);
    FPROF_MARK(tf);
    if (has_next) fused_item_scales(itn, nxt_bounds, scale_s[par ^ 1], p.fx_shift);
    cp_async_wait_all();
    FPROF_MARK(ta0);
    __syncthreads();  // [A] flush complete (tile zero), next velocity tile ready
    wi = wnext;
#ifdef FUSED_PROFILE
    {
      const long long ta1 = fprof_clock_dep(*(volatile int*)&scale_s[par ^ 1][0]);
      pr[0] += tb0 - tA; pr[1] += tb1 - tb0; pr[2] += tf - tb1; pr[3] += ta0 - tf; pr[4] += ta1 - ta0;
      tA = ta1;
    }
#endif
  }
#ifdef FUSED_PROFILE
  if ((threadIdx.x & 31) == 0)
    for (int k = 0; k < 5; ++k) atomicAdd(&g_fprof[k], pr[k]);
  if (threadIdx.x == 0) atomicAdd(&g_fprof[5], 1ull);
#endif
  warp_count_add(p.inverted, inverted);
  warp_count_add(p.stats, guard);
}

template <bool SINGLE>
__global__ void __launch_bounds__(FUSED_K_THREADS, FUSED_MIN_BLOCKS) fused_kernel(Params p, float4* __restrict__ bounds_in,
                                                                                  float4* __restrict__ bounds_out,
                                                                                  int* __restrict__ item_box) {
#ifdef FUSED_PROFILE
  const unsigned long long t0 = gtimer();
  if (threadIdx.x == 0) atomicMin(&g_bub[2], t0);
#endif
  fused_phase<SINGLE>(p, bounds_in, bounds_out, item_box, true, true);
#ifdef FUSED_PROFILE
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long t_end = gtimer();
    atomicAdd(&g_fwin[2], t_end - t0);
    atomicAdd(&g_fwin[3], 1ull);
    atomicMax(&g_bub[0], t_end);
    if (atomicAdd(&g_bub[3], 1ull) == gridDim.x - 1) {
      const unsigned long long st = atomicExch(&g_bub[2], ~0ull), ge = g_bub[1];
      atomicAdd(&g_fwin[0], gtimer() - st);
      atomicAdd(&g_fwin[1], 1ull);
      if (ge && st > ge && st - ge < 50000ull) {
        atomicAdd(&g_bub[6], st - ge);
        atomicAdd(&g_bub[7], 1ull);
      }
      g_bub[3] = 0;
    }
  }
#endif
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

// Final G2P of a fast-path stretch, one work item at a time: the item's
// velocity tile (the node box its particles scattered to in the stretch's
// last substep, item_box) is staged in shared memory with LDGSTS and the
// gathers read it (the global grid for a particle outside it), then advect
// and x / v / C.  Same sums in the same order as g2p_kernel.
template <bool SINGLE>
__global__ void __launch_bounds__(256) g2p_tile_kernel(Params p, const int* __restrict__ item_box) {
  extern __shared__ float smem[];
  const int nwork = *p.nwork;
  for (int wi = blockIdx.x; wi < nwork; wi += gridDim.x) {
    const int4 item = p.work[wi];
    TileVel tv;
    tv.t = smem;
    fused_item_geometry(p, item, item_box[wi], tv);
    __syncthreads();  // the previous item's gathers are done with the tile
    fused_item_vtile_issue(p, tv, smem);
    cp_async_wait_all();
    __syncthreads();
    for (long long i = (long long)item.y + threadIdx.x; i < item.z; i += blockDim.x) {
      float x[3] = {ldf(p, FX, i), ldf(p, FX + 1, i), ldf(p, FX + 2, i)};
      int b[3];
      float f[3], w[3][3];
      bool in_tile = true;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        stencil(x[a], p.inv_dx, p.res[a], b[a], f[a], w[a]);
        in_tile &= (b[a] - tv.org[a] >= tv.lo[a]) && (b[a] - tv.org[a] <= tv.hi[a]);
      }
      float v[3], C[9];
      if (in_tile)
        g2p_gather_pk(p, tv, b, f, w, v, C);
      else
        g2p_gather(p, global_vel(p), b, f, w, v, C);
      advect<SINGLE>(p, x, v);
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        stf(p, FX + a, i, x[a]);
        stf(p, FV + a, i, v[a]);
      }
#pragma unroll
      for (int q = 0; q < 9; ++q) stf(p, FC + q, i, C[q]);
    }
  }
}

// Exact fp64 field + contact response at one massive node inside the fp32
// prefilter band.  Out of line: only a few percent of the nodes get here, and
// keeping its fp64 register footprint out of grid_op_kernel lets 4 CTAs of
// the streaming path reside per SM.
__device__ __noinline__ float3 grid_contact(const Colliders cs, double cap, double wx, double wy, double wz, float v0,
                                            float v1, float v2) {
  double best;
#ifdef FUSED_PROFILE
  long long tq = clock64();
#endif
  const int ci = nearest_collider(cs, wx, wy, wz, cap, best);
  CPH_MARK(0, tq);
  if (best < cs.theta && ci >= 0) {
    double vv[3] = {v0, v1, v2};
    resolve_contact(cs, ci, wx, wy, wz, vv);
    CPH_MARK(3, tq);
    return make_float3((float)vv[0], (float)vv[1], (float)vv[2]);
  }
  return make_float3(v0, v1, v2);
}

// Grid op (kernels.py:347-436) over active bricks (or all bricks when DENSE):
// one warp per 4^3 brick, two nodes per lane (both loads in flight).
// Zero-mass nodes pass momentum through unchanged (kernels.py:364-365).
// Collider distances are exact fp64 (collide.cuh), but a node is only sent
// through them when the conservative fp32 far-field bound of some collider
// (collide.cuh: collider_far) is below theta + margin -- nodes the bound
// clears cannot be in contact, so results are unchanged.  When `clear`, gm
// is zeroed for the next P2G.
__device__ __forceinline__ float4 grid_node(const Params& p, const Colliders& cs_all, const ColliderNearF* nf,
                                            bool single_env, double cap, float4 a, int gi, int gj, int gk) {
  if (!(a.w > 0.0f) || gi >= p.res[0] || gj >= p.res[1] || gk >= p.res[2]) return a;
  // global node coordinates (slab window offset), environment tile, tile-local coordinates
  gi += p.goff[0];
  gj += p.goff[1];
  gk += p.goff[2];
  int li = gi, lj = gj, lk = gk;
  Colliders cs = cs_all;
  if (!single_env) {
    const int ei = (int)p.fd_env[0].div((unsigned)gi), ej = (int)p.fd_env[1].div((unsigned)gj),
              ek = (int)p.fd_env[2].div((unsigned)gk);
    cs = env_colliders(cs_all, ei, ej, ek);
    li = gi - ei * p.env_res[0];
    lj = gj - ej * p.env_res[1];
    lk = gk - ek * p.env_res[2];
  }
  const float inv_m = 1.0f / a.w;
  float v0 = a.x * inv_m + p.dt * p.gravity[0];
  float v1 = a.y * inv_m + p.dt * p.gravity[1];
  float v2 = a.z * inv_m + p.dt * p.gravity[2];
  if (cs.theta >= 0.0 && cs.count > 0) {
    const float fx = (float)gi * p.dx, fy = (float)gj * p.dx, fz = (float)gk * p.dx;
    bool near = false;
    if (nf) {
      for (int ci = 0; ci < cs.count; ++ci) near |= nf[ci].near(fx, fy, fz);
    } else {
      for (int ci = 0; ci < cs.count; ++ci) near |= collider_near(cs, ci, fx, fy, fz, cs.theta_f);
    }
    if (near) {
#ifdef FUSED_PROFILE
      const long long c0 = clock64();
#endif
      const float3 v = grid_contact(cs, cap, (double)gi * p.dx64, (double)gj * p.dx64, (double)gk * p.dx64, v0, v1, v2);
#ifdef FUSED_PROFILE
      const long long c1 = clock64();
      const unsigned m = __activemask();
      if ((int)(threadIdx.x & 31) == __ffs(m) - 1) {
        atomicAdd(&g_cprof[0], 1ull);
        atomicAdd(&g_cprof[1], (unsigned long long)__popc(m));
        atomicAdd(&g_cprof[2], (unsigned long long)(c1 - c0));
        atomicMax(&g_cprof[3], (unsigned long long)(c1 - c0));
      }
#endif
      v0 = v.x;
      v1 = v.y;
      v2 = v.z;
    }
  }
  const int bw = p.bwidth;
  const int rx = p.env_res[0], ry = p.env_res[1], rz = p.env_res[2];
  if (p.stick) {
    if (li < bw || li >= rx - bw || lj < bw || lj >= ry - bw || lk < bw || lk >= rz - bw) v0 = v1 = v2 = 0.0f;
  } else {
    if (li < bw && v0 < 0.0f) v0 = 0.0f;
    if (li >= rx - bw && v0 > 0.0f) v0 = 0.0f;
    if (lj < bw && v1 < 0.0f) v1 = 0.0f;
    if (lj >= ry - bw && v1 > 0.0f) v1 = 0.0f;
    if (lk < bw && v2 < 0.0f) v2 = 0.0f;
    if (lk >= rz - bw && v2 > 0.0f) v2 = 0.0f;
  }
  return make_float4(v0, v1, v2, a.w);
}

// The grid op as a CTA-level phase (grid_op_kernel, and once per substep in
// the cooperative substeps_kernel).
template <bool DENSE>
__device__ __forceinline__ void grid_phase(const Params& p, const Colliders& cs, int clear, bool dep_wait = false) {
  // one table for the whole grid: the fp32 prefilter boxes are staged in
  // shared memory once per CTA (per-environment tables use collider_near)
  __shared__ ColliderNearF nf_s[MAX_COLLIDERS];
  const bool staged = !cs.per_env && cs.theta >= 0.0 && cs.count > 0 && cs.count <= MAX_COLLIDERS;
  if (staged && threadIdx.x < cs.count) nf_s[threadIdx.x] = make_near_f(cs, threadIdx.x, cs.theta_f);
  // collider tables come from the host: staged before the dependency wait
  if (dep_wait) {
    griddep_wait();
    griddep_trigger();
  }
  const int lane = threadIdx.x & 31;
  const long long stride = (long long)gridDim.x * (blockDim.x >> 5);
  const long long first = (long long)(threadIdx.x >> 5) * gridDim.x + blockIdx.x;
  const long long nbt = (long long)p.nb[0] * p.nb[1] * p.nb[2];
  // the brick count and this warp's first 32 list entries are loaded
  // together (entries past the count are ignored): one dependent round trip
  // to the first momentum loads instead of two
  const long long spec_it = first + (long long)lane * stride;
  const int spec_b = !DENSE && spec_it < nbt ? p.active_list[spec_it] : 0;
  const long long nitems = DENSE ? nbt : (long long)*p.active_count;
  __syncthreads();
  const ColliderNearF* nf = staged ? nf_s : nullptr;
  const bool single_env = p.env_res[0] == p.gres[0] && p.env_res[1] == p.gres[1] && p.env_res[2] == p.gres[2];
  const double cap = 2.0 * cs.theta;
  const int lj = (lane >> 2) & 3, lk = lane & 3, li0 = lane >> 4;
  // this warp's bricks: first, first + stride, ... (strided so that the
  // expensive contact bricks, clustered in the list, spread over warps).
  // Their list entries are fetched 32 at a time (one per lane) and the
  // momentum of the brick after next is loaded while one is processed.
  // warp-major numbering (warp w of CTA c is w * gridDim + c): consecutive
  // list entries -- one item's bricks, e.g. a tool's contact band -- land in
  // different CTAs / SMs instead of the 8 warps of one CTA
  const long long nmine = nitems > first ? (nitems - first + stride - 1) / stride : 0;
  for (long long base = 0; base < nmine; base += 32) {
    const int cnt = (int)min(32LL, nmine - base);
    const long long my_it = first + (base + lane) * stride;
    const int myb = lane < cnt ? (DENSE ? (int)my_it : (base == 0 ? spec_b : p.active_list[my_it])) : 0;
    long long b0 = __shfl_sync(0xffffffffu, myb, 0), b1 = __shfl_sync(0xffffffffu, myb, cnt > 1 ? 1 : 0);
    float4 a00 = p.gm[(b0 << 6) | lane], a01 = p.gm[((b0 << 6) | lane) + 32];
    float4 a10 = a00, a11 = a01;
    if (cnt > 1) {
      a10 = p.gm[(b1 << 6) | lane];
      a11 = p.gm[((b1 << 6) | lane) + 32];
    }
    for (int k = 0; k < cnt; ++k) {
      long long b2 = b1;
      float4 a20 = a10, a21 = a11;
      if (k + 2 < cnt) {
        b2 = __shfl_sync(0xffffffffu, myb, k + 2);
        a20 = p.gm[(b2 << 6) | lane];
        a21 = p.gm[((b2 << 6) | lane) + 32];
      }
      const unsigned t12 = p.fd_nb2.div((unsigned)b0);
      const int bk = (int)((unsigned)b0 - t12 * p.nb[2]);
      const int bi = (int)p.fd_nb1.div(t12), bj = (int)t12 - bi * p.nb[1];
      const long long i0 = (b0 << 6) | lane, i1 = i0 + 32;
      const float4 o0 = grid_node(p, cs, nf, single_env, cap, a00, bi * 4 + li0, bj * 4 + lj, bk * 4 + lk);
      const float4 o1 = grid_node(p, cs, nf, single_env, cap, a01, bi * 4 + li0 + 2, bj * 4 + lj, bk * 4 + lk);
      p.gv[i0] = o0;
      p.gv[i1] = o1;
      if (clear) {
        p.gm[i0] = make_float4(0.f, 0.f, 0.f, 0.f);
        p.gm[i1] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      if (lane == 0) p.brick_flag[b0] = 0;
      b0 = b1;
      a00 = a10;
      a01 = a11;
      b1 = b2;
      a10 = a20;
      a11 = a21;
    }
  }
}

template <bool DENSE>
__global__ void __launch_bounds__(256, GRIDOP_MIN_BLOCKS) grid_op_kernel(Params p, Colliders cs, int clear, int* done) {
#ifdef FUSED_PROFILE
  unsigned long long g_t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_t0));
#endif
  grid_phase<DENSE>(p, cs, clear, true);
#ifdef FUSED_PROFILE
  {
    __syncthreads();
    unsigned long long g_t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_t1));
    if (threadIdx.x == 0) {
      if (done) {  // window accounting over clearing launches only (reset by their last CTA)
        atomicMin(&g_gwin[0], g_t0);
        atomicMax(&g_gwin[1], g_t1);
        atomicMax(&g_gwin[3], g_t0);
      }
      atomicAdd(&g_gprof[0], g_t1 - g_t0);
      atomicMax(&g_gprof[1], g_t1 - g_t0);
      atomicAdd(&g_gprof[2], 1ull);
      if (blockIdx.x == 0) atomicAdd(&g_gprof[3], 1ull);
    }
  }
#endif
  // clearing launch of the fast path: the last CTA out zeroes the brick-list
  // and work-item counters for the next substep (no memset nodes per substep)
  if (done) {
    __syncthreads();
    // (every CTA read the counters before its increment; the next launch
    // sees the reset across the kernel boundary: no fences needed)
    if (threadIdx.x == 0) {
      if (atomicAdd(done, 1) == (int)gridDim.x - 1) {
#ifdef FUSED_PROFILE
        atomicAdd(&g_gprof[4], atomicExch(&g_gprof[1], 0ull));
        atomicAdd(&g_gprof[5], 1ull);
        atomicAdd(&g_gprof[6], (unsigned long long)*p.active_count);
        {
          const unsigned long long fe = g_bub[0];
          if (fe && g_gwin[0] > fe && g_gwin[0] - fe < 50000ull) {  // same substep only
            atomicAdd(&g_bub[4], g_gwin[0] - fe);
            atomicAdd(&g_bub[5], 1ull);
          }
          atomicMax(&g_bub[1], gtimer());
        }
        {
          const unsigned long long a = atomicExch(&g_gwin[0], ~0ull), b = atomicExch(&g_gwin[1], 0ull);
          const unsigned long long c = atomicExch(&g_gwin[3], 0ull);
          atomicAdd(&g_gwin[2], ((b - a) << 20) | min(c - a, (1ull << 20) - 1));  // window ns (hi), start spread ns (lo)
        }
#endif
        *p.active_count = 0;
        *p.work_next = 0;
        *done = 0;
      }
    }
  }
}

// Grid op, plain form: one warp per active brick (two nodes per lane), no
// software prefetch pipeline (2 CTAs of 8 warps per SM, the fp64 contact
// chain out of line).  Same node math
// (grid_node) and the same last-CTA counter reset as grid_op_kernel.
#ifndef MPM_GRIDOP_SIMPLE_MINB
#define MPM_GRIDOP_SIMPLE_MINB 2
#endif
__global__ void __launch_bounds__(256, MPM_GRIDOP_SIMPLE_MINB)
    grid_op_simple_kernel(Params p, Colliders cs, int clear, int* done) {
  __shared__ ColliderNearF nf_s[MAX_COLLIDERS];
  const bool staged = !cs.per_env && cs.theta >= 0.0 && cs.count > 0 && cs.count <= MAX_COLLIDERS;
  if (staged && threadIdx.x < cs.count) nf_s[threadIdx.x] = make_near_f(cs, threadIdx.x, cs.theta_f);
  // collider tables come from the host: staged before the dependency wait (a
  // no-op unless launched with programmatic dependent launch)
  griddep_wait();
  griddep_trigger();
  const int lane = threadIdx.x & 31;
  const long long nitems = *p.active_count;
  __syncthreads();
  const ColliderNearF* nf = staged ? nf_s : nullptr;
  const bool single_env = p.env_res[0] == p.gres[0] && p.env_res[1] == p.gres[1] && p.env_res[2] == p.gres[2];
  const double cap = 2.0 * cs.theta;
  const int lj = (lane >> 2) & 3, lk = lane & 3, li0 = lane >> 4;
  const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long it = (long long)(threadIdx.x >> 5) * gridDim.x + blockIdx.x; it < nitems; it += nw) {
    const long long b = p.active_list[it];
    const long long i0 = (b << 6) | lane, i1 = i0 + 32;
    const float4 a0 = p.gm[i0], a1 = p.gm[i1];
    const unsigned t12 = p.fd_nb2.div((unsigned)b);
    const int bk = (int)((unsigned)b - t12 * p.nb[2]);
    const int bi = (int)p.fd_nb1.div(t12), bj = (int)t12 - bi * p.nb[1];
    p.gv[i0] = grid_node(p, cs, nf, single_env, cap, a0, bi * 4 + li0, bj * 4 + lj, bk * 4 + lk);
    p.gv[i1] = grid_node(p, cs, nf, single_env, cap, a1, bi * 4 + li0 + 2, bj * 4 + lj, bk * 4 + lk);
    if (clear) {
      p.gm[i0] = make_float4(0.f, 0.f, 0.f, 0.f);
      p.gm[i1] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (lane == 0) p.brick_flag[b] = 0;
  }
  if (done) {
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(done, 1) == (int)gridDim.x - 1) {
      *p.active_count = 0;
      *p.work_next = 0;
      *done = 0;
    }
  }
}

// Substeps 2..L of a stretch in ONE cooperative launch: per substep the
// fused phase (all items) and the grid-op phase (all active bricks),
// separated by grid-wide barriers, so the kernel boundaries (launch, ramp,
// tail, the grid op's fixed per-launch work) of two launches per substep
// disappear.  Brick-list and work-item counters are double-buffered by
// substep parity (ctr[0..1] active bricks, ctr[2..3] work cursor; both of the
// first pair zero at launch): substep t uses parity t & 1 and CTA 0 re-arms
// parity t + 1, whose last users finished before the previous barrier.  The
// item bounds swap per substep exactly as across fused_kernel launches.
// Collider pose rows: row0 + t, clamped to the table.
__global__ void __launch_bounds__(FUSED_K_THREADS, FUSED_MIN_BLOCKS)
    substeps_kernel(Params p, Colliders cs, const ColliderPose* __restrict__ pose_base, int pose_rows,
                    int pose_stride, int row0, int nsub, int last_clear, float4* __restrict__ bounds_in,
                    float4* __restrict__ bounds_out, int* __restrict__ item_box, int* __restrict__ ctr,
                    int* __restrict__ final_active) {
  cg::grid_group grid = cg::this_grid();
  for (int t = 0; t < nsub; ++t) {
    Params q = p;
    q.active_count = ctr + (t & 1);
    q.work_next = ctr + 2 + (t & 1);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      ctr[(t + 1) & 1] = 0;
      ctr[2 + ((t + 1) & 1)] = 0;
    }
    fused_phase<false>(q, bounds_in, bounds_out, item_box, t == 0);
    float4* tmp = bounds_in;
    bounds_in = bounds_out;
    bounds_out = tmp;
    grid.sync();
    Colliders c = cs;
    if (pose_base) c.pose = pose_base + (long long)min(row0 + t, pose_rows - 1) * pose_stride;
    const int clear = t < nsub - 1 || last_clear;
    grid_phase<false>(q, c, clear);
    if (t == nsub - 1 && !clear && blockIdx.x == 0 && threadIdx.x == 0) *final_active = *q.active_count;
    grid.sync();
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

}  // namespace mpm

#include "binning.cuh"
#include "determinism.cuh"
#include "conversions.cuh"
#include "frame_ops.cuh"
#include "slab_halo.cuh"
