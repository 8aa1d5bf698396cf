// common.cuh -- layouts, launch parameters and stencil math shared by the
// B200 MLS-MPM kernels.
//
// HBM layout:
//   * particles: SoA fp32, NF float fields of `cap` entries each (x0..2,
//     v0..2, F00..F22, C00..C22, mass, vol0) + int32 material id + int32
//     original index, double-buffered so re-binning is a gather-free scatter;
//     the device order is "grouped by 8^3-cell bin", the host order is the
//     caller's.
//   * grid: blocked-dense float4 arrays, 4^3-node bricks of 1 KiB each
//     (node (i,j,k) -> brick ((i>>2,j>>2,k>>2)) * 64 + local (i&3,j&3,k&3)),
//     `gm` = (momentum xyz, mass) accumulated by P2G, `gv` = velocity
//     written by the grid op and read by G2P.  Only bricks touched by P2G
//     (the active list) are visited by the grid op.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace mpm {

constexpr int BRICK_SHIFT = 2;            // 4^3 nodes per layout brick
constexpr int BRICK_NODES = 64;
constexpr int BIN = 8;                    // particle bin edge (cells)
constexpr int BIN_SHIFT = 3;
#ifndef MPM_MARGIN
#define MPM_MARGIN 2
#endif
constexpr int MARGIN = MPM_MARGIN;        // tile margin for particles drifting out of their bin
#ifndef MPM_TILE
#define MPM_TILE (BIN + 2 + 2 * MPM_MARGIN)
#endif
// nodes per tile edge (14): base cells org + [0, TILE - 3], i.e. drift of
// MARGIN - 1 cells below the bin and TILE - BIN - 1 - MARGIN above
constexpr int TILE = MPM_TILE;
#ifndef MPM_TILE_ZSTRIDE
#define MPM_TILE_ZSTRIDE TILE
#endif
#ifndef MPM_PLANE_PAD
#define MPM_PLANE_PAD 0
#endif
// smem tile layout: node (x, y, z) at (x TILE + y) TILE_Z + z of a channel
// plane of TILE_NODES words (z stride and plane padding tune the bank map)
constexpr int TILE_Z = MPM_TILE_ZSTRIDE;
constexpr int TILE_NODES = TILE * TILE * TILE_Z + MPM_PLANE_PAD;
// the velocity tile holds (vx, vy) float2 pairs and its buffers start at
// multiples of 3 * TILE_NODES floats: 8-byte alignment needs an even plane
static_assert(TILE_NODES % 2 == 0, "TILE_NODES must be even (float2 velocity tile)");
constexpr int FUSED_THREADS = 256;      // stage A (g2p_stress_kernel)
#ifndef MPM_FUSED_THREADS
#define MPM_FUSED_THREADS 256
#endif
#ifndef MPM_FUSED_MINB
#define MPM_FUSED_MINB 2
#endif
constexpr int FUSED_K_THREADS = MPM_FUSED_THREADS;  // fused steady-state kernel
constexpr int FUSED_MIN_BLOCKS = MPM_FUSED_MINB;
constexpr int P2G_THREADS = 256;        // stage B (p2g_tile_kernel)
constexpr int P2G_MIN_BLOCKS = 3;
#ifndef MPM_GRIDOP_MINB
#define MPM_GRIDOP_MINB 2
#endif
constexpr int GRIDOP_MIN_BLOCKS = MPM_GRIDOP_MINB;
// dynamic shared memory of the fused kernel: velocity tile (3 planes), int32
// scatter tile (4 channel planes) and the per-cell particle counts of the
// fixed-point overflow guard (1 plane); stage B: scatter tile + counts
#ifndef EXP_SMEM_PAD
#define EXP_SMEM_PAD 0  // timing experiment: extra shared memory per fused CTA (occupancy sensitivity)
#endif
constexpr unsigned FUSED_SMEM = sizeof(float) * 8 * TILE_NODES + EXP_SMEM_PAD;
constexpr unsigned P2G_SMEM = sizeof(int) * 5 * TILE_NODES;
constexpr int NPAY = 13;                // payload floats per particle: m v (3), A (9), m
constexpr int CHUNK = 4096;               // max particles per work item (larger bins split evenly)
constexpr int MIN_CHUNK = 256;            // small scenes: items shrink to this so every SM gets work
// 4^3 layout bricks overlapped by a tile: org = 8b - MARGIN is even, so a tile edge of TILE nodes spans
constexpr int TILE_BRICKS = (TILE + 3 + 3) / 4;
constexpr int NF = 26;                    // float fields per particle

enum Field : int { FX = 0, FV = 3, FF = 6, FC = 15, FMASS = 24, FVOL = 25 };

// Division of a non-negative 32-bit value by a runtime-constant divisor with
// one multiply-high (round-up method: q = (umulhi(n, m) + n) >> s, exact for
// all n < 2^32), precomputed on the host.
struct FastDiv {
  unsigned m;
  int s;
  __device__ __forceinline__ unsigned div(unsigned n) const {
    return (unsigned)(((unsigned long long)__umulhi(n, m) + n) >> s);
  }
};

inline FastDiv make_fastdiv(int d) {
  int l = 0;
  while ((1LL << l) < d) ++l;
  FastDiv f;
  f.m = (unsigned)((((1ULL << 32) * ((1ULL << l) - (unsigned long long)d)) / (unsigned long long)d) + 1);
  f.s = l;
  return f;
}

struct Params {
  // grid
  int res[3];      // node resolution
  int nb[3];       // layout bricks per axis
  FastDiv fd_nb1, fd_nb2;  // / nb[1], / nb[2]
  int nbin[3];     // particle bins per axis
  FastDiv fd_nbin1, fd_nbin2;  // / nbin[1], / nbin[2]
  float dx, inv_dx, dt;
  float gravity[3];
  float lo, hi[3];  // particle margin clamp (core.py:51-56), env-local
  int env_res[3];   // nodes per environment tile (== gres for one environment)
  float env_ext[3]; // env_res * dx
  FastDiv fd_env[3];  // / env_res
  float inv_env_ext[3];  // 1 / env_ext
  // slab decomposition (config 5): this context's grid is the window of the
  // global grid (gres nodes) starting at global node goff; particle positions
  // on the device are window-local (global - goff * dx)
  int goff[3];
  int gres[3];
  float goffx[3];   // goff * dx
  float stress_coef;  // -4 dt / dx^2 (kernels.py:207)
  float apic_coef;    // 4 / dx^2 (kernels.py:448)
  double dx64, dt64;
  int bwidth, stick, stress_form;
  // grid buffers
  float4* gm;
  float4* gv;
  int* brick_flag;
  int* active_list;
  int* active_count;
  // particles
  float* P;
  float* Pf[NF];  // per-field base pointers into P (kernel-parameter constants: one address add per access)
  int* mat;
  int* orig;
  long long cap;
  long long n;
  const float* mu;
  const float* lam;
  unsigned long long* inverted;
  // fixed-point overflow guard: stats[0] counts particles routed to the float
  // path because their cell exceeded the item's count limit; fx_shift (test
  // hook, default 0) scales the tile up by 2^fx_shift and the limit down
  unsigned long long* stats;
  int fx_shift;
  // slab windows between a migrant extraction and the next re-binning:
  // slots [0, hole_n) whose hole_flag is set have left (skipped by bin_key)
  const int* hole_flag;
  long long hole_n;
  // work items (bin, start, end, 0)
  const int4* work;
  const int* nwork;
  int* work_next;    // dynamic work-item counter (zeroed per launch)
};

// Bin index -> bin coordinates (x-major, z fastest) by multiply-high division.
__device__ __forceinline__ void bin_coords(const Params& p, int bin, int& bx, int& by, int& bz) {
  const unsigned t = p.fd_nbin2.div((unsigned)bin);
  bz = bin - (int)t * p.nbin[2];
  bx = (int)p.fd_nbin1.div(t);
  by = (int)t - bx * p.nbin[1];
}

__host__ __device__ inline long long node_index(int i, int j, int k, int nby, int nbz) {
  long long b = ((long long)(i >> BRICK_SHIFT) * nby + (j >> BRICK_SHIFT)) * nbz + (k >> BRICK_SHIFT);
  return (b << 6) | ((i & 3) << 4) | ((j & 3) << 2) | (k & 3);
}

__device__ inline void brick_coords(long long b, const int nb[3], int& bi, int& bj, int& bk) {
  bk = (int)(b % nb[2]);
  long long t = b / nb[2];
  bj = (int)(t % nb[1]);
  bi = (int)(t / nb[1]);
}

// Quadratic B-spline stencil of one coordinate (kernels.py:277-294), fp32,
// base clamped to [0, r-3] (fp32 rounding can push x/dx past the fp64
// margin of core.py:55; the clamp keeps the 3-node stencil in the grid).
__device__ __forceinline__ void stencil(float xc, float inv_dx, int r, int& b, float& f,
                                        float w[3]) {
  float g = xc * inv_dx;
  int bb = (int)floorf(g - 0.5f);
  bb = max(0, min(bb, r - 3));
  f = g - (float)bb;
  float t0 = 1.5f - f, t1 = f - 1.0f, t2 = f - 0.5f;
  w[0] = 0.5f * (t0 * t0);
  w[1] = 0.75f - t1 * t1;
  w[2] = 0.5f * (t2 * t2);
  b = bb;
}

// Exactly-rounded variant (no FMA contraction) used by the deterministic
// mode; must equal oracle/mpm_oracle.c:stencil_axis32 bit for bit.
__device__ __forceinline__ void stencil_rn(float xc, float inv_dx, int r, int& b, float& f,
                                           float w[3]) {
  float g = __fmul_rn(xc, inv_dx);
  int bb = (int)floorf(__fsub_rn(g, 0.5f));
  bb = max(0, min(bb, r - 3));
  f = __fsub_rn(g, (float)bb);
  float t0 = __fsub_rn(1.5f, f), t1 = __fsub_rn(f, 1.0f), t2 = __fsub_rn(f, 0.5f);
  w[0] = __fmul_rn(0.5f, __fmul_rn(t0, t0));
  w[1] = __fsub_rn(0.75f, __fmul_rn(t1, t1));
  w[2] = __fmul_rn(0.5f, __fmul_rn(t2, t2));
  b = bb;
}

// Packed fp32 pairs (sm_100a FFMA2 / FMUL2 / FADD2): one issue slot for two
// lanes of fp32 math.  Measured on B200 (tools/microbench/ffma2.cu): FFMA2
// occupies the FMA pipe for 2 cycles (no extra FLOP rate) but halves the
// issue slots of paired math, which is what the issue-bound fused kernel
// needs.  A scalar broadcast (f2_bc) compiles to the .F32 operand form, no MOV.
typedef unsigned long long f2p;
__device__ __forceinline__ f2p f2_pack(float a, float b) {
  f2p r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ f2p f2_bc(float a) { return f2_pack(a, a); }
__device__ __forceinline__ float f2_lo(f2p v) {
  float a;
  asm("mov.b64 {%0, _}, %1;" : "=f"(a) : "l"(v));
  return a;
}
__device__ __forceinline__ float f2_hi(f2p v) {
  float b;
  asm("mov.b64 {_, %0}, %1;" : "=f"(b) : "l"(v));
  return b;
}
__device__ __forceinline__ f2p f2_fma(f2p a, f2p b, f2p c) {
  f2p d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ f2p f2_mul(f2p a, f2p b) {
  f2p d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f2p f2_add(f2p a, f2p b) {
  f2p d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

__device__ __forceinline__ float ldf(const Params& p, int field, long long i) {
  return p.Pf[field][i];
}
__device__ __forceinline__ void stf(const Params& p, int field, long long i, float v) {
  p.Pf[field][i] = v;
}

// F' = (I + dt C) F (kernels.py:213-231), then the Neo-Hookean affine
// momentum A = m C + k P F'^T (kernels.py:233-275).  Returns det(F').
template <bool RN>
__device__ __forceinline__ float affine_update(float F[9], const float C[9], float m, float vol,
                                               float mu, float lam, float dt, float stress_coef,
                                               int stress_form, float A[9]);

template <>
__device__ __forceinline__ float affine_update<false>(float F[9], const float C[9], float m,
                                                      float vol, float mu, float lam, float dt,
                                                      float stress_coef, int stress_form,
                                                      float A[9]) {
  float f[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      f[3 * r + c] = F[3 * r + c] + dt * (C[3 * r] * F[c] + C[3 * r + 1] * F[3 + c] +
                                          C[3 * r + 2] * F[6 + c]);
#pragma unroll
  for (int q = 0; q < 9; ++q) F[q] = f[q];
  float cof[9];
  cof[0] = f[4] * f[8] - f[5] * f[7];
  cof[1] = f[5] * f[6] - f[3] * f[8];
  cof[2] = f[3] * f[7] - f[4] * f[6];
  cof[3] = f[2] * f[7] - f[1] * f[8];
  cof[4] = f[0] * f[8] - f[2] * f[6];
  cof[5] = f[1] * f[6] - f[0] * f[7];
  cof[6] = f[1] * f[5] - f[2] * f[4];
  cof[7] = f[2] * f[3] - f[0] * f[5];
  cof[8] = f[0] * f[4] - f[1] * f[3];
  float det = f[0] * cof[0] + f[1] * cof[1] + f[2] * cof[2];
  float js = det > 1.0e-6f ? det : 1.0e-6f;
  float g = (lam * logf(js) - mu) * (det != 0.0f ? 1.0f / det : 0.0f);
  float k = stress_coef * vol;
  float P[9];
  if (stress_form == 0) {
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) P[3 * r + c] = mu * f[3 * r + c] + g * cof[3 * c + r];
  } else {
#pragma unroll
    for (int q = 0; q < 9; ++q) P[q] = mu * f[q] + g * cof[q];
  }
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      A[3 * r + c] = m * C[3 * r + c] +
                     k * (P[3 * r] * f[3 * c] + P[3 * r + 1] * f[3 * c + 1] + P[3 * r + 2] * f[3 * c + 2]);
  return det;
}

// Round-to-nearest twin of the above (no contraction) for the deterministic
// mode; mirrors oracle/mpm_oracle.c:orc32_p2g_sorted operation by operation.
template <>
__device__ __forceinline__ float affine_update<true>(float F[9], const float C[9], float m,
                                                     float vol, float mu, float lam, float dt,
                                                     float stress_coef, int stress_form,
                                                     float A[9]) {
  float f[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      float s = __fadd_rn(__fadd_rn(__fmul_rn(C[3 * r], F[c]), __fmul_rn(C[3 * r + 1], F[3 + c])),
                          __fmul_rn(C[3 * r + 2], F[6 + c]));
      f[3 * r + c] = __fadd_rn(F[3 * r + c], __fmul_rn(dt, s));
    }
#pragma unroll
  for (int q = 0; q < 9; ++q) F[q] = f[q];
  auto dif = [](float a, float b, float c, float d) { return __fsub_rn(__fmul_rn(a, b), __fmul_rn(c, d)); };
  float cof[9];
  cof[0] = dif(f[4], f[8], f[5], f[7]);
  cof[1] = dif(f[5], f[6], f[3], f[8]);
  cof[2] = dif(f[3], f[7], f[4], f[6]);
  float det = __fadd_rn(__fadd_rn(__fmul_rn(f[0], cof[0]), __fmul_rn(f[1], cof[1])), __fmul_rn(f[2], cof[2]));
  cof[3] = dif(f[2], f[7], f[1], f[8]);
  cof[4] = dif(f[0], f[8], f[2], f[6]);
  cof[5] = dif(f[1], f[6], f[0], f[7]);
  cof[6] = dif(f[1], f[5], f[2], f[4]);
  cof[7] = dif(f[2], f[3], f[0], f[5]);
  cof[8] = dif(f[0], f[4], f[1], f[3]);
  float js = det > 1.0e-6f ? det : 1.0e-6f;
  float lj = logf(js);
  float id = det != 0.0f ? __fdiv_rn(1.0f, det) : 0.0f;
  float g = __fmul_rn(__fsub_rn(__fmul_rn(lam, lj), mu), id);
  float P[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      float cv = stress_form == 0 ? cof[3 * c + r] : cof[3 * r + c];
      P[3 * r + c] = __fadd_rn(__fmul_rn(mu, f[3 * r + c]), __fmul_rn(g, cv));
    }
  float k = __fmul_rn(stress_coef, vol);
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      float s = __fadd_rn(__fadd_rn(__fmul_rn(P[3 * r], f[3 * c]), __fmul_rn(P[3 * r + 1], f[3 * c + 1])),
                          __fmul_rn(P[3 * r + 2], f[3 * c + 2]));
      A[3 * r + c] = __fadd_rn(__fmul_rn(m, C[3 * r + c]), __fmul_rn(k, s));
    }
  return det;
}

}  // namespace mpm
