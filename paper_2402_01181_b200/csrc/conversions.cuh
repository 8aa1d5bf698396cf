// conversions.cuh -- host <-> device field conversions (sm_100a).
// Part of the kernel set included by kernels.cuh (namespace mpm).
#pragma once

namespace mpm {

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

// The same with the host-converted fp32 wire format (mpm.cu host_xfer: the
// caller's fp64 arrays are narrowed on host threads, exactly as the device's
// round-to-nearest cvt would, and only fp32 crosses PCIe); unmasked fields
// are null.
__global__ void upload_fields32_kernel(Params p, const float* __restrict__ x, const float* __restrict__ v,
                                       const float* __restrict__ F, const float* __restrict__ C) {
  long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s >= p.n) return;
  long long o = p.orig[s];
  if (x)
    for (int a = 0; a < 3; ++a) stf(p, FX + a, s, x[3 * o + a]);
  if (v)
    for (int a = 0; a < 3; ++a) stf(p, FV + a, s, v[3 * o + a]);
  if (F)
    for (int q = 0; q < 9; ++q) stf(p, FF + q, s, F[9 * o + q]);
  if (C)
    for (int q = 0; q < 9; ++q) stf(p, FC + q, s, C[9 * o + q]);
}

__global__ void download_fields32_kernel(Params p, float* __restrict__ x, float* __restrict__ v,
                                         float* __restrict__ F, float* __restrict__ C) {
  long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s >= p.n) return;
  long long o = p.orig[s];
  if (x)
    for (int a = 0; a < 3; ++a) x[3 * o + a] = ldf(p, FX + a, s);
  if (v)
    for (int a = 0; a < 3; ++a) v[3 * o + a] = ldf(p, FV + a, s);
  if (F)
    for (int q = 0; q < 9; ++q) F[9 * o + q] = ldf(p, FF + q, s);
  if (C)
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
  gi += p.goff[0];
  gj += p.goff[1];
  gk += p.goff[2];
  const Colliders ce = env_colliders(cs, gi / p.env_res[0], gj / p.env_res[1], gk / p.env_res[2]);
  double best;
  int id = nearest_collider(ce, (double)gi * p.dx64, (double)gj * p.dx64, (double)gk * p.dx64, cap, best);
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
