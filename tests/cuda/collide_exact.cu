// Bitwise self-check of collide.cuh's shortcut paths (box_sd_fast and the
// axis-aligned normal) against the plain formulas of the reference
// (kernels.py:30-45, 116-158) on many points near faces, edges, corners and
// inside rotated boxes.  Built and run by tests/test_gpu_collide_exact.py.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include "../../paper_2402_01181_b200/csrc/collide.cuh"
using namespace mpm;

__device__ double plain_box_sd(double px, double py, double pz, const double h[3]) {
  double qx = ds(fabs(px), h[0]), qy = ds(fabs(py), h[1]), qz = ds(fabs(pz), h[2]);
  double ox = qx > 0.0 ? qx : 0.0, oy = qy > 0.0 ? qy : 0.0, oz = qz > 0.0 ? qz : 0.0;
  double outside = __dsqrt_rn(da(da(dm(ox, ox), dm(oy, oy)), dm(oz, oz)));
  double qm = qx;
  if (qy > qm) qm = qy;
  if (qz > qm) qm = qz;
  return da(outside, qm < 0.0 ? qm : 0.0);
}

__device__ void plain_normal(const ColliderGeo& g, const ColliderPose& q, double wx, double wy, double wz, double n[3]) {
  double px, py, pz;
  to_local(q, wx, wy, wz, px, py, pz);
  double h = g.half[0];
  if (g.half[1] < h) h = g.half[1];
  if (g.half[2] < h) h = g.half[2];
  h = dm(1.0e-3, h);
  if (h < 1.0e-6) h = 1.0e-6;
  double gx = ds(plain_box_sd(da(px, h), py, pz, g.half), plain_box_sd(ds(px, h), py, pz, g.half));
  double gy = ds(plain_box_sd(px, da(py, h), pz, g.half), plain_box_sd(px, ds(py, h), pz, g.half));
  double gz = ds(plain_box_sd(px, py, da(pz, h), g.half), plain_box_sd(px, py, ds(pz, h), g.half));
  double norm = __dsqrt_rn(da(da(dm(gx, gx), dm(gy, gy)), dm(gz, gz)));
  if (norm < 1.0e-12) {
    double fx = ds(wx, q.T[0]), fy = ds(wy, q.T[1]), fz = ds(wz, q.T[2]);
    double fn = __dsqrt_rn(da(da(dm(fx, fx), dm(fy, fy)), dm(fz, fz)));
    if (fn < 1.0e-12) { n[0] = 0.0; n[1] = 1.0; n[2] = 0.0; return; }
    n[0] = __ddiv_rn(fx, fn); n[1] = __ddiv_rn(fy, fn); n[2] = __ddiv_rn(fz, fn);
    return;
  }
  gx = __ddiv_rn(gx, norm); gy = __ddiv_rn(gy, norm); gz = __ddiv_rn(gz, norm);
  n[0] = da(da(dm(q.R[0], gx), dm(q.R[1], gy)), dm(q.R[2], gz));
  n[1] = da(da(dm(q.R[3], gx), dm(q.R[4], gy)), dm(q.R[5], gz));
  n[2] = da(da(dm(q.R[6], gx), dm(q.R[7], gy)), dm(q.R[8], gz));
}

__device__ unsigned long long mix(unsigned long long x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return x;
}
__device__ double u01(unsigned long long& s) { s = mix(s + 0x9e3779b97f4a7c15ull); return (s >> 11) * (1.0 / 9007199254740992.0); }

__global__ void check(const ColliderGeo* geos, const ColliderPose* poses, int ncol, long long n, unsigned long long* bad,
                      unsigned long long* fast_hits) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned long long s = mix(i * 7919ull + 17ull);
  const int ci = (int)(i % ncol);
  const ColliderGeo& g = geos[ci];
  const ColliderPose& q = poses[ci];
  // a local point near the box surface: each axis at -h, +h, inside, or just beyond,
  // jittered by a few multiples of the finite-difference step (and sometimes exactly on it)
  double p[3];
  for (int a = 0; a < 3; ++a) {
    const double h = g.half[a];
    const int kind = (int)(u01(s) * 6.0);
    const double sgn = u01(s) < 0.5 ? -1.0 : 1.0;
    const double jit = (u01(s) - 0.5) * 8.0e-3 * h;
    p[a] = kind == 0 ? sgn * h : kind <= 2 ? sgn * (h + jit) : (u01(s) - 0.5) * 2.0 * h * 1.2;
  }
  // to world: w = R p + T
  double w[3];
  for (int r = 0; r < 3; ++r) w[r] = q.T[r] + q.R[3 * r] * p[0] + q.R[3 * r + 1] * p[1] + q.R[3 * r + 2] * p[2];
  Colliders cs{};
  cs.count = ncol;
  cs.geo = geos;
  cs.pose = poses;
  double a[3], b[3];
  world_normal(cs, ci, w[0], w[1], w[2], a);
  plain_normal(g, q, w[0], w[1], w[2], b);
  double lx, ly, lz;
  to_local(q, w[0], w[1], w[2], lx, ly, lz);
  const double d0 = world_sd(cs, ci, w[0], w[1], w[2]), d1 = plain_box_sd(lx, ly, lz, g.half);
  bool okf;
  box_sd_fast(lx, ly, lz, g.half, okf);
  if (okf) atomicAdd(fast_hits, 1ull);
  bool same = __double_as_longlong(d0) == __double_as_longlong(d1);
  for (int k = 0; k < 3; ++k) same &= __double_as_longlong(a[k]) == __double_as_longlong(b[k]);
  if (!same) atomicAdd(bad, 1ull);
}

int main(int argc, char** argv) {
  const long long n = argc > 1 ? atoll(argv[1]) : (1ll << 24);
  const int ncol = 4;
  std::vector<ColliderGeo> geo(ncol);
  std::vector<ColliderPose> pose(ncol);
  srand(7);
  for (int c = 0; c < ncol; ++c) {
    memset(&geo[c], 0, sizeof(ColliderGeo));
    memset(&pose[c], 0, sizeof(ColliderPose));
    const double hs[4][3] = {{0.08, 0.03, 0.08}, {0.01, 0.02, 0.3}, {0.25, 0.25, 0.25}, {1e-3, 5e-4, 2e-3}};
    for (int a = 0; a < 3; ++a) geo[c].half[a] = hs[c][a];
    // rotation from a quaternion (identity for collider 0: the axis-aligned C3 tool)
    double qx = 0, qy = 0, qz = 0, qw = 1;
    if (c) { qx = rand() / (double)RAND_MAX - 0.5; qy = rand() / (double)RAND_MAX - 0.5; qz = rand() / (double)RAND_MAX - 0.5; qw = 0.7; }
    const double nn = sqrt(qx * qx + qy * qy + qz * qz + qw * qw);
    qx /= nn; qy /= nn; qz /= nn; qw /= nn;
    double* R = pose[c].R;
    R[0] = 1 - 2 * (qy * qy + qz * qz); R[1] = 2 * (qx * qy - qz * qw); R[2] = 2 * (qx * qz + qy * qw);
    R[3] = 2 * (qx * qy + qz * qw); R[4] = 1 - 2 * (qx * qx + qz * qz); R[5] = 2 * (qy * qz - qx * qw);
    R[6] = 2 * (qx * qz - qy * qw); R[7] = 2 * (qy * qz + qx * qw); R[8] = 1 - 2 * (qx * qx + qy * qy);
    pose[c].T[0] = 0.5 + 0.01 * c; pose[c].T[1] = 0.2; pose[c].T[2] = 0.5 - 0.003 * c;
  }
  ColliderGeo* dg; ColliderPose* dp; unsigned long long* dbad;
  cudaMalloc(&dg, sizeof(ColliderGeo) * ncol);
  cudaMalloc(&dp, sizeof(ColliderPose) * ncol);
  cudaMalloc(&dbad, 16);
  cudaMemcpy(dg, geo.data(), sizeof(ColliderGeo) * ncol, cudaMemcpyHostToDevice);
  cudaMemcpy(dp, pose.data(), sizeof(ColliderPose) * ncol, cudaMemcpyHostToDevice);
  cudaMemset(dbad, 0, 16);
  check<<<(unsigned)((n + 255) / 256), 256>>>(dg, dp, ncol, n, dbad, dbad + 1);
  unsigned long long h[2] = {0, 0};
  if (cudaMemcpy(h, dbad, 16, cudaMemcpyDeviceToHost) != cudaSuccess) { printf("cuda error\n"); return 2; }
  printf("points %lld mismatches %llu fast-path %llu\n", n, h[0], h[1]);
  return h[0] == 0 ? 0 : 1;
}
