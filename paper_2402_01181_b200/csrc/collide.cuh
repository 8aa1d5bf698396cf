// collide.cuh -- rigid-tool geometry and contact response on the device.
//
// fp64 with every product/sum explicitly rounded (no FMA contraction) so the
// merged distance field and contact normals equal the reference's numba
// kernels bit for bit (kernels.py:30-191, fastmath off):
//   box_sd      <- _box_signed_distance      kernels.py:30-45
//   baked_sd    <- _sample_baked             kernels.py:48-88
//   world_sd    <- _collider_world_distance  kernels.py:102-113
//   world_normal<- _collider_world_normal    kernels.py:116-158
//   resolve     <- grid_update contact block kernels.py:371-411
// Only massive nodes inside the band evaluate these (the reference rebuilds
// the field over every node, kernels.py:161-191; the result at consumed nodes
// is identical).
#pragma once
#include <cstdint>

namespace mpm {

constexpr int MAX_COLLIDERS = 16;
#ifdef FUSED_PROFILE
__device__ unsigned long long g_cph[4];  // contact phases: nearest, pre-normal, normal, rest (cycles)
#define CPH_MARK(k, t) do { const long long _t = clock64(); atomicAdd(&g_cph[k], (unsigned long long)(_t - (t))); t = _t; } while (0)
#else
#define CPH_MARK(k, t) do { } while (0)
#endif

struct ColliderGeo {
  int kind;  // 0 box, 1 baked
  double half[3];
  double fric;
  int mode;  // packed (frozen) mode
  long long sdf_off;
  int sdf_res[3];
  double sdf_bmin[3];
  double sdf_ext;
  // far-field prefilter (host-computed): box -> |half|; baked -> the smallest
  // sampled distance on the lattice's outer layer (what any query outside
  // the lattice box evaluates to, kernels.py:52-66 clamping)
  float far_r;
  float far_min;
};

struct ColliderPose {
  double R[9];
  double T[3];
  double lv[3];
  double av[3];
  int mode;
};

struct Colliders {
  int count;      // colliders acting on one environment tile
  double theta;   // < 0: disabled
  float theta_f;  // theta + prefilter margin (fp32)
  const ColliderGeo* geo;
  const ColliderPose* pose;  // row for this substep
  const double* sdf;
  int per_env;        // 0: one table for the whole grid; else count per tile, tile-major
  int env_tiles[3];
};

// The collider sub-table of environment tile (ei, ej, ek).
__device__ __forceinline__ Colliders env_colliders(const Colliders& cs, int ei, int ej, int ek) {
  if (!cs.per_env) return cs;
  Colliders c = cs;
  const int e = (ei * cs.env_tiles[1] + ej) * cs.env_tiles[2] + ek;
  c.geo += (long long)e * cs.per_env;
  c.pose += (long long)e * cs.per_env;
  return c;
}

__device__ __forceinline__ double dm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double da(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double ds(double a, double b) { return __dsub_rn(a, b); }

// The reference's sqrt(ox*ox + oy*oy + oz*oz) for ox, oy, oz >= +0 without
// the library square root when at most one term is non-zero: in radix 2,
// sqrt(RN(x*x)) == |x| absent under/overflow, and adding +0 is exact, so the
// result is that term bit for bit.  Near a face (the common contact case)
// this keeps the branchy sqrt sequence -- which serialises everything around
// it -- out of the six finite-difference evaluations of world_normal.
// `ok` is false when the full square root is needed.
__device__ __forceinline__ double box_sd_fast(double px, double py, double pz, const double h[3], bool& ok) {
  const double qx = ds(fabs(px), h[0]), qy = ds(fabs(py), h[1]), qz = ds(fabs(pz), h[2]);
  const bool ax = qx > 0.0, ay = qy > 0.0, az = qz > 0.0;
  // the one positive term (adding the +0 others is exact): selects, no adds
  const double one = ax ? qx : ay ? qy : az ? qz : 0.0;
  ok = ((int)ax + (int)ay + (int)az <= 1) & ((one == 0.0) | ((one > 1e-150) & (one < 1e150)));  // no branches
  double qm = qx;
  if (qy > qm) qm = qy;
  if (qz > qm) qm = qz;
  // outside + inside: one of the two is +0 (a positive term makes qm > 0)
  return one > 0.0 ? one : (qm < 0.0 ? qm : 0.0);
}

__device__ inline double box_sd(double px, double py, double pz, const double h[3]) {
  bool ok;
  const double fast = box_sd_fast(px, py, pz, h, ok);
  if (ok) return fast;
  double qx = ds(fabs(px), h[0]), qy = ds(fabs(py), h[1]), qz = ds(fabs(pz), h[2]);
  double ox = qx > 0.0 ? qx : 0.0, oy = qy > 0.0 ? qy : 0.0, oz = qz > 0.0 ? qz : 0.0;
  double outside = __dsqrt_rn(da(da(dm(ox, ox), dm(oy, oy)), dm(oz, oz)));
  double qm = qx;
  if (qy > qm) qm = qy;
  if (qz > qm) qm = qz;
  return da(outside, qm < 0.0 ? qm : 0.0);
}

__device__ inline double baked_sd(const ColliderGeo& g, const double* sdf, double px, double py,
                                  double pz) {
  const double p[3] = {px, py, pz};
  long long i0[3];
  double fr[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double r = (double)g.sdf_res[a];
    double c = ds(dm(__ddiv_rn(ds(p[a], g.sdf_bmin[a]), g.sdf_ext), r), 0.5);
    if (c < 0.0) c = 0.0;
    if (c > r - 1.0) c = r - 1.0;
    long long ii = (long long)c;
    if (ii > g.sdf_res[a] - 2) ii = g.sdf_res[a] - 2;
    i0[a] = ii;
    fr[a] = ds(c, (double)ii);
  }
  const double* v = sdf + g.sdf_off;
  long long rx = g.sdf_res[0], ry = g.sdf_res[1];
  double s = 0.0;
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    double wa = a ? fr[0] : ds(1.0, fr[0]);
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      double wb = b ? fr[1] : ds(1.0, fr[1]);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        double wc = c ? fr[2] : ds(1.0, fr[2]);
        long long idx = (i0[0] + a) + rx * ((i0[1] + b) + ry * (i0[2] + c));
        s = da(s, dm(dm(dm(wa, wb), wc), __ldg(v + idx)));
      }
    }
  }
  return dm(s, g.sdf_ext);
}

__device__ inline double local_sd(const ColliderGeo& g, const double* sdf, double px, double py,
                                  double pz) {
  if (g.kind == 0) return box_sd(px, py, pz, g.half);
  return baked_sd(g, sdf, px, py, pz);
}

__device__ inline void to_local(const ColliderPose& q, double wx, double wy, double wz,
                                double& px, double& py, double& pz) {
  double d0 = ds(wx, q.T[0]), d1 = ds(wy, q.T[1]), d2 = ds(wz, q.T[2]);
  px = da(da(dm(q.R[0], d0), dm(q.R[3], d1)), dm(q.R[6], d2));
  py = da(da(dm(q.R[1], d0), dm(q.R[4], d1)), dm(q.R[7], d2));
  pz = da(da(dm(q.R[2], d0), dm(q.R[5], d1)), dm(q.R[8], d2));
}

__device__ inline double world_sd(const Colliders& cs, int ci, double wx, double wy, double wz) {
  double px, py, pz;
  to_local(cs.pose[ci], wx, wy, wz, px, py, pz);
  return local_sd(cs.geo[ci], cs.sdf, px, py, pz);
}

// Conservative fp32 test: may collider ci be closer than theta_m to world
// point (x, y, z)?  false only when the exact fp64 distance is certainly
// >= theta (theta_m carries a margin far above fp32 rounding).
__device__ __forceinline__ bool collider_near(const Colliders& cs, int ci, float x, float y, float z,
                                              float theta_m) {
  const ColliderGeo& g = cs.geo[ci];
  const ColliderPose& q = cs.pose[ci];
  const float d0 = x - (float)q.T[0], d1 = y - (float)q.T[1], d2 = z - (float)q.T[2];
  if (g.kind == 0) {
    // box SDF >= max_a (|p_a| - h_a): test the theta-inflated oriented box
    const float px = (float)q.R[0] * d0 + (float)q.R[3] * d1 + (float)q.R[6] * d2;
    const float py = (float)q.R[1] * d0 + (float)q.R[4] * d1 + (float)q.R[7] * d2;
    const float pz = (float)q.R[2] * d0 + (float)q.R[5] * d1 + (float)q.R[8] * d2;
    return fabsf(px) < (float)g.half[0] + theta_m && fabsf(py) < (float)g.half[1] + theta_m &&
           fabsf(pz) < (float)g.half[2] + theta_m;
  }
  // baked: outside the lattice box the sample is >= far_min
  if (g.far_min >= theta_m) {
    const float px = (float)q.R[0] * d0 + (float)q.R[3] * d1 + (float)q.R[6] * d2;
    const float py = (float)q.R[1] * d0 + (float)q.R[4] * d1 + (float)q.R[7] * d2;
    const float pz = (float)q.R[2] * d0 + (float)q.R[5] * d1 + (float)q.R[8] * d2;
    const float m = 1e-4f * (float)g.sdf_ext + 1e-6f;
    const float lo0 = (float)g.sdf_bmin[0] - m, lo1 = (float)g.sdf_bmin[1] - m, lo2 = (float)g.sdf_bmin[2] - m;
    const float e = (float)g.sdf_ext + 2.0f * m;
    const bool inside = px >= lo0 && px <= lo0 + e && py >= lo1 && py <= lo1 + e && pz >= lo2 && pz <= lo2 + e;
    return inside;
  }
  return true;
}

// The same test with the fp32 pose and the inflated box precomputed once per
// CTA: local p in [lo, hi] per axis (non-strict: at least as conservative).
struct ColliderNearF {
  float R[9], T[3];
  float lo[3], hi[3];
  __device__ __forceinline__ bool near(float x, float y, float z) const {
    const float d0 = x - T[0], d1 = y - T[1], d2 = z - T[2];
    const float px = R[0] * d0 + R[3] * d1 + R[6] * d2;
    const float py = R[1] * d0 + R[4] * d1 + R[7] * d2;
    const float pz = R[2] * d0 + R[5] * d1 + R[8] * d2;
    return px >= lo[0] && px <= hi[0] && py >= lo[1] && py <= hi[1] && pz >= lo[2] && pz <= hi[2];
  }
};

__device__ inline ColliderNearF make_near_f(const Colliders& cs, int ci, float theta_m) {
  const ColliderGeo& g = cs.geo[ci];
  const ColliderPose& q = cs.pose[ci];
  ColliderNearF f;
  for (int k = 0; k < 9; ++k) f.R[k] = (float)q.R[k];
  for (int k = 0; k < 3; ++k) f.T[k] = (float)q.T[k];
  if (g.kind == 0) {
    for (int k = 0; k < 3; ++k) {
      f.hi[k] = (float)g.half[k] + theta_m;
      f.lo[k] = -f.hi[k];
    }
  } else if (g.far_min >= theta_m) {
    const float m = 1e-4f * (float)g.sdf_ext + 1e-6f;
    const float e = (float)g.sdf_ext + 2.0f * m;
    for (int k = 0; k < 3; ++k) {
      f.lo[k] = (float)g.sdf_bmin[k] - m;
      f.hi[k] = f.lo[k] + e;
    }
  } else {
    for (int k = 0; k < 3; ++k) {
      f.lo[k] = -INFINITY;
      f.hi[k] = INFINITY;
    }
  }
  return f;
}

// Merged field at one node: min distance, ties to the lowest index, id -1
// beyond cap = 2 theta (kernels.py:180-191).
__device__ inline int nearest_collider(const Colliders& cs, double wx, double wy, double wz,
                                       double cap, double& best) {
  best = 1.0e30;
  int id = -1;
  for (int ci = 0; ci < cs.count; ++ci) {
    double d = world_sd(cs, ci, wx, wy, wz);
    if (d < best) {
      best = d;
      id = ci;
    }
  }
  return best >= cap ? -1 : id;
}

__device__ inline void world_normal(const Colliders& cs, int ci, double wx, double wy, double wz,
                                    double n[3]) {
  const ColliderGeo& g = cs.geo[ci];
  const ColliderPose& q = cs.pose[ci];
  double px, py, pz;
  to_local(q, wx, wy, wz, px, py, pz);
  double h;
  if (g.kind == 0) {
    h = g.half[0];
    if (g.half[1] < h) h = g.half[1];
    if (g.half[2] < h) h = g.half[2];
    h = dm(1.0e-3, h);
    if (h < 1.0e-6) h = 1.0e-6;
  } else {
    h = __ddiv_rn(g.sdf_ext, (double)g.sdf_res[0]);
  }
  double gx, gy, gz;
  if (g.kind == 0) {
    // six straight-line evaluations; the exact square roots only at edges
    bool ok[6];
    const double s0 = box_sd_fast(da(px, h), py, pz, g.half, ok[0]), s1 = box_sd_fast(ds(px, h), py, pz, g.half, ok[1]);
    const double s2 = box_sd_fast(px, da(py, h), pz, g.half, ok[2]), s3 = box_sd_fast(px, ds(py, h), pz, g.half, ok[3]);
    const double s4 = box_sd_fast(px, py, da(pz, h), g.half, ok[4]), s5 = box_sd_fast(px, py, ds(pz, h), g.half, ok[5]);
    gx = ds(s0, s1);
    gy = ds(s2, s3);
    gz = ds(s4, s5);
    if (!(ok[0] & ok[1] & ok[2] & ok[3] & ok[4] & ok[5])) {
      gx = ds(box_sd(da(px, h), py, pz, g.half), box_sd(ds(px, h), py, pz, g.half));
      gy = ds(box_sd(px, da(py, h), pz, g.half), box_sd(px, ds(py, h), pz, g.half));
      gz = ds(box_sd(px, py, da(pz, h), g.half), box_sd(px, py, ds(pz, h), g.half));
    }
  } else {
    gx = ds(baked_sd(g, cs.sdf, da(px, h), py, pz), baked_sd(g, cs.sdf, ds(px, h), py, pz));
    gy = ds(baked_sd(g, cs.sdf, px, da(py, h), pz), baked_sd(g, cs.sdf, px, ds(py, h), pz));
    gz = ds(baked_sd(g, cs.sdf, px, py, da(pz, h)), baked_sd(g, cs.sdf, px, py, ds(pz, h)));
  }
  // axis-aligned gradient (a face): norm = |g| exactly (see box_sd_fast) and
  // g / norm = (+-1, +-0, +-0) -- the divisions are exact, so skip them
  const double ag = gx != 0.0 ? fabs(gx) : gy != 0.0 ? fabs(gy) : fabs(gz);
  if (((int)(gx != 0.0) + (int)(gy != 0.0) + (int)(gz != 0.0) == 1) & (ag >= 1.0e-12) & (ag < 1e150)) {
    gx = gx > 0.0 ? 1.0 : gx < 0.0 ? -1.0 : gx;
    gy = gy > 0.0 ? 1.0 : gy < 0.0 ? -1.0 : gy;
    gz = gz > 0.0 ? 1.0 : gz < 0.0 ? -1.0 : gz;
    n[0] = da(da(dm(q.R[0], gx), dm(q.R[1], gy)), dm(q.R[2], gz));
    n[1] = da(da(dm(q.R[3], gx), dm(q.R[4], gy)), dm(q.R[5], gz));
    n[2] = da(da(dm(q.R[6], gx), dm(q.R[7], gy)), dm(q.R[8], gz));
    return;
  }
  double norm = __dsqrt_rn(da(da(dm(gx, gx), dm(gy, gy)), dm(gz, gz)));
  if (norm < 1.0e-12) {
    double fx = ds(wx, q.T[0]), fy = ds(wy, q.T[1]), fz = ds(wz, q.T[2]);
    double fn = __dsqrt_rn(da(da(dm(fx, fx), dm(fy, fy)), dm(fz, fz)));
    if (fn < 1.0e-12) {
      n[0] = 0.0; n[1] = 1.0; n[2] = 0.0;
      return;
    }
    n[0] = __ddiv_rn(fx, fn); n[1] = __ddiv_rn(fy, fn); n[2] = __ddiv_rn(fz, fn);
    return;
  }
  gx = __ddiv_rn(gx, norm); gy = __ddiv_rn(gy, norm); gz = __ddiv_rn(gz, norm);
  n[0] = da(da(dm(q.R[0], gx), dm(q.R[1], gy)), dm(q.R[2], gz));
  n[1] = da(da(dm(q.R[3], gx), dm(q.R[4], gy)), dm(q.R[5], gz));
  n[2] = da(da(dm(q.R[6], gx), dm(q.R[7], gy)), dm(q.R[8], gz));
}

// Contact response at a massive node inside the band (kernels.py:371-411).
__device__ inline void resolve_contact(const Colliders& cs, int ci, double wx, double wy, double wz,
                                       double v[3]) {
#ifdef FUSED_PROFILE
  long long tp = clock64();
#endif
  const ColliderPose& q = cs.pose[ci];
  double rx = ds(wx, q.T[0]), ry = ds(wy, q.T[1]), rz = ds(wz, q.T[2]);
  double co0 = ds(da(q.lv[0], dm(q.av[1], rz)), dm(q.av[2], ry));
  double co1 = ds(da(q.lv[1], dm(q.av[2], rx)), dm(q.av[0], rz));
  double co2 = ds(da(q.lv[2], dm(q.av[0], ry)), dm(q.av[1], rx));
  double r0 = ds(v[0], co0), r1 = ds(v[1], co1), r2 = ds(v[2], co2);
  double n[3];
  CPH_MARK(1, tp);
  world_normal(cs, ci, wx, wy, wz, n);
  CPH_MARK(2, tp);
  double vn = da(da(dm(r0, n[0]), dm(r1, n[1])), dm(r2, n[2]));
  if (!(vn < 0.0)) return;
  if (q.mode == 1) {
    v[0] = co0; v[1] = co1; v[2] = co2;
    return;
  }
  double t0 = ds(r0, dm(vn, n[0])), t1 = ds(r1, dm(vn, n[1])), t2 = ds(r2, dm(vn, n[2]));
  double tn = __dsqrt_rn(da(da(dm(t0, t0), dm(t1, t1)), dm(t2, t2)));
  double muf = cs.geo[ci].fric;
  if (tn <= dm(muf, -vn)) {
    v[0] = co0; v[1] = co1; v[2] = co2;
  } else {
    double scale = da(1.0, __ddiv_rn(dm(muf, vn), tn));
    v[0] = da(dm(t0, scale), co0);
    v[1] = da(dm(t1, scale), co1);
    v[2] = da(dm(t2, scale), co2);
  }
}

}  // namespace mpm
