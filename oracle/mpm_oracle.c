/*
 * mpm_oracle.c -- CPU restatement of the reference MLS-MPM substep.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path links or calls this
 * file: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` leg load liboracle.so, and only as the checker or as the
 * timed CPU baseline.
 *
 * What it restates (all file:line citations are into the reference package
 * /root/reference/pkg/src/softmpm):
 *
 *   O1 (fp64, drop-in parity target) -- the numba kernels of kernels.py with
 *      the same arithmetic order (left-to-right sums, no FMA contraction:
 *      build with -ffp-contract=off, numba runs with fastmath off,
 *      kernels.py:12) and the same fixed-chunk deterministic accumulation
 *      (kernels.py:8-12):
 *        orc_p2g_scatter         kernels.py:198-314  (stress_form 0 = the
 *                                kernel's F^-1 form, 1 = the spec F^-T form,
 *                                SURVEY F1)
 *        orc_p2g_reduce          kernels.py:317-340
 *        orc_build_collision_field kernels.py:161-191 (+ helpers 30-158)
 *        orc_grid_update         kernels.py:347-436
 *        orc_g2p_advect          kernels.py:443-534
 *        orc_substep             core.py:261-277 (p2g -> field -> grid -> g2p)
 *   O2 (fp64 loop-nest spec oracle) -- reference.py:14-200 (F^-T stress,
 *      no colliders): orc_reference_substep.
 *   O3 (fp32 deterministic-order P2G) -- not in the reference: the summation
 *      order the GPU "sorted deterministic" mode promises (ascending
 *      (base-cell key, original particle index), sequential from 0.0f,
 *      explicit round-to-nearest products and sums) so grid mass can be
 *      checked bit-for-bit: orc32_p2g_sorted.
 *
 * Parallelism: the chunked kernels use OpenMP over chunks / nodes / particles
 * exactly where numba uses prange, so results do not depend on thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define BIG_DISTANCE 1.0e30
#define KIND_BOX 0
#define KIND_BAKED 1
#define MODE_STICKY 1

int orc_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void orc_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

/* Quadratic B-spline stencil of one coordinate (kernels.py:277-294). */
static inline void stencil_axis(double xc, double inv_dx, long *base, double *frac,
                                double w[3]) {
  double g = xc * inv_dx;
  long b = (long)floor(g - 0.5);
  double f = g - (double)b;
  double t0 = 1.5 - f, t1 = f - 1.0, t2 = f - 0.5;
  w[0] = 0.5 * (t0 * t0);
  w[1] = 0.75 - t1 * t1;
  w[2] = 0.5 * (t2 * t2);
  *base = b;
  *frac = f;
}

/* ------------------------------------------------------------------------- */
/* collider geometry (kernels.py:30-158)                                     */
/* ------------------------------------------------------------------------- */

typedef struct {
  int ncol;
  const int32_t *kind;     /* (k,)   */
  const double *half;      /* (k,3)  */
  const double *R;         /* (k,3,3) row-major */
  const double *T;         /* (k,3)  */
  const double *lin_vel;   /* (k,3)  */
  const double *ang_vel;   /* (k,3)  */
  const double *fric;      /* (k,)   */
  const int32_t *mode;     /* (k,)   */
  const double *sdf_vals;  /* flat, x-fastest per collider */
  const int64_t *sdf_off;  /* (k,)   */
  const int32_t *sdf_res;  /* (k,3)  */
  const double *sdf_bmin;  /* (k,3)  */
  const double *sdf_ext;   /* (k,)   */
} colliders_t;

static double box_sd(double px, double py, double pz, double hx, double hy, double hz) {
  double qx = fabs(px) - hx, qy = fabs(py) - hy, qz = fabs(pz) - hz;
  double ox = qx > 0.0 ? qx : 0.0;
  double oy = qy > 0.0 ? qy : 0.0;
  double oz = qz > 0.0 ? qz : 0.0;
  double outside = sqrt(ox * ox + oy * oy + oz * oz);
  double qm = qx;
  if (qy > qm) qm = qy;
  if (qz > qm) qm = qz;
  return outside + (qm < 0.0 ? qm : 0.0);
}

static double baked_sd(const colliders_t *c, int ci, double px, double py, double pz) {
  const double *bmin = c->sdf_bmin + 3 * ci;
  double ext = c->sdf_ext[ci];
  long rx = c->sdf_res[3 * ci], ry = c->sdf_res[3 * ci + 1], rz = c->sdf_res[3 * ci + 2];
  double q[3] = {(px - bmin[0]) / ext * (double)rx - 0.5,
                 (py - bmin[1]) / ext * (double)ry - 0.5,
                 (pz - bmin[2]) / ext * (double)rz - 0.5};
  long r[3] = {rx, ry, rz}, i0[3];
  double fr[3];
  for (int a = 0; a < 3; ++a) {
    if (q[a] < 0.0) q[a] = 0.0;
    if (q[a] > (double)r[a] - 1.0) q[a] = (double)r[a] - 1.0;
    long ii = (long)q[a];
    if (ii > r[a] - 2) ii = r[a] - 2;
    i0[a] = ii;
    fr[a] = q[a] - (double)ii;
  }
  const double *vals = c->sdf_vals + c->sdf_off[ci];
  double s = 0.0;
  for (int a = 0; a < 2; ++a) {
    double wa = a ? fr[0] : 1.0 - fr[0];
    for (int b = 0; b < 2; ++b) {
      double wb = b ? fr[1] : 1.0 - fr[1];
      for (int cc = 0; cc < 2; ++cc) {
        double wc = cc ? fr[2] : 1.0 - fr[2];
        long idx = (i0[0] + a) + rx * ((i0[1] + b) + ry * (i0[2] + cc));
        s += wa * wb * wc * vals[idx];
      }
    }
  }
  return s * ext;
}

static double local_sd(const colliders_t *c, int ci, double px, double py, double pz) {
  if (c->kind[ci] == KIND_BOX)
    return box_sd(px, py, pz, c->half[3 * ci], c->half[3 * ci + 1], c->half[3 * ci + 2]);
  return baked_sd(c, ci, px, py, pz);
}

/* x_ref = R^T (x - T) */
static void to_local(const colliders_t *c, int ci, double wx, double wy, double wz,
                     double *px, double *py, double *pz) {
  const double *R = c->R + 9 * ci, *T = c->T + 3 * ci;
  double d0 = wx - T[0], d1 = wy - T[1], d2 = wz - T[2];
  *px = R[0] * d0 + R[3] * d1 + R[6] * d2;
  *py = R[1] * d0 + R[4] * d1 + R[7] * d2;
  *pz = R[2] * d0 + R[5] * d1 + R[8] * d2;
}

static double world_sd(const colliders_t *c, int ci, double wx, double wy, double wz) {
  double px, py, pz;
  to_local(c, ci, wx, wy, wz, &px, &py, &pz);
  return local_sd(c, ci, px, py, pz);
}

static void world_normal(const colliders_t *c, int ci, double wx, double wy, double wz,
                         double n[3]) {
  double px, py, pz;
  to_local(c, ci, wx, wy, wz, &px, &py, &pz);
  double h;
  if (c->kind[ci] == KIND_BOX) {
    const double *hh = c->half + 3 * ci;
    h = hh[0];
    if (hh[1] < h) h = hh[1];
    if (hh[2] < h) h = hh[2];
    h = 1.0e-3 * h;
    if (h < 1.0e-6) h = 1.0e-6;
  } else {
    h = c->sdf_ext[ci] / (double)c->sdf_res[3 * ci];
  }
  double gx = local_sd(c, ci, px + h, py, pz) - local_sd(c, ci, px - h, py, pz);
  double gy = local_sd(c, ci, px, py + h, pz) - local_sd(c, ci, px, py - h, pz);
  double gz = local_sd(c, ci, px, py, pz + h) - local_sd(c, ci, px, py, pz - h);
  double norm = sqrt(gx * gx + gy * gy + gz * gz);
  const double *T = c->T + 3 * ci;
  if (norm < 1.0e-12) {
    double fx = wx - T[0], fy = wy - T[1], fz = wz - T[2];
    double fn = sqrt(fx * fx + fy * fy + fz * fz);
    if (fn < 1.0e-12) {
      n[0] = 0.0; n[1] = 1.0; n[2] = 0.0;
      return;
    }
    n[0] = fx / fn; n[1] = fy / fn; n[2] = fz / fn;
    return;
  }
  gx /= norm; gy /= norm; gz /= norm;
  const double *R = c->R + 9 * ci;
  n[0] = R[0] * gx + R[1] * gy + R[2] * gz;
  n[1] = R[3] * gx + R[4] * gy + R[5] * gz;
  n[2] = R[6] * gx + R[7] * gy + R[8] * gz;
}

void orc_build_collision_field(double dx, int nx, int ny, int nz, double *dist,
                               int32_t *obj, double cap, int ncol, const int32_t *kind,
                               const double *half, const double *R, const double *T,
                               const double *sdf_vals, const int64_t *sdf_off,
                               const int32_t *sdf_res, const double *sdf_bmin,
                               const double *sdf_ext) {
  colliders_t c = {ncol, kind, half, R, T, NULL, NULL, NULL, NULL,
                   sdf_vals, sdf_off, sdf_res, sdf_bmin, sdf_ext};
  long nn = (long)nx * ny * nz;
#pragma omp parallel for schedule(static)
  for (long node = 0; node < nn; ++node) {
    long ix = node / ((long)ny * nz), rem = node - ix * ((long)ny * nz);
    long iy = rem / nz, iz = rem - iy * nz;
    double best = BIG_DISTANCE;
    int best_id = -1;
    for (int ci = 0; ci < ncol; ++ci) {
      double d = world_sd(&c, ci, (double)ix * dx, (double)iy * dx, (double)iz * dx);
      if (d < best) {
        best = d;
        best_id = ci;
      }
    }
    dist[node] = best;
    obj[node] = best >= cap ? -1 : best_id;
  }
}

/* ------------------------------------------------------------------------- */
/* P2G (kernels.py:198-340)                                                  */
/* ------------------------------------------------------------------------- */

/* Affine momentum matrix A = m C + k P F'^T with F' = (I + dt C) F written
 * back (kernels.py:213-275).  Returns 1 when det(F') <= 0. */
static int particle_affine(double *Fp, const double *Cp, double m, double vol0,
                           double mu, double lam, double dt, double stress_coef,
                           int stress_form, double A[9]) {
  double f[9];
  for (int r = 0; r < 3; ++r)
    for (int col = 0; col < 3; ++col)
      f[3 * r + col] = Fp[3 * r + col] +
                       dt * (Cp[3 * r] * Fp[col] + Cp[3 * r + 1] * Fp[3 + col] +
                             Cp[3 * r + 2] * Fp[6 + col]);
  memcpy(Fp, f, sizeof f);
  /* cofactors cof[i][j] of f (so that f^-T = cof / det) */
  double cof[9];
  cof[0] = f[4] * f[8] - f[5] * f[7];
  cof[1] = f[5] * f[6] - f[3] * f[8];
  cof[2] = f[3] * f[7] - f[4] * f[6];
  double det = f[0] * cof[0] + f[1] * cof[1] + f[2] * cof[2];
  cof[3] = f[2] * f[7] - f[1] * f[8];
  cof[4] = f[0] * f[8] - f[2] * f[6];
  cof[5] = f[1] * f[6] - f[0] * f[7];
  cof[6] = f[1] * f[5] - f[2] * f[4];
  cof[7] = f[2] * f[3] - f[0] * f[5];
  cof[8] = f[0] * f[4] - f[1] * f[3];
  double j_safe = det > 1.0e-6 ? det : 1.0e-6;
  double log_j = log(j_safe);
  double inv_det = det != 0.0 ? 1.0 / det : 0.0;
  double g = (lam * log_j - mu) * inv_det;
  double P[9];
  for (int r = 0; r < 3; ++r)
    for (int col = 0; col < 3; ++col) {
      /* kernel form pairs P[r][c] with cof[c][r] (F^-1, kernels.py:254-262);
       * spec form with cof[r][c] (F^-T, materials.py:59-60) */
      double cv = stress_form == 0 ? cof[3 * col + r] : cof[3 * r + col];
      P[3 * r + col] = mu * f[3 * r + col] + g * cv;
    }
  double k = stress_coef * vol0;
  for (int r = 0; r < 3; ++r)
    for (int col = 0; col < 3; ++col)
      A[3 * r + col] = m * Cp[3 * r + col] +
                       k * (P[3 * r] * f[3 * col] + P[3 * r + 1] * f[3 * col + 1] +
                            P[3 * r + 2] * f[3 * col + 2]);
  return det <= 0.0;
}

void orc_p2g_scatter(long n, const double *x, const double *v, double *F, const double *C,
                     const double *mass, const double *vol0, const int32_t *mat_id,
                     const double *mu_arr, const double *lam_arr, double dt, double dx,
                     int ny, int nz, long nn, double *buf, int nchunks,
                     int64_t *inverted_counts, int stress_form) {
  double inv_dx = 1.0 / dx;
  double stress_coef = -4.0 * dt * inv_dx * inv_dx;
#pragma omp parallel for schedule(static, 1)
  for (int c = 0; c < nchunks; ++c) {
    long lo = (long)c * n / nchunks, hi = (long)(c + 1) * n / nchunks;
    double *cb = buf + (size_t)c * nn * 4;
    int64_t inverted = 0;
    for (long p = lo; p < hi; ++p) {
      double A[9];
      int mid = mat_id[p];
      inverted += particle_affine(F + 9 * p, C + 9 * p, mass[p], vol0[p], mu_arr[mid],
                                  lam_arr[mid], dt, stress_coef, stress_form, A);
      long b[3];
      double fr[3], w[3][3];
      for (int a = 0; a < 3; ++a) stencil_axis(x[3 * p + a], inv_dx, &b[a], &fr[a], w[a]);
      double m = mass[p];
      double mv0 = m * v[3 * p], mv1 = m * v[3 * p + 1], mv2 = m * v[3 * p + 2];
      for (int i = 0; i < 3; ++i) {
        double dp0 = ((double)i - fr[0]) * dx;
        for (int j = 0; j < 3; ++j) {
          double wij = w[0][i] * w[1][j];
          double dp1 = ((double)j - fr[1]) * dx;
          long row = ((b[0] + i) * ny + (b[1] + j)) * nz + b[2];
          for (int kk = 0; kk < 3; ++kk) {
            double wt = wij * w[2][kk];
            double dp2 = ((double)kk - fr[2]) * dx;
            double *cell = cb + (row + kk) * 4;
            cell[0] += wt * (mv0 + A[0] * dp0 + A[1] * dp1 + A[2] * dp2);
            cell[1] += wt * (mv1 + A[3] * dp0 + A[4] * dp1 + A[5] * dp2);
            cell[2] += wt * (mv2 + A[6] * dp0 + A[7] * dp1 + A[8] * dp2);
            cell[3] += wt * m;
          }
        }
      }
    }
    inverted_counts[c] = inverted;
  }
}

void orc_p2g_reduce(double *buf, double *grid_mv, double *grid_m, long nn, int nchunks) {
#pragma omp parallel for schedule(static)
  for (long node = 0; node < nn; ++node) {
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    for (int c = 0; c < nchunks; ++c) {
      double *e = buf + ((size_t)c * nn + node) * 4;
      for (int q = 0; q < 4; ++q) {
        s[q] += e[q];
        e[q] = 0.0;
      }
    }
    grid_mv[3 * node] = s[0];
    grid_mv[3 * node + 1] = s[1];
    grid_mv[3 * node + 2] = s[2];
    grid_m[node] = s[3];
  }
}

/* ------------------------------------------------------------------------- */
/* grid update (kernels.py:347-436)                                          */
/* ------------------------------------------------------------------------- */

void orc_grid_update(double *grid_mv, const double *grid_m, int nx, int ny, int nz,
                     double dt, double gx, double gy, double gz, double dx, int bwidth,
                     int stick, double theta, const double *col_dist,
                     const int32_t *col_obj, int ncol, const int32_t *kind,
                     const double *half, const double *R, const double *T,
                     const double *lin_vel, const double *ang_vel, const double *fric,
                     const int32_t *mode, const double *sdf_vals, const int64_t *sdf_off,
                     const int32_t *sdf_res, const double *sdf_bmin,
                     const double *sdf_ext) {
  colliders_t c = {ncol, kind, half, R, T, lin_vel, ang_vel, fric, mode,
                   sdf_vals, sdf_off, sdf_res, sdf_bmin, sdf_ext};
  long nn = (long)nx * ny * nz;
#pragma omp parallel for schedule(static)
  for (long node = 0; node < nn; ++node) {
    long ix = node / ((long)ny * nz), rem = node - ix * ((long)ny * nz);
    long iy = rem / nz, iz = rem - iy * nz;
    double m = grid_m[node];
    if (m <= 0.0) continue;
    double inv_m = 1.0 / m;
    double *mv = grid_mv + 3 * node;
    double v[3] = {mv[0] * inv_m + dt * gx, mv[1] * inv_m + dt * gy,
                   mv[2] * inv_m + dt * gz};
    if (theta >= 0.0 && col_dist[node] < theta) {
      int ci = col_obj[node];
      if (ci >= 0) {
        double w[3] = {(double)ix * dx, (double)iy * dx, (double)iz * dx};
        const double *Tc = T + 3 * ci, *lv = lin_vel + 3 * ci, *av = ang_vel + 3 * ci;
        double r[3] = {w[0] - Tc[0], w[1] - Tc[1], w[2] - Tc[2]};
        double co[3] = {lv[0] + av[1] * r[2] - av[2] * r[1],
                        lv[1] + av[2] * r[0] - av[0] * r[2],
                        lv[2] + av[0] * r[1] - av[1] * r[0]};
        double rel[3] = {v[0] - co[0], v[1] - co[1], v[2] - co[2]};
        double nrm[3];
        world_normal(&c, ci, w[0], w[1], w[2], nrm);
        double vn = rel[0] * nrm[0] + rel[1] * nrm[1] + rel[2] * nrm[2];
        if (vn < 0.0) {
          if (mode[ci] == MODE_STICKY) {
            v[0] = co[0]; v[1] = co[1]; v[2] = co[2];
          } else {
            double t[3] = {rel[0] - vn * nrm[0], rel[1] - vn * nrm[1], rel[2] - vn * nrm[2]};
            double tn = sqrt(t[0] * t[0] + t[1] * t[1] + t[2] * t[2]);
            double mu_f = fric[ci];
            if (tn <= mu_f * (-vn)) {
              v[0] = co[0]; v[1] = co[1]; v[2] = co[2];
            } else {
              double scale = 1.0 + mu_f * vn / tn;
              for (int a = 0; a < 3; ++a) v[a] = t[a] * scale + co[a];
            }
          }
        }
      }
    }
    long idx[3] = {ix, iy, iz}, res[3] = {nx, ny, nz};
    if (stick) {
      int band = 0;
      for (int a = 0; a < 3; ++a)
        if (idx[a] < bwidth || idx[a] >= res[a] - bwidth) band = 1;
      if (band) v[0] = v[1] = v[2] = 0.0;
    } else {
      for (int a = 0; a < 3; ++a) {
        if (idx[a] < bwidth && v[a] < 0.0) v[a] = 0.0;
        if (idx[a] >= res[a] - bwidth && v[a] > 0.0) v[a] = 0.0;
      }
    }
    mv[0] = v[0]; mv[1] = v[1]; mv[2] = v[2];
  }
}

/* ------------------------------------------------------------------------- */
/* G2P + advection (kernels.py:443-534)                                      */
/* ------------------------------------------------------------------------- */

void orc_g2p_advect(long n, double *x, double *v, double *C, const double *grid_v,
                    int ny, int nz, double dt, double dx, double hi_x, double hi_y,
                    double hi_z) {
  double inv_dx = 1.0 / dx;
  double coef = 4.0 * inv_dx * inv_dx;
  double lo = 1.5 * dx;
  double hi[3] = {hi_x, hi_y, hi_z};
#pragma omp parallel for schedule(static)
  for (long p = 0; p < n; ++p) {
    long b[3];
    double fr[3], w[3][3];
    for (int a = 0; a < 3; ++a) stencil_axis(x[3 * p + a], inv_dx, &b[a], &fr[a], w[a]);
    double nv[3] = {0.0, 0.0, 0.0};
    double cc[9] = {0.0};
    for (int i = 0; i < 3; ++i) {
      double dp0 = ((double)i - fr[0]) * dx;
      for (int j = 0; j < 3; ++j) {
        double wij = w[0][i] * w[1][j];
        double dp1 = ((double)j - fr[1]) * dx;
        for (int kk = 0; kk < 3; ++kk) {
          double wt = wij * w[2][kk];
          double dp2 = ((double)kk - fr[2]) * dx;
          const double *g = grid_v + 3 * (((b[0] + i) * ny + (b[1] + j)) * nz + b[2] + kk);
          double dp[3] = {dp0, dp1, dp2};
          for (int a = 0; a < 3; ++a) nv[a] += wt * g[a];
          for (int a = 0; a < 3; ++a)
            for (int q = 0; q < 3; ++q) cc[3 * a + q] += coef * wt * g[a] * dp[q];
        }
      }
    }
    for (int a = 0; a < 3; ++a) v[3 * p + a] = nv[a];
    memcpy(C + 9 * p, cc, sizeof cc);
    for (int a = 0; a < 3; ++a) {
      double q = x[3 * p + a] + dt * nv[a];
      if (q < lo) q = lo;
      if (q > hi[a]) q = hi[a];
      x[3 * p + a] = q;
    }
  }
}

/* ------------------------------------------------------------------------- */
/* whole substep (core.py:261-277), O1                                       */
/* ------------------------------------------------------------------------- */

typedef struct {
  int nx, ny, nz;
  double dx, dt, gx, gy, gz;
  int bwidth, stick;
  double theta; /* < 0: no colliders; else collision band (core.py:268-269) */
  double hi[3];
  int nchunks;
  int stress_form;
} orc_params;

/* One substep on caller-owned fp64 state.  buf: (nchunks, nodes, 4) zeroed,
 * dist/obj: node-sized scratch.  Returns the inverted-element count. */
int64_t orc_substep(const orc_params *pp, long n, double *x, double *v, double *F,
                    double *C, const double *mass, const double *vol0,
                    const int32_t *mat_id, const double *mu_arr, const double *lam_arr,
                    double *grid_mv, double *grid_m, double *buf, double *dist,
                    int32_t *obj, int ncol, const int32_t *kind, const double *half,
                    const double *R, const double *T, const double *lin_vel,
                    const double *ang_vel, const double *fric, const int32_t *mode,
                    const double *sdf_vals, const int64_t *sdf_off,
                    const int32_t *sdf_res, const double *sdf_bmin,
                    const double *sdf_ext) {
  long nn = (long)pp->nx * pp->ny * pp->nz;
  int64_t inv[256];
  int nch = pp->nchunks > 256 ? 256 : pp->nchunks;
  orc_p2g_scatter(n, x, v, F, C, mass, vol0, mat_id, mu_arr, lam_arr, pp->dt, pp->dx,
                  pp->ny, pp->nz, nn, buf, nch, inv, pp->stress_form);
  orc_p2g_reduce(buf, grid_mv, grid_m, nn, nch);
  double theta = -1.0;
  if (ncol > 0 && pp->theta >= 0.0) {
    theta = pp->theta;
    orc_build_collision_field(pp->dx, pp->nx, pp->ny, pp->nz, dist, obj, 2.0 * theta, ncol,
                              kind, half, R, T, sdf_vals, sdf_off, sdf_res, sdf_bmin,
                              sdf_ext);
  }
  orc_grid_update(grid_mv, grid_m, pp->nx, pp->ny, pp->nz, pp->dt, pp->gx, pp->gy, pp->gz,
                  pp->dx, pp->bwidth, pp->stick, theta, dist, obj, ncol, kind, half, R, T,
                  lin_vel, ang_vel, fric, mode, sdf_vals, sdf_off, sdf_res, sdf_bmin,
                  sdf_ext);
  orc_g2p_advect(n, x, v, C, grid_mv, pp->ny, pp->nz, pp->dt, pp->dx, pp->hi[0], pp->hi[1],
                 pp->hi[2]);
  int64_t tot = 0;
  for (int c = 0; c < nch; ++c) tot += inv[c];
  return tot;
}

/* ------------------------------------------------------------------------- */
/* O2: loop-nest spec oracle (reference.py:14-200)                           */
/* ------------------------------------------------------------------------- */

void orc_reference_substep(long n, double *x, double *v, double *F, double *C,
                           const double *mass, const double *vol0, const int32_t *mat_id,
                           const double *mu_arr, const double *lam_arr, double *grid_mv,
                           double *grid_m, int nx, int ny, int nz, double dt, double dx,
                           double gx, double gy, double gz, int bwidth, int stick,
                           double hi_x, double hi_y, double hi_z) {
  long nn = (long)nx * ny * nz;
  double inv_dx = 1.0 / dx;
  memset(grid_mv, 0, sizeof(double) * 3 * nn);
  memset(grid_m, 0, sizeof(double) * nn);
  for (long p = 0; p < n; ++p) {
    double Fn[9];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double s = F[9 * p + 3 * i + j];
        for (int k = 0; k < 3; ++k) s += dt * C[9 * p + 3 * i + k] * F[9 * p + 3 * k + j];
        Fn[3 * i + j] = s;
      }
    memcpy(F + 9 * p, Fn, sizeof Fn);
    double det = Fn[0] * (Fn[4] * Fn[8] - Fn[5] * Fn[7]) - Fn[1] * (Fn[3] * Fn[8] - Fn[5] * Fn[6]) +
                 Fn[2] * (Fn[3] * Fn[7] - Fn[4] * Fn[6]);
    double id = 1.0 / det;
    double Fit[9];
    Fit[0] = (Fn[4] * Fn[8] - Fn[5] * Fn[7]) * id;
    Fit[1] = (Fn[5] * Fn[6] - Fn[3] * Fn[8]) * id;
    Fit[2] = (Fn[3] * Fn[7] - Fn[4] * Fn[6]) * id;
    Fit[3] = (Fn[2] * Fn[7] - Fn[1] * Fn[8]) * id;
    Fit[4] = (Fn[0] * Fn[8] - Fn[2] * Fn[6]) * id;
    Fit[5] = (Fn[1] * Fn[6] - Fn[0] * Fn[7]) * id;
    Fit[6] = (Fn[1] * Fn[5] - Fn[2] * Fn[4]) * id;
    Fit[7] = (Fn[2] * Fn[3] - Fn[0] * Fn[5]) * id;
    Fit[8] = (Fn[0] * Fn[4] - Fn[1] * Fn[3]) * id;
    double mu = mu_arr[mat_id[p]], lam = lam_arr[mat_id[p]];
    double js = det > 1.0e-6 ? det : 1.0e-6;
    double lj = log(js);
    double P[9], A[9];
    for (int q = 0; q < 9; ++q) P[q] = mu * (Fn[q] - Fit[q]) + lam * lj * Fit[q];
    double m = mass[p];
    double coef = -4.0 * dt * inv_dx * inv_dx * vol0[p];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double s = 0.0;
        for (int k = 0; k < 3; ++k) s += P[3 * i + k] * Fn[3 * j + k];
        A[3 * i + j] = m * C[9 * p + 3 * i + j] + coef * s;
      }
    long b[3];
    double fr[3], w[3][3];
    for (int a = 0; a < 3; ++a) stencil_axis(x[3 * p + a], inv_dx, &b[a], &fr[a], w[a]);
    for (int i = 0; i < 3; ++i) {
      double dp0 = ((double)i - fr[0]) * dx;
      for (int j = 0; j < 3; ++j) {
        double dp1 = ((double)j - fr[1]) * dx;
        for (int k = 0; k < 3; ++k) {
          double dp2 = ((double)k - fr[2]) * dx;
          double wt = w[0][i] * w[1][j] * w[2][k];
          long node = ((b[0] + i) * ny + (b[1] + j)) * nz + b[2] + k;
          for (int a = 0; a < 3; ++a)
            grid_mv[3 * node + a] +=
                wt * (m * v[3 * p + a] + A[3 * a] * dp0 + A[3 * a + 1] * dp1 + A[3 * a + 2] * dp2);
          grid_m[node] += wt * m;
        }
      }
    }
  }
  for (long node = 0; node < nn; ++node) {
    long gi = node / ((long)ny * nz), rem = node - gi * ((long)ny * nz);
    long gj = rem / nz, gk = rem - gj * nz;
    double m = grid_m[node];
    if (m <= 0.0) continue;
    double vv[3] = {grid_mv[3 * node] / m + dt * gx, grid_mv[3 * node + 1] / m + dt * gy,
                    grid_mv[3 * node + 2] / m + dt * gz};
    long idx[3] = {gi, gj, gk}, res[3] = {nx, ny, nz};
    if (stick) {
      int band = 0;
      for (int a = 0; a < 3; ++a)
        if (idx[a] < bwidth || idx[a] >= res[a] - bwidth) band = 1;
      if (band) vv[0] = vv[1] = vv[2] = 0.0;
    } else {
      for (int a = 0; a < 3; ++a) {
        if (idx[a] < bwidth && vv[a] < 0.0) vv[a] = 0.0;
        if (idx[a] >= res[a] - bwidth && vv[a] > 0.0) vv[a] = 0.0;
      }
    }
    for (int a = 0; a < 3; ++a) grid_mv[3 * node + a] = vv[a];
  }
  double lo = 1.5 * dx, hi[3] = {hi_x, hi_y, hi_z};
  for (long p = 0; p < n; ++p) {
    long b[3];
    double fr[3], w[3][3];
    for (int a = 0; a < 3; ++a) stencil_axis(x[3 * p + a], inv_dx, &b[a], &fr[a], w[a]);
    double nv[3] = {0.0, 0.0, 0.0};
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j)
        for (int k = 0; k < 3; ++k) {
          double wt = w[0][i] * w[1][j] * w[2][k];
          const double *g = grid_mv + 3 * (((b[0] + i) * ny + (b[1] + j)) * nz + b[2] + k);
          for (int a = 0; a < 3; ++a) nv[a] += wt * g[a];
        }
    double coef = 4.0 * inv_dx * inv_dx;
    for (int a = 0; a < 3; ++a)
      for (int bb = 0; bb < 3; ++bb) {
        double s = 0.0;
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j)
            for (int k = 0; k < 3; ++k) {
              double wt = w[0][i] * w[1][j] * w[2][k];
              double gv = grid_mv[3 * (((b[0] + i) * ny + (b[1] + j)) * nz + b[2] + k) + a];
              double d = bb == 0 ? ((double)i - fr[0]) * dx
                                 : (bb == 1 ? ((double)j - fr[1]) * dx : ((double)k - fr[2]) * dx);
              s += coef * wt * gv * d;
            }
        C[9 * p + 3 * a + bb] = s;
      }
    for (int a = 0; a < 3; ++a) {
      v[3 * p + a] = nv[a];
      double q = x[3 * p + a] + dt * v[3 * p + a];
      if (q < lo) q = lo;
      if (q > hi[a]) q = hi[a];
      x[3 * p + a] = q;
    }
  }
}

/* ------------------------------------------------------------------------- */
/* O3: fp32 deterministic-order P2G                                          */
/* ------------------------------------------------------------------------- */

/*
 * Same physics as orc_p2g_scatter, in fp32, scattered in the order given by
 * `order` (the GPU's sorted permutation: ascending base-cell key, ties by
 * original index).  Every product and sum is a separately rounded fp32 op
 * (-ffp-contract=off), matching the explicit __fmul_rn/__fadd_rn chain of
 * the GPU deterministic gather kernel for the mass channel:
 *     w  = (wx[i] * wy[j]) * wz[k]
 *     m += w * mass
 * F is updated in place (fp32) and the momentum channel follows the same
 * order (its stress uses logf, so it is compared with a tolerance).
 */
static inline void stencil_axis32(float xc, float inv_dx, int r, int *base, float *frac,
                                  float w[3]) {
  float g = xc * inv_dx;
  int b = (int)floorf(g - 0.5f);
  if (b > r - 3) b = r - 3;
  if (b < 0) b = 0;
  float f = g - (float)b;
  float t0 = 1.5f - f, t1 = f - 1.0f, t2 = f - 0.5f;
  w[0] = 0.5f * (t0 * t0);
  w[1] = 0.75f - t1 * t1;
  w[2] = 0.5f * (t2 * t2);
  *base = b;
  *frac = f;
}

void orc32_p2g_sorted(long n, const int64_t *order, const float *x, const float *v, float *F,
                      const float *C, const float *mass, const float *vol0,
                      const int32_t *mat_id, const float *mu_arr, const float *lam_arr,
                      float dt, float dx, int nx, int ny, int nz, float *grid_mv, float *grid_m,
                      int stress_form, int64_t *inverted) {
  float inv_dx = 1.0f / dx;
  float stress_coef = -4.0f * dt * inv_dx * inv_dx;
  int64_t inv = 0;
  for (long q = 0; q < n; ++q) {
    long p = order ? order[q] : q;
    const float *Fp = F + 9 * p, *Cp = C + 9 * p;
    float f[9];
    for (int r = 0; r < 3; ++r)
      for (int col = 0; col < 3; ++col)
        f[3 * r + col] = Fp[3 * r + col] + dt * (Cp[3 * r] * Fp[col] + Cp[3 * r + 1] * Fp[3 + col] +
                                                 Cp[3 * r + 2] * Fp[6 + col]);
    memcpy(F + 9 * p, f, sizeof f);
    float cof[9];
    cof[0] = f[4] * f[8] - f[5] * f[7];
    cof[1] = f[5] * f[6] - f[3] * f[8];
    cof[2] = f[3] * f[7] - f[4] * f[6];
    float det = f[0] * cof[0] + f[1] * cof[1] + f[2] * cof[2];
    cof[3] = f[2] * f[7] - f[1] * f[8];
    cof[4] = f[0] * f[8] - f[2] * f[6];
    cof[5] = f[1] * f[6] - f[0] * f[7];
    cof[6] = f[1] * f[5] - f[2] * f[4];
    cof[7] = f[2] * f[3] - f[0] * f[5];
    cof[8] = f[0] * f[4] - f[1] * f[3];
    if (det <= 0.0f) ++inv;
    int mid = mat_id[p];
    float mu = mu_arr[mid], lam = lam_arr[mid];
    float js = det > 1.0e-6f ? det : 1.0e-6f;
    float lj = logf(js);
    float id = det != 0.0f ? 1.0f / det : 0.0f;
    float g = (lam * lj - mu) * id;
    float P[9], A[9];
    for (int r = 0; r < 3; ++r)
      for (int col = 0; col < 3; ++col) {
        float cv = stress_form == 0 ? cof[3 * col + r] : cof[3 * r + col];
        P[3 * r + col] = mu * f[3 * r + col] + g * cv;
      }
    float m = mass[p];
    float k = stress_coef * vol0[p];
    for (int r = 0; r < 3; ++r)
      for (int col = 0; col < 3; ++col)
        A[3 * r + col] = m * Cp[3 * r + col] +
                         k * (P[3 * r] * f[3 * col] + P[3 * r + 1] * f[3 * col + 1] +
                              P[3 * r + 2] * f[3 * col + 2]);
    int b[3];
    float fr[3], w[3][3];
    int rr[3] = {nx, ny, nz};
    for (int a = 0; a < 3; ++a) stencil_axis32(x[3 * p + a], inv_dx, rr[a], &b[a], &fr[a], w[a]);
    float mv[3] = {m * v[3 * p], m * v[3 * p + 1], m * v[3 * p + 2]};
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        float wij = w[0][i] * w[1][j];
        for (int kk = 0; kk < 3; ++kk) {
          float wt = wij * w[2][kk];
          float dp[3] = {((float)i - fr[0]) * dx, ((float)j - fr[1]) * dx,
                         ((float)kk - fr[2]) * dx};
          long node = ((long)(b[0] + i) * ny + (b[1] + j)) * nz + b[2] + kk;
          for (int a = 0; a < 3; ++a)
            grid_mv[3 * node + a] += wt * (mv[a] + A[3 * a] * dp[0] + A[3 * a + 1] * dp[1] +
                                           A[3 * a + 2] * dp[2]);
          grid_m[node] += wt * m;
        }
      }
  }
  if (inverted) *inverted = inv;
}

/* ------------------------------------------------------------------------- */
/* density splat (kernels.py:541-588, surfacing.py:45-67)                    */
/* ------------------------------------------------------------------------- */

/* kernels.splat_mass: chunk c deposits particles [c n / nchunks, (c + 1) n /
 * nchunks) into its private buffer, same expression order (weights
 * 0.5 * (t * t), w_ij = w_i * w_j, w = w_ij * w_k, buf += w * m).  The
 * reference does not bounds-check; nodes outside the lattice are skipped. */
void orc_splat_mass(long n, const double *x, const double *mass, double dx, int nx, int ny, int nz,
                    double *buf, int nchunks) {
  const double inv_dx = 1.0 / dx;
  const long nn = (long)nx * ny * nz;
#pragma omp parallel for schedule(static, 1)
  for (int c = 0; c < nchunks; ++c) {
    const long lo = (long)c * n / nchunks, hi = (long)(c + 1) * n / nchunks;
    double *cb = buf + (size_t)c * nn;
    for (long p = lo; p < hi; ++p) {
      double g[3], w[3][3];
      long b[3];
      for (int a = 0; a < 3; ++a) {
        g[a] = x[3 * p + a] * inv_dx;
        b[a] = (long)floor(g[a] - 0.5);
        const double f = g[a] - (double)b[a];
        w[a][0] = 0.5 * ((1.5 - f) * (1.5 - f));
        w[a][1] = 0.75 - (f - 1.0) * (f - 1.0);
        w[a][2] = 0.5 * ((f - 0.5) * (f - 0.5));
      }
      const double m = mass[p];
      for (int i = 0; i < 3; ++i) {
        const long xi = b[0] + i;
        for (int j = 0; j < 3; ++j) {
          const long yj = b[1] + j;
          const double wij = w[0][i] * w[1][j];
          for (int k = 0; k < 3; ++k) {
            const long zk = b[2] + k;
            if (xi < 0 || xi >= nx || yj < 0 || yj >= ny || zk < 0 || zk >= nz) continue;
            const double wt = wij * w[2][k];
            cb[(xi * ny + yj) * nz + zk] += wt * m;
          }
        }
      }
    }
  }
}

/* kernels.splat_reduce: node sums in chunk order 0..nchunks-1 from 0.0,
 * times 1/dx^3; buffers re-zeroed. */
void orc_splat_reduce(double *buf, double *out, long nn, int nchunks, double inv_cell_volume) {
#pragma omp parallel for schedule(static)
  for (long node = 0; node < nn; ++node) {
    double s = 0.0;
    for (int c = 0; c < nchunks; ++c) {
      s += buf[(size_t)c * nn + node];
      buf[(size_t)c * nn + node] = 0.0;
    }
    out[node] = s * inv_cell_volume;
  }
}
