// frame_ops.cuh -- frame consumers: metrics, density splat, marching cubes, frame encoding (sm_100a).
// Part of the kernel set included by kernels.cuh (namespace mpm).
#pragma once

namespace mpm {

// ---------------------------------------------------------------------------
// frame-level consumers of the state: metrics and density splat
// ---------------------------------------------------------------------------

// compute_metrics (scene.py:204-220) without a particle download: per block
// {lifted count, detached count, sum |det F - 1|, max |x - x0|} in fp64 over
// a fixed grid-stride partition (block partials are summed on the host in
// block order).  x0 is in the caller's order, indexed by original id.
constexpr int METRICS_THREADS = 256;

__global__ void __launch_bounds__(METRICS_THREADS) metrics_kernel(Params p, const double* __restrict__ x0, double dx,
                                                                  double* __restrict__ part) {
  double sum = 0.0, mx = 0.0, c_lift = 0.0, c_det = 0.0;
  for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < p.n;
       s += (long long)gridDim.x * blockDim.x) {
    const long long id = p.orig[s];
    // the device holds positions in fp32; a coordinate equal to the fp32
    // rounding of x0 did not move (the host mirror keeps the caller's fp64
    // value there, core.SimState._download), so its displacement is exactly
    // zero, as scene.py:210-219 computes it on the host state
    double d[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const float xa = ldf(p, FX + a, s);
      const double x0a = x0[3 * id + a];
      d[a] = xa == (float)x0a ? 0.0 : (double)xa - x0a;
    }
    const double d0 = d[0], d1 = d[1], d2 = d[2];
    c_lift += d1 > 2.0 * dx ? 1.0 : 0.0;
    c_det += d1 > dx ? 1.0 : 0.0;
    double F[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) F[q] = (double)ldf(p, FF + q, s);
    const double det = F[0] * (F[4] * F[8] - F[5] * F[7]) - F[1] * (F[3] * F[8] - F[5] * F[6]) +
                       F[2] * (F[3] * F[7] - F[4] * F[6]);
    sum += fabs(det - 1.0);
    mx = fmax(mx, sqrt(d0 * d0 + d1 * d1 + d2 * d2));
  }
  // fixed-order reduction: warp shuffles, then warps in index order
  for (int o = 16; o > 0; o >>= 1) {
    sum += __shfl_down_sync(0xffffffffu, sum, o);
    c_lift += __shfl_down_sync(0xffffffffu, c_lift, o);
    c_det += __shfl_down_sync(0xffffffffu, c_det, o);
    mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, o));
  }
  __shared__ double red[METRICS_THREADS / 32][4];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[w][0] = c_lift;
    red[w][1] = c_det;
    red[w][2] = sum;
    red[w][3] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double r[4] = {0.0, 0.0, 0.0, 0.0};
    for (int k = 0; k < METRICS_THREADS / 32; ++k) {
      r[0] += red[k][0];
      r[1] += red[k][1];
      r[2] += red[k][2];
      r[3] = fmax(r[3], red[k][3]);
    }
    for (int k = 0; k < 4; ++k) part[4 * blockIdx.x + k] = r[k];
  }
}

// splat_mass (kernels.py:541-576): quadratic B-spline mass deposit on a
// dense (rx, ry, rz) lattice of spacing 1/inv_dx, C order.  fp64 weights and
// fp64 atomic accumulation (partition of unity to ~1e-16, so the field
// integrates to the total mass); the caller scales by 1/dx^3
// (splat_reduce, kernels.py:579-588).  Source: the context's fp32
// particles (pos == nullptr) or caller fp64 arrays.  Nodes outside the
// lattice are skipped (the reference does not bounds-check).
__global__ void splat_kernel(Params p, const double* __restrict__ pos, const double* __restrict__ mass, long long n,
                             int rx, int ry, int rz, double inv_dx, double* __restrict__ out) {
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s >= n) return;
  double g[3], m;
  if (pos) {
    g[0] = pos[3 * s] * inv_dx;
    g[1] = pos[3 * s + 1] * inv_dx;
    g[2] = pos[3 * s + 2] * inv_dx;
    m = mass[s];
  } else {
#pragma unroll
    for (int a = 0; a < 3; ++a) g[a] = (double)ldf(p, FX + a, s) * inv_dx;
    m = (double)ldf(p, FMASS, s);
  }
  int b[3];
  double w[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    b[a] = (int)floor(g[a] - 0.5);
    const double f = g[a] - b[a];
    w[a][0] = 0.5 * ((1.5 - f) * (1.5 - f));
    w[a][1] = 0.75 - (f - 1.0) * (f - 1.0);
    w[a][2] = 0.5 * ((f - 0.5) * (f - 0.5));
  }
  for (int i = 0; i < 3; ++i) {
    const int xi = b[0] + i;
    if (xi < 0 || xi >= rx) continue;
    for (int j = 0; j < 3; ++j) {
      const int yj = b[1] + j;
      if (yj < 0 || yj >= ry) continue;
      const double wij = w[0][i] * w[1][j];
      const long long row = ((long long)xi * ry + yj) * rz;
      for (int k = 0; k < 3; ++k) {
        const int zk = b[2] + k;
        if (zk < 0 || zk >= rz) continue;
        atomicAdd(out + row + zk, wij * w[2][k] * m);
      }
    }
  }
}

__global__ void scale_kernel(double* v, long long n, double s) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) v[i] *= s;
}

// Isosurface of a dense (nx, ny, nz) C-order fp64 field (marching cubes,
// the surfacing step after the splat; surfacing.py:70-95).  Case table:
// mc_table.h (tools/gen_mc_table.py).  One vertex per crossed lattice edge
// (edge id = node * 3 + axis, numbered by a scan over the crossing flags), so
// the mesh is indexed and welded like the reference's; normals are the
// normalised negative field gradient (central differences, one-sided at the
// border) interpolated along the edge, i.e. outward from the dense side.
__device__ __forceinline__ long long mc_node(int i, int j, int k, int ny, int nz) {
  return ((long long)i * ny + j) * nz + k;
}

__global__ void mc_edge_flag_kernel(const double* __restrict__ f, int nx, int ny, int nz, double iso,
                                    int* __restrict__ flag) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long nn = (long long)nx * ny * nz;
  if (e >= 3 * nn) return;
  const long long node = e / 3;
  const int axis = (int)(e - node * 3);
  const int k = (int)(node % nz), j = (int)((node / nz) % ny), i = (int)(node / ((long long)ny * nz));
  const int i2 = i + (axis == 0), j2 = j + (axis == 1), k2 = k + (axis == 2);
  int c = 0;
  if (i2 < nx && j2 < ny && k2 < nz) c = (f[node] >= iso) != (f[mc_node(i2, j2, k2, ny, nz)] >= iso);
  flag[e] = c;
}

__device__ __forceinline__ void mc_grad(const double* f, int nx, int ny, int nz, int i, int j, int k, double g[3]) {
  const int ii[3] = {i, j, k}, nn[3] = {nx, ny, nz};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    int lo[3] = {i, j, k}, hi[3] = {i, j, k};
    lo[a] = max(ii[a] - 1, 0);
    hi[a] = min(ii[a] + 1, nn[a] - 1);
    const double span = (double)(hi[a] - lo[a]);
    g[a] = span > 0.0 ? (f[mc_node(hi[0], hi[1], hi[2], ny, nz)] - f[mc_node(lo[0], lo[1], lo[2], ny, nz)]) / span
                      : 0.0;
  }
}

__global__ void mc_edge_vertex_kernel(const double* __restrict__ f, int nx, int ny, int nz, double iso, double dx,
                                      const int* __restrict__ flag, const int* __restrict__ vid,
                                      double* __restrict__ verts, double* __restrict__ normals) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long nn = (long long)nx * ny * nz;
  if (e >= 3 * nn || !flag[e]) return;
  const long long node = e / 3;
  const int axis = (int)(e - node * 3);
  const int k = (int)(node % nz), j = (int)((node / nz) % ny), i = (int)(node / ((long long)ny * nz));
  const int i2 = i + (axis == 0), j2 = j + (axis == 1), k2 = k + (axis == 2);
  const double f0 = f[node], f1 = f[mc_node(i2, j2, k2, ny, nz)];
  const double t = (iso - f0) / (f1 - f0);
  const long long v = vid[e];
  const double p0[3] = {(double)i, (double)j, (double)k}, p1[3] = {(double)i2, (double)j2, (double)k2};
  double g0[3], g1[3];
  mc_grad(f, nx, ny, nz, i, j, k, g0);
  mc_grad(f, nx, ny, nz, i2, j2, k2, g1);
  double n[3], nrm = 0.0;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    verts[3 * v + a] = (p0[a] + t * (p1[a] - p0[a])) * dx;
    n[a] = -(g0[a] + t * (g1[a] - g0[a]));
    nrm += n[a] * n[a];
  }
  nrm = nrm > 1e-60 ? 1.0 / sqrt(nrm) : 0.0;
#pragma unroll
  for (int a = 0; a < 3; ++a) normals[3 * v + a] = n[a] * nrm;
}

__device__ __forceinline__ int mc_case(const double* f, int ny, int nz, int i, int j, int k, double iso) {
  int c = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int di = (q == 1 || q == 2 || q == 5 || q == 6), dj = (q == 2 || q == 3 || q == 6 || q == 7), dk = q >= 4;
    c |= (f[mc_node(i + di, j + dj, k + dk, ny, nz)] >= iso) << q;
  }
  return c;
}

__global__ void mc_cell_count_kernel(const double* __restrict__ f, int nx, int ny, int nz, double iso,
                                     int* __restrict__ cnt) {
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long nc = (long long)(nx - 1) * (ny - 1) * (nz - 1);
  if (c >= nc) return;
  const int k = (int)(c % (nz - 1)), j = (int)((c / (nz - 1)) % (ny - 1)), i = (int)(c / ((long long)(ny - 1) * (nz - 1)));
  cnt[c] = MC_NTRI[mc_case(f, ny, nz, i, j, k, iso)];
}

__global__ void mc_cell_emit_kernel(const double* __restrict__ f, int nx, int ny, int nz, double iso,
                                    const int* __restrict__ cnt, const int* __restrict__ off,
                                    const int* __restrict__ vid, int* __restrict__ tris) {
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long nc = (long long)(nx - 1) * (ny - 1) * (nz - 1);
  if (c >= nc || !cnt[c]) return;
  const int k = (int)(c % (nz - 1)), j = (int)((c / (nz - 1)) % (ny - 1)), i = (int)(c / ((long long)(ny - 1) * (nz - 1)));
  const int cs = mc_case(f, ny, nz, i, j, k, iso);
  const int nt = MC_NTRI[cs];
  const long long o = off[c];
  for (int q = 0; q < 3 * nt; ++q) {
    const int e = MC_TRI[cs][q];
    const int a = MC_EDGE[e][0], b = MC_EDGE[e][1];
    // lower corner of the edge and its axis
    const int ca = min(a, b) == a ? a : b;
    const int ai = (a == 1 || a == 2 || a == 5 || a == 6), aj = (a == 2 || a == 3 || a == 6 || a == 7), ak = a >= 4;
    const int bi = (b == 1 || b == 2 || b == 5 || b == 6), bj = (b == 2 || b == 3 || b == 6 || b == 7), bk = b >= 4;
    (void)ca;
    const int li = min(ai, bi), lj = min(aj, bj), lk = min(ak, bk);
    const int axis = ai != bi ? 0 : (aj != bj ? 1 : 2);
    tris[3 * o + q] = vid[mc_node(i + li, j + lj, k + lk, ny, nz) * 3 + axis];
  }
}

// MPMF frame body (server.py:65-92) from the device mesh: f32 vertices, f32
// normals, f32 planar UVs (surfacing.py:92-101: u = clip(x / ext0, 0, 1),
// v = clip(z / ext2, 0, 1), in fp64 then rounded like numpy's astype) and u32
// triangle indices, each array contiguous and little-endian, back to back.
__global__ void mesh_encode_kernel(const double* __restrict__ v, const double* __restrict__ nrm, long long nv,
                                   const int* __restrict__ tris, long long nt, double ext0, double ext2,
                                   float* __restrict__ ov, float* __restrict__ on, float* __restrict__ ouv,
                                   unsigned* __restrict__ ot) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < 3 * nv; i += stride) {
    ov[i] = __double2float_rn(v[i]);
    on[i] = __double2float_rn(nrm[i]);
  }
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nv; i += stride) {
    double u = __ddiv_rn(v[3 * i], ext0), w = __ddiv_rn(v[3 * i + 2], ext2);
    u = u < 0.0 ? 0.0 : (u > 1.0 ? 1.0 : u);
    w = w < 0.0 ? 0.0 : (w > 1.0 ? 1.0 : w);
    ouv[2 * i] = __double2float_rn(u);
    ouv[2 * i + 1] = __double2float_rn(w);
  }
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < 3 * nt; i += stride)
    ot[i] = (unsigned)tris[i];
}

}  // namespace mpm
