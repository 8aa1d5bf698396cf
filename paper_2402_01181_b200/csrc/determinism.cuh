// determinism.cuh -- deterministic mode: cell-sorted permutation, payload and node-owner gather (sm_100a).
// Part of the kernel set included by kernels.cuh (namespace mpm).
#pragma once

namespace mpm {

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

}  // namespace mpm
