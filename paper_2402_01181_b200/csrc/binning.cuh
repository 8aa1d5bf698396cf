// binning.cuh -- re-binning: counting sort of particle slots by bin and local cell, work list, exclusive scan (sm_100a).
// Part of the kernel set included by kernels.cuh (namespace mpm).
#pragma once

namespace mpm {

// ---------------------------------------------------------------------------
// binning (counting sort by 8^3-cell bin)
// ---------------------------------------------------------------------------

// Re-binning = counting sort of particle slots by (8^3-cell bin, local cell):
// bin_key (warp-aggregated counters) -> scan -> bin_fill -> bin_local_sort
// (per-bin counting sort over the 512 local cells in shared memory) ->
// gather_permute (coalesced writes).  Lanes of a warp then share cells, so
// shared-memory tile reads broadcast and int atomics hit few banks.
__global__ void bin_key_kernel(Params p, int* key, int* lcell, int* rank, int* bin_count) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  // slots vacated by migrants (slab windows) are dropped by this re-binning
  const bool valid = i < p.n && !(i < p.hole_n && p.hole_flag[i] != 0);
  const unsigned mask = __ballot_sync(0xffffffffu, valid);
  if (!valid) {
    if (i < p.n) key[i] = -1;
    return;
  }
  int c[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    float g = ldf(p, FX + a, i) * p.inv_dx;
    int bb = (int)floorf(g - 0.5f);
    c[a] = max(0, min(bb, p.res[a] - 3));
  }
  const int k = ((c[0] >> BIN_SHIFT) * p.nbin[1] + (c[1] >> BIN_SHIFT)) * p.nbin[2] + (c[2] >> BIN_SHIFT);
  key[i] = k;
  lcell[i] = (((c[0] & (BIN - 1)) * BIN) + (c[1] & (BIN - 1))) * BIN + (c[2] & (BIN - 1));
  const unsigned peers = __match_any_sync(mask, k);
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(peers) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(bin_count + k, __popc(peers));
  base = __shfl_sync(peers, base, leader);
  rank[i] = base + __popc(peers & ((1u << lane) - 1u));
}

__global__ void bin_fill_kernel(const int* key, const int* lcell, const int* rank, const int* start,
                                int* sidx, int* slc, long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n || key[i] < 0) return;
  const int d = start[key[i]] + rank[i];
  sidx[d] = (int)i;
  slc[d] = lcell[i];
}

constexpr int LOCAL_CELLS = BIN * BIN * BIN;

// One CTA per bin (grid-stride): counting sort of the bin's slots by local cell.
// The CTA's bins are screened 256 at a time (one count load per thread) and
// only the occupied ones visited -- most bins of a sparse scene are empty,
// and walking them one dependent load at a time dominated the kernel.
__global__ void __launch_bounds__(256) bin_local_sort_kernel(const int* bin_count, const int* bin_start,
                                                             int nbins, const int* sidx, const int* slc,
                                                             int* rk, int* perm, int* bin_maxcnt) {
  __shared__ int cnt[LOCAL_CELLS];
  __shared__ int wsum[8];
  __shared__ int wmax[8];
  __shared__ int occ[256];
  __shared__ int nocc;
  for (long long j0 = 0; (long long)blockIdx.x + j0 * gridDim.x < nbins; j0 += 256) {
    if (threadIdx.x == 0) nocc = 0;
    __syncthreads();
    {
      const long long b = (long long)blockIdx.x + (j0 + threadIdx.x) * gridDim.x;
      if (b < nbins && bin_count[b] > 0) occ[atomicAdd(&nocc, 1)] = (int)b;
    }
    __syncthreads();
    const int nvisit = nocc;
    __syncthreads();  // nocc read by all before the next screen resets it
  for (int v = 0; v < nvisit; ++v) {
    const int b = occ[v];
    const int nb = bin_count[b];
    const int s = bin_start[b];
    for (int c = threadIdx.x; c < LOCAL_CELLS; c += blockDim.x) cnt[c] = 0;
    __syncthreads();
    for (int e = threadIdx.x; e < nb; e += blockDim.x) rk[s + e] = atomicAdd(&cnt[slc[s + e]], 1);
    __syncthreads();
    // exclusive scan of 512 counters: 2 per thread (and the densest cell)
    const int c0 = cnt[2 * threadIdx.x], c1 = cnt[2 * threadIdx.x + 1];
    int incl = c0 + c1;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int cm = __reduce_max_sync(0xffffffffu, max(c0, c1));
    if (lane == 0) wmax[wid] = cm;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    int woff = 0;
    for (int w = 0; w < wid; ++w) woff += wsum[w];
    if (threadIdx.x == 0) {
      int mm = 0;
      for (int w = 0; w < 8; ++w) mm = max(mm, wmax[w]);
      bin_maxcnt[b] = mm;
    }
    const int excl = woff + incl - c0 - c1;
    __syncthreads();
    cnt[2 * threadIdx.x] = excl;
    cnt[2 * threadIdx.x + 1] = excl + c0;
    __syncthreads();
    for (int e = threadIdx.x; e < nb; e += blockDim.x) perm[s + cnt[slc[s + e]] + rk[s + e]] = sidx[s + e];
    __syncthreads();
  }
  }
}

__global__ void gather_permute_kernel(const float* __restrict__ src, const int* __restrict__ src_mat,
                                      const int* __restrict__ src_orig, float* __restrict__ dst,
                                      int* __restrict__ dst_mat, int* __restrict__ dst_orig,
                                      const int* __restrict__ perm, long long n, long long cap) {
  const long long d = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (d >= n) return;
  const long long s = perm[d];
#pragma unroll
  for (int f = 0; f < NF; ++f) dst[f * cap + d] = __ldg(src + f * cap + s);
  dst_mat[d] = __ldg(src_mat + s);
  dst_orig[d] = __ldg(src_orig + s);
}

// Work list, sorted by decreasing size class (whole CTA rounds of
// FUSED_K_THREADS particles) so that the dynamically scheduled kernels hand
// out the large items first (longest-processing-time order) and finish on
// the small ones.  Three launches: count per class, class offsets, emit.
constexpr int WORK_CLASSES = CHUNK / 256 + 2;

__device__ __forceinline__ int work_items_of(int c, int chunk, int& per) {
  const int items = (c + chunk - 1) / chunk;
  per = (c + items - 1) / items;  // equal splits (no tiny tail item)
  return items;
}

__device__ __forceinline__ int work_class(int size) {
  return min((size + FUSED_K_THREADS - 1) / FUSED_K_THREADS, WORK_CLASSES - 1);
}

__global__ void make_work_count_kernel(const int* bin_count, int nbins, int chunk, int* class_count) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nbins) return;
  const int c = bin_count[b];
  if (!c) return;
  int per;
  const int items = work_items_of(c, chunk, per);
  for (int t = 0; t < items; ++t) atomicAdd(&class_count[work_class(min(per, c - t * per))], 1);
}

__global__ void make_work_offsets_kernel(const int* class_count, int* class_cursor, int* nwork) {
  if (threadIdx.x != 0) return;
  int s = 0;
  for (int k = WORK_CLASSES - 1; k >= 0; --k) {
    class_cursor[k] = s;
    s += class_count[k];
  }
  *nwork = s;
}

__global__ void make_work_kernel(const int* bin_count, const int* bin_start, const int* bin_maxcnt, int nbins,
                                 int4* work, int* class_cursor, int chunk) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nbins) return;
  const int c = bin_count[b];
  if (!c) return;
  int per;
  const int items = work_items_of(c, chunk, per);
  const int s = bin_start[b];
  for (int t = 0; t < items; ++t) {
    const int size = min(per, c - t * per);
    const int pos = atomicAdd(&class_cursor[work_class(size)], 1);
    work[pos] = make_int4(b, s + t * per, s + t * per + size, bin_maxcnt[b]);
  }
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

}  // namespace mpm
