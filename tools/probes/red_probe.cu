// L2 reduction throughput on B200: n float4 reductions (REDG.F32x4) into m
// nodes, vs scalar fp32 / int32 reductions and plain stores, for distinct
// and overlapping targets.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/probes/red_probe.cu -o /tmp/rp && /tmp/rp
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned hash(unsigned x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16;
  return x;
}

// mode 0: red f32x4, 1: 4 x red f32, 2: 4 x red s32, 3: st.v4, 4: red f32x4 to (i*stride)%m contiguous runs
template <int MODE>
__global__ void k(float4* g, long long n, unsigned m, int runs) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
    // contiguous runs of 32 nodes (a warp writes one brick row), run start hashed
    const unsigned run = (unsigned)(i >> 5), lane = (unsigned)(i & 31);
    const unsigned node = (runs ? (hash(run % (m / 32)) % (m / 32)) * 32 + lane : (unsigned)(i % m));
    float4 v = make_float4(1.f, 2.f, 3.f, 4.f);
    if (MODE == 0) atomicAdd(g + node, v);
    if (MODE == 1) { float* f = (float*)(g + node); atomicAdd(f, 1.f); atomicAdd(f + 1, 2.f); atomicAdd(f + 2, 3.f); atomicAdd(f + 3, 4.f); }
    if (MODE == 2) { int* f = (int*)(g + node); atomicAdd(f, 1); atomicAdd(f + 1, 2); atomicAdd(f + 2, 3); atomicAdd(f + 3, 4); }
    if (MODE == 3) g[node] = v;
  }
}

template <int MODE>
float run(float4* g, long long n, unsigned m, int runs) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  k<MODE><<<148 * 8, 256>>>(g, n, m, runs);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) k<MODE><<<148 * 8, 256>>>(g, n, m, runs);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / 5;
}

int main() {
  const unsigned m = 600000;  // nodes (C3: ~593 K in active bricks)
  float4* g; cudaMalloc(&g, sizeof(float4) * m);
  cudaMemset(g, 0, sizeof(float4) * m);
  for (long long n : {1500000LL, 3000000LL}) {
    for (int runs : {0, 1}) {
      printf("n %lld (%.1f per node) %s: red.f32x4 %.1f us  4xred.f32 %.1f us  4xred.s32 %.1f us  st.v4 %.1f us\n", n,
             (double)n / m, runs ? "hashed 32-node runs" : "sequential", 1e3 * run<0>(g, n, m, runs),
             1e3 * run<1>(g, n, m, runs), 1e3 * run<2>(g, n, m, runs), 1e3 * run<3>(g, n, m, runs));
    }
  }
  return 0;
}
