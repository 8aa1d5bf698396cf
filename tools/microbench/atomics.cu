// Microbenchmarks that decide the P2G accumulation strategy on B200:
//   smem fp32 atomicAdd (compiles to ATOMS.CAST.SPIN loop on sm_100a),
//   smem int32 atomicAdd (native ATOMS.ADD), global REDG.F32 / REDG.F32x4,
//   shuffle throughput.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s line %d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

template<int MODE>
__global__ void smem_atom(float* out, int iters, int spread) {
  __shared__ float s[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = 0.f;
  __syncthreads();
  float v = 1.0f + threadIdx.x * 1e-7f;
  int base = (threadIdx.x / spread) * 37 + (threadIdx.x % spread);  // lanes share addresses in groups
  for (int it = 0; it < iters; ++it) {
    int a = (base + it * 97) & 8191;
    if (MODE == 0) atomicAdd(&s[a], v);
    else atomicAdd((int*)&s[a], 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[threadIdx.x];
}

__global__ void smem_add_plain(float* out, int iters) {
  __shared__ float s[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = 0.f;
  __syncthreads();
  float v = 1.0f;
  for (int it = 0; it < iters; ++it) {
    int a = (threadIdx.x + it * 97) & 8191;
    s[a] += v;  // non-atomic RMW: LDS+FADD+STS (lower bound)
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[0];
}

__global__ void gred(float* g, int iters, size_t n, int vec) {
  size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  float v = 1.0f;
  for (int it = 0; it < iters; ++it) {
    size_t a = (tid * 4 + (size_t)it * 1048576 * 4 * 7) % n;   // distinct 16B slots
    if (vec) atomicAdd((float4*)&g[a & ~(size_t)3], make_float4(v, v, v, v));
    else atomicAdd(&g[a], v);
  }
}

__global__ void gred_hot(float* g, int iters, int nodes) {
  // realistic: each warp hammers a small window of nodes (like a tile flush)
  size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    size_t node = ((tid >> 3) + it * 13) % nodes;
    atomicAdd((float4*)&g[node * 4], make_float4(1.f, 1.f, 1.f, 1.f));
  }
}

__global__ void shfl_bench(float* out, int iters) {
  float v = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    v += __shfl_down_sync(0xffffffff, v, 1);
    v += __shfl_down_sync(0xffffffff, v, 2);
    v += __shfl_down_sync(0xffffffff, v, 4);
    v += __shfl_down_sync(0xffffffff, v, 8);
  }
  if (v == 12345.f) out[0] = v;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  printf("%s SMs=%d L2=%d MB smemPerBlockOptin=%zu clock=%d kHz\n", p.name, p.multiProcessorCount,
         p.l2CacheSize >> 20, p.sharedMemPerBlockOptin, p.clockRate);
  int sms = p.multiProcessorCount;
  float* out; CK(cudaMalloc(&out, 1 << 20));
  size_t n = 256ull << 20;  // 1 GiB of floats
  float* g; CK(cudaMalloc(&g, n * 4)); CK(cudaMemset(g, 0, n * 4));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  int iters = 4096;
  int blocks = sms * 4, thr = 512;
  for (int spread : {1, 2, 4, 8, 32}) {
    smem_atom<0><<<blocks, thr>>>(out, iters, 32 / spread > 0 ? (spread) : 1);
    cudaEventRecord(a);
    smem_atom<0><<<blocks, thr>>>(out, iters, spread);
    cudaEventRecord(b); CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b);
    double ops = (double)blocks * thr * iters;
    printf("smem f32 atomicAdd lanes/addr-group=%d: %.3f Gop/s  %.2f lane-cyc/op/SM\n", spread,
           ops / ms * 1e-6, (ms * 1e-3 * p.clockRate * 1e3 * sms) / ops);
    smem_atom<1><<<blocks, thr>>>(out, iters, spread);
    cudaEventRecord(a);
    smem_atom<1><<<blocks, thr>>>(out, iters, spread);
    cudaEventRecord(b); CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b);
    printf("smem i32 atomicAdd spread=%d: %.3f Gop/s  %.2f lane-cyc/op/SM\n", spread,
           ops / ms * 1e-6, (ms * 1e-3 * p.clockRate * 1e3 * sms) / ops);
  }
  smem_add_plain<<<blocks, thr>>>(out, iters);
  cudaEventRecord(a);
  smem_add_plain<<<blocks, thr>>>(out, iters);
  cudaEventRecord(b); CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b);
  { double ops = (double)blocks * thr * iters;
    printf("smem plain RMW: %.3f Gop/s  %.2f lane-cyc/op/SM\n", ops / ms * 1e-6, (ms * 1e-3 * p.clockRate * 1e3 * sms) / ops); }
  for (int vec : {0, 1}) {
    int gi = 64; int gb = sms * 8;
    gred<<<gb, 256>>>(g, gi, n, vec);
    cudaEventRecord(a);
    gred<<<gb, 256>>>(g, gi, n, vec);
    cudaEventRecord(b); CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b);
    double ops = (double)gb * 256 * gi;
    printf("global red %s spread: %.3f Gop/s\n", vec ? "F32x4" : "F32", ops / ms * 1e-6);
  }
  for (int nodes : {1 << 16, 1 << 20, 1 << 22}) {
    int gi = 64; int gb = sms * 8;
    gred_hot<<<gb, 256>>>(g, gi, nodes);
    cudaEventRecord(a);
    gred_hot<<<gb, 256>>>(g, gi, nodes);
    cudaEventRecord(b); CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b);
    double ops = (double)gb * 256 * gi;
    printf("global red F32x4 8-lane-shared nodes=%d: %.3f Gop/s\n", nodes, ops / ms * 1e-6);
  }
  shfl_bench<<<blocks, thr>>>(out, iters);
  cudaEventRecord(a);
  shfl_bench<<<blocks, thr>>>(out, iters);
  cudaEventRecord(b); CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b);
  { double ops = (double)blocks * thr * iters * 4;
    printf("shfl: %.3f G lane-op/s  %.2f lane-cyc/op/SM\n", ops / ms * 1e-6, (ms * 1e-3 * p.clockRate * 1e3 * sms) / ops); }
  CK(cudaGetLastError());
  return 0;
}
