// Issue/pipe throughput of FFMA vs packed FFMA2 (sm_100a) and of int32
// ATOMS.ADD with and without bank conflicts: cycles per warp instruction per
// SM sub-partition, measured with clock64 over a long unrolled loop.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma2 ffma2.cu
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
  u64 d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ u64 pk(float a, float b) {
  u64 r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
constexpr int IT = 4096;
__global__ void k_ffma(float* out, float a, float b, long long* cyc) {
  float x[8];
  for (int q = 0; q < 8; ++q) x[q] = threadIdx.x + q;
  float c = b + threadIdx.x * 1e-9f;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < IT; ++i) {
#pragma unroll
    for (int q = 0; q < 8; ++q) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[q]) : "f"(a), "f"(c));
  }
  long long t1 = clock64();
  float s = 0;
  for (int q = 0; q < 8; ++q) s += x[q];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void k_ffma2(float* out, float a, float b, long long* cyc) {
  u64 x[8];
  for (int q = 0; q < 8; ++q) x[q] = pk(threadIdx.x + q, q);
  u64 aa = pk(a, a * 0.5f), cc = pk(b + threadIdx.x * 1e-9f, b);
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < IT; ++i) {
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = fma2(x[q], aa, cc);
  }
  long long t1 = clock64();
  float s = 0;
  for (int q = 0; q < 8; ++q) s += __int_as_float((int)x[q]) + __int_as_float((int)(x[q] >> 32));
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
// shared int atomics: stride 1 (conflict-free) or stride 32 (32-way conflicts)
__global__ void k_atoms(int* out, int stride, long long* cyc) {
  __shared__ int t[32 * 33 * 8];
  for (int i = threadIdx.x; i < 32 * 33 * 8; i += blockDim.x) t[i] = 0;
  __syncthreads();
  int base = ((threadIdx.x & 31) * stride) % (32 * 33) + (threadIdx.x >> 5) * 4;
  long long t0 = clock64();
  for (int i = 0; i < IT; ++i) {
#pragma unroll
    for (int q = 0; q < 8; ++q) atomicAdd(&t[base + q * 32 * 33 / 8 % 1024], i + q);
  }
  long long t1 = clock64();
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = t[threadIdx.x];
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* out;
  int* iout;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&iout, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  long long h[148];
  for (int warps : {4, 8, 16, 32}) {
    int thr = warps * 32;
    k_ffma<<<148, thr>>>(out, 1.0001f, 0.5f, cyc);
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    double ffma = (double)h[0] / (IT * 8.0 * warps / 4);
    k_ffma2<<<148, thr>>>(out, 1.0001f, 0.5f, cyc);
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    double ffma2 = (double)h[0] / (IT * 8.0 * warps / 4);
    k_atoms<<<148, thr>>>(iout, 1, cyc);
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    double at1 = (double)h[0] / (IT * 8.0 * warps / 4);
    k_atoms<<<148, thr>>>(iout, 32, cyc);
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    double at33 = (double)h[0] / (IT * 8.0 * warps / 4);
    k_atoms<<<148, thr>>>(iout, 2, cyc);
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    double at2 = (double)h[0] / (IT * 8.0 * warps / 4);
    printf("warps/SM %2d: cycles per warp-instr per SMSP: FFMA %.2f  FFMA2 %.2f  ATOMS(no conflict) %.2f  ATOMS(32-way) %.2f  ATOMS(2-way) %.2f\n",
           warps, ffma, ffma2, at1, at33, at2);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
