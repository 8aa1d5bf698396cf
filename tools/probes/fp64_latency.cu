#include <cstdio>
__global__ void k(double* io, long long* out, float* fio) {
  double a = io[0], b = io[1];
  float fa = fio[0], fb = fio[1];
  long long t0 = clock64();
#pragma unroll
  for (int i = 0; i < 64; ++i) a = __dadd_rn(a, b);
  long long t1 = clock64();
#pragma unroll
  for (int i = 0; i < 64; ++i) a = __dmul_rn(a, b);
  long long t2 = clock64();
#pragma unroll
  for (int i = 0; i < 64; ++i) a = a > b ? a : b + a;
  long long t3 = clock64();
#pragma unroll
  for (int i = 0; i < 64; ++i) fa = __fadd_rn(fa, fb);
  long long t4 = clock64();
  io[2] = a; fio[2] = fa;
  out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = t4 - t3;
}
int main() {
  double* d; long long* o; float* f;
  cudaMalloc(&d, 64); cudaMalloc(&o, 64); cudaMalloc(&f, 64);
  double h[3] = {1.0, 1e-9, 0}; float hf[3] = {1.f, 1e-9f, 0};
  cudaMemcpy(d, h, 24, cudaMemcpyHostToDevice); cudaMemcpy(f, hf, 12, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(d, o, f); k<<<1, 32>>>(d, o, f);
  long long r[4]; cudaMemcpy(r, o, 32, cudaMemcpyDeviceToHost);
  printf("per-op latency (cycles): dadd %.1f dmul %.1f dcmp+sel+dadd %.1f fadd %.1f\n", r[0] / 64., r[1] / 64., r[2] / 64., r[3] / 64.);
}
