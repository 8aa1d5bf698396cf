// Can stream memory operations (cuStreamWaitValue32 / cuStreamWriteValue32)
// be captured into a CUDA graph and replayed?  Two streams, one signals the
// other through a device counter; the pair is captured as one graph (fork /
// join through events) and replayed 3 times with the counter reset between.
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
typedef CUresult (*WaitFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*WriteFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
__global__ void add(int* x, int v) { atomicAdd(x, v); }
int main() {
  void *fw = nullptr, *fr = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuStreamWaitValue32", &fw, cudaEnableDefault, &q);
  cudaGetDriverEntryPoint("cuStreamWriteValue32", &fr, cudaEnableDefault, &q);
  WaitFn wait = (WaitFn)fw;
  WriteFn write = (WriteFn)fr;
  int *cnt, *x;
  cudaMalloc(&cnt, 8);
  cudaMalloc(&x, 4);
  cudaMemset(cnt, 0, 8);
  cudaMemset(x, 0, 4);
  cudaStream_t a, b;
  cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
  cudaEvent_t fork, join;
  cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&join, cudaEventDisableTiming);
  cudaGraph_t g;
  cudaError_t e = cudaStreamBeginCapture(a, cudaStreamCaptureModeThreadLocal);
  printf("begin capture: %s\n", cudaGetErrorString(e));
  cudaMemsetAsync(cnt, 0, 4, a);
  cudaEventRecord(fork, a);
  cudaStreamWaitEvent(b, fork, 0);
  CUresult r1 = wait((CUstream)b, (CUdeviceptr)cnt, 1, CU_STREAM_WAIT_VALUE_GEQ);  // b waits for a's signal
  add<<<1, 1, 0, b>>>(x, 10);
  add<<<1, 1, 0, a>>>(x, 1);
  CUresult r2 = write((CUstream)a, (CUdeviceptr)cnt, 1, CU_STREAM_WRITE_VALUE_DEFAULT);
  cudaEventRecord(join, b);
  cudaStreamWaitEvent(a, join, 0);
  e = cudaStreamEndCapture(a, &g);
  printf("wait in capture: %d, write in capture: %d, end capture: %s\n", (int)r1, (int)r2, cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  cudaGraphExec_t ge;
  e = cudaGraphInstantiate(&ge, g, 0);
  printf("instantiate: %s\n", cudaGetErrorString(e));
  for (int k = 0; k < 3; ++k) cudaGraphLaunch(ge, a);
  e = cudaStreamSynchronize(a);
  int h = 0;
  cudaMemcpy(&h, x, 4, cudaMemcpyDeviceToHost);
  printf("replays done: %s, x = %d (expect 33)\n", cudaGetErrorString(e), h);
  return 0;
}
