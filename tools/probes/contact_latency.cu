// Single-warp latency of the contact pieces (collide.cuh) for a node just
// below the bottom face of an axis-aligned box (the C3 tool):
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/probes/contact_latency.cu -o /tmp/cl && /tmp/cl
#include <cstdio>
#include <cstring>
#include "../../paper_2402_01181_b200/csrc/collide.cuh"
using namespace mpm;

__global__ void lat(const ColliderGeo* geo, const ColliderPose* pose, long long* out, double* sink) {
  Colliders cs{};
  cs.count = 1;
  cs.geo = geo;
  cs.pose = pose;
  cs.theta = 0.5 / 256;
  const double wx = 0.5 + 0.01 * threadIdx.x / 32.0, wy = 0.2 - 0.03 - 0.3 / 256, wz = 0.5;
  double acc = 0.0;
  for (int rep = 0; rep < 3; ++rep) {  // rep 0 warms L1
    long long t0 = clock64();
    double best;
    const int ci = nearest_collider(cs, wx, wy + acc * 1e-30, wz, 2 * cs.theta, best);
    long long t1 = clock64();
    double n[3];
    world_normal(cs, ci < 0 ? 0 : ci, wx, wy + best * 1e-30, wz, n);
    long long t2 = clock64();
    double v[3] = {0.1 + n[0] * 1e-30, -0.2, 0.05};
    resolve_contact(cs, 0, wx, wy, wz, v);
    long long t3 = clock64();
    acc += v[0] + v[1] + v[2] + n[1];
    if (threadIdx.x == 0 && rep == 2) {
      out[0] = t1 - t0;
      out[1] = t2 - t1;
      out[2] = t3 - t2;
    }
  }
  sink[threadIdx.x] = acc;
}

int main() {
  ColliderGeo g;
  ColliderPose q;
  memset(&g, 0, sizeof g);
  memset(&q, 0, sizeof q);
  g.half[0] = 0.08; g.half[1] = 0.03; g.half[2] = 0.08; g.fric = 0.4;
  q.R[0] = q.R[4] = q.R[8] = 1.0;
  q.T[0] = 0.5; q.T[1] = 0.2; q.T[2] = 0.5; q.lv[1] = -0.5;
  ColliderGeo* dg; ColliderPose* dq; long long* dout; double* sink;
  cudaMalloc(&dg, sizeof g); cudaMalloc(&dq, sizeof q); cudaMalloc(&dout, 64); cudaMalloc(&sink, 256);
  cudaMemcpy(dg, &g, sizeof g, cudaMemcpyHostToDevice);
  cudaMemcpy(dq, &q, sizeof q, cudaMemcpyHostToDevice);
  lat<<<1, 32>>>(dg, dq, dout, sink);
  long long h[3];
  cudaMemcpy(h, dout, sizeof h, cudaMemcpyDeviceToHost);
  printf("cycles: nearest %lld  world_normal %lld  resolve_contact %lld\n", h[0], h[1], h[2]);
  return 0;
}
