// Cost of warp_route_token (route_common.cuh) per call, warm and cold:
// one warp, E logits in shared memory, clock64() around each call.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2605_17889_b200/csrc tools/probes/route_probe.cu -o /tmp/route_probe
#include <cstdio>
#include "route_common.cuh"

__global__ void probe(int E, int k, int mode, int reps, long long* cyc, int* idx, float* w, int* hist) {
  __shared__ float lg[256];
  __shared__ int s_sel[8];
  __shared__ float s_selv[8];
  const int lane = threadIdx.x;
  for (int r = 0; r < reps; ++r) {
    for (int e = lane; e < E; e += 32) lg[e] = __sinf(0.37f * e + r);
    __syncwarp();
    long long t0 = clock64();
    cox::warp_route_token(lg, E, k, mode, lane, s_sel, s_selv, idx, w, hist);
    long long t1 = clock64();
    if (lane == 0) cyc[r] = t1 - t0;
  }
}

int main() {
  long long* cyc;
  int *idx, *hist;
  float* w;
  cudaMalloc(&cyc, 64 * sizeof(long long));
  cudaMalloc(&idx, 64);
  cudaMalloc(&w, 64);
  cudaMalloc(&hist, 1024);
  int cfg[3][3] = {{64, 6, 1}, {8, 2, 0}, {64, 6, 0}};
  for (auto& c : cfg) {
    probe<<<1, 32>>>(c[0], c[1], c[2], 16, cyc, idx, w, hist);
    long long h[16];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("E=%d k=%d mode=%d: first call %lld cycles, then", c[0], c[1], c[2], h[0]);
    for (int i = 1; i < 6; ++i) printf(" %lld", h[i]);
    printf("\n");
  }
  return 0;
}
