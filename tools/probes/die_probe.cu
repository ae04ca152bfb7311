// Probe: per-SM L2-hit latency to a set of lines spread over the address space.
// SMs on the same die see the same near/far pattern (address -> home die is a
// hash), so clustering the per-SM latency vectors recovers the SM -> die map.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/die_probe tools/probes/die_probe.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

__global__ void probe(const int* __restrict__ buf, int nlines, int stride_ints, unsigned* lat, int* smid_out) {
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if (threadIdx.x) return;
  smid_out[blockIdx.x] = smid;
  int sink = 0;
  for (int i = 0; i < nlines; ++i) {  // warm: lines become L2-resident
    int v;
    asm volatile("ld.global.cg.s32 %0, [%1];" : "=r"(v) : "l"(buf + (long)i * stride_ints));
    sink += v;
  }
  for (int i = 0; i < nlines; ++i) {
    const long long t0 = clock64();
    int v;
    asm volatile("ld.global.cg.s32 %0, [%1];" : "=r"(v) : "l"(buf + (long)i * stride_ints + (sink & 1)));
    sink += v;
    const long long t1 = clock64();
    lat[blockIdx.x * nlines + i] = (unsigned)(t1 - t0);
  }
  if (sink == 123456789) lat[0] = 0;
}

int main() {
  const int nlines = 256, stride = 512 * 3;  // 6 KB apart
  int* buf;
  cudaMalloc(&buf, (size_t)nlines * stride * 4 + 64);
  cudaMemset(buf, 0, (size_t)nlines * stride * 4 + 64);
  const int nb = 148 * 4;
  unsigned* lat;
  int* sm;
  cudaMalloc(&lat, (size_t)nb * nlines * 4);
  cudaMalloc(&sm, nb * 4);
  probe<<<nb, 32>>>(buf, nlines, stride, lat, sm);
  probe<<<nb, 32>>>(buf, nlines, stride, lat, sm);
  if (cudaDeviceSynchronize() != cudaSuccess) {
    fprintf(stderr, "kernel failed\n");
    return 1;
  }
  std::vector<unsigned> h((size_t)nb * nlines);
  std::vector<int> hs(nb);
  cudaMemcpy(h.data(), lat, h.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(hs.data(), sm, nb * 4, cudaMemcpyDeviceToHost);
  for (int b = 0; b < nb; ++b) {
    printf("%d", hs[b]);
    for (int i = 0; i < nlines; ++i) printf(" %u", h[(size_t)b * nlines + i]);
    printf("\n");
  }
  return 0;
}
