// Probe: TMA tile::gather4 on sm_100a — 4 arbitrary rows x 64 bf16 (128 B) into smem,
// 128B-swizzled, compared against the expected swizzled layout.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__global__ void k(const __grid_constant__ CUtensorMap map, int* rows, uint16_t* out) {
  __shared__ __align__(1024) uint16_t sm[8 * 64];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(sm), b = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(8 * 128));
    for (int g = 0; g < 2; ++g)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(s + g * 512),
          "l"(&map), "r"(0), "r"(rows[4 * g]), "r"(rows[4 * g + 1]), "r"(rows[4 * g + 2]), "r"(rows[4 * g + 3]),
          "r"(b)
          : "memory");
  }
  asm volatile(
      "{\n.reg .pred P;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W;\n}" ::"r"(b));
  for (int i = threadIdx.x; i < 8 * 64; i += blockDim.x) out[i] = sm[i];
}

int main() {
  const int R = 1000, C = 64;
  std::vector<uint16_t> h(R * C);
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < C; ++c) h[r * C + c] = (uint16_t)(r * 64 + c);
  uint16_t* d;
  cudaMalloc(&d, h.size() * 2);
  cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R};
  cuuint64_t str[1] = {(cuuint64_t)C * 2};
  cuuint32_t box[2] = {64, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult cr = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)cr);
  int rows_h[8] = {7, 3, 999, 500, 1, 2, 42, 0};
  int* rows;
  cudaMalloc(&rows, 32);
  cudaMemcpy(rows, rows_h, 32, cudaMemcpyHostToDevice);
  uint16_t* out;
  cudaMalloc(&out, 8 * 64 * 2);
  k<<<1, 128>>>(m, rows, out);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel %s\n", cudaGetErrorString(e));
  std::vector<uint16_t> o(8 * 64);
  cudaMemcpy(o.data(), out, o.size() * 2, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int r = 0; r < 8; ++r)
    for (int c = 0; c < 64; ++c) {
      // 128B swizzle: 16-byte chunk index (c/8) XOR (row within 8-row atom)
      const int chunk = (c / 8) ^ (r & 7);
      const uint16_t got = o[r * 64 + chunk * 8 + (c % 8)];
      if (got != (uint16_t)(rows_h[r] * 64 + c)) ++bad;
    }
  printf("mismatches %d\n", bad);
  return 0;
}
