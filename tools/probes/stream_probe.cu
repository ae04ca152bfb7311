// Probe: how fast can 148 SMs stream a 1.1 GB weight set into shared memory?
// (the decode expert FFN is this plus a few KB of activations)
//   mode 0: 2-D TMA boxes {64 cols, 64 rows} of a row-major [rows, 2048] bf16
//           matrix (the tiled-weight pattern: 128 B from each of 64 rows 4 KB apart)
//   mode 1: same, KA=2 (two K-adjacent boxes per stage = 256 B per row)
//   mode 2: 1-D cp.async.bulk of contiguous 16 KB blocks (a packed, tile-major layout)
//   mode 3: 1-D cp.async.bulk of contiguous 32 KB blocks
// Each CTA owns a contiguous range of 512 KB "units" (claimed from an atomic
// counter); the consumer only waits and frees the slot.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/stream_probe tools/probes/stream_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint32_t b, uint32_t ph) {
  asm volatile(
      "{\n\t.reg .pred P;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@P bra D_%=;\n\tbra W_%=;\nD_%=:\n\t}" ::"r"(b),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");
}
__device__ __forceinline__ void tma2d(uint32_t dst, const CUtensorMap* m, uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          dst),
      "l"(m), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void bulk(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

constexpr int RING = 192 * 1024;

__global__ void __launch_bounds__(64, 1)
    stream_kernel(const __grid_constant__ CUtensorMap map, const uint8_t* base, int mode, int n_units, int* counter,
                  int stage_bytes) {
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[24], empty[24];
  __shared__ int s_unit[2];
  const int stages = RING / stage_bytes;
  if (threadIdx.x == 0) {
    s_unit[0] = 0;
    s_unit[1] = 0;
    for (int i = 0; i < stages; ++i) {
      mbar_init(su32(&full[i]), 1);
      mbar_init(su32(&empty[i]), 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int unit_bytes = 512 * 1024;
  const int steps = unit_bytes / stage_bytes;
  if (threadIdx.x == 0) {
    uint32_t st = 0, ph = 0;
    for (;;) {
      const int u = atomicAdd(counter, 1);
      if (u >= n_units) break;
      for (int s = 0; s < steps; ++s) {
        mbar_wait(su32(&empty[st]), ph ^ 1);
        const uint32_t fb = su32(&full[st]);
        mbar_expect(fb, stage_bytes);
        const uint32_t dst = su32(sm + st * stage_bytes);
        if (mode == 0 || mode == 1) {
          // unit = 128 rows x 2048 cols; stage = 128 rows x (64 * KA) cols as 64-row boxes
          const int ka = mode == 0 ? 1 : 2;
          for (int a = 0; a < ka; ++a)
            for (int h = 0; h < 2; ++h) tma2d(dst + (a * 2 + h) * 8192, &map, fb, (s * ka + a) * 64, u * 128 + h * 64);
        } else {
          bulk(dst, base + (size_t)u * unit_bytes + (size_t)s * stage_bytes, stage_bytes, fb);
        }
        *(volatile int*)&s_unit[1] += 1;
        if (++st == (uint32_t)stages) {
          st = 0;
          ph ^= 1;
        }
      }
    }
    __threadfence_block();
    *(volatile int*)&s_unit[0] = -1;
  } else if (threadIdx.x == 32) {
    uint32_t st = 0, ph = 0;
    for (int consumed = 0;;) {
      const int issued = *(volatile int*)&s_unit[1];
      if (consumed == issued) {
        if (*(volatile int*)&s_unit[0] == -1 && *(volatile int*)&s_unit[1] == consumed) break;
        continue;
      }
      mbar_wait(su32(&full[st]), ph);
      mbar_arrive(su32(&empty[st]));
      ++consumed;
      if (++st == (uint32_t)stages) {
        st = 0;
        ph ^= 1;
      }
    }
  }
}

int main() {
  const size_t rows = 128 * 2240;  // 2240 units of 512 KB = 1.17 GB
  const size_t cols = 2048;
  const int n_units = (int)(rows / 128);
  uint8_t* buf;
  cudaMalloc(&buf, rows * cols * 2);
  cudaMemset(buf, 1, rows * cols * 2);
  int* counter;
  cudaMalloc(&counter, 4);
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap map;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, 64};
  cuuint32_t es[2] = {1, 1};
  enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, RING + 1024);
  const char* names[] = {"tma2d box64x64 KA=1 (16KB stages)", "tma2d KA=2 (32KB stages)", "bulk 16KB contiguous",
                         "bulk 32KB contiguous", "bulk 64KB contiguous"};
  const int sb[] = {16384, 32768, 16384, 32768, 65536};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 0; mode < 5; ++mode) {
    float best = 1e9;
    for (int it = 0; it < 6; ++it) {
      cudaMemset(counter, 0, 4);
      cudaEventRecord(e0);
      stream_kernel<<<148, 64, RING + 1024>>>(map, buf, mode >= 2 ? 2 : mode, n_units, counter, sb[mode]);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    printf("%-36s %8.1f us  %7.0f GB/s  %s\n", names[mode], best * 1e3, rows * cols * 2 / (best * 1e-3) / 1e9,
           cudaGetErrorString(err));
  }
  return 0;
}
