// HBM write ceilings on B200: how fast can an SM push bytes to HBM through
//   (a) TMA tiled stores from shared memory (box shapes of the GEMM / chain
//       epilogues: 32 rows x 64 B, 32 x 128 B, 128 x 128 B),
//   (b) plain 16-byte STG from registers,
// against an LDG/STG copy (the 1:1 read+write mix of the write-heavy layers).
// One persistent CTA per SM, 1 GiB destination, rows of 2 KB (N = 1024 bf16).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2006_05096_b200/csrc \
//        tools/tma_write.cu -lcuda -o tools/tma_write && tools/tma_write
#include <cstdio>
#include <cuda.h>
#include "common.cuh"

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                          const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                          CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                          CUtensorMapFloatOOBfill);

constexpr long ROW_ELEMS = 1024;            // 2 KB rows
constexpr long BYTES = 1l << 30;
constexpr long ROWS = BYTES / (ROW_ELEMS * 2);

// Each CTA walks boxes b = blockIdx.x, += gridDim.x; box b covers rows
// (b / nbx) * box_rows.., columns (b % nbx) * box_cols.
__global__ void __launch_bounds__(256, 1)
    tma_store_kernel(const __grid_constant__ CUtensorMap m, int box_rows, int box_cols, int depth,
                     const __grid_constant__ CUtensorMap src, int mix) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[1];
  const int box_bytes = box_rows * box_cols * 2;
  for (int i = threadIdx.x; i < depth * box_bytes / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sm)[i] = 0x3f803f80u;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  __syncthreads();
  // `mix` > 1: that many issuing warps (lane 0 each), boxes interleaved
  const int issuers = mix > 1 ? mix : 1;
  const int wi = threadIdx.x >> 5;
  if ((threadIdx.x & 31) != 0 || wi >= issuers) return;
  if (mix > 1) mix = 0;
  sm += wi * depth * box_bytes;
  const long nbx = ROW_ELEMS / box_cols;
  const long nbox = (ROWS / box_rows) * nbx;
  int k = 0;
  uint32_t ph = 0;
  for (long b = (long)blockIdx.x * issuers + wi; b < nbox; b += (long)gridDim.x * issuers, ++k) {
    const int slot = k % depth;
    const int c0 = (int)(b % nbx) * box_cols, r0 = (int)(b / nbx) * box_rows;
    if (mix) {   // read one box (from the other half of the buffer) into the slot first
      bulk_wait_read<0>();
      mbar_arrive_expect_tx(bar, box_bytes);
      tma_load_2d(sm + slot * box_bytes, &src, bar, c0, r0);
      mbar_wait(bar, ph);
      ph ^= 1;
    } else if (k >= depth) {   // throttle: at most `depth` stores in flight
      switch (depth) {
        case 2: bulk_wait_read<1>(); break;
        case 4: bulk_wait_read<3>(); break;
        case 8: bulk_wait_read<7>(); break;
        case 16: bulk_wait_read<15>(); break;
        default: bulk_wait_read<31>(); break;
      }
    }
    tma_store_2d(&m, sm + slot * box_bytes, c0, r0);
    bulk_commit();
  }
  bulk_wait<0>();
}

__global__ void stg_kernel(uint4* p, long n) {
  const uint4 v = make_uint4(0x3f803f80u, 0x3f803f80u, 0x3f803f80u, 0x3f803f80u);
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    p[i] = v;
}

__global__ void copy_kernel(const uint4* s, uint4* d, long n) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    d[i] = s[i];
}

int main() {
  void *dst, *srcp;
  cudaMalloc(&dst, BYTES);
  cudaMalloc(&srcp, BYTES);
  cudaMemset(srcp, 0, BYTES);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  EncFn fn = (EncFn)fp;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(tma_store_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](auto&& launch) {
    launch();
    cudaDeviceSynchronize();
    float best = 1e9f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    return best;
  };
  struct Shape { int rows, cols; CUtensorMapSwizzle sw; const char* name; };
  Shape shapes[] = {{32, 32, CU_TENSOR_MAP_SWIZZLE_64B, "32 rows x 64 B (gemm epilogue)"},
                    {32, 64, CU_TENSOR_MAP_SWIZZLE_128B, "32 rows x 128 B"},
                    {128, 32, CU_TENSOR_MAP_SWIZZLE_64B, "128 rows x 64 B"},
                    {64, 64, CU_TENSOR_MAP_SWIZZLE_128B, "64 rows x 128 B"},
                    {128, 64, CU_TENSOR_MAP_SWIZZLE_128B, "128 rows x 128 B (chain)"},
                    {256, 64, CU_TENSOR_MAP_SWIZZLE_128B, "256 rows x 128 B"},
                    {64, 256, CU_TENSOR_MAP_SWIZZLE_NONE, "64 rows x 512 B (no swizzle)"}};
  for (auto& s : shapes) {
    CUtensorMap m, ms;
    cuuint64_t dims[2] = {(cuuint64_t)ROW_ELEMS, (cuuint64_t)ROWS};
    cuuint64_t str[1] = {(cuuint64_t)ROW_ELEMS * 2};
    cuuint32_t box[2] = {(cuuint32_t)s.cols, (cuuint32_t)s.rows}, es[2] = {1, 1};
    CUresult r1 = fn(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dst, dims, str, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, s.sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUresult r2 = fn(&ms, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, srcp, dims, str, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, s.sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r1 || r2) { printf("%s: encode failed %d %d\n", s.name, (int)r1, (int)r2); continue; }
    const int bb = s.rows * s.cols * 2;
    for (int depth : {4, 8, 16, 32}) {
      if (depth * bb > 190 * 1024) continue;
      const float ms_ = timeit([&] {
        tma_store_kernel<<<sms, 128, depth * bb + 1024>>>(m, s.rows, s.cols, depth, ms, 0);
      });
      printf("TMA store  %-32s depth %2d: %6.2f TB/s\n", s.name, depth, BYTES / ms_ / 1e9);
    }
    for (int iss : {2, 4, 8}) {   // several issuing warps per SM, depth 2 each
      if (iss * 2 * bb > 190 * 1024) continue;
      const float ms_ = timeit([&] {
        tma_store_kernel<<<sms, 256, iss * 2 * bb + 1024>>>(m, s.rows, s.cols, 2, ms, iss);
      });
      printf("TMA store  %-32s %d issuers x depth 2: %6.2f TB/s\n", s.name, iss, BYTES / ms_ / 1e9);
    }
  }
  for (int bpsm : {4, 8, 16}) {
    const float ms_ = timeit([&] { stg_kernel<<<sms * bpsm, 256>>>((uint4*)dst, BYTES / 16); });
    printf("STG.128 write-only (%2d blocks/SM): %6.2f TB/s\n", bpsm, BYTES / ms_ / 1e9);
  }
  const float mc = timeit([&] { copy_kernel<<<sms * 8, 256>>>((const uint4*)srcp, (uint4*)dst, BYTES / 16); });
  printf("LDG/STG copy: %6.2f TB/s moved (read + write)\n", 2.0 * BYTES / mc / 1e9);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
