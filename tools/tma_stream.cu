// Micro-benchmark: streaming HBM reads through a TMA ring, the A-operand path
// of the memory-bound GEMMs.  One CTA per SM; one elected thread issues 2D
// tensor loads (128 rows x 128 B, SWIZZLE_128B, 16 KB) into an S-stage ring,
// a consumer warp waits each stage and releases it (no math).  Reports GB/s
// for S in {2, 4, 8, 12} and box heights {64, 128, 256}, over a 1 GiB tensor.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2006_05096_b200/csrc tma_stream.cu -o tma_stream -lcuda
#include <cuda.h>
#include <cstdio>
#include "common.cuh"

__global__ void __launch_bounds__(64, 1) stream_kernel(const __grid_constant__ CUtensorMap tm,
                                                       const __grid_constant__ CUtensorMap tw,
                                                       int tiles, int box_rows, int stages,
                                                       int wbox) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int box_bytes = box_rows * 128;
  const int stage_bytes = box_bytes + wbox * 128;   // + an L2-resident "weights" box
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * stage_bytes);
  uint64_t* empty = full + stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (warp == 0 && lane == 0) {
    int st = 0;
    uint32_t ph = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
      mbar_wait(&empty[st], ph ^ 1);
      mbar_arrive_expect_tx(&full[st], stage_bytes);
      tma_load_2d(smem + st * stage_bytes, &tm, &full[st], 0, t * box_rows);
      if (wbox) tma_load_2d(smem + st * stage_bytes + box_bytes, &tw, &full[st], 0, 0);
      if (++st == stages) { st = 0; ph ^= 1; }
    }
  } else if (warp == 1 && lane == 0) {
    int st = 0;
    uint32_t ph = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
      mbar_wait(&full[st], ph);
      mbar_arrive(&empty[st]);
      if (++st == stages) { st = 0; ph ^= 1; }
    }
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t bytes = 1ull << 30;
  const uint64_t rows = bytes / 128;
  void* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  EncodeFn enc = reinterpret_cast<EncodeFn>(fp);
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  void* wbuf;
  cudaMalloc(&wbuf, 1 << 20);
  cudaMemset(wbuf, 1, 1 << 20);
  for (int oob : {0, 1})
  for (int wbox : {0, 32})
  for (int box_rows : {128}) {
    CUtensorMap tm, tw;
    {
      cuuint64_t wd[2] = {64, (cuuint64_t)(oob ? 16 : 4096)};
      cuuint64_t wst[1] = {128};
      cuuint32_t wb[2] = {64, (cuuint32_t)(wbox ? wbox : 32)};
      cuuint32_t wes[2] = {1, 1};
      enc(&tw, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, wbuf, wd, wst, wb, wes,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    // oob = 1: a 32-column (64 B) tensor read with the 64-column box, half of
    // every box row out of bounds (the narrow-K GEMM A operand); weights box
    // of 32 rows over a 16-row tensor
    cuuint64_t dims[2] = {(cuuint64_t)(oob ? 32 : 64), oob ? rows * 2 : rows};
    cuuint64_t str[1] = {(cuuint64_t)(oob ? 64 : 128)};
    cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, box, es,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int tiles = (int)((oob ? rows * 2 : rows) / box_rows);
    for (int stages : {2, 4, 8}) {
      const int smem = stages * (box_rows + wbox) * 128 + 2048;
      if (smem > 232448) continue;
      stream_kernel<<<sms, 64, smem>>>(tm, tw, tiles, box_rows, stages, wbox);
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) stream_kernel<<<sms, 64, smem>>>(tm, tw, tiles, box_rows, stages, wbox);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("oob %d wbox %2d  box %3d rows (%3d KB) stages %2d (%4d KB in flight/SM): %7.1f GB/s  (%s)\n", oob, wbox, box_rows,
             box_rows * 128 / 1024, stages, stages * box_rows * 128 / 1024,
             5.0 * bytes / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
