// Does a tiled TMA store accept negative / partially out-of-bounds box
// coordinates (clipping), like tiled loads do?  4D bf16 map, 64B swizzle.
#include <cstdio>
#include <cuda.h>
#include "common.cuh"
typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                          const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                          CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                          CUtensorMapFloatOOBfill);
__global__ void k(const __grid_constant__ CUtensorMap m, int c1, int c2) {
  __shared__ __align__(1024) uint8_t buf[2048];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) reinterpret_cast<uint16_t*>(buf)[i] = 0x3f80;
  fence_proxy_async_smem();
  __syncthreads();
  if (threadIdx.x == 0) {
    tma_store_4d(&m, buf, 0, c1, c2, 0);
    bulk_commit();
    bulk_wait<0>();
  }
}
int main() {
  void* p; cudaMalloc(&p, 64 * 56 * 56 * 2 * 2);
  void* fp = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  EncFn fn = (EncFn)fp;
  CUtensorMap m;
  cuuint64_t dims[4] = {64, 56, 56, 2};
  cuuint64_t str[3] = {128, 56 * 128, 56 * 56 * 128};
  cuuint32_t box[4] = {32, 32, 1, 1}, es[4] = {1, 1, 1, 1};
  printf("encode %d\n", (int)fn(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, p, dims, str, box, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  int cases[][2] = {{0, 0}, {40, 0}, {-5, 1}, {-40, 2}, {0, -1}};
  for (auto& c : cases) {
    k<<<1, 128>>>(m, c[0], c[1]);
    printf("store at w=%d h=%d: %s\n", c[0], c[1], cudaGetErrorString(cudaDeviceSynchronize()));
  }
}
