#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
typedef CUresult (*PFN)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main(){
  void* p; cudaDriverEntryPointQueryResult q; cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  PFN enc=(PFN)p; double* y; cudaMalloc(&y, 1<<20); CUtensorMap m;
  cuuint64_t d1[1]={1000}; cuuint32_t b1[1]={32}; cuuint32_t es[2]={1,1}; cuuint64_t st[1]={8000};
  printf("rank1 null strides: %d\n", enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 1, y, d1, nullptr, b1, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  printf("rank1 dummy strides: %d\n", enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 1, y, d1, st, b1, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  printf("rank1 no promo: %d\n", enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 1, y, d1, st, b1, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  cuuint64_t d2[2]={1000,1}; cuuint32_t b2[2]={32,1}; cuuint64_t s2[1]={8000};
  printf("rank2 {n,1}: %d\n", enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, y, d2, s2, b2, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  cuuint64_t d3[1]={1000}; cuuint32_t b3[1]={32};
  printf("rank1 L2_128: %d\n", enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 1, y, d3, st, b3, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  return 0;
}
