// tma_test.cu -- standalone check of the pair-row TMA view used by k_search_tma (debugging aid).
// Loads one {bw x bh} box of a {2n, rows/2} FLOAT64 view of an n x rows array (n odd) with
// cp.async.bulk.tensor.2d + mbarrier, and compares with the expected elements.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tma_test tools/tma_test.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void k_tma(const __grid_constant__ CUtensorMap map, const CUtensorMap* gmap, int x, int y, int bw,
                      int bh, double* out, int* status) {
  const CUtensorMap* mp = (MODE == 2) ? gmap : &map;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar;
  double* box = (double*)(((uintptr_t)sm + 127) & ~(uintptr_t)127);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)),
                 "r"(bw * bh * 8) : "memory");
    if (MODE == 3)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(box)), "l"((const void*)gmap), "r"(bw * bh * 8), "r"(smem_u32(&bar)) : "memory");
    else if (MODE == 0)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
          ::"r"(smem_u32(box)), "l"((uint64_t)mp), "r"(x), "r"(y), "r"(smem_u32(&bar)) : "memory");
    else
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
          ::"r"(smem_u32(box)), "l"((uint64_t)mp), "r"(x), "r"(y), "r"(smem_u32(&bar)) : "memory");
  }
  uint32_t done = 0;
  long long spin = 0;
  while (!done && spin < (1LL << 26)) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done) : "r"(smem_u32(&bar)), "r"(0) : "memory");
    ++spin;
  }
  if (threadIdx.x == 0) *status = done ? 1 : -1;
  __syncthreads();
  if (done)
    for (int e = threadIdx.x; e < bw * bh; e += blockDim.x) out[e] = box[e];
}

int main(int argc, char** argv) {
  const int only = argc > 1 ? atoi(argv[1]) : -1;
  const int n = 257, rows = 257;
  int bw = 36, bh = 7;
  int dtype_f32 = 0, promo_none = 0;
  if (only >= 6) {  // argv: mode bw bh f32 promo_none
    bw = atoi(argv[2]);
    bh = atoi(argv[3]);
    dtype_f32 = atoi(argv[4]);
    promo_none = atoi(argv[5]);
  }
  std::vector<double> h((size_t)n * rows);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
  double *d, *out;
  int* st;
  cudaMalloc(&d, h.size() * 8);
  cudaMalloc(&out, bw * bh * 8);
  cudaMalloc(&st, 4);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeTiledFn enc = (EncodeTiledFn)p;
  CUtensorMap map;
  const cuuint64_t dims[2] = {2ull * n, (cuuint64_t)(rows / 2)};
  const cuuint64_t strides[1] = {2ull * n * 8};
  const cuuint32_t box[2] = {(cuuint32_t)bw, (cuuint32_t)bh};
  const cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: %d (entry point query %d)\n", (int)r, (int)q);
  const int x = n + 40, y = 60;  // odd rows of pair-row 60.. : local rows 121, 123, ...
  CUtensorMap* gmap;
  cudaMalloc(&gmap, sizeof(CUtensorMap));
  cudaMemcpy(gmap, &map, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
  if (only >= 6) {
    CUtensorMap m3;
    const int es_b = dtype_f32 ? 4 : 8;
    const cuuint64_t dims3[2] = {(cuuint64_t)(2 * n * 8 / es_b), (cuuint64_t)(rows / 2)};
    const cuuint32_t box3[2] = {(cuuint32_t)bw, (cuuint32_t)bh};
    CUresult r3 = enc(&m3, dtype_f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims3,
                      strides, box3, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      promo_none ? CU_TENSOR_MAP_L2_PROMOTION_NONE : CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaMemset(st, 0, 4);
    const int bytes_total = bw * bh * es_b;
    const int cx = argc > 6 ? atoi(argv[6]) : 8, cy = argc > 7 ? atoi(argv[7]) : 3;
    k_tma<0><<<1, 128, bytes_total + 256>>>(m3, gmap, cx, cy, bytes_total / 8, 1, out, st);
    cudaError_t e = cudaDeviceSynchronize();
    int hs = 0;
    cudaMemcpy(&hs, st, 4, cudaMemcpyDeviceToHost);
    printf("mode %d: box {%d,%d} at (%d,%d) %s promo %s encode=%d -> err=%s status=%d\n", only, bw, bh, cx, cy,
           dtype_f32 ? "F32" : "F64", promo_none ? "none" : "256B", (int)r3, cudaGetErrorString(e), hs);
    return 0;
  }
  for (int mode = 0; mode < 6; ++mode) {
    if (only >= 0 && mode != only) continue;
    cudaMemset(st, 0, 4);
    const size_t smem = bw * bh * 8 + 128;
    CUtensorMap m2 = map;
    if (mode >= 4) {
      CUresult r2 = enc(&m2, mode == 4 ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : CU_TENSOR_MAP_DATA_TYPE_INT64, 2, d, dims,
                        strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      printf("encode mode %d: %d\n", mode, (int)r2);
    }
    if (mode == 0 || mode >= 4) k_tma<0><<<1, 128, smem>>>(m2, gmap, x, y, bw, bh, out, st);
    else if (mode == 1) k_tma<1><<<1, 128, smem>>>(map, gmap, x, y, bw, bh, out, st);
    else if (mode == 2) k_tma<2><<<1, 128, smem>>>(map, gmap, x, y, bw, bh, out, st);
    else k_tma<3><<<1, 128, smem>>>(map, (const CUtensorMap*)(d + (size_t)y * 2 * n + (x & ~1)), x, y, bw, bh, out, st);
    cudaError_t e = cudaDeviceSynchronize();
    int hs = 0;
    cudaMemcpy(&hs, st, 4, cudaMemcpyDeviceToHost);
    std::vector<double> o(bw * bh);
    cudaMemcpy(o.data(), out, o.size() * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int j = 0; j < bh && hs == 1; ++j)
      for (int i = 0; i < bw; ++i) {
        const size_t el = mode == 3 ? (size_t)y * 2 * n + (x & ~1) + j * bw + i   // 1D bulk copy
                                    : (size_t)(y + j) * 2 * n + (x + i);          // element in the flat array
        if (o[j * bw + i] != h[el]) ++bad;
      }
    printf("mode %d (%s): err=%s status=%d mismatches=%d\n", mode,
           mode == 0 ? ".tile, param map, F64" : mode == 1 ? "no .tile, param map" : mode == 2 ? ".tile, global map"
           : mode == 3 ? "1D cp.async.bulk" : mode == 4 ? ".tile, UINT64 map" : ".tile, INT64 map",
           cudaGetErrorString(e), hs, bad);
  }
  return 0;
}
