// Probe: can a TMA tensor store (cp.async.bulk.tensor) target peer-mapped
// memory (cudaDeviceEnablePeerAccess)?  GPU 0 stores a 32x32 fp32 box into a
// buffer that lives on GPU 1; the host checks it.  Also times 1 GiB of boxes.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

using EncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                              const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                              const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__global__ void store_boxes(const __grid_constant__ CUtensorMap map, int rows, int cols, int iters) {
  __shared__ alignas(128) float box[32 * 32];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) box[i] = (float)(blockIdx.x * 1024 + i);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    const int nbx = cols / 32, nby = rows / 32, nb = nbx * nby;
    for (int it = 0; it < iters; ++it)
      for (int b = blockIdx.x; b < nb; b += gridDim.x) {
        int c0 = (b % nbx) * 32, r0 = (b / nbx) * 32;
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                         reinterpret_cast<uint64_t>(&map)), "r"(c0), "r"(r0),
                     "r"((uint32_t)__cvta_generic_to_shared(box))
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory");
      }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

int main() {
  int n = 0;
  cudaGetDeviceCount(&n);
  if (n < 2) { printf("SKIP need 2 GPUs\n"); return 0; }
  const int rows = 16384, cols = 16384;  // 1 GiB fp32
  float *dst = nullptr;
  cudaSetDevice(1);
  cudaMalloc(&dst, (size_t)rows * cols * 4);
  cudaMemset(dst, 0, (size_t)rows * cols * 4);
  cudaDeviceSynchronize();
  cudaSetDevice(0);
  cudaError_t e = cudaDeviceEnablePeerAccess(1, 0);
  printf("peer access: %s\n", cudaGetErrorString(e));
  void *fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fp;
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
  cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dst, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode on peer pointer: %d\n", (int)r);
  store_boxes<<<148, 128>>>(map, rows, cols, 1);
  e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<float> h(32 * 32);
  cudaMemcpy2D(h.data(), 128, dst, (size_t)cols * 4, 128, 32, cudaMemcpyDefault);
  bool ok = true;
  for (int i = 0; i < 1024; ++i) ok &= h[i] == (float)i;  // box 0 written by block 0
  printf("box 0 check: %s (h[5]=%f)\n", ok ? "OK" : "BAD", h[5]);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int grid : {16, 32, 74, 148}) {
    cudaEventRecord(a);
    store_boxes<<<grid, 128>>>(map, rows, cols, 3);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("grid %d: TMA store to peer %.1f GB/s\n", grid, 3.0 * rows * cols * 4 / ms / 1e6);
  }
  printf("%s\n", ok ? "PASS" : "FAIL");
  return ok ? 0 : 1;
}
