// Latency probe kernels (scripts/probes/latency_probe.py): what does one
// graph-launched handshake kernel cost on B200, piece by piece?
//   empty      : a 1-thread kernel doing nothing (launch floor)
//   fence      : fence.acq_rel.sys only
//   fence_sc   : fence.sc.sys (= __threadfence_system) only
//   store      : relaxed .sys store of a u64 to (peer) memory
//   fence_store: fence.acq_rel.sys + relaxed .sys store (our post)
//   poll       : wait until *flag >= v (ld.acquire.sys, no sleep)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC
//        -o latency_kernels.so latency_kernels.cu
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_empty() {}
__global__ void k_fence() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__global__ void k_fence_sc() { asm volatile("fence.sc.sys;" ::: "memory"); }
__global__ void k_store(uint64_t *p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__global__ void k_fence_store(uint64_t *p, uint64_t v) {
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__global__ void k_poll(const uint64_t *p, uint64_t v) {
  uint64_t x;
  do {
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(x) : "l"(p) : "memory");
  } while (x < v);
}

extern "C" int probe_launch(int which, void *p, uint64_t v, void *stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  switch (which) {
    case 0: k_empty<<<1, 1, 0, s>>>(); break;
    case 1: k_fence<<<1, 1, 0, s>>>(); break;
    case 2: k_fence_sc<<<1, 1, 0, s>>>(); break;
    case 3: k_store<<<1, 1, 0, s>>>(static_cast<uint64_t *>(p), v); break;
    case 4: k_fence_store<<<1, 1, 0, s>>>(static_cast<uint64_t *>(p), v); break;
    case 5: k_poll<<<1, 1, 0, s>>>(static_cast<const uint64_t *>(p), v); break;
    default: return -1;
  }
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}
