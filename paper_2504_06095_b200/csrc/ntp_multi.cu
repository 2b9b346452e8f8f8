// R-way gradient sync across DP > 2 replicas with arbitrary (nonuniform) layouts.
//
// The reference syncs exactly two replicas nonuniformly (tpnumerics.py:289-356)
// and R identically laid out replicas uniformly (263-286).  A DP=4 x TP2 job with
// one replica degraded to TP1 (BASELINE configs[2]) needs both at once: every
// unit j has R owners (one per replica, each in its own layout) and ends as
//   v_j = sum_r w_r * g_r[j]      (replica order, explicit fp32 rounding)
// in all R owners.  One kernel reads the R copies of each unit once and writes
// the result R times: 2*R*U*b bytes per unit, the HBM minimum when all replicas
// are local.  Plans are host-built tables of chunks; each chunk carries R
// (buffer, offset) pairs in structure-of-arrays form.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <new>
#include <string>
#include <vector>

#include "ntp_internal.h"

namespace ntp {
namespace multi {

constexpr int kMaxR = 8;
constexpr int kThreads = 256;
constexpr uint32_t kChunkVecs = 1024;  // 16 KiB per replica per chunk

struct Table {
  uint32_t *off[kMaxR];  // grains
  uint16_t *buf[kMaxR];
  uint32_t *len;
};

struct Weights {
  float w[kMaxR];
  double wd[kMaxR];
};

struct BufTable {
  char *p[kMaxBufs];
};

__device__ __forceinline__ float f(float x) { return x; }

template <typename T>
struct Vec;
template <>
struct Vec<float> {
  static constexpr int n = 4;
  __device__ static void unpack(uint4 v, float *o) {
    o[0] = __uint_as_float(v.x); o[1] = __uint_as_float(v.y);
    o[2] = __uint_as_float(v.z); o[3] = __uint_as_float(v.w);
  }
  __device__ static uint4 pack(const float *o) {
    return make_uint4(__float_as_uint(o[0]), __float_as_uint(o[1]), __float_as_uint(o[2]),
                      __float_as_uint(o[3]));
  }
};
template <>
struct Vec<__nv_bfloat16> {
  static constexpr int n = 8;
  __device__ static void unpack(uint4 v, float *o) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __nv_bfloat162 h = *reinterpret_cast<const __nv_bfloat162 *>(&w[i]);
      float2 t = __bfloat1622float2(h);
      o[2 * i] = t.x;
      o[2 * i + 1] = t.y;
    }
  }
  __device__ static uint4 pack(const float *o) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __nv_bfloat162 h = __floats2bfloat162_rn(o[2 * i], o[2 * i + 1]);
      w[i] = *reinterpret_cast<uint32_t *>(&h);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
  }
};

// op: 0 sum (replica order), 1 true mean (sum then / R, tpnumerics.py:280-283),
// 2 weighted sum_r w_r x_r
template <typename T, int R>
__global__ void __launch_bounds__(kThreads)
multi_kernel(Table tab, int n_chunks, BufTable bufs, Weights wts, int op) {
  constexpr int E = Vec<T>::n;
  for (int c = blockIdx.x; c < n_chunks; c += gridDim.x) {
    uint4 *ptr[R];
#pragma unroll
    for (int r = 0; r < R; ++r)
      ptr[r] = reinterpret_cast<uint4 *>(bufs.p[__ldg(tab.buf[r] + c)]) + __ldg(tab.off[r] + c);
    const int len = (int)__ldg(tab.len + c);
    for (int i = threadIdx.x; i < len; i += kThreads) {
      uint4 v[R];
#pragma unroll
      for (int r = 0; r < R; ++r) v[r] = __ldcs(ptr[r] + i);
      float acc[E], x[E];
      Vec<T>::unpack(v[0], acc);
      if (op == 2) {
#pragma unroll
        for (int e = 0; e < E; ++e) acc[e] = __fmul_rn(wts.w[0], acc[e]);
      } else if (op == 1) {
#pragma unroll
        for (int e = 0; e < E; ++e) acc[e] = __fadd_rn(0.0f, acc[e]);
      }
#pragma unroll
      for (int r = 1; r < R; ++r) {
        Vec<T>::unpack(v[r], x);
#pragma unroll
        for (int e = 0; e < E; ++e)
          acc[e] = __fadd_rn(acc[e], op == 2 ? __fmul_rn(wts.w[r], x[e]) : x[e]);
      }
      if (op == 1) {
#pragma unroll
        for (int e = 0; e < E; ++e) acc[e] = __fdiv_rn(acc[e], (float)R);
      }
      const uint4 o = Vec<T>::pack(acc);
#pragma unroll
      for (int r = 0; r < R; ++r) __stcs(ptr[r] + i, o);
    }
  }
}

// ---------------------------------------------------------------------------
// TMA-bulk variant (R <= 4): a producer warp streams the R copies of each chunk
// into a shared-memory ring with cp.async.bulk (mbarrier complete_tx), four
// consumer warps combine them in place, and one thread bulk-stores the result
// to all R owners.  Up to 192 KiB per SM in flight: with peer-mapped copies the
// NVLink reads of the next chunks overlap the stores of this one.

constexpr int kBulkConsumers = 128;
constexpr int kBulkThreads = kBulkConsumers + 32;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

template <int R, int kStages>
struct BulkSmem {
  uint4 slot[kStages][R][kChunkVecs];
  uint64_t full[kStages];
  uint64_t empty[kStages];
};

template <typename T, int R, int kStages>
__global__ void __launch_bounds__(kBulkThreads, 1)
multi_kernel_bulk(Table tab, int n_chunks, BufTable bufs, Weights wts, int op) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  auto &sm = *reinterpret_cast<BulkSmem<R, kStages> *>(smem_raw);
  constexpr int E = Vec<T>::n;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid >= kBulkConsumers) {
    // ---- producer ----
    if (tid == kBulkConsumers) {
      int stage = 0;
      uint32_t phase = 0;
      for (int c = blockIdx.x; c < n_chunks; c += gridDim.x) {
        const uint32_t bytes = __ldg(tab.len + c) * 16u;
        mbar_wait(&sm.empty[stage], phase ^ 1u);
        mbar_expect_tx(&sm.full[stage], R * bytes);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const uint4 *src =
              reinterpret_cast<const uint4 *>(bufs.p[__ldg(tab.buf[r] + c)]) + __ldg(tab.off[r] + c);
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  smem_u32(sm.slot[stage][r])),
              "l"(src), "r"(bytes), "r"(smem_u32(&sm.full[stage]))
              : "memory");
        }
        if (++stage == kStages) { stage = 0; phase ^= 1u; }
      }
    }
    return;
  }
  // ---- consumers ----
  int stage = 0, prev_stage = -1;
  uint32_t phase = 0;
  for (int c = blockIdx.x; c < n_chunks; c += gridDim.x) {
    const int len = (int)__ldg(tab.len + c);
    mbar_wait(&sm.full[stage], phase);
    for (int i = tid; i < len; i += kBulkConsumers) {
      float acc[E], x[E];
      Vec<T>::unpack(sm.slot[stage][0][i], acc);
      if (op == 2) {
#pragma unroll
        for (int e = 0; e < E; ++e) acc[e] = __fmul_rn(wts.w[0], acc[e]);
      } else if (op == 1) {
#pragma unroll
        for (int e = 0; e < E; ++e) acc[e] = __fadd_rn(0.0f, acc[e]);
      }
#pragma unroll
      for (int r = 1; r < R; ++r) {
        Vec<T>::unpack(sm.slot[stage][r][i], x);
#pragma unroll
        for (int e = 0; e < E; ++e)
          acc[e] = __fadd_rn(acc[e], op == 2 ? __fmul_rn(wts.w[r], x[e]) : x[e]);
      }
      if (op == 1) {
#pragma unroll
        for (int e = 0; e < E; ++e) acc[e] = __fdiv_rn(acc[e], (float)R);
      }
      sm.slot[stage][0][i] = Vec<T>::pack(acc);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("bar.sync 1, %0;" ::"r"(kBulkConsumers) : "memory");
    if (tid == 0) {
      const uint32_t bytes = (uint32_t)len * 16u;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        uint4 *dst = reinterpret_cast<uint4 *>(bufs.p[__ldg(tab.buf[r] + c)]) + __ldg(tab.off[r] + c);
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                     "r"(smem_u32(sm.slot[stage][0])), "r"(bytes)
                     : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      // the previous stage's stores have finished reading shared memory
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      if (prev_stage >= 0) mbar_arrive(&sm.empty[prev_stage]);
    }
    prev_stage = stage;
    if (++stage == kStages) { stage = 0; phase ^= 1u; }
  }
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <typename T, int R, int kStages>
static cudaError_t launch_bulk(const Table &tab, int nc, const BufTable &bt, const Weights &wts,
                               int op, int sms, cudaStream_t s) {
  auto k = multi_kernel_bulk<T, R, kStages>;
  const int smem = (int)sizeof(BulkSmem<R, kStages>);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int grid = nc < sms ? nc : sms;
  k<<<grid, kBulkThreads, smem, s>>>(tab, nc, bt, wts, op);
  return cudaGetLastError();
}

// 0: AUTO (bulk for R <= 4 and >= 2 chunks per SM), 1: LDG, 2: bulk when R <= 4
std::atomic<int> g_multi_kernel{0};

}  // namespace multi
}  // namespace ntp

struct ntp_mplan {
  int dtype = NTP_BF16;
  int R = 0;
  bool finalized = false;
  int64_t n_units = 0, elems = 0;
  int max_buf = -1;
  // merged runs: R (buf, off) pairs + length, elements
  std::vector<int32_t> run_buf;   // R per run
  std::vector<int64_t> run_off;   // R per run
  std::vector<int64_t> run_len;
  // chunk table (host, SoA)
  std::vector<uint32_t> c_off;    // R x n_chunks (replica-major)
  std::vector<uint16_t> c_buf;
  std::vector<uint32_t> c_len;
  void *d_mem = nullptr;
  int device = -1;
};

using namespace ntp;

extern "C" {

int ntp_mplan_create(ntp_mplan **out, int dtype, int R) {
  if (!out) return fail(NTP_EINVAL, "null plan pointer");
  if (dtype != NTP_BF16 && dtype != NTP_F32)
    return fail(NTP_EINVAL, "R-way sync supports bf16 and fp32");
  if (R < 2 || R > multi::kMaxR) return fail(NTP_EINVAL, "replica count must be in [2, 8]");
  ntp_mplan *p = new (std::nothrow) ntp_mplan();
  if (!p) return fail(NTP_ENOMEM, "out of host memory");
  p->dtype = dtype;
  p->R = R;
  *out = p;
  return NTP_OK;
}

// bufs, offs: [R][n_units] (replica-major), element offsets.
int ntp_mplan_add_units(ntp_mplan *p, int64_t n_units, int64_t unit_elems, const int32_t *bufs,
                        const int64_t *offs) {
  if (!p) return fail(NTP_EINVAL, "null plan");
  if (p->finalized) return fail(NTP_ESTATE, "plan already finalized");
  if (n_units < 0 || unit_elems <= 0) return fail(NTP_EINVAL, "bad unit count or size");
  const int R = p->R;
  for (int64_t j = 0; j < n_units; ++j) {
    bool merge = !p->run_len.empty();
    const size_t base = p->run_len.size() * (size_t)R;
    for (int r = 0; r < R; ++r) {
      const int32_t b = bufs[(size_t)r * n_units + j];
      const int64_t o = offs[(size_t)r * n_units + j];
      if (b < 0 || b >= kMaxBufs) return fail(NTP_EINVAL, "buffer index out of range (max 64)");
      if (o < 0) return fail(NTP_EINVAL, "negative offset");
      p->max_buf = std::max(p->max_buf, (int)b);
      if (merge) {
        const size_t q = base - R + r;
        if (p->run_buf[q] != b || p->run_off[q] + p->run_len.back() != o) merge = false;
      }
    }
    if (merge) {
      p->run_len.back() += unit_elems;
      continue;
    }
    for (int r = 0; r < R; ++r) {
      p->run_buf.push_back(bufs[(size_t)r * n_units + j]);
      p->run_off.push_back(offs[(size_t)r * n_units + j]);
    }
    p->run_len.push_back(unit_elems);
  }
  p->n_units += n_units;
  p->elems += n_units * unit_elems;
  return NTP_OK;
}

int ntp_mplan_finalize(ntp_mplan *p) {
  if (!p) return fail(NTP_EINVAL, "null plan");
  if (p->finalized) return NTP_OK;
  const int R = p->R;
  const int64_t vec = 16 / dtype_bytes(p->dtype);
  const size_t nr = p->run_len.size();
  std::vector<uint32_t> off;
  std::vector<uint16_t> buf;
  std::vector<uint32_t> len;
  for (size_t i = 0; i < nr; ++i) {
    if (p->run_len[i] % vec) return fail(NTP_EINVAL, "R-way sync needs 16-byte aligned units");
    for (int r = 0; r < R; ++r)
      if (p->run_off[i * R + r] % vec) return fail(NTP_EINVAL, "R-way sync needs 16-byte aligned units");
    const int64_t g = p->run_len[i] / vec;
    const int64_t pieces = (g + multi::kChunkVecs - 1) / multi::kChunkVecs;
    for (int64_t c = 0; c < pieces; ++c) {
      const int64_t lo = g * c / pieces, hi = g * (c + 1) / pieces;
      len.push_back((uint32_t)(hi - lo));
      for (int r = 0; r < R; ++r) {
        const int64_t o = p->run_off[i * R + r] / vec + lo;
        if (o + (hi - lo) > UINT32_MAX) return fail(NTP_EINVAL, "offset exceeds 32-bit grains");
        off.push_back((uint32_t)o);
        buf.push_back((uint16_t)p->run_buf[i * R + r]);
      }
    }
  }
  // chunk-major -> replica-major SoA
  const size_t nc = len.size();
  p->c_off.assign(nc * R, 0);
  p->c_buf.assign(nc * R, 0);
  for (size_t c = 0; c < nc; ++c)
    for (int r = 0; r < R; ++r) {
      p->c_off[r * nc + c] = off[c * R + r];
      p->c_buf[r * nc + c] = buf[c * R + r];
    }
  p->c_len = std::move(len);
  p->finalized = true;
  return NTP_OK;
}

int64_t ntp_mplan_chunks(const ntp_mplan *p) {
  if (!p || !p->finalized) return fail(NTP_ESTATE, "plan not finalized");
  return (int64_t)p->c_len.size();
}

int ntp_mplan_upload(ntp_mplan *p, int device) {
  if (!p || !p->finalized) return fail(NTP_ESTATE, "plan not finalized");
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return fail(NTP_ECUDA, cudaGetErrorString(e));
  if (p->d_mem) {
    cudaFree(p->d_mem);
    p->d_mem = nullptr;
  }
  p->device = device;
  const size_t nc = p->c_len.size();
  if (!nc) return NTP_OK;
  const size_t bytes = nc * 4 * p->R + nc * 2 * p->R + nc * 4 + 64;
  e = cudaMalloc(&p->d_mem, bytes);
  if (e != cudaSuccess) return fail(NTP_ECUDA, cudaGetErrorString(e));
  char *d = static_cast<char *>(p->d_mem);
  cudaMemcpy(d, p->c_off.data(), nc * 4 * p->R, cudaMemcpyHostToDevice);
  cudaMemcpy(d + nc * 4 * p->R, p->c_len.data(), nc * 4, cudaMemcpyHostToDevice);
  e = cudaMemcpy(d + nc * 4 * p->R + nc * 4, p->c_buf.data(), nc * 2 * p->R, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return fail(NTP_ECUDA, cudaGetErrorString(e));
  return NTP_OK;
}

void ntp_mplan_destroy(ntp_mplan *p) {
  if (!p) return;
  if (p->d_mem) device_free(p->d_mem, p->device);
  delete p;
}

int ntp_multi_sync(const ntp_mplan *p, void *const *bufs, int n_bufs, int op, const double *w,
                   void *stream) {
  if (!p || !p->finalized) return fail(NTP_ESTATE, "plan not finalized");
  if (p->device < 0) return fail(NTP_ESTATE, "plan not uploaded");
  if (op < NTP_OP_SUM || op > NTP_OP_WEIGHTED) return fail(NTP_EINVAL, "unknown reduction op");
  if (op == NTP_OP_WEIGHTED && !w) return fail(NTP_EINVAL, "weighted op needs R weights");
  if (n_bufs <= p->max_buf || n_bufs > kMaxBufs)
    return fail(NTP_EINVAL, "plan references more buffers than were passed");
  const size_t nc = p->c_len.size();
  if (!nc) return NTP_OK;
  cudaSetDevice(p->device);
  multi::BufTable bt{};
  for (int i = 0; i < n_bufs; ++i) {
    bt.p[i] = static_cast<char *>(bufs[i]);
    if (reinterpret_cast<uintptr_t>(bt.p[i]) & 15u)
      return fail(NTP_EINVAL, "buffer not 16-byte aligned");
  }
  multi::Table tab{};
  char *d = static_cast<char *>(p->d_mem);
  for (int r = 0; r < p->R; ++r) {
    tab.off[r] = reinterpret_cast<uint32_t *>(d) + r * nc;
    tab.buf[r] = reinterpret_cast<uint16_t *>(d + nc * 4 * p->R + nc * 4) + r * nc;
  }
  tab.len = reinterpret_cast<uint32_t *>(d + nc * 4 * p->R);
  multi::Weights wts{};
  for (int r = 0; r < p->R; ++r) {
    wts.w[r] = w ? (float)w[r] : 1.0f;
    wts.wd[r] = w ? w[r] : 1.0;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->device);
  const int grid = (int)std::min<size_t>(nc, (size_t)sms * 4);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int variant = multi::g_multi_kernel.load();
  // AUTO: the bulk ring pays off when copies live on peers (NVLink latency);
  // with every copy in local HBM the 128-bit-load kernel is faster (0.958 vs
  // 0.922 of HBM on the C3 shape, scripts/multi_bench.py)
  bool any_peer = false;
  if (variant == 0)
    for (int i = 0; i < n_bufs && !any_peer; ++i) {
      cudaPointerAttributes a{};
      if (cudaPointerGetAttributes(&a, bufs[i]) == cudaSuccess && a.device != p->device)
        any_peer = true;
    }
  const bool bulk =
      p->R <= 4 && (variant == 2 || (variant == 0 && any_peer && nc >= (size_t)sms * 2));
  if (bulk) {
    cudaError_t e = cudaSuccess;
    const int n = (int)nc;
    if (p->dtype == NTP_BF16) {
      if (p->R == 2) e = multi::launch_bulk<__nv_bfloat16, 2, 6>(tab, n, bt, wts, op, sms, s);
      else if (p->R == 3) e = multi::launch_bulk<__nv_bfloat16, 3, 4>(tab, n, bt, wts, op, sms, s);
      else e = multi::launch_bulk<__nv_bfloat16, 4, 3>(tab, n, bt, wts, op, sms, s);
    } else {
      if (p->R == 2) e = multi::launch_bulk<float, 2, 6>(tab, n, bt, wts, op, sms, s);
      else if (p->R == 3) e = multi::launch_bulk<float, 3, 4>(tab, n, bt, wts, op, sms, s);
      else e = multi::launch_bulk<float, 4, 3>(tab, n, bt, wts, op, sms, s);
    }
    if (e != cudaSuccess) return fail(NTP_ECUDA, std::string("multi sync (bulk): ") + cudaGetErrorString(e));
    return NTP_OK;
  }
#define NTP_MULTI_CASE(TT, RR) \
  case RR: multi::multi_kernel<TT, RR><<<grid, multi::kThreads, 0, s>>>(tab, (int)nc, bt, wts, op); break;
  if (p->dtype == NTP_BF16) {
    switch (p->R) {
      NTP_MULTI_CASE(__nv_bfloat16, 2) NTP_MULTI_CASE(__nv_bfloat16, 3)
      NTP_MULTI_CASE(__nv_bfloat16, 4) NTP_MULTI_CASE(__nv_bfloat16, 5)
      NTP_MULTI_CASE(__nv_bfloat16, 6) NTP_MULTI_CASE(__nv_bfloat16, 7)
      NTP_MULTI_CASE(__nv_bfloat16, 8)
    }
  } else {
    switch (p->R) {
      NTP_MULTI_CASE(float, 2) NTP_MULTI_CASE(float, 3) NTP_MULTI_CASE(float, 4)
      NTP_MULTI_CASE(float, 5) NTP_MULTI_CASE(float, 6) NTP_MULTI_CASE(float, 7)
      NTP_MULTI_CASE(float, 8)
    }
  }
#undef NTP_MULTI_CASE
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(NTP_ECUDA, std::string("multi sync: ") + cudaGetErrorString(e));
  return NTP_OK;
}

// Kernel variant for ntp_multi_sync: 0 AUTO, 1 LDG, 2 TMA bulk (R <= 4).
int ntp_multi_set_kernel(int variant) {
  if (variant < 0 || variant > 2) return fail(NTP_EINVAL, "multi kernel variant must be 0..2");
  multi::g_multi_kernel.store(variant);
  return NTP_OK;
}

}  // extern "C"
