// Device side of the NTP gradient reshard-and-reduce (sm_100a).
//
// One kernel family covers the whole data path of the reference's
// nonuniform_grad_sync (pkg/src/ntpsim/tpnumerics.py:289-356): instead of
// gathering the healthy replica into the reduced layout (323-333), reducing
// pairwise (338-347) and scattering back (349-356), every unit is read once
// from each of its two owners -- local HBM or a peer GPU's HBM through an
// NVLink-mapped pointer -- reduced in fp32 (fp64 for fp64 data) and written
// once to each owner.  A plan is a table of 16-byte chunk records (see
// ntp_internal.h) built on the host; a persistent grid walks it.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <atomic>
#include <mutex>
#include <string>

#include "ntp_internal.h"

namespace ntp {

static int cuda_fail(cudaError_t e, const char *what) {
  std::string msg = std::string(what) + ": " + cudaGetErrorString(e);
  return fail(NTP_ECUDA, msg);
}

#define NTP_CUDA(call)                                   \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) return cuda_fail(_e, #call);  \
  } while (0)

int device_free(void *p, int device) {
  int prev = 0;
  cudaGetDevice(&prev);
  if (device >= 0) cudaSetDevice(device);
  cudaFree(p);
  if (device >= 0) cudaSetDevice(prev);
  return NTP_OK;
}

struct BufTable {
  char *p[kMaxBufs];
};

// Cap on sync-kernel CTAs (0 = one wave over all SMs).  Lets a sync that is
// overlapped with the backward GEMMs leave most SMs to the tensor cores.
static std::atomic<int> g_max_ctas{0};
static uint64_t *g_trace = nullptr;  // debug: ntp_debug_sync_trace
static std::atomic<int> g_l2_hint{0};  // NTP_OPT_SYNC_L2

struct SignalArgs {
  uint64_t *wait[16];
  uint64_t *post[16];
  int n_wait, n_post;
  // single-launch step (ntp_grad_sync_step): `pre` words are posted before the
  // wait (this process's "ready"), `fin` words are waited for after the post
  // (the partners' "done"); both empty for ntp_grad_sync_signaled
  uint64_t *pre[16];
  uint64_t *fin[16];
  int n_pre, n_fin;
  uint64_t epoch;
  uint64_t spin_ns;
  int *status;
  unsigned int *counter;  // CTA completion counter (device, zeroed)
  int wmask = 3;          // bit 0: write side A, bit 1: write side B
  // device-resident epochs (CUDA-graph replayable steps): when set, the epoch
  // of this launch is *epoch_word + 1 (the word counts completed steps), and
  // the step's final kernel (advance = 1) stores that epoch back
  uint64_t *epoch_word = nullptr;
  int advance = 0;
  // debug only (ntp_debug_sync_trace, not in the header): globaltimer stamps
  // [0] CTA 0 start, [1] ready posted, [2] ready seen by CTA 0, [3] last CTA
  // entered its finish, [4] done posted, [5] partners' done seen
  uint64_t *trace = nullptr;
  // L2 policy of the bulk kernel's copies (NTP_OPT_SYNC_L2): 0 none, 1 loads
  // evict_first, 2 loads and stores evict_first
  int l2_hint = 0;
};

enum { OP_COPY = 3 };
constexpr int kThreads = 256;
constexpr int kUnroll = kChunkVecs / kThreads;  // 4 x 16 B per side per thread

// ---------------------------------------------------------------------------
// element math

template <typename T>
struct Acc { using type = float; };
template <>
struct Acc<double> { using type = double; };

// Explicitly rounded operations: no FMA contraction, so the device result is
// the IEEE evaluation of the written expression (identical to the oracle's).
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }

template <int OP, typename A>
__device__ __forceinline__ A combine(A a, A b, A wa, A wb) {
  if constexpr (OP == NTP_OP_SUM) return add_rn(a, b);                      // tpnumerics.py:257
  else if constexpr (OP == NTP_OP_MEAN) return mul_rn(add_rn(a, b), A(0.5));  // 259: (a+b)/2.0 (exact *0.5)
  else return add_rn(mul_rn(wa, a), mul_rn(wb, b));                       // w_a*a + w_b*b
}

template <typename T> __device__ __forceinline__ float2 to_f2(uint32_t w);
template <>
__device__ __forceinline__ float2 to_f2<__nv_bfloat16>(uint32_t w) {
  __nv_bfloat162 h = *reinterpret_cast<__nv_bfloat162 *>(&w);
  return __bfloat1622float2(h);
}
template <>
__device__ __forceinline__ float2 to_f2<__half>(uint32_t w) {
  __half2 h = *reinterpret_cast<__half2 *>(&w);
  return __half22float2(h);
}
template <typename T> __device__ __forceinline__ uint32_t from_f2(float2 v);
template <>
__device__ __forceinline__ uint32_t from_f2<__nv_bfloat16>(float2 v) {
  __nv_bfloat162 h = __float22bfloat162_rn(v);
  return *reinterpret_cast<uint32_t *>(&h);
}
template <>
__device__ __forceinline__ uint32_t from_f2<__half>(float2 v) {
  __half2 h = __float22half2_rn(v);
  return *reinterpret_cast<uint32_t *>(&h);
}

// Reduce one 16-byte vector of each side.
template <typename T, int OP>
__device__ __forceinline__ uint4 combine_vec(uint4 a, uint4 b, float wa, float wb);

template <int OP>
__device__ __forceinline__ uint4 combine_vec_f32(uint4 a, uint4 b, float wa, float wb) {
  uint4 o;
  o.x = __float_as_uint(combine<OP, float>(__uint_as_float(a.x), __uint_as_float(b.x), wa, wb));
  o.y = __float_as_uint(combine<OP, float>(__uint_as_float(a.y), __uint_as_float(b.y), wa, wb));
  o.z = __float_as_uint(combine<OP, float>(__uint_as_float(a.z), __uint_as_float(b.z), wa, wb));
  o.w = __float_as_uint(combine<OP, float>(__uint_as_float(a.w), __uint_as_float(b.w), wa, wb));
  return o;
}

template <typename H, int OP>
__device__ __forceinline__ uint32_t combine_w16(uint32_t a, uint32_t b, float wa, float wb) {
  float2 x = to_f2<H>(a), y = to_f2<H>(b);
  return from_f2<H>(make_float2(combine<OP, float>(x.x, y.x, wa, wb),
                                combine<OP, float>(x.y, y.y, wa, wb)));
}

template <typename T, int OP>
struct VecOp {
  __device__ static __forceinline__ uint4 run(uint4 a, uint4 b, typename Acc<T>::type wa,
                                              typename Acc<T>::type wb) {
    uint4 o;
    o.x = combine_w16<T, OP>(a.x, b.x, wa, wb);
    o.y = combine_w16<T, OP>(a.y, b.y, wa, wb);
    o.z = combine_w16<T, OP>(a.z, b.z, wa, wb);
    o.w = combine_w16<T, OP>(a.w, b.w, wa, wb);
    return o;
  }
};
template <int OP>
struct VecOp<float, OP> {
  __device__ static __forceinline__ uint4 run(uint4 a, uint4 b, float wa, float wb) {
    return combine_vec_f32<OP>(a, b, wa, wb);
  }
};
template <int OP>
struct VecOp<double, OP> {
  __device__ static __forceinline__ uint4 run(uint4 a, uint4 b, double wa, double wb) {
    double2 x = *reinterpret_cast<double2 *>(&a), y = *reinterpret_cast<double2 *>(&b);
    double2 o = make_double2(combine<OP, double>(x.x, y.x, wa, wb),
                             combine<OP, double>(x.y, y.y, wa, wb));
    return *reinterpret_cast<uint4 *>(&o);
  }
};

// scalar element path (plans whose runs are not 16-byte aligned)
template <typename T, int OP>
__device__ __forceinline__ T combine_scalar(T a, T b, typename Acc<T>::type wa,
                                            typename Acc<T>::type wb) {
  using A = typename Acc<T>::type;
  return T(combine<OP, A>(A(a), A(b), wa, wb));
}

// streaming loads/stores: every byte is touched exactly once per launch
__device__ __forceinline__ uint4 ld_stream(const uint4 *p) { return __ldcs(p); }
__device__ __forceinline__ void st_stream(uint4 *p, uint4 v) { __stcs(p, v); }

// ---------------------------------------------------------------------------
// cross-GPU signals (release/acquire at system scope)

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t *p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// A release pattern for several flag words: ONE system-scope acq_rel fence,
// then relaxed system-scope stores.  (st.release.sys per word compiles to a
// MEMBAR.ALL.SYS per word, and __threadfence_system() to a MEMBAR.SC.SYS on
// top: each costs microseconds on a peer-memory path; SASS-checked.)
__device__ __forceinline__ void fence_acq_rel_sys() {
  asm volatile("fence.acq_rel.sys;" ::: "memory");
}
__device__ __forceinline__ void st_relaxed_sys(uint64_t *p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void release_words(uint64_t *const *w, int n, uint64_t v) {
  if (n == 0) return;
  fence_acq_rel_sys();
  for (int i = 0; i < n; ++i) st_relaxed_sys(w[i], v);
}
__device__ __forceinline__ uint64_t global_timer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// This launch's epoch: the host value, or (graph-replayable steps) one past
// the device word that counts completed steps.
__device__ __forceinline__ uint64_t sig_epoch(const SignalArgs &sig) {
  if (!sig.epoch_word) return sig.epoch;
  return *reinterpret_cast<volatile const uint64_t *>(sig.epoch_word) + 1;
}
__device__ __forceinline__ void sig_advance(const SignalArgs &sig, uint64_t e) {
  if (sig.epoch_word && sig.advance) *reinterpret_cast<volatile uint64_t *>(sig.epoch_word) = e;
}

// Returns false on timeout (status set).
__device__ bool wait_signals(uint64_t *const *wait, int n, uint64_t epoch, uint64_t spin_ns,
                             int *status) {
  const uint64_t t0 = global_timer_ns();
  for (int i = 0; i < n; ++i) {
    while (ld_acquire_sys(wait[i]) < epoch) {
      if (global_timer_ns() - t0 > spin_ns) {
        if (status) atomicExch(status, NTP_ETIMEOUT);
        return false;
      }
      __nanosleep(256);
    }
  }
  return true;
}

// ---------------------------------------------------------------------------
// the plan kernels

__device__ __forceinline__ void post_signals(uint64_t *const *post, int n, uint64_t epoch) {
  release_words(post, n, epoch);
}

// The plan's 256-byte counter block: u32 word 0 counts finished CTAs of the
// current launch, u64 word 1 records the last epoch whose ready words were
// posted, u32 word 4 counts CTAs of the current launch that timed out.
__device__ __forceinline__ unsigned int *failed_ctas(const SignalArgs &sig) { return sig.counter + 4; }

// Last CTA of a signalled launch: every CTA's stores are fenced -- reset the
// block for the next launch, then post the done words and (single-launch
// step) wait for the partners' done words.  If any CTA of this launch timed
// out (it skipped its chunks) the done words are NOT posted: the partners
// then time out too instead of consuming a partly reduced result, and every
// process's status reports the failure.
__device__ __forceinline__ void last_cta_finish(const SignalArgs &sig) {
  if (sig.trace) sig.trace[3] = global_timer_ns();
  fence_acq_rel_sys();  // acquire: every CTA's fenced stores happen-before what follows
  const uint64_t e = sig_epoch(sig);
  const unsigned int failed = atomicExch(failed_ctas(sig), 0u);
  *sig.counter = 0u;
  if (!failed) {
    release_words(sig.post, sig.n_post, e);
    if (sig.trace) sig.trace[4] = global_timer_ns();
    if (sig.n_fin) wait_signals(sig.fin, sig.n_fin, e, sig.spin_ns, sig.status);
    if (sig.trace) sig.trace[5] = global_timer_ns();
  }
  sig_advance(sig, e);  // every CTA has read the word: it is safe to move on
}

// A CTA whose ready-wait timed out does no work but still counts itself, so
// the counter block is reset by whichever CTA finishes last.
template <bool kSignaled>
__device__ __forceinline__ void cta_abort(const SignalArgs &sig) {
  if constexpr (kSignaled) {
    if (threadIdx.x == 0) {
      atomicAdd(failed_ctas(sig), 1u);
      __threadfence();
      const unsigned int done = atomicAdd(sig.counter, 1u);
      if (done == gridDim.x - 1) last_cta_finish(sig);
    }
  }
}

template <bool kSignaled>
__device__ __forceinline__ bool cta_prologue(const SignalArgs &sig) {
  if constexpr (kSignaled) {
    __shared__ int ok;
    if (threadIdx.x == 0) {
      // the first CTA to start posts this process's ready words, so no CTA
      // waits on a post that an unscheduled CTA would make (word 1 of the
      // plan's counter block records the last epoch posted)
      const bool tr = sig.trace && blockIdx.x == 0;
      if (tr) sig.trace[0] = global_timer_ns();
      const uint64_t e = sig_epoch(sig);
      if (sig.n_pre && atomicMax(reinterpret_cast<unsigned long long *>(sig.counter) + 1,
                                 (unsigned long long)e) < e)
        post_signals(sig.pre, sig.n_pre, e);
      if (tr) sig.trace[1] = global_timer_ns();
      ok = wait_signals(sig.wait, sig.n_wait, e, sig.spin_ns, sig.status) ? 1 : 0;
      if (tr) sig.trace[2] = global_timer_ns();
    }
    __syncthreads();
    return ok != 0;
  } else {
    return true;
  }
}

template <bool kSignaled>
__device__ __forceinline__ void cta_epilogue(const SignalArgs &sig) {
  if constexpr (kSignaled) {
    fence_acq_rel_sys();  // release this thread's peer/local stores, system scope
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned int done = atomicAdd(sig.counter, 1u);
      if (done == gridDim.x - 1) last_cta_finish(sig);  // every CTA's stores are fenced
    }
  }
}

// 128-bit path.  Each CTA walks chunks blockIdx.x, +gridDim.x, ...; the next
// record is prefetched while the current chunk's loads are in flight.
template <typename T, int OP, bool kSignaled>
__global__ void __launch_bounds__(kThreads)
plan_kernel_vec(const Chunk *__restrict__ chunks, int n_chunks, BufTable bufs,
                typename Acc<T>::type wa, typename Acc<T>::type wb, SignalArgs sig) {
  if (!cta_prologue<kSignaled>(sig)) {
    cta_abort<kSignaled>(sig);
    return;
  }
  const int tid = threadIdx.x;
  int c = blockIdx.x;
  uint4 rec = c < n_chunks ? __ldg(reinterpret_cast<const uint4 *>(chunks) + c) : make_uint4(0, 0, 0, 0);
  for (; c < n_chunks; c += gridDim.x) {
    const int cn = c + gridDim.x;
    const uint4 next = cn < n_chunks ? __ldg(reinterpret_cast<const uint4 *>(chunks) + cn) : rec;
    uint4 *a = reinterpret_cast<uint4 *>(bufs.p[rec.w & 0xffffu]) + rec.x;
    uint4 *b = reinterpret_cast<uint4 *>(bufs.p[rec.w >> 16]) + rec.y;
    const int len = (int)rec.z;
    for (int base = 0; base < len; base += kChunkVecs) {
      uint4 va[kUnroll], vb[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int i = base + u * kThreads + tid;
        if (i < len) {
          va[u] = ld_stream(a + i);
          if constexpr (OP != OP_COPY) vb[u] = ld_stream(b + i);
        }
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int i = base + u * kThreads + tid;
        if (i < len) {
          if constexpr (OP == OP_COPY) {
            st_stream(b + i, va[u]);
          } else {
            const uint4 o = VecOp<T, OP>::run(va[u], vb[u], wa, wb);
            if (sig.wmask & 1) st_stream(a + i, o);
            if (sig.wmask & 2) st_stream(b + i, o);
          }
        }
      }
    }
    rec = next;
  }
  cta_epilogue<kSignaled>(sig);
}

// ---------------------------------------------------------------------------
// TMA bulk-copy variant: a producer warp streams both sides of each chunk into
// shared memory with cp.async.bulk (mbarrier complete_tx), four consumer warps
// reduce in shared memory, and one consumer thread writes the result back to
// both owners with cp.async.bulk stores.  kStages chunk-sized stages keep
// ~kStages*32 KiB of loads in flight per CTA without register staging.

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
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
__device__ __forceinline__ void bulk_load(void *smem_dst, const void *gsrc, uint32_t bytes,
                                          uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_load_hint(void *smem_dst, const void *gsrc, uint32_t bytes,
                                               uint64_t *bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], "
      "%2, [%3], %4;" ::"r"(smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bulk_store_hint(void *gdst, const void *smem_src, uint32_t bytes,
                                                uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(
                   gdst),
               "r"(smem_u32(smem_src)), "r"(bytes), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void bulk_store(void *gdst, const void *smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"(smem_u32(smem_src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

constexpr int kBulkConsumers = 128;                 // 4 consumer warps
constexpr int kBulkThreads = kBulkConsumers + 32;   // + 1 producer warp

template <int kStages>
struct BulkSmem {
  uint4 a[kStages][kChunkVecs];
  uint4 b[kStages][kChunkVecs];
  uint64_t full[kStages];
  uint64_t empty[kStages];
};

template <typename T, int OP, int kStages, bool kSignaled>
__global__ void __launch_bounds__(kBulkThreads, 1)
plan_kernel_bulk(const Chunk *__restrict__ chunks, int n_chunks, BufTable bufs,
                 typename Acc<T>::type wa, typename Acc<T>::type wb, SignalArgs sig) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  auto &sm = *reinterpret_cast<BulkSmem<kStages> *>(smem_raw);
  if (!cta_prologue<kSignaled>(sig)) {
    cta_abort<kSignaled>(sig);
    return;
  }
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint4 *recs = reinterpret_cast<const uint4 *>(chunks);
  if (warp == kBulkConsumers / 32) {
    // ---- producer: one elected lane issues the bulk loads ----
    if ((tid & 31) == 0) {
      const uint64_t pol = sig.l2_hint ? policy_evict_first() : 0;
      int stage = 0;
      uint32_t phase = 0;
      for (int c = blockIdx.x; c < n_chunks; c += gridDim.x) {
        const uint4 rec = __ldg(recs + c);
        const uint32_t bytes = rec.z * 16u;
        mbar_wait(&sm.empty[stage], phase ^ 1u);
        const uint4 *ga = reinterpret_cast<const uint4 *>(bufs.p[rec.w & 0xffffu]) + rec.x;
        const uint4 *gb = reinterpret_cast<const uint4 *>(bufs.p[rec.w >> 16]) + rec.y;
        if constexpr (OP == OP_COPY) {
          mbar_expect_tx(&sm.full[stage], bytes);
          if (sig.l2_hint) bulk_load_hint(sm.a[stage], ga, bytes, &sm.full[stage], pol);
          else bulk_load(sm.a[stage], ga, bytes, &sm.full[stage]);
        } else {
          mbar_expect_tx(&sm.full[stage], 2u * bytes);
          if (sig.l2_hint) {
            bulk_load_hint(sm.a[stage], ga, bytes, &sm.full[stage], pol);
            bulk_load_hint(sm.b[stage], gb, bytes, &sm.full[stage], pol);
          } else {
            bulk_load(sm.a[stage], ga, bytes, &sm.full[stage]);
            bulk_load(sm.b[stage], gb, bytes, &sm.full[stage]);
          }
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
    const uint4 rec = __ldg(recs + c);
    const int len = (int)rec.z;
    mbar_wait(&sm.full[stage], phase);
    if constexpr (OP != OP_COPY) {
      for (int i = tid; i < len; i += kBulkConsumers)
        sm.a[stage][i] = VecOp<T, OP>::run(sm.a[stage][i], sm.b[stage][i], wa, wb);
      fence_proxy_async_smem();
    }
    named_bar_sync(1, kBulkConsumers);
    if (tid == 0) {
      uint4 *ga = reinterpret_cast<uint4 *>(bufs.p[rec.w & 0xffffu]) + rec.x;
      uint4 *gb = reinterpret_cast<uint4 *>(bufs.p[rec.w >> 16]) + rec.y;
      if (sig.l2_hint == 2) {
        const uint64_t pol = policy_evict_first();
        if constexpr (OP != OP_COPY) {
          if (sig.wmask & 1) bulk_store_hint(ga, sm.a[stage], rec.z * 16u, pol);
          if (sig.wmask & 2) bulk_store_hint(gb, sm.a[stage], rec.z * 16u, pol);
        } else {
          bulk_store_hint(gb, sm.a[stage], rec.z * 16u, pol);
        }
      } else if constexpr (OP != OP_COPY) {
        if (sig.wmask & 1) bulk_store(ga, sm.a[stage], rec.z * 16u);
        if (sig.wmask & 2) bulk_store(gb, sm.a[stage], rec.z * 16u);
      } else {
        bulk_store(gb, sm.a[stage], rec.z * 16u);
      }
      bulk_commit();
      // the previous stage's stores have finished reading shared memory
      bulk_wait_read<1>();
      if (prev_stage >= 0) mbar_arrive(&sm.empty[prev_stage]);
    }
    prev_stage = stage;
    if (++stage == kStages) { stage = 0; phase ^= 1u; }
  }
  if (tid == 0) {
    bulk_wait_all();  // this CTA's result stores are complete
    if constexpr (kSignaled) {
      // async-proxy (bulk) global writes -> generic release at system scope
      asm volatile("fence.proxy.async.global;" ::: "memory");
      fence_acq_rel_sys();
      const unsigned int done = atomicAdd(sig.counter, 1u);
      if (done == gridDim.x - 1) last_cta_finish(sig);
    }
  }
}

template <typename T, int OP, bool kSignaled>
__global__ void __launch_bounds__(kThreads)
plan_kernel_scalar(const Chunk *__restrict__ chunks, int n_chunks, BufTable bufs,
                   typename Acc<T>::type wa, typename Acc<T>::type wb, SignalArgs sig) {
  if (!cta_prologue<kSignaled>(sig)) {
    cta_abort<kSignaled>(sig);
    return;
  }
  for (int c = blockIdx.x; c < n_chunks; c += gridDim.x) {
    const uint4 rec = __ldg(reinterpret_cast<const uint4 *>(chunks) + c);
    T *a = reinterpret_cast<T *>(bufs.p[rec.w & 0xffffu]) + rec.x;
    T *b = reinterpret_cast<T *>(bufs.p[rec.w >> 16]) + rec.y;
    for (int i = threadIdx.x; i < (int)rec.z; i += kThreads) {
      if constexpr (OP == OP_COPY) {
        b[i] = a[i];
      } else {
        const T o = combine_scalar<T, OP>(a[i], b[i], wa, wb);
        if (sig.wmask & 1) a[i] = o;
        if (sig.wmask & 2) b[i] = o;
      }
    }
  }
  cta_epilogue<kSignaled>(sig);
}

// uniform_grad_sync over R local replicas (tpnumerics.py:263-286).  Weights
// travel by value in the launch (no device buffer, no per-call allocation).
struct RepWeights {
  double w[kMaxBufs];
};

template <typename T>
__device__ __forceinline__ typename Acc<T>::type uniform_elem(const BufTable &reps, int R, int op,
                                                              const RepWeights &w, int64_t e) {
  using A = typename Acc<T>::type;
  A acc;
  if (op == NTP_OP_MEAN) {  // true mean over all replicas (tpnumerics.py:280-283)
    acc = A(0);
    for (int r = 0; r < R; ++r) acc = add_rn(acc, A(reinterpret_cast<const T *>(reps.p[r])[e]));
    acc = acc / A(R);
  } else if (op == NTP_OP_SUM) {  // replica order (tpnumerics.py:276-279)
    acc = A(reinterpret_cast<const T *>(reps.p[0])[e]);
    for (int r = 1; r < R; ++r) acc = add_rn(acc, A(reinterpret_cast<const T *>(reps.p[r])[e]));
  } else {
    acc = mul_rn(A(w.w[0]), A(reinterpret_cast<const T *>(reps.p[0])[e]));
    for (int r = 1; r < R; ++r)
      acc = add_rn(acc, mul_rn(A(w.w[r]), A(reinterpret_cast<const T *>(reps.p[r])[e])));
  }
  return acc;
}

// 16-byte vectors when every replica base is 16-byte aligned: each thread
// reduces 16/sizeof(T) consecutive elements with 128-bit loads and stores
// (same per-element arithmetic and order as the scalar path); the tail and
// unaligned buffers take the scalar path.
template <typename T>
__global__ void __launch_bounds__(kThreads)
uniform_kernel(BufTable reps, int R, int64_t n, int op, RepWeights w, int64_t n_vec, BufTable dst,
               int n_dst) {
  using A = typename Acc<T>::type;
  constexpr int kPer = 16 / sizeof(T);
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  const int64_t tid = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  for (int64_t v = tid; v < n_vec; v += stride) {
    A acc[kPer];
    {
      const uint4 x = ld_stream(reinterpret_cast<const uint4 *>(reps.p[0]) + v);
      const T *xe = reinterpret_cast<const T *>(&x);
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        const A a = A(xe[j]);
        acc[j] = op == NTP_OP_WEIGHTED ? mul_rn(A(w.w[0]), a)
                 : op == NTP_OP_MEAN    ? add_rn(A(0), a)  // as the scalar path: 0 + a
                                        : a;
      }
    }
    for (int r = 1; r < R; ++r) {
      const uint4 x = ld_stream(reinterpret_cast<const uint4 *>(reps.p[r]) + v);
      const T *xe = reinterpret_cast<const T *>(&x);
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        const A a = A(xe[j]);
        acc[j] = add_rn(acc[j], op == NTP_OP_WEIGHTED ? mul_rn(A(w.w[r]), a) : a);
      }
    }
    uint4 o;
    T *oe = reinterpret_cast<T *>(&o);
#pragma unroll
    for (int j = 0; j < kPer; ++j) oe[j] = T(op == NTP_OP_MEAN ? acc[j] / A(R) : acc[j]);
    if (n_dst) {
      for (int d = 0; d < n_dst; ++d) st_stream(reinterpret_cast<uint4 *>(dst.p[d]) + v, o);
    } else {
      for (int r = 0; r < R; ++r) st_stream(reinterpret_cast<uint4 *>(reps.p[r]) + v, o);
    }
  }
  for (int64_t e = n_vec * kPer + tid; e < n; e += stride) {
    const T o = T(uniform_elem<T>(reps, R, op, w, e));
    if (n_dst) {
      for (int d = 0; d < n_dst; ++d) reinterpret_cast<T *>(dst.p[d])[e] = o;
    } else {
      for (int r = 0; r < R; ++r) reinterpret_cast<T *>(reps.p[r])[e] = o;
    }
  }
}

__global__ void signal_post_kernel(SignalArgs sig) {
  const uint64_t e = sig_epoch(sig);
  release_words(sig.post, sig.n_post, e);
  sig_advance(sig, e);
}

__global__ void signal_wait_kernel(SignalArgs sig) {
  const uint64_t e = sig_epoch(sig);
  wait_signals(sig.wait, sig.n_wait, e, sig.spin_ns, sig.status);
  sig_advance(sig, e);
}

// a step with nothing to compute: post ready, wait ready, post done, wait done
__global__ void signal_step_kernel(SignalArgs sig) {
  const uint64_t e = sig_epoch(sig);
  post_signals(sig.pre, sig.n_pre, e);
  if (wait_signals(sig.wait, sig.n_wait, e, sig.spin_ns, sig.status)) {
    post_signals(sig.post, sig.n_post, e);
    wait_signals(sig.fin, sig.n_fin, e, sig.spin_ns, sig.status);
  }
  sig_advance(sig, e);
}

// ---------------------------------------------------------------------------
// launch helpers

static int sm_count(int device) {
  static std::mutex mu;
  static int cache[64] = {0};
  std::lock_guard<std::mutex> g(mu);
  if (device < 0 || device >= 64) return 148;
  if (!cache[device]) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || n <= 0)
      n = 148;
    cache[device] = n;
  }
  return cache[device];
}

template <typename K>
static int grid_for(K kernel, int device, int n_items) {
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kThreads, 0) != cudaSuccess ||
      occ <= 0)
    occ = 4;
  int g = sm_count(device) * occ;
  const int cap = g_max_ctas.load();
  if (cap > 0 && g > cap) g = cap;
  return n_items < g ? (n_items > 0 ? n_items : 1) : g;
}

static std::atomic<int> g_sync_kernel{NTP_KERNEL_AUTO};

template <typename T, int OP, int kStages, bool kSig>
static int launch_bulk(const ntp_plan *p, const BufTable &bt, typename Acc<T>::type wa,
                       typename Acc<T>::type wb, int ctas_per_sm, const SignalArgs &sig,
                       cudaStream_t s) {
  auto k = plan_kernel_bulk<T, OP, kStages, kSig>;
  const int smem = (int)sizeof(BulkSmem<kStages>);
  static std::once_flag once[64];
  const int dev = p->device >= 0 && p->device < 64 ? p->device : 0;
  std::call_once(once[dev], [&] {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  });
  const int n = (int)p->chunks.size();
  int grid = sm_count(p->device) * ctas_per_sm;
  const int cap = g_max_ctas.load();
  if (cap > 0 && grid > cap) grid = cap;
  if (n < grid) grid = n > 0 ? n : 1;
  SignalArgs sg = sig;
  sg.l2_hint = g_l2_hint.load();
  k<<<grid, kBulkThreads, smem, s>>>(p->d_chunks, n, bt, wa, wb, sg);
  return NTP_OK;
}

template <typename T, int OP, bool kSig>
static int launch_plan_t(const ntp_plan *p, const BufTable &bt, double wa, double wb,
                         const SignalArgs &sig, cudaStream_t s) {
  using A = typename Acc<T>::type;
  const int n = (int)p->chunks.size();
  int variant = g_sync_kernel.load();
  if (variant == NTP_KERNEL_AUTO)  // small plans are latency-bound: no smem pipeline fill
    variant = n < 4 * sm_count(p->device) ? NTP_KERNEL_LDG : NTP_KERNEL_BULK;
  if (p->vectorized && (variant == NTP_KERNEL_BULK || variant == NTP_KERNEL_BULK2)) {
    if (variant == NTP_KERNEL_BULK)
      return launch_bulk<T, OP, 4, kSig>(p, bt, A(wa), A(wb), 1, sig, s);
    return launch_bulk<T, OP, 3, kSig>(p, bt, A(wa), A(wb), 2, sig, s);
  }
  if (p->vectorized) {
    auto k = plan_kernel_vec<T, OP, kSig>;
    k<<<grid_for(k, p->device, n), kThreads, 0, s>>>(p->d_chunks, n, bt, A(wa), A(wb), sig);
  } else {
    auto k = plan_kernel_scalar<T, OP, kSig>;
    k<<<grid_for(k, p->device, n), kThreads, 0, s>>>(p->d_chunks, n, bt, A(wa), A(wb), sig);
  }
  return NTP_OK;
}

template <typename T, bool kSig>
static int launch_plan_op(const ntp_plan *p, int op, const BufTable &bt, double wa, double wb,
                          const SignalArgs &sig, cudaStream_t s) {
  switch (op) {
    case NTP_OP_SUM: return launch_plan_t<T, NTP_OP_SUM, kSig>(p, bt, wa, wb, sig, s);
    case NTP_OP_MEAN: return launch_plan_t<T, NTP_OP_MEAN, kSig>(p, bt, wa, wb, sig, s);
    case NTP_OP_WEIGHTED: return launch_plan_t<T, NTP_OP_WEIGHTED, kSig>(p, bt, wa, wb, sig, s);
    case OP_COPY: return launch_plan_t<T, OP_COPY, kSig>(p, bt, wa, wb, sig, s);
    default: return fail(NTP_EINVAL, "unknown reduction op");
  }
}

template <bool kSig>
static int launch_plan(const ntp_plan *p, int op, const BufTable &bt, double wa, double wb,
                       const SignalArgs &sig, cudaStream_t s) {
  switch (p->dtype) {
    case NTP_F32: return launch_plan_op<float, kSig>(p, op, bt, wa, wb, sig, s);
    case NTP_BF16: return launch_plan_op<__nv_bfloat16, kSig>(p, op, bt, wa, wb, sig, s);
    case NTP_F16: return launch_plan_op<__half, kSig>(p, op, bt, wa, wb, sig, s);
    case NTP_F64: return launch_plan_op<double, kSig>(p, op, bt, wa, wb, sig, s);
    default: return fail(NTP_EINVAL, "unsupported dtype");
  }
}

static int check_exec(const ntp_plan *p, void *const *bufs, int n_bufs, BufTable &bt) {
  if (!p) return fail(NTP_EINVAL, "null plan");
  if (!p->finalized) return fail(NTP_ESTATE, "plan not finalized");
  if (p->device < 0 || (!p->d_chunks && !p->chunks.empty()))
    return fail(NTP_ESTATE, "plan not uploaded to a device");
  if (n_bufs <= p->max_buf || n_bufs > kMaxBufs)
    return fail(NTP_EINVAL, "plan references more buffers than were passed");
  for (int i = 0; i < kMaxBufs; ++i) bt.p[i] = nullptr;
  for (int i = 0; i < n_bufs; ++i) {
    bt.p[i] = static_cast<char *>(bufs[i]);
    if (i <= p->max_buf && !bt.p[i]) return fail(NTP_EINVAL, "null buffer pointer");
    if (p->vectorized && (reinterpret_cast<uintptr_t>(bt.p[i]) & 15u))
      return fail(NTP_EINVAL, "buffer not 16-byte aligned for a vectorized plan");
  }
  return NTP_OK;
}

static int set_device(int device) {
  int cur = -1;
  NTP_CUDA(cudaGetDevice(&cur));
  if (cur != device) NTP_CUDA(cudaSetDevice(device));
  return NTP_OK;
}

// Launches with no plan (handshake kernels) go to the stream's own device,
// whatever the caller's current device is.
static int set_device_of(cudaStream_t s) {
  if (!s) return NTP_OK;  // legacy default stream: the current device's
  // cudaStreamGetDevice is not permitted on a capturing stream; a capture
  // records the launch onto the stream's own graph whatever the current device
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  NTP_CUDA(cudaStreamIsCapturing(s, &cs));
  if (cs != cudaStreamCaptureStatusNone) return NTP_OK;
  int dev = -1;
  NTP_CUDA(cudaStreamGetDevice(s, &dev));
  return set_device(dev);
}

}  // namespace ntp

using namespace ntp;

extern "C" {

int ntp_set_option(int option, int64_t value) {
  if (option == NTP_OPT_SYNC_L2) {
    if (value < 0 || value > 2) return fail(NTP_EINVAL, "L2 hint must be 0, 1 or 2");
    g_l2_hint.store((int)value);
    return NTP_OK;
  }
  if (option == NTP_OPT_PLAN_MIN_CHUNKS) {
    if (value < 0 || value > 1 << 24) return fail(NTP_EINVAL, "bad minimum chunk count");
    g_min_chunks.store(value);
    return NTP_OK;
  }
  if (option == NTP_OPT_SYNC_MAX_CTAS) {
    if (value < 0 || value > 1 << 20) return fail(NTP_EINVAL, "bad CTA cap");
    g_max_ctas.store((int)value);
    return NTP_OK;
  }
  if (option != NTP_OPT_SYNC_KERNEL) return fail(NTP_EINVAL, "unknown option");
  if (value < NTP_KERNEL_AUTO || value > NTP_KERNEL_BULK2)
    return fail(NTP_EINVAL, "unknown sync kernel variant");
  g_sync_kernel.store((int)value);
  return NTP_OK;
}

int64_t ntp_get_option(int option) {
  if (option == NTP_OPT_SYNC_L2) return g_l2_hint.load();
  if (option == NTP_OPT_PLAN_MIN_CHUNKS) return g_min_chunks.load();
  if (option == NTP_OPT_SYNC_MAX_CTAS) return g_max_ctas.load();
  if (option != NTP_OPT_SYNC_KERNEL) return fail(NTP_EINVAL, "unknown option");
  return g_sync_kernel.load();
}

int ntp_plan_upload(ntp_plan *p, int device) {
  if (!p) return fail(NTP_EINVAL, "null plan");
  if (!p->finalized) return fail(NTP_ESTATE, "plan not finalized");
  int st = set_device(device);
  if (st) return st;
  if (p->d_chunks) {
    device_free(p->d_chunks, p->device);
    p->d_chunks = nullptr;
  }
  if (p->d_counter) {
    device_free(p->d_counter, p->device);
    p->d_counter = nullptr;
  }
  p->device = device;
  NTP_CUDA(cudaMalloc(&p->d_counter, 256));
  NTP_CUDA(cudaMemset(p->d_counter, 0, 256));
  if (p->chunks.empty()) return NTP_OK;
  const size_t bytes = p->chunks.size() * sizeof(Chunk);
  NTP_CUDA(cudaMalloc(&p->d_chunks, bytes));
  NTP_CUDA(cudaMemcpy(p->d_chunks, p->chunks.data(), bytes, cudaMemcpyHostToDevice));
  return NTP_OK;
}

int ntp_grad_sync(const ntp_plan *p, void *const *bufs, int n_bufs, int op, double w_a,
                  double w_b, void *stream) {
  BufTable bt;
  int st = check_exec(p, bufs, n_bufs, bt);
  if (st) return st;
  if (op < NTP_OP_SUM || op > NTP_OP_WEIGHTED) {
    char buf[64];
    snprintf(buf, sizeof buf, "unknown reduction op %d", op);
    return fail(NTP_EINVAL, buf);
  }
  if (p->chunks.empty()) return NTP_OK;
  if ((st = set_device(p->device))) return st;
  SignalArgs sig{};
  st = launch_plan<false>(p, op, bt, w_a, w_b, sig, static_cast<cudaStream_t>(stream));
  if (st) return st;
  NTP_CUDA(cudaGetLastError());
  return NTP_OK;
}

int ntp_grad_sync_ex(const ntp_plan *p, void *const *bufs, int n_bufs, int op, double w_a,
                     double w_b, int write_mask, void *stream) {
  BufTable bt;
  int st = check_exec(p, bufs, n_bufs, bt);
  if (st) return st;
  if (op < NTP_OP_SUM || op > NTP_OP_WEIGHTED) return fail(NTP_EINVAL, "unknown reduction op");
  if (write_mask < 1 || write_mask > 3) return fail(NTP_EINVAL, "write_mask must be 1, 2 or 3");
  if (p->chunks.empty()) return NTP_OK;
  if ((st = set_device(p->device))) return st;
  SignalArgs sig{};
  sig.wmask = write_mask;
  st = launch_plan<false>(p, op, bt, w_a, w_b, sig, static_cast<cudaStream_t>(stream));
  if (st) return st;
  NTP_CUDA(cudaGetLastError());
  return NTP_OK;
}

int ntp_reshard(const ntp_plan *p, void *const *bufs, int n_bufs, void *stream) {
  BufTable bt;
  int st = check_exec(p, bufs, n_bufs, bt);
  if (st) return st;
  if (p->chunks.empty()) return NTP_OK;
  if ((st = set_device(p->device))) return st;
  SignalArgs sig{};
  st = launch_plan<false>(p, OP_COPY, bt, 0.0, 0.0, sig, static_cast<cudaStream_t>(stream));
  if (st) return st;
  NTP_CUDA(cudaGetLastError());
  return NTP_OK;
}

static int uniform_reduce(void *const *reps, int R, int64_t n, int dtype, int op,
                          const double *w, void *const *dsts, int n_dst, void *stream) {
  if (R < 1 || R > kMaxBufs) return fail(NTP_EINVAL, "replica count must be in [1, 64]");
  if (n_dst < 0 || n_dst > kMaxBufs) return fail(NTP_EINVAL, "destination count must be in [0, 64]");
  if (op < NTP_OP_SUM || op > NTP_OP_WEIGHTED) return fail(NTP_EINVAL, "unknown reduction op");
  if (n <= 0) return NTP_OK;
  cudaPointerAttributes attr{};
  NTP_CUDA(cudaPointerGetAttributes(&attr, reps[0]));
  int st = set_device(attr.device);
  if (st) return st;
  BufTable bt{}, dt{};
  bool aligned = true;
  for (int d = 0; d < n_dst; ++d) {
    if (!dsts[d]) return fail(NTP_EINVAL, "null destination");
    dt.p[d] = static_cast<char *>(dsts[d]);
    aligned &= (reinterpret_cast<uintptr_t>(dsts[d]) & 15u) == 0;
  }
  for (int r = 0; r < R; ++r) {
    bt.p[r] = static_cast<char *>(reps[r]);
    aligned &= (reinterpret_cast<uintptr_t>(reps[r]) & 15u) == 0;
  }
  RepWeights wv{};
  if (op == NTP_OP_WEIGHTED) {
    if (!w) return fail(NTP_EINVAL, "weighted op needs one weight per replica");
    for (int r = 0; r < R; ++r) wv.w[r] = w[r];
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int esize = dtype == NTP_F64 ? 8 : dtype == NTP_F32 ? 4 : 2;
  const int64_t n_vec = aligned ? n * esize / 16 : 0;
  const int64_t work = n_vec + (n - n_vec * 16 / esize);
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((work + kThreads - 1) / kThreads,
                                                                 sm_count(attr.device) * 8));
  switch (dtype) {
    case NTP_F32: uniform_kernel<float><<<blocks, kThreads, 0, s>>>(bt, R, n, op, wv, n_vec, dt, n_dst); break;
    case NTP_BF16: uniform_kernel<__nv_bfloat16><<<blocks, kThreads, 0, s>>>(bt, R, n, op, wv, n_vec, dt, n_dst); break;
    case NTP_F16: uniform_kernel<__half><<<blocks, kThreads, 0, s>>>(bt, R, n, op, wv, n_vec, dt, n_dst); break;
    case NTP_F64: uniform_kernel<double><<<blocks, kThreads, 0, s>>>(bt, R, n, op, wv, n_vec, dt, n_dst); break;
    default: return fail(NTP_EINVAL, "unsupported dtype");
  }
  NTP_CUDA(cudaGetLastError());
  return NTP_OK;
}

int ntp_uniform_sync(void *const *reps, int R, int64_t n, int dtype, int op, const double *w,
                     void *stream) {
  return uniform_reduce(reps, R, n, dtype, op, w, nullptr, 0, stream);
}

int ntp_reduce_into(void *const *srcs, int R, int64_t n, int dtype, void *const *dsts, int n_dst,
                    void *stream) {
  if (n_dst < 1) return fail(NTP_EINVAL, "at least one destination is required");
  return uniform_reduce(srcs, R, n, dtype, NTP_OP_SUM, nullptr, dsts, n_dst, stream);
}

// --------------------------------------------------------------------------
// multi-GPU plumbing

int ntp_alloc(int device, int64_t bytes, void **out) {
  if (!out || bytes <= 0) return fail(NTP_EINVAL, "bad allocation request");
  int st = set_device(device);
  if (st) return st;
  NTP_CUDA(cudaMalloc(out, (size_t)bytes));
  NTP_CUDA(cudaMemset(*out, 0, (size_t)bytes));
  return NTP_OK;
}

int ntp_free(void *ptr) {
  if (!ptr) return NTP_OK;
  cudaPointerAttributes attr{};
  NTP_CUDA(cudaPointerGetAttributes(&attr, ptr));
  int st = set_device(attr.device);
  if (st) return st;
  NTP_CUDA(cudaFree(ptr));
  return NTP_OK;
}

int ntp_ipc_get_handle(void *dev_ptr, void *handle_out) {
  static_assert(sizeof(cudaIpcMemHandle_t) == NTP_IPC_HANDLE_BYTES, "ipc handle size");
  cudaPointerAttributes attr{};
  NTP_CUDA(cudaPointerGetAttributes(&attr, dev_ptr));
  int st = set_device(attr.device);
  if (st) return st;
  cudaIpcMemHandle_t h;
  NTP_CUDA(cudaIpcGetMemHandle(&h, dev_ptr));
  memcpy(handle_out, &h, sizeof h);
  return NTP_OK;
}

int ntp_ipc_open(int device, const void *handle, void **dev_ptr_out) {
  int st = set_device(device);
  if (st) return st;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof h);
  NTP_CUDA(cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess));
  return NTP_OK;
}

int ntp_ipc_close(void *dev_ptr) {
  NTP_CUDA(cudaIpcCloseMemHandle(dev_ptr));
  return NTP_OK;
}

static int fill_signals(SignalArgs &sig, uint64_t *const *wait, int n_wait, uint64_t *const *post,
                        int n_post, uint64_t epoch, uint64_t spin_ns, int *status) {
  if (n_wait < 0 || n_wait > 16 || n_post < 0 || n_post > 16)
    return fail(NTP_EINVAL, "at most 16 wait and 16 post signals");
  sig = SignalArgs{};
  for (int i = 0; i < n_wait; ++i) sig.wait[i] = wait[i];
  for (int i = 0; i < n_post; ++i) sig.post[i] = post[i];
  sig.n_wait = n_wait;
  sig.n_post = n_post;
  sig.epoch = epoch;
  sig.spin_ns = spin_ns;
  sig.status = status;
  return NTP_OK;
}

static int grad_sync_signaled(const ntp_plan *p, void *const *bufs, int n_bufs, int op,
                              double w_a, double w_b, uint64_t *const *wait, int n_wait,
                              uint64_t *const *post, int n_post, uint64_t epoch,
                              uint64_t *epoch_word, uint64_t spin_ns, int *status, void *stream) {
  BufTable bt;
  int st = check_exec(p, bufs, n_bufs, bt);
  if (st) return st;
  if (op < NTP_OP_SUM || op > NTP_OP_WEIGHTED) return fail(NTP_EINVAL, "unknown reduction op");
  if ((st = set_device(p->device))) return st;
  SignalArgs sig;
  if ((st = fill_signals(sig, wait, n_wait, post, n_post, epoch, spin_ns, status))) return st;
  sig.counter = p->d_counter;
  sig.trace = g_trace;
  sig.epoch_word = epoch_word;  // never advanced here: the step's done-wait advances
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (p->chunks.empty()) {
    signal_wait_kernel<<<1, 1, 0, s>>>(sig);
    signal_post_kernel<<<1, 1, 0, s>>>(sig);
  } else {
    st = launch_plan<true>(p, op, bt, w_a, w_b, sig, s);
    if (st) return st;
  }
  NTP_CUDA(cudaGetLastError());
  return NTP_OK;
}

int ntp_grad_sync_signaled(const ntp_plan *p, void *const *bufs, int n_bufs, int op, double w_a,
                           double w_b, uint64_t *const *wait, int n_wait, uint64_t *const *post,
                           int n_post, uint64_t epoch, uint64_t spin_ns, int *status,
                           void *stream) {
  return grad_sync_signaled(p, bufs, n_bufs, op, w_a, w_b, wait, n_wait, post, n_post, epoch,
                            nullptr, spin_ns, status, stream);
}

int ntp_grad_sync_signaled_dev(const ntp_plan *p, void *const *bufs, int n_bufs, int op,
                               double w_a, double w_b, uint64_t *const *wait, int n_wait,
                               uint64_t *const *post, int n_post, uint64_t *epoch_word,
                               uint64_t spin_ns, int *status, void *stream) {
  if (!epoch_word) return fail(NTP_EINVAL, "epoch_word is required");
  return grad_sync_signaled(p, bufs, n_bufs, op, w_a, w_b, wait, n_wait, post, n_post, 0,
                            epoch_word, spin_ns, status, stream);
}

static int grad_sync_step(const ntp_plan *p, void *const *bufs, int n_bufs, int op, double w_a,
                          double w_b, uint64_t *const *post_ready, int n_post_ready,
                          uint64_t *const *wait_ready, int n_wait_ready,
                          uint64_t *const *post_done, int n_post_done,
                          uint64_t *const *wait_done, int n_wait_done, uint64_t epoch,
                          uint64_t *epoch_word, uint64_t spin_ns, int *status, void *stream) {
  if (n_post_ready < 0 || n_post_ready > 16 || n_wait_done < 0 || n_wait_done > 16)
    return fail(NTP_EINVAL, "at most 16 wait and 16 post signals");
  SignalArgs sig;
  int st = fill_signals(sig, wait_ready, n_wait_ready, post_done, n_post_done, epoch, spin_ns,
                        status);
  if (st) return st;
  for (int i = 0; i < n_post_ready; ++i) sig.pre[i] = post_ready[i];
  for (int i = 0; i < n_wait_done; ++i) sig.fin[i] = wait_done[i];
  sig.n_pre = n_post_ready;
  sig.n_fin = n_wait_done;
  sig.epoch_word = epoch_word;
  sig.advance = 1;  // one launch is the whole step
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (!p || p->chunks.empty()) {
    if ((st = p ? set_device(p->device) : set_device_of(s))) return st;
    signal_step_kernel<<<1, 1, 0, s>>>(sig);
    NTP_CUDA(cudaGetLastError());
    return NTP_OK;
  }
  BufTable bt;
  if ((st = check_exec(p, bufs, n_bufs, bt))) return st;
  if (op < NTP_OP_SUM || op > NTP_OP_WEIGHTED) return fail(NTP_EINVAL, "unknown reduction op");
  if ((st = set_device(p->device))) return st;
  sig.counter = p->d_counter;
  sig.trace = g_trace;
  if ((st = launch_plan<true>(p, op, bt, w_a, w_b, sig, s))) return st;
  NTP_CUDA(cudaGetLastError());
  return NTP_OK;
}

int ntp_grad_sync_step(const ntp_plan *p, void *const *bufs, int n_bufs, int op, double w_a,
                       double w_b, uint64_t *const *post_ready, int n_post_ready,
                       uint64_t *const *wait_ready, int n_wait_ready, uint64_t *const *post_done,
                       int n_post_done, uint64_t *const *wait_done, int n_wait_done,
                       uint64_t epoch, uint64_t spin_ns, int *status, void *stream) {
  return grad_sync_step(p, bufs, n_bufs, op, w_a, w_b, post_ready, n_post_ready, wait_ready,
                        n_wait_ready, post_done, n_post_done, wait_done, n_wait_done, epoch,
                        nullptr, spin_ns, status, stream);
}

int ntp_grad_sync_step_dev(const ntp_plan *p, void *const *bufs, int n_bufs, int op, double w_a,
                           double w_b, uint64_t *const *post_ready, int n_post_ready,
                           uint64_t *const *wait_ready, int n_wait_ready,
                           uint64_t *const *post_done, int n_post_done,
                           uint64_t *const *wait_done, int n_wait_done, uint64_t *epoch_word,
                           uint64_t spin_ns, int *status, void *stream) {
  if (!epoch_word) return fail(NTP_EINVAL, "epoch_word is required");
  return grad_sync_step(p, bufs, n_bufs, op, w_a, w_b, post_ready, n_post_ready, wait_ready,
                        n_wait_ready, post_done, n_post_done, wait_done, n_wait_done, 0,
                        epoch_word, spin_ns, status, stream);
}

static int signal_post(uint64_t *const *post, int n_post, uint64_t epoch, uint64_t *epoch_word,
                       void *stream) {
  SignalArgs sig;
  int st = fill_signals(sig, nullptr, 0, post, n_post, epoch, 0, nullptr);
  if (st) return st;
  sig.epoch_word = epoch_word;
  if ((st = set_device_of(static_cast<cudaStream_t>(stream)))) return st;
  signal_post_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(sig);
  NTP_CUDA(cudaGetLastError());
  return NTP_OK;
}

static int signal_wait(uint64_t *const *wait, int n_wait, uint64_t epoch, uint64_t *epoch_word,
                       int advance, uint64_t spin_ns, int *status, void *stream) {
  SignalArgs sig;
  int st = fill_signals(sig, wait, n_wait, nullptr, 0, epoch, spin_ns, status);
  if (st) return st;
  sig.epoch_word = epoch_word;
  sig.advance = advance ? 1 : 0;
  if ((st = set_device_of(static_cast<cudaStream_t>(stream)))) return st;
  signal_wait_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(sig);
  NTP_CUDA(cudaGetLastError());
  return NTP_OK;
}

// Debug hook, not in the header: device buffer of >= 6 u64 that signalled
// sync launches stamp with globaltimer (nullptr: off).
int ntp_debug_sync_trace(void *buf) {
  g_trace = static_cast<uint64_t *>(buf);
  return NTP_OK;
}

int ntp_signal_post(uint64_t *const *post, int n_post, uint64_t epoch, void *stream) {
  return signal_post(post, n_post, epoch, nullptr, stream);
}

int ntp_signal_wait(uint64_t *const *wait, int n_wait, uint64_t epoch, uint64_t spin_ns,
                    int *status, void *stream) {
  return signal_wait(wait, n_wait, epoch, nullptr, 0, spin_ns, status, stream);
}

int ntp_signal_post_dev(uint64_t *const *post, int n_post, uint64_t *epoch_word, void *stream) {
  if (!epoch_word) return fail(NTP_EINVAL, "epoch_word is required");
  return signal_post(post, n_post, 0, epoch_word, stream);
}

int ntp_signal_wait_dev(uint64_t *const *wait, int n_wait, uint64_t *epoch_word, int advance,
                        uint64_t spin_ns, int *status, void *stream) {
  if (!epoch_word) return fail(NTP_EINVAL, "epoch_word is required");
  return signal_wait(wait, n_wait, 0, epoch_word, advance, spin_ns, status, stream);
}

}  // extern "C"
