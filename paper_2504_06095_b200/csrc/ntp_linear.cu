// Uneven-shard column/row-parallel linears on the 5th-gen tensor cores (sm_100a).
//
// The only dense contraction of the NTP path: per TP rank i with
// n_i ffn columns (n_i ragged: 4779, 1366, ... -- shardmap.py:160-165),
//   forward   H_i = X A_i,  Y_i = GeLU(H_i),  Z_i = Y_i B_i     (tpnumerics.py:177-185)
//   backward  dB_i = Y_i^T G,  D_i = (G B_i^T) * GeLU'(H_i),  dA_i = X^T D_i
//                                                              (tpnumerics.py:238-252)
// One kernel template computes C[M x N] = epilogue(sum_k A[m,k] B[n,k]) with
//   * operands staged by TMA (cp.async.bulk.tensor, 128B swizzle, OOB zero fill
//     for the ragged M/N/K tails) into a 4-stage shared-memory ring,
//   * tcgen05.mma (kind::f16, bf16 x bf16 -> fp32) issued by one thread, the
//     accumulator in TMEM,
//   * K-major or MN-major operands (the wgrad GEMMs contract over tokens, so
//     both of their operands are MN-major views of token-major activations),
//   * fused epilogues read back from TMEM with tcgen05.ld: GeLU (stores H and
//     Y), GeLU' multiply (backward), plain store -- and an arbitrary output row
//     stride, so the weight-gradient GEMMs write straight into the unit-major
//     gradient arena the sync kernel consumes (ldc = 2*hidden).
// Warp roles: warp 0 TMA producer, warp 1 TMEM allocator + MMA issuer,
// warps 2-5 epilogue (warp w reads TMEM lanes 32*(w%4)..+31).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <atomic>
#include <cstring>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "ntp_internal.h"

namespace ntp {
namespace gemm {

constexpr int BM = 128;
constexpr int BK = 64;          // 64 bf16 = 128 B: one swizzle-128B row
constexpr int kThreads = 192;   // 6 warps: TMA, MMA, 4 x epilogue

enum Epi { EPI_NONE = 0, EPI_GELU = 1, EPI_DGELU = 2, EPI_RED = 3, EPI_PUSH = 4 };

constexpr int kMaxPeers = 8;

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
__device__ __forceinline__ bool mbar_try(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Bounded wait: a pipeline bug traps (a CUDA error the host sees) after ~4 s
// instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  if (mbar_try(bar, parity)) return;
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (!mbar_try(bar, parity)) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 4000000000ull) asm volatile("trap;");
  }
}
// Long waits (the epilogue waiting a whole tile for its accumulator): poll
// with a short sleep so the spinning warps leave issue slots to the producer
// and MMA warps that share their SM sub-partitions.
__device__ __forceinline__ void mbar_wait_sleepy(uint64_t *bar, uint32_t parity) {
  if (mbar_try(bar, parity)) return;
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (!mbar_try(bar, parity)) {
    __nanosleep(64);
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 4000000000ull) asm volatile("trap;");
  }
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void tma_load_2d(void *smem_dst, const CUtensorMap *map, int c0, int c1,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t *bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Shared-memory matrix descriptor, SWIZZLE_128B (layout type 2), sm100 version 1.
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr & 0x3FFFFu) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (2ull << 61);
}

// tcgen05 instruction descriptor, kind::f16: bf16 A/B, fp32 D.
__host__ __device__ constexpr uint32_t instr_desc(int m, int n, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

// MUFU.TANH (max rel. error ~2^-11, below the bf16 output rounding of 2^-9)
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float gelu_f(float x) {
  // tanh GeLU, tpnumerics.py:25-28
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  return 0.5f * x * (1.0f + tanh_fast(k0 * (x + k1 * x * x * x)));
}
__device__ __forceinline__ float gelu_grad_f(float x) {
  // tpnumerics.py:31-36
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  const float t = tanh_fast(k0 * (x + k1 * x * x * x));
  const float du = k0 * (1.0f + 3.0f * k1 * x * x);
  return 0.5f * (1.0f + t) + 0.5f * x * (1.0f - t * t) * du;
}

struct Params {
  int M, N, K;
  int a_mn, b_mn;          // 1 = operand is MN-major in global memory
  int c_f32;               // 1: fp32 output, 0: bf16
  int epi;
  const __nv_bfloat16 *aux;  // EPI_DGELU: H (read directly)
  long long ld_aux;
  float alpha;
  int num_m, num_n;        // tile grid
  void *C, *H;             // outputs (H: EPI_GELU pre-activation)
  long long ldc, ldh;
  int c_tma, h_tma;        // 1: 16-byte aligned pitch -> TMA store; 0: warp copy
  // EPI_RED (fused wgrad + NTP sync): row m of the tile is added (red.add) to
  // the local C row and to row red_row[m] of peer copy red_buf[m] (-1: none)
  const int *red_buf;
  const int *red_row;
  char *red_base[kMaxPeers];
  long long red_ld;        // elements
  // split-K tail: tiles [0, full_items) run whole; each of the remaining tiles is
  // cut into `split` K ranges run by different CTA pairs, whose fp32 partials
  // meet in `ws`; the last arriving piece of each warp slice sums and stores
  int full_items, split;
  int *tile_cnt;
  float *ws;
  unsigned long long split_window_ns;  // how long a piece waits for the others
  // debug only (ntp_gemm_debug_trace): per (CTA, local item) 8 u64:
  // {item, t_full, t_done, t_kernel_start, t_prod_first, t_prod_last, t_mma_first, t_mma_last}
  unsigned long long *trace;
  // debug only (ntp_gemm_debug_counters): per leader CTA 4 u64 of clock64
  // cycles: {-, MMA waiting for full stages, MMA waiting for a free
  // accumulator, MMA loop total}
  unsigned long long *counters;
  // EPI_PUSH with push_tma = 1: a 32-row box whose rows map to consecutive rows
  // of one peer copy goes there as one TMA tensor store (peer_maps[pb]) from the
  // same smem staging as the local store; other boxes fall back to row stores
  int push_tma;
  // EPI_RED with tma_red = 1: the box is added into the local copy and the
  // partner's copy with TMA bulk tensor reductions (cp.reduce.async.bulk.tensor
  // .add) from the same smem staging -- no per-thread remote atomics
  int tma_red;
  // programmatic dependent launch: 0 off; 1 = wait for the previous kernel in
  // the stream before touching global memory (prologue overlaps its tail);
  // 2 = this GEMM's inputs and outputs are independent of the previous kernel
  // (runs under its tail), but the grid does not complete before it does
  int pdl;
  // tile order: tiles are walked in groups of `raster` M-tile rows (M fastest
  // inside a group); 0 = one group of all M rows
  int raster;
  int epi_sleep;  // 1: the epilogue polls its accumulator barrier with a sleep
  int debug;      // experiments: 1 = no operand loads, 2 = no epilogue output,
                  // 4 = MMA skips the full-stage waits, 8 = no stage commits (no producer)
  // TMA stores clip the inner dimension at 16-byte granularity, not per
  // element (found by tests/test_bounds_gpu.py: with N*esize % 16 != 0 a box
  // at the row end also wrote the bytes up to the next 16-byte boundary, i.e.
  // into the pitch gap -- in a unit-major arena, the next half-unit).  Boxes
  // that reach past tma_cols are stored element by element instead.
  int tma_cols;
};

// tile t -> (M-tile, N-tile) under the grouped raster order
__device__ __forceinline__ void tile_coords(int t, const Params &p, int &tm, int &tn) {
  const int G = (p.raster > 0 && p.raster < p.num_m) ? p.raster : p.num_m;
  const int span = G * p.num_n, g = t / span, w = t - g * span;
  const int gsz = min(G, p.num_m - g * G);
  tm = g * G + w % gsz;
  tn = w / gsz;
}

// Tensor maps over the peer copies (EPI_PUSH, push_tma): boxes of 32 x 32 at
// the GEMM output's element type, row pitch red_ld.
struct PeerMaps {
  CUtensorMap m[kMaxPeers];
};

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
constexpr int kTraceItems = 16;

struct Work {
  int t, kb_lo, kb_hi, tail, piece;
};

__device__ __forceinline__ Work decode_work(int item, const Params &p, int nk) {
  if (item < p.full_items) return Work{item, 0, nk, -1, 0};
  const int j = item - p.full_items, tail = j / p.split, piece = j % p.split;
  return Work{p.full_items + tail, nk * piece / p.split, nk * (piece + 1) / p.split, tail, piece};
}

// 16-byte stores of 32 consecutive values (fp32 or bf16 destination, aligned)
__device__ __forceinline__ void store_row32(void *dst, const float *f, int c_f32) {
  if (c_f32) {
    float4 *d = reinterpret_cast<float4 *>(dst);
#pragma unroll
    for (int j = 0; j < 32; j += 4) d[j / 4] = make_float4(f[j], f[j + 1], f[j + 2], f[j + 3]);
  } else {
    uint4 *d = reinterpret_cast<uint4 *>(dst);
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
      uint32_t w[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        __nv_bfloat162 t = __floats2bfloat162_rn(f[j + 2 * e], f[j + 2 * e + 1]);
        w[e] = *reinterpret_cast<uint32_t *>(&t);
      }
      d[j / 8] = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}

// red.add of 32 consecutive values (fp32 or bf16 destination, 16-byte aligned)
__device__ __forceinline__ void red_row32(void *dst, const float *f, int c_f32) {
  if (c_f32) {
    float *d = reinterpret_cast<float *>(dst);
#pragma unroll
    for (int j = 0; j < 32; j += 4)
      asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(d + j), "f"(f[j]),
                   "f"(f[j + 1]), "f"(f[j + 2]), "f"(f[j + 3])
                   : "memory");
  } else {
    __nv_bfloat16 *d = reinterpret_cast<__nv_bfloat16 *>(dst);
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
      uint32_t w[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        __nv_bfloat162 t = __floats2bfloat162_rn(f[j + 2 * e], f[j + 2 * e + 1]);
        w[e] = *reinterpret_cast<uint32_t *>(&t);
      }
      asm volatile("red.global.add.noftz.v4.bf16x2 [%0], {%1, %2, %3, %4};" ::"l"(d + j),
                   "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3])
                   : "memory");
    }
  }
}

// Staged 32 x 32 output boxes are swizzled like the TMA maps that store them
// (fp32: 128-byte rows, SWIZZLE_128B; bf16: 64-byte rows, SWIZZLE_64B): the
// 16-byte chunk c of row r sits at chunk c ^ swz(r), so the 32 lanes of a warp
// (one row each) write conflict-free instead of all hitting the same banks.
__device__ __forceinline__ int stage_swz(int r, int esize) {
  return esize == 4 ? (r & 7) : ((r >> 1) & 3);
}

// Copy a staged 32 x 32 box to global with row/column masking (pitches a TMA
// map cannot describe).  esize = 2 (bf16) or 4 (fp32).
__device__ __forceinline__ void box_store(const unsigned char *stage, void *g, long long ld,
                                          int esize, int row0, int col0, int M, int N, int lane) {
  const int col = col0 + lane;
  if (col >= N) return;
  const int b = lane * esize, rp = 32 * esize;
  for (int r = 0; r < 32; ++r) {
    const int row = row0 + r;
    if (row >= M) break;
    const unsigned char *src = stage + r * rp + ((((b >> 4) ^ stage_swz(r, esize)) << 4) | (b & 15));
    if (esize == 4)
      reinterpret_cast<float *>(g)[(long long)row * ld + col] = *reinterpret_cast<const float *>(src);
    else
      reinterpret_cast<__nv_bfloat16 *>(g)[(long long)row * ld + col] =
          *reinterpret_cast<const __nv_bfloat16 *>(src);
  }
}

// Output staging per epilogue warp: a 32 x 32 box (bf16 C [+ bf16 H], or fp32 C).
constexpr int kStageBytes = 32 * 32 * 4;

template <int BN, int kPair, int kStg>
struct Smem {
  alignas(1024) __nv_bfloat16 a[kStg][BM * BK];
  alignas(1024) __nv_bfloat16 b[kStg][(BN / kPair) * BK];
  alignas(1024) unsigned char out[4][2][kStageBytes];  // double-buffered per epilogue warp (swizzled)
  uint64_t full[kStg];
  uint64_t empty[kStg];
  uint64_t tmem_full[2];
  uint64_t tmem_empty[2];
  uint32_t tmem_base;
};

__device__ __forceinline__ void tma_store_2d(const CUtensorMap *map, const void *smem_src, int c0,
                                             int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(smem_u32(smem_src))
               : "memory");
}
__device__ __forceinline__ void tma_reduce_add_2d(const CUtensorMap *map, const void *smem_src,
                                                  int c0, int c1) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(c0), "r"(c1), "r"(smem_u32(smem_src))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
// arrive on the barrier at the same smem offset in cluster CTA `rank`
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t *bar, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote)
               : "memory");
}
// 2-SM TMA load: bytes land in this CTA's smem, completion is counted on the
// leader CTA's barrier (peer bit cleared), as CUTLASS's SM100_TMA_2SM_LOAD.
__device__ __forceinline__ void tma_load_2d_pair(void *smem_dst, const CUtensorMap *map, int c0,
                                                 int c1, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar) & 0xFEFFFFFFu)
      : "memory");
}
__device__ __forceinline__ void tc_mma2(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                        uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_commit2(uint64_t *bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}

// Persistent, warp-specialized: warp 0 streams operand tiles (TMA) through a
// kStg ring, warp 1 issues tcgen05.mma into one of two TMEM accumulators
// (2 x BN columns), warps 2-5 drain the other accumulator (tcgen05.ld ->
// fused epilogue -> smem -> TMA store) so the epilogue of tile i overlaps the
// MMAs of tile i+1.  kPair = 2: a CTA pair (cluster of 2) computes a 256 x BN
// tile with tcgen05.mma.cta_group::2 -- each CTA stages its 128 rows of A and
// half of B, the leader issues the MMAs, both drain their own TMEM half.
// kEpi: the fused epilogue, one instantiation each (see launch()).
// TMEM allocations are a power of two columns (>= 32): the two BN-column
// accumulators of a 224-wide tile take 512.
__host__ __device__ constexpr uint32_t tmem_cols(int bn) {
  return 2 * bn <= 32 ? 32u : 2 * bn <= 64 ? 64u : 2 * bn <= 128 ? 128u : 2 * bn <= 256 ? 256u : 512u;
}

template <int BN, int kPair, int kStg, int kEpi>
__global__ void __launch_bounds__(kThreads, 1)
gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
            const __grid_constant__ CUtensorMap map_c, const __grid_constant__ CUtensorMap map_h,
            const __grid_constant__ PeerMaps peer_maps, Params p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t base = smem_u32(smem_raw);
  unsigned char *aligned = smem_raw + ((1024u - (base & 1023u)) & 1023u);
  Smem<BN, kPair, kStg> &sm = *reinterpret_cast<Smem<BN, kPair, kStg> *>(aligned);
  constexpr int BNC = BN / kPair;  // B rows staged by this CTA
  constexpr int TM = BM * kPair;   // tile rows of the pair

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nk = (p.K + BK - 1) / BK;
  const int num_tiles = p.num_m * p.num_n;
  const int num_items = p.full_items + (num_tiles - p.full_items) * p.split;
  const uint32_t rank = kPair == 2 ? cluster_rank() : 0u;
  const bool leader = rank == 0;
  const int unit_id = blockIdx.x / kPair, num_units = gridDim.x / kPair;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStg; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&sm.tmem_full[a], 1);
      mbar_init(&sm.tmem_empty[a], 4 * kPair);  // one arrive per epilogue warp of the pair
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {  // TMEM: two BN-column fp32 accumulators x 128 lanes
    if constexpr (kPair == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(&sm.tmem_base)),
                   "r"(tmem_cols(BN)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(&sm.tmem_base)),
                   "r"(tmem_cols(BN)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  if constexpr (kPair == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  if (p.pdl) {
    // every CTA is resident (persistent grid): the next kernel may launch now
    // and set up under this one's tail
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (p.pdl == 1) asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  if (p.trace && threadIdx.x == 0) p.trace[(size_t)blockIdx.x * kTraceItems * 8 + 3] = gtime();

  if (warp == 0) {
    {
      // ---- TMA producer (both CTAs of a pair) ----
      // The whole warp walks the schedule (warp-uniform values stay in uniform
      // registers, which the TMA instructions take) and one elected lane issues.
      const uint32_t cta_bytes = (BM + BNC) * BK * 2;
      int it = 0, plocal = 0;
      for (int item = unit_id; item < num_items && !(p.debug & 8); item += num_units, ++plocal) {
        const Work w = decode_work(item, p, nk);
        const int t = w.t;
        int tm, tn;
        tile_coords(t, p, tm, tn);
        const int m0 = tm * TM + (int)rank * BM;
        const int n0 = tn * BN + (int)rank * BNC;
        unsigned long long *trp =
            p.trace && lane == 0 && plocal < kTraceItems ? p.trace + ((size_t)blockIdx.x * kTraceItems + plocal) * 8 : nullptr;
        for (int kb = w.kb_lo; kb < w.kb_hi; ++kb, ++it) {
          const int s = it % kStg;
          mbar_wait(&sm.empty[s], ((it / kStg) & 1) ^ 1);
          if (trp && kb == w.kb_lo) trp[4] = gtime();
          if (trp && kb == w.kb_hi - 1) trp[5] = gtime();
          if (p.debug & 1) {  // debug: no operand loads (MMA ceiling on stale smem)
            if (leader && lane == 0) mbar_arrive(&sm.full[s]);
            __syncwarp();
            continue;
          }
          if (elect_one()) {
            if (leader) mbar_expect_tx(&sm.full[s], cta_bytes * kPair);
            const int k0 = kb * BK;
            auto load = [&](void *dst, const CUtensorMap *m, int c0, int c1) {
              if constexpr (kPair == 2) tma_load_2d_pair(dst, m, c0, c1, &sm.full[s]);
              else tma_load_2d(dst, m, c0, c1, &sm.full[s]);
            };
            if (!p.a_mn) {
              load(sm.a[s], &map_a, k0, m0);
            } else {
#pragma unroll
              for (int j = 0; j < BM / 64; ++j) load(sm.a[s] + j * 64 * BK, &map_a, m0 + 64 * j, k0);
            }
            if (!p.b_mn) {
              load(sm.b[s], &map_b, k0, n0);
            } else {
#pragma unroll
              for (int j = 0; j < BNC / 64; ++j) load(sm.b[s] + j * 64 * BK, &map_b, n0 + 64 * j, k0);
            }
          }
          __syncwarp();
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // ---- MMA issuer (the leader CTA of a pair) ----
      // The whole warp walks the schedule (every value below is warp-uniform,
      // so the descriptors live in uniform registers) and one elected lane
      // issues the MMAs and commits -- no per-MMA uniform-register waterfall.
      const uint32_t idesc = instr_desc(TM, BN, p.a_mn, p.b_mn);
      // K-major: rows of 128 B, 8-row atoms 1024 B apart (SBO); K advance +32 B per k16.
      // MN-major: 64-element MN blocks of BK rows (LBO = BK*128 B), 8-row K groups
      // 1024 B apart (SBO); K advance +2048 B per k16.
      const uint32_t a_lbo = p.a_mn ? BK * 128 : 16, b_lbo = p.b_mn ? BK * 128 : 16;
      const uint32_t k_step_a = p.a_mn ? 2048u : 32u, k_step_b = p.b_mn ? 2048u : 32u;
      const uint64_t ad0 = smem_desc(smem_u32(sm.a[0]), a_lbo, 1024);
      const uint64_t bd0 = smem_desc(smem_u32(sm.b[0]), b_lbo, 1024);
      constexpr uint32_t a_stage16 = (BM * BK * 2) >> 4, b_stage16 = (BNC * BK * 2) >> 4;
      int it = 0, local = 0;
      long long cnt_full = 0, cnt_acc = 0;
      const long long c_start = p.counters ? clock64() : 0;
      for (int item = unit_id; item < num_items; item += num_units, ++local) {
        const Work w = decode_work(item, p, nk);
        const int acc = local & 1;
        if (p.counters) {
          const long long c0 = clock64();
          mbar_wait(&sm.tmem_empty[acc], ((local >> 1) & 1) ^ 1);
          cnt_acc += clock64() - c0;
        } else {
          mbar_wait(&sm.tmem_empty[acc], ((local >> 1) & 1) ^ 1);
        }
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(acc * BN);
        unsigned long long *trp =
            p.trace && lane == 0 && local < kTraceItems ? p.trace + ((size_t)blockIdx.x * kTraceItems + local) * 8 : nullptr;
        for (int kb = w.kb_lo; kb < w.kb_hi; ++kb, ++it) {
          const int s = it % kStg;
          if (p.counters) {
            const long long c0 = clock64();
            mbar_wait(&sm.full[s], (it / kStg) & 1);
            cnt_full += clock64() - c0;
          } else if (!(p.debug & 4)) {
            mbar_wait(&sm.full[s], (it / kStg) & 1);
          }
          if (trp && kb == w.kb_lo) trp[6] = gtime();
          if (trp && kb == w.kb_hi - 1) trp[7] = gtime();
          tc_fence_after();
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              // descriptors advance in 16-byte units in their low field
              const uint64_t ad = ad0 + (uint64_t)(s * a_stage16 + ((kk * k_step_a) >> 4));
              const uint64_t bd = bd0 + (uint64_t)(s * b_stage16 + ((kk * k_step_b) >> 4));
              const uint32_t accum = (kb > w.kb_lo || kk) ? 1u : 0u;
              if constexpr (kPair == 2) tc_mma2(d, ad, bd, idesc, accum);
              else tc_mma(d, ad, bd, idesc, accum);
            }
            // frees the stage (in both CTAs) once these MMAs have read it
            if (!(p.debug & 8)) {
              if constexpr (kPair == 2) tc_commit2(&sm.empty[s], 0x3); else tc_commit(&sm.empty[s]);
            }
          }
          __syncwarp();
        }
        if (elect_one()) {
          if constexpr (kPair == 2) tc_commit2(&sm.tmem_full[acc], 0x3); else tc_commit(&sm.tmem_full[acc]);
        }
        __syncwarp();
      }
      if (p.counters && lane == 0) {
        unsigned long long *c = p.counters + (size_t)blockIdx.x * 4;
        c[1] = (unsigned long long)cnt_full;
        c[2] = (unsigned long long)cnt_acc;
        c[3] = (unsigned long long)(clock64() - c_start);
      }
    }
  } else {
    // ---- epilogue: TMEM -> registers -> fused op -> smem -> TMA store ----
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    int sbuf = 0;
    int local = 0;
    // one 32-column chunk of this warp's 32-row slice: raw fp32 sums -> fused
    // epilogue -> global (TMA store, warp copy, or fused-sync stores)
    auto emit = [&](const int n0, const int row0, const int c, float *f) {
      const int row = row0 + lane;
        const int col0 = n0 + c;
        if (col0 >= p.N || row0 >= p.M) return;  // warp-uniform: nothing of this box is stored
#pragma unroll
        for (int j = 0; j < 32; ++j) f[j] *= p.alpha;
        if ((kEpi == EPI_RED && !p.tma_red) || (kEpi == EPI_PUSH && !p.push_tma)) {
          // fused sync: this replica's weighted contribution goes into its own copy
          // and, over NVLink, into the partner replica's copy (EPI_RED: red.add
          // into zeroed arenas) or the partner's staging arena (EPI_PUSH: plain
          // stores; the partner adds staging into its arena after the done
          // handshake).  Two-term fp sums commute: both replicas end bit-identical.
          if (row < p.M && col0 + 32 <= p.N) {
            const int ce = p.c_f32 ? 4 : 2;
            char *own = static_cast<char *>(p.C) + ((long long)row * p.ldc + col0) * ce;
            const int pb = p.red_buf[row];
            char *peer = pb >= 0 ? p.red_base[pb] + ((long long)p.red_row[row] * p.red_ld + col0) * ce
                                 : nullptr;
            if (kEpi == EPI_RED) {
              red_row32(own, f, p.c_f32);
              if (peer) red_row32(peer, f, p.c_f32);
            } else {
              store_row32(own, f, p.c_f32);
              if (peer) store_row32(peer, f, p.c_f32);
            }
          }
          return;
        }
        // staging alternates between two boxes: the store issued two boxes ago
        // (the last-but-one bulk group) must have finished reading this one
        unsigned char *stage = sm.out[q][sbuf];
        sbuf ^= 1;
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncwarp();
        if (kEpi == EPI_GELU) {
          // H = bf16(acc) (kept for the backward), Y = GeLU(H)
          uint4 *hs = reinterpret_cast<uint4 *>(stage + 2048 + lane * 64);
          uint4 *ys = reinterpret_cast<uint4 *>(stage + lane * 64);
          const int sw = stage_swz(lane, 2);
#pragma unroll
          for (int j = 0; j < 32; j += 8) {
            uint32_t hw[4], yw[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              __nv_bfloat162 hh = __floats2bfloat162_rn(f[j + 2 * e], f[j + 2 * e + 1]);
              const float2 hf = __bfloat1622float2(hh);
              __nv_bfloat162 yy = __floats2bfloat162_rn(gelu_f(hf.x), gelu_f(hf.y));
              hw[e] = *reinterpret_cast<uint32_t *>(&hh);
              yw[e] = *reinterpret_cast<uint32_t *>(&yy);
            }
            hs[(j / 8) ^ sw] = make_uint4(hw[0], hw[1], hw[2], hw[3]);
            ys[(j / 8) ^ sw] = make_uint4(yw[0], yw[1], yw[2], yw[3]);
          }
        } else {
          if (kEpi == EPI_DGELU && row < p.M) {
            const __nv_bfloat16 *h = p.aux + (long long)row * p.ld_aux + col0;
            const int nc = min(32, p.N - col0);
            if (nc == 32 && !(reinterpret_cast<uintptr_t>(h) & 15u)) {
#pragma unroll
              for (int j = 0; j < 32; j += 8) {
                const uint4 w = __ldg(reinterpret_cast<const uint4 *>(h + j));
                const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const float2 hf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&ww[e]));
                  f[j + 2 * e] *= gelu_grad_f(hf.x);
                  f[j + 2 * e + 1] *= gelu_grad_f(hf.y);
                }
              }
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (j < nc) f[j] *= gelu_grad_f(__bfloat162float(h[j]));
            }
          }
          if (p.c_f32) {
            float4 *cs = reinterpret_cast<float4 *>(stage + lane * 128);
            const int sw = stage_swz(lane, 4);
#pragma unroll
            for (int j = 0; j < 32; j += 4)
              cs[(j / 4) ^ sw] = make_float4(f[j], f[j + 1], f[j + 2], f[j + 3]);
          } else {
            uint4 *cs = reinterpret_cast<uint4 *>(stage + lane * 64);
            const int sw = stage_swz(lane, 2);
#pragma unroll
            for (int j = 0; j < 32; j += 8) {
              uint32_t w[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                __nv_bfloat162 tt = __floats2bfloat162_rn(f[j + 2 * e], f[j + 2 * e + 1]);
                w[e] = *reinterpret_cast<uint32_t *>(&tt);
              }
              cs[(j / 8) ^ sw] = make_uint4(w[0], w[1], w[2], w[3]);
            }
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        // EPI_PUSH (TMA): the box also goes to the partner replica's staging copy
        // -- one TMA store over NVLink when its 32 rows are consecutive rows of
        // one peer copy, else row stores from registers (run boundaries, ragged M)
        int peer_box = -1, peer_row0 = 0;
        const bool reduce = kEpi == EPI_RED;  // only reached with tma_red
        const bool tma_box = col0 + 32 <= p.tma_cols;
        if (kEpi == EPI_PUSH || reduce) {
          const int pb = row < p.M ? p.red_buf[row] : -1;
          const int pr = row < p.M ? p.red_row[row] : 0;
          const int pb0 = __shfl_sync(0xffffffffu, pb, 0), pr0 = __shfl_sync(0xffffffffu, pr, 0);
          if (__all_sync(0xffffffffu, pb == pb0 && pb0 >= 0 && pr == pr0 + lane)) {
            peer_box = pb0;
            peer_row0 = pr0;
          } else if (pb >= 0 && col0 + 32 <= p.N) {
            const int ce = p.c_f32 ? 4 : 2;
            char *dst = p.red_base[pb] + ((long long)pr * p.red_ld + col0) * ce;
            if (reduce) red_row32(dst, f, p.c_f32);
            else store_row32(dst, f, p.c_f32);
          }
        }
        if (lane == 0) {
          if (reduce) {
            tma_reduce_add_2d(&map_c, stage, col0, row0);
            if (peer_box >= 0) tma_reduce_add_2d(&peer_maps.m[peer_box], stage, col0, peer_row0);
          } else {
            // TMA clips rows >= M; columns only up to tma_cols (16-byte granules)
            if (p.c_tma && tma_box) tma_store_2d(&map_c, stage, col0, row0);
            if (kEpi == EPI_GELU && p.h_tma && tma_box)
              tma_store_2d(&map_h, stage + 2048, col0, row0);
            if (peer_box >= 0) tma_store_2d(&peer_maps.m[peer_box], stage, col0, peer_row0);
          }
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        if (!p.c_tma || !tma_box) box_store(stage, p.C, p.ldc, p.c_f32 ? 4 : 2, row0, col0, p.M, p.N, lane);
        if (kEpi == EPI_GELU && (!p.h_tma || !tma_box))
          box_store(stage + 2048, p.H, p.ldh, 2, row0, col0, p.M, p.N, lane);
        __syncwarp();
    };
    for (int item = unit_id; item < num_items; item += num_units, ++local) {
      const Work w = decode_work(item, p, nk);
      const int t = w.t;
      const int acc = local & 1;
      int tm, tn;
      tile_coords(t, p, tm, tn);
      const int m0 = tm * TM + (int)rank * BM, n0 = tn * BN;
      const int row0 = m0 + q * 32;
      // split-K piece: this warp's 32 x BN partial lives in ws, float4 column
      // groups outermost so each warp access is 512 contiguous bytes
      float4 *slice = w.tail >= 0
          ? reinterpret_cast<float4 *>(
                p.ws + ((((size_t)w.tail * p.split + w.piece) * kPair + rank) * 4 + q) * 32 * BN)
          : nullptr;
      if (p.epi_sleep) mbar_wait_sleepy(&sm.tmem_full[acc], (local >> 1) & 1);
      else mbar_wait(&sm.tmem_full[acc], (local >> 1) & 1);
      const bool tr = p.trace && q == 0 && lane == 0 && local < kTraceItems;
      unsigned long long *trp = tr ? p.trace + ((size_t)blockIdx.x * kTraceItems + local) * 8 : nullptr;
      if (tr) { trp[0] = (unsigned long long)item; trp[1] = gtime(); }
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t v[32];
        const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + c);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, "
            "%10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, "
            "%27, %28, %29, %30, %31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
              "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
              "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
              "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
              "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
              "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (c + 32 >= BN) {
          // all of this accumulator has been read: hand it back to the MMA warp
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if constexpr (kPair == 2) mbar_arrive_cluster(&sm.tmem_empty[acc], 0);
            else mbar_arrive(&sm.tmem_empty[acc]);
          }
        }
        if (slice) {
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            __stcg(slice + (c / 4 + j / 4) * 32 + lane,
                   make_float4(__uint_as_float(v[j]), __uint_as_float(v[j + 1]),
                               __uint_as_float(v[j + 2]), __uint_as_float(v[j + 3])));
        } else if (!(p.debug & 2)) {
          float f[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]);
          emit(n0, row0, c, f);
        }
      }
      if (slice) {
        // Fixup without a blocking barrier.  Every piece publishes its partial
        // and arrives; a piece that sees all `split` pieces arrive within a
        // short window sums every partial, in piece order (deterministic), for
        // its own 32-column chunks i, i+split, ...; chunks are claimed
        // atomically, and the last piece to arrive sums every chunk nobody has
        // claimed.  Nothing waits for a piece that is not running, so the GEMM
        // stays deadlock-free next to kernels that hold SMs; with all pieces
        // co-resident (the normal case) the fixup work is spread over them.
        // Slot layout per warp slice: [arrive, depart, claim[BN/32]].
        constexpr int kSlot = 2 + BN / 32;
        __threadfence();
        __syncwarp();
        int *cnt = p.tile_cnt + (((size_t)w.tail * kPair + rank) * 4 + q) * kSlot;
        int old = 0, arrived = 0;
        if (lane == 0) {
          old = atomicAdd(cnt, 1);
          arrived = old + 1;
          const unsigned long long t0 = gtime();
          while (arrived < p.split && gtime() - t0 < p.split_window_ns) {
            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(arrived) : "l"(cnt) : "memory");
          }
        }
        old = __shfl_sync(0xffffffffu, old, 0);
        arrived = __shfl_sync(0xffffffffu, arrived, 0);
        __threadfence();
        const size_t piece_stride = (size_t)kPair * BM * BN / 4;  // float4s
        const float4 *base = slice - (size_t)w.piece * piece_stride;
        auto fix = [&](const int c) {
          int won = 0;
          if (lane == 0) won = atomicExch(cnt + 2 + c / 32, 1) == 0;
          if (!__shfl_sync(0xffffffffu, won, 0)) return;
          float f[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) f[j] = 0.0f;
          int pc = 0;
          for (; pc + 1 < p.split; pc += 2) {  // two partials' loads in flight
            float4 x[8], y[8];
            const float4 *s0 = base + pc * piece_stride + (c / 4) * 32 + lane;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              x[j] = __ldcg(s0 + j * 32);
              y[j] = __ldcg(s0 + piece_stride + j * 32);
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              f[4 * j] += x[j].x; f[4 * j + 1] += x[j].y; f[4 * j + 2] += x[j].z; f[4 * j + 3] += x[j].w;
              f[4 * j] += y[j].x; f[4 * j + 1] += y[j].y; f[4 * j + 2] += y[j].z; f[4 * j + 3] += y[j].w;
            }
          }
          if (pc < p.split) {
            const float4 *s0 = base + pc * piece_stride + (c / 4) * 32 + lane;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float4 x = __ldcg(s0 + j * 32);
              f[4 * j] += x.x; f[4 * j + 1] += x.y; f[4 * j + 2] += x.z; f[4 * j + 3] += x.w;
            }
          }
          emit(n0, row0, c, f);
        };
        if (arrived >= p.split) {  // everyone published: my own chunks
#pragma unroll 1
          for (int c = w.piece * 32; c < BN; c += 32 * p.split) fix(c);
        }
        if (old == p.split - 1) {  // last arrival: every chunk still unclaimed
#pragma unroll 1
          for (int c = 0; c < BN; c += 32) fix(c);
        }
        // the last piece to leave resets the slot for the next launch
        __syncwarp();
        if (lane == 0 && atomicAdd(cnt + 1, 1) == p.split - 1) {
          __threadfence();
          for (int t = 0; t < kSlot; ++t) cnt[t] = 0;
        }
      }
      if (tr) trp[2] = gtime();
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  if constexpr (kPair == 2) cluster_sync(); else __syncthreads();
  // independent GEMM (pdl 2): completes only after its predecessor, so a later
  // kernel that waits on this one also sees the predecessor's results
  if (p.pdl == 2) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (warp == 1) {
    tc_fence_after();
    if constexpr (kPair == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols(BN)));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols(BN)));
  }
}

// ---------------------------------------------------------------------------
// host side: tensor maps through the driver entry point (no -lcuda link)

using EncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                              const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                              const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

// 2-D tensor map over a row-major [outer][ld] array with logical inner extent
// `inner`: box {box_inner, box_outer}.
static std::atomic<int> g_l2promo{3};

static int make_map(CUtensorMap *m, const void *ptr, CUtensorMapDataType dt, int esize,
                    long long inner, long long outer, long long ld, int box_inner, int box_outer,
                    CUtensorMapSwizzle swz) {
  EncodeFn enc = encode_fn();
  if (!enc) return fail(NTP_ECUDA, "cuTensorMapEncodeTiled unavailable");
  if ((reinterpret_cast<uintptr_t>(ptr) & 15u) || ((ld * esize) & 15))
    return fail(NTP_EINVAL, "GEMM tensors need 16-byte aligned bases and row pitches");
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * esize)};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
  cuuint32_t es[2] = {1u, 1u};
  CUresult r = enc(m, dt, 2, const_cast<void *>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swz, (CUtensorMapL2promotion)g_l2promo.load(),
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char b[96];
    snprintf(b, sizeof b, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return fail(NTP_EINVAL, b);
  }
  return NTP_OK;
}

static int sm_count_dev() {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!cache[dev & 63]) {
    int n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev & 63] = n;
  }
  return cache[dev & 63];
}

static std::atomic<int> g_pair{1};
static std::atomic<int> g_max_ctas{0};
static std::atomic<int> g_split_k{1};
static std::atomic<int> g_pdl{0};
static std::atomic<int> g_raster{0};
static std::atomic<int> g_epi_sleep{1};
static std::atomic<int> g_debug{0};
static unsigned long long *g_trace = nullptr;
static unsigned long long *g_counters = nullptr;
static std::atomic<unsigned long long> g_split_window_ns{250000};

// Split-K partials and per-slice arrival counters, one set per (device, stream)
// so GEMMs on different streams never share them.  Grow-only; counters are
// zeroed on allocation and reset by the last arriving piece.
struct Workspace {
  float *ws = nullptr;
  int *cnt = nullptr;
  size_t ws_bytes = 0, cnt_bytes = 0;
  int ensure(size_t need_ws, size_t need_cnt, cudaStream_t s) {
    if (need_ws > ws_bytes) {
      if (ws) cudaFree(ws);
      if (cudaMalloc(&ws, need_ws) != cudaSuccess) {
        ws = nullptr;
        ws_bytes = 0;
        return fail(NTP_ECUDA, "split-K workspace allocation failed");
      }
      ws_bytes = need_ws;
    }
    if (need_cnt > cnt_bytes) {
      if (cnt) cudaFree(cnt);
      if (cudaMalloc(&cnt, need_cnt) != cudaSuccess || cudaMemsetAsync(cnt, 0, need_cnt, s) != cudaSuccess) {
        cnt = nullptr;
        cnt_bytes = 0;
        return fail(NTP_ECUDA, "split-K counter allocation failed");
      }
      cnt_bytes = need_cnt;
    }
    return NTP_OK;
  }
};

// A ring of 4 per stream: with programmatic dependent launch up to three
// consecutive GEMMs of one stream can be in flight at once, and each launch
// that splits K takes the next workspace of the ring.
struct StreamWorkspaces {
  Workspace w[4];
  unsigned next = 0;
};

static Workspace &workspace_for(cudaStream_t s) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<int, cudaStream_t>, StreamWorkspaces *>> table;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  for (auto &e : table)
    if (e.first.first == dev && e.first.second == s) return e.second->w[e.second->next++ & 3];
  table.push_back({{dev, s}, new StreamWorkspaces()});
  StreamWorkspaces *sw = table.back().second;
  return sw->w[sw->next++ & 3];
}

template <int BN, int kPair, int kStg>
static int launch(const void *A, long long lda, int a_mn, const void *B, long long ldb, int b_mn,
                  void *C, long long ldc, void *H, long long ldh, Params p, cudaStream_t s) {
  constexpr int BNC = BN / kPair;
  CUtensorMap ma, mb, mc, mh;
  const auto BF = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  // operands: SWIZZLE_128B; staged output boxes: 128B (fp32) / 64B (bf16) swizzle
  const auto SW = CU_TENSOR_MAP_SWIZZLE_128B, SW64 = CU_TENSOR_MAP_SWIZZLE_64B;
  int st;
  // A is logically [M x K]: K-major stored [M][lda], MN-major stored [K][lda]
  if ((st = a_mn ? make_map(&ma, A, BF, 2, p.M, p.K, lda, 64, BK, SW)
                 : make_map(&ma, A, BF, 2, p.K, p.M, lda, 64, BM, SW)))
    return st;
  if ((st = b_mn ? make_map(&mb, B, BF, 2, p.N, p.K, ldb, 64, BK, SW)
                 : make_map(&mb, B, BF, 2, p.K, p.N, ldb, 64, BNC, SW)))
    return st;
  const int ce = p.c_f32 ? 4 : 2;
  p.C = C;
  p.H = H;
  p.ldc = ldc;
  p.ldh = ldh;
  PeerMaps pm;
  memset(&pm, 0, sizeof pm);
  const bool c_aligned = !((reinterpret_cast<uintptr_t>(C) & 15u) || ((ldc * ce) & 15));
  if (p.epi == EPI_RED && p.tma_red && !c_aligned) p.tma_red = 0;  // per-thread red.add path
  if ((p.epi == EPI_PUSH && p.push_tma) || (p.epi == EPI_RED && p.tma_red)) {
    // rows: any row a box is checked to own (red_row) -- the extent only bounds the map
    bool ok = true;
    for (int i = 0; i < kMaxPeers && ok; ++i)
      if (p.red_base[i] &&
          make_map(&pm.m[i], p.red_base[i],
                   p.c_f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : BF, ce, p.N, 1ll << 24, p.red_ld,
                   32, 32, p.c_f32 ? SW : SW64))
        ok = false;
    if (!ok) p.push_tma = p.tma_red = 0;  // unaligned peer copy: per-row stores / red.add
  }
  p.c_tma = (p.epi != EPI_RED || p.tma_red) && (p.epi != EPI_PUSH || p.push_tma) && c_aligned;
  p.h_tma = p.epi == EPI_GELU && !((reinterpret_cast<uintptr_t>(H) & 15u) || ((ldh * 2) & 15));
  // whole rows end on a 16-byte boundary: every box may go through TMA; else only
  // the boxes that end inside the row (the last column box is stored per element)
  const bool row_end_aligned = ((p.N * ce) % 16 == 0) && (p.epi != EPI_GELU || (p.N * 2) % 16 == 0);
  p.tma_cols = row_end_aligned ? p.N : (p.N / 32) * 32;
  memset(&mc, 0, sizeof mc);
  memset(&mh, 0, sizeof mh);
  if (p.c_tma && (st = p.c_f32 ? make_map(&mc, C, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, p.N, p.M, ldc,
                                          32, 32, SW)
                               : make_map(&mc, C, BF, 2, p.N, p.M, ldc, 32, 32, SW64)))
    return st;
  if (p.h_tma && (st = make_map(&mh, H, BF, 2, p.N, p.M, ldh, 32, 32, SW64))) return st;
  // one kernel per (producer style, epilogue): each instantiation carries only
  // its own epilogue, which keeps the kernel's code within the instruction cache
  // (measured: the all-epilogue kernel, ~150 KB of SASS, slowed the fused-GeLU
  // GEMMs by 10-15 %)
  using Kern = void (*)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const CUtensorMap,
                        const PeerMaps, Params);
  static const Kern table[5] = {
      gemm_kernel<BN, kPair, kStg, EPI_NONE>, gemm_kernel<BN, kPair, kStg, EPI_GELU>,
      gemm_kernel<BN, kPair, kStg, EPI_DGELU>, gemm_kernel<BN, kPair, kStg, EPI_RED>,
      gemm_kernel<BN, kPair, kStg, EPI_PUSH>};
  if (p.epi < 0 || p.epi > EPI_PUSH) return fail(NTP_EINVAL, "unknown GEMM epilogue");
  auto kern = table[p.epi];
  const int smem = (int)sizeof(Smem<BN, kPair, kStg>) + 1024;
  static std::once_flag once[5][64];
  int dev = 0;
  cudaGetDevice(&dev);
  std::call_once(once[p.epi][dev & 63], [&] {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  });
  p.num_m = (p.M + BM * kPair - 1) / (BM * kPair);
  p.num_n = (p.N + BN - 1) / BN;
  const int tiles = p.num_m * p.num_n;
  int sms = sm_count_dev();
  const int cap = g_max_ctas.load();
  if (cap > 0 && cap < sms) sms = cap;  // leave SMs to a concurrent sync kernel
  const int units = sms / kPair > 0 ? sms / kPair : 1;
  // split-K for the last, partial wave: its R tiles are cut into S K-ranges so
  // the wave is filled instead of leaving most SMs idle for a whole tile time
  p.full_items = tiles;
  p.split = 1;
  p.tile_cnt = nullptr;
  p.ws = nullptr;
  p.trace = g_trace;
  p.counters = g_counters;
  p.raster = g_raster.load();
  p.epi_sleep = g_epi_sleep.load();
  p.debug = g_debug.load();
  p.split_window_ns = g_split_window_ns.load();
  const int rem = tiles % units, nkb = (p.K + BK - 1) / BK;
  if (g_split_k.load() && rem > 0) {
    const int cap_s = g_split_k.load() >= 2 ? g_split_k.load() : 8;
    int S = units / rem;
    if (S > cap_s) S = cap_s;          // bound the fixup's partial reads
    if (S > nkb / 4) S = nkb / 4;      // >= 4 k-blocks per piece
    if (S > BN / 32) S = BN / 32;      // every piece fixes up >= 1 column chunk
    Workspace &w = workspace_for(s);
    const size_t need_ws = (size_t)rem * S * kPair * BM * BN * sizeof(float);
    const size_t need_cnt = (size_t)rem * kPair * 4 * (2 + BN / 32) * sizeof(int);
    cudaStreamCaptureStatus cap_st = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cap_st);
    // never allocate inside a graph capture: run whole tiles instead
    const bool fits = need_ws <= w.ws_bytes && need_cnt <= w.cnt_bytes;
    if (S >= 2 && (fits || cap_st == cudaStreamCaptureStatusNone)) {
      int st2 = w.ensure(need_ws, need_cnt, s);
      if (st2) return st2;
      p.full_items = tiles - rem;
      p.split = S;
      p.ws = w.ws;
      p.tile_cnt = w.cnt;
    }
  }
  const int items = p.full_items + (tiles - p.full_items) * p.split;
  const int grid = (items < units ? items : units) * kPair;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kPair;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = p.pdl ? 2 : 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ma, mb, mc, mh, pm, p);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return fail(NTP_ECUDA, std::string("gemm launch: ") + cudaGetErrorString(e));
  return NTP_OK;
}


}  // namespace gemm
}  // namespace ntp

namespace ntp {
namespace gemm {
int dispatch(const void *A, long long lda, int a_mn, const void *B, long long ldb, int b_mn,
             void *C, long long ldc, void *H, long long ld_aux, Params p, cudaStream_t s);
}  // namespace gemm
}  // namespace ntp

using namespace ntp;

extern "C" int ntp_gemm_bf16_ex(const void *A, int64_t lda, int a_mn, const void *B,
                                int64_t ldb, int b_mn, void *C, int64_t ldc, int c_f32, int64_t M,
                                int64_t N, int64_t K, int epilogue, const void *aux,
                                int64_t ld_aux, float alpha, int pdl, void *stream);

extern "C" int ntp_gemm_bf16(const void *A, int64_t lda, int a_mn, const void *B, int64_t ldb,
                             int b_mn, void *C, int64_t ldc, int c_f32, int64_t M, int64_t N,
                             int64_t K, int epilogue, const void *aux, int64_t ld_aux,
                             float alpha, void *stream) {
  return ntp_gemm_bf16_ex(A, lda, a_mn, B, ldb, b_mn, C, ldc, c_f32, M, N, K, epilogue, aux,
                          ld_aux, alpha, gemm::g_pdl.load(), stream);
}

extern "C" int ntp_gemm_bf16_ex(const void *A, int64_t lda, int a_mn, const void *B,
                                int64_t ldb, int b_mn, void *C, int64_t ldc, int c_f32, int64_t M,
                                int64_t N, int64_t K, int epilogue, const void *aux,
                                int64_t ld_aux, float alpha, int pdl, void *stream) {
  if (pdl < 0 || pdl > 2) return fail(NTP_EINVAL, "pdl must be 0, 1 (after) or 2 (independent)");
  if (M <= 0 || N <= 0 || K <= 0) return fail(NTP_EINVAL, "GEMM extents must be positive");
  if (M > (1ll << 31) || N > (1ll << 31) || K > (1ll << 31))
    return fail(NTP_EINVAL, "GEMM extent too large");
  if (epilogue < 0 || epilogue > 2) return fail(NTP_EINVAL, "unknown GEMM epilogue");
  if (epilogue != gemm::EPI_NONE && !aux) return fail(NTP_EINVAL, "epilogue needs an aux tensor");
  if (epilogue == gemm::EPI_GELU && c_f32) return fail(NTP_EINVAL, "GeLU epilogue writes bf16");
  gemm::Params p{(int)M, (int)N, (int)K, a_mn ? 1 : 0, b_mn ? 1 : 0, c_f32 ? 1 : 0, epilogue,
                 static_cast<const __nv_bfloat16 *>(aux), ld_aux, alpha, 0, 0,
                 nullptr, nullptr, 0, 0, 0, 0};
  p.pdl = pdl;
  return gemm::dispatch(A, lda, a_mn, B, ldb, b_mn, C, ldc, const_cast<void *>(aux), ld_aux, p,
                        static_cast<cudaStream_t>(stream));
}

// Fused weight-gradient GEMM + NTP gradient sync (EPI_RED, see the epilogue).
extern "C" int ntp_gemm_bf16_red(const void *A, int64_t lda, int a_mn, const void *B,
                                 int64_t ldb, int b_mn, void *C, int64_t ldc, int c_f32,
                                 int64_t M, int64_t N, int64_t K, float alpha,
                                 const int32_t *red_buf, const int32_t *red_row,
                                 void *const *red_base, int n_red, int64_t red_ld, int mode,
                                 void *stream) {
  if (mode < 0 || mode > 3)
    return fail(NTP_EINVAL,
                "fused mode must be 0 (red), 1 (push), 2 (push, TMA boxes) or 3 (red, TMA boxes)");
  if (M <= 0 || N <= 0 || K <= 0) return fail(NTP_EINVAL, "GEMM extents must be positive");
  if (N % 32) return fail(NTP_EINVAL, "fused sync GEMM needs N % 32 == 0");
  if (n_red < 0 || n_red > gemm::kMaxPeers) return fail(NTP_EINVAL, "at most 8 peer copies");
  if (!red_buf || !red_row) return fail(NTP_EINVAL, "fused sync GEMM needs a row map");
  const int ce = c_f32 ? 4 : 2;
  if ((reinterpret_cast<uintptr_t>(C) & 15u) || ((ldc * ce) & 15) || ((red_ld * ce) & 15))
    return fail(NTP_EINVAL, "fused sync GEMM needs 16-byte aligned rows");
  gemm::Params p{(int)M, (int)N, (int)K, a_mn ? 1 : 0, b_mn ? 1 : 0, c_f32 ? 1 : 0,
                 (mode == 1 || mode == 2) ? gemm::EPI_PUSH : gemm::EPI_RED, nullptr, 0, alpha,
                 0, 0, nullptr,
                 nullptr, 0, 0, 0, 0};
  p.red_buf = red_buf;
  p.red_row = red_row;
  for (int i = 0; i < gemm::kMaxPeers; ++i)
    p.red_base[i] = i < n_red ? static_cast<char *>(red_base[i]) : nullptr;
  for (int i = 0; i < n_red; ++i)
    if (reinterpret_cast<uintptr_t>(p.red_base[i]) & 15u)
      return fail(NTP_EINVAL, "peer copies must be 16-byte aligned");
  p.red_ld = red_ld;
  p.push_tma = mode == 2;
  p.tma_red = mode == 3;
  p.pdl = gemm::g_pdl.load();
  return gemm::dispatch(A, lda, a_mn, B, ldb, b_mn, C, ldc, nullptr, 0, p,
                        static_cast<cudaStream_t>(stream));
}

namespace ntp {
namespace gemm {
int dispatch(const void *A, long long lda, int a_mn, const void *B, long long ldb, int b_mn,
             void *C, long long ldc, void *H, long long ld_aux, Params p, cudaStream_t s) {
  const long long M = p.M, N = p.N;
  if (!gemm::g_pair.load()) {
    if (N > 128) return gemm::launch<256, 1, 4>(A, lda, a_mn, B, ldb, b_mn, C, ldc, H, ld_aux, p, s);
    return gemm::launch<128, 1, 4>(A, lda, a_mn, B, ldb, b_mn, C, ldc, H, ld_aux, p, s);
  }
  // CTA-pair tiles 256 x 256 or 256 x 128: pick the one with the fewer per-SM
  // MACs over the whole (wave-quantized) persistent schedule -- a ragged tile
  // count that spills a few tiles into an extra wave costs a full wave.
  int sms = gemm::sm_count_dev();
  const int cap = gemm::g_max_ctas.load();
  if (cap > 0 && cap < sms) sms = cap;
  const long long pairs = sms / 2 > 0 ? sms / 2 : 1;
  auto cost = [&](long long bn) {
    const long long tiles = ((M + 255) / 256) * ((N + bn - 1) / bn);
    return ((tiles + pairs - 1) / pairs) * bn;  // rounds x per-SM tile width
  };
  const int mode = gemm::g_pair.load();
  // Measured (profiles/r01_gemm_bench_v5.json): 256-wide pair tiles beat 128-wide
  // ones by 1.3-1.6x on every C4 GEMM even where they lose a wave to quantization
  // (the narrow tile doubles the A-operand bytes per MAC), so AUTO only takes
  // the narrow tile when the wide one would need twice the waves.
  const bool wide = mode == 3 || mode == 4 || (mode == 1 && cost(256) <= 2 * cost(128));
  // 256 x 224 pair tiles (K-major B only: an MN-major B box is loaded in 64-row
  // blocks per CTA) remove the wave quantisation of N = 3584 (14 -> 16 N-tiles:
  // 448 -> 512 tiles on 74 pairs) but measured 3-9 % slower than 256 x 256 on
  // the C4 shapes (lower MACs per operand byte; profiles/r02/gemm_bench_c4_bn224.json),
  // so only the explicit mode 4 takes them
  const bool n224 = !b_mn && N > 192 && mode == 4;
  if (n224) return gemm::launch<224, 2, 6>(A, lda, a_mn, B, ldb, b_mn, C, ldc, H, ld_aux, p, s);
  if (N > 128 && mode != 2 && wide)
    return gemm::launch<256, 2, 6>(A, lda, a_mn, B, ldb, b_mn, C, ldc, H, ld_aux, p, s);
  return gemm::launch<128, 2, 8>(A, lda, a_mn, B, ldb, b_mn, C, ldc, H, ld_aux, p, s);
}
}  // namespace gemm
}  // namespace ntp

// 1 (default): split-K the last partial wave into <= 8 pieces per tile;
// n >= 2: at most n pieces; 0: whole tiles only.
extern "C" int ntp_gemm_set_split_k(int on) {
  if (on < 0 || on > 64) return fail(NTP_EINVAL, "split_k must be in [0, 64]");
  gemm::g_split_k.store(on);
  return NTP_OK;
}

// Debug hook, deliberately not in include/ntp_b200.h: device buffer of
// gridDim * 16 * 8 u64 receiving per-item epilogue timestamps (nullptr: off).
// Debug hook, not in the header: how long a split-K piece waits for the other
// pieces of its tile before leaving the fixup to the last arrival (default
// 250 us; 0 forces the last-arrival path).
extern "C" int ntp_gemm_debug_split_window(unsigned long long ns) {
  gemm::g_split_window_ns.store(ns);
  return NTP_OK;
}

// Debug hook, not in the header: tile order (groups of n M-tile rows; 0 = all)
extern "C" int ntp_gemm_debug_raster(int n) {
  if (n < 0) return fail(NTP_EINVAL, "bad raster group");
  gemm::g_raster.store(n);
  return NTP_OK;
}

// Debug hook, not in the header: 1 (default) the epilogue's accumulator wait
// sleeps between polls; 0 spins
extern "C" int ntp_gemm_debug_epi_sleep(int on) {
  gemm::g_epi_sleep.store(on ? 1 : 0);
  return NTP_OK;
}

// Debug hook, not in the header: experiment bits (1 no loads, 2 no epilogue output)
// Debug hook, not in the header: TMA L2 promotion of the GEMM maps (0 none,
// 1 64B, 2 128B, 3 256B = default)
extern "C" int ntp_gemm_debug_l2promo(int v) {
  if (v < 0 || v > 3) return fail(NTP_EINVAL, "bad L2 promotion");
  gemm::g_l2promo.store(v);
  return NTP_OK;
}

extern "C" int ntp_gemm_debug_mode(int bits) {
  gemm::g_debug.store(bits);
  return NTP_OK;
}

// Debug hook, not in the header: device buffer of gridDim * 4 u64 receiving
// per-CTA wait-cycle counters (nullptr: off)
extern "C" int ntp_gemm_debug_counters(void *buf) {
  gemm::g_counters = static_cast<unsigned long long *>(buf);
  return NTP_OK;
}

extern "C" int ntp_gemm_debug_trace(void *buf) {
  gemm::g_trace = static_cast<unsigned long long *>(buf);
  return NTP_OK;
}

// 1: every GEMM launch (ntp_gemm_bf16, ntp_gemm_bf16_red) uses programmatic
// dependent launch, waiting for its predecessor before touching memory; 0: off.
extern "C" int ntp_gemm_set_pdl(int on) {
  gemm::g_pdl.store(on ? 1 : 0);
  return NTP_OK;
}

// Cap on persistent GEMM CTAs (0 = all SMs): overlap with a CTA-capped sync.
extern "C" int ntp_gemm_set_max_ctas(int n) {
  if (n < 0) return fail(NTP_EINVAL, "bad CTA cap");
  gemm::g_max_ctas.store(n);
  return NTP_OK;
}

extern "C" int ntp_gemm_get_max_ctas(void) { return gemm::g_max_ctas.load(); }

// 1 (default): CTA-pair tiles (tcgen05 cta_group::2), width picked per shape;
// 0: 1-SM tiles; 2 / 3 / 4: force 256x128 / 256x256 / 256x224 pair tiles
// (224 only with a K-major B operand; otherwise 256).
extern "C" int ntp_gemm_set_pair(int mode) {
  if (mode < 0 || mode > 4) return fail(NTP_EINVAL, "pair mode must be 0..4");
  gemm::g_pair.store(mode);
  return NTP_OK;
}
