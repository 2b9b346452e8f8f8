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
#include <cstring>
#include <mutex>
#include <string>

#include "ntp_internal.h"

namespace ntp {
namespace gemm {

constexpr int BM = 128;
constexpr int BK = 64;          // 64 bf16 = 128 B: one swizzle-128B row
constexpr int kStages = 4;
constexpr int kThreads = 192;   // 6 warps
constexpr int kEpiWarp0 = 2;

enum Epi { EPI_NONE = 0, EPI_GELU = 1, EPI_DGELU = 2 };

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

__device__ __forceinline__ float gelu_f(float x) {
  // tanh GeLU, tpnumerics.py:25-28
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  return 0.5f * x * (1.0f + tanhf(k0 * (x + k1 * x * x * x)));
}
__device__ __forceinline__ float gelu_grad_f(float x) {
  // tpnumerics.py:31-36
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  const float t = tanhf(k0 * (x + k1 * x * x * x));
  const float du = k0 * (1.0f + 3.0f * k1 * x * x);
  return 0.5f * (1.0f + t) + 0.5f * x * (1.0f - t * t) * du;
}

struct Params {
  int M, N, K;
  int a_mn, b_mn;          // 1 = operand is MN-major in global memory
  void *C;
  long long ldc;           // elements
  int c_f32;               // 1: fp32 output, 0: bf16
  int epi;
  const __nv_bfloat16 *aux;  // EPI_DGELU: H (read), EPI_GELU: H (written)
  long long ld_aux;
  float alpha;
};

template <int BN>
struct Smem {
  alignas(1024) __nv_bfloat16 a[kStages][BM * BK];
  alignas(1024) __nv_bfloat16 b[kStages][BN * BK];
  uint64_t full[kStages];
  uint64_t empty[kStages];
  uint64_t tmem_full;
  uint32_t tmem_base;
};

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
            Params p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // align the dynamic smem base to 1024 B (swizzle-128B atoms)
  const uint32_t base = smem_u32(smem_raw);
  unsigned char *aligned = smem_raw + ((1024u - (base & 1023u)) & 1023u);
  Smem<BN> &sm = *reinterpret_cast<Smem<BN> *>(aligned);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * BM;
  const int n0 = blockIdx.x * BN;
  const int nk = (p.K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], 1);
    }
    mbar_init(&sm.tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {  // TMEM: BN fp32 columns x 128 lanes
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&sm.tmem_base)),
                 "r"(BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer ----
      const uint32_t stage_bytes = (BM + BN) * BK * 2;
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % kStages;
        mbar_wait(&sm.empty[s], ((kb / kStages) & 1) ^ 1);
        mbar_expect_tx(&sm.full[s], stage_bytes);
        const int k0 = kb * BK;
        if (!p.a_mn) {
          tma_load_2d(sm.a[s], &map_a, k0, m0, &sm.full[s]);
        } else {
#pragma unroll
          for (int j = 0; j < BM / 64; ++j)
            tma_load_2d(sm.a[s] + j * 64 * BK, &map_a, m0 + 64 * j, k0, &sm.full[s]);
        }
        if (!p.b_mn) {
          tma_load_2d(sm.b[s], &map_b, k0, n0, &sm.full[s]);
        } else {
#pragma unroll
          for (int j = 0; j < BN / 64; ++j)
            tma_load_2d(sm.b[s] + j * 64 * BK, &map_b, n0 + 64 * j, k0, &sm.full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---- MMA issuer ----
      const uint32_t idesc = instr_desc(BM, BN, p.a_mn, p.b_mn);
      // K-major: rows of 128 B, 8-row atoms 1024 B apart (SBO); K advance +32 B per k16.
      // MN-major: 64-element MN blocks of BK rows (LBO = BK*128 B), 8-row K groups
      // 1024 B apart (SBO); K advance +2048 B per k16.
      const uint32_t a_lbo = p.a_mn ? BK * 128 : 16, b_lbo = p.b_mn ? BK * 128 : 16;
      const uint32_t k_step_a = p.a_mn ? 2048u : 32u, k_step_b = p.b_mn ? 2048u : 32u;
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % kStages;
        mbar_wait(&sm.full[s], (kb / kStages) & 1);
        tc_fence_after();
        const uint32_t a_addr = smem_u32(sm.a[s]), b_addr = smem_u32(sm.b[s]);
#pragma unroll
        for (int kk = 0; kk < BK / 16; ++kk) {
          const uint64_t ad = smem_desc(a_addr + kk * k_step_a, a_lbo, 1024);
          const uint64_t bd = smem_desc(b_addr + kk * k_step_b, b_lbo, 1024);
          tc_mma(tmem, ad, bd, idesc, (kb | kk) ? 1u : 0u);
        }
        tc_commit(&sm.empty[s]);  // frees the stage once these MMAs have read it
      }
      tc_commit(&sm.tmem_full);
    }
  } else {
    // ---- epilogue: TMEM -> registers -> fused op -> global ----
    const int q = warp & 3;                      // TMEM lane quarter this warp may access
    const int row = m0 + q * 32 + lane;
    mbar_wait(&sm.tmem_full, 0);
    tc_fence_after();
    const bool row_ok = row < p.M;
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      uint32_t v[32];
      const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c;
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
      if (!row_ok) continue;
      const int col0 = n0 + c;
      if (col0 >= p.N) continue;
      const int ncols = min(32, p.N - col0);
      float f[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]) * p.alpha;
      if (p.epi == EPI_GELU) {
        __nv_bfloat16 *h = const_cast<__nv_bfloat16 *>(p.aux) + (long long)row * p.ld_aux + col0;
        for (int j = 0; j < ncols; ++j) {
          h[j] = __float2bfloat16_rn(f[j]);
          f[j] = gelu_f(__bfloat162float(h[j]));
        }
      } else if (p.epi == EPI_DGELU) {
        const __nv_bfloat16 *h = p.aux + (long long)row * p.ld_aux + col0;
        for (int j = 0; j < ncols; ++j) f[j] *= gelu_grad_f(__bfloat162float(h[j]));
      }
      if (p.c_f32) {
        float *out = reinterpret_cast<float *>(p.C) + (long long)row * p.ldc + col0;
        for (int j = 0; j < ncols; ++j) out[j] = f[j];
      } else {
        __nv_bfloat16 *out = reinterpret_cast<__nv_bfloat16 *>(p.C) + (long long)row * p.ldc + col0;
        if (ncols == 32 && ((reinterpret_cast<uintptr_t>(out) & 15u) == 0)) {
#pragma unroll
          for (int j = 0; j < 32; j += 8) {
            uint4 w;
            __nv_bfloat162 t0 = __floats2bfloat162_rn(f[j], f[j + 1]);
            __nv_bfloat162 t1 = __floats2bfloat162_rn(f[j + 2], f[j + 3]);
            __nv_bfloat162 t2 = __floats2bfloat162_rn(f[j + 4], f[j + 5]);
            __nv_bfloat162 t3 = __floats2bfloat162_rn(f[j + 6], f[j + 7]);
            w.x = *reinterpret_cast<uint32_t *>(&t0);
            w.y = *reinterpret_cast<uint32_t *>(&t1);
            w.z = *reinterpret_cast<uint32_t *>(&t2);
            w.w = *reinterpret_cast<uint32_t *>(&t3);
            *reinterpret_cast<uint4 *>(out + j) = w;
          }
        } else {
          for (int j = 0; j < ncols; ++j) out[j] = __float2bfloat16_rn(f[j]);
        }
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(BN));
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

// 2-D bf16 tensor map: inner (contiguous) extent `inner`, outer extent `outer`,
// row pitch `ld` elements, box {64, box_outer}, 128B swizzle, OOB -> 0.
static int make_map(CUtensorMap *m, const void *ptr, long long inner, long long outer,
                    long long ld, int box_outer) {
  EncodeFn enc = encode_fn();
  if (!enc) return fail(NTP_ECUDA, "cuTensorMapEncodeTiled unavailable");
  if ((reinterpret_cast<uintptr_t>(ptr) & 15u) || ((ld * 2) & 15))
    return fail(NTP_EINVAL, "GEMM operands need 16-byte aligned base and row pitch");
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {64u, (cuuint32_t)box_outer};
  cuuint32_t es[2] = {1u, 1u};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(ptr), dims, strides,
                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char b[96];
    snprintf(b, sizeof b, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return fail(NTP_EINVAL, b);
  }
  return NTP_OK;
}

template <int BN>
static int launch(const void *A, long long lda, int a_mn, const void *B, long long ldb, int b_mn,
                  const Params &p, cudaStream_t s) {
  CUtensorMap ma, mb;
  int st;
  // A is logically [M x K]: K-major stored [M][lda], MN-major stored [K][lda]
  if ((st = a_mn ? make_map(&ma, A, p.M, p.K, lda, BK) : make_map(&ma, A, p.K, p.M, lda, BM)))
    return st;
  if ((st = b_mn ? make_map(&mb, B, p.N, p.K, ldb, BK) : make_map(&mb, B, p.K, p.N, ldb, BN)))
    return st;
  const int smem = (int)sizeof(Smem<BN>) + 1024;
  static std::once_flag once[64];
  int dev = 0;
  cudaGetDevice(&dev);
  std::call_once(once[dev & 63], [&] {
    cudaFuncSetAttribute(gemm_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  });
  dim3 grid((p.N + BN - 1) / BN, (p.M + BM - 1) / BM);
  gemm_kernel<BN><<<grid, kThreads, smem, s>>>(ma, mb, p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(NTP_ECUDA, std::string("gemm launch: ") + cudaGetErrorString(e));
  return NTP_OK;
}

}  // namespace gemm
}  // namespace ntp

using namespace ntp;

extern "C" int ntp_gemm_bf16(const void *A, int64_t lda, int a_mn, const void *B, int64_t ldb,
                             int b_mn, void *C, int64_t ldc, int c_f32, int64_t M, int64_t N,
                             int64_t K, int epilogue, const void *aux, int64_t ld_aux,
                             float alpha, void *stream) {
  if (M <= 0 || N <= 0 || K <= 0) return fail(NTP_EINVAL, "GEMM extents must be positive");
  if (M > (1ll << 31) || N > (1ll << 31) || K > (1ll << 31))
    return fail(NTP_EINVAL, "GEMM extent too large");
  if (epilogue < 0 || epilogue > 2) return fail(NTP_EINVAL, "unknown GEMM epilogue");
  if (epilogue != gemm::EPI_NONE && !aux) return fail(NTP_EINVAL, "epilogue needs an aux tensor");
  gemm::Params p{(int)M, (int)N, (int)K, a_mn ? 1 : 0, b_mn ? 1 : 0, C, ldc, c_f32 ? 1 : 0,
                 epilogue, static_cast<const __nv_bfloat16 *>(aux), ld_aux, alpha};
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (N > 128) return gemm::launch<256>(A, lda, a_mn, B, ldb, b_mn, p, s);
  return gemm::launch<128>(A, lda, a_mn, B, ldb, b_mn, p, s);
}
