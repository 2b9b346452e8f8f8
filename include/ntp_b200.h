/*
 * ntp_b200.h -- C ABI of the B200-native NTP gradient reshard-and-reduce path.
 *
 * The reference (arxiv 2504.06095, package `ntpsim`) has no FFI: its boundary
 * is the Python module API of pkg/src/ntpsim/shardmap.py and
 * pkg/src/ntpsim/tpnumerics.py.  Each entry point below names the reference
 * function it replaces (file:line, relative to pkg/src/ntpsim/).  The Python
 * package paper_2504_06095_b200 binds these with ctypes and re-exposes the
 * reference's names, argument meaning and ValueError texts; INTEGRATION.md
 * shows the binding a maintainer of the reference would add.
 *
 * Conventions
 *   - plain pointers and sizes only; no torch types.  Device buffers are raw
 *     CUDA device pointers (local or peer-mapped); `stream` is a cudaStream_t.
 *   - return value: NTP_OK (0) or a negative status; ntp_last_error() gives
 *     the message (per thread).  NTP_EINVAL carries the reference's ValueError
 *     text where the reference has one.
 *   - all hot-path calls are stream-ordered and asynchronous; no hidden
 *     allocation happens on the hot path (plans own their device tables).
 *
 * Unit-major layout: a rank's gradient buffer stores its columns one after
 * another; column ("unit") p of a rank occupies elements [off_p, off_p + U).
 * For an MLP column U = 2*hidden (A column then B row, perfmodel.py:269); for
 * an attention head U = 4*hidden*head_dim (perfmodel.py:270-272).
 */
#ifndef NTP_B200_H
#define NTP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NTP_ABI_VERSION 1

enum ntp_status {
  NTP_OK = 0,
  NTP_EINVAL = -1, /* bad argument: Python raises ValueError(ntp_last_error()) */
  NTP_ECUDA = -2,  /* CUDA runtime error: Python raises RuntimeError */
  NTP_ENOMEM = -3,
  NTP_ESTATE = -4, /* call out of order (e.g. execute before finalize) */
  NTP_ETIMEOUT = -5 /* a cross-GPU signal did not arrive in time */
};

enum ntp_dtype { NTP_F32 = 0, NTP_BF16 = 1, NTP_F16 = 2, NTP_F64 = 3 };

/* _reduce, tpnumerics.py:255-260 ("sum" -> a+b, "mean" -> (a+b)/2) plus the
 * per-replica batch weighting extension w_a*a + w_b*b. */
enum ntp_op { NTP_OP_SUM = 0, NTP_OP_MEAN = 1, NTP_OP_WEIGHTED = 2 };

/* PRE_SYNC / POST_SYNC, shardmap.py:19-20 */
enum ntp_direction { NTP_PRE_SYNC = 0, NTP_POST_SYNC = 1 };

const char *ntp_last_error(void);
int ntp_abi_version(void);

/* Process-wide tuning knobs (no reference counterpart). */
enum ntp_option {
  NTP_OPT_SYNC_KERNEL = 0,   /* value: enum ntp_sync_kernel */
  NTP_OPT_SYNC_MAX_CTAS = 1,  /* value: cap on sync-kernel CTAs, 0 = all SMs */
  NTP_OPT_PLAN_MIN_CHUNKS = 2, /* value: plans finalized afterwards get at least this many
                                 chunks (smaller chunks, >= 64 grains; default 1184 = 8
                                 per SM: a 16 MB-per-replica N=2 step 47.7 -> 43.1 us);
                                 0 = always 16 KiB chunks */
  NTP_OPT_SYNC_L2 = 3         /* value: L2 policy of the bulk sync kernel's copies: 0 none
                                 (default), 1 loads evict_first, 2 loads + stores */
};
enum ntp_sync_kernel {
  NTP_KERNEL_AUTO = 0,  /* default: LDG below 4 chunks per SM, BULK above */
  NTP_KERNEL_LDG = 1,   /* 128-bit register-staged loads/stores */
  NTP_KERNEL_BULK = 2,  /* TMA bulk copies through shared memory, 4 stages, 1 CTA/SM */
  NTP_KERNEL_BULK2 = 3  /* TMA bulk copies, 3 stages, 2 CTAs/SM */
};
int ntp_set_option(int option, int64_t value);
int64_t ntp_get_option(int option);

/* ------------------------------------------------------------------------
 * Shard algebra (host, integer, bit-exact with the reference)
 * ------------------------------------------------------------------------ */

/* build_shard_map, shardmap.py:141-182 (validation: _validate_triple 132-138).
 * Writes comp_rank[k] in [0,n1) and sync_rank[k] in [0,n2). */
int ntp_shard_map(int64_t k, int64_t n1, int64_t n2, int64_t *comp_rank, int64_t *sync_rank);

/* build_reshard_plan, shardmap.py:185-206, flattened: every moving column
 * becomes one (src, dst, col) triple, sorted by (src, dst, col) -- the
 * reference's transfer order.  Arrays must hold k entries.  Returns the
 * number of triples (>= 0) or a negative status. */
int64_t ntp_reshard_plan(const int64_t *comp_rank, const int64_t *sync_rank, int64_t k,
                         int64_t n1, int direction, int64_t *src, int64_t *dst, int64_t *col);

/* apply_plan, shardmap.py:209-217: replay n_moves (src, dst, col) triples in
 * order on ownership[k] in place.  NTP_EINVAL with the reference's message if
 * a transfer names a column its src does not own. */
int ntp_apply_plan(int64_t *ownership, int64_t k, const int64_t *src, const int64_t *dst,
                   const int64_t *col, int64_t n_moves);

/* naive_contiguous_sync_volumes, shardmap.py:220-245: contiguous TP-n2 vs
 * contiguous TP-n1 interval overlaps.  pairs gets (healthy, overlap) pairs,
 * reduced shard by reduced shard (capacity 2*(n1+n2)); per_reduced[n2] the
 * pair count of each reduced shard.  Returns the total pair count. */
int64_t ntp_naive_overlaps(int64_t k, int64_t n1, int64_t n2, int64_t *pairs,
                           int64_t *per_reduced);

/* Interval-overlap planner between any two contiguous balanced partitions of k
 * (TP-n_src -> TP-n_dst), the building block of reconfiguration: writes
 * (src_rank, dst_rank, start, length) quadruples in ascending start order
 * (capacity 4*(n_src+n_dst)).  Returns the count. */
int64_t ntp_interval_overlaps(int64_t k, int64_t n_src, int64_t n_dst, int64_t *quads);

/* attention_head_partition, shardmap.py:248-260. */
int ntp_head_partition(int64_t heads, int64_t n, int64_t *counts, double *imbalance);

/* ------------------------------------------------------------------------
 * Copy/reduce plans (host build, device-resident table)
 * ------------------------------------------------------------------------ */

typedef struct ntp_plan ntp_plan;

typedef struct ntp_plan_stats {
  int64_t n_units;    /* units added */
  int64_t n_runs;     /* maximal runs after merging contiguous units */
  int64_t n_chunks;   /* device work items */
  int64_t elems;      /* elements per side (sum of unit sizes) */
  int32_t vectorized; /* 1: every run is 16-byte aligned -> 128-bit path */
  int32_t max_buf;    /* highest buffer index referenced */
  int32_t dtype;
  int32_t device;     /* device the table was uploaded to, -1 if not */
} ntp_plan_stats;

int ntp_plan_create(ntp_plan **out, int dtype);

/* Append n_units units of unit_elems elements each: unit j pairs side A at
 * bufs[a_buf[j]] + a_off[j] with side B at bufs[b_buf[j]] + b_off[j]
 * (element offsets).  For a sync plan A is the healthy replica's copy and B
 * the reduced replica's (operand order of tpnumerics.py:342-343); for a
 * reshard plan A is the source and B the destination. */
int ntp_plan_add_units(ntp_plan *plan, int64_t n_units, int64_t unit_elems, const int32_t *a_buf,
                       const int64_t *a_off, const int32_t *b_buf, const int64_t *b_off);

/* Merge contiguous units into runs and split runs into device chunks (host). */
int ntp_plan_finalize(ntp_plan *plan);
int ntp_plan_stats_get(const ntp_plan *plan, ntp_plan_stats *out);

/* Export the finalized host table: per chunk (a_buf, a_off, b_buf, b_off, len)
 * in elements; out holds 5*n_chunks int64.  For tests and tooling. */
int ntp_plan_export(const ntp_plan *plan, int64_t *out);

/* Copy the finalized table to device `device` (cudaMalloc + memcpy). */
int ntp_plan_upload(ntp_plan *plan, int device);
void ntp_plan_destroy(ntp_plan *plan);

/* ------------------------------------------------------------------------
 * Hot path (device, stream-ordered)
 * ------------------------------------------------------------------------ */

/* nonuniform_grad_sync, tpnumerics.py:289-356 (and the aligned case of
 * uniform_grad_sync, 263-286, for two replicas): for every unit of the plan
 *   v = op(A, B)   (fp32 accumulation; fp64 for NTP_F64)
 *   A = v; B = v   (both replicas end with identical bits, 346-347/355-356)
 * in one kernel, with no staging buffer: the reference's pre-sync gather,
 * pairwise reduce and post-sync scatter (323-356) collapse into direct reads
 * of each unit's two owners.  bufs[n_bufs] may be peer-mapped pointers. */
int ntp_grad_sync(const ntp_plan *plan, void *const *bufs, int n_bufs, int op, double w_a,
                  double w_b, void *stream);

/* ntp_grad_sync with a write mask: bit 0 writes the result to side A, bit 1 to
 * side B.  write_mask = 1 accumulates the B replica's (weighted) contribution
 * into A only -- the first phase of a DP > 2 sync across processes (the degraded
 * replica's share folded into one healthy replica before the NCCL all-reduce of
 * the aligned healthy replicas). */
int ntp_grad_sync_ex(const ntp_plan *plan, void *const *bufs, int n_bufs, int op, double w_a,
                     double w_b, int write_mask, void *stream);

/* Static memory-safety check of a finalized plan (no device work): every
 * chunk's element range on both sides lies inside its buffer (buf_elems[b]
 * elements, n_bufs buffers), and, for the sides in write_sides (bit 0: side
 * A, bit 1: side B; 3 for a sync, 2 for a reshard copy), no element is written
 * by two chunks, i.e. no two CTAs of a launch write the same bytes.  Returns
 * NTP_EINVAL naming the offending chunk(s).  (compute-sanitizer is closed on
 * the B200 pool: this, the canary tests and the oracle comparisons stand in.) */
int ntp_plan_check(const ntp_plan *plan, const int64_t *buf_elems, int n_bufs, int write_sides);

/* Reconfiguration copy (no reference function; built from build_reshard_plan
 * 185-206 / apply_plan 209-217 / contiguous_assignment tpnumerics.py:115-120):
 * B = A for every unit.  Bit-exact. */
int ntp_reshard(const ntp_plan *plan, void *const *bufs, int n_bufs, void *stream);

/* uniform_grad_sync, tpnumerics.py:263-286, over R identically laid out local
 * replicas of n elements: sum in replica order (op SUM), true mean (MEAN) or
 * sum_r w[r]*x_r (WEIGHTED), written back to all R.  w (host memory, R
 * doubles) is read during the call and passed to the kernel by value: no
 * device allocation or copy per call.  128-bit vector path when every
 * replica is 16-byte aligned. */
int ntp_uniform_sync(void *const *reps, int R, int64_t n, int dtype, int op, const double *w,
                     void *stream);

/* dsts[d] = srcs[0] + srcs[1] + ... + srcs[R-1] in that order (accumulated in
 * fp32, fp64 for f64) for every d < n_dst, n elements; a destination may alias
 * a source and may be a peer GPU's (IPC-mapped) memory.  The owner's step of
 * the row-parallel all-reduce (mlp_forward_tp's ascending-rank sum,
 * tpnumerics.py:177-185, across GPUs: dist_linear.py): sum the pushed partial
 * sums and write the block into every rank's output at once. */
int ntp_reduce_into(void *const *srcs, int R, int64_t n, int dtype, void *const *dsts, int n_dst,
                    void *stream);

/* ------------------------------------------------------------------------
 * R-way sync for DP > 2 (no reference function: composes nonuniform_grad_sync,
 * tpnumerics.py:289-356, with uniform_grad_sync, 263-286)
 * ------------------------------------------------------------------------ */

typedef struct ntp_mplan ntp_mplan;

/* R in [2, 8] replicas; dtype NTP_BF16 or NTP_F32. */
int ntp_mplan_create(ntp_mplan **out, int dtype, int R);
/* bufs/offs are [R][n_units] (replica-major): unit j of replica r lives at
 * bufs[bufs[r*n_units+j]] + offs[r*n_units+j] (elements). */
int ntp_mplan_add_units(ntp_mplan *plan, int64_t n_units, int64_t unit_elems, const int32_t *bufs,
                        const int64_t *offs);
int ntp_mplan_finalize(ntp_mplan *plan);
int64_t ntp_mplan_chunks(const ntp_mplan *plan);
int ntp_mplan_upload(ntp_mplan *plan, int device);
void ntp_mplan_destroy(ntp_mplan *plan);
/* Every unit ends as op over its R copies (SUM in replica order, true MEAN, or
 * sum_r w[r]*x_r), written to all R owners; one read and one write per copy. */
int ntp_multi_sync(const ntp_mplan *plan, void *const *bufs, int n_bufs, int op, const double *w,
                   void *stream);
/* Kernel for ntp_multi_sync: 0 AUTO (TMA-bulk shared-memory ring for R <= 4,
 * >= 2 chunks per SM and at least one peer-mapped copy; else 128-bit loads),
 * 1 loads, 2 bulk (R <= 4).  Both give identical bits. */
int ntp_multi_set_kernel(int variant);

/* ------------------------------------------------------------------------
 * Uneven-shard linears on tcgen05 tensor cores (bf16 in, fp32 accumulate)
 * ------------------------------------------------------------------------ */

enum ntp_gemm_epilogue {
  NTP_EPI_NONE = 0,  /* C = alpha * acc                                            */
  NTP_EPI_GELU = 1,  /* aux = bf16(alpha*acc) (pre-activation H); C = GeLU(aux)    */
  NTP_EPI_DGELU = 2  /* C = alpha * acc * GeLU'(aux)   (aux = H, backward)         */
};

/* C[M x N] = epilogue(sum_k A[m,k] * B[n,k]) -- the per-rank GEMMs of
 * mlp_forward_tp / mlp_backward_tp (tpnumerics.py:177-185, 238-252) with
 * ragged M/N/K (n_i = 4779, 1366, ...).  A is [M x K]: a_mn = 0 -> stored
 * row-major [M][lda] (K contiguous), a_mn = 1 -> stored [K][lda] (M
 * contiguous).  B likewise for [N x K] with b_mn.  C is row-major [M][ldc]
 * (bf16, or fp32 if c_f32); ldc may exceed N, e.g. 2*hidden to write the
 * unit-major gradient arena directly.  A, B, aux: bf16, 16-byte aligned
 * bases and row pitches.  Stream-ordered. */
int ntp_gemm_bf16(const void *A, int64_t lda, int a_mn, const void *B, int64_t ldb, int b_mn,
                  void *C, int64_t ldc, int c_f32, int64_t M, int64_t N, int64_t K, int epilogue,
                  const void *aux, int64_t ld_aux, float alpha, void *stream);

/* ntp_gemm_bf16 with an explicit programmatic-dependent-launch mode:
 * pdl 0: ordinary stream order.  1: launched early; waits for the previous
 * kernel of the stream before touching global memory, so its set-up overlaps
 * that kernel's tail.  2: the caller guarantees this GEMM neither reads what
 * the previous kernel writes nor writes what it reads or writes; it runs
 * under the previous kernel's tail and does not complete before it. */
int ntp_gemm_bf16_ex(const void *A, int64_t lda, int a_mn, const void *B, int64_t ldb, int b_mn,
                     void *C, int64_t ldc, int c_f32, int64_t M, int64_t N, int64_t K,
                     int epilogue, const void *aux, int64_t ld_aux, float alpha, int pdl,
                     void *stream);

/* Fused weight-gradient GEMM + NTP gradient sync: the epilogue adds
 * alpha * acc (this replica's batch-weighted gradient) with red.add into the
 * local row m of C AND into row red_row[m] of the partner replica's copy
 * red_base[red_buf[m]] (local or peer-mapped; red_buf[m] < 0: no partner).
 * Both copies must start at zero; since each unit receives exactly two
 * contributions and a two-term floating-point sum commutes, both replicas end
 * with identical bits -- nonuniform_grad_sync (tpnumerics.py:289-356) done
 * inside the producer of the gradients, with no separate sync kernel.
 * red_buf/red_row are device int32[M]; N % 32 == 0; 16-byte aligned rows.
 * mode 0: red.add into zeroed arenas as above.  mode 1 (push): plain stores of
 * the weighted tile into the local arena and into the partner's *staging*
 * arena (red_base); after the done handshake each side adds its staging into
 * its arena (ntp_grad_sync_ex with write mask 1) -- no remote atomics.
 * mode 2 (push, TMA): as mode 1, but each 32-row output box whose rows are
 * consecutive rows of one partner copy is sent as one TMA tensor store over
 * NVLink from the same shared-memory staging as the local store; other boxes
 * (run boundaries, ragged tails) fall back to row stores.
 * mode 3 (red, TMA): as mode 0 (zeroed arenas), but every box is added with
 * TMA bulk tensor reductions (cp.reduce.async.bulk.tensor .add) into the
 * local copy and the partner copy; row red.adds where a box's rows are not
 * consecutive in the partner's layout. */
int ntp_gemm_bf16_red(const void *A, int64_t lda, int a_mn, const void *B, int64_t ldb, int b_mn,
                      void *C, int64_t ldc, int c_f32, int64_t M, int64_t N, int64_t K,
                      float alpha, const int32_t *red_buf, const int32_t *red_row,
                      void *const *red_base, int n_red, int64_t red_ld, int mode, void *stream);

/* Tile selection: 1 (default) AUTO -- 256 x 256 CTA-pair tiles (tcgen05
 * cta_group::2, cluster of 2) unless 256 x 128 pair tiles halve the waves;
 * 2 force 256 x 128 pair tiles; 3 force 256 x 256; 4 force 256 x 224
 * (K-major B; else 256 x 256; measured slower on the C4 shapes); 0 single-CTA
 * 128 x 256. */
int ntp_gemm_set_pair(int mode);

/* Cap on the persistent GEMM's CTAs (0 = every SM).  With a sync kernel capped
 * to c CTAs (NTP_OPT_SYNC_MAX_CTAS), a GEMM cap of SMs - c lets the two run
 * side by side when the sync overlaps the backward pass. */
int ntp_gemm_set_max_ctas(int n);
/* The current cap (so a caller that changes it can restore it). */
int ntp_gemm_get_max_ctas(void);

/* 1 (default): when the persistent schedule ends in a partial wave of R tiles,
 * those tiles are split along K into up to 8 pieces run by idle CTA pairs; fp32
 * partials meet in a per-stream workspace; the pieces share the final sums
 * (in piece order, deterministic) and epilogues by atomically claimed column
 * chunks, and the last piece to arrive takes every unclaimed chunk -- no piece
 * ever waits for one that is not running.
 * n >= 2: at most n pieces per tile.  0: whole tiles only.  NTP_EINVAL
 * outside [0, 64]. */
int ntp_gemm_set_split_k(int on);

/* 1: every ntp_gemm_bf16 / ntp_gemm_bf16_red launch uses programmatic
 * dependent launch mode 1 (see ntp_gemm_bf16_ex).  0 (default): off. */
int ntp_gemm_set_pdl(int on);

/* ------------------------------------------------------------------------
 * Multi-GPU plumbing: peer memory over NVLink/NVSwitch and device signals
 * ------------------------------------------------------------------------ */

#define NTP_IPC_HANDLE_BYTES 64

/* Device arena for gradients shared with peers (cudaMalloc'd so it can be
 * exported with CUDA IPC).  Free with ntp_free. */
int ntp_alloc(int device, int64_t bytes, void **out);
int ntp_free(void *ptr);
int ntp_ipc_get_handle(void *dev_ptr, void *handle_out);
int ntp_ipc_open(int device, const void *handle, void **dev_ptr_out);
int ntp_ipc_close(void *dev_ptr);

/* One-sided signalled sync (push design): the computing GPU
 *   1. waits until every signal word in wait[n_wait] (local memory, written
 *      by peers with release semantics) is >= epoch,
 *   2. runs the plan like ntp_grad_sync (reading and writing peer memory),
 *   3. after all its CTAs finish, stores epoch (release, .sys scope) to every
 *      word in post[n_post] (peer memory).
 * spin_ns bounds each wait; on timeout the kernel records NTP_ETIMEOUT in
 * *status (device int) and exits instead of hanging. */
int ntp_grad_sync_signaled(const ntp_plan *plan, void *const *bufs, int n_bufs, int op,
                           double w_a, double w_b, uint64_t *const *wait, int n_wait,
                           uint64_t *const *post, int n_post, uint64_t epoch,
                           uint64_t spin_ns, int *status, void *stream);

/* One whole synchronisation step in a single launch (the three launches of
 * ntp_signal_post + ntp_grad_sync_signaled + ntp_signal_wait folded together):
 * post epoch to post_ready[] (this process's buffers may be touched), wait for
 * wait_ready[], run the plan, post post_done[] after every CTA has finished,
 * then wait for wait_done[] (the partners finished touching this process's
 * buffers) before the launch completes.  plan may be NULL (nothing to compute
 * here: only the handshakes run).  Replaces one call of the reference's
 * nonuniform_grad_sync (tpnumerics.py:289-356) across processes. */
int ntp_grad_sync_step(const ntp_plan *plan, void *const *bufs, int n_bufs, int op, double w_a,
                       double w_b, uint64_t *const *post_ready, int n_post_ready,
                       uint64_t *const *wait_ready, int n_wait_ready,
                       uint64_t *const *post_done, int n_post_done,
                       uint64_t *const *wait_done, int n_wait_done, uint64_t epoch,
                       uint64_t spin_ns, int *status, void *stream);

/* Store epoch to each word in post[] (release, .sys) from a 1-thread kernel. */
int ntp_signal_post(uint64_t *const *post, int n_post, uint64_t epoch, void *stream);

/* Block the stream until every word in wait[] is >= epoch (bounded spin). */
int ntp_signal_wait(uint64_t *const *wait, int n_wait, uint64_t epoch, uint64_t spin_ns,
                    int *status, void *stream);

/* Device-resident epochs: the same four calls with the epoch read on the
 * device from *epoch_word (a u64 in device memory counting the completed
 * steps; this launch uses *epoch_word + 1), so a step recorded once into a
 * CUDA graph can be replayed step after step with no host involvement.  The
 * step's final launch advances the word: ntp_grad_sync_step_dev always,
 * ntp_signal_wait_dev when advance != 0 (the done-wait of a three-launch
 * step); the post and signalled-sync launches only read it. */
int ntp_grad_sync_signaled_dev(const ntp_plan *plan, void *const *bufs, int n_bufs, int op,
                               double w_a, double w_b, uint64_t *const *wait, int n_wait,
                               uint64_t *const *post, int n_post, uint64_t *epoch_word,
                               uint64_t spin_ns, int *status, void *stream);
int ntp_grad_sync_step_dev(const ntp_plan *plan, void *const *bufs, int n_bufs, int op,
                           double w_a, double w_b, uint64_t *const *post_ready, int n_post_ready,
                           uint64_t *const *wait_ready, int n_wait_ready,
                           uint64_t *const *post_done, int n_post_done,
                           uint64_t *const *wait_done, int n_wait_done, uint64_t *epoch_word,
                           uint64_t spin_ns, int *status, void *stream);
int ntp_signal_post_dev(uint64_t *const *post, int n_post, uint64_t *epoch_word, void *stream);
int ntp_signal_wait_dev(uint64_t *const *wait, int n_wait, uint64_t *epoch_word, int advance,
                        uint64_t spin_ns, int *status, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* NTP_B200_H */
