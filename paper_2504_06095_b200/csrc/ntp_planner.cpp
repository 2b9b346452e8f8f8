// Host-side planner: the reference's shard algebra (shardmap.py) and the
// builder of device copy/reduce plans.  Integer work only; bit-exact with the
// reference (tests/test_planner.py pins it against tests/golden/).
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "ntp_internal.h"

namespace ntp {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }

std::atomic<int64_t> g_min_chunks{1184};  // 8 per SM of a B200 (measured: scripts/sweep.py)

int fail(int status, const std::string &msg) {
  set_error(msg);
  return status;
}

// _balanced_sizes, shardmap.py:23-27: remainder to the lowest ranks.
static inline int64_t balanced_size(int64_t k, int64_t n, int64_t i) {
  return k / n + (i < k % n ? 1 : 0);
}
static inline int64_t balanced_start(int64_t k, int64_t n, int64_t i) {
  int64_t q = k / n, r = k % n;
  return i * q + std::min(i, r);
}

// _validate_triple, shardmap.py:132-138, same ValueError texts.
static int validate_triple(int64_t k, int64_t n1, int64_t n2) {
  char buf[256];
  if (k <= 0 || n1 <= 0 || n2 <= 0) {
    snprintf(buf, sizeof buf, "k, n1, n2 must be positive, got (%lld, %lld, %lld)",
             (long long)k, (long long)n1, (long long)n2);
    return fail(NTP_EINVAL, buf);
  }
  if (n2 > n1) {
    snprintf(buf, sizeof buf, "reduced degree n2=%lld exceeds healthy degree n1=%lld",
             (long long)n2, (long long)n1);
    return fail(NTP_EINVAL, buf);
  }
  if (n1 > k) {
    snprintf(buf, sizeof buf, "TP degree n1=%lld exceeds partition size k=%lld", (long long)n1,
             (long long)k);
    return fail(NTP_EINVAL, buf);
  }
  return NTP_OK;
}

}  // namespace ntp

using namespace ntp;

extern "C" {

const char *ntp_last_error(void) { return g_last_error.c_str(); }
int ntp_abi_version(void) { return NTP_ABI_VERSION; }

// build_shard_map, shardmap.py:141-182, in closed form: sync shard i is the
// balanced contiguous block [s_i, s_i + z_i) over n2 ranks; it keeps its
// first m_i = min(cap_i, z_i) columns (cap_i = balanced size over n1); the
// offloaded columns, enumerated in global order (idx), go to n2 + idx % (n1-n2).
// The enumeration index of an offloaded column is O_i + (q - m_i), O_i being
// the number of columns offloaded by shards 0..i-1, so every column is placed
// independently of the others.
int ntp_shard_map(int64_t k, int64_t n1, int64_t n2, int64_t *comp_rank, int64_t *sync_rank) {
  int st = validate_triple(k, n1, n2);
  if (st) return st;
  const int64_t n_off = n1 - n2;
  int64_t offloaded_before = 0;
  for (int64_t i = 0; i < n2; ++i) {
    const int64_t s = balanced_start(k, n2, i), z = balanced_size(k, n2, i);
    const int64_t m = std::min(balanced_size(k, n1, i), z);
    if (z > m && n_off == 0)  // unreachable for valid triples (shardmap.py:175-178)
      return fail(NTP_EINVAL, "offloaded columns with no offload ranks");
    for (int64_t q = 0; q < z; ++q) {
      sync_rank[s + q] = i;
      comp_rank[s + q] = q < m ? i : n2 + (offloaded_before + q - m) % n_off;
    }
    offloaded_before += z - m;
  }
  return NTP_OK;
}

// build_reshard_plan, shardmap.py:185-206: stable counting sort of the moving
// columns on the ordered (src, dst) link.
int64_t ntp_reshard_plan(const int64_t *comp, const int64_t *sync, int64_t k, int64_t n1,
                         int direction, int64_t *src, int64_t *dst, int64_t *col) {
  if (direction != NTP_PRE_SYNC && direction != NTP_POST_SYNC)
    return fail(NTP_EINVAL, "direction must be 'pre_sync' or 'post_sync'");
  if (k < 0 || n1 <= 0) return fail(NTP_EINVAL, "bad plan arguments");
  std::vector<int64_t> start((size_t)(n1 * n1) + 1, 0);
  for (int64_t j = 0; j < k; ++j) {
    if (comp[j] == sync[j]) continue;
    if (comp[j] < 0 || comp[j] >= n1 || sync[j] < 0 || sync[j] >= n1)
      return fail(NTP_EINVAL, "rank out of range in shard map");
    const int64_t s = direction == NTP_PRE_SYNC ? comp[j] : sync[j];
    const int64_t d = direction == NTP_PRE_SYNC ? sync[j] : comp[j];
    ++start[(size_t)(s * n1 + d) + 1];
  }
  for (size_t i = 1; i < start.size(); ++i) start[i] += start[i - 1];
  const int64_t total = start.back();
  for (int64_t j = 0; j < k; ++j) {
    if (comp[j] == sync[j]) continue;
    const int64_t s = direction == NTP_PRE_SYNC ? comp[j] : sync[j];
    const int64_t d = direction == NTP_PRE_SYNC ? sync[j] : comp[j];
    const int64_t at = start[(size_t)(s * n1 + d)]++;
    src[at] = s;
    dst[at] = d;
    col[at] = j;
  }
  return total;
}

// apply_plan, shardmap.py:209-217.  The reference checks a whole transfer
// before writing it; columns are unique within a plan, so checking each
// (src, dst, col) triple in order before its write is equivalent.
int ntp_apply_plan(int64_t *own, int64_t k, const int64_t *src, const int64_t *dst,
                   const int64_t *col, int64_t n) {
  for (int64_t t = 0; t < n; ++t) {
    if (col[t] < 0 || col[t] >= k || own[col[t]] != src[t]) {
      char buf[160];
      snprintf(buf, sizeof buf, "transfer %lld->%lld names columns not owned by %lld",
               (long long)src[t], (long long)dst[t], (long long)src[t]);
      return fail(NTP_EINVAL, buf);
    }
    own[col[t]] = dst[t];
  }
  return NTP_OK;
}

// naive_contiguous_sync_volumes, shardmap.py:220-245, as a two-pointer merge
// of the two sets of balanced interval bounds.
int64_t ntp_naive_overlaps(int64_t k, int64_t n1, int64_t n2, int64_t *pairs,
                           int64_t *per_reduced) {
  int st = validate_triple(k, n1, n2);
  if (st) return st;
  int64_t total = 0, h = 0;
  for (int64_t i = 0; i < n2; ++i) {
    const int64_t lo = balanced_start(k, n2, i), hi = lo + balanced_size(k, n2, i);
    per_reduced[i] = 0;
    while (h < n1 && balanced_start(k, n1, h) + balanced_size(k, n1, h) <= lo) ++h;
    for (int64_t g = h; g < n1; ++g) {
      const int64_t a = balanced_start(k, n1, g), b = a + balanced_size(k, n1, g);
      if (a >= hi) break;
      const int64_t ov = std::min(hi, b) - std::max(lo, a);
      if (ov > 0) {
        pairs[2 * total] = g;
        pairs[2 * total + 1] = ov;
        ++total;
        ++per_reduced[i];
      }
    }
  }
  return total;
}

int64_t ntp_interval_overlaps(int64_t k, int64_t n_src, int64_t n_dst, int64_t *quads) {
  if (k <= 0 || n_src <= 0 || n_dst <= 0 || n_src > k || n_dst > k)
    return fail(NTP_EINVAL, "interval overlaps need 0 < n_src, n_dst <= k");
  int64_t total = 0, s = 0, d = 0, pos = 0;
  while (pos < k) {
    const int64_t s_end = balanced_start(k, n_src, s) + balanced_size(k, n_src, s);
    const int64_t d_end = balanced_start(k, n_dst, d) + balanced_size(k, n_dst, d);
    const int64_t end = std::min(s_end, d_end);
    if (end > pos) {
      quads[4 * total + 0] = s;
      quads[4 * total + 1] = d;
      quads[4 * total + 2] = pos;
      quads[4 * total + 3] = end - pos;
      ++total;
    }
    pos = end;
    if (s_end == end) ++s;
    if (d_end == end) ++d;
  }
  return total;
}

// attention_head_partition, shardmap.py:248-260.
int ntp_head_partition(int64_t heads, int64_t n, int64_t *counts, double *imbalance) {
  char buf[160];
  if (heads <= 0 || n <= 0) {
    snprintf(buf, sizeof buf, "heads and n must be positive, got (%lld, %lld)",
             (long long)heads, (long long)n);
    return fail(NTP_EINVAL, buf);
  }
  if (n > heads) {
    snprintf(buf, sizeof buf, "TP degree n=%lld exceeds head count %lld", (long long)n,
             (long long)heads);
    return fail(NTP_EINVAL, buf);
  }
  int64_t mx = 0;
  for (int64_t i = 0; i < n; ++i) {
    counts[i] = balanced_size(heads, n, i);
    mx = std::max(mx, counts[i]);
  }
  *imbalance = (double)mx / ((double)heads / (double)n);
  return NTP_OK;
}

// ---------------------------------------------------------------------------
// copy/reduce plans

int ntp_plan_create(ntp_plan **out, int dtype) {
  if (!out) return fail(NTP_EINVAL, "null plan pointer");
  if (dtype_bytes(dtype) == 0) return fail(NTP_EINVAL, "unsupported dtype");
  ntp_plan *p = new (std::nothrow) ntp_plan();
  if (!p) return fail(NTP_ENOMEM, "out of host memory");
  p->dtype = dtype;
  *out = p;
  return NTP_OK;
}

int ntp_plan_add_units(ntp_plan *p, int64_t n_units, int64_t unit_elems, const int32_t *a_buf,
                       const int64_t *a_off, const int32_t *b_buf, const int64_t *b_off) {
  if (!p) return fail(NTP_EINVAL, "null plan");
  if (p->finalized) return fail(NTP_ESTATE, "plan already finalized");
  if (n_units < 0 || unit_elems <= 0) return fail(NTP_EINVAL, "bad unit count or size");
  for (int64_t j = 0; j < n_units; ++j) {
    const int32_t ab = a_buf[j], bb = b_buf[j];
    if (ab < 0 || ab >= kMaxBufs || bb < 0 || bb >= kMaxBufs)
      return fail(NTP_EINVAL, "buffer index out of range (max 64 buffers)");
    if (a_off[j] < 0 || b_off[j] < 0) return fail(NTP_EINVAL, "negative offset");
    p->max_buf = std::max(p->max_buf, std::max(ab, bb));
    if (!p->runs.empty()) {
      Run &r = p->runs.back();
      if (r.a_buf == ab && r.b_buf == bb && r.a_off + r.len == a_off[j] &&
          r.b_off + r.len == b_off[j]) {
        r.len += unit_elems;
        continue;
      }
    }
    p->runs.push_back(Run{ab, bb, a_off[j], b_off[j], unit_elems});
  }
  p->n_units += n_units;
  p->elems += n_units * unit_elems;
  return NTP_OK;
}

int ntp_plan_finalize(ntp_plan *p) {
  if (!p) return fail(NTP_EINVAL, "null plan");
  if (p->finalized) return NTP_OK;
  const int64_t vec = 16 / dtype_bytes(p->dtype);
  bool vectorized = true;
  for (const Run &r : p->runs)
    if (r.a_off % vec || r.b_off % vec || r.len % vec) vectorized = false;
  const int64_t grain = vectorized ? vec : 1;
  int64_t chunk = vectorized ? kChunkVecs : kChunkElems;
  const int64_t min_chunks = g_min_chunks.load();
  if (min_chunks > 0) {
    // the target is set in elements, a multiple of 8, so plans over the same
    // units split identically in every dtype (grains are 2, 4 or 8 elements)
    int64_t elems = 0;
    for (const Run &r : p->runs) elems += r.len;
    const int64_t target = std::max<int64_t>(512, elems / min_chunks / 8 * 8);
    if (target / grain < chunk) chunk = target / grain;
  }
  p->chunks.clear();
  for (const Run &r : p->runs) {
    const int64_t g = r.len / grain;
    const int64_t pieces = (g + chunk - 1) / chunk;
    // split on 8-element boundaries when the run allows it, so the same units
    // cut at the same elements in every dtype (grains are 2, 4 or 8 elements)
    const int64_t q = (vectorized && r.len % 8 == 0) ? 8 / grain : 1;
    const int64_t gq = g / q;
    for (int64_t c = 0; c < pieces; ++c) {
      // near-equal pieces so a long run does not leave a tiny tail chunk
      const int64_t lo = gq * c / pieces * q, hi = gq * (c + 1) / pieces * q;
      if (hi <= lo) continue;
      const int64_t ao = r.a_off / grain + lo, bo = r.b_off / grain + lo;
      if (ao + (hi - lo) > UINT32_MAX || bo + (hi - lo) > UINT32_MAX)
        return fail(NTP_EINVAL, "buffer offset exceeds the 32-bit grain range of a plan");
      p->chunks.push_back(Chunk{(uint32_t)ao, (uint32_t)bo, (uint32_t)(hi - lo),
                                (uint16_t)r.a_buf, (uint16_t)r.b_buf});
    }
  }
  p->vectorized = vectorized;
  p->finalized = true;
  return NTP_OK;
}

int ntp_plan_stats_get(const ntp_plan *p, ntp_plan_stats *s) {
  if (!p || !s) return fail(NTP_EINVAL, "null argument");
  s->n_units = p->n_units;
  s->n_runs = (int64_t)p->runs.size();
  s->n_chunks = (int64_t)p->chunks.size();
  s->elems = p->elems;
  s->vectorized = p->vectorized ? 1 : 0;
  s->max_buf = p->max_buf;
  s->dtype = p->dtype;
  s->device = p->device;
  return NTP_OK;
}

int ntp_plan_export(const ntp_plan *p, int64_t *out) {
  if (!p || !out) return fail(NTP_EINVAL, "null argument");
  if (!p->finalized) return fail(NTP_ESTATE, "plan not finalized");
  const int64_t grain = p->vectorized ? 16 / dtype_bytes(p->dtype) : 1;
  for (size_t i = 0; i < p->chunks.size(); ++i) {
    const Chunk &c = p->chunks[i];
    out[5 * i + 0] = c.a_buf;
    out[5 * i + 1] = (int64_t)c.a_off * grain;
    out[5 * i + 2] = c.b_buf;
    out[5 * i + 3] = (int64_t)c.b_off * grain;
    out[5 * i + 4] = (int64_t)c.len * grain;
  }
  return NTP_OK;
}

int ntp_plan_check(const ntp_plan *p, const int64_t *buf_elems, int n_bufs, int write_sides) {
  if (!p || (!buf_elems && n_bufs)) return fail(NTP_EINVAL, "null argument");
  if (!p->finalized) return fail(NTP_ESTATE, "plan not finalized");
  if (write_sides < 0 || write_sides > 3) return fail(NTP_EINVAL, "write_sides must be 0..3");
  const int64_t grain = p->vectorized ? 16 / dtype_bytes(p->dtype) : 1;
  struct Range {
    int64_t buf, lo, hi, chunk;
  };
  std::vector<Range> writes;
  writes.reserve(2 * p->chunks.size());
  for (size_t i = 0; i < p->chunks.size(); ++i) {
    const Chunk &c = p->chunks[i];
    const int64_t len = (int64_t)c.len * grain;
    const int64_t side_buf[2] = {c.a_buf, c.b_buf};
    const int64_t side_off[2] = {(int64_t)c.a_off * grain, (int64_t)c.b_off * grain};
    for (int side = 0; side < 2; ++side) {
      const int64_t b = side_buf[side], lo = side_off[side];
      if (b >= n_bufs)
        return fail(NTP_EINVAL, "chunk " + std::to_string(i) + " uses buffer " + std::to_string(b) +
                                    " of " + std::to_string(n_bufs));
      if (lo + len > buf_elems[b])
        return fail(NTP_EINVAL, "chunk " + std::to_string(i) + ": buffer " + std::to_string(b) +
                                    " elements [" + std::to_string(lo) + ", " +
                                    std::to_string(lo + len) + ") exceed its " +
                                    std::to_string(buf_elems[b]));
      if (write_sides & (1 << side)) writes.push_back(Range{b, lo, lo + len, (int64_t)i});
    }
  }
  // every element is written by one chunk at most: no two CTAs race on it
  std::sort(writes.begin(), writes.end(), [](const Range &x, const Range &y) {
    return x.buf != y.buf ? x.buf < y.buf : x.lo < y.lo;
  });
  for (size_t i = 1; i < writes.size(); ++i)
    if (writes[i].buf == writes[i - 1].buf && writes[i].lo < writes[i - 1].hi)
      return fail(NTP_EINVAL, "chunks " + std::to_string(writes[i - 1].chunk) + " and " +
                                  std::to_string(writes[i].chunk) + " write overlapping elements of buffer " +
                                  std::to_string(writes[i].buf));
  return NTP_OK;
}

void ntp_plan_destroy(ntp_plan *p) {
  if (!p) return;
  if (p->d_chunks) device_free(p->d_chunks, p->device);
  if (p->d_counter) device_free(p->d_counter, p->device);
  delete p;
}

}  // extern "C"
