// Internal declarations shared by the planner (host C++) and the CUDA side.
#pragma once

#include <atomic>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/ntp_b200.h"

namespace ntp {

// Per-thread last error (ntp_last_error()).
void set_error(const std::string &msg);
int fail(int status, const std::string &msg);

inline int dtype_bytes(int dtype) {
  switch (dtype) {
    case NTP_F32: return 4;
    case NTP_BF16: return 2;
    case NTP_F16: return 2;
    case NTP_F64: return 8;
    default: return 0;
  }
}

// One device work item: 16 bytes, loaded with a single 128-bit load.
// Offsets and length are in "grains": 16-byte vectors for a vectorized plan,
// single elements otherwise.
struct Chunk {
  uint32_t a_off;
  uint32_t b_off;
  uint32_t len;   // grains
  uint16_t a_buf;
  uint16_t b_buf;
};
static_assert(sizeof(Chunk) == 16, "chunk record must be 16 bytes");

// Grains per chunk: 1024 x 16 B = 16 KiB per side for the vector path.
constexpr uint32_t kChunkVecs = 1024;
constexpr uint32_t kChunkElems = 4096;  // scalar path
// NTP_OPT_PLAN_MIN_CHUNKS (default 1184 = 8 per SM): plans finalized while
// this is > 0 shrink their chunks (down to 64 grains) so the plan has at least
// this many -- small plans then spread over every SM several times, which
// shortens the tail.
extern std::atomic<int64_t> g_min_chunks;

constexpr int kMaxBufs = 64;

struct Run {
  int32_t a_buf, b_buf;
  int64_t a_off, b_off, len;  // elements
};

}  // namespace ntp

struct ntp_plan {
  int dtype = NTP_F32;
  bool finalized = false;
  bool vectorized = false;
  int64_t n_units = 0;
  int64_t elems = 0;
  int32_t max_buf = -1;
  std::vector<ntp::Run> runs;      // merged, in insertion order
  std::vector<ntp::Chunk> chunks;  // host table
  ntp::Chunk *d_chunks = nullptr;  // device table
  unsigned int *d_counter = nullptr;  // CTA completion counter (signalled launches)
  int device = -1;
};

// CUDA-side helpers implemented in ntp_sync.cu.
namespace ntp {
int device_free(void *p, int device);
}
