// Definitions shared by the decode-attention kernels (paged_decode_attn.cu:
// the stream-K persistent grid; decode_split.cu: the split-pair CTA kernel for
// small calls): page geometry, launch arguments, tuning constants.
#pragma once

#include "adr_internal.h"

namespace adr {
namespace dec {

constexpr int kPage = 16;                  // tokens per page (block_size)
constexpr int kTileBytes = kPage * 128;    // one 16-row x 64-col bf16 half page
constexpr int kMaxWarpsPerSm = 16;         // workspace sizing bound over all variants
constexpr int kChunksPerWarp = 12;         // chunk grid: at most this many chunks per grid warp
constexpr int kMinChunk = 16;              // units per chunk, lower bound
constexpr int kMinChunkSmall = 8;          // ... when that shortens the per-warp path (Chunks)
constexpr int kStaticMaxChunk = 32;        // static grid (one chunk per warp) up to this chunk size
constexpr int kClaimAhead = 4;             // claim the next chunk this many units before the end
constexpr int kSpinNs = 256;               // merge-task poll back-off
constexpr int kPrefetchUnits = 8;          // default pages of its chunk-to-be a warp warms L2 with (sweep: 8 > 4, 12 > 0, 16)
constexpr long long kMaxPairs = 1 << 17;   // (request, kv-head) counters in the workspace
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kNegBig = -1.0e30f;

#ifdef ADR_TIMELINE
// Diagnostic build only (scripts/timeline.py): per-warp globaltimer stamps of
// the last launch — entry, before the dependency wait, after it, first page
// landed, chunk stream exhausted, merge phase done.
constexpr int kTlWarps = 4096, kTlPoints = 12;
__device__ unsigned long long g_timeline[kTlWarps][kTlPoints];
__device__ __forceinline__ unsigned long long tl_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define ADR_TL(k)                                                                   \
  do {                                                                              \
    const int tlw = (threadIdx.x >> 5) * gridDim.x + blockIdx.x;                    \
    if ((threadIdx.x & 31) == 0 && tlw < kTlWarps) g_timeline[tlw][k] = tl_now();   \
  } while (0)
#else
#define ADR_TL(k) \
  do {            \
  } while (0)
#endif

struct DecodeArgs {
  const __nv_bfloat16* q;
  const __nv_bfloat16* k_new;  // fused append (nullable): [B, Hkv, D] token at seq_len - 1
  const __nv_bfloat16* v_new;
  __nv_bfloat16* k_cache;      // written only by the fused append
  __nv_bfloat16* v_cache;
  const int32_t* block_table;
  const int32_t* seq_lens;
  void* out;
  float* lse;
  float* part;       // 2 slots per chunk, slot_floats each
  int32_t* counter;  // [B*Hkv] arrivals per split pair (zero between calls)
  int32_t* claim;    // [0] next dynamic chunk, [1] warps done, [2] next merge task (zero between calls)
  int32_t* status;   // ADR_STATUS_* bits of rejected input (sticky; read by adr_decode_status)
  // Row maps (nullable): request b reads q / k_new / v_new row in_rows[b] and
  // writes out / lse row out_rows[b]. With peer pointers this is the zero-copy
  // offload: an executor kernel reads the decode GPU's q/k/v rows and writes
  // its outputs straight into the decode GPU's rows over NVLink.
  const int32_t* in_rows;
  const int32_t* out_rows;
  int B, Hq, Hkv, G, max_blocks, num_blocks, out_f32, slot_floats;
  int min_chunk, chunks_per_warp, split_rule;  // chunk grid knobs (tuning; see Chunks)
  int prefetch_units;                          // L2 warm-up pages per chunk (<= 32)
  int static_mode;                             // 0 never, 1 small calls, 2 always (tests)
  int static_min;                              // static-grid chunk floor (0: kMinChunkSmall)
  int pdl;                                     // launched with programmatic dependent launch
  int part_slots;                              // partial slots in the workspace (split kernel)
  int split_item_cost;                         // split kernel: fixed cost of an item, in pages per warp
  int split_force_k;                           // split kernel: > 0 forces k runs per longest pair (tuning)
  int split_dynamic;                           // split kernel items: 0 static, 1 claimed, 2 by the path model
  int split_dyn_cost;                          // split kernel: claimed item cost, pages per warp
  int split_merge_cost;                        // split kernel: merge of a split pair, pages per warp
  float scale_log2;
};

template <int D>
struct Geometry {
  static constexpr int kHalves = D / 64;
  static constexpr int kStageBytes = 2 * kHalves * kTileBytes;  // K + V
  static constexpr int kKSteps = D / 16;                         // QK MMAs per page
  static constexpr int kMTiles = D / 16;                         // PV m-tiles per page
};


__device__ __forceinline__ int upper_bound_smem(const int32_t* a, int n, int key) {
  // first index i in [0, n) with a[i] > key (a non-decreasing)
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] <= key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Floats per partial slot: acc [G][D] | m[8] | l[8], rounded up to whole
// 128-byte lines so a merged row can be discarded from L2 line by line.
inline int slot_floats(int G, int D) { return (G * D + 16 + 31) / 32 * 32; }

}  // namespace dec
}  // namespace adr
