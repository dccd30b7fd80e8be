// Paged decode attention for sm_100a.
//
// What it computes (the real work priced by costs.attention_step_latency,
// costs.py:73-80): for each request b, q-head h,
//     out[b,h] = softmax(scale * q[b,h] . K_b^T) . V_b   over seq_lens[b] tokens
// with K/V paged in 16-token pages [num_blocks, Hkv, 16, D] bf16 and GQA
// grouping (q-head h reads kv-head h / G, G = Hq/Hkv <= 8).
//
// Design (B200-first):
//  * Work unit = one page of one (request, kv-head) pair: 16 tokens x D x {K,V}
//    (8 KiB at D=128). Units are flattened in (request, kv-head, page) order and
//    cut into a fixed grid of equal power-of-two chunks (16..64 units at the
//    BASELINE shapes). Warps of a persistent grid CLAIM chunks from a global
//    counter: HBM serves SMs unevenly (a static equal split left warps finishing
//    up to 250 us apart in a 600 us call), so fast warps simply take more chunks
//    and every warp finishes within a chunk of the others. No chunk is owned in
//    advance, so a warp that never gets an SM leaves nothing undone. The chunk
//    grid, not the claim order, fixes every partial's slot and the merge order,
//    so results stay bit-identical from run to run.
//  * Each warp is an independent producer/consumer: lane 0 issues TMA tile loads
//    (cp.async.bulk.tensor, 128B-swizzled, L2 evict-first) of the K and V page
//    halves into a private kStages-deep smem ring guarded by mbarriers; the warp
//    consumes the ring with ldmatrix + mma.sync m16n8k16 (bf16 in, fp32 acc):
//      S^T[16 tok x 8 heads] = K[16 x D] . Q^T[D x 8]     (D/16 MMAs)
//      O^T[D x 8 heads]     += V^T[D x 16] . P^T[16 x 8]   (2 x D/16 MMAs:
//                                         P split into bf16 hi + lo parts)
//    The 8 MMA columns carry the G q-heads of the kv-head (padding columns are
//    zero). P^T is rebuilt from the S^T accumulator with movmatrix.trans, so no
//    shared-memory round trip is needed between the two MMAs.
//  * Online softmax in the log2 domain per (warp, head). A pair inside one chunk
//    is normalised and written directly. A pair cut by chunk boundaries leaves
//    fp32 partials (acc [G][D], m, l) in the workspace, one slot per piece,
//    announced with a release increment of the pair's arrival counter (no
//    round trip). Warps whose chunk stream is exhausted take (request, q-head)
//    merge tasks: wait for the pair's pieces (acquire), then max / sum over the
//    pieces lane-parallel and each lane accumulates its 4 dims in chunk order —
//    deterministic, in the same kernel, counters self-cleaning. Merged rows are
//    discarded from L2 (dead scratch would otherwise be written back behind
//    the grid's last warp), and the merge code is kept compact: it runs once
//    per warp at the end of the call, when it is no longer in the i-cache.
//  * Small calls use a static grid instead (Chunks::stat): one chunk per warp,
//    no claims, the first TMA loads issued before the dependency wait, and the
//    warp publishing a pair's last piece merges all its heads (no merge phase,
//    no waiting, hence no deadlock if some CTAs start late).
//  * The step's new K/V row can be appended in the same pass (fused append): the
//    warp owning a pair's last page patches the row into its smem tile and
//    writes it to the cache.
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <type_traits>

#include "decode_common.cuh"

namespace adr {

namespace {

using namespace dec;

// Fixed chunk grid over the U units: chunk c = [c*CH, min(U, (c+1)*CH)).
// A pair cut by the grid leaves one partial per chunk it touches, in slot
// 2c (the chunk's leading piece, or the whole chunk) or 2c + 1 (a piece that
// starts inside the chunk and runs past its end).
// CH >= 16 (8 for small problems) and >= ~sqrt(0.6 x mean pair length): small problems would otherwise
// cut every pair into many pieces and make the merge (one partial read per
// piece) the critical path; and at most kChunksPerWarp chunks per grid warp
// (bounds the workspace).
struct Chunks {
  const int32_t* cu;
  int Hkv;
  long long U, CH, n;
  bool stat;  // static grid: one chunk per grid warp (see the kernel)
  // Per-warp critical path of a chunk size in pages: chunk size x rounds of
  // chunks over the grid (the wave quantisation that decides small problems).
  // All chunk-grid math is 32-bit (units < 2^31, checked on the host): every
  // warp runs it once at startup, where 64-bit division calls are slow cold code.
  __device__ static int path(int u, int ch, int gw) {
    const int n = (u + ch - 1) / ch;
    return ch * ((n + gw - 1) / gw);
  }
  __device__ Chunks(const int32_t* cu_, int B, int Hkv_, int G, long long grid_warps, int stages,
                    int min_chunk, int per_warp, int split_rule, int static_mode, int static_min)
      : cu(cu_), Hkv(Hkv_), U(cu_[B]), stat(false) {
    const int u = cu_[B], gw = (int)grid_warps;
    const int pairs = cu_[B + 1] * Hkv_;  // non-empty (request, kv-head) pairs
    // floor: 16 units, or 8 when that shortens the per-warp path enough to pay
    // for twice the pieces (GQA pieces are G x larger: a higher bar). Measured
    // (knob_sweep, r01k): 8 wins 4-27% at B=4-16 ctx 512-1024 and B=16-64 ctx 1024,
    // 16 wins where 8 only adds a nearly empty second round (B=8 ctx 1024 MHA:
    // 27.0 vs 36.3 us) or more GQA pieces (B=40 ctx 2048 GQA-4: 58.6 vs 62.8 us).
    int floor_ch = min_chunk;
    if (floor_ch <= 0) {
      const long long p8 = path(u, kMinChunkSmall, gw), p16 = path(u, kMinChunk, gw);
      floor_ch = 10 * p8 < (G > 1 ? 7 : 8) * p16 ? kMinChunkSmall : kMinChunk;
    }
    int ch = floor_ch > stages + 1 ? floor_ch : stages + 1;
    if (pairs > 0 && split_rule) {
      const int mu = (int)sqrtf(0.6f * (float)u / (float)pairs);
      if (mu > ch) ch = mu;
    }
    const int cap = (u + per_warp * gw - 1) / (per_warp * gw);
    if (cap > ch) ch = cap;
    if (split_rule >= 2) {  // power of two: chunks then tile power-of-two pair lengths
      int p2 = 4;  // next power of two >= ch (ch >= min_chunk)
      while (p2 < ch) p2 <<= 1;
      if (split_rule == 3 && p2 > ch && p2 / 2 >= 16 && p2 / 2 >= cap) p2 >>= 1;  // round down
      ch = p2;
    }
    CH = ch;
    n = (u + ch - 1) / ch;
    // Static grid: one chunk of ceil(U / warps) units (>= 8) per grid warp. Chosen
    // automatically for small calls where it pays (static_grid_*_r01l.txt): when
    // the chunks tile the pairs and the last-arriving warp's merge stays small
    // (pieces x G <= 32 rows), or when the dynamic grid above would need a
    // second, mostly idle round of chunks. (Misaligned static chunks against a
    // one-round dynamic grid lose: B=8 ctx 1024 MHA 27.9 vs 28.7 us.)
    if (static_mode > 0 && pairs > 0) {
      int chs = (u + gw - 1) / gw;
      const int smin = static_min > 0 ? static_min : kMinChunkSmall;
      if (chs < smin) chs = smin;
      if (chs < stages + 1) chs = stages + 1;
      const int pair_len = u / pairs, np_s = (pair_len + chs - 1) / chs;
      const bool pays = (pair_len % chs == 0 && np_s * G <= 32) || n > grid_warps;
      if (static_mode == 2 || (chs <= kStaticMaxChunk && pays)) {
        stat = true;
        CH = chs;
        n = (u + chs - 1) / chs;
      }
    }
  }
  __device__ long long lo(long long c) const { return c * CH; }
  __device__ long long hi(long long c) const { return (c + 1) * CH < U ? (c + 1) * CH : U; }
};

template <int D, int kWarps, int kStages, int kCtas>
__global__ void __launch_bounds__(kWarps * 32, kCtas)
decode_attn_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                   const DecodeArgs p) {
  using Geo = Geometry<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* stages = smem;
  uint64_t* bars = reinterpret_cast<uint64_t*>(stages + kWarps * kStages * Geo::kStageBytes);
  int32_t* cu = reinterpret_cast<int32_t*>(bars + kWarps * kStages);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  // Programmatic dependent launch: let the next kernel on the stream start its
  // CTAs as soon as SMs free up (it waits for our completion before touching
  // anything we write). No-op without the launch attribute.
  griddep_launch_dependents();
  ADR_TL(0);
  if (threadIdx.x == 0) {
    prefetch_tmap(&tmK);
    prefetch_tmap(&tmV);
  }
  // Units prefix over requests: cu[b] = sum_{b' < b} ceil(seq[b'] / 16) * Hkv.
  // All threads load the lengths at once (independent loads), then a two-level
  // block scan: each thread sums a contiguous chunk, warps scan the chunk sums.
  constexpr int kThreads = kWarps * 32;
  // A request whose seq_len is negative or runs past its block-table row
  // (> 16 x max_blocks) is rejected: it owns no unit (output zero, lse -inf,
  // nothing appended) and sets ADR_STATUS_BAD_SEQ_LEN.
  for (int b = threadIdx.x; b < p.B; b += kThreads) {
    const int sl = p.seq_lens[b];
    const bool ok = sl >= 0 && sl <= p.max_blocks * kPage;
    if (!ok && blockIdx.x == 0) atomicOr(p.status, ADR_STATUS_BAD_SEQ_LEN);
    cu[b + 1] = ok ? cdiv(sl, kPage) * p.Hkv : 0;
  }
  if (threadIdx.x < kWarps * kStages) mbar_init(&bars[threadIdx.x], 1);
  fence_mbar_init();
  __syncthreads();
  {
    __shared__ int warp_tot[kWarps];
    __shared__ int nonempty_tot[kWarps];
    const int per = cdiv(p.B, kThreads);
    const int c0 = min(p.B, threadIdx.x * per), c1 = min(p.B, c0 + per);
    int sum = 0, ne = 0;
    for (int b = c0; b < c1; ++b) {
      sum += cu[b + 1];
      ne += cu[b + 1] > 0;
    }
    int incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ne += __shfl_xor_sync(kFull, ne, o);
    if (lane == 31) warp_tot[warp] = incl;
    if (lane == 0) nonempty_tot[warp] = ne;
    __syncthreads();
    int before = incl - sum;
    for (int w = 0; w < warp; ++w) before += warp_tot[w];
    int run = before;
    for (int b = c0; b < c1; ++b) {
      run += cu[b + 1];
      cu[b + 1] = run;  // each thread rewrites only its own chunk
    }
    if (threadIdx.x == 0) {
      cu[0] = 0;
      int tot = 0;
      for (int w = 0; w < kWarps; ++w) tot += nonempty_tot[w];
      cu[p.B + 1] = tot;  // count of requests with context
    }
  }
  __syncthreads();

  // Requests with no context own no unit: zero output, lse = -inf.
  // (Global writes wait for the preceding kernel: griddep_wait here / below.)
  bool waited = false;
  for (int b = blockIdx.x; b < p.B; b += gridDim.x) {
    if (cu[b + 1] != cu[b]) continue;
    if (!waited) {  // only CTAs that write a zero row wait here
      griddep_wait();
      waited = true;
    }
    const size_t base = (size_t)(p.out_rows ? p.out_rows[b] : b) * p.Hq;
    for (int e = threadIdx.x; e < p.Hq * D; e += blockDim.x) {
      if (p.out_f32) reinterpret_cast<float*>(p.out)[base * D + e] = 0.f;
      else reinterpret_cast<__nv_bfloat16*>(p.out)[base * D + e] = __float2bfloat16(0.f);
    }
    if (p.lse != nullptr)
      for (int e = threadIdx.x; e < p.Hq; e += blockDim.x) p.lse[base + e] = -INFINITY;
  }

  const long long GW = (long long)gridDim.x * kWarps;
  const Chunks ck(cu, p.B, p.Hkv, p.G, GW, kStages, p.min_chunk, p.chunks_per_warp, p.split_rule,
                  p.static_mode, p.static_min);
  const int Hkv = p.Hkv;
  uint8_t* ring = stages + warp * kStages * Geo::kStageBytes;
  uint64_t* ring_bar = bars + warp * kStages;

  // ---- producer: a stream of chunks; page rows one per lane, 32-unit windows --
  auto page_row = [&](int u) -> int {
    const int b = upper_bound_smem(cu, p.B + 1, u) - 1;
    const int nblk = (cu[b + 1] - cu[b]) / Hkv;
    const int local = u - cu[b];
    const int h = local / nblk;
    const int blk = local - h * nblk;
    int page = __ldg(&p.block_table[(size_t)b * p.max_blocks + blk]);
    if ((unsigned)page >= (unsigned)p.num_blocks) {  // never read outside the cache
      atomicOr(p.status, ADR_STATUS_BAD_PAGE);
      page = 0;
    }
    return (page * Hkv + h) * kPage;
  };
  auto window = [&](long long base, long long end) -> int {
    return (base + lane < end) ? page_row((int)(base + lane)) : 0;
  };
  // current chunk [p_lo, p_hi), next unit pu, window base p_wb (rows in row_cur,
  // the chunk's next window in row_nxt); claimed next chunk [n_lo, n_hi) with the
  // rows of its first window in row_nc (n_lo < 0: none; claimed = asked for one)
  long long p_lo = 0, p_hi = 0, pu = 0, p_wb = 0, n_lo = -1, n_hi = -1;
  bool claimed = false;
  int row_cur = 0, row_nxt = 0, row_nc = 0;
  const uint64_t policy = l2_evict_first_policy();
  int32_t* claim_ctr = p.claim;
  auto claim = [&]() {  // warp-uniform; only after griddep_wait (the counter is reused per call)
    if (ck.stat) {  // static grid: the warp's one chunk is all it streams
      claimed = true;
      return;
    }
    int c = 0;
    if (lane == 0) c = atomicAdd(claim_ctr, 1);
    const long long cc = __shfl_sync(kFull, c, 0);
    claimed = true;
    if (cc < ck.n) {
      n_lo = ck.lo(cc);
      n_hi = ck.hi(cc);
      row_nc = window(n_lo, n_hi);
    }
  };
  // Issue the next unit into stage s; false when the stream is exhausted.
  auto issue = [&](int s) -> bool {  // warp-uniform
    if (pu == p_hi) {  // next chunk
      if (n_lo < 0) return false;
      p_lo = p_wb = pu = n_lo;
      p_hi = n_hi;
      n_lo = n_hi = -1;
      claimed = false;
      row_cur = row_nc;
      row_nxt = window(p_lo + 32, p_hi);
    } else if (pu == p_wb + 32) {  // next window of this chunk
      p_wb += 32;
      row_cur = row_nxt;
      row_nxt = window(p_wb + 32, p_hi);
    }
    const int row = __shfl_sync(kFull, row_cur, (int)(pu - p_wb));
    if (lane == 0) {
      uint8_t* st = ring + s * Geo::kStageBytes;
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(&ring_bar[s], Geo::kStageBytes);
#pragma unroll
      for (int hf = 0; hf < Geo::kHalves; ++hf) {
        tma_load_2d(st + hf * kTileBytes, &tmK, hf * 64, row, &ring_bar[s], policy);
        tma_load_2d(st + (Geo::kHalves + hf) * kTileBytes, &tmV, hf * 64, row, &ring_bar[s],
                    policy);
      }
    }
    ++pu;
    return true;
  };
  // Claim the following chunk a few units before this one runs out: late
  // enough to keep the finish balanced, early enough to hide the row lookups.
  auto maybe_claim = [&]() {
    if (!claimed && p_hi - pu <= kClaimAhead) claim();
  };
  uint32_t live = 0;  // bit s: stage s holds an issued unit
  // Every chunk is claimed, none is owned in advance: a warp that never gets an
  // SM (another kernel holding them) then leaves no piece unprocessed, so the
  // merge phase below never waits on a warp that has not started. Claims start
  // after the dependency wait (the previous call on this workspace is done with
  // the counters by then).
  // Before the wait, warp w warms L2 with the first pages of chunk w: the first
  // claims hand out chunks 0, 1, 2, ... so whichever warp gets chunk w finds
  // them there, and HBM works through the preceding kernel's tail. (A hint
  // only: the cache and tables are inputs of the step.)
  long long c_first_lo = -1, c_first_hi = -1;
  bool pre_issued = false;
  if (ck.stat) {
    // Static grid (small calls): warp w owns chunk w, so its table lookups and,
    // when no appended row can be stale (fused append patches it, or no PDL
    // overlap), its first TMA loads are issued before the dependency wait. No
    // claim counter, no merge phase: the warp that publishes a pair's last
    // piece merges the pair. Nothing ever waits on another warp, so a warp
    // that starts late delays the result but cannot deadlock it.
    const long long w = (long long)warp * gridDim.x + blockIdx.x;
    claimed = true;
    if (w < ck.n) {
      n_lo = ck.lo(w);
      n_hi = ck.hi(w);
      row_nc = window(n_lo, n_hi);
    }
    c_first_lo = n_lo;
    c_first_hi = n_hi;
    if (p.k_new != nullptr || !p.pdl) {
#pragma unroll
      for (int k = 0; k < kStages; ++k)
        if (issue(k)) live |= 1u << k;
      pre_issued = true;
    }
  } else {
    const long long w = (long long)warp * gridDim.x + blockIdx.x;
    if (w < ck.n) {
      const long long u0 = ck.lo(w);
      const int r = (u0 + lane < ck.hi(w) && lane < p.prefetch_units) ? page_row((int)(u0 + lane)) : -1;
      if (r >= 0) {
#pragma unroll
        for (int hf = 0; hf < Geo::kHalves; ++hf) {
          tma_prefetch_l2_2d(&tmK, hf * 64, r);
          tma_prefetch_l2_2d(&tmV, hf * 64, r);
        }
      }
    }
  }
  ADR_TL(1);
  if (!waited) griddep_wait();
  ADR_TL(2);
  if (!ck.stat) {
    claim();
    c_first_lo = n_lo;
    c_first_hi = n_hi;
  }
  if (!pre_issued) {
#pragma unroll
    for (int k = 0; k < kStages; ++k) {
      if (issue(k)) live |= 1u << k;
      maybe_claim();
    }
  }
  auto retire = [&]() {  // every warp, once: the last one leaves the claim counters at zero
    int done = 0;
    if (lane == 0) done = atomicAdd(p.claim + 1, 1);
    if (lane == 0 && done == GW - 1) {
      atomicExch(p.claim, 0);      // chunk claims
      atomicExch(p.claim + 2, 0);  // merge-task claims
      atomicExch(p.claim + 1, 0);  // warps done
    }
  };
  const bool streams = c_first_lo >= 0;

  // ---- consumer cursor: chunk [c_lo, c_hi), unit cur ------------------------
  long long c_lo = c_first_lo, c_hi = c_first_hi, cur = c_lo;
  int b = 0, nblk = 1, h = 0, blk = 0, seq = 0;
  auto locate = [&](long long u) {
    b = upper_bound_smem(cu, p.B + 1, (int)u) - 1;
    nblk = (cu[b + 1] - cu[b]) / Hkv;
    h = ((int)u - cu[b]) / nblk;
    blk = ((int)u - cu[b]) - h * nblk;
    seq = p.seq_lens[b];
  };
  if (streams) locate(c_lo);

  const int g = lane >> 2;  // MMA group id (row of A / column of B)
  const int t = lane & 3;   // thread in group
  const int head0 = 2 * t, head1 = 2 * t + 1;
  const int T = (p.G + 1) >> 1;  // lanes t < T carry live heads (compact partials)
  const int acc_floats = Geo::kMTiles * 4 * 8 * T;  // slot = acc (live lanes) | m[8] | l[8]

  // pieces of pair (bb, hh) on the chunk grid
  const int CHi = (int)ck.CH;  // units < 2^31 (checked on the host)
  auto pair_pieces = [&](int bb, int hh) -> int {
    const int nb = (cu[bb + 1] - cu[bb]) / Hkv;
    const int S = cu[bb] + hh * nb;
    return nb > 0 ? (S + nb - 1) / CHi - S / CHi + 1 : 0;
  };
  int n_mine = 0, mine_b0 = 0, mine_h0 = 0, mine_b1 = 0, mine_h1 = 0;  // static grid: pairs to merge

  uint32_t qf[Geo::kKSteps][2];
  float acc[Geo::kMTiles][4];
  float m0, m1, l0, l1;
  bool seg_at_chunk_start = true;  // the current piece began at c_lo (slot 2c, else 2c + 1)
  bool seg_from_page0 = (blk == 0);

  // Fused KV append: lane j < 2*D/8 owns one 16-byte chunk of the new K (j < D/8)
  // or V row; fetched when the pair starts, written when its last page arrives.
  constexpr int kChunks = D / 8;
  const bool app_lane = p.k_new != nullptr && lane < 2 * kChunks;
  const bool app_is_v = lane >= kChunks;
  const int app_c = app_is_v ? lane - kChunks : lane;
  uint4 app_val = make_uint4(0, 0, 0, 0);
  int app_page = 0;
  auto load_append = [&]() {
    // only the warp whose range reaches the pair's last page appends
    if (app_lane && cu[b] + h * nblk + nblk - 1 < c_hi) {
      const __nv_bfloat16* src =
          (app_is_v ? p.v_new : p.k_new) + ((size_t)(p.in_rows ? p.in_rows[b] : b) * Hkv + h) * D;
      app_val = __ldcg(reinterpret_cast<const uint4*>(src) + app_c);  // L2-coherent: may be a peer's
      app_page = __ldg(&p.block_table[(size_t)b * p.max_blocks + nblk - 1]);
      if ((unsigned)app_page >= (unsigned)p.num_blocks) app_page = -1;  // flagged by page_row
    }
  };

  auto load_q = [&]() {
    const bool live = g < p.G;
    const __nv_bfloat16* qrow =
        p.q + ((size_t)(p.in_rows ? p.in_rows[b] : b) * p.Hq + (size_t)h * p.G + (live ? g : 0)) * D;
#pragma unroll
    for (int kk = 0; kk < Geo::kKSteps; ++kk) {  // L2-coherent loads: q may live on a peer GPU
      qf[kk][0] = live ? __ldcg(reinterpret_cast<const uint32_t*>(qrow + kk * 16 + 2 * t)) : 0u;
      qf[kk][1] = live ? __ldcg(reinterpret_cast<const uint32_t*>(qrow + kk * 16 + 8 + 2 * t)) : 0u;
    }
#pragma unroll
    for (int mt = 0; mt < Geo::kMTiles; ++mt)
      acc[mt][0] = acc[mt][1] = acc[mt][2] = acc[mt][3] = 0.f;
    m0 = m1 = kNegBig;
    l0 = l1 = 0.f;
    load_append();
  };
  if (streams) load_q();

  // Per-lane ldmatrix row geometry (constant across pages).
  const int lm_j = lane >> 3;                         // which 8x8 matrix this lane addresses
  const int k_tok = (lane & 7) + ((lm_j & 1) << 3);   // K (non-trans) row
  const int k_chunk_off = lm_j >> 1;                  // +0 / +1 chunk
  const int v_tok = (lane & 7) + ((lm_j >> 1) << 3);  // V (trans) row
  const int v_chunk_off = lm_j & 1;

  // Normalise the register state and write out[] / lse[] of the current pair.
  auto store_output = [&]() {
    const float inv0 = 1.f / l0, inv1 = 1.f / l1;
    const size_t row_base = (size_t)(p.out_rows ? p.out_rows[b] : b) * p.Hq + (size_t)h * p.G;
    if (p.out_f32) {
      float* o = reinterpret_cast<float*>(p.out);
#pragma unroll
      for (int mt = 0; mt < Geo::kMTiles; ++mt) {
        if (head0 < p.G) {
          o[(row_base + head0) * D + mt * 16 + g] = acc[mt][0] * inv0;
          o[(row_base + head0) * D + mt * 16 + g + 8] = acc[mt][2] * inv0;
        }
        if (head1 < p.G) {
          o[(row_base + head1) * D + mt * 16 + g] = acc[mt][1] * inv1;
          o[(row_base + head1) * D + mt * 16 + g + 8] = acc[mt][3] * inv1;
        }
      }
    } else {
      __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(p.out);
#pragma unroll
      for (int mt = 0; mt < Geo::kMTiles; ++mt) {
        // rows = dims, cols = heads -> transpose so each lane owns 2 adjacent dims of one head
        const uint32_t y0 = movmatrix_trans(pack_bf16x2(acc[mt][0] * inv0, acc[mt][1] * inv1));
        const uint32_t y1 = movmatrix_trans(pack_bf16x2(acc[mt][2] * inv0, acc[mt][3] * inv1));
        if (g < p.G) {
          uint32_t* dst = reinterpret_cast<uint32_t*>(o + (row_base + g) * D + mt * 16 + 2 * t);
          dst[0] = y0;
          dst[4] = y1;  // +8 elements
        }
      }
    }
    if (p.lse != nullptr && g == 0) {
      if (head0 < p.G) p.lse[row_base + head0] = (m0 + __log2f(l0)) * kLn2;
      if (head1 < p.G) p.lse[row_base + head1] = (m1 + __log2f(l1)) * kLn2;
    }
  };

  auto finalize = [&](bool complete) {
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      l0 += __shfl_xor_sync(kFull, l0, o);
      l1 += __shfl_xor_sync(kFull, l1, o);
    }
    if (complete) {
      store_output();
      return;
    }
    // ---- split pair: publish this piece ([G][D] acc | m[8] | l[8]); the pair is
    // merged after the stream phase, so nothing here waits on memory ----
    float* sl = p.part + (size_t)(2 * ((int)c_lo / CHi) + (seg_at_chunk_start ? 0 : 1)) * p.slot_floats;
#pragma unroll
    for (int mt = 0; mt < Geo::kMTiles; ++mt) {
      if (head0 < p.G) {
        sl[head0 * D + mt * 16 + g] = acc[mt][0];
        sl[head0 * D + mt * 16 + g + 8] = acc[mt][2];
      }
      if (head1 < p.G) {
        sl[head1 * D + mt * 16 + g] = acc[mt][1];
        sl[head1 * D + mt * 16 + g + 8] = acc[mt][3];
      }
    }
    const int GD = p.G * D;
    if (g == 0) {
      if (head0 < p.G) {
        sl[GD + head0] = m0;
        sl[GD + 8 + head0] = l0;
      }
      if (head1 < p.G) {
        sl[GD + head1] = m1;
        sl[GD + 8 + head1] = l1;
      }
    }
    __syncwarp();  // the lanes' stores precede lane 0's release (cumulative)
    if (ck.stat) {  // static grid: the warp publishing a pair's last piece merges it (after its stream)
      int old = 0;
      if (lane == 0) old = atom_add_acq_rel_s32(p.counter + (size_t)b * Hkv + h, 1);
      old = __shfl_sync(kFull, old, 0);
      if (old == pair_pieces(b, h) - 1) {
        if (n_mine == 0) { mine_b0 = b; mine_h0 = h; } else { mine_b1 = b; mine_h1 = h; }
        ++n_mine;  // <= 2: only a chunk's first and last pairs can be split
      }
    } else if (lane == 0) {
      red_release_add(p.counter + (size_t)b * Hkv + h, 1);
    }
  };

  // Per-lane ldmatrix bases. The 128B swizzle XOR of chunk c = 2j + off with the
  // row's (tok & 7) splits into a lane constant and j, so each of the 4 K and 4
  // V chunk pairs gets one register; stage and half-page offsets are immediates.
  const uint32_t ring_s = smem_addr(ring);
  uint32_t kaddr[4], vaddr[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    kaddr[j] = ring_s + k_tok * 128 + (((2 * j + k_chunk_off) ^ (k_tok & 7)) << 4);
    vaddr[j] = ring_s + Geo::kHalves * kTileBytes + v_tok * 128 +
               (((2 * j + v_chunk_off) ^ (v_tok & 7)) << 4);
  }

#ifdef ADR_STAGE_UNROLL
  constexpr int kStageUnroll = ADR_STAGE_UNROLL;  // experiment: smaller stream-loop code
#else
  constexpr int kStageUnroll = kStages;
#endif
  uint32_t phase = 0;
  bool done = !streams;
  while (!done) {
#pragma unroll kStageUnroll
    for (int s = 0; s < kStages; ++s) {  // unrolled: stage offsets are immediates
      if (done || !((live >> s) & 1u)) {  // stages fill in consumption order: the first empty one ends it
        done = true;
        continue;
      }
      mbar_wait(&ring_bar[s], phase);
#ifdef ADR_TIMELINE
      if (cur == c_first_lo) ADR_TL(3);
#endif
      const uint32_t so = s * Geo::kStageBytes;
      if (p.k_new != nullptr && blk == nblk - 1) {
        // the page holding this step's token: the TMA copy predates the append, so
        // patch the row in shared memory and write it to the cache (the append)
        if (app_lane) {
          const int r = (seq - 1) & (kPage - 1);
          const int half = app_c >> 3, cc = app_c & 7;
          const uint32_t dst = ring_s + so + (app_is_v ? Geo::kHalves * kTileBytes : 0) +
                               half * kTileBytes + r * 128 + ((cc ^ (r & 7)) << 4);
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dst), "r"(app_val.x),
                       "r"(app_val.y), "r"(app_val.z), "r"(app_val.w)
                       : "memory");
          __nv_bfloat16* cache = app_is_v ? p.v_cache : p.k_cache;
          if (app_page >= 0)  // never write outside the cache
            reinterpret_cast<uint4*>(cache + (((size_t)app_page * Hkv + h) * kPage + r) * D)[app_c] =
                app_val;
        }
        __syncwarp();
      }

      // ---- S^T = K . Q^T ----
      float c[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int kk = 0; kk < Geo::kKSteps; ++kk) {
        uint32_t a[4];
        ldmatrix_x4(a, kaddr[kk & 3] + so + (kk >> 2) * kTileBytes);
        mma_16816(c, a, qf[kk][0], qf[kk][1]);
      }
      float s00 = c[0] * p.scale_log2;  // tok g,   head 2t
      float s01 = c[1] * p.scale_log2;  // tok g,   head 2t+1
      float s10 = c[2] * p.scale_log2;  // tok g+8, head 2t
      float s11 = c[3] * p.scale_log2;  // tok g+8, head 2t+1
      if (blk == nblk - 1) {  // only a pair's last page can run past seq_len
        const int tok0 = blk * kPage + g;
        if (tok0 >= seq) s00 = s01 = -INFINITY;
        if (tok0 + 8 >= seq) s10 = s11 = -INFINITY;
      }

      // ---- online softmax (per head, log2 domain) ----
      float mx0 = fmaxf(s00, s10), mx1 = fmaxf(s01, s11);
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        mx0 = fmaxf(mx0, __shfl_xor_sync(kFull, mx0, o));
        mx1 = fmaxf(mx1, __shfl_xor_sync(kFull, mx1, o));
      }
      const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
      const float al0 = fast_exp2(m0 - mn0), al1 = fast_exp2(m1 - mn1);
      m0 = mn0;
      m1 = mn1;
      const float p00 = fast_exp2(s00 - mn0), p01 = fast_exp2(s01 - mn1);
      const float p10 = fast_exp2(s10 - mn0), p11 = fast_exp2(s11 - mn1);
      // P = P_hi + P_lo, both bf16: rounding P to one bf16 alone leaves a 2^-9
      // relative weight error that does not average out (mean-rel ~1e-3); the
      // second PV MMA on the residual brings it to ~2^-17 for 8 extra HMMAs/page.
      const uint32_t x0 = pack_bf16x2(p00, p01);
      const uint32_t x1 = pack_bf16x2(p10, p11);
      const uint32_t r0 = pack_bf16x2(p00 - bf16_lo(x0), p01 - bf16_hi(x0));
      const uint32_t r1 = pack_bf16x2(p10 - bf16_lo(x1), p11 - bf16_hi(x1));
      l0 = l0 * al0 + (p00 + p10);
      l1 = l1 * al1 + (p01 + p11);
      if (__any_sync(kFull, (al0 != 1.f) | (al1 != 1.f))) {
#pragma unroll
        for (int mt = 0; mt < Geo::kMTiles; ++mt) {
          acc[mt][0] *= al0;
          acc[mt][1] *= al1;
          acc[mt][2] *= al0;
          acc[mt][3] *= al1;
        }
      }
      const uint32_t pb0 = movmatrix_trans(x0);  // P^T rows tok 2t..2t+1, col head g
      const uint32_t pb1 = movmatrix_trans(x1);  // tok 8+2t..
      const uint32_t pr0 = movmatrix_trans(r0);
      const uint32_t pr1 = movmatrix_trans(r1);

      // ---- O^T += V^T . P^T ----
#pragma unroll
      for (int mt = 0; mt < Geo::kMTiles; ++mt) {
        uint32_t a[4];
        ldmatrix_x4_trans(a, vaddr[mt & 3] + so + (mt >> 2) * kTileBytes);
        mma_16816(acc[mt], a, pb0, pb1);
        mma_16816(acc[mt], a, pr0, pr1);
      }

      __syncwarp();
      live = issue(s) ? (live | (1u << s)) : (live & ~(1u << s));
      maybe_claim();

      const bool last_of_pair = (blk == nblk - 1);
      const bool last_of_chunk = (cur == c_hi - 1);
      if (last_of_pair || last_of_chunk) {
        finalize(seg_from_page0 && last_of_pair);
        if (last_of_chunk) {
          // the consumer's next chunk is the producer's current one (the producer
          // runs kStages < chunk units ahead); unchanged = the stream has ended
          if (p_lo != c_lo) {
            c_lo = cur = p_lo;
            c_hi = p_hi;
            locate(c_lo);
            seg_at_chunk_start = true;
            seg_from_page0 = (blk == 0);
            load_q();
          }
        } else {
          ++cur;
          blk = 0;
          if (++h == Hkv) {
            h = 0;
            do { ++b; } while (cu[b + 1] == cu[b]);
            nblk = (cu[b + 1] - cu[b]) / Hkv;
            seq = p.seq_lens[b];
          }
          seg_at_chunk_start = false;
          seg_from_page0 = true;
          load_q();
        }
      } else {
        ++cur;
        ++blk;
      }
    }
    phase ^= 1u;
  }

  ADR_TL(4);
  // ---- merge phase: this warp's chunk stream is exhausted --------------------
  // Tasks = (request, q-head) in order; a split pair's pieces are merged per
  // head once all of them are published: lane-parallel max / sum over the
  // pieces, then each lane accumulates its 4 dims over the pieces in chunk
  // order (fixed order: bit-identical whichever warp merges). Pairs complete
  // roughly in unit order, so early finishers take the early pairs.
  // Kept compact on purpose: a warp runs this code once, at the end of the
  // call, when it is no longer in the instruction cache (the stream loop is
  // ~100 KB of SASS); every extra cache line of code is an L2 round trip on the
  // critical tail. Integer math is 32-bit (units < 2^31, checked on the host).
  //
  // merge_head: out[mb, mh*G + k] from the np published pieces of pair (mb, mh)
  // (their writes already acquired by every lane), in piece order; the merged
  // rows are then dropped from L2.
  const int GD = p.G * D;
  const bool dl = lane * 4 < D;  // this lane carries 4 dims of the head's row
  auto merge_head = [&](int mb, int mh, int k, int np) {
    const int nb = (cu[mb + 1] - cu[mb]) / Hkv;
    const int S = cu[mb] + mh * nb;  // the pair's first unit
    const int cf = S / CHi;
    const float* part0 = p.part + (size_t)(2 * cf) * p.slot_floats;
    const int first_odd = (cf * CHi < S) ? 1 : 0;
    auto slot = [&](int i) -> const float* {
      return part0 + (size_t)(2 * i + (i == 0 ? first_odd : 0)) * p.slot_floats;
    };
    // statistics: lane i holds piece i (32r + i in round r); max over all first
    float m0 = kNegBig, l0 = 0.f;
    if (lane < np) {
      m0 = __ldcg(slot(lane) + GD + k);
      l0 = __ldcg(slot(lane) + GD + 8 + k);
    }
    float M = m0;
    for (int i = lane + 32; i < np; i += 32) M = fmaxf(M, __ldcg(slot(i) + GD + k));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(kFull, M, o));
    // rows in piece order, 8 loads in flight per batch; weights from lane i
    float L = 0.f;
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 1
    for (int r = 0; r < np; r += 32) {
      const int i = r + lane;
      float wi = 0.f;
      if (i < np) {
        const float mi = r == 0 ? m0 : __ldcg(slot(i) + GD + k);
        const float li = r == 0 ? l0 : __ldcg(slot(i) + GD + 8 + k);
        wi = exp2f(mi - M);
        L += wi * li;
      }
      const int cnt = min(32, np - r);
#pragma unroll 1
      for (int j = 0; j < cnt; j += 8) {
        float4 x[8];
#pragma unroll
        for (int q = 0; q < 8; ++q)
          x[q] = (j + q < cnt && dl)
                     ? __ldcg(reinterpret_cast<const float4*>(slot(r + j + q) + k * D) + lane)
                     : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float w = __shfl_sync(kFull, wi, (j + q) & 31);
          if (j + q < cnt) {
            a.x += w * x[q].x;
            a.y += w * x[q].y;
            a.z += w * x[q].z;
            a.w += w * x[q].w;
          }
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(kFull, L, o);
    // The head's rows are dead now (every lane has consumed its loads): drop
    // them from L2 instead of leaving ~16 MB of dirty scratch to be written
    // back behind the call's last warp.
    if (lane < D / 32)
      for (int i = 0; i < np; ++i) discard_l2_line(slot(i) + k * D + lane * 32);
#ifdef ADR_TIMELINE
    if (dl && a.x == 12345.f) a.y += 1.f;  // force the loads before the stamp
    ADR_TL(9);  // rows loaded and accumulated
#endif
    const size_t orow = (size_t)(p.out_rows ? p.out_rows[mb] : mb) * p.Hq + (size_t)mh * p.G + k;
    if (dl) {
      const float inv = 1.f / L;
      const size_t o = orow * D + lane * 4;
      if (p.out_f32) {
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(p.out) + o) =
            make_float4(a.x * inv, a.y * inv, a.z * inv, a.w * inv);
      } else {
        uint2 v2;
        v2.x = pack_bf16x2(a.x * inv, a.y * inv);
        v2.y = pack_bf16x2(a.z * inv, a.w * inv);
        *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(p.out) + o) = v2;
      }
    }
    if (p.lse != nullptr && lane == 0) p.lse[orow] = (M + __log2f(L)) * kLn2;
  };

  // merge_heads<V>: all G heads of pair (mb, mh) at once, for the static grid's
  // last-arriving warp: 32 / G' lanes per head (G' = G rounded up to a power of
  // two), V float4 of the head's row per lane (V = D G' / 128), 16 row loads in
  // flight per batch of 16 / V pieces, pieces accumulated in order (deterministic).
  // One pass of round trips for the whole pair instead of G merges in a row.
  auto merge_heads = [&](int mb, int mh, int np, auto vtag) {
    constexpr int V = decltype(vtag)::value;
    constexpr int PB = 16 / V;  // pieces per batch
    const int lph = D / (4 * V);  // lanes per head
    const int hk = lane / lph, sl = lane - hk * lph;
    const bool live = hk < p.G;
    const int hkc = live ? hk : 0;
    const int nb = (cu[mb + 1] - cu[mb]) / Hkv;
    const int S = cu[mb] + mh * nb;
    const int cf = S / CHi;
    const float* part0 = p.part + (size_t)(2 * cf) * p.slot_floats;
    const int first_odd = (cf * CHi < S) ? 1 : 0;
    auto slot = [&](int i) -> const float* {
      return part0 + (size_t)(2 * i + (i == 0 ? first_odd : 0)) * p.slot_floats;
    };
    // one pass, online: each batch's statistics and rows are loaded together
    // and folded in with a running max (no separate max pass over the pieces)
    float M = kNegBig, L = 0.f;
    float4 acc[V];
#pragma unroll
    for (int v = 0; v < V; ++v) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 1
    for (int j0 = 0; j0 < np; j0 += PB) {
      float4 x[PB][V];
      float mq[PB], lq[PB];
#pragma unroll
      for (int q = 0; q < PB; ++q) {
        const bool ok = j0 + q < np;
        const float* sp = slot(ok ? j0 + q : 0);
        mq[q] = ok ? __ldcg(sp + GD + hkc) : kNegBig;
        lq[q] = ok ? __ldcg(sp + GD + 8 + hkc) : 0.f;
#pragma unroll
        for (int v = 0; v < V; ++v)
          x[q][v] = ok ? __ldcg(reinterpret_cast<const float4*>(sp + hkc * D) + sl * V + v)
                       : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      float mb = M;
#pragma unroll
      for (int q = 0; q < PB; ++q) mb = fmaxf(mb, mq[q]);
      const float r = exp2f(M - mb);  // rescale what is accumulated so far
      L *= r;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        acc[v].x *= r;
        acc[v].y *= r;
        acc[v].z *= r;
        acc[v].w *= r;
      }
      M = mb;
#pragma unroll
      for (int q = 0; q < PB; ++q) {
        const float wq = j0 + q < np ? exp2f(mq[q] - M) : 0.f;
        L += wq * lq[q];
#pragma unroll
        for (int v = 0; v < V; ++v) {
          acc[v].x += wq * x[q][v].x;
          acc[v].y += wq * x[q][v].y;
          acc[v].z += wq * x[q][v].z;
          acc[v].w += wq * x[q][v].w;
        }
      }
    }
    __syncwarp();  // every lane has consumed its loads: the pair's lines are dead
    const int lines = (p.G * D) / 32 + 1;  // the heads' rows and the statistics line
    for (int j = 0; j < np; ++j)
      for (int ln = lane; ln < lines; ln += 32) discard_l2_line(slot(j) + ln * 32);
    if (live) {
      const size_t orow = (size_t)(p.out_rows ? p.out_rows[mb] : mb) * p.Hq + (size_t)mh * p.G + hk;
      const float inv = 1.f / L;
      const size_t o = orow * D + (size_t)sl * V * 4;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        if (p.out_f32) {
          reinterpret_cast<float4*>(reinterpret_cast<float*>(p.out) + o)[v] =
              make_float4(acc[v].x * inv, acc[v].y * inv, acc[v].z * inv, acc[v].w * inv);
        } else {
          uint2 v2;
          v2.x = pack_bf16x2(acc[v].x * inv, acc[v].y * inv);
          v2.y = pack_bf16x2(acc[v].z * inv, acc[v].w * inv);
          reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(p.out) + o)[v] = v2;
        }
      }
      if (p.lse != nullptr && sl == 0) p.lse[orow] = (M + __log2f(L)) * kLn2;
    }
  };

  if (ck.stat) {
    // ---- static grid: merge the pairs this warp completed (0-2), no claims ----
    const int gp = p.G <= 1 ? 1 : p.G <= 2 ? 2 : p.G <= 4 ? 4 : 8;  // G rounded up
    const int vv = D * gp / 128;                                      // float4 per lane
    for (int m = 0; m < n_mine; ++m) {
      const int mb = m == 0 ? mine_b0 : mine_b1, mh = m == 0 ? mine_h0 : mine_h1;
      int* arrivals = p.counter + (size_t)mb * Hkv + mh;
      (void)ld_acquire(arrivals);  // every lane acquires the other pieces' writes
      const int np = pair_pieces(mb, mh);
      if (vv == 2) merge_heads(mb, mh, np, std::integral_constant<int, 2>{});
      else if (vv == 4) merge_heads(mb, mh, np, std::integral_constant<int, 4>{});
      else if (vv == 8) merge_heads(mb, mh, np, std::integral_constant<int, 8>{});
      else for (int k = 0; k < p.G; ++k) merge_head(mb, mh, k, np);  // one row per warp
      __syncwarp();
      if (lane == 0) *arrivals = 0;  // every piece has arrived: free for the next call
    }
    ADR_TL(5);
    ADR_TL(11);
    return;
  }

  // ---- dynamic grid: merge tasks (request, q-head) claimed in order ----------
  const int tasks = p.B * p.Hq;
  int tk = 0;
  if (lane == 0) tk = atom_add_s32(p.claim + 2, 1);
  tk = __shfl_sync(kFull, tk, 0);
  while (tk < tasks) {
    const int mb = tk / p.Hq, qh = tk - mb * p.Hq;
    const int mh = qh / p.G, k = qh - mh * p.G;
    const int np = pair_pieces(mb, mh);
    if (np <= 1) {  // empty request (zeroed above) or a pair written in the stream phase
      if (lane == 0) tk = atom_add_s32(p.claim + 2, 1);
      tk = __shfl_sync(kFull, tk, 0);
      continue;
    }
    int* arrivals = p.counter + (size_t)mb * Hkv + mh;
    int* heads_done = p.counter + kMaxPairs + (size_t)mb * Hkv + mh;
#ifdef ADR_TIMELINE
    ADR_TL(6);  // task claimed (last one wins)
#endif
    if (lane == 0)
      while (ld_relaxed_s32(arrivals) < np) __nanosleep(kSpinNs);
    __syncwarp();
    (void)ld_acquire(arrivals);  // every lane acquires the pieces' writes
#ifdef ADR_TIMELINE
    ADR_TL(7);  // its pieces all published
    {
      const int tlw = (threadIdx.x >> 5) * gridDim.x + blockIdx.x;
      if (lane == 0 && tlw < kTlWarps) g_timeline[tlw][8] += 1;  // tasks merged
    }
#endif
    // next task and this head's "merged" count: round trips overlap the loads
    int nxt = 0, hd = 0;
    if (lane == 0) {
      nxt = atom_add_s32(p.claim + 2, 1);
      hd = atom_add_s32(heads_done, 1);
    }
    merge_head(mb, mh, k, np);
    // the pair's last head task leaves its counters at zero for the next call
    // (every head task has passed the wait once all G have counted themselves)
    if (lane == 0 && hd == p.G - 1) {
      *arrivals = 0;
      *heads_done = 0;
    }
    tk = __shfl_sync(kFull, nxt, 0);
#ifdef ADR_TIMELINE
    ADR_TL(10);  // next task index known
#endif
  }
  ADR_TL(5);
  retire();
#ifdef ADR_TIMELINE
  __syncwarp();
  ADR_TL(11);  // retired (lane 0's atomic returned)
#endif
}

// ---- variants (warps per CTA, pages in flight per warp, CTAs per SM) ---------

// (warps per CTA, pages in flight per warp, CTAs per SM); index 0 is the default.
#define ADR_DECODE_VARIANTS(X) \
  X(0, 4, 4, 1)                \
  X(1, 4, 2, 3)                \
  X(2, 8, 3, 1)                \
  X(3, 4, 3, 2)                \
  X(4, 4, 5, 1)                \
  X(5, 4, 6, 1)                \
  X(6, 2, 8, 1)                \
  X(7, 3, 4, 2)                \
  X(8, 2, 4, 3)                \
  X(9, 8, 2, 1)                \
  X(10, 6, 3, 1)               \
  X(11, 2, 12, 1)
constexpr int kNumVariants = 12;

// Default: variant 1 (12 warps x 2 pages per SM). Its 3x per-SM issue capacity
// over variant 0 (4 warps x 4 pages) keeps the whole-device rate when sustained
// load power-caps the SM clock (6.61 vs 6.38 TB/s in the 1 s bench loop; variant
// 0 only wins isolated calls at full clock), and lets an SM partition of ~43%
// of the SMs saturate HBM (colocation curves).
// ADR_DECODE_VARIANT overrides it (tuning experiments).
//
// Coarse chunk grids (few chunks per warp: long pairs with few of them, where the
// chunk size follows sqrt(pair pages)) go to fewer, deeper warps: the last round
// of 64-page chunks is what the call waits on, and 8 warps x 3 pages (variant 2)
// or 8 x 2 (variant 9) per SM give each warp more chunks and more pages in
// flight. Measured (graph-timed, same box, two repeats; profiles/variant_coarse_r02.txt):
// ~1.2 chunks per variant-1 warp (B=8 ctx 32k GQA-4/8) 185.6 -> 159.5 us with
// variant 9; ~2.3 (C5, B=4 ctx 32k MHA, B=16 ctx 16k GQA-4) -1.2 to -1.8% with
// variant 2 (one 2.3 shape +1%); >= 4.6 (C2, C3, B=8 ctx 16k MHA) variant 1 wins
// by 1-7%. The host estimates the grid from the uniform bound
// (units <= B x Hkv x max_blocks_per_seq, the kernel's own chunk rule); ragged
// batches overestimate units and stay on variant 1. Applied to whole-device
// launches only: SM partitions keep variant 1, the grid the colocation curves
// and closed loop were measured with.
int pick_variant(int num_sms, int device_sms, long long units_bound = 0, int max_pages = 0) {
  static int forced = [] {
    const char* e = getenv("ADR_DECODE_VARIANT");
    if (e == nullptr) return -1;
    int x = atoi(e);
    return (x >= 0 && x < kNumVariants) ? x : -1;
  }();
  if (forced >= 0) return forced;
  if (num_sms > 0 && num_sms < device_sms) return 1;
  if (units_bound > 0 && max_pages > 0) {
    const long long gw = (long long)device_sms * 12;  // variant 1: 4 warps x 3 CTAs
    long long ch = (long long)sqrtf(0.6f * (float)max_pages);
    if (ch < kMinChunk) ch = kMinChunk;
    const long long cap = (units_bound + 12 * gw - 1) / (12 * gw);
    if (cap > ch) ch = cap;
    long long p2 = 4;
    while (p2 < ch) p2 <<= 1;
    const long long chunks = (units_bound + p2 - 1) / p2;
    if (chunks < 2 * gw) return 9;
    if (chunks < 3 * gw) return 2;
  }
  return 1;
}

int variant_warps_per_sm(int v) {
  switch (v) {
#define ADR_WPS(I, W, S, C) \
  case I: return W * C;
    ADR_DECODE_VARIANTS(ADR_WPS)
#undef ADR_WPS
    default: return 4;
  }
}

template <int D, int W, int S>
constexpr size_t smem_bytes(int B) {
  return 1024 + (size_t)W * S * Geometry<D>::kStageBytes + W * S * 8 + (size_t)(B + 2) * 4;
}

constexpr int kMaxDevices = 64;

template <int D, int W, int S, int C>
int launch_variant(const CUtensorMap& tmK, const CUtensorMap& tmV, const DecodeArgs& a, int sms,
                   int workers, bool pdl, int dev, cudaStream_t stream) {

  auto kern = decode_attn_kernel<D, W, S, C>;
  // The shared-memory limit is a per-device attribute of the function: a
  // process driving two GPUs (peer offload) must set it on each.
  static std::atomic<bool> configured[kMaxDevices];
  if (dev < 0 || dev >= kMaxDevices) return fail(ADR_ERR_UNSUPPORTED, "device %d", dev);
  if (!configured[dev].load(std::memory_order_acquire)) {
    if (!cuda_ok(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem_bytes<D, W, S>(kMaxBatch)),
                 "cudaFuncSetAttribute(decode_attn_kernel)"))
      return ADR_ERR_CUDA;
    configured[dev].store(true, std::memory_order_release);
  }
  int ctas = (workers + W - 1) / W;
  if (workers <= 0) {
    // persistent grid: every CTA must be resident at once (large B grows the
    // shared-memory prefix arrays and can lower the CTAs that fit per SM)
    int fit = 0;
    if (!cuda_ok(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fit, kern, W * 32,
                                                               smem_bytes<D, W, S>(a.B)),
                 "cudaOccupancyMaxActiveBlocksPerMultiprocessor"))
      return ADR_ERR_CUDA;
    ctas = sms * (fit < C ? (fit > 0 ? fit : 1) : C);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(W * 32);
  cfg.dynamicSmemBytes = smem_bytes<D, W, S>(a.B);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cuda_ok(cudaLaunchKernelEx(&cfg, kern, tmK, tmV, a), "decode_attn_kernel launch")
             ? ADR_OK : ADR_ERR_CUDA;
}

// sms = SMs the persistent grid should cover (whole device or a partition).
template <int D>
int launch_decode(int variant, const CUtensorMap& tmK, const CUtensorMap& tmV,
                  const DecodeArgs& a, int sms, int workers, bool pdl, int dev, cudaStream_t s) {
  switch (variant) {
#define ADR_CASE(I, W, S, C) \
  case I: return launch_variant<D, W, S, C>(tmK, tmV, a, sms, workers, pdl, dev, s);
    ADR_DECODE_VARIANTS(ADR_CASE)
#undef ADR_CASE
    default: return fail(ADR_ERR_INVALID, "bad decode variant");
  }
}

int device_sms(int device) {
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return 0;
  return sms;
}

// Workspace: [arrival counters (fixed capacity, kMaxPairs int32) | claim
// counters and status (256 B) | 2 partial slots per chunk of the largest chunk
// grid]. The counter offsets depend on neither the call's batch nor its head
// count, and every call leaves all counters at zero, so one zero-filled
// workspace serves any sequence of calls with the same or a smaller GQA group,
// head_dim and (request, kv-head, page) unit count.
constexpr size_t kCounterBytes = 2 * kMaxPairs * 4;  // piece arrivals | head merges done
constexpr size_t kClaimBytes = 256;
constexpr int kStatusWord = 8;      // claim[8]: ADR_STATUS_* bits (sticky)
constexpr int kFirstBadWord = 9;    // claim[9]: B - (first rejected request), adr_check_decode_tables
constexpr int kMinChunkAny = 4;     // every chunk grid uses chunks of >= 4 units (bounds the slots)
constexpr int kSplitItemCost = 4;     // split kernel item cost (pages per warp; ADR_SPLIT_ITEM_COST)
constexpr int kSplitDynamic = 0;      // split kernel item order: 0 static (ADR_SPLIT_DYNAMIC)
constexpr int kSplitDynCost = 4;      // split kernel claimed-item cost (ADR_SPLIT_DYN_COST)
constexpr int kSplitMergeCost = 5;    // split kernel merge cost, pages per warp (ADR_SPLIT_MERGE_COST)
constexpr long long kSplitMaxUnits = 65536;  // split-pair kernel up to this unit bound (measured crossover)

// units_bound: an upper bound on the (request, kv-head, page) units of any
// call (B x max_blocks_per_seq x Hkv), or <= 0 for none. Chunks number at most
// kChunksPerWarp per grid warp and at most ceil(units / kMinChunkAny).
size_t workspace_layout(int sms, int num_workers, int G, int D, long long units_bound,
                        size_t* part_off) {
  // explicit worker counts round up to whole CTAs (<= 15 extra warps)
  const long long warps = num_workers > 0 ? (long long)num_workers + 16
                                          : (long long)sms * kMaxWarpsPerSm;
  long long chunks = (long long)kChunksPerWarp * warps;
  if (units_bound > 0) {
    const long long by_units = (units_bound + kMinChunkAny - 1) / kMinChunkAny;
    if (by_units < chunks) chunks = by_units;
  }
  *part_off = kCounterBytes + kClaimBytes;
  return *part_off + (size_t)2 * chunks * slot_floats(G, D) * sizeof(float);
}

// One thread per request: seq_len within [0, 16 x max_blocks] and, for each of
// its pages, block_table entry within [0, num_blocks).
__global__ void check_tables_kernel(const int32_t* __restrict__ block_table,
                                    const int32_t* __restrict__ seq_lens, int B, int max_blocks,
                                    int num_blocks, int32_t* status, int32_t* first_bad) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int sl = seq_lens[b];
  int bits = 0;
  if (sl < 0 || sl > max_blocks * kPage) {
    bits = ADR_STATUS_BAD_SEQ_LEN;
  } else {
    const int n = cdiv(sl, kPage);
    for (int i = 0; i < n; ++i) {
      const int pg = block_table[(size_t)b * max_blocks + i];
      if ((unsigned)pg >= (unsigned)num_blocks) {
        bits = ADR_STATUS_BAD_PAGE;
        break;
      }
    }
  }
  if (bits) {
    atomicOr(status, bits);
    atomicMax(first_bad, B - b);
  }
}

}  // namespace

// decode_split.cu: the split-pair CTA kernel for small calls.
int launch_decode_split(const CUtensorMap& tmK, const CUtensorMap& tmV, const DecodeArgs& a, int D,
                        int sms, bool pdl, int dev, cudaStream_t s);

}  // namespace adr

using namespace adr;

extern "C" int32_t adr_decode_warps_per_sm(int32_t num_sms) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  int sms = device_sms(dev);
  if (sms <= 0) sms = 148;
  return variant_warps_per_sm(pick_variant(num_sms, sms));
}

extern "C" size_t adr_decode_workspace_size(int32_t B, int32_t Hq, int32_t Hkv, int32_t D,
                                            int32_t max_blocks_per_seq, int32_t num_workers) {
  clear_error();
  if (B < 0 || B > kMaxBatch || Hq <= 0 || Hkv <= 0 || Hq % Hkv != 0 || Hq / Hkv > 8 ||
      (D != 64 && D != 128) || max_blocks_per_seq < 0)
    return 0;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  int sms = device_sms(dev);
  if (sms <= 0) sms = 148;
  size_t off;
  const long long units = max_blocks_per_seq > 0 ? (long long)(B > 0 ? B : 1) * max_blocks_per_seq * Hkv : 0;
  return workspace_layout(sms, num_workers, Hq / Hkv, D, units, &off);
}

extern "C" size_t adr_decode_workspace_bytes(int32_t B, int32_t Hq, int32_t Hkv, int32_t D,
                                             int32_t num_workers) {
  return adr_decode_workspace_size(B, Hq, Hkv, D, 0, num_workers);
}

extern "C" int32_t adr_decode_status(void* workspace, size_t workspace_bytes, int32_t clear,
                                     int32_t* status, void* stream) {
  clear_error();
  if (!workspace || !status) return fail(ADR_ERR_INVALID, "null pointer");
  if (workspace_bytes < kCounterBytes + kClaimBytes)
    return fail(ADR_ERR_WORKSPACE, "workspace %zu bytes too small", workspace_bytes);
  int32_t* word = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(workspace) + kCounterBytes) + kStatusWord;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (!cuda_ok(cudaMemcpyAsync(status, word, 4, cudaMemcpyDeviceToHost, s), "status read"))
    return ADR_ERR_CUDA;
  if (clear && !cuda_ok(cudaMemsetAsync(word, 0, 4, s), "status clear")) return ADR_ERR_CUDA;
  return cuda_ok(cudaStreamSynchronize(s), "cudaStreamSynchronize") ? ADR_OK : ADR_ERR_CUDA;
}

extern "C" int32_t adr_check_decode_tables(const int32_t* block_table, const int32_t* seq_lens,
                                           int32_t B, int32_t max_blocks_per_seq,
                                           int64_t num_blocks, void* workspace,
                                           size_t workspace_bytes, void* stream) {
  clear_error();
  if (B == 0) return ADR_OK;
  if (B < 0 || max_blocks_per_seq <= 0 || num_blocks <= 0 || num_blocks >= ((int64_t)1 << 31))
    return fail(ADR_ERR_INVALID, "bad shape B=%d max_blocks_per_seq=%d num_blocks=%lld", B,
                max_blocks_per_seq, (long long)num_blocks);
  if (!block_table || !seq_lens || !workspace) return fail(ADR_ERR_INVALID, "null pointer");
  if (workspace_bytes < kCounterBytes + kClaimBytes)
    return fail(ADR_ERR_WORKSPACE, "workspace %zu bytes too small", workspace_bytes);
  int32_t* words = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(workspace) + kCounterBytes);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  check_tables_kernel<<<cdiv(B, 128), 128, 0, s>>>(block_table, seq_lens, B, max_blocks_per_seq,
                                                   (int)num_blocks, words + kStatusWord,
                                                   words + kFirstBadWord);
  if (!cuda_ok(cudaGetLastError(), "check_tables_kernel launch")) return ADR_ERR_CUDA;
  int32_t host[2] = {0, 0};
  if (!cuda_ok(cudaMemcpyAsync(host, words + kStatusWord, 8, cudaMemcpyDeviceToHost, s), "status read") ||
      !cuda_ok(cudaMemsetAsync(words + kStatusWord, 0, 8, s), "status clear") ||
      !cuda_ok(cudaStreamSynchronize(s), "cudaStreamSynchronize"))
    return ADR_ERR_CUDA;
  if (host[0] == 0) return ADR_OK;
  const int b = B - host[1];
  int32_t sl = 0;
  if (b >= 0 && b < B) cudaMemcpy(&sl, seq_lens + b, 4, cudaMemcpyDeviceToHost);
  if (sl < 0 || sl > max_blocks_per_seq * kPage)
    return fail(ADR_ERR_INVALID, "request %d: seq_len %d outside [0, %d] (max_blocks_per_seq x 16)",
                b, sl, max_blocks_per_seq * kPage);
  return fail(ADR_ERR_INVALID, "request %d: block_table entry outside [0, %lld) among its %d pages",
              b, (long long)num_blocks, cdiv(sl, kPage));
}

extern "C" int32_t adr_paged_decode_attn_rows(
    const void* q, const void* k_new, const void* v_new, const int32_t* in_rows, void* k_cache,
    void* v_cache, const int32_t* block_table, const int32_t* seq_lens, void* out, float* lse,
    const int32_t* out_rows, int32_t B, int32_t Hq, int32_t Hkv, int32_t D, int32_t block_size,
    int32_t max_blocks_per_seq, int64_t num_blocks, float scale, int32_t num_sms,
    int32_t num_workers, int32_t out_dtype, uint32_t flags, void* workspace,
    size_t workspace_bytes, void* stream) {
  clear_error();
  if (B == 0) return ADR_OK;
  if (B < 0 || B > kMaxBatch) return fail(ADR_ERR_INVALID, "B must be in [0, %d], got %d", kMaxBatch, B);
  if (!q || !k_cache || !v_cache || !block_table || !seq_lens || !out)
    return fail(ADR_ERR_INVALID, "null tensor pointer");
  if (Hq <= 0 || Hkv <= 0 || Hq % Hkv != 0)
    return fail(ADR_ERR_INVALID, "Hq (%d) must be a positive multiple of Hkv (%d)", Hq, Hkv);
  if (Hq / Hkv > 8) return fail(ADR_ERR_UNSUPPORTED, "GQA group %d > 8", Hq / Hkv);
  if (D != 64 && D != 128) return fail(ADR_ERR_UNSUPPORTED, "head_dim %d (need 64 or 128)", D);
  if (block_size != kPage) return fail(ADR_ERR_UNSUPPORTED, "block_size %d (need 16)", block_size);
  if (max_blocks_per_seq <= 0 || num_blocks <= 0)
    return fail(ADR_ERR_INVALID, "max_blocks_per_seq and num_blocks must be positive");
  if (num_blocks * Hkv * kPage >= (int64_t)1 << 31)
    return fail(ADR_ERR_UNSUPPORTED, "cache too large for 32-bit page rows");
  if ((int64_t)B * max_blocks_per_seq * Hkv >= (int64_t)1 << 31)
    return fail(ADR_ERR_UNSUPPORTED, "too many (request, head, page) units");
  if (out_dtype != ADR_DTYPE_BF16 && out_dtype != ADR_DTYPE_F32)
    return fail(ADR_ERR_INVALID, "out_dtype %d", out_dtype);
  if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k_cache) |
       reinterpret_cast<uintptr_t>(v_cache) | reinterpret_cast<uintptr_t>(k_new) |
       reinterpret_cast<uintptr_t>(v_new) | reinterpret_cast<uintptr_t>(out)) & 15)
    return fail(ADR_ERR_INVALID, "q / k_new / v_new / caches / out must be 16-byte aligned");
  if (reinterpret_cast<uintptr_t>(lse) & 3) return fail(ADR_ERR_INVALID, "lse must be 4-byte aligned");
  if ((k_new == nullptr) != (v_new == nullptr))
    return fail(ADR_ERR_INVALID, "k_new and v_new must both be given or both be null");
  if (flags & ~uint32_t(ADR_DECODE_PDL | ADR_DECODE_GRID_DYNAMIC | ADR_DECODE_GRID_STATIC |
                        ADR_DECODE_GRID_SPLIT))
    return fail(ADR_ERR_INVALID, "unknown flags 0x%x", flags);
  {
    const uint32_t grids = flags & (ADR_DECODE_GRID_DYNAMIC | ADR_DECODE_GRID_STATIC | ADR_DECODE_GRID_SPLIT);
    if (grids & (grids - 1))
      return fail(ADR_ERR_INVALID, "ADR_DECODE_GRID_DYNAMIC / _STATIC / _SPLIT exclude each other");
  }

  int dev = 0;
  if (!cuda_ok(cudaGetDevice(&dev), "cudaGetDevice")) return ADR_ERR_CUDA;
  const int dev_sms = device_sms(dev);
  if (dev_sms <= 0) return fail(ADR_ERR_CUDA, "cannot query SM count");
  if (num_sms < 0 || num_sms > dev_sms)
    return fail(ADR_ERR_INVALID, "num_sms %d outside [0, %d]", num_sms, dev_sms);
  if (num_workers < 0 || num_workers > dev_sms * kMaxWarpsPerSm * 64)
    return fail(ADR_ERR_INVALID, "num_workers %d out of range", num_workers);
  const int sms = num_sms > 0 ? num_sms : dev_sms;
  const int variant = num_workers > 0 ? pick_variant(num_sms, dev_sms)
                                      : pick_variant(num_sms, dev_sms,
                                                     (long long)B * Hkv * max_blocks_per_seq,
                                                     max_blocks_per_seq);
  if ((long long)B * Hkv > kMaxPairs)
    return fail(ADR_ERR_UNSUPPORTED, "B*Hkv = %lld pairs > %lld", (long long)B * Hkv, kMaxPairs);
  size_t part_off;
  const size_t need = workspace_layout(dev_sms, num_workers, Hq / Hkv, D,
                                       (long long)B * max_blocks_per_seq * Hkv, &part_off);
  if (workspace == nullptr || workspace_bytes < need)
    return fail(ADR_ERR_WORKSPACE, "workspace %zu bytes < required %zu", workspace_bytes, need);

  CUtensorMap tmK, tmV;
  const uint64_t rows = (uint64_t)num_blocks * Hkv * kPage;
  int rc = encode_page_tmap(&tmK, k_cache, D, rows);
  if (rc != ADR_OK) return rc;
  rc = encode_page_tmap(&tmV, v_cache, D, rows);
  if (rc != ADR_OK) return rc;

  DecodeArgs a;
  a.q = static_cast<const __nv_bfloat16*>(q);
  a.k_new = static_cast<const __nv_bfloat16*>(k_new);
  a.v_new = static_cast<const __nv_bfloat16*>(v_new);
  a.k_cache = static_cast<__nv_bfloat16*>(k_cache);
  a.v_cache = static_cast<__nv_bfloat16*>(v_cache);
  a.block_table = block_table;
  a.seq_lens = seq_lens;
  a.out = out;
  a.lse = lse;
  a.in_rows = in_rows;
  a.out_rows = out_rows;
  a.counter = static_cast<int32_t*>(workspace);
  a.claim = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(workspace) + kCounterBytes);
  a.status = a.claim + kStatusWord;
  a.part = reinterpret_cast<float*>(static_cast<uint8_t*>(workspace) + part_off);
  a.slot_floats = slot_floats(Hq / Hkv, D);
  // chunk-grid tuning knobs (ADR_CHUNK_MIN >= 16, ADR_CHUNKS_PER_WARP <= the
  // workspace bound, ADR_SPLIT_RULE 0/1); defaults are the measured best
  static const int env_min = [] { const char* e = getenv("ADR_CHUNK_MIN"); return e ? atoi(e) : 0; }();
  static const int env_cpw = [] { const char* e = getenv("ADR_CHUNKS_PER_WARP"); return e ? atoi(e) : 0; }();
  static const int env_rule = [] { const char* e = getenv("ADR_SPLIT_RULE"); return e ? atoi(e) : -1; }();
  static const int env_pf = [] { const char* e = getenv("ADR_PREFETCH_UNITS"); return e ? atoi(e) : -1; }();
  a.min_chunk = env_min >= 4 ? env_min : 0;  // 0: size rule (kMinChunk / kMinChunkSmall)
  a.chunks_per_warp = (env_cpw > 0 && env_cpw <= kChunksPerWarp) ? env_cpw : kChunksPerWarp;
  a.split_rule = env_rule >= 0 ? env_rule : 2;
  a.prefetch_units = (env_pf >= 0 && env_pf <= 32) ? env_pf : kPrefetchUnits;
  static const int env_static = [] { const char* e = getenv("ADR_STATIC_GRID"); return e ? atoi(e) : -1; }();
  a.static_mode = (flags & ADR_DECODE_GRID_STATIC) ? 2 : (flags & ADR_DECODE_GRID_DYNAMIC) ? 0
                : (env_static >= 0 && env_static <= 2) ? env_static : 1;
  a.pdl = (flags & ADR_DECODE_PDL) ? 1 : 0;
  static const int env_smin = [] { const char* e = getenv("ADR_STATIC_MIN"); return e ? atoi(e) : 0; }();
  a.static_min = env_smin >= kMinChunkAny ? env_smin : 0;  // the grid clamps it to >= stages + 1
  a.B = B;
  a.Hq = Hq;
  a.Hkv = Hkv;
  a.G = Hq / Hkv;
  a.max_blocks = max_blocks_per_seq;
  a.num_blocks = (int)num_blocks;
  a.out_f32 = out_dtype == ADR_DTYPE_F32;
  a.scale_log2 = scale * kLog2e;
  a.part_slots = (int)std::min<size_t>((workspace_bytes - part_off) / ((size_t)a.slot_floats * 4),
                                       (size_t)1 << 30);
  static const int env_item = [] { const char* e = getenv("ADR_SPLIT_ITEM_COST"); return e ? atoi(e) : -1; }();
  a.split_item_cost = (env_item >= 0 && env_item <= 64) ? env_item : kSplitItemCost;
  static const int env_k = [] { const char* e = getenv("ADR_SPLIT_FORCE_K"); return e ? atoi(e) : 0; }();
  a.split_force_k = env_k;
  static const int env_dyn = [] { const char* e = getenv("ADR_SPLIT_DYNAMIC"); return e ? atoi(e) : -1; }();
  static const int env_dcost = [] { const char* e = getenv("ADR_SPLIT_DYN_COST"); return e ? atoi(e) : -1; }();
  a.split_dynamic = (env_dyn >= 0 && env_dyn <= 2) ? env_dyn : kSplitDynamic;
  a.split_dyn_cost = (env_dcost >= 0 && env_dcost <= 64) ? env_dcost : kSplitDynCost;
  static const int env_mcost = [] { const char* e = getenv("ADR_SPLIT_MERGE_COST"); return e ? atoi(e) : -1; }();
  a.split_merge_cost = (env_mcost >= 0 && env_mcost <= 64) ? env_mcost : kSplitMergeCost;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool pdl = (flags & ADR_DECODE_PDL) != 0;
  // Small calls (the executor's per-layer offloaded batches): the split-pair CTA
  // kernel (decode_split.cu) when the call's unit bound (B x table width x Hkv)
  // is at most ADR_SPLIT_MAX_UNITS (measured crossover), unless a
  // grid is forced. The split is chosen on the device from the real lengths.
  static const long long split_max = [] {
    const char* e = getenv("ADR_SPLIT_MAX_UNITS");
    return e ? atoll(e) : kSplitMaxUnits;
  }();
  const long long unit_bound = (long long)B * max_blocks_per_seq * Hkv;
  const bool forced = flags & (ADR_DECODE_GRID_DYNAMIC | ADR_DECODE_GRID_STATIC);
  // GQA groups > 4 (the 4x2 split variant): the split kernel stays ahead up to 2x the bound
  // (1 GB at D=128: 155-167 vs 164-186 us; 2 GB: 325 vs 316; profiles/split_gqa8_r02q.txt)
  const long long bound = Hq / Hkv > 4 ? 2 * split_max : split_max;
  if ((flags & ADR_DECODE_GRID_SPLIT) || (!forced && num_workers == 0 && unit_bound <= bound))
    return launch_decode_split(tmK, tmV, a, D, sms, pdl, dev, s);
  return D == 128 ? launch_decode<128>(variant, tmK, tmV, a, sms, num_workers, pdl, dev, s)
                  : launch_decode<64>(variant, tmK, tmV, a, sms, num_workers, pdl, dev, s);
}

extern "C" int32_t adr_paged_decode_attn(const void* q, const void* k_new, const void* v_new,
                                         void* k_cache, void* v_cache,
                                         const int32_t* block_table, const int32_t* seq_lens,
                                         void* out, float* lse, int32_t B, int32_t Hq, int32_t Hkv,
                                         int32_t D, int32_t block_size, int32_t max_blocks_per_seq,
                                         int64_t num_blocks, float scale, int32_t num_sms,
                                         int32_t num_workers, int32_t out_dtype, uint32_t flags,
                                         void* workspace, size_t workspace_bytes, void* stream) {
  return adr_paged_decode_attn_rows(q, k_new, v_new, nullptr, k_cache, v_cache, block_table,
                                    seq_lens, out, lse, nullptr, B, Hq, Hkv, D, block_size,
                                    max_blocks_per_seq, num_blocks, scale, num_sms, num_workers,
                                    out_dtype, flags, workspace, workspace_bytes, stream);
}

#ifdef ADR_TIMELINE
extern "C" ADR_API int32_t adr_debug_timeline(void* dst, size_t bytes) {
  return cudaMemcpyFromSymbol(dst, g_timeline, bytes < sizeof(g_timeline) ? bytes : sizeof(g_timeline)) ==
                 cudaSuccess
             ? 0
             : -3;
}
#endif
