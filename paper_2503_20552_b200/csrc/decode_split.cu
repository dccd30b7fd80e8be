// Split-pair CTA kernel: paged decode attention for SMALL calls (sm_100a).
//
// Same arithmetic as decode_attn_kernel (paged_decode_attn.cu): per page of one
// (request, kv-head) pair, S^T = K.Q^T and O^T += V^T.P^T on mma.sync m16n8k16
// tiles from a TMA-filled, 128B-swizzled shared-memory ring, online softmax in
// the log2 domain, P split into bf16 hi + lo parts, fused KV append.
//
// What differs is the work split, built for calls whose KV fits in the
// device's shared-memory pipelines a few times over (the executor's per-layer
// offloaded batches):
//  * An ITEM is a run of P consecutive pages of one pair. Every pair of n pages
//    is cut into ceil(n / P) items; P (a multiple of the warps per CTA) is picked
//    on the device from the call's total pages so that the items fill one round
//    of the persistent grid. CTA c takes items c, c + grid, ...
//  * Inside an item the CTA's W warps interleave pages (warp w: pages w, w + W,
//    ...), so every warp of every SM streams from the first microsecond and all
//    of a warp's pages are usually in flight at once (in the stream-K kernel a
//    small call leaves most warps idle and the busy ones latency-bound).
//  * The W per-warp states are combined through shared memory (fixed warp
//    order). An item that is a whole pair writes out / lse directly; otherwise
//    it publishes one fp32 partial and the CTA that publishes a pair's last
//    partial merges them (fixed item order): one global merge per pair, over a
//    handful of pieces, with the whole CTA's threads.
//  * Before the dependency wait (PDL) it reads only step inputs the preceding
//    kernel may not write (seq_lens, block table, cache pages): the unit scan,
//    the split choice, the table lookups and the first TMA loads all overlap the
//    previous kernel's tail.
// Results are deterministic (fixed combine and merge orders).
#include <atomic>
#include <climits>
#include <cstdlib>

#include "decode_common.cuh"

namespace adr {
namespace {

using namespace dec;

// Block-wide exclusive scan of one int per thread; `total` receives the sum.
template <int kWarps>
__device__ __forceinline__ int block_excl_scan(int v, int* tmp, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int x = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += x;
  }
  if (lane == 31) tmp[warp] = incl;
  __syncthreads();
  int before = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    const int t = tmp[w];
    before += w < warp ? t : 0;
    tot += t;
  }
  __syncthreads();  // tmp is reused by the next scan
  total = tot;
  return before + incl - v;
}

// out[o .. o+3] = A * inv (fp32 or bf16 rows; o is a multiple of 4)
__device__ __forceinline__ void store_row4(const DecodeArgs& p, size_t o, float4 A, float inv) {
  if (p.out_f32) {
    *reinterpret_cast<float4*>(reinterpret_cast<float*>(p.out) + o) =
        make_float4(A.x * inv, A.y * inv, A.z * inv, A.w * inv);
  } else {
    uint2 v;
    v.x = pack_bf16x2(A.x * inv, A.y * inv);
    v.y = pack_bf16x2(A.z * inv, A.w * inv);
    *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(p.out) + o) = v;
  }
}

// Split-size candidates: the longest pair cut into k runs (see the kernel),
// k = 1 .. 12, then 16, 24, 32, 48, ... 512, 768 (c < 24).
constexpr int kNumSplitK = 24;
constexpr int kSplitClaimWord = 4;  // claim[4]: dynamic item claims, claim[5]: CTAs done
__device__ __forceinline__ int split_k(int c) {
  return c < 12 ? c + 1 : ((((c - 12) & 1) ? 3 : 2) << ((c - 12) >> 1)) << 3;
}

struct SplitItem {
  int b, h, lo, hi, n, ns, s;  // pages [lo, hi) of pair (b, h) with n pages; split s of ns
};

template <int D, int kW, int kS, int kCtas>
__global__ void __launch_bounds__(kW * 32, kCtas)
decode_split_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                    const DecodeArgs p) {
  using Geo = Geometry<D>;
  constexpr int kThreads = kW * 32;
  constexpr int kRowPad = D + 4;  // combine rows padded against bank conflicts
  constexpr int kFpt = (8 * D / 4 + kThreads - 1) / kThreads;  // float4 of a pair's rows per thread (G <= 8)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* stages = smem;
  uint64_t* bars = reinterpret_cast<uint64_t*>(stages + kW * kS * Geo::kStageBytes);
  const int G = p.G;
  const int comb_floats = G * kRowPad + 16;  // per warp: acc [G][D+4] | m[8] | l[8]
  float* comb = reinterpret_cast<float*>(bars + kW * kS);
  float* hst = comb + kW * comb_floats;  // head statistics: M[8] | L[8] | weights [W][8] (or rescale[8])
  int32_t* pg = reinterpret_cast<int32_t*>(hst + 16 + 8 * kW);        // [B+1] page prefix
  int32_t* icu = pg + (p.B + 1);                                      // [B+1] item prefix
  __shared__ int scan_tmp[kW];
  __shared__ int cand_tmp[kW][kNumSplitK];
  __shared__ int s_last;
  __shared__ int s_items[4];  // dynamic claims: item k of this CTA in slot k & 3 (k <= s_known)
  __shared__ int s_known;
  __shared__ int s_dyn;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int Hkv = p.Hkv;

  griddep_launch_dependents();
  ADR_TL(0);
  if (threadIdx.x == 0) {
    prefetch_tmap(&tmK);
    prefetch_tmap(&tmV);
  }
  if (threadIdx.x < kW * kS) mbar_init(&bars[threadIdx.x], 1);
  fence_mbar_init();

  // ---- pages per request (rejected requests own none) and their prefix ----
  const int per = cdiv(p.B, kThreads);
  const int c0 = min(p.B, (int)threadIdx.x * per), c1 = min(p.B, c0 + per);
  int sum = 0;
  for (int b = c0; b < c1; ++b) {
    const int sl = p.seq_lens[b];
    const bool ok = sl >= 0 && sl <= p.max_blocks * kPage;
    if (!ok && blockIdx.x == 0) atomicOr(p.status, ADR_STATUS_BAD_SEQ_LEN);
    const int n = ok ? cdiv(sl, kPage) : 0;
    pg[b + 1] = n;
    sum += n;
  }
  int total_pages = 0;
  int run = block_excl_scan<kW>(sum, scan_tmp, total_pages);
  for (int b = c0; b < c1; ++b) {
    run += pg[b + 1];
    pg[b + 1] = run;
  }
  if (threadIdx.x == 0) pg[0] = 0;
  ADR_TL(6);
  // ---- split size P ------------------------------------------------------------
  // Candidates: the longest pair cut into k equal runs (k = split_k(c)), rounded
  // to whole warp rounds. Each gives ni items and a per-CTA critical path of
  // ceil(ni / grid) rounds x (P / W pages per warp + the item's fixed cost);
  // take the shortest path, then the fewest items (fewer partials to merge).
  // Lane c of every warp evaluates candidate c over the warp's requests, so the
  // whole choice is one short parallel pass (it runs cold, once per call, before
  // the first page: a serial loop over the candidates cost ~15 us here).
  // Every CTA computes the same P: same integer math, same prefix.
  const int GC = gridDim.x;
  auto round_w = [](int x) { return (x + kW - 1) / kW * kW; };
  auto count_items = [&](int P) {
    int c = 0;
    for (int b = c0; b < c1; ++b) c += cdiv(pg[b + 1] - pg[b], P);  // pg is final: read-only
    return c;
  };
  __syncthreads();  // pg complete
  int nmax = 0;
  for (int b = c0; b < c1; ++b) nmax = max(nmax, pg[b + 1] - pg[b]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nmax = max(nmax, __shfl_xor_sync(kFull, nmax, o));
  if (lane == 0) scan_tmp[warp] = nmax;
  __syncthreads();
  nmax = 0;
#pragma unroll
  for (int w = 0; w < kW; ++w) nmax = max(nmax, scan_tmp[w]);
  const bool cand = lane < kNumSplitK;
  const int Pc = round_w(max(kW, cdiv(max(nmax, 1), split_k(cand ? lane : 0))));
  {
    int m = 0;
    if (cand)
      for (int b = warp; b < p.B; b += kW) m += cdiv(pg[b + 1] - pg[b], Pc);
    if (cand) cand_tmp[warp][lane] = m;
  }
  __syncthreads();
  int P, ni = 0;
  {
    int m = 0;
#pragma unroll
    for (int w = 0; w < kW; ++w) m += cand ? cand_tmp[w][lane] : 0;
    m *= Hkv;
    const bool ok = cand && m <= p.part_slots &&
                    (p.split_force_k <= 0 || split_k(lane) == p.split_force_k);  // tuning knob
    // static items (CTA c: items c, c + grid, ...): rounds x (pages + item cost);
    // dynamic items (first static, then claimed): average pages per CTA + the
    // last item (tail) + the items' costs — both in pages of one CTA
    // (+ the merge of split pairs: the last-arriving CTA of a pair merges it)
    const int merge = nmax > Pc ? p.split_merge_cost * kW : 0;
    const long long path_s = (long long)cdiv(m, GC) * (Pc + p.split_item_cost * kW) + merge;
    const long long path_d = (long long)cdiv(total_pages * Hkv, GC) + Pc +
                             (long long)cdiv(m, GC) * p.split_dyn_cost * kW + merge;
    const bool dyn_c = p.split_dynamic == 1 || (p.split_dynamic == 2 && path_d < path_s);
    long long path = ok ? (dyn_c ? path_d : path_s) : LLONG_MAX;
    long long best = path;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(kFull, best, o));
    int mm = path == best ? m : INT_MAX;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mm = min(mm, __shfl_xor_sync(kFull, mm, o));
    const unsigned win = __ballot_sync(kFull, path == best && m == mm);
    // no candidate fits the workspace: the longest runs, doubled below until they do
    const int wl = best == LLONG_MAX ? 0 : __ffs(win) - 1;
    P = __shfl_sync(kFull, Pc, wl);
    const int dw = __shfl_sync(kFull, (int)dyn_c, wl);
    if (threadIdx.x == 0) s_dyn = dw && best != LLONG_MAX;
  }
  ADR_TL(7);
  int mine = count_items(P);
  int ex = block_excl_scan<kW>(mine, scan_tmp, ni);
  ni *= Hkv;
  while (ni > p.part_slots && P < (1 << 24)) {  // workspace bound (rare: tiny workspaces)
    P *= 2;
    mine = count_items(P);
    ex = block_excl_scan<kW>(mine, scan_tmp, ni);
    ni *= Hkv;
  }
  {
    int r = ex * Hkv;
    for (int b = c0; b < c1; ++b) {
      icu[b] = r;
      r += Hkv * cdiv(pg[b + 1] - pg[b], P);
    }
    if (threadIdx.x == 0) icu[p.B] = ni;
  }
  __syncthreads();
  ADR_TL(9);

  // Requests with no context own no item: zero output, lse = -inf.
  bool waited = false;
  for (int b = blockIdx.x; b < p.B; b += gridDim.x) {
    if (pg[b + 1] != pg[b]) continue;
    if (!waited) {
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

  auto item_at = [&](int i) -> SplitItem {
    SplitItem it;
    it.b = upper_bound_smem(icu, p.B + 1, i) - 1;
    it.n = pg[it.b + 1] - pg[it.b];
    it.ns = cdiv(it.n, P);
    const int local = i - icu[it.b];
    it.h = local / it.ns;
    it.s = local - it.h * it.ns;
    it.lo = it.s * P;
    it.hi = min(it.n, it.lo + P);
    return it;
  };
  // pages of this warp in an item: lo + warp + kW * j, j < count
  auto warp_pages = [&](const SplitItem& it) -> int {
    return it.hi - it.lo > warp ? (it.hi - it.lo - warp + kW - 1) / kW : 0;
  };

  uint8_t* ring = stages + warp * kS * Geo::kStageBytes;
  uint64_t* ring_bar = bars + warp * kS;
  const uint64_t policy = l2_evict_first_policy();

  // ---- this CTA's item sequence --------------------------------------------
  // static: items c, c + grid, c + 2 grid, ...; dynamic: item c first, then
  // items grid + (claims of a global counter), claimed by thread 0 three items
  // ahead of the consumers (slot k & 3). `known` is this thread's copy of the
  // highest claimed index, refreshed only after a __syncthreads.
  const bool dyn = s_dyn != 0;
  constexpr int kStall = -2;  // item not claimed yet (dynamic): retry after the next item
  int known = 0;
  auto item_seq = [&](int k) -> int {
    if (!dyn) {
      const long long i = (long long)blockIdx.x + (long long)k * GC;
      return i < ni ? (int)i : -1;
    }
    if (k == 0) return (int)blockIdx.x < ni ? (int)blockIdx.x : -1;
    return k <= known ? *reinterpret_cast<volatile int*>(&s_items[k & 3]) : kStall;
  };
  int32_t* dyn_claim = p.claim + kSplitClaimWord;
  bool claims_out = false;  // thread 0: the counter ran past the items
  auto claim_items = [&](int k0, int n) {  // thread 0: claim items k0 .. k0 + n - 1
    int v = claims_out ? ni : atomicAdd(dyn_claim, n);
    for (int j = 0; j < n; ++j) {
      const int i = GC + v + j;
      const bool in = !claims_out && i < ni;
      s_items[(k0 + j) & 3] = in ? i : -1;
      if (!in) claims_out = true;
    }
    s_known = k0 + n - 1;
  };

  // ---- producer: this warp's pages of the CTA's items, in sequence order -----
  int pidx = 0;  // producing item (index in the sequence)
  int prod = 0;  // pages issued by this warp (ring position)
  SplitItem pit{};
  int pk = 0, pj = 0, pwb = 0, prow = 0;  // pages in item, next page, row window base, rows
  auto load_rows = [&]() {  // rows of pages j in [pwb, pwb + 32) of item pit, one per lane
    const int j = pwb + lane;
    int row = 0;
    if (j < pk) {
      const int pgi = pit.lo + warp + kW * j;
      int page = __ldg(&p.block_table[(size_t)pit.b * p.max_blocks + pgi]);
      if ((unsigned)page >= (unsigned)p.num_blocks) {  // never read outside the cache
        atomicOr(p.status, ADR_STATUS_BAD_PAGE);
        page = 0;
      }
      row = (page * Hkv + pit.h) * kPage;
    }
    prow = row;
  };
  bool prod_live = true;
  {
    // first item of this CTA
    const int pi = item_seq(0);
    if (pi >= 0) {
      pit = item_at(pi);
      pk = warp_pages(pit);
      pj = 0;
      pwb = 0;
      if (pk > 0) load_rows();
    } else {
      prod_live = false;
    }
  }
  auto issue = [&]() -> bool {  // next page into stage prod % kS; false: none (yet)
    if (!prod_live) return false;
    if (pj >= pk) {
      // move to the next item this warp has pages in
      for (;;) {
        const int pi = item_seq(pidx + 1);
        if (pi == kStall) return false;  // not claimed yet: refilled after the item
        ++pidx;
        if (pi < 0) {
          prod_live = false;
          return false;
        }
        pit = item_at(pi);
        pk = warp_pages(pit);
        pj = 0;
        pwb = 0;
        if (pk > 0) {
          load_rows();
          break;
        }
      }
    } else if (pj == pwb + 32) {
      pwb += 32;
      load_rows();
    }
    const int row = __shfl_sync(kFull, prow, pj - pwb);
    const int s = prod % kS;
    if (lane == 0) {
      uint8_t* st = ring + s * Geo::kStageBytes;
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(&ring_bar[s], Geo::kStageBytes);
#pragma unroll
      for (int hf = 0; hf < Geo::kHalves; ++hf) {
        tma_load_2d(st + hf * kTileBytes, &tmK, hf * 64, row, &ring_bar[s], policy);
        tma_load_2d(st + (Geo::kHalves + hf) * kTileBytes, &tmV, hf * 64, row, &ring_bar[s], policy);
      }
    }
    ++pj;
    ++prod;
    return true;
  };
  ADR_TL(10);
  // A warp with no pages in its first item moves on (the loop in issue()).
  if (prod_live && pk == 0) pj = pk;  // forces the advance on the first issue
  const bool pre = p.k_new != nullptr || !p.pdl;  // no appended row can be stale in smem
  if (pre) {
#pragma unroll
    for (int s = 0; s < kS; ++s) issue();
  }
  ADR_TL(1);
  if (!waited) griddep_wait();
  ADR_TL(2);
  int cons = 0;  // pages consumed by this warp (ring position)
  auto refill = [&]() {
    while (prod - cons < kS && issue()) {
    }
  };
  if (dyn) {  // the claim counter is free once the preceding kernel is done
    if (threadIdx.x == 0) claim_items(1, 2);
    __syncthreads();
    known = *reinterpret_cast<volatile int*>(&s_known);
  }
  refill();

  // ---- consumer --------------------------------------------------------------
  const int g = lane >> 2;
  const int t = lane & 3;
  const int head0 = 2 * t, head1 = 2 * t + 1;
  const int lm_j = lane >> 3;
  const int k_tok = (lane & 7) + ((lm_j & 1) << 3);
  const int k_chunk_off = lm_j >> 1;
  const int v_tok = (lane & 7) + ((lm_j >> 1) << 3);
  const int v_chunk_off = lm_j & 1;
  const uint32_t ring_s = smem_addr(ring);
  uint32_t kaddr[4], vaddr[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    kaddr[j] = ring_s + k_tok * 128 + (((2 * j + k_chunk_off) ^ (k_tok & 7)) << 4);
    vaddr[j] = ring_s + Geo::kHalves * kTileBytes + v_tok * 128 +
               (((2 * j + v_chunk_off) ^ (v_tok & 7)) << 4);
  }
  constexpr int kChunks = D / 8;
  const bool app_lane = p.k_new != nullptr && lane < 2 * kChunks;
  const bool app_is_v = lane >= kChunks;
  const int app_c = app_is_v ? lane - kChunks : lane;

  float* my = comb + warp * comb_floats;
  const int GD = G * D;

  for (int k = 0;; ++k) {  // block-uniform
    const int i = item_seq(k);
    if (i < 0) break;
    const SplitItem it = item_at(i);
    const int ck = warp_pages(it);
    const int seq = p.seq_lens[it.b];
    uint32_t qf[Geo::kKSteps][2];
    float acc[Geo::kMTiles][4];
#pragma unroll
    for (int mt = 0; mt < Geo::kMTiles; ++mt) acc[mt][0] = acc[mt][1] = acc[mt][2] = acc[mt][3] = 0.f;
    float m0 = kNegBig, m1 = kNegBig, l0 = 0.f, l1 = 0.f;
    uint4 app_val = make_uint4(0, 0, 0, 0);
    int app_page = -1;
    if (ck > 0) {
      const bool qlive = g < G;
      const __nv_bfloat16* qrow = p.q + ((size_t)(p.in_rows ? p.in_rows[it.b] : it.b) * p.Hq +
                                         (size_t)it.h * G + (qlive ? g : 0)) * D;
#pragma unroll
      for (int kk = 0; kk < Geo::kKSteps; ++kk) {  // L2-coherent: q may live on a peer GPU
        qf[kk][0] = qlive ? __ldcg(reinterpret_cast<const uint32_t*>(qrow + kk * 16 + 2 * t)) : 0u;
        qf[kk][1] = qlive ? __ldcg(reinterpret_cast<const uint32_t*>(qrow + kk * 16 + 8 + 2 * t)) : 0u;
      }
      // fused append: the warp holding the pair's last page
      if (app_lane && it.hi == it.n && (it.n - 1 - it.lo) % kW == warp) {
        const __nv_bfloat16* src =
            (app_is_v ? p.v_new : p.k_new) + ((size_t)(p.in_rows ? p.in_rows[it.b] : it.b) * Hkv + it.h) * D;
        app_val = __ldcg(reinterpret_cast<const uint4*>(src) + app_c);
        app_page = __ldg(&p.block_table[(size_t)it.b * p.max_blocks + it.n - 1]);
        if ((unsigned)app_page >= (unsigned)p.num_blocks) app_page = -1;
      }
    }
    for (int j = 0; j < ck; ++j) {
      const int s = cons % kS;
      const uint32_t phase = (uint32_t)(cons / kS) & 1u;
      ++cons;
      mbar_wait(&ring_bar[s], phase);
#ifdef ADR_TIMELINE
      if (cons == 1) ADR_TL(3);
#endif
      const uint32_t so = s * Geo::kStageBytes;
      const int pgi = it.lo + warp + kW * j;
      const bool last_page = pgi == it.n - 1;
      if (p.k_new != nullptr && last_page) {
        if (app_lane) {
          const int r = (seq - 1) & (kPage - 1);
          const int half = app_c >> 3, cc = app_c & 7;
          const uint32_t dst = ring_s + so + (app_is_v ? Geo::kHalves * kTileBytes : 0) +
                               half * kTileBytes + r * 128 + ((cc ^ (r & 7)) << 4);
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dst), "r"(app_val.x),
                       "r"(app_val.y), "r"(app_val.z), "r"(app_val.w)
                       : "memory");
          __nv_bfloat16* cache = app_is_v ? p.v_cache : p.k_cache;
          if (app_page >= 0)
            reinterpret_cast<uint4*>(cache + (((size_t)app_page * Hkv + it.h) * kPage + r) * D)[app_c] =
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
      float s00 = c[0] * p.scale_log2, s01 = c[1] * p.scale_log2;
      float s10 = c[2] * p.scale_log2, s11 = c[3] * p.scale_log2;
      if (last_page) {
        const int tok0 = pgi * kPage + g;
        if (tok0 >= seq) s00 = s01 = -INFINITY;
        if (tok0 + 8 >= seq) s10 = s11 = -INFINITY;
      }
      // ---- online softmax (log2 domain) ----
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
      const uint32_t pb0 = movmatrix_trans(x0), pb1 = movmatrix_trans(x1);
      const uint32_t pr0 = movmatrix_trans(r0), pr1 = movmatrix_trans(r1);
      // ---- O^T += V^T . P^T ----
#pragma unroll
      for (int mt = 0; mt < Geo::kMTiles; ++mt) {
        uint32_t a[4];
        ldmatrix_x4_trans(a, vaddr[mt & 3] + so + (mt >> 2) * kTileBytes);
        mma_16816(acc[mt], a, pb0, pb1);
        mma_16816(acc[mt], a, pr0, pr1);
      }
      __syncwarp();
      refill();  // into the stage just read
    }
    ADR_TL(4);
    // ---- this warp's state -> shared memory ----
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      l0 += __shfl_xor_sync(kFull, l0, o);
      l1 += __shfl_xor_sync(kFull, l1, o);
    }
#pragma unroll
    for (int mt = 0; mt < Geo::kMTiles; ++mt) {
      if (head0 < G) {
        my[head0 * kRowPad + mt * 16 + g] = acc[mt][0];
        my[head0 * kRowPad + mt * 16 + g + 8] = acc[mt][2];
      }
      if (head1 < G) {
        my[head1 * kRowPad + mt * 16 + g] = acc[mt][1];
        my[head1 * kRowPad + mt * 16 + g + 8] = acc[mt][3];
      }
    }
    if (g == 0) {
      if (head0 < G) {
        my[G * kRowPad + head0] = m0;
        my[G * kRowPad + 8 + head0] = l0;
      }
      if (head1 < G) {
        my[G * kRowPad + head1] = m1;
        my[G * kRowPad + 8 + head1] = l1;
      }
    }
    __syncthreads();
    if (dyn && threadIdx.x == 0) claim_items(k + 3, 1);  // slot of item k - 1, consumed
    // ---- combine the warps (fixed order) ----
    // per head: M = max over warps, weights w = exp2(m_w - M), L = sum w l_w
    // (lane w of warp k % W); then float4 rows A = sum_w w A_w in warp order
    for (int k = warp; k < G; k += kW) {
      const float m = lane < kW ? comb[lane * comb_floats + G * kRowPad + k] : kNegBig;
      const float l = lane < kW ? comb[lane * comb_floats + G * kRowPad + 8 + k] : 0.f;
      float M = m;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(kFull, M, o));
      const float w = lane < kW ? exp2f(m - M) : 0.f;
      float L = w * l;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(kFull, L, o);
      if (lane < kW) hst[16 + lane * 8 + k] = w;
      if (lane == 0) {
        hst[k] = M;
        hst[8 + k] = L;
      }
    }
    __syncthreads();
    const size_t orow0 = (size_t)(p.out_rows ? p.out_rows[it.b] : it.b) * p.Hq + (size_t)it.h * G;
    float* slot = p.part + (size_t)i * p.slot_floats;
    const int F = GD / 4;  // float4 of the G x D rows
    for (int f = threadIdx.x; f < F; f += kThreads) {
      const int k = (4 * f) / D, d = 4 * f - k * D;
      float4 A = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int w = 0; w < kW; ++w) {
        const float wt = hst[16 + w * 8 + k];
        const float4 c = *reinterpret_cast<const float4*>(comb + w * comb_floats + k * kRowPad + d);
        A.x += wt * c.x;
        A.y += wt * c.y;
        A.z += wt * c.z;
        A.w += wt * c.w;
      }
      if (it.ns == 1) {
        const float inv = 1.f / hst[8 + k];
        store_row4(p, (orow0 + k) * D + d, A, inv);
        if (p.lse != nullptr && d == 0) p.lse[orow0 + k] = (hst[k] + __log2f(hst[8 + k])) * kLn2;
      } else {
        *reinterpret_cast<float4*>(slot + k * D + d) = A;
        if (d == 0) {
          slot[GD + k] = hst[k];
          slot[GD + 8 + k] = hst[8 + k];
        }
      }
    }
    if (it.ns > 1) {
      // publish the partial; the CTA publishing the pair's last one merges them
      __syncthreads();
      int32_t* arrivals = p.counter + (size_t)it.b * Hkv + it.h;
      if (threadIdx.x == 0) s_last = atom_add_acq_rel_s32(arrivals, 1) == it.ns - 1;
      __syncthreads();
      if (s_last) {
        // Merge the ns pieces in piece order, in chunks whose statistics fit in
        // shared memory (usually one): per chunk, the piece statistics are
        // staged once, turned into per-(piece, head) weights with a running
        // max, and every thread folds its float4 rows in with all of the
        // chunk's loads in flight (no serial round trips per piece).
        const float* base = p.part + (size_t)(i - it.s) * p.slot_floats;
        const int cap = (kW * comb_floats) / (2 * G);  // pieces per chunk (m and l staged)
        float* wq = comb;              // [chunk][G] m, then weights (comb is free now)
        float* lq = comb + cap * G;    // [chunk][G] l
        float4 A[kFpt];
#pragma unroll
        for (int r = 0; r < kFpt; ++r) A[r] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (threadIdx.x < G) {
          hst[threadIdx.x] = kNegBig;       // running M per head
          hst[8 + threadIdx.x] = 0.f;       // running L per head
        }
        for (int q0 = 0; q0 < it.ns; q0 += cap) {
          const int nq = min(cap, it.ns - q0);
          // the rows of the chunk's first 8 pieces go out together with the
          // statistics: one round trip for the common (ns <= 8) merge
          float4 v[kFpt][8];
#pragma unroll
          for (int r = 0; r < kFpt; ++r) {
            const int f = threadIdx.x + r * kThreads;
#pragma unroll
            for (int j = 0; j < 8; ++j)
              v[r][j] = (f < F && j < nq)
                            ? __ldcg(reinterpret_cast<const float4*>(base + (size_t)(q0 + j) * p.slot_floats) + f)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
          }
          for (int x = threadIdx.x; x < nq * G; x += kThreads) {
            const float* st = base + (size_t)(q0 + x / G) * p.slot_floats + GD + x % G;
            wq[x] = __ldcg(st);
            lq[x] = __ldcg(st + 8);
          }
          __syncthreads();
          for (int k = warp; k < G; k += kW) {
            float M = hst[k];
            for (int j = lane; j < nq; j += 32) M = fmaxf(M, wq[j * G + k]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(kFull, M, o));
            float Ls = 0.f;
            for (int j = lane; j < nq; j += 32) {
              const float w = exp2f(wq[j * G + k] - M);
              Ls += w * lq[j * G + k];
              wq[j * G + k] = w;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) Ls += __shfl_xor_sync(kFull, Ls, o);
            __syncwarp();
            if (lane == 0) {
              const float r = exp2f(hst[k] - M);  // rescale of the chunks before
              hst[16 + k] = r;
              hst[8 + k] = hst[8 + k] * r + Ls;
              hst[k] = M;
            }
          }
          __syncthreads();
#pragma unroll
          for (int r = 0; r < kFpt; ++r) {
            const int f = threadIdx.x + r * kThreads;
            if (f < F) {
              const int k = (4 * f) / D;
              const float rs = hst[16 + k];
              A[r].x *= rs;
              A[r].y *= rs;
              A[r].z *= rs;
              A[r].w *= rs;
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float w = j < nq ? wq[j * G + k] : 0.f;
                A[r].x += w * v[r][j].x;
                A[r].y += w * v[r][j].y;
                A[r].z += w * v[r][j].z;
                A[r].w += w * v[r][j].w;
              }
              for (int j0 = 8; j0 < nq; j0 += 8) {
                float4 u[8];
#pragma unroll
                for (int j = 0; j < 8; ++j)
                  u[j] = j0 + j < nq ? __ldcg(reinterpret_cast<const float4*>(
                                           base + (size_t)(q0 + j0 + j) * p.slot_floats) + f)
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                  const float w = j0 + j < nq ? wq[(j0 + j) * G + k] : 0.f;
                  A[r].x += w * u[j].x;
                  A[r].y += w * u[j].y;
                  A[r].z += w * u[j].z;
                  A[r].w += w * u[j].w;
                }
              }
            }
          }
          __syncthreads();  // wq, lq and the running statistics are reused by the next chunk
        }
#pragma unroll
        for (int r = 0; r < kFpt; ++r) {
          const int f = threadIdx.x + r * kThreads;
          if (f < F) {
            const int k = (4 * f) / D, d = 4 * f - k * D;
            store_row4(p, (orow0 + k) * D + d, A[r], 1.f / hst[8 + k]);
            if (p.lse != nullptr && d == 0) p.lse[orow0 + k] = (hst[k] + __log2f(hst[8 + k])) * kLn2;
          }
        }
        // every thread has consumed the pieces (the last __syncthreads): drop them from L2
        const int lines = (GD + 16 + 31) / 32;
        for (int x = threadIdx.x; x < it.ns * lines; x += kThreads) {
          const int q = x / lines, ln = x - q * lines;
          discard_l2_line(base + (size_t)q * p.slot_floats + ln * 32);
        }
        if (threadIdx.x == 0) *arrivals = 0;  // every piece has arrived: free for the next call
      }
    }
    __syncthreads();  // comb is rewritten by the next item
    if (dyn) {
      known = *reinterpret_cast<volatile int*>(&s_known);
      refill();  // a producer that reached an unclaimed item resumes
    }
    ADR_TL(5);
  }
  if (dyn && threadIdx.x == 0) {  // the last CTA out frees the claim counter for the next call
    if (atom_add_acq_rel_s32(dyn_claim + 1, 1) == (int)gridDim.x - 1) {
      dyn_claim[0] = 0;
      dyn_claim[1] = 0;
    }
  }
  ADR_TL(11);
}

// (warps per CTA, pages in flight per warp, CTAs per SM); index 0 is the default.
#define ADR_SPLIT_VARIANTS(X) \
  X(0, 4, 3, 2)               \
  X(1, 4, 2, 3)               \
  X(2, 8, 2, 1)               \
  X(3, 8, 3, 1)               \
  X(4, 4, 4, 1)               \
  X(5, 2, 4, 3)
constexpr int kNumSplitVariants = 6;

constexpr int kMaxDevices = 64;

template <int D, int W, int S>
size_t split_smem_bytes(int B, int G) {
  return 1024 + (size_t)W * S * Geometry<D>::kStageBytes + (size_t)W * S * 8 +
         (size_t)W * (G * (D + 4) + 16) * 4 + (size_t)(16 + 8 * W) * 4 + (size_t)(2 * (B + 1)) * 4;
}

template <int D, int W, int S, int C>
int launch_split_variant(const CUtensorMap& tmK, const CUtensorMap& tmV, const DecodeArgs& a,
                         int sms, bool pdl, int dev, cudaStream_t stream) {
  auto kern = decode_split_kernel<D, W, S, C>;
  static std::atomic<bool> configured[kMaxDevices];
  if (dev < 0 || dev >= kMaxDevices) return fail(ADR_ERR_UNSUPPORTED, "device %d", dev);
  if (!configured[dev].load(std::memory_order_acquire)) {
    if (!cuda_ok(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)split_smem_bytes<D, W, S>(kMaxBatch, 8)),
                 "cudaFuncSetAttribute(decode_split_kernel)"))
      return ADR_ERR_CUDA;
    configured[dev].store(true, std::memory_order_release);
  }
  const size_t smem = split_smem_bytes<D, W, S>(a.B, a.G);
  int fit = 0;
  if (!cuda_ok(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fit, kern, W * 32, smem),
               "cudaOccupancyMaxActiveBlocksPerMultiprocessor"))
    return ADR_ERR_CUDA;
  const int ctas = sms * (fit < C ? (fit > 0 ? fit : 1) : C);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(W * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cuda_ok(cudaLaunchKernelEx(&cfg, kern, tmK, tmV, a), "decode_split_kernel launch")
             ? ADR_OK : ADR_ERR_CUDA;
}

}  // namespace

// Variant for a call: ADR_SPLIT_VARIANT if set, else 4x3x2 (24 pages in flight
// per SM) for G <= 4, and 4x2x3 for G > 4, where the larger combine buffers
// leave room for one 4x3x2 CTA per SM only (12 pages in flight) but for two
// 4x2x3 CTAs (16): 7-22% faster on GQA-8 calls (profiles/split_gqa8_r02q.txt).
int split_variant(int G) {
  static int env = [] {
    const char* e = getenv("ADR_SPLIT_VARIANT");
    const int x = e ? atoi(e) : -1;
    return (x >= 0 && x < kNumSplitVariants) ? x : -1;
  }();
  return env >= 0 ? env : (G > 4 ? 1 : 0);
}

// Launch the split-pair kernel for D in {64, 128} (called by adr_paged_decode_attn_rows).
int launch_decode_split(const CUtensorMap& tmK, const CUtensorMap& tmV, const DecodeArgs& a, int D,
                        int sms, bool pdl, int dev, cudaStream_t s) {
  const int v = split_variant(a.G);
  switch (v) {
#define ADR_SPLIT_CASE(I, W, S, C)                                                        \
  case I:                                                                                 \
    return D == 128 ? launch_split_variant<128, W, S, C>(tmK, tmV, a, sms, pdl, dev, s)   \
                    : launch_split_variant<64, W, S, C>(tmK, tmV, a, sms, pdl, dev, s);
    ADR_SPLIT_VARIANTS(ADR_SPLIT_CASE)
#undef ADR_SPLIT_CASE
    default: return fail(ADR_ERR_INVALID, "bad split variant");
  }
}

}  // namespace adr

#ifdef ADR_TIMELINE
extern "C" ADR_API int32_t adr_debug_timeline_split(void* dst, size_t bytes) {
  using adr::dec::g_timeline;
  return cudaMemcpyFromSymbol(dst, g_timeline, bytes < sizeof(g_timeline) ? bytes : sizeof(g_timeline)) ==
                 cudaSuccess
             ? 0
             : -3;
}
#endif
