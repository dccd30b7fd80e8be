// KV-streaming probe (diagnostic, not product code): how fast can the C2 paged
// KV cache be streamed into shared memory with no attention math at all, for
// different load shapes, in-flight depths, unit orders and cache hints? It
// separates "memory pipeline limit" from "consumer turnaround limit" for
// paged_decode_attn.
//
// Layout = the product's: K, V [num_pages, Hkv, 16, D] bf16, (Llama-2-7B C2:
// B=64, ctx 4096, Hkv=32, D=128), pages a seeded random permutation.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o kv_stream_probe \
//        kv_stream_probe.cu -L/usr/local/cuda/lib64/stubs -lcuda
//   ./kv_stream_probe [W,S,C,PPS,hint,order,spin ...]    (defaults: a built-in sweep)
//     W warps/CTA, S stages per warp, C CTAs/SM, PPS pages (K+V) per stage,
//     hint 0 none / 1 evict_first / 2 evict_normal,
//     order 0 (request, head, page) / 1 (request, page, head) / 2 sequential pages,
//     spin: fake consumer work per page (SM cycles).
//   Producer-warp variant: W<0 -> |W| consumer warps + 1 producer warp sharing a
//   CTA ring of S stages.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <random>
#include <string>
#include <vector>

#include "../../paper_2503_20552_b200/csrc/adr_device.cuh"

using namespace adr;

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e = (x);                                                             \
    if (e != cudaSuccess) {                                                          \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

constexpr int D = 128, kPage = 16;
constexpr int kPageBytes = kPage * D * 2;  // 4 KiB per (page, head) for K or for V

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar, uint64_t policy, int hint) {
  if (hint) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
        : "memory");
  } else {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1], %2, [%3];" ::"r"(smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
  }
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

struct Args {
  const int32_t* rows;  // [U] page row (page*Hkv + h)*16 per unit
  const uint8_t* k;
  const uint8_t* v;
  long long U;
  int spin, pps, stages, hint;
  unsigned* sink;
  unsigned long long* t_end;  // [warps] globaltimer at each warp's (or CTA's) last page
  int chunk;                  // > 0: dynamic claiming of `chunk`-unit chunks (warp ring)
  int static_pct;             // dyn: this % of the units split statically first, the rest pooled
  unsigned* counter;          // this launch's chunk counter (zero at launch)
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint64_t make_policy(int hint) {
  uint64_t pol = 0;
  if (hint == 1) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  if (hint == 2) asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ void fake_work(int spin) {
  if (spin > 0) {
    const long long t0 = clock64();
    while (clock64() - t0 < spin) {}
  }
}

// Per-warp rings (the product's structure): each warp issues its own loads.
__global__ void warp_ring_kernel(Args a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x >> 5;
  const int S = a.stages, P = a.pps;
  const int kStage = 2 * kPageBytes * P;
  uint8_t* ring = smem + (size_t)warp * S * kStage;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)W * S * kStage) + warp * S;
  if (lane < S) mbar_init(&bars[lane], 1);
  fence_mbar_init();
  __syncwarp();
  const long long NW = (long long)gridDim.x * W;
  const long long gw = (long long)warp * gridDim.x + blockIdx.x;
  const long long lo = gw * a.U / NW, hi = (gw + 1) * a.U / NW;
  const int n = (int)((hi - lo + P - 1) / P);  // stages of P units
  const uint64_t pol = make_policy(a.hint);
  auto issue = [&](int k, int s) {
    if (lane == 0) {
      uint8_t* st = ring + s * kStage;
      const long long u0 = lo + (long long)k * P;
      const int cnt = (int)min((long long)P, hi - u0);
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(&bars[s], 2 * kPageBytes * cnt);
      for (int j = 0; j < cnt; ++j) {
        const size_t off = (size_t)a.rows[u0 + j] * D * 2;
        bulk_load(st + j * kPageBytes, a.k + off, kPageBytes, &bars[s], pol, a.hint);
        bulk_load(st + (P + j) * kPageBytes, a.v + off, kPageBytes, &bars[s], pol, a.hint);
      }
    }
  };
  for (int k = 0; k < S && k < n; ++k) issue(k, k);
  unsigned x = 0;
  uint32_t phase = 0;
  for (int i = 0; i < n; ++i) {
    const int s = i % S;
    mbar_wait(&bars[s], phase);
    x ^= *reinterpret_cast<const unsigned*>(ring + s * kStage + lane * 4);
    fake_work(a.spin * P);
    __syncwarp();
    if (i + S < n) issue(i + S, s);
    if (s == S - 1) phase ^= 1u;
  }
  if (lane == 0) a.t_end[gw] = gtimer();
  if (x == 0x12345678u) a.sink[0] = x;
}

// Per-warp rings with dynamic work: warps claim `chunk`-unit chunks from a
// global counter (claims run kStages ahead with the loads), so fast warps take
// more chunks and all warps finish together.
template <int S>
__global__ void dyn_ring_kernel(Args a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x >> 5;
  constexpr int kStage = 2 * kPageBytes;
  uint8_t* ring = smem + (size_t)warp * S * kStage;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)W * S * kStage) + warp * S;
  if (lane < S) mbar_init(&bars[lane], 1);
  fence_mbar_init();
  __syncwarp();
  const long long gw = (long long)warp * gridDim.x + blockIdx.x;
  const uint64_t pol = make_policy(a.hint);
  const long long NW = (long long)gridDim.x * W;
  const long long Us = a.U * a.static_pct / 100;  // static part
  const long long nchunks = (a.U - Us + a.chunk - 1) / a.chunk;
  // producer cursor: current range [cu, ce); first the warp's static range
  long long cu = gw * Us / NW, ce = (gw + 1) * Us / NW;
  // static_pct < 0: guided tiers — tier t hands out NW segments of
  // max(chunk, U / (2^(t+1) NW)) units, then `chunk`-unit segments to the end.
  const bool guided = a.static_pct < 0;
  auto segment = [&](long long c, long long& st, long long& en) -> bool {
    long long base = 0;
    for (int t = 0; t < 40; ++t) {
      long long sz = (a.U >> (t + 1)) / NW;
      if (sz <= a.chunk) break;
      if (c < NW) {
        st = base + c * sz;
        en = min(a.U, st + sz);
        return st < a.U;
      }
      c -= NW;
      base += NW * sz;
    }
    st = base + c * a.chunk;
    en = min(a.U, st + a.chunk);
    return st < a.U;
  };
  if (guided) cu = ce = 0;
  auto next_unit = [&]() -> long long {
    if (cu >= ce) {
      unsigned c = 0;
      if (lane == 0) c = atomicAdd(a.counter, 1u);
      c = __shfl_sync(kFull, c, 0);
      if (guided) {
        if (!segment(c, cu, ce)) return -1;
      } else {
        if (c >= nchunks) return -1;
        cu = Us + (long long)c * a.chunk;
        ce = min(a.U, cu + a.chunk);
      }
    }
    return cu++;
  };
  bool live[S];
  auto issue = [&](int s) {
    const long long u = next_unit();
    live[s] = u >= 0;
    if (u >= 0 && lane == 0) {
      uint8_t* st = ring + s * kStage;
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(&bars[s], kStage);
      const size_t off = (size_t)a.rows[u] * D * 2;
      bulk_load(st, a.k + off, kPageBytes, &bars[s], pol, a.hint);
      bulk_load(st + kPageBytes, a.v + off, kPageBytes, &bars[s], pol, a.hint);
    }
  };
#pragma unroll
  for (int s = 0; s < S; ++s) issue(s);
  unsigned x = 0;
  uint32_t phase = 0;
  bool done = false;
  while (!done) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      if (done || !live[s]) {  // claims are monotonic: the first dead stage ends the stream
        done = true;
        continue;
      }
      mbar_wait(&bars[s], phase);
      x ^= *reinterpret_cast<const unsigned*>(ring + s * kStage + lane * 4);
      fake_work(a.spin);
      __syncwarp();
      issue(s);
    }
    phase ^= 1u;
  }
  if (lane == 0) a.t_end[gw] = gtimer();
  if (x == 0x12345678u) a.sink[0] = x;
}

// One producer warp per CTA fills a CTA ring of S stages (P pages each); the
// consumer warps take stages round-robin (stage i -> consumer i % Wc) and
// release them on an "empty" barrier. CTA range = contiguous units.
__global__ void producer_kernel(Args a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int Wc = (blockDim.x >> 5) - 1;
  const int S = a.stages, P = a.pps;
  const int kStage = 2 * kPageBytes * P;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * kStage);
  uint64_t* empty = full + S;
  if (threadIdx.x < S) {
    mbar_init(&full[threadIdx.x], 1);
    mbar_init(&empty[threadIdx.x], 1);
  }
  fence_mbar_init();
  __syncthreads();
  const long long lo = (long long)blockIdx.x * a.U / gridDim.x;
  const long long hi = (long long)(blockIdx.x + 1) * a.U / gridDim.x;
  const int n = (int)((hi - lo + P - 1) / P);
  if (warp == Wc) {  // producer
    const uint64_t pol = make_policy(a.hint);
    long long wbase = lo;  // rows of units [wbase, wbase + 32) held one per lane
    int myrow = (wbase + lane < hi) ? a.rows[wbase + lane] : 0;
    int nxtrow = (wbase + 32 + lane < hi) ? a.rows[wbase + 32 + lane] : 0;
    for (int k = 0; k < n; ++k) {
      const int s = k % S;
      if (k >= S) mbar_wait(&empty[s], ((k / S) - 1) & 1);
      uint8_t* st = smem + (size_t)s * kStage;
      const long long u0 = lo + (long long)k * P;
      const int cnt = (int)min((long long)P, hi - u0);
      if (lane == 0) mbar_arrive_expect_tx(&full[s], 2 * kPageBytes * cnt);
      for (int j = 0; j < cnt; ++j) {
        const long long u = u0 + j;
        if (u >= wbase + 32) {
          wbase += 32;
          myrow = nxtrow;
          nxtrow = (wbase + 32 + lane < hi) ? a.rows[wbase + 32 + lane] : 0;
        }
        const int row = __shfl_sync(kFull, myrow, (int)(u - wbase));
        if (lane == 0) {
          const size_t off = (size_t)row * D * 2;
          bulk_load(st + j * kPageBytes, a.k + off, kPageBytes, &full[s], pol, a.hint);
          bulk_load(st + (P + j) * kPageBytes, a.v + off, kPageBytes, &full[s], pol, a.hint);
        }
      }
    }
    return;
  }
  unsigned x = 0;
  for (int k = warp; k < n; k += Wc) {
    const int s = k % S;
    mbar_wait(&full[s], (k / S) & 1);
    x ^= *reinterpret_cast<const unsigned*>(smem + (size_t)s * kStage + lane * 4);
    fake_work(a.spin * P);
    __syncwarp();
    if (lane == 0) {
      fence_proxy_async_smem();
      mbar_arrive(&empty[s]);
    }
  }
  if (lane == 0) a.t_end[(long long)blockIdx.x * Wc + warp] = gtimer();
  if (x == 0x12345678u) a.sink[0] = x;
}

int main(int argc, char** argv) {
  const int B = 64, Hkv = 32, ctx = 4096;
  const int ppr = ctx / kPage;
  const int num_pages = B * ppr;
  const long long U = (long long)B * Hkv * ppr;
  const size_t cache_bytes = (size_t)num_pages * Hkv * kPageBytes;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int nbuf = 4;  // distinct caches cycled (>> L2)
  std::vector<uint8_t*> K(nbuf), V(nbuf);
  for (int i = 0; i < nbuf; ++i) {
    CK(cudaMalloc(&K[i], cache_bytes));
    CK(cudaMalloc(&V[i], cache_bytes));
    CK(cudaMemset(K[i], 1, cache_bytes));
    CK(cudaMemset(V[i], 2, cache_bytes));
  }
  std::vector<int> perm(num_pages);
  std::iota(perm.begin(), perm.end(), 0);
  std::shuffle(perm.begin(), perm.end(), std::mt19937(1));
  auto build_rows = [&](int order) {
    std::vector<int32_t> rows(U);
    long long u = 0;
    for (int b = 0; b < B; ++b) {
      if (order == 1) {
        for (int p = 0; p < ppr; ++p)
          for (int h = 0; h < Hkv; ++h) rows[u++] = (perm[b * ppr + p] * Hkv + h) * kPage;
      } else {
        for (int h = 0; h < Hkv; ++h)
          for (int p = 0; p < ppr; ++p) {
            const int pg = order == 2 ? b * ppr + p : perm[b * ppr + p];
            rows[u++] = (pg * Hkv + h) * kPage;
          }
      }
    }
    int32_t* d;
    CK(cudaMalloc(&d, U * 4));
    CK(cudaMemcpy(d, rows.data(), U * 4, cudaMemcpyHostToDevice));
    return d;
  };
  int32_t* rows_by_order[3] = {build_rows(0), build_rows(1), build_rows(2)};
  unsigned* sink;
  CK(cudaMalloc(&sink, 4));
  unsigned long long* t_end;
  const int max_warps = sms * 64;
  CK(cudaMalloc(&t_end, (size_t)max_warps * 8));
  unsigned long long* t_start;
  CK(cudaMalloc(&t_start, 8));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const double bytes = 2.0 * U * kPageBytes;

  unsigned* counters;
  CK(cudaMalloc(&counters, 4096 * 4));
  auto run = [&](int W, int S, int C, int P, int hint, int order, int spin, int chunk, int spct) {
    Args a{rows_by_order[order], nullptr, nullptr, U, spin, P, S, hint, sink, t_end, chunk,
           spct, counters};
    const bool prod = W < 0;
    const int warps = prod ? -W + 1 : W;
    const size_t stage = (size_t)2 * kPageBytes * P;
    const size_t smem = prod ? 1024 + S * stage + 16 * S : 1024 + (size_t)W * S * stage + W * S * 8;
    auto kern = prod ? producer_kernel : warp_ring_kernel;
    if (chunk > 0) {
      if (S == 2) kern = dyn_ring_kernel<2>;
      else if (S == 3) kern = dyn_ring_kernel<3>;
      else if (S == 4) kern = dyn_ring_kernel<4>;
      else { printf("dyn needs S in 2..4\n"); return; }
    }
    if (smem > 232448 ||
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess) {
      printf("W=%d S=%d C=%d P=%d skipped (smem %zu)\n", W, S, C, P, smem);
      cudaGetLastError();
      return;
    }
    int fit = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fit, kern, warps * 32, smem);
    if (fit < C) {
      printf("W=%d S=%d C=%d P=%d skipped (fit %d)\n", W, S, C, P, fit);
      return;
    }
    int launch_id = 0;
    auto launch = [&](int i) {
      a.k = K[i % nbuf];
      a.v = V[i % nbuf];
      if (launch_id % 4096 == 0) CK(cudaMemsetAsync(counters, 0, 4096 * 4));
      a.counter = counters + (launch_id++ % 4096);
      kern<<<sms * C, warps * 32, smem>>>(a);
    };
    for (int i = 0; i < 8; ++i) launch(i);
    CK(cudaDeviceSynchronize());
    const int reps = 40;
    CK(cudaEventRecord(e0));
    for (int i = 0; i < reps; ++i) launch(i);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double us = 1e3 * ms / reps;
    // completion spread of one isolated launch: when do warps finish, relative
    // to the last one? (a long spread = a bandwidth tail)
    const int nw = prod ? sms * C * (-W) : sms * C * W;
    CK(cudaMemset(t_end, 0, (size_t)max_warps * 8));
    CK(cudaDeviceSynchronize());
    launch(0);
    CK(cudaDeviceSynchronize());
    std::vector<unsigned long long> te(nw);
    CK(cudaMemcpy(te.data(), t_end, nw * 8, cudaMemcpyDeviceToHost));
    std::sort(te.begin(), te.end());
    const double last = (double)te[nw - 1];
    auto q = [&](double f) { return (last - (double)te[(size_t)(f * (nw - 1))]) / 1e3; };
    const size_t inflight = prod ? S * stage * C : W * S * stage * C;
    printf("%s static=%d%% chunk=%d W=%d S=%d C=%d P=%d hint=%d order=%d spin=%d: %7.1f us %7.1f GB/s (smem ring/SM %zu KiB)"
           " finish before last: p0 %.1f p10 %.1f p50 %.1f p90 %.1f us\n",
           prod ? "producer " : (chunk > 0 ? "dyn-ring " : "warp-ring"), spct, chunk, W, S, C, P, hint,
           order, spin, us, bytes / us / 1e3,
           inflight >> 10, q(0), q(0.1), q(0.5), q(0.9));
    fflush(stdout);
  };
  std::vector<std::string> cfgs;
  for (int i = 1; i < argc; ++i) cfgs.push_back(argv[i]);
  if (cfgs.empty())
    cfgs = {
        "4,2,3,1,1,0,0", "4,4,1,1,1,0,0", "4,2,3,1,1,1,0",
        "-4,24,1,1,1,0,0", "-8,24,1,1,1,0,0", "-8,12,1,2,1,0,0", "-4,12,2,1,1,0,0",
        "-2,12,2,1,1,0,0", "-12,24,1,1,1,0,0", "-8,24,1,1,1,1,0",
        "-8,24,1,1,1,0,300", "-8,24,1,1,1,0,1000", "4,2,3,1,1,0,300", "4,2,3,1,1,0,1000",
    };
  for (const std::string& c : cfgs) {
    int v[9] = {4, 2, 3, 1, 1, 0, 0, 0, 0};
    sscanf(c.c_str(), "%d,%d,%d,%d,%d,%d,%d,%d,%d", &v[0], &v[1], &v[2], &v[3], &v[4], &v[5],
           &v[6], &v[7], &v[8]);
    run(v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7], v[8]);
  }
  return 0;
}
