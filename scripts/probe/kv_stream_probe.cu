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
};

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
    if (lane == 0) {
      const uint64_t pol = make_policy(a.hint);
      for (int k = 0; k < n; ++k) {
        const int s = k % S;
        if (k >= S) mbar_wait(&empty[s], ((k / S) - 1) & 1);
        uint8_t* st = smem + (size_t)s * kStage;
        const long long u0 = lo + (long long)k * P;
        const int cnt = (int)min((long long)P, hi - u0);
        mbar_arrive_expect_tx(&full[s], 2 * kPageBytes * cnt);
        for (int j = 0; j < cnt; ++j) {
          const size_t off = (size_t)a.rows[u0 + j] * D * 2;
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
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const double bytes = 2.0 * U * kPageBytes;

  auto run = [&](int W, int S, int C, int P, int hint, int order, int spin) {
    Args a{rows_by_order[order], nullptr, nullptr, U, spin, P, S, hint, sink};
    const bool prod = W < 0;
    const int warps = prod ? -W + 1 : W;
    const size_t stage = (size_t)2 * kPageBytes * P;
    const size_t smem = prod ? 1024 + S * stage + 16 * S : 1024 + (size_t)W * S * stage + W * S * 8;
    auto kern = prod ? producer_kernel : warp_ring_kernel;
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
    auto launch = [&](int i) {
      a.k = K[i % nbuf];
      a.v = V[i % nbuf];
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
    const size_t inflight = prod ? S * stage * C : W * S * stage * C;
    printf("%s W=%d S=%d C=%d P=%d hint=%d order=%d spin=%d: %7.1f us %7.1f GB/s (smem ring/SM %zu KiB)\n",
           prod ? "producer " : "warp-ring", W, S, C, P, hint, order, spin, us, bytes / us / 1e3,
           inflight >> 10);
    fflush(stdout);
  };
  std::vector<std::string> cfgs;
  for (int i = 1; i < argc; ++i) cfgs.push_back(argv[i]);
  if (cfgs.empty())
    cfgs = {
        "4,2,3,1,1,0,0", "4,2,3,1,0,0,0", "4,2,3,1,2,0,0", "4,2,3,1,1,1,0", "4,2,3,1,1,2,0",
        "4,1,3,2,1,0,0", "4,1,6,1,1,0,0", "8,1,3,1,1,0,0", "2,1,6,2,1,0,0", "4,1,2,3,1,0,0",
        "1,2,12,1,1,0,0", "1,1,24,1,1,0,0", "16,1,1,1,1,0,0", "12,2,1,1,1,0,0",
        "-4,24,1,1,1,0,0", "-8,24,1,1,1,0,0", "-8,12,1,2,1,0,0", "-8,6,1,4,1,0,0",
        "-4,12,2,1,1,0,0", "-4,6,2,2,1,0,0", "-8,26,1,1,1,0,0", "-12,24,1,1,1,0,0",
        "-8,24,1,1,0,0,0", "-8,24,1,1,1,1,0",
        "4,2,3,1,1,0,300", "-8,24,1,1,1,0,300", "-8,24,1,1,1,0,1000", "4,2,3,1,1,0,1000",
    };
  for (const std::string& c : cfgs) {
    int v[7] = {4, 2, 3, 1, 1, 0, 0};
    sscanf(c.c_str(), "%d,%d,%d,%d,%d,%d,%d", &v[0], &v[1], &v[2], &v[3], &v[4], &v[5], &v[6]);
    run(v[0], v[1], v[2], v[3], v[4], v[5], v[6]);
  }
  return 0;
}
