// Byte-moving kernels of the decode step: fused KV append (the per-step KV
// growth of engine.py:416-421 made real) and the offload exchange packing /
// scattering (the q/k/v send and output return priced at engine.py:436-438).
//
// All of them are pure 16-byte vector copies: HBM-bound, one warp (or CTA) per
// row, no shared memory. Indices come from device-resident int32/int64 tables
// so the calls are graph-capturable.
#include "adr_internal.h"

namespace adr {
namespace {

using vec16 = uint4;

// One warp per (request, kv-head): the warp's first half copies the K row, the
// second half the V row (D=128 -> 16 lanes x 16 B each).
__global__ void __launch_bounds__(128)
kv_append_kernel(const __nv_bfloat16* __restrict__ k_new, const __nv_bfloat16* __restrict__ v_new,
                 __nv_bfloat16* __restrict__ k_cache, __nv_bfloat16* __restrict__ v_cache,
                 const int64_t* __restrict__ slots, int B, int Hkv, int D, int block_size,
                 int64_t num_blocks) {
  const int pair = blockIdx.x * 4 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (pair >= B * Hkv) return;
  const int b = pair / Hkv;
  const int h = pair - b * Hkv;
  const int64_t slot = slots[b];
  if (slot < 0) return;  // padded row
  const int64_t page = slot / block_size;
  if (page >= num_blocks) return;  // out-of-range slot: ignored (see header)
  const int off = (int)(slot - page * block_size);
  const int chunks = D / 8;  // 16-byte chunks per row
  const size_t src = ((size_t)b * Hkv + h) * D;
  const size_t dst = (((size_t)page * Hkv + h) * block_size + off) * D;
  for (int c = lane; c < 2 * chunks; c += 32) {
    const bool is_v = c >= chunks;
    const int cc = is_v ? c - chunks : c;
    const vec16 val = __ldg(reinterpret_cast<const vec16*>((is_v ? v_new : k_new) + src) + cc);
    reinterpret_cast<vec16*>((is_v ? v_cache : k_cache) + dst)[cc] = val;
  }
}

// Message row i = [ q[r] | k[r] | v[r] ], r = row_idx[i]; one CTA per row.
__global__ void __launch_bounds__(256)
pack_qkv_kernel(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k,
                const __nv_bfloat16* __restrict__ v, const int32_t* __restrict__ row_idx, int Hq,
                int Hkv, int D, __nv_bfloat16* __restrict__ dst) {
  const int i = blockIdx.x;
  const int r = row_idx[i];
  const int qc = Hq * D / 8, kc = Hkv * D / 8;
  const int row_chunks = qc + 2 * kc;
  vec16* out = reinterpret_cast<vec16*>(dst) + (size_t)i * row_chunks;
  const vec16* qs = reinterpret_cast<const vec16*>(q) + (size_t)r * qc;
  const vec16* ks = reinterpret_cast<const vec16*>(k) + (size_t)r * kc;
  const vec16* vs = reinterpret_cast<const vec16*>(v) + (size_t)r * kc;
  for (int c = threadIdx.x; c < row_chunks; c += blockDim.x) {
    vec16 val;
    if (c < qc) val = __ldg(qs + c);
    else if (c < qc + kc) val = __ldg(ks + (c - qc));
    else val = __ldg(vs + (c - qc - kc));
    out[c] = val;
  }
}

__global__ void __launch_bounds__(256)
unpack_qkv_kernel(const __nv_bfloat16* __restrict__ msg, int Hq, int Hkv, int D,
                  __nv_bfloat16* __restrict__ q, __nv_bfloat16* __restrict__ k,
                  __nv_bfloat16* __restrict__ v) {
  const int i = blockIdx.x;
  const int qc = Hq * D / 8, kc = Hkv * D / 8;
  const int row_chunks = qc + 2 * kc;
  const vec16* in = reinterpret_cast<const vec16*>(msg) + (size_t)i * row_chunks;
  for (int c = threadIdx.x; c < row_chunks; c += blockDim.x) {
    const vec16 val = __ldg(in + c);
    if (c < qc) reinterpret_cast<vec16*>(q)[(size_t)i * qc + c] = val;
    else if (c < qc + kc) reinterpret_cast<vec16*>(k)[(size_t)i * kc + (c - qc)] = val;
    else reinterpret_cast<vec16*>(v)[(size_t)i * kc + (c - qc - kc)] = val;
  }
}

__global__ void __launch_bounds__(256)
scatter_out_kernel(const __nv_bfloat16* __restrict__ src, const int32_t* __restrict__ row_idx,
                   int row_chunks, __nv_bfloat16* __restrict__ out) {
  const int i = blockIdx.x;
  const int r = row_idx[i];
  const vec16* s = reinterpret_cast<const vec16*>(src) + (size_t)i * row_chunks;
  vec16* d = reinterpret_cast<vec16*>(out) + (size_t)r * row_chunks;
  for (int c = threadIdx.x; c < row_chunks; c += blockDim.x) d[c] = __ldg(s + c);
}

// Page migration: dst page dst_pages[i] <- src page src_pages[i] for K and V
// (one CTA per page; 2 x Hkv x 16 x D x 2 bytes). src may live on a peer GPU
// (peer-mapped pointer): the loads then travel over NVLink.
__global__ void __launch_bounds__(256)
kv_transfer_kernel(const uint4* __restrict__ src_k, const uint4* __restrict__ src_v,
                   const int32_t* __restrict__ src_pages, uint4* __restrict__ dst_k,
                   uint4* __restrict__ dst_v, const int32_t* __restrict__ dst_pages,
                   int page_chunks) {
  const int i = blockIdx.x;
  const size_t s = (size_t)src_pages[i] * page_chunks;
  const size_t d = (size_t)dst_pages[i] * page_chunks;
  for (int c = threadIdx.x; c < 2 * page_chunks; c += blockDim.x) {
    if (c < page_chunks) dst_k[d + c] = src_k[s + c];
    else dst_v[d + c - page_chunks] = src_v[s + c - page_chunks];
  }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace
}  // namespace adr

using namespace adr;

extern "C" int32_t adr_kv_append(const void* k_new, const void* v_new, void* k_cache,
                                 void* v_cache, const int64_t* slot_mapping, int32_t B,
                                 int32_t Hkv, int32_t D, int32_t block_size, int64_t num_blocks,
                                 void* stream) {
  clear_error();
  if (B == 0) return ADR_OK;
  if (B < 0 || Hkv <= 0 || D <= 0 || block_size <= 0 || num_blocks <= 0)
    return fail(ADR_ERR_INVALID, "bad shape B=%d Hkv=%d D=%d block_size=%d", B, Hkv, D, block_size);
  if (D % 8 != 0) return fail(ADR_ERR_UNSUPPORTED, "head_dim %d not a multiple of 8", D);
  if (!k_new || !v_new || !k_cache || !v_cache || !slot_mapping)
    return fail(ADR_ERR_INVALID, "null tensor pointer");
  if (!aligned16(k_new) || !aligned16(v_new) || !aligned16(k_cache) || !aligned16(v_cache))
    return fail(ADR_ERR_INVALID, "tensors must be 16-byte aligned");
  const int pairs = B * Hkv;
  kv_append_kernel<<<(pairs + 3) / 4, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(k_new), static_cast<const __nv_bfloat16*>(v_new),
      static_cast<__nv_bfloat16*>(k_cache), static_cast<__nv_bfloat16*>(v_cache), slot_mapping, B,
      Hkv, D, block_size, num_blocks);
  return cuda_ok(cudaGetLastError(), "kv_append_kernel launch") ? ADR_OK : ADR_ERR_CUDA;
}

extern "C" int32_t adr_pack_qkv(const void* q, const void* k, const void* v,
                                const int32_t* row_idx, int32_t n_rows, int32_t Hq, int32_t Hkv,
                                int32_t D, void* dst, void* stream) {
  clear_error();
  if (n_rows == 0) return ADR_OK;
  if (n_rows < 0 || Hq <= 0 || Hkv <= 0 || D <= 0 || D % 8 != 0)
    return fail(ADR_ERR_INVALID, "bad shape n_rows=%d Hq=%d Hkv=%d D=%d", n_rows, Hq, Hkv, D);
  if (!q || !k || !v || !row_idx || !dst) return fail(ADR_ERR_INVALID, "null pointer");
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(dst))
    return fail(ADR_ERR_INVALID, "tensors must be 16-byte aligned");
  pack_qkv_kernel<<<n_rows, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(k),
      static_cast<const __nv_bfloat16*>(v), row_idx, Hq, Hkv, D, static_cast<__nv_bfloat16*>(dst));
  return cuda_ok(cudaGetLastError(), "pack_qkv_kernel launch") ? ADR_OK : ADR_ERR_CUDA;
}

extern "C" int32_t adr_unpack_qkv(const void* msg, int32_t n_rows, int32_t Hq, int32_t Hkv,
                                  int32_t D, void* q, void* k, void* v, void* stream) {
  clear_error();
  if (n_rows == 0) return ADR_OK;
  if (n_rows < 0 || Hq <= 0 || Hkv <= 0 || D <= 0 || D % 8 != 0)
    return fail(ADR_ERR_INVALID, "bad shape n_rows=%d Hq=%d Hkv=%d D=%d", n_rows, Hq, Hkv, D);
  if (!msg || !q || !k || !v) return fail(ADR_ERR_INVALID, "null pointer");
  if (!aligned16(msg) || !aligned16(q) || !aligned16(k) || !aligned16(v))
    return fail(ADR_ERR_INVALID, "tensors must be 16-byte aligned");
  unpack_qkv_kernel<<<n_rows, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(msg), Hq, Hkv, D, static_cast<__nv_bfloat16*>(q),
      static_cast<__nv_bfloat16*>(k), static_cast<__nv_bfloat16*>(v));
  return cuda_ok(cudaGetLastError(), "unpack_qkv_kernel launch") ? ADR_OK : ADR_ERR_CUDA;
}

extern "C" int32_t adr_scatter_out(const void* src, const int32_t* row_idx, int32_t n_rows,
                                   int32_t Hq, int32_t D, void* out, void* stream) {
  clear_error();
  if (n_rows == 0) return ADR_OK;
  if (n_rows < 0 || Hq <= 0 || D <= 0 || D % 8 != 0)
    return fail(ADR_ERR_INVALID, "bad shape n_rows=%d Hq=%d D=%d", n_rows, Hq, D);
  if (!src || !row_idx || !out) return fail(ADR_ERR_INVALID, "null pointer");
  if (!aligned16(src) || !aligned16(out)) return fail(ADR_ERR_INVALID, "tensors must be 16-byte aligned");
  scatter_out_kernel<<<n_rows, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(src), row_idx, Hq * D / 8, static_cast<__nv_bfloat16*>(out));
  return cuda_ok(cudaGetLastError(), "scatter_out_kernel launch") ? ADR_OK : ADR_ERR_CUDA;
}

extern "C" int32_t adr_kv_transfer(const void* src_k, const void* src_v, const int32_t* src_pages,
                                   void* dst_k, void* dst_v, const int32_t* dst_pages,
                                   int32_t n_pages, int32_t Hkv, int32_t D, int32_t block_size,
                                   void* stream) {
  clear_error();
  if (n_pages == 0) return ADR_OK;
  if (n_pages < 0 || Hkv <= 0 || D <= 0 || block_size <= 0 || D % 8 != 0)
    return fail(ADR_ERR_INVALID, "bad shape n_pages=%d Hkv=%d D=%d", n_pages, Hkv, D);
  if (!src_k || !src_v || !src_pages || !dst_k || !dst_v || !dst_pages)
    return fail(ADR_ERR_INVALID, "null pointer");
  if (!aligned16(src_k) || !aligned16(src_v) || !aligned16(dst_k) || !aligned16(dst_v))
    return fail(ADR_ERR_INVALID, "caches must be 16-byte aligned");
  const int page_chunks = Hkv * block_size * D / 8;
  kv_transfer_kernel<<<n_pages, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint4*>(src_k), static_cast<const uint4*>(src_v), src_pages,
      static_cast<uint4*>(dst_k), static_cast<uint4*>(dst_v), dst_pages, page_chunks);
  return cuda_ok(cudaGetLastError(), "kv_transfer_kernel launch") ? ADR_OK : ADR_ERR_CUDA;
}
