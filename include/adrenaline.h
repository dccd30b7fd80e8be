/*
 * adrenaline.h — C-ABI of libadrenaline.so, the B200 (sm_100a) implementation of
 * Adrenaline's offloaded decode-attention path (arXiv 2503.20552).
 *
 * The reference (/root/reference/pkg/src/adrenaline_sim) is a pure-Python
 * simulator with no FFI: its "operators" are the Python cost functions that
 * price the path. Each entry point below is the real computation that sits
 * under one of those functions; the reference symbol it replaces is cited on
 * every declaration (file:line under pkg/src/adrenaline_sim/).
 *
 * Conventions (all entry points):
 *   - return int32 status: ADR_OK (0) or a negative ADR_ERR_* code; the message
 *     is available from adr_last_error() (thread-local);
 *   - take an explicit CUDA stream (cudaStream_t passed as void*), never
 *     synchronise the host and never allocate: the caller owns every buffer,
 *     including the workspace, so every call is CUDA-graph capturable;
 *   - dtypes: bf16 (__nv_bfloat16, passed as void*) for q/k/v/out, fp32 for
 *     lse and scale, int32 for block tables, sequence lengths and row indices,
 *     int64 for slot mappings;
 *   - layouts are dense and contiguous:
 *       q        [B, Hq, D]
 *       k_cache  [num_blocks, Hkv, block_size, D]   (one 4 KiB page per
 *       v_cache  [num_blocks, Hkv, block_size, D]    (block, kv-head) at D=128)
 *       block_table [B, max_blocks_per_seq], seq_lens [B]
 *       out      [B, Hq, D] (bf16, or fp32 when out_dtype == ADR_DTYPE_F32)
 *       lse      [B, Hq] natural-log log-sum-exp of the scaled scores
 *   - q-head h reads kv-head h / (Hq / Hkv)  (GQA grouping).
 * There is no CPU fallback: on a host without a usable sm_100 device every
 * compute entry point returns ADR_ERR_CUDA.
 */
#ifndef ADRENALINE_H_
#define ADRENALINE_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define ADR_API __attribute__((visibility("default")))
#else
#define ADR_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define ADR_OK 0
#define ADR_ERR_INVALID (-1)     /* bad argument (shape, null pointer, alignment) */
#define ADR_ERR_UNSUPPORTED (-2) /* valid but not implemented (e.g. D=96, GQA group > 8) */
#define ADR_ERR_CUDA (-3)        /* CUDA runtime / driver failure */
#define ADR_ERR_WORKSPACE (-4)   /* workspace missing or too small */

#define ADR_DTYPE_BF16 0
#define ADR_DTYPE_F32 1

/* adr_paged_decode_attn flags */
#define ADR_DECODE_PDL 1u /* programmatic dependent launch: overlap this call's
                             prologue and first KV loads with the preceding
                             kernel's tail (see the function's contract) */
/* Work split of adr_paged_decode_attn (testing / tuning; default: automatic).
 * Dynamic grid: warps claim chunks from a counter, split pairs are merged by a
 * merge phase. Static grid (chosen for small calls): one chunk per warp, the
 * warp publishing a pair's last piece merges it, the first KV loads may be
 * issued before the dependency wait. Results are deterministic in either. */
#define ADR_DECODE_GRID_DYNAMIC 2u
#define ADR_DECODE_GRID_STATIC 4u
/* Split-pair CTA kernel (chosen automatically for small calls): each pair is
 * cut into items of P pages, a CTA's warps interleave an item's pages and
 * combine through shared memory, the CTA publishing a pair's last item merges. */
#define ADR_DECODE_GRID_SPLIT 8u

/* Library version, (major << 16) | minor. */
ADR_API int32_t adr_version(void);

/* Last error message of the calling thread ("" when none). */
ADR_API const char* adr_last_error(void);

/* Device facts the host planner needs (SM count, compute capability). */
ADR_API int32_t adr_device_info(int32_t device, int32_t* num_sms, int32_t* cc_major, int32_t* cc_minor);

/* Bytes of caller-provided workspace adr_paged_decode_attn needs for this
 * shape (B = the largest batch the workspace will serve; the partial slots are
 * sized for the GQA group Hq / Hkv and head_dim D, so one workspace serves any
 * call with the same or a smaller group and head_dim). num_workers <= 0
 * selects the default persistent grid (every resident warp).
 * The workspace must be zero-filled before its first use; every successful
 * call leaves it ready for the next one (its claim and per-pair counters are
 * reset by the warps that finish last). Calls sharing a workspace must be
 * ordered (same stream, or event-ordered). Returns 0 on invalid input. */
ADR_API size_t adr_decode_workspace_bytes(int32_t B, int32_t Hq, int32_t Hkv, int32_t D,
                                  int32_t num_workers);

/* As adr_decode_workspace_bytes, sized for calls whose block tables have at
 * most max_blocks_per_seq columns (0 = no bound): the partial slots then scale
 * with B x max_blocks_per_seq x Hkv instead of the whole device's grid (a
 * B=8 ctx-1024 executor needs ~6 MB instead of ~240 MB at GQA-8). A call
 * whose B x max_blocks_per_seq x Hkv exceeds what the workspace was sized for
 * returns ADR_ERR_WORKSPACE. */
ADR_API size_t adr_decode_workspace_size(int32_t B, int32_t Hq, int32_t Hkv, int32_t D,
                                 int32_t max_blocks_per_seq, int32_t num_workers);

/* Status bits of rejected decode input (sticky in the workspace). The kernel
 * never reads or writes outside the caches on bad tables: a request whose
 * seq_len is negative or exceeds 16 x max_blocks_per_seq owns no work (zero
 * output, lse -inf, nothing appended); a block-table entry outside
 * [0, num_blocks) is read as page 0 and its append is skipped. */
#define ADR_STATUS_BAD_SEQ_LEN 1
#define ADR_STATUS_BAD_PAGE 2

/* Synchronous diagnostics (they synchronise `stream`; not for the hot path):
 * adr_decode_status reads (and with clear != 0 resets) the ADR_STATUS_* bits
 * the decode calls on this workspace recorded. adr_check_decode_tables
 * validates block_table / seq_lens before a call: ADR_OK, or ADR_ERR_INVALID
 * naming the first offending request. */
ADR_API int32_t adr_decode_status(void* workspace, size_t workspace_bytes, int32_t clear,
                          int32_t* status, void* stream);
ADR_API int32_t adr_check_decode_tables(const int32_t* block_table, const int32_t* seq_lens,
                                int32_t B, int32_t max_blocks_per_seq, int64_t num_blocks,
                                void* workspace, size_t workspace_bytes, void* stream);

/* Warps per SM the decode-attention kernel keeps resident for a launch
 * confined to num_sms SMs (0 = the whole device). */
ADR_API int32_t adr_decode_warps_per_sm(int32_t num_sms);

/*
 * Paged decode attention: for every request b and q-head h,
 *   out[b,h,:] = softmax(scale * q[b,h,:] . K[b, 0:seq_lens[b], kvh, :]^T) . V[b, 0:seq_lens[b], kvh, :]
 * where token t of request b lives in page block_table[b, t / block_size] at
 * row t % block_size. fp32 accumulation; one persistent pass: the (request,
 * kv-head, page) space is cut into a fixed grid of equal chunks that warps
 * claim dynamically; a pair cut by the grid is merged by log-sum-exp over its
 * pieces in chunk order, inside the same launch (bit-identical run to run).
 *
 * Fused append (k_new, v_new non-null, [B, Hkv, D] bf16): the step's new token
 * of request b is position seq_lens[b] - 1; its K/V rows are written into the
 * cache (k_cache/v_cache, bit-exact) and used by this same attention — the
 * separate adr_kv_append call is then unnecessary.
 *
 * Replaces costs.attention_step_latency (costs.py:73-80), called for local
 * attention at engine.py:424-425 and per executor at engine.py:439-440.
 * block_size must be 16; D in {64, 128}; Hq % Hkv == 0 and Hq / Hkv <= 8;
 * num_blocks is the page count of the cache (bounds the TMA descriptors).
 * num_sms: SMs the launch may occupy — 0 for the whole device, or the size of
 * the SM partition (green context) whose stream is passed, so the persistent
 * grid fits it. num_workers: 0, or an explicit warp count (testing knob).
 * flags: ADR_DECODE_PDL — the caller guarantees that block_table, seq_lens and
 * the cache (other than the appended rows) are not written by the kernel
 * immediately preceding this call on the stream (q, k_new, v_new may be).
 */
ADR_API int32_t adr_paged_decode_attn(const void* q, const void* k_new, const void* v_new,
                              void* k_cache, void* v_cache, const int32_t* block_table,
                              const int32_t* seq_lens, void* out, float* lse, int32_t B,
                              int32_t Hq, int32_t Hkv, int32_t D, int32_t block_size,
                              int32_t max_blocks_per_seq, int64_t num_blocks, float scale,
                              int32_t num_sms, int32_t num_workers, int32_t out_dtype,
                              uint32_t flags, void* workspace, size_t workspace_bytes,
                              void* stream);

/*
 * adr_paged_decode_attn with request row maps (zero-copy offload over NVLink):
 * request b reads its q / k_new / v_new rows at in_rows[b] (of [*, Hq, D] /
 * [*, Hkv, D] tensors) and writes its out / lse rows at out_rows[b]; either
 * map may be null (identity). q, k_new, v_new, out and lse may be peer-GPU
 * pointers (peer access enabled, or CUDA-IPC mapped): the executor's attention
 * then reads the offloaded requests' q/k/v from the decode GPU and writes
 * their outputs into the decode GPU's output rows directly — no pack, copy,
 * unpack or scatter kernels (replaces the send/recv legs of the remote path,
 * engine.py:427-445, in the kernel's own loads and stores). Cache, tables and
 * workspace are the executor's own. Ordering against the decode GPU's
 * producer/consumer kernels is the caller's (events or adr_signal/adr_wait).
 */
ADR_API int32_t adr_paged_decode_attn_rows(const void* q, const void* k_new, const void* v_new,
                                   const int32_t* in_rows, void* k_cache, void* v_cache,
                                   const int32_t* block_table, const int32_t* seq_lens, void* out,
                                   float* lse, const int32_t* out_rows, int32_t B, int32_t Hq,
                                   int32_t Hkv, int32_t D, int32_t block_size,
                                   int32_t max_blocks_per_seq, int64_t num_blocks, float scale,
                                   int32_t num_sms, int32_t num_workers, int32_t out_dtype,
                                   uint32_t flags, void* workspace, size_t workspace_bytes,
                                   void* stream);

/*
 * CUDA IPC for the zero-copy offload between processes (one process per GPU).
 * adr_ipc_export: handle (ADR_IPC_HANDLE_BYTES) of the device allocation that
 * contains ptr, and ptr's byte offset in it. adr_ipc_import (other process):
 * maps it (peer access enabled lazily) and returns ptr = mapped base + offset
 * and the base to pass to adr_ipc_close. The decode process exports its
 * per-layer q/k/v/out rows and uint32 flags once; the executor passes the
 * mapped pointers to adr_paged_decode_attn_rows, adr_wait and adr_signal.
 */
#define ADR_IPC_HANDLE_BYTES 64
ADR_API int32_t adr_ipc_export(const void* ptr, void* handle, uint64_t* offset);
ADR_API int32_t adr_ipc_import(const void* handle, uint64_t offset, void** ptr, void** base);
ADR_API int32_t adr_ipc_close(void* base);

/*
 * Fused KV append: for each request b with slot_mapping[b] >= 0,
 *   k_cache[slot / block_size, :, slot % block_size, :] = k_new[b]
 *   v_cache[slot / block_size, :, slot % block_size, :] = v_new[b]
 * (k_new, v_new: [B, Hkv, D] bf16; slot = page * block_size + offset).
 * Bit-exact copy. Replaces the per-step KV growth of engine.py:416-421
 * (reservation +1 token per running request).
 */
ADR_API int32_t adr_kv_append(const void* k_new, const void* v_new, void* k_cache, void* v_cache,
                      const int64_t* slot_mapping, int32_t B, int32_t Hkv, int32_t D,
                      int32_t block_size, int64_t num_blocks, void* stream);

/*
 * Pack the offloaded rows' q, k, v into one contiguous message (one send per
 * layer): dst[i] = [ q[row_idx[i]] (Hq*D) | k[row_idx[i]] (Hkv*D) | v[row_idx[i]] (Hkv*D) ]
 * bf16, i < n_rows. Replaces the q/k/v send pricing of engine.py:436-437.
 */
ADR_API int32_t adr_pack_qkv(const void* q, const void* k, const void* v, const int32_t* row_idx,
                     int32_t n_rows, int32_t Hq, int32_t Hkv, int32_t D, void* dst, void* stream);

/*
 * Split a received message (layout of adr_pack_qkv, n_rows rows) into dense
 * q [n_rows, Hq, D], k [n_rows, Hkv, D], v [n_rows, Hkv, D] on the executor.
 */
ADR_API int32_t adr_unpack_qkv(const void* msg, int32_t n_rows, int32_t Hq, int32_t Hkv, int32_t D,
                       void* q, void* k, void* v, void* stream);

/*
 * Scatter returned executor outputs into the decode batch order beside the
 * local outputs: out[row_idx[i]] = src[i] (src [n_rows, Hq, D] bf16).
 * The "merge outputs from two attention kernels" step; replaces
 * the output-return pricing of engine.py:438.
 */
ADR_API int32_t adr_scatter_out(const void* src, const int32_t* row_idx, int32_t n_rows, int32_t Hq,
                        int32_t D, void* out, void* stream);

/*
 * Prefill -> decode KV migration with block-table remap: for i < n_pages,
 *   dst_k[dst_pages[i]] = src_k[src_pages[i]], dst_v[dst_pages[i]] = src_v[src_pages[i]]
 * (whole pages [Hkv, block_size, D] bf16). src_* may be peer-mapped pointers of
 * the prefill GPU (enable peer access first): the kernel then pulls the pages
 * over NVLink. Replaces the KV-transfer pricing of engine.py:231-238
 * (prefill_len * kv_tok / interconnect_bandwidth per local request). Offloaded
 * requests skip it: their KV stays on the executor (engine.py:239-241).
 */
ADR_API int32_t adr_kv_transfer(const void* src_k, const void* src_v, const int32_t* src_pages,
                                void* dst_k, void* dst_v, const int32_t* dst_pages,
                                int32_t n_pages, int32_t Hkv, int32_t D, int32_t block_size,
                                void* stream);

/* Enable peer access between two devices (both directions). Idempotent. */
ADR_API int32_t adr_peer_open(int32_t dev_a, int32_t dev_b);

/*
 * SM partition of one GPU for colocation (replaces the reference's
 * attn_sm_ratio split, config.py:125-132): two green contexts, attn_sms SMs
 * (rounded to the architecture's granularity, 8 on sm_100) for the executor's
 * attention and the rest for prefill, each with one non-blocking stream of
 * the given priority (lower = higher priority; cudaDeviceGetStreamPriorityRange).
 * The executor's stream should have the higher priority: the block scheduler
 * otherwise dispatches a grid's CTAs only after the CTAs of every grid launched
 * before it, so an attention call queued behind a prefill GEMM waits for that
 * GEMM's CTAs (measured: +100-350 us per call, profiles/exec_prio_r02u.txt).
 * *handle is released with adr_sm_partition_destroy (after the streams' work).
 */
ADR_API int32_t adr_sm_partition_create(int32_t device, int32_t attn_sms, int32_t attn_priority,
                                        int32_t prefill_priority, void** attn_stream,
                                        void** prefill_stream, int32_t* attn_sms_out,
                                        int32_t* prefill_sms_out, void** handle);
ADR_API int32_t adr_sm_partition_destroy(void* handle);

/* Asynchronous device-to-device copy across GPUs (NVLink when peer access is
 * enabled). Replaces the scalar interconnect pricing of engine.py:431-444. */
ADR_API int32_t adr_copy_peer(void* dst, int32_t dst_dev, const void* src, int32_t src_dev, size_t bytes,
                      void* stream);

/* Stream-ordered flag signalling on (possibly peer-mapped) device memory:
 * adr_signal writes `value` to *flag once prior work on `stream` is done;
 * adr_wait blocks `stream` (not the host) until *flag >= value. */
ADR_API int32_t adr_signal(uint32_t* flag, uint32_t value, void* stream);
ADR_API int32_t adr_wait(const uint32_t* flag, uint32_t value, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* ADRENALINE_H_ */
