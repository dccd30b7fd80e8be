// Host-side helpers shared by the libadrenaline.so translation units.
#pragma once

#include <cstdarg>
#include <cstddef>
#include <cstdint>

#include "adr_device.cuh"
#include "../../include/adrenaline.h"

namespace adr {

// Largest decode batch one adr_paged_decode_attn call accepts (the per-CTA
// unit prefix lives in shared memory).
constexpr int kMaxBatch = 2048;

void clear_error();
// Record a printf-style message as the thread's last error and return `code`.
int fail(int code, const char* fmt, ...);
// True on cudaSuccess, otherwise records "<what>: <cuda error>" and returns false.
bool cuda_ok(cudaError_t err, const char* what);

// 2-D TMA descriptor over a paged cache viewed as [rows, D] bf16 with a
// 64-column x 16-row box and 128-byte swizzle (one half page per load).
int encode_page_tmap(CUtensorMap* map, const void* base, int D, uint64_t rows);

}  // namespace adr
