/*
 * attn_oracle.c — CPU restatement of the decode-attention path.
 *
 * TEST INFRASTRUCTURE ONLY. This file is the checker for libadrenaline.so:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load it. The product path never calls it (no CPU fallback).
 *
 * Parity status: UNPINNED against the reference for attention outputs. The
 * reference (/root/reference/pkg/src/adrenaline_sim) contains no attention
 * arithmetic — decode attention exists there only as a cost,
 *   attention_step_latency = resident_kv_bytes / (bandwidth * bw_fraction)
 * (costs.py:73-80, called engine.py:424-425 and 439-440) — and KV memory only as
 * token counters (engine.py:331-349, 416-421). This restates the standard
 * per-layer decode attention the paper runs on vLLM:
 *   out[b,h] = softmax(scale * q[b,h] . K_b^T) . V_b
 * over the request's paged context with GQA (q-head h reads kv-head h / (Hq/Hkv)),
 * on the fp32 upcast of the same bf16 inputs the GPU sees, accumulating in
 * double. The KV append is the paged scatter slot = page * block_size + offset.
 *
 * Pinned (in place of the reference) to the paper prototype's kernel family:
 * vLLM paged_attention_v2 + reshape_and_cache (the vLLM v0.6.3 algorithm the
 * paper ran; vLLM 0.22 in this image) and FlashInfer TRT-LLM-gen
 * outputs committed in tests/golden/attn_libraries.npz (generator:
 * tests/golden/make_attn_golden.py; check: tests/test_oracle_cpu.py).
 *
 * Layouts match include/adrenaline.h: q [B,Hq,D]; caches [NB,Hkv,bs,D];
 * block_table [B,max_blocks]; seq_lens [B]; out [B,Hq,D] fp32; lse [B,Hq].
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <pthread.h>
#include <string.h>
#include <unistd.h>

static inline float bf16_to_f32(uint16_t x) {
  uint32_t u = (uint32_t)x << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

int oracle_max_threads(void) {
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}

typedef struct {
  const uint16_t *q, *k_cache, *v_cache;
  const int32_t *block_table, *seq_lens;
  float *out, *lse;
  int B, Hq, Hkv, D, block_size, max_blocks;
  float scale;
  long long begin, end; /* (b, h) rows [begin, end) */
} AttnJob;

static void attn_rows(const AttnJob* j) {
  const int G = j->Hq / j->Hkv;
  const int D = j->D;
  double* acc = (double*)malloc(sizeof(double) * (size_t)D);
  float* qf = (float*)malloc(sizeof(float) * (size_t)D);
  double* sc = NULL;
  int sc_cap = 0;
  for (long long bh = j->begin; bh < j->end; ++bh) {
    const int b = (int)(bh / j->Hq);
    const int h = (int)(bh % j->Hq);
    const int kvh = h / G;
    const int n = j->seq_lens[b] > 0 ? j->seq_lens[b] : 0;
    float* o = j->out + (size_t)bh * D;
    for (int d = 0; d < D; ++d) qf[d] = bf16_to_f32(j->q[(size_t)bh * D + d]);
    if (n == 0) {
      for (int d = 0; d < D; ++d) o[d] = 0.f;
      if (j->lse) j->lse[bh] = -INFINITY;
      continue;
    }
    if (n > sc_cap) {
      free(sc);
      sc = (double*)malloc(sizeof(double) * (size_t)n);
      sc_cap = n;
    }
    double mx = -INFINITY;
    for (int t = 0; t < n; ++t) {
      const int page = j->block_table[(size_t)b * j->max_blocks + t / j->block_size];
      const uint16_t* kr =
          j->k_cache + (((size_t)page * j->Hkv + kvh) * j->block_size + t % j->block_size) * D;
      double s = 0.0;
      for (int d = 0; d < D; ++d) s += (double)qf[d] * (double)bf16_to_f32(kr[d]);
      s *= (double)j->scale;
      sc[t] = s;
      if (s > mx) mx = s;
    }
    double sum = 0.0;
    for (int d = 0; d < D; ++d) acc[d] = 0.0;
    for (int t = 0; t < n; ++t) {
      const double p = exp(sc[t] - mx);
      sum += p;
      const int page = j->block_table[(size_t)b * j->max_blocks + t / j->block_size];
      const uint16_t* vr =
          j->v_cache + (((size_t)page * j->Hkv + kvh) * j->block_size + t % j->block_size) * D;
      for (int d = 0; d < D; ++d) acc[d] += p * (double)bf16_to_f32(vr[d]);
    }
    for (int d = 0; d < D; ++d) o[d] = (float)(acc[d] / sum);
    if (j->lse) j->lse[bh] = (float)(mx + log(sum));
  }
  free(acc);
  free(qf);
  free(sc);
}

static void* attn_thread(void* arg) {
  attn_rows((const AttnJob*)arg);
  return NULL;
}

/* Returns 0 on success, -1 on invalid arguments. num_threads <= 0: all cores. */
int oracle_paged_decode_attn(const uint16_t* q, const uint16_t* k_cache, const uint16_t* v_cache,
                             const int32_t* block_table, const int32_t* seq_lens, float* out,
                             float* lse, int B, int Hq, int Hkv, int D, int block_size,
                             int max_blocks, float scale, int num_threads) {
  if (B < 0 || Hq <= 0 || Hkv <= 0 || Hq % Hkv != 0 || D <= 0 || block_size <= 0) return -1;
  const long long total = (long long)B * Hq;
  int nt = num_threads > 0 ? num_threads : oracle_max_threads();
  if (nt > total) nt = total > 0 ? (int)total : 1;
  AttnJob* jobs = (AttnJob*)calloc((size_t)nt, sizeof(AttnJob));
  pthread_t* th = (pthread_t*)calloc((size_t)nt, sizeof(pthread_t));
  for (int i = 0; i < nt; ++i) {
    AttnJob j = {q, k_cache, v_cache, block_table, seq_lens, out, lse, B, Hq, Hkv, D, block_size,
                 max_blocks, scale, total * i / nt, total * (i + 1) / nt};
    jobs[i] = j;
  }
  for (int i = 1; i < nt; ++i) pthread_create(&th[i], NULL, attn_thread, &jobs[i]);
  if (nt > 0) attn_rows(&jobs[0]);
  for (int i = 1; i < nt; ++i) pthread_join(th[i], NULL);
  free(jobs);
  free(th);
  return 0;
}

/* slot < 0 rows are skipped; returns the number of rows written or -1. */
int oracle_kv_append(const uint16_t* k_new, const uint16_t* v_new, uint16_t* k_cache,
                     uint16_t* v_cache, const int64_t* slots, int B, int Hkv, int D,
                     int block_size, long long num_blocks) {
  if (B < 0 || Hkv <= 0 || D <= 0 || block_size <= 0) return -1;
  int written = 0;
  for (int b = 0; b < B; ++b) {
    const int64_t slot = slots[b];
    if (slot < 0) continue;
    const int64_t page = slot / block_size;
    if (page >= num_blocks) continue;
    const int off = (int)(slot % block_size);
    for (int h = 0; h < Hkv; ++h) {
      const size_t dst = (((size_t)page * Hkv + h) * block_size + off) * D;
      const size_t src = ((size_t)b * Hkv + h) * D;
      memcpy(k_cache + dst, k_new + src, sizeof(uint16_t) * (size_t)D);
      memcpy(v_cache + dst, v_new + src, sizeof(uint16_t) * (size_t)D);
    }
    ++written;
  }
  return written;
}
