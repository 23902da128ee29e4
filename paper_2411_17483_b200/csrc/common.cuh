// Shared device helpers and the internal index layout of libsofa (sm_100a).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <array>
#include <atomic>
#include <string>
#include <vector>

#include "../../include/sofa.h"

#define SOFA_TRACE_FIELDS 24

namespace sofa {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kThreads = 256;     // every kernel of the hot path runs 8 warps per CTA
constexpr int kQueryBatch = 1024;  // sofa_knn runs larger batches as consecutive sub-batches

extern std::atomic<int64_t> g_launches;
void set_error(const std::string& msg);

#define SOFA_CK(call)                                                                  \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess) {                                                           \
      ::sofa::set_error(std::string(#call) + ": " + cudaGetErrorString(e_));           \
      return e_ == cudaErrorMemoryAllocation ? SOFA_ENOMEM : SOFA_ECUDA;               \
    }                                                                                  \
  } while (0)

#define SOFA_LAUNCHED()                                                                \
  do {                                                                                 \
    ::sofa::g_launches.fetch_add(1);                                                   \
    cudaError_t e_ = cudaGetLastError();                                               \
    if (e_ != cudaSuccess) {                                                           \
      ::sofa::set_error(std::string("kernel launch: ") + cudaGetErrorString(e_));      \
      return SOFA_ECUDA;                                                               \
    }                                                                                  \
  } while (0)

// Device-side copy of the model: LT = l rounded up to 16/32/64 (padded rows are inert:
// zero basis, +inf edges, zero tables).
struct DevModel {
  int len, l, LT, a, a_bits, WS;  // WS = word stride in bytes (l rounded up to 16)
  const float* basis32;            // LT x len   float32 cos/-sin(2 pi k t/n)/sqrt(n)
  const double* basis64;           // LT x len   float64 (query projection)
  const float* edges32;            // LT x 256   float32, row padded with +inf
  const double* edges64;           // LT x 256   float64, row padded with +inf
  float weights[SOFA_MAX_L];
};

// ---------------------------------------------------------------------------------------------
// streaming loads (read-once data: do not allocate in L1)
__device__ __forceinline__ float4 ld_stream(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ld_stream_u4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(FULL, v, m);
  return v;
}
__device__ __forceinline__ float warp_sum_f32(float v) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(FULL, v, m);
  return v;
}

// Lanes per row in the row layout of a1 (k_transform and the query prep): each lane of a group of G
// lanes holds 8 float4 of the row (float4 index g + G f), G = ceil(n/32) rounded up to a power of two.
__host__ __device__ constexpr int row_group(int nf4) {
  int G = 1;
  while (G * 8 < nf4) G *= 2;
  return G;
}

// a1 (Def. 2, population std, reading 1): per-row statistics with a fixed arithmetic order,
// shared by the series transform and the query prep so that a query equal to a stored row
// z-normalises to the same float32 bits (exact duplicates -> d = 0).  Each lane of the row's group
// sums its float4s in float32, the G partials are combined in float64 by an xor butterfly (every
// lane of the group ends with the same value).  Returns mu (float32 and float64) and inv_sigma
// (float64; 0 for a constant row).
// ALLSLOTS (compile time; it was once named FULL and shadowed the shuffle mask): the caller knows nf4 == 8 G (every lane's 8 float4 are in the row): the same
// arithmetic without the per-slot guards.
template <int G, bool ALLSLOTS = false>
__device__ __forceinline__ void row_stats_g(const float4 (&x)[8], int nf4, int g, int len, float& muf, double& mu64,
                                            double& inv64) {
  float p = 0.f;
#pragma unroll
  for (int f = 0; f < 8; ++f)
    if (ALLSLOTS || g + G * f < nf4) p = __fadd_rn(p, __fadd_rn(__fadd_rn(x[f].x, x[f].y), __fadd_rn(x[f].z, x[f].w)));
  double sp = (double)p;
#pragma unroll
  for (int m = G / 2; m >= 1; m >>= 1) sp += __shfl_xor_sync(FULL, sp, m);
  mu64 = sp / (double)len;
  muf = (float)mu64;
  float s = 0.f;
#pragma unroll
  for (int f = 0; f < 8; ++f)
    if (ALLSLOTS || g + G * f < nf4) {
      const float a = __fsub_rn(x[f].x, muf), b = __fsub_rn(x[f].y, muf);
      const float c = __fsub_rn(x[f].z, muf), d = __fsub_rn(x[f].w, muf);
      s = __fadd_rn(s, __fadd_rn(__fmaf_rn(a, a, __fmul_rn(b, b)), __fmaf_rn(c, c, __fmul_rn(d, d))));
    }
  double ss = (double)s;
#pragma unroll
  for (int m = G / 2; m >= 1; m >>= 1) ss += __shfl_xor_sync(FULL, ss, m);
  const double var = ss / (double)len;
  const double sd = sqrt(var);
  inv64 = sd < 1e-12 ? 0.0 : 1.0 / sd;
}

// exact squared z-ED with early abandoning (a8) for R candidate rows at once: one warp, float4
// loads of all R rows issued together (R rows in flight per warp), chunks of 2 float4 per lane
// (256 values), partial sums warp-reduced after each chunk and compared with the BSF.
template <int NF, int R>
__device__ __forceinline__ void ed_warp_multi(const float* const (&rows)[R], const float2 (&st)[R],
                                              const bool (&on)[R], const float4* s_qh4, int nf4, float bsf,
                                              float (&d2)[R], bool (&ab)[R]) {
  const int lane = threadIdx.x & 31;
  constexpr int CH = (NF < 2 || R >= 8) ? 1 : 2;  // float4 per lane per chunk (8 rows in flight: 1)
#pragma unroll
  for (int r = 0; r < R; ++r) {
    d2[r] = 0.f;
    ab[r] = false;
  }
#pragma unroll
  for (int f0 = 0; f0 < NF; f0 += CH) {
    float4 x[R][CH];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        const int fi = lane + 32 * (f0 + c);
        x[r][c] = (on[r] && !ab[r] && fi < nf4) ? ld_stream(reinterpret_cast<const float4*>(rows[r]) + fi)
                                                : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      float acc = 0.f;
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        const int fi = lane + 32 * (f0 + c);
        if (fi < nf4) {
          const float4 q = s_qh4[fi];
          const float e0 = __fsub_rn(__fmul_rn(__fsub_rn(x[r][c].x, st[r].x), st[r].y), q.x);
          const float e1 = __fsub_rn(__fmul_rn(__fsub_rn(x[r][c].y, st[r].x), st[r].y), q.y);
          const float e2 = __fsub_rn(__fmul_rn(__fsub_rn(x[r][c].z, st[r].x), st[r].y), q.z);
          const float e3 = __fsub_rn(__fmul_rn(__fsub_rn(x[r][c].w, st[r].x), st[r].y), q.w);
          acc = __fmaf_rn(e0, e0, acc);
          acc = __fmaf_rn(e1, e1, acc);
          acc = __fmaf_rn(e2, e2, acc);
          acc = __fmaf_rn(e3, e3, acc);
        }
      }
      d2[r] += warp_sum_f32(acc);
      if (f0 + CH < NF && d2[r] > bsf) ab[r] = true;
    }
  }
}

// One query's result (a8 -> caller), written by ONE thread.  The top-k is kept sorted by (d^2, row);
// the caller's order is (d, global index) with d = sqrtf(d^2) (include/sofa.h), which differs only
// where distinct d^2 round to the same d: an insertion pass (k <= 128, almost always a no-op) puts
// those runs in index order, so every writer — and the cross-shard merge (a9), which only sees d —
// agrees on one order.  Missing entries pad with (+inf, -1).
__device__ __forceinline__ void write_topk(const volatile float* td, const volatile int* ti, int n, int k,
                                           int64_t goff, float* __restrict__ od, int64_t* __restrict__ oi) {
  for (int r = 0; r < k; ++r) {
    const float d = r < n ? sqrtf(td[r]) : INFINITY;
    const int64_t i = r < n ? goff + ti[r] : -1;
    int p = r;
    while (p > 0 && i >= 0 && od[p - 1] == d && oi[p - 1] > i) {
      od[p] = od[p - 1];
      oi[p] = oi[p - 1];
      --p;
    }
    od[p] = d;
    oi[p] = i;
  }
}

// upper_bound over a 256-entry edge row padded with +inf: number of edges <= v (symbol of v;
// bins [beta(s), beta(s+1)) — P:225-228, value on an edge goes right).
template <typename E>
__device__ __forceinline__ int bin_of(const E* __restrict__ e, double v) {
  int pos = 0;
#pragma unroll
  for (int step = 128; step >= 1; step >>= 1)
    if ((double)e[pos + step - 1] <= v) pos += step;
  return pos;
}

// 64-bit block-ordering key of a word (a4): symbols normalised to 8 bits, 2-bit groups taken
// MSB-first round-robin over the first min(l,16) positions (SURVEY SIM-4: 2-bit interleaving
// gives the fewest surviving blocks).  Only the order of blocks depends on it, never a result.
__device__ __forceinline__ uint64_t word_key(const uint8_t* w, int l, int a_bits) {
  const int P = l < 16 ? l : 16;
  // symbols 4i..4i+3 normalised to 8 bits in v[i], position 4i in the most significant byte
  uint32_t v[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint32_t x = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int p = 4 * i + b;
      const uint32_t s = p < P ? ((uint32_t)w[p] << (8 - a_bits)) & 0xffu : 0u;
      x |= s << (24 - 8 * b);
    }
    v[i] = x;
  }
  // round r: the r-th 2-bit digit (MSB first) of every symbol, packed position-major into 32 bits
  // with byte-parallel masks; the first 2P bits hold positions 0..P-1
  uint64_t key = 0;
  int nbits = 0;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    if (nbits >= 64) break;
    uint32_t packed = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t m = (v[i] >> (6 - 2 * r)) & 0x03030303u;
      packed = (packed << 8) | ((m >> 18) & 0xC0u) | ((m >> 12) & 0x30u) | ((m >> 6) & 0x0Cu) | (m & 0x03u);
    }
    const int bits = 2 * P;
    const int take = bits < 64 - nbits ? bits : 64 - nbits;
    const uint64_t grp = packed >> (32 - bits);
    key = (key << take) | (grp >> (bits - take));
    nbits += take;
  }
  return nbits < 64 ? key << (64 - nbits) : key;
}

}  // namespace sofa

// Dense-path (f1) scratch, per index, grown on demand (dense.cu).  counters (64 ints): [0] dense query
// slots, [1] overflowed slots, [2..3] candidate count (u64), [4] finished CTAs, [6..7] estimated
// sparse refines of the flagged queries (u64, the batch decision); then 1024 ints of per-CTA progress.
struct DenseScratch {
  int q_cap = 0, k_cap = 0, len = 0;
  int64_t cand_cap = 0;
  float* qhat = nullptr;           // slot x len: z-normalised query (float32, same bits as the sparse path)
  __nv_bfloat16* qb16 = nullptr;   // slot x xb_ld: the same, bfloat16 (the screen's B operand)
  float4* qparams = nullptr;       // slot: (|q^|^2, eps, -, -)
  int* qidx = nullptr;             // slot -> query index
  float* binit = nullptr;          // slot -> caller's bound
  float* bsf = nullptr;            // slot -> exact k-th best squared distance (or the bound)
  float* thr = nullptr;            // slot -> proven bound on the k-th best (screening threshold)
  float* tkd = nullptr;            // slot x k_cap
  int* tki = nullptr;              // slot x k_cap (local rows)
  int* tkn = nullptr;
  unsigned long long* key1 = nullptr;  // slot: k = 1 best as (d^2 bits << 32 | local row), lock-free min
  int* lock = nullptr;
  float* ubl = nullptr;            // slot x k_cap: k smallest upper bounds of candidate rows (k > 1)
  float* ubsnap = nullptr;         // slot x screen CTA x (k_cap + 2): each CTA's UB list, seqlock-published (k > 1)
  int* ubn = nullptr;
  int* ub_lock = nullptr;
  int* overflow = nullptr;
  int* ovf_list = nullptr;
  unsigned long long* cand = nullptr;
  int* counters = nullptr;
  alignas(64) unsigned char tmap_q[128];  // CUtensorMap of qb16, encoded for tmap_q_rows rows
  alignas(64) unsigned char tmap_x[128];  // CUtensorMap of the index's bf16 rows
  int tmap_q_rows = -1;
};

// Host-side index object (opaque in the C ABI).
struct sofa_index {
  int64_t n = 0, nb = 0, global_offset = 0, global_n = 0;
  int32_t len = 0, l = 0, a = 0, B = 256, LT = 16, WS = 16;
  sofa_model model{};
  const float* series = nullptr;  // borrowed
  uint8_t* words = nullptr;       // n x WS, sorted by key
  float2* stats = nullptr;        // n, sorted order: (mu, 1/sigma)
  float2* stats_orig = nullptr;   // n, original row order (dense path)
  __nv_bfloat16* xb16 = nullptr;  // n x xb_ld, original row order: z-normalised rows in bfloat16 (dense screen)
  int xb_ld = 0;                  // row stride of xb16 (len rounded up to 8: 16-byte TMA rows)
  int32_t dense_permille = 5;     // dense path when >= this many permille of probed words pass (0: off)
  double build_ms[4] = {};        // model, transform, sort, gather + envelopes (CUDA events)
  DenseScratch dense;
  int32_t* perm = nullptr;        // n: sorted position -> local row
  uint8_t* env = nullptr;         // nb x 2 x WS
  uint64_t* bkey = nullptr;       // nb first keys
  int nlev = 1;                   // envelope tree levels (level 0 = blocks, fan-out 16)
  int64_t lvl_off[8] = {}, lvl_cnt[8] = {};
  float* basis32 = nullptr;
  double* basis64 = nullptr;
  float* edges32 = nullptr;
  double* edges64 = nullptr;
  // query scratch
  unsigned long long* gscratch = nullptr;
  int64_t gscratch_ctas = 0;
  int* qcounter = nullptr;
  // front/scan split (query.cu): per-query state, tables, the leaf pool and the scan tasks
  void *qstate = nullptr, *q_T = nullptr, *q_hat = nullptr, *pool = nullptr, *tasks = nullptr,
       *rank_count = nullptr;
  void *fifo = nullptr, *fifo_seq = nullptr;  // fused scan: published set-0 tasks in publication order
  int* fcount = nullptr;  // fused-scan counters (512 B: one 128-byte line each)
  int epoch = 0;  // front launch number: FIFO entries and query states are valid when they carry it
  int64_t scan_q_cap = 0, pool_cap = 0, task_cap = 0, rank_cap = 0;
  int scan_LT = 0;
  unsigned long long* dstats = nullptr;
  long long* trace = nullptr;  // per-query trace (filled when stats are requested)
  int64_t trace_cap = 0;
  int trace_on = 0;
  // live per-launch-group timing (sofa_kernel_timing): 4 events per sub-batch, read back lazily
  int ktime_on = 0;
  std::vector<std::array<cudaEvent_t, 5>> ktime_pending, ktime_free;
  double ktime_ms[4] = {0, 0, 0, 0};
  int64_t ktime_groups = 0;
  int64_t trace_off = 0;  // first query row of the current sub-batch in the trace
  int32_t trace_q = 0;
  // host-path staging
  float* hq_dev = nullptr;
  float* hd_dev = nullptr;
  int64_t* hi_dev = nullptr;
  int64_t h_cap = 0;
  int device = 0;
  int sms = 148;        // multiprocessors of `device` (queried once at build time)
  int dense_clusters = 0;  // resident clusters of 2 of the dense screen (queried at its first cluster launch)
  sofa_tuning tune{};   // query-kernel tuning (sofa_set_tuning; defaults from sofa_default_tuning)
  sofa::DevModel dm{};
};

namespace sofa {
int upload_model(const sofa_model& m, int len, sofa_index* ix, cudaStream_t st);
int launch_transform(const float* X, int64_t N, const DevModel& dm, const sofa_model& m, uint8_t* words,
                     float2* stats, uint64_t* keys, double* vals, uint8_t* words_l, __nv_bfloat16* xb16,
                     cudaStream_t st, cudaEvent_t t_start = nullptr);
int launch_envelopes(const uint8_t* words, int64_t n, int B, int WS, const uint64_t* skeys, uint8_t* env,
                     uint64_t* bkey, cudaStream_t st);
int launch_env_up(const uint8_t* child, int64_t nchild, int WS, uint8_t* parent, cudaStream_t st);
int launch_gather(const uint8_t* words, const float2* stats, const int32_t* perm, int64_t n, int WS,
                  uint8_t* words_out, float2* stats_out, cudaStream_t st);
int learn_model_dev(const float* sample, int64_t S, int len, int l, int a, int binning, int cand_limit,
                    cudaStream_t st, sofa_model* out);
int isax_model(int len, int l, int a, sofa_model* out);
int launch_query(sofa_index* ix, const float* Q, int q, int k, const float* bsf_init, float* od, int64_t* oi,
                 cudaStream_t st, bool scan = false, int64_t lb_m = 0, float* lb_out = nullptr,
                 float* ed_out = nullptr, int64_t* lb_rows = nullptr, float* seed_out = nullptr);
// batch-level dense decision (f1): the tensor-core pass runs iff the flagged queries' estimated sparse
// refines add up to at least this many rows.  Default n / 5: one dense pass streams 2 len bytes per row
// at ~6 TB/s, a sparse refine reads 4 len bytes of a random row at ~2.6 TB/s (configs[3], measured), so
// the pass pays for itself from ~0.22 n refines on (tools/latency_probe.py cfg4: batches of 8 with two
// or three unprunable queries 23.5 ms at n, 8.9 ms at n / 4 and below; one such query 10.4 -> 8.7 ms)
inline int64_t dense_batch_rows(const sofa_index* ix) {
  return ix->tune.dense_batch_rows > 0 ? ix->tune.dense_batch_rows : (ix->n >= 5 ? ix->n / 5 : 1);
}
int launch_dense(sofa_index* ix, int q, int k, float* od, int64_t* oi, bool stats, cudaStream_t st,
                 cudaEvent_t after_screen = nullptr);
int ensure_dense_scratch(sofa_index* ix, int q, int k);
int dense_dots(const float* rows, int64_t m, int len, const float* queries, int q, float* out, cudaStream_t st);
void free_dense_scratch(sofa_index* ix);
int launch_merge(const float* d, const int64_t* i, int parts, int q, int k, float* od, int64_t* oi, cudaStream_t st);
int launch_fill_pad(float* od, int64_t* oi, int64_t cnt, cudaStream_t st);
int launch_fill_value(float* o, int64_t cnt, float v, cudaStream_t st);
}  // namespace sofa
