// a5..a8: the exact k-NN query path.  One persistent kernel, k_query, in three modes:
//   front (mode 0): one CTA of 8 warps per query at a time (atomic query counter);
//   scan  (mode 1): every CTA pulls scan tasks (chunks of any query's remaining leaf list);
//   lower bounds (mode 2): sofa_lower_bounds (TLB evaluation).
//
// Front, per query:
//   a5  z-norm (shared row_stats, float32 q-hat for the refine, float64 for the projection),
//       float64 projection onto the l selected positions, then three l x 256 tables in shared
//       memory, each entry rounded DOWN to float32 (reading 15):
//         T  [j][s] = w_j * mind_j(q_j, s)^2                   word LB  (d_SFA)
//         Tlo[j][s] = w_j * max(0, beta_j(s)   - q_j)^2        envelope lower side
//         Thi[j][s] = w_j * max(0, q_j - beta_j(s+1))^2        envelope upper side
//   a6  seed: the query's own-key block (MESSI's approximate search) found by a 256-way
//       parallel search over the blocks' first keys, scanned + refined -> BSF0; the envelope tree
//       descent (leaf LB) -> the surviving leaves; top-M seeding (the 32 lowest word
//       LBs of the ~64 lowest-LB leaves are refined, SURVEY SIM-6) and a re-filter; the dense-path
//       decision (dense.cu); then up to a budget of leaves in ascending LB with MESSI's stop rule
//       (priority queue order), the rest published as scan tasks.
//   a7+a8  scan_blocks: barrier-free, warp-centric: a warp takes the next leaf, computes its words'
//       LBs (Alg. 3, chunks of 8 positions with early abandoning) and refines its
//       candidates in ascending LB, R rows at a time (exact squared z-ED with early abandoning,
//       P:382), improvements into the top-k sorted by (d^2, index).
// Scan: a rank-major task pool (every query's lowest-LB chunk first); a chunk whose first leaf LB
// exceeds the query's BSF is rejected unread; the CTA finishing a query's last task writes it.
// thr = BSF * (1 + 1e-4) + 1e-5 (squared units): prune only when the float32 lower bound clearly
// exceeds the float32 k-th best; this absorbs the data-side projection error (reading 15).
#include "common.cuh"

// This file is compiled twice: as itself (8-warp CTAs, 3 per SM: batches with several queries per
// CTA) and through query512.cu (16-warp CTAs, one per SM: batches of at most one query per SM,
// where a query's latency sets the step).  Each copy lives in its own namespace.
#ifndef SOFA_QTHREADS
#define SOFA_QTHREADS 256
#define SOFA_QNS q256
#define SOFA_QMAIN 1
#endif

namespace sofa {
namespace SOFA_QNS {

constexpr int kQThreads = SOFA_QTHREADS;  // threads per k_query CTA
constexpr int CAP_B = 2048;  // surviving blocks sorted in shared memory
constexpr int CAP_C = 2048;  // words per scan batch (l <= 16)
constexpr int TOPM_MIN_LEAVES = 256;  // top-M seeding for queries whose leaf list is longer than this (at least)
constexpr int TOPM_LEAVES = 64;       // ... over (about) this many lowest-LB leaves
constexpr int KMAX = SOFA_MAX_K;
constexpr int kFan = 16;  // envelope tree fan-out

// Front / scan split.  The front mode of k_query does the per-query steps (a5 tables, a6 seed and
// envelope descent, top-M seeding, the dense-path decision, a budget of leaves) and publishes the rest of
// the query's leaf list as scan tasks (chunks of leaves) into a global pool; the scan mode spreads
// all queries' tasks over all CTAs, so a heavy query no longer sits on one CTA.  A query's top-k
// lives in its QState while tasks are in flight; the CTA that finishes its last task writes the
// output.  Results do not depend on which CTA scans which chunk.
struct QState {
  int tkn, lock, ntasks, done;
  int ready;  // == the front launch's epoch once the front has handed the query over (tables, top-k, ntasks)
  float bsf, bsf_init;
  float tkd[SOFA_MAX_K];
  int tki[SOFA_MAX_K];
};
struct ScanTask {
  int64_t off;    // into the leaf pool
  int q;
  int cnt_flags;  // leaves | sorted << 30
};
// cnt_flags: leaf count | sorted list | range task (off = first leaf, no pool entries: every leaf of
// [off, off + cnt) in storage order)
constexpr int kTaskSorted = 1 << 30, kTaskRange = 1 << 29, kTaskCnt = (1 << 29) - 1;

struct QArgs {
  const float* series;
  int64_t n, nb;
  int len, l, a, WS, B;
  const uint8_t* words;
  const float2* stats;
  const int32_t* perm;
  const uint8_t* env;
  const uint64_t* bkey;
  const double* edges64;
  const double* basis64;
  const float* Q;
  int q, k;
  const float* bsf_init;
  float* od;
  int64_t* oi;
  int64_t goff;
  unsigned long long* gscratch;
  int nlev;
  int64_t lvl_off[8], lvl_cnt[8];
  int* qcounter;
  unsigned long long* dstats;
  long long* trace;  // nullable: per query SOFA_TRACE_FIELDS int64
  // dense path (f1, dense.cu): a query for which >= dense_pm permille of a strided word probe pass
  // its seed threshold is handed over before the tree descent (0 = never)
  int dense_pm;
  int64_t dense_rows;  // batch decision: dense pass iff the flagged queries' estimated refines >= this
  int dense_force;     // dense_permille >= 1000: every query with a surviving leaf goes dense (tests)
  int mode;            // 0: front, 1: scan, 2: lower-bound evaluation (sofa_lower_bounds), 3: seed bound
  float* seed_out;     // mode 3: per query, the k-th best squared distance of the seeded rows
  int64_t lb_m;        // mode 2: rows evaluated per query
  float *lb_out, *ed_out;
  int64_t* lb_rows;
  int front_batches;  // word batches of LB-ordered leaves the front scans itself per query
  int rev_rounds;     // scan_blocks: refine rounds per unit before it is deferred to the revisit pass
  int topm_min, topm_leaves;  // top-M seeding for lists longer than topm_min, over ~topm_leaves leaves
  QState* qs;          // q
  float* q_T;          // q x 3 x LT x 256: word-LB table T, then (range tasks only) Tlo, Thi
  float* q_hat;        // q x len z-normalised queries
  unsigned long long* pool;  // q x nb leaf entries (LB, block)
  unsigned long long* pool_used;
  // two task sets, rank-major: tasks[s][r * q + i] = i-th chunk of rank r (a query's r-th lowest-LB
  // chunk) in set s; set 0 = ordinary queries, set 1 = dense candidates (scanned only if the batch
  // skips the dense pass)
  ScanTask* tasks;     // 2 x rank_cap x q
  int* rank_count;     // 2 x rank_cap
  int rank_cap;
  int* counters;       // [2s] ranks used in set s, [2s+1] its cursor
  int* fcount;         // fused scan, one 128-byte line each: [0] fronts finished, [32] FIFO entries
                       // reserved, [64] FIFO tickets taken
  ScanTask* fifo;      // fused scan: set-0 tasks in publication order (instead of the rank-major table)
  int* fifo_seq;       // == epoch once fifo[i] is written (fifo_cap entries)
  int64_t fifo_cap;
  int epoch;
  int fused;           // front CTAs without a query left scan the set-0 tasks other fronts publish
  int* qd_counter;
  float* d_qhat;
  __nv_bfloat16* d_qb16;
  int xb_ld;
  int *d_ubn, *d_ublock;
  float4* d_qparams;
  int* d_qidx;
  float *d_binit, *d_bsf, *d_thr, *d_tkd;
  int *d_tki, *d_tkn, *d_lock, *d_overflow;
  unsigned long long* d_key1;
  float weights[SOFA_MAX_L];
};

__device__ __forceinline__ float thr_of(float bsf) { return isinf(bsf) ? INFINITY : bsf * (1.0f + 1e-4f) + 1e-5f; }

__device__ __forceinline__ unsigned long long pack(float lb, uint32_t id) {
  return ((unsigned long long)__float_as_uint(lb) << 32) | id;
}
__device__ __forceinline__ float lb_of(unsigned long long e) { return __uint_as_float((uint32_t)(e >> 32)); }

__device__ void bitonic_sort_u64(unsigned long long* s, int n) {
  int P2 = 1;
  while (P2 < n) P2 <<= 1;
  for (int i = n + threadIdx.x; i < P2; i += kQThreads) s[i] = ~0ull;
  __syncthreads();
  for (int k = 2; k <= P2; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P2; i += kQThreads) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const unsigned long long a = s[i], b = s[ixj];
          const bool up = (i & k) == 0;
          if ((a > b) == up) {
            s[i] = b;
            s[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
}

// warp-aggregated append of (key) into buf[*counter ...]
__device__ __forceinline__ void warp_append(bool pass, unsigned long long key, unsigned long long* buf, int* counter) {
  const unsigned m = __ballot_sync(FULL, pass);
  if (!m) return;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(m) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(counter, __popc(m));
  base = __shfl_sync(FULL, base, leader);
  if (pass) buf[base + __popc(m & ((1u << lane) - 1u))] = key;
}

struct QShared {
  int qi, cnt, tkn, take, rem, next, lock, gslot, chunk, chsz, ntask, nrev;
  long long off;
  float bsf, bsf_init, thr;
  // per query: 0 blocks_survived, 1 words_scanned, 2 candidates, 3 refined, 4 abandoned, 5 env_nodes,
  // 6 list_blocks, 7 rounds, 8 batches, 9 waves
  unsigned int st[10];
  int fpos[2], fcnt[2], nf;  // fused scan: this query's FIFO ranges, made visible at its handoff
};

// word LB (d_SFA^2 from the T table) with chunked early abandoning: Alg. 3.  The word's
// 16-byte chunks were loaded beforehand (all loads of a batch are in flight together).
template <int LT>
__device__ __forceinline__ float word_lb(const uint4 (&w)[LT / 16], const float* __restrict__ sT, float thr) {
  float lb = 0.f;
#pragma unroll
  for (int c = 0; c < LT / 16; ++c) {
    const uint32_t wv[4] = {w[c].x, w[c].y, w[c].z, w[c].w};
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // two chunks of 8 positions per 16 bytes
      float t[8];
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {
        const int j = c * 16 + h * 8 + jj;
        const uint32_t sym = (wv[(h * 8 + jj) >> 2] >> (8 * (jj & 3))) & 0xffu;
        t[jj] = sT[j * 256 + sym];
      }
      // pairwise sum: dependency depth 3 instead of 8 (LB rounding is absorbed by thr's slack)
      lb += ((t[0] + t[1]) + (t[2] + t[3])) + ((t[4] + t[5]) + (t[6] + t[7]));
      if (lb > thr) return lb;
    }
  }
  return lb;
}

// top-k insertion under a shared-memory spin lock (one lane of one warp at a time); updates the
// BSF (k-th best squared distance, or the caller's bound) and the pruning threshold.
__device__ void topk_insert(const QArgs& A, QShared& S, float* s_tkd, int* s_tki, float d, int i) {
  if (d > S.bsf_init) return;  // above the caller's bound: never part of the answer
  if (S.gslot >= 0) {          // scan mode: the query's top-k lives in its QState
    QState* h = &A.qs[S.gslot];
    while (atomicCAS(&h->lock, 0, 1) != 0) {
    }
    __threadfence();
    volatile float* td = h->tkd;
    volatile int* ti = h->tki;
    const int k = A.k;
    const int n = *(volatile int*)&h->tkn;
    float b = INFINITY;
    bool dup = false;  // a row refined twice (top-M seeding, then the scan) enters once
    for (int p = 0; p < n; ++p) dup |= ti[p] == i;
    if (!dup && (n < k || d < td[n - 1] || (d == td[n - 1] && i < ti[n - 1]))) {
      int p = n < k ? n : k - 1;
      while (p > 0 && (td[p - 1] > d || (td[p - 1] == d && ti[p - 1] > i))) {
        td[p] = td[p - 1];
        ti[p] = ti[p - 1];
        --p;
      }
      td[p] = d;
      ti[p] = i;
      const int nn = n < k ? n + 1 : k;
      *(volatile int*)&h->tkn = nn;
      if (nn == k) {
        b = fminf(S.bsf_init, td[k - 1]);
        *(volatile float*)&h->bsf = b;
      }
    }
    __threadfence();
    atomicExch(&h->lock, 0);
    if (b < INFINITY) {  // local mirror of the BSF (monotone: atomicMin on the bit patterns)
      atomicMin(reinterpret_cast<unsigned int*>(&S.bsf), __float_as_uint(b));
      atomicMin(reinterpret_cast<unsigned int*>(&S.thr), __float_as_uint(thr_of(b)));
    }
    return;
  }
  while (atomicCAS(&S.lock, 0, 1) != 0) {
  }
  __threadfence_block();
  const int k = A.k;
  const int n = S.tkn;
  bool dup = false;  // a row refined twice (top-M seeding, then the scan) enters once
  for (int p = 0; p < n; ++p) dup |= s_tki[p] == i;
  if (!dup && (n < k || d < s_tkd[n - 1] || (d == s_tkd[n - 1] && i < s_tki[n - 1]))) {
    int p = n < k ? n : k - 1;
    while (p > 0 && (s_tkd[p - 1] > d || (s_tkd[p - 1] == d && s_tki[p - 1] > i))) {
      s_tkd[p] = s_tkd[p - 1];
      s_tki[p] = s_tki[p - 1];
      --p;
    }
    s_tkd[p] = d;
    s_tki[p] = i;
    if (n < k) S.tkn = n + 1;
    if (S.tkn == k) {
      const float b = fminf(S.bsf_init, s_tkd[k - 1]);
      *(volatile float*)&S.bsf = b;
      *(volatile float*)&S.thr = thr_of(b);
    }
  }
  __threadfence_block();
  atomicExch(&S.lock, 0);
}

// rows a warp refines together in scan_blocks (R): more rows give more loads in flight, but R = 4 at
// n <= 256 spills at the 80-register cap of 3 CTAs per SM (configs[1] 9% slower than R = 2)
template <int NF>
__host__ __device__ constexpr int refine_rows() { return NF <= 4 ? 2 : 1; }

// a7 + a8 over a list of leaves, barrier-free and warp-centric.  Each warp pulls the next unit (a
// leaf, or a part of one) from a shared counter — in ascending leaf LB when the list is sorted, and
// stopping at the first leaf whose LB exceeds the BSF (MESSI's priority order and stop rule,
// P:173-176) — loads its words with 128-bit loads, computes their LBs from the shared-memory table
// (Alg. 3, chunks of 8 positions with early abandoning), then refines its candidates in ascending
// LB: R at a time (the R smallest by warp-min extraction), exact squared ED with early abandoning
// (P:382), improvements into the shared top-k.  The BSF every warp reads is the shared one, so a
// warp's improvement prunes the other warps' candidates at once; no CTA barrier inside the loop.
template <int LT, int NF, int RR = refine_rows<NF>()>
__device__ void scan_blocks(const QArgs& A, QShared& S, const unsigned long long* list, int cnt, bool sorted,
                            const float* s_T, float* s_tkd, int* s_tki, const float4* s_qh4, int seed_rounds = 0,
                            int64_t range0 = 0, const float* s_env = nullptr) {
  // list == nullptr: the leaves range0, range0 + 1, ... in storage order, each pruned by its envelope LB
  // (Tlo = s_env, Thi = s_env + LT * 256) before its words are read
  constexpr int NC = LT / 16;
  constexpr int WMAX = 8 / NC;                          // words per lane per unit
  constexpr int R = RR;  // rows refined together per warp
  constexpr int NW = kQThreads / 32;
  const int tid = threadIdx.x, lane = tid & 31;
  if (cnt <= 0) return;
  const int B = A.B;
  int ppl = B / (32 * WMAX);  // units per leaf
  if (ppl < 1) ppl = 1;
  while (ppl * 2 <= B / 32 && cnt * ppl < 2 * NW) ppl *= 2;  // short lists: split leaves over the warps
  const int span = B / ppl, wpl = span / 32;
  const int units = cnt * ppl;
  const int nf4 = A.len >> 2;
  // Pass 0 scans the list; a unit with more candidates than A.rev_rounds x R refines only its lowest
  // ones now (so the BSF keeps improving) and is queued for pass 1, which rescans it after the whole
  // list — under a BSF that is by then nearly final — skipping the candidates already refined.
  constexpr int REV_CAP = 128;
  __shared__ int s_rev_u[REV_CAP];
  __shared__ unsigned long long s_rev_k[REV_CAP];
  __syncthreads();
  if (tid == 0) {
    S.next = 0;
    S.nrev = 0;
  }
  __syncthreads();
  unsigned n_words = 0, n_cand = 0, n_ref = 0, n_ab = 0, n_units = 0, n_leaf = 0;
  for (int pass = 0; pass < 2; ++pass) {
    const int total = pass == 0 ? units : (S.nrev < REV_CAP ? S.nrev : REV_CAP);
    for (;;) {
      int idx = 0;
      float thr = 0.f;
      if (lane == 0) {
        idx = atomicAdd(&S.next, 1);
        thr = *(volatile float*)&S.thr;
      }
      idx = __shfl_sync(FULL, idx, 0);
      thr = __shfl_sync(FULL, thr, 0);
      if (idx >= total) break;
      const int u = pass == 0 ? idx : s_rev_u[idx];
      const unsigned long long done_key = pass == 0 ? 0ull : s_rev_k[idx];  // refined in pass 0: keys <= this
      const int e = u / ppl, part = u % ppl;
      unsigned long long ent;
      if (list) {
        // a pool list may have been written by another SM in this launch (fused scan): read it from L2
        ent = __isGlobal(list + e) ? __ldcg(list + e) : list[e];
      } else {  // range task: the leaf's envelope LB, lane j < LT takes position j
        const int64_t leaf = range0 + e;
        const uint8_t* ev = A.env + leaf * 2 * A.WS;
        float lbe = 0.f;
        if (lane < LT && lane < A.l) lbe = s_env[lane * 256 + ev[lane]] + s_env[(LT + lane) * 256 + ev[A.WS + lane]];
        if (LT > 32 && lane + 32 < A.l)
          lbe += s_env[(lane + 32) * 256 + ev[lane + 32]] + s_env[(LT + lane + 32) * 256 + ev[A.WS + lane + 32]];
        lbe = warp_sum_f32(lbe);
        ent = pack(lbe, (uint32_t)leaf);
      }
      if (lb_of(ent) > thr) {
        if (sorted && pass == 0) break;  // every later leaf has a larger LB
        continue;
      }
      if (pass == 0) {
        ++n_units;
        n_leaf += part == 0;
      }
      const int64_t base = (int64_t)(uint32_t)ent * B + (int64_t)part * span;
      uint4 wr[WMAX][NC];
      bool ok[WMAX];
#pragma unroll
      for (int i = 0; i < WMAX; ++i) {
        const int64_t pos = base + i * 32 + lane;
        ok[i] = i < wpl && pos < A.n;
#pragma unroll
        for (int c = 0; c < NC; ++c) wr[i][c] = ok[i] ? ld_stream_u4(A.words + pos * A.WS + 16 * c) : make_uint4(0u, 0u, 0u, 0u);
      }
      float lbv[WMAX];
#pragma unroll
      for (int i = 0; i < WMAX; ++i) {
        lbv[i] = ok[i] ? word_lb<LT>(wr[i], s_T, thr) : __int_as_float(0x7fffffff);  // NaN: never <= thr
        if (pass == 1 && ok[i] && pack(lbv[i], (uint32_t)(i * 32 + lane)) <= done_key)
          lbv[i] = __int_as_float(0x7fffffff);  // refined in pass 0
        if (pass == 0) {
          n_words += ok[i];
          n_cand += lbv[i] <= thr;
        }
      }
      unsigned long long last_key = 0ull;
      for (int rounds = 0;; ++rounds) {  // refine this unit's candidates, R lowest LBs at a time
        float bsf = 0.f;
        if (lane == 0) {
          thr = *(volatile float*)&S.thr;
          bsf = *(volatile float*)&S.bsf;
        }
        thr = __shfl_sync(FULL, thr, 0);
        bsf = __shfl_sync(FULL, bsf, 0);
        bool mine = false;
#pragma unroll
        for (int i = 0; i < WMAX; ++i) mine |= lbv[i] <= thr;
        if (!__any_sync(FULL, mine)) break;  // the common case: no candidate left in this unit
        if (seed_rounds > 0 && rounds == seed_rounds) break;  // seed leaf: it is scanned again from the list
        if (pass == 0 && rounds == A.rev_rounds) {  // many candidates: a loose BSF; revisit the rest later
          int slot = 0;
          if (lane == 0) slot = atomicAdd(&S.nrev, 1);
          slot = __shfl_sync(FULL, slot, 0);
          if (slot < REV_CAP) {
            if (lane == 0) {
              s_rev_u[slot] = u;
              s_rev_k[slot] = last_key;
            }
            break;
          }
        }
        const float* rows[R];
        float2 st[R];
        bool on[R];
        int oidx[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          unsigned long long best = ~0ull;
#pragma unroll
          for (int i = 0; i < WMAX; ++i)
            if (lbv[i] <= thr) {
              const unsigned long long key = pack(lbv[i], (uint32_t)(i * 32 + lane));
              best = key < best ? key : best;
            }
#pragma unroll
          for (int o = 16; o >= 1; o >>= 1) {
            const unsigned long long other = __shfl_xor_sync(FULL, best, o);
            best = other < best ? other : best;
          }
          on[r] = best != ~0ull;
          oidx[r] = -1;
          rows[r] = A.series;
          st[r] = make_float2(0.f, 0.f);
          if (on[r]) {
            last_key = best;
            const int slot = (int)(uint32_t)best;
#pragma unroll
            for (int i = 0; i < WMAX; ++i)
              if (slot == i * 32 + lane) lbv[i] = __int_as_float(0x7fffffff);  // taken
            const int64_t pos = base + slot;
            oidx[r] = A.perm[pos];
            st[r] = A.stats[pos];
            rows[r] = A.series + (int64_t)oidx[r] * A.len;
          }
        }
        float d2[R];
        bool ab[R];
        ed_warp_multi<NF, R>(rows, st, on, s_qh4, nf4, bsf, d2, ab);
        if (lane == 0) {
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if (!on[r]) continue;
            ++n_ref;
            if (ab[r]) {
              ++n_ab;
              continue;
            }
            bool ins;
            if (S.gslot >= 0) {
              ins = d2[r] <= *(volatile float*)&S.bsf;
            } else {
              const int n = *(volatile int*)&S.tkn;
              const float kd = *(volatile float*)&s_tkd[n > 0 ? n - 1 : 0];
              ins = n < A.k || d2[r] <= kd;
            }
            if (ins) topk_insert(A, S, s_tkd, s_tki, d2[r], oidx[r]);
          }
        }
      }
    }
    __syncthreads();
    if (tid == 0) S.next = 0;
    __syncthreads();
    if (S.nrev == 0) break;
  }
  n_cand = __reduce_add_sync(FULL, n_cand);
  n_words = __reduce_add_sync(FULL, n_words);
  if (lane == 0) {
    if (n_leaf) atomicAdd(&S.st[0], n_leaf);
    if (n_words) atomicAdd(&S.st[1], n_words);
    if (n_cand) atomicAdd(&S.st[2], n_cand);
    if (n_ref) atomicAdd(&S.st[3], n_ref);
    if (n_ab) atomicAdd(&S.st[4], n_ab);
    if (n_units) atomicAdd(&S.st[8], n_units);
    if (n_ref) atomicAdd(&S.st[9], (n_ref + R - 1) / R);
  }
  __syncthreads();
}

// leaves per word batch, per scan task (8 batches) and the front's own budget (64 batches)
template <int LT>
__device__ __forceinline__ int batch_blocks(int B) {
  constexpr int BW = LT == 16 ? CAP_C : (LT == 32 ? CAP_C / 2 : CAP_C / 4);
  return B <= BW ? BW / B : 1;
}
template <int LT>
__device__ __forceinline__ int chunk_blocks(int B) { return 8 * batch_blocks<LT>(B); }

// front: append `n` leaf entries of query q to the pool as scan tasks of ranks S.ntask, S.ntask+1, ...
template <int LT>
__device__ void publish_tasks(const QArgs& A, QShared& S, int q, const unsigned long long* list, int n, bool sorted,
                              bool dense_cand) {
  if (n <= 0) return;
  const int tid = threadIdx.x;
  const int set = dense_cand ? 1 : 0;
  if (tid == 0) {
    // ranks left for this query (rank_cap covers ceil(nb / CH) + 2 ranks; a query publishes at most
    // twice, so this never binds today): if the list needed more, its chunks grow instead of being
    // dropped — every published task is stored, so the query's done counter always reaches ntasks
    int CH = chunk_blocks<LT>(A.B);
    const int left = A.rank_cap - S.ntask;
    if (left <= 0) __trap();
    if ((n + CH - 1) / CH > left) CH = (n + left - 1) / left;
    S.chsz = CH;
    S.off = (long long)atomicAdd(A.pool_used, (unsigned long long)n);
    S.chunk = S.ntask;
    S.ntask += (n + CH - 1) / CH;
    if (!(A.fused && set == 0)) atomicMax(&A.counters[2 * set], S.ntask);
  }
  __syncthreads();
  const int CH = S.chsz;
  const int nt = (n + CH - 1) / CH;
  const int64_t off = S.off;
  const int r0 = S.chunk;
  for (int i = tid; i < n; i += kQThreads) A.pool[off + i] = list[i];
  const int flags = sorted ? kTaskSorted : 0;
  if (A.fused && set == 0) {
    // fused scan: a contiguous FIFO range for this call's tasks; their sequence numbers are written at
    // the query's handoff (after its state), so a consumer never holds a task it cannot start yet
    if (tid == 0) {
      S.fpos[S.nf] = atomicAdd(A.fcount + 32, nt);
      S.fcnt[S.nf] = nt;
      S.nf++;
    }
    __syncthreads();
    const int p0 = S.fpos[S.nf - 1];
    for (int i = tid; i < nt; i += kQThreads) {
      ScanTask t;
      t.off = off + (int64_t)i * CH;
      t.q = q;
      t.cnt_flags = (n - i * CH < CH ? n - i * CH : CH) | flags;
      A.fifo[p0 + i] = t;
    }
    __threadfence();  // this thread's pool entries and records, before the handoff's sequence numbers
    __syncthreads();
    return;
  }
  ScanTask* tasks = A.tasks + (int64_t)set * A.rank_cap * A.q;
  int* rc = A.rank_count + set * A.rank_cap;
  for (int i = tid; i < nt; i += kQThreads) {
    ScanTask t;
    t.off = off + (int64_t)i * CH;
    t.q = q;
    t.cnt_flags = (n - i * CH < CH ? n - i * CH : CH) | flags;
    const int r = r0 + i;  // < rank_cap by the CH choice above
    tasks[(int64_t)r * A.q + atomicAdd(&rc[r], 1)] = t;
  }
  __syncthreads();
}

// front: every leaf of the index as range tasks of the dense-candidate set (a query sent to the dense
// path before its tree descent; scanned only if the batch skips the dense pass)
template <int LT>
__device__ void publish_range(const QArgs& A, QShared& S, int q) {
  const int64_t n = A.nb;
  if (n <= 0) return;
  const int tid = threadIdx.x;
  if (tid == 0) {
    int64_t CH = chunk_blocks<LT>(A.B);
    const int left = A.rank_cap - S.ntask;
    if (left <= 0) __trap();
    if ((n + CH - 1) / CH > left) CH = (n + left - 1) / left;
    S.chsz = (int)CH;
    S.chunk = S.ntask;
    S.ntask += (int)((n + CH - 1) / CH);
    atomicMax(&A.counters[2], S.ntask);
  }
  __syncthreads();
  const int CH = S.chsz;
  const int nt = (int)((n + CH - 1) / CH);
  const int r0 = S.chunk;
  ScanTask* tasks = A.tasks + (int64_t)A.rank_cap * A.q;
  int* rc = A.rank_count + A.rank_cap;
  for (int i = tid; i < nt; i += kQThreads) {
    ScanTask t;
    t.off = (int64_t)i * CH;
    t.q = q;
    t.cnt_flags = (int)(n - (int64_t)i * CH < CH ? n - (int64_t)i * CH : CH) | kTaskRange;
    const int r = r0 + i;
    tasks[(int64_t)r * A.q + atomicAdd(&rc[r], 1)] = t;
  }
  __syncthreads();
}

// scan mode: all CTAs pull tasks until the pool is drained; rank-major order (every query's lowest-
// LB chunk first), so a query's later chunks usually meet its final BSF and are rejected unread
template <int LT, int NF, int RR = refine_rows<NF>()>
__device__ void scan_tasks(const QArgs& A, QShared& S, float* s_T, float* s_tkd, int* s_tki, float4* s_qh4,
                           float* s_env, bool fused = false) {
  const int tid = threadIdx.x;
  bool dense_go = false;
  if (A.qd_counter) {
    const int qd = *A.qd_counter;
    const unsigned long long est = *reinterpret_cast<const unsigned long long*>(A.qd_counter + 6);
    dense_go = qd > 0 && est >= (unsigned long long)A.dense_rows;
  }
  const int nsets = dense_go ? 1 : 2;
  __shared__ ScanTask s_task;
  __shared__ int s_have;
  if (tid == 0) {
    for (int i = 0; i < 10; ++i) S.st[i] = 0;
    S.gslot = -1;
  }
  int cur = -1, cur_env = -1;
  for (;;) {
    if (fused && tid == 0) {
      // a ticket = the next FIFO entry in publication order; wait until it is published, or until every
      // front has finished and the FIFO ends before it (then this CTA is done).  Every cross-CTA read
      // below is volatile or ld.global.cg (no L1-invalidating fence on the consumer side).
      // The counters live on separate 128-byte lines and a waiting CTA backs off exponentially (64 ns
      // .. 4 us): hundreds of idle CTAs polling one L2 line at full rate slowed the fronts still running.
      int have = 0;
      const int t = atomicAdd(A.fcount + 64, 1);
      unsigned ns = 64;
      for (;;) {
        if (t < A.fifo_cap && *(volatile int*)&A.fifo_seq[t] == A.epoch) {
          have = 1;
          break;
        }
        if (*(volatile int*)A.fcount >= A.q && *(volatile int*)(A.fcount + 32) <= t) break;
        __nanosleep(ns);
        ns = ns < 4096 ? 2 * ns : 4096;
      }
      s_have = have;
      if (have) {
        const volatile ScanTask* vt = &A.fifo[t];
        ScanTask tk;
        tk.off = vt->off;
        tk.q = vt->q;
        tk.cnt_flags = vt->cnt_flags;
        s_task = tk;
        volatile QState* h = &A.qs[tk.q];
        while (h->ready != A.epoch) __nanosleep(64);  // its front is still publishing
        const float thr = thr_of(h->bsf);
        S.take = (tk.cnt_flags & kTaskSorted) && lb_of(__ldcg(A.pool + tk.off)) > thr;
      }
    } else if (tid == 0) {
      int have = 0;
      for (int set = 0; set < nsets && !have; ++set) {
        const int ranks = A.counters[2 * set] < A.rank_cap ? A.counters[2 * set] : A.rank_cap;
        unsigned* cursor = reinterpret_cast<unsigned*>(&A.counters[2 * set + 1]);
        const int* rc = A.rank_count + set * A.rank_cap;
        for (;;) {  // rank-major cursor over tasks[r * q + i], jumping over each bucket's empty tail
          const unsigned t = atomicAdd(cursor, 1u);
          const int r = (int)(t / (unsigned)A.q), i = (int)(t % (unsigned)A.q);
          if (r >= ranks) break;
          if (i < rc[r]) {
            s_task = A.tasks[(int64_t)set * A.rank_cap * A.q + t];
            have = 1;
            break;
          }
          atomicMax(cursor, (unsigned)(r + 1) * (unsigned)A.q);
        }
      }
      s_have = have;
      if (have) {  // quick reject: a sorted chunk whose first leaf's LB is above the query's BSF
        volatile QState* h = &A.qs[s_task.q];
        const float thr = thr_of(h->bsf);
        S.take = (s_task.cnt_flags & kTaskSorted) && lb_of(A.pool[s_task.off]) > thr;
      }
    }
    __syncthreads();
    if (!s_have) break;
    const ScanTask tk = s_task;
    const int q = tk.q;
    volatile QState* h = &A.qs[q];
    if (!S.take) {
      if (q != cur) {
        const float4* T4 = reinterpret_cast<const float4*>(A.q_T + (int64_t)q * 3 * LT * 256);
        for (int i = tid; i < LT * 64; i += kQThreads) reinterpret_cast<float4*>(s_T)[i] = __ldcg(T4 + i);
        for (int i = tid; i < A.len; i += kQThreads)
          reinterpret_cast<float*>(s_qh4)[i] = __ldcg(A.q_hat + (int64_t)q * A.len + i);
        cur = q;
      }
      if (tid == 0) {
        S.gslot = q;
        S.bsf_init = h->bsf_init;
        S.bsf = h->bsf;
        S.thr = thr_of(S.bsf);
        S.next = 0;
        S.lock = 0;
      }
      __syncthreads();
      const bool range = (tk.cnt_flags & kTaskRange) != 0;
      if (range && q != cur_env) {  // the query's envelope tables Tlo / Thi (stored by the front)
        const float4* E4 = reinterpret_cast<const float4*>(A.q_T + ((int64_t)q * 3 + 1) * LT * 256);
        for (int i = tid; i < 2 * LT * 64; i += kQThreads) reinterpret_cast<float4*>(s_env)[i] = __ldcg(E4 + i);
        cur_env = q;
        __syncthreads();
      }
      scan_blocks<LT, NF, RR>(A, S, range ? nullptr : A.pool + tk.off, tk.cnt_flags & kTaskCnt,
                              (tk.cnt_flags & kTaskSorted) != 0, s_T, s_tkd, s_tki, s_qh4, 0, range ? tk.off : 0,
                              s_env);
      __syncthreads();
    }
    if (tid == 0) {
      __threadfence();
      S.take = atomicAdd(const_cast<int*>(&h->done), 1) == h->ntasks - 1;
      if (S.take) __threadfence();
      S.gslot = -1;
    }
    __syncthreads();
    if (S.take && tid == 0)  // last task of this query: write its result
      write_topk(h->tkd, h->tki, h->tkn, A.k, A.goff, A.od + (int64_t)q * A.k, A.oi + (int64_t)q * A.k);
    __syncthreads();
  }
  if (tid == 0 && A.dstats)
    for (int i = 0; i < 10; ++i)
      if (S.st[i]) atomicAdd(&A.dstats[2 + i], (unsigned long long)S.st[i]);
}

// envelope LB of a node (leaf LB): sum_j Tlo[j][min_j] + Thi[j][max_j]
template <int LT>
__device__ __forceinline__ float env_lb(const uint4 (&mn)[LT / 16], const uint4 (&mx)[LT / 16], const float* sTlo,
                                        const float* sThi) {
  float lb = 0.f;
#pragma unroll
  for (int c = 0; c < LT / 16; ++c) {
    const uint32_t vn[4] = {mn[c].x, mn[c].y, mn[c].z, mn[c].w}, vx[4] = {mx[c].x, mx[c].y, mx[c].z, mx[c].w};
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) {
      const int j = c * 16 + jj;
      lb += sTlo[j * 256 + ((vn[jj >> 2] >> (8 * (jj & 3))) & 0xffu)];
      lb += sThi[j * 256 + ((vx[jj >> 2] >> (8 * (jj & 3))) & 0xffu)];
    }
  }
  return lb;
}

// One level of the envelope tree: either every node of the level (parents == nullptr) or the
// F children of each listed parent whose LB is still <= thr.  Survivors (LB, node) -> out.
template <int LT>
__device__ void env_level(const QArgs& A, int L, const unsigned long long* parents, int nparents, int64_t b0,
                          float thr, const float* sTlo, const float* sThi, unsigned long long* out, int* counter,
                          unsigned int& stat_env) {
  constexpr int NC = LT / 16, U = 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int WS = A.WS;
  const uint8_t* base = A.env + A.lvl_off[L] * 2 * WS;
  const int64_t ncnt = A.lvl_cnt[L];
  const int64_t total = parents ? (int64_t)nparents * kFan : ncnt;
  for (int64_t ii = (int64_t)warp * 32 * U; ii < total; ii += (int64_t)kQThreads * U) {
    int64_t node[U];
    bool ok[U];
    uint4 mn[U][NC], mx[U][NC];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t idx = ii + u * 32 + lane;
      ok[u] = idx < total;
      node[u] = idx;
      if (ok[u] && parents) {
        const unsigned long long pe = parents[idx / kFan];
        node[u] = (int64_t)(uint32_t)pe * kFan + idx % kFan;
        ok[u] = lb_of(pe) <= thr && node[u] < ncnt;
      }
      ok[u] = ok[u] && !(L == 0 && node[u] == b0);
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        mn[u][c] = ok[u] ? ld_stream_u4(base + node[u] * 2 * WS + 16 * c) : make_uint4(0u, 0u, 0u, 0u);
        mx[u][c] = ok[u] ? ld_stream_u4(base + node[u] * 2 * WS + WS + 16 * c) : make_uint4(0u, 0u, 0u, 0u);
      }
    }
    unsigned int nev = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const float lb = ok[u] ? env_lb<LT>(mn[u], mx[u], sTlo, sThi) : INFINITY;
      nev += ok[u];
      warp_append(ok[u] && lb <= thr, pack(lb, (uint32_t)node[u]), out, counter);
    }
    nev = __reduce_add_sync(FULL, nev);
    if (lane == 0 && nev) atomicAdd(&stat_env, nev);
  }
}

// One pass over a block list: entries with LB > thr are dropped; entries with LB <= tau go to
// the shared-memory list `take` (up to CAP_B of them), the rest to `rem`.  4 entries per thread
// per iteration with all loads issued first.
__device__ void filter_list(const unsigned long long* src, int cnt, float thr, float tau, unsigned long long* take,
                            int* ntake, unsigned long long* rem, int* nrem, int cap = CAP_B) {
  constexpr int U = 4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int ee = warp * 32 * U; ee < cnt; ee += kQThreads * U) {
    unsigned long long ent[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = ee + u * 32 + lane;
      ent[u] = e < cnt ? src[e] : ~0ull;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = ee + u * 32 + lane;
      const float lbe = lb_of(ent[u]);
      const bool keep = e < cnt && lbe <= thr;
      const bool tk = keep && lbe <= tau;
      const unsigned m = __ballot_sync(FULL, tk);
      int base = 0;
      if (m) {
        const int leader = __ffs(m) - 1;
        if (lane == leader) base = atomicAdd(ntake, __popc(m));
        base = __shfl_sync(FULL, base, leader);
      }
      const int slot = base + __popc(m & ((1u << lane) - 1u));
      const bool got = tk && slot < cap;
      if (got) take[slot] = ent[u];
      if (rem) warp_append(keep && !got, ent[u], rem, nrem);
    }
  }
}

// Top-M seeding (SURVEY SIM-6): word LBs of the leaves in `list` (LB only, no refinement), then
// only the M = 32 lowest-LB words are refined (each warp keeps its 4 lowest in registers and
// refines them).  The lowest word LBs of the most promising leaves almost always include the true
// nearest neighbour, so the BSF is (nearly) final before the real scan starts — instead of being
// tightened one greedy batch at a time from the own-key seed.
template <int LT, int NF>
__device__ void seed_topm(const QArgs& A, QShared& S, const unsigned long long* list, int cnt, const float* s_T,
                          float* s_tkd, int* s_tki, const float4* s_qh4) {
  constexpr int NC = LT / 16;
  constexpr int WMAX = 8 / NC;
  constexpr int M = 4;  // per warp
  constexpr int NW = kQThreads / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int B = A.B;
  int ppl = B / (32 * WMAX);
  if (ppl < 1) ppl = 1;
  const int span = B / ppl, wpl = span / 32;
  const float thr = S.thr;
  unsigned long long best[M];
#pragma unroll
  for (int r = 0; r < M; ++r) best[r] = ~0ull;
  unsigned n_words = 0;
  for (int u = warp; u < cnt * ppl; u += NW) {
    const unsigned long long ent = list[u / ppl];
    const int64_t base = (int64_t)(uint32_t)ent * B + (int64_t)(u % ppl) * span;
    uint4 wr[WMAX][NC];  // all loads of the unit in flight together
#pragma unroll
    for (int i = 0; i < WMAX; ++i) {
      const int64_t pos = base + i * 32 + lane;
      const bool ok = i < wpl && pos < A.n;
#pragma unroll
      for (int c = 0; c < NC; ++c) wr[i][c] = ok ? ld_stream_u4(A.words + pos * A.WS + 16 * c) : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int i = 0; i < WMAX; ++i) {
      const int64_t pos = base + i * 32 + lane;
      if (i < wpl && pos < A.n) {
        const float lb = word_lb<LT>(wr[i], s_T, thr);
        ++n_words;
        unsigned long long key = lb <= thr ? pack(lb, (uint32_t)pos) : ~0ull;
#pragma unroll
        for (int r = 0; r < M; ++r)  // insert into this lane's sorted best-M
          if (key < best[r]) {
            const unsigned long long t = best[r];
            best[r] = key;
            key = t;
          }
      }
    }
  }
  // the warp's M lowest: M rounds of warp-min over the lanes' list heads
  const float* rows[M];
  float2 st[M];
  bool on[M];
  int oidx[M];
#pragma unroll
  for (int r = 0; r < M; ++r) {
    unsigned long long m = best[0];
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      const unsigned long long other = __shfl_xor_sync(FULL, m, o);
      m = other < m ? other : m;
    }
    on[r] = m != ~0ull;
    if (on[r] && best[0] == m) {  // the owner pops its head (keys are unique: they hold the position)
#pragma unroll
      for (int s = 0; s < M - 1; ++s) best[s] = best[s + 1];
      best[M - 1] = ~0ull;
    }
    oidx[r] = -1;
    rows[r] = A.series;
    st[r] = make_float2(0.f, 0.f);
    if (on[r]) {
      const uint32_t pos = (uint32_t)m;
      oidx[r] = A.perm[pos];
      st[r] = A.stats[pos];
      rows[r] = A.series + (int64_t)oidx[r] * A.len;
    }
  }
  float bsf = 0.f;
  if (lane == 0) bsf = *(volatile float*)&S.bsf;
  bsf = __shfl_sync(FULL, bsf, 0);
  float d2[M];
  bool ab[M];
  ed_warp_multi<NF, M>(rows, st, on, s_qh4, A.len >> 2, bsf, d2, ab);
  if (lane == 0) {
    unsigned n_ref = 0;
#pragma unroll
    for (int r = 0; r < M; ++r) {
      if (!on[r]) continue;
      ++n_ref;
      if (ab[r]) continue;
      const int n = *(volatile int*)&S.tkn;
      const float kd = *(volatile float*)&s_tkd[n > 0 ? n - 1 : 0];
      if (n < A.k || d2[r] <= kd) topk_insert(A, S, s_tkd, s_tki, d2[r], oidx[r]);
    }
    if (n_ref) atomicAdd(&S.st[3], n_ref);
  }
  n_words = __reduce_add_sync(FULL, n_words);
  if (lane == 0 && n_words) atomicAdd(&S.st[1], n_words);
  __syncthreads();
}

// f1 decision probe: the word LBs (against the query's current threshold) of kProbe words at strided
// positions of the sorted words; the passing fraction estimates the fraction of ALL rows the sparse path
// would refine (the stride covers the key order uniformly).  Returns the passing count (every thread).
constexpr int kProbe = 2048;
constexpr int kEarlyPermille = 100;     // stage 1 (before the tree descent): >= 10% of the probe passes
constexpr long long kDenseMinRows = 4096;  // ... and the estimate is at least this many rows
template <int LT>
__device__ long long dense_probe(const QArgs& A, QShared& S, const float* s_T) {
  constexpr int U = 128 / LT;  // words per thread in flight (8 x 16 B at l <= 16)
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t P = A.n < kProbe ? A.n : kProbe;
  if (tid == 0) S.take = 0;
  __syncthreads();
  const float thr = S.thr;
  int pass = 0;
  for (int64_t j0 = tid; j0 < P; j0 += (int64_t)kQThreads * U) {
    uint4 wr[U][LT / 16];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = j0 + (int64_t)u * kQThreads;
      const int64_t pos = j < P ? j * A.n / P : 0;
#pragma unroll
      for (int c = 0; c < LT / 16; ++c) wr[u][c] = ld_stream_u4(A.words + pos * A.WS + 16 * c);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (j0 + (int64_t)u * kQThreads < P) pass += word_lb<LT>(wr[u], s_T, thr) <= thr;
  }
  pass = __reduce_add_sync(FULL, pass);
  if (lane == 0 && pass) atomicAdd(&S.take, pass);
  __syncthreads();
  const long long npass = S.take;
  __syncthreads();
  return npass;
}
// flagged: at least `permille` of the probe passes AND that estimate is at least kDenseMinRows rows (a
// few hundred refines are cheaper than a share of a pass over all rows)
__device__ __forceinline__ bool dense_flag(const QArgs& A, long long npass, int64_t P, int permille) {
  return npass * 1000 >= (long long)permille * P && npass * A.n >= kDenseMinRows * P;
}
// thread 0: take a dense slot and add the query's estimated sparse refines to the batch decision
__device__ __forceinline__ int flag_dense(const QArgs& A, long long npass, int64_t P) {
  const unsigned long long est =
      A.dense_force ? (unsigned long long)A.dense_rows : (unsigned long long)(npass * A.n / (P > 0 ? P : 1));
  atomicAdd(reinterpret_cast<unsigned long long*>(A.qd_counter + 6), est);
  return atomicAdd(A.qd_counter, 1);
}

template <int LT, int NF, int RR = refine_rows<NF>()>
__global__ void __launch_bounds__(kQThreads, kQThreads == 256 ? 3 : 1) k_query(const __grid_constant__ QArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ QShared S;
  constexpr int UB0 = 2 * LT * 256 * 4, UB1 = CAP_B * 8, UB2 = NF * 128 * 8;
  constexpr int UB = UB0 > UB1 ? (UB0 > UB2 ? UB0 : UB2) : (UB1 > UB2 ? UB1 : UB2);
  float4* s_qh4 = reinterpret_cast<float4*>(smem);                         // NF*32 float4
  double* s_qproj = reinterpret_cast<double*>(smem + NF * 128 * 4);        // LT
  float* s_T = reinterpret_cast<float*>(smem + NF * 128 * 4 + LT * 8);     // LT*256
  unsigned char* s_u = smem + NF * 128 * 4 + LT * 8 + LT * 256 * 4;        // union
  float* s_Tlo = reinterpret_cast<float*>(s_u);
  float* s_Thi = s_Tlo + LT * 256;
  double* s_qd = reinterpret_cast<double*>(s_u);
  unsigned long long* s_blist = reinterpret_cast<unsigned long long*>(s_u);
  unsigned long long* s_samp = reinterpret_cast<unsigned long long*>(s_u + UB);  // strided list sample
  float* s_tkd = reinterpret_cast<float*>(s_samp + kQThreads);
  int* s_tki = reinterpret_cast<int*>(s_tkd + KMAX);
  __shared__ uint8_t s_qw[SOFA_MAX_L];
  __shared__ unsigned long long s_seed;
  __shared__ int s_dense;
  __shared__ long long s_dec[4];  // dense decision: flagged (1 stage 1, 2 stage 2), stage-2 pass, stage-1 pass, probe words

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int len = A.len, nf4 = len >> 2, l = A.l, a = A.a;
  unsigned long long* gl = A.gscratch + (int64_t)blockIdx.x * 2 * A.nb;  // the two halves swap roles
  unsigned long long* gl2 = gl + A.nb;

  if (A.mode == 1) {
    scan_tasks<LT, NF, RR>(A, S, s_T, s_tkd, s_tki, s_qh4, s_Tlo);
    return;
  }
  for (;;) {
    if (tid == 0) S.qi = atomicAdd(A.qcounter, 1);
    __syncthreads();
    const int qi = S.qi;
    if (qi >= A.q) break;
    long long t_phase[5], t_sub[2] = {0, 0}, t_blocks = 0;
    t_phase[0] = clock64();
    // ---------------------------------------------------------------- a5: z-norm + projection
    if (warp == 0) {
      // the row layout and statistics of k_transform (row_stats_g): every group of G lanes holds the
      // whole query, group 0 writes q-hat
      const float4* q4 = reinterpret_cast<const float4*>(A.Q + (int64_t)qi * len);
      const int G = row_group(nf4), g = lane & (G - 1);
      float4 x[8];
#pragma unroll
      for (int f = 0; f < 8; ++f) {
        const int fi = g + G * f;
        x[f] = fi < nf4 ? q4[fi] : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      float muf;
      double mu64, inv64;
      switch (G) {
        case 1: row_stats_g<1>(x, nf4, g, len, muf, mu64, inv64); break;
        case 2: row_stats_g<2>(x, nf4, g, len, muf, mu64, inv64); break;
        case 4: row_stats_g<4>(x, nf4, g, len, muf, mu64, inv64); break;
        case 8: row_stats_g<8>(x, nf4, g, len, muf, mu64, inv64); break;
        case 16: row_stats_g<16>(x, nf4, g, len, muf, mu64, inv64); break;
        default: row_stats_g<32>(x, nf4, g, len, muf, mu64, inv64); break;
      }
      const float invf = (float)inv64;
#pragma unroll
      for (int f = 0; f < 8; ++f) {
        const int fi = lane + G * f;
        if (lane < G && fi < nf4) {
          float4 h;
          h.x = __fmul_rn(__fsub_rn(x[f].x, muf), invf);
          h.y = __fmul_rn(__fsub_rn(x[f].y, muf), invf);
          h.z = __fmul_rn(__fsub_rn(x[f].z, muf), invf);
          h.w = __fmul_rn(__fsub_rn(x[f].w, muf), invf);
          s_qh4[fi] = h;
          s_qd[4 * fi + 0] = ((double)x[f].x - mu64) * inv64;
          s_qd[4 * fi + 1] = ((double)x[f].y - mu64) * inv64;
          s_qd[4 * fi + 2] = ((double)x[f].z - mu64) * inv64;
          s_qd[4 * fi + 3] = ((double)x[f].w - mu64) * inv64;
        }
      }
      if (lane == 0) {
        S.cnt = 0;
        S.tkn = 0;
        S.next = 0;
        S.lock = 0;
        S.gslot = -1;
        for (int i = 0; i < 10; ++i) S.st[i] = 0;
        const float bi = A.bsf_init ? A.bsf_init[qi] : INFINITY;
        S.bsf_init = bi;
        S.bsf = bi;
        S.thr = thr_of(bi);
      }
    }
    __syncthreads();
    for (int j = warp; j < LT; j += kQThreads / 32) {
      double acc = 0.0;
      if (j < l)
        for (int t0 = lane; t0 < len; t0 += 32 * 8) {  // 8 loads in flight, same summation order
          double b[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) b[u] = t0 + 32 * u < len ? A.basis64[(int64_t)j * len + t0 + 32 * u] : 0.0;
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (t0 + 32 * u < len) acc = fma(s_qd[t0 + 32 * u], b[u], acc);
        }
      acc = warp_sum_f64(acc);
      if (lane == 0) s_qproj[j] = acc;
    }
    __syncthreads();
    // ---------------------------------------------------------------- a5: LB tables (round down)
    for (int e0 = tid; e0 < LT * 256; e0 += kQThreads * 4) {
      double elo[4], ehi[4];  // the bin edges of 4 entries, loads in flight together
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = e0 + u * kQThreads, j = e >> 8, s = e & 255;
        const bool v = e < LT * 256 && j < l && s < a;
        elo[u] = !v || s == 0 ? -INFINITY : A.edges64[j * 256 + s - 1];
        ehi[u] = !v || s == a - 1 ? INFINITY : A.edges64[j * 256 + s];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * kQThreads;
      if (e >= LT * 256) break;
      const int j = e >> 8, s = e & 255;
      float t = 0.f, tlo = 0.f, thi = 0.f;
      if (j < l && s < a) {
        const double qv = s_qproj[j], w = (double)A.weights[j];
        const double lo = elo[u];
        const double hi = ehi[u];
        const double dl = fmax(0.0, lo - qv), dh = fmax(0.0, qv - hi);
        tlo = __double2float_rd(w * dl * dl);
        thi = __double2float_rd(w * dh * dh);
        t = __double2float_rd(w * (dl * dl + dh * dh));
        if (lo <= qv && qv < hi) s_qw[j] = (uint8_t)s;  // the query's own symbol
      }
      if (j >= l && s == 0 && j < SOFA_MAX_L) s_qw[j] = 0;
      s_T[e] = t;
      s_Tlo[e] = tlo;
      s_Thi[e] = thi;
      }
    }
    __syncthreads();
    if (A.mode == 2) {
      // lower-bound evaluation (TLB): for rows at sorted positions floor(j n / m), the squared
      // word LB from this query's table (no abandoning) and the exact squared z-ED
      for (int64_t j = warp; j < A.lb_m; j += kQThreads / 32) {
        const int64_t pos = j * A.n / A.lb_m;
        const float* rows[1] = {A.series + (int64_t)A.perm[pos] * len};
        const float2 st[1] = {A.stats[pos]};
        const bool on[1] = {true};
        float d2[1];
        bool ab[1];
        ed_warp_multi<NF, 1>(rows, st, on, s_qh4, nf4, INFINITY, d2, ab);
        if (lane == 0) {
          uint4 wr[LT / 16];
#pragma unroll
          for (int c = 0; c < LT / 16; ++c) wr[c] = ld_stream_u4(A.words + pos * A.WS + 16 * c);
          A.lb_out[(int64_t)qi * A.lb_m + j] = word_lb<LT>(wr, s_T, INFINITY);
          A.ed_out[(int64_t)qi * A.lb_m + j] = d2[0];
          if (qi == 0) A.lb_rows[j] = A.goff + A.perm[pos];
        }
      }
      __syncthreads();
      continue;
    }
    // ---------------------------------------------------------------- a6: seed block
    const uint64_t key = word_key(s_qw, l, 31 - __clz(a));
    int64_t lo = 0, hi = A.nb;
    while (hi - lo > 1) {  // 256-way parallel search: largest b with bkey[b] <= key
      const int64_t step = (hi - lo + kQThreads - 1) / kQThreads;
      const int64_t idx = lo + (int64_t)tid * step;
      const int c = __syncthreads_count(idx < hi && A.bkey[idx] <= key);
      if (c == 0) {
        hi = lo + 1;
        break;
      }
      const int64_t nlo = lo + (int64_t)(c - 1) * step;
      hi = nlo + step < hi ? nlo + step : hi;
      lo = nlo;
    }
    const int64_t b0 = lo;
    t_phase[1] = clock64();
    if (tid == 0) s_seed = pack(0.f, (uint32_t)b0);
    __syncthreads();
    // own-key seed: the R lowest-LB words of each warp's part of the leaf, as many rounds as it
    // takes to fill k; no revisit (the leaf is not excluded from the tree descent below: b0 = -1,
    // so its remaining candidates are scanned again from the list)
    scan_blocks<LT, NF, RR>(A, S, &s_seed, A.nb > 0 ? 1 : 0, true, s_T, s_tkd, s_tki, s_qh4,
                            1 + (A.k - 1) / (kQThreads / 32 * RR));
    t_phase[2] = clock64();
    if (A.mode == 3) {  // sofa_knn_seed: this shard's own-key bound on the k-th best, nothing else
      if (tid == 0) A.seed_out[qi] = S.tkn == A.k ? S.bsf : INFINITY;
      __syncthreads();
      continue;
    }
    // ---------------------------------------------------------------- f1: dense-path decision, stage 1
    // Before the tree descent: a query for which >= 10% of a strided word probe (dense_probe) passes the
    // seed's threshold is one the SFA bound cannot prune (high-frequency data, noisy members with
    // sigma = 1): it goes to the batched tensor-core screen (dense.cu) without walking the envelope
    // tree.  Queries below that are decided again after top-M seeding (stage 2) at dense_pm.
    if (tid == 0) {
      s_dense = -1;
      s_dec[0] = s_dec[1] = s_dec[2] = s_dec[3] = 0;
    }
    __syncthreads();
    if (A.mode == 0 && A.dense_pm > 0) {
      const long long npass = dense_probe<LT>(A, S, s_T);
      const int64_t P = A.n < kProbe ? A.n : kProbe;
      if (tid == 0) {
        if (A.dense_force || dense_flag(A, npass, P, kEarlyPermille)) {
          s_dense = flag_dense(A, npass, P);
          s_dec[0] = 1;
        }
        s_dec[2] = npass;
        s_dec[3] = P;
      }
      __syncthreads();
    }
    const bool early_dense = s_dense >= 0;
    if (tid == 0) S.cnt = 0;
    __syncthreads();
    // ---------------------------------------------------------------- a6: envelope tree descent
    // top level: every node; lower levels: the kFan children of each surviving parent
    // (the MESSI-style tree over sorted SFA-word blocks, P:159-166 / P:171-173)
    if (!early_dense) {
      const float thr = S.thr;
      unsigned long long* cur = gl;
      unsigned long long* nxt = gl2;
      env_level<LT>(A, A.nlev - 1, nullptr, 0, -1, thr, s_Tlo, s_Thi, cur, &S.cnt, S.st[5]);
      for (int L = A.nlev - 2; L >= 0; --L) {
        __syncthreads();
        const int np = S.cnt;
        if (tid == 0) S.rem = 0;
        __syncthreads();
        env_level<LT>(A, L, cur, np, -1, S.thr, s_Tlo, s_Thi, nxt, &S.rem, S.st[5]);
        __syncthreads();
        if (tid == 0) S.cnt = S.rem;
        unsigned long long* t = cur;
        cur = nxt;
        nxt = t;
      }
      if (cur != gl) {  // the rounds below start from gl
        __syncthreads();
        for (int i = tid; i < S.cnt; i += kQThreads) gl[i] = cur[i];
      }
      __syncthreads();  // S.cnt and gl are final for every thread
    }
    t_phase[3] = clock64();
    // ---------------------------------------------------------------- a6 -> a7/a8: LB-ordered processing
    // MESSI processes leaves in ascending LB from priority queues and abandons a queue at the
    // first leaf whose LB exceeds the BSF.  Here: if the surviving blocks fit in
    // shared memory they are bitonic-sorted and scanned in ascending LB with that stop rule.
    // Otherwise the ~CAP_B lowest-LB blocks (threshold tau from a sorted strided sample) are
    // sorted and scanned first — that tightens the BSF to (nearly) its final value — and the rest
    // is re-filtered against it and scanned in storage order (LB re-checked per block).
    {
      int cnt = S.cnt;
      if (tid == 0) S.st[6] += cnt;
      if (cnt > A.topm_min) {
        // top-M seeding over the TOPM_LEAVES lowest-LB leaves (threshold from a sorted strided sample)
        s_samp[tid] = gl[((int64_t)tid * cnt) / kQThreads];
        if (tid == 0) S.take = 0;
        __syncthreads();
        bitonic_sort_u64(s_samp, kQThreads);
        int r = (int)(((int64_t)kQThreads * A.topm_leaves) / cnt);
        r = r < 0 ? 0 : (r > kQThreads - 1 ? kQThreads - 1 : r);
        const float tau = lb_of(s_samp[r]);
        filter_list(gl, cnt, S.thr, tau, s_blist, &S.take, nullptr, nullptr, A.topm_leaves);
        __syncthreads();
        const int nt = S.take < A.topm_leaves ? S.take : A.topm_leaves;
        seed_topm<LT, NF>(A, S, s_blist, nt, s_T, s_tkd, s_tki, s_qh4);
        // re-filter the leaf list against the (nearly final) BSF
        if (tid == 0) {
          S.take = 0;
          S.rem = 0;
        }
        __syncthreads();
        filter_list(gl, cnt, S.thr, -1.f, s_blist, &S.take, gl2, &S.rem);
        __syncthreads();
        cnt = S.rem;
        unsigned long long* t = gl;
        gl = gl2;
        gl2 = t;
      }
      t_sub[0] = clock64();  // top-M seeding done
      // f1 stage 2: the same probe under the (nearly final) bound of top-M seeding, at dense_pm permille —
      // only once the batch's dense pass is certain (the flagged estimates already add up to dense_rows;
      // the sum only grows), so a query flagged here never falls back to the scan pool's dense-candidate
      // set, and a batch without a dense pass keeps every query on the ordinary sparse path
      // (read once by thread 0: the counter moves, and the branch below must be block-uniform)
      if (tid == 0)
        S.take = A.qd_counter && *reinterpret_cast<volatile unsigned long long*>(A.qd_counter + 6) >=
                                     (unsigned long long)A.dense_rows;
      __syncthreads();
      const bool batch_dense = S.take != 0;
      __syncthreads();
      if (A.mode == 0 && A.dense_pm > 0 && !early_dense && cnt > 0 && batch_dense) {
        const long long npass = dense_probe<LT>(A, S, s_T);
        const int64_t P = A.n < kProbe ? A.n : kProbe;
        if (tid == 0) {
          if (dense_flag(A, npass, P, A.dense_pm)) {
            s_dense = flag_dense(A, npass, P);
            s_dec[0] = 2;
          }
          s_dec[1] = npass;
        }
        __syncthreads();
      }
      if (s_dense >= 0) {
        // publish the query's state to its dense slot; dense.cu finishes it
        const int slot = s_dense;
        for (int t = tid; t < len; t += kQThreads) {
          const float v = reinterpret_cast<const float*>(s_qh4)[t];
          A.d_qhat[(int64_t)slot * len + t] = v;
          A.d_qb16[(int64_t)slot * A.xb_ld + t] = __float2bfloat16_rn(v);  // the screen's operand
        }
        for (int r = tid; r < S.tkn; r += kQThreads) {
          A.d_tkd[(int64_t)slot * A.k + r] = s_tkd[r];
          A.d_tki[(int64_t)slot * A.k + r] = s_tki[r];
        }
        if (warp == 0) {
          double nq = 0.0;
          for (int t = lane; t < len; t += 32) {
            const double v = reinterpret_cast<const float*>(s_qh4)[t];
            nq += v * v;
          }
          nq = warp_sum_f64(nq);
          if (lane == 0) {
            // bf16 operands round to nearest (relative error <= 2^-8 each), products are exact, the
            // fp32 accumulation is bounded as a naive sum (K 2^-24) and doubled: |dot error| <=
            // gamma |x^| |q^| with |x^| <= sqrt(1.0001 n); plus slack for |x^|^2 = n (float32
            // statistics) and the refine's own float32 rounding (dense.cu header, DESIGN reading 29)
            const double gamma = 0x1p-7 + 0x1p-15 + (double)len * 0x1p-23;
            const double eps = 2.0 * gamma * sqrt(1.0001 * len) * sqrt(nq) + 2e-4 * (nq + len) + 1e-3;
            A.d_qparams[slot] = make_float4((float)nq, (float)eps, 0.f, 0.f);
            A.d_qidx[slot] = qi;
            A.d_binit[slot] = S.bsf_init;
            A.d_bsf[slot] = S.bsf;
            A.d_thr[slot] = S.tkn == A.k ? S.bsf : S.bsf_init;  // proven bound on the k-th best (or +inf)
            A.d_tkn[slot] = S.tkn;
            A.d_key1[slot] = S.tkn > 0 ? ((unsigned long long)__float_as_uint(s_tkd[0]) << 32) | (uint32_t)s_tki[0] : ~0ull;
            A.d_lock[slot] = 0;
            A.d_ubn[slot] = 0;
            A.d_ublock[slot] = 0;
            A.d_overflow[slot] = 0;
          }
        }
      }
      t_sub[1] = clock64();  // dense decision done
      // the remaining leaves, in ascending LB (MESSI's priority-queue order): up to
      // `budget` of them are scanned here with the stop rule; what a heavy query has left beyond that
      // becomes scan tasks spread over all CTAs.  A dense candidate's leaves are only published
      // (scanned only if the batch decides against the dense pass).
      const bool dc = s_dense >= 0;
      const int CH = chunk_blocks<LT>(A.B);
      const int budget = A.front_batches * batch_blocks<LT>(A.B);  // leaves the front scans itself
      if (tid == 0) {
        S.ntask = 0;
        S.nf = 0;
      }
      __syncthreads();
      if (dc && early_dense) {
        // a dense candidate's rows are only needed if the batch skips the dense pass: every leaf, in
        // storage order, as range tasks (no list is built for a query that usually never scans)
        publish_range<LT>(A, S, qi);
      } else if (dc) {
        // flagged at stage 2, when the batch's dense pass was already certain: nothing to publish
      } else if (cnt <= CAP_B) {
        for (int i = tid; i < cnt; i += kQThreads) s_blist[i] = gl[i];
        __syncthreads();
        bitonic_sort_u64(s_blist, cnt);
        int nloc = dc ? 0 : (cnt < budget ? cnt : budget);
        if (!dc && cnt - nloc <= CH) nloc = cnt;  // short remainder: finish it here
        if (nloc) {
          const long long c0 = clock64();
          scan_blocks<LT, NF, RR>(A, S, s_blist, nloc, true, s_T, s_tkd, s_tki, s_qh4);
          t_blocks += clock64() - c0;
        }
        int rest = cnt - nloc;
        if (!dc && rest > 0 && lb_of(s_blist[nloc]) > S.thr) rest = 0;  // stop rule: nothing left below the BSF
        publish_tasks<LT>(A, S, qi, s_blist + nloc, rest, true, dc);
      } else {
        if (tid == 0) S.st[7] += 1;
        s_samp[tid] = gl[((int64_t)tid * cnt) / kQThreads];
        if (tid == 0) {
          S.take = 0;
          S.rem = 0;
        }
        __syncthreads();
        bitonic_sort_u64(s_samp, kQThreads);
        int r = (int)(((int64_t)kQThreads * (CAP_B * 3 / 4)) / cnt);
        r = r < 0 ? 0 : (r > kQThreads - 1 ? kQThreads - 1 : r);
        const float tau = lb_of(s_samp[r]);
        filter_list(gl, cnt, S.thr, tau, s_blist, &S.take, gl2, &S.rem);
        __syncthreads();
        const int ntake = S.take < CAP_B ? S.take : CAP_B;
        const int nrem = S.rem;
        bitonic_sort_u64(s_blist, ntake);
        const int nloc = dc ? 0 : (ntake < budget ? ntake : budget);
        if (nloc) {
          const long long c0 = clock64();
          scan_blocks<LT, NF, RR>(A, S, s_blist, nloc, true, s_T, s_tkd, s_tki, s_qh4);
          t_blocks += clock64() - c0;
        }
        int rest = ntake - nloc;
        if (!dc && rest > 0 && lb_of(s_blist[nloc]) > S.thr) rest = 0;
        publish_tasks<LT>(A, S, qi, s_blist + nloc, rest, true, dc);
        if (nrem > 0) {
          if (tid == 0) {
            S.take = 0;
            S.rem = 0;
          }
          __syncthreads();
          filter_list(gl2, nrem, S.thr, -1.f, s_blist, &S.take, gl, &S.rem);
          __syncthreads();
          publish_tasks<LT>(A, S, qi, gl, S.rem, false, dc);
        }
      }
      __syncthreads();
      if (S.ntask > 0) {  // hand the query's state to the scan CTAs
        QState* h = &A.qs[qi];
        if (tid == 0 && A.dstats) {
          atomicAdd(&A.dstats[22], (unsigned long long)S.ntask);
          atomicAdd(&A.dstats[23], 1ull);
        }
        for (int i = tid; i < LT * 256; i += kQThreads) A.q_T[(int64_t)qi * 3 * LT * 256 + i] = s_T[i];
        if (early_dense)  // range tasks prune leaves by their envelope LB: they need Tlo / Thi too
          for (int i = tid; i < 2 * LT * 256; i += kQThreads) A.q_T[((int64_t)qi * 3 + 1) * LT * 256 + i] = s_Tlo[i];
        for (int i = tid; i < len; i += kQThreads) A.q_hat[(int64_t)qi * len + i] = reinterpret_cast<const float*>(s_qh4)[i];
        for (int r = tid; r < S.tkn; r += kQThreads) {
          h->tkd[r] = s_tkd[r];
          h->tki[r] = s_tki[r];
        }
        __syncthreads();
        if (tid == 0) {
          h->tkn = S.tkn;
          h->lock = 0;
          h->ntasks = S.ntask;
          h->done = 0;
          h->bsf = S.bsf;
          h->bsf_init = S.bsf_init;
          __threadfence();  // tables, q-hat, top-k and ntasks before the flag the FIFO consumers wait on
          *(volatile int*)&h->ready = A.epoch;
        }
        __syncthreads();
        for (int f = 0; f < S.nf; ++f)  // the query's FIFO entries become visible only now
          for (int i = tid; i < S.fcnt[f]; i += kQThreads) *(volatile int*)&A.fifo_seq[S.fpos[f] + i] = A.epoch;
      }
    }
    // ---------------------------------------------------------------- output
    if (s_dense < 0 && S.ntask == 0 && tid == 0)
      write_topk(s_tkd, s_tki, S.tkn, A.k, A.goff, A.od + (int64_t)qi * A.k, A.oi + (int64_t)qi * A.k);
    t_phase[4] = clock64();
    if (tid == 0 && A.dstats) {
      atomicAdd(&A.dstats[0], 1ull);
      atomicAdd(&A.dstats[1], (unsigned long long)A.nb);
      for (int i = 0; i < 10; ++i) atomicAdd(&A.dstats[2 + i], (unsigned long long)S.st[i]);
      for (int i = 0; i < 4; ++i) atomicAdd(&A.dstats[12 + i], (unsigned long long)(t_phase[i + 1] - t_phase[i]));
      atomicMax(&A.dstats[16], (unsigned long long)(t_phase[4] - t_phase[0]));
      atomicMax(&A.dstats[17], (unsigned long long)S.st[6]);
      atomicMax(&A.dstats[18], (unsigned long long)S.st[8]);
    }
    if (tid == 0 && A.trace) {
      long long* tr = A.trace + (int64_t)qi * SOFA_TRACE_FIELDS;
      for (int i = 0; i < 4; ++i) tr[i] = t_phase[i + 1] - t_phase[i];
      // the scan phase split: top-M seeding, dense decision, front scan_blocks, the rest (sorts,
      // filters, task publishing)
      if (t_sub[0] && t_sub[1]) {
        tr[20] = t_sub[0] - t_phase[3];
        tr[21] = t_sub[1] - t_sub[0];
        tr[22] = t_blocks;
        tr[23] = t_phase[4] - t_sub[1] - t_blocks;
      } else {
        tr[20] = tr[21] = tr[22] = tr[23] = 0;
      }
      for (int i = 0; i < 10; ++i) tr[4 + i] = S.st[i];
      tr[14] = blockIdx.x;
      for (int i = 0; i < 4; ++i) tr[16 + i] = s_dec[i];
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      tr[15] = smid;
    }
    if (tid == 0 && A.fused) {  // this query's front is finished (its tasks and state are published)
      __threadfence();
      atomicAdd(A.fcount, 1);
    }
    __syncthreads();
  }
  // no query left for this CTA: drain the FIFO of set-0 tasks other fronts publish (or still will)
  if (A.mode == 0 && A.fused) scan_tasks<LT, NF, RR>(A, S, s_T, s_tkd, s_tki, s_qh4, s_Tlo, true);
}

template <int LT, int NF, int RR = refine_rows<NF>()>
static int launch_query_t(sofa_index* ix, const QArgs& A0, cudaStream_t st) {
  QArgs A = A0;
  constexpr int UB0 = 2 * LT * 256 * 4, UB1 = CAP_B * 8, UB2 = NF * 128 * 8;
  constexpr int UB = UB0 > UB1 ? (UB0 > UB2 ? UB0 : UB2) : (UB1 > UB2 ? UB1 : UB2);
  const size_t smem = NF * 128 * 4 + LT * 8 + LT * 256 * 4 + UB + kQThreads * 8 + KMAX * 8;
  auto kern = k_query<LT, NF, RR>;
  // launch shape, once per instantiation and device (no driver queries on the per-call path; racing
  // first calls set the same attribute and store the same value)
  static std::atomic<int> per_sm_cache[16];
  std::atomic<int>& slot = per_sm_cache[ix->device & 15];
  int per_sm = slot.load();
  if (per_sm == 0) {
    SOFA_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    SOFA_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kQThreads, smem));
    if (per_sm < 1) per_sm = 1;
    slot.store(per_sm);
  }
  const int sms = ix->sms;
  // the whole GPU even for a small batch: CTAs without a query of their own help heavy ones
  const int grid = sms * per_sm;
  const int64_t need = (int64_t)grid * 2 * (ix->nb > 0 ? ix->nb : 1);
  if (ix->gscratch_ctas < need) {
    if (ix->gscratch) cudaFree(ix->gscratch);
    ix->gscratch = nullptr;
    SOFA_CK(cudaMalloc(&ix->gscratch, need * 8));
    ix->gscratch_ctas = need;
  }
  A.gscratch = ix->gscratch;
  // qcounter ints: [0] query queue, [2..3] leaf pool entries used (u64), [4..7] scan counters
  A.pool_used = reinterpret_cast<unsigned long long*>(ix->qcounter + 2);
  A.counters = ix->qcounter + 4;
  if (A.mode == 0) {
    const int BW = LT == 16 ? CAP_C : (LT == 32 ? CAP_C / 2 : CAP_C / 4);
    const int CH = 8 * (ix->B <= BW ? BW / ix->B : 1);
    const int64_t qn = A.q, nb = ix->nb > 0 ? ix->nb : 1;
    const int64_t ranks = (nb + CH - 1) / CH + 2;  // chunks one query can publish
    const int64_t pool_need = qn * nb, task_need = qn * ranks;
    if (ix->scan_q_cap != qn || ix->scan_LT != LT || ix->pool_cap < pool_need || ix->task_cap < task_need) {
      void* old[] = {ix->qstate, ix->q_T, ix->q_hat, ix->pool, ix->tasks, ix->rank_count};
      for (void* o : old)
        if (o) cudaFree(o);
      ix->qstate = ix->q_T = ix->q_hat = ix->pool = ix->tasks = ix->rank_count = nullptr;
      SOFA_CK(cudaMalloc(&ix->qstate, (size_t)qn * sizeof(QState)));
      SOFA_CK(cudaMalloc(&ix->q_T, (size_t)qn * 3 * LT * 256 * 4));
      SOFA_CK(cudaMalloc(&ix->q_hat, (size_t)qn * SOFA_MAX_LEN * 4));
      SOFA_CK(cudaMalloc(&ix->pool, (size_t)pool_need * 8));
      SOFA_CK(cudaMalloc(&ix->tasks, (size_t)2 * task_need * sizeof(ScanTask)));
      SOFA_CK(cudaMalloc(&ix->rank_count, (size_t)2 * ranks * 4));
      if (ix->fifo) cudaFree(ix->fifo);
      if (ix->fifo_seq) cudaFree(ix->fifo_seq);
      SOFA_CK(cudaMalloc(&ix->fifo, (size_t)task_need * sizeof(ScanTask)));
      SOFA_CK(cudaMalloc(&ix->fifo_seq, (size_t)(task_need + 4096) * 4));
      // epoch-tagged entries and states: zeroed once, so no stale value can match an epoch (>= 1)
      SOFA_CK(cudaMemsetAsync(ix->fifo_seq, 0, (size_t)(task_need + 4096) * 4, st));
      SOFA_CK(cudaMemsetAsync(ix->qstate, 0, (size_t)qn * sizeof(QState), st));
      ix->scan_q_cap = qn;
      ix->scan_LT = LT;
      ix->pool_cap = pool_need;
      ix->task_cap = task_need;
      ix->rank_cap = ranks;
    }
    SOFA_CK(cudaMemsetAsync(ix->qcounter, 0, 16 * sizeof(int), st));
    SOFA_CK(cudaMemsetAsync(ix->rank_count, 0, (size_t)2 * ix->rank_cap * 4, st));
    if (!ix->fcount) SOFA_CK(cudaMalloc(&ix->fcount, 512));
    SOFA_CK(cudaMemsetAsync(ix->fcount, 0, 512, st));
    ix->epoch = ix->epoch + 1 > 0 ? ix->epoch + 1 : 1;  // a new front launch
  } else if (A.mode >= 2) {
    SOFA_CK(cudaMemsetAsync(ix->qcounter, 0, 16 * sizeof(int), st));
  }
  A.rank_count = reinterpret_cast<int*>(ix->rank_count);
  A.rank_cap = (int)ix->rank_cap;
  A.fifo = reinterpret_cast<ScanTask*>(ix->fifo);
  A.fifo_seq = reinterpret_cast<int*>(ix->fifo_seq);
  A.fifo_cap = ix->task_cap + 4096;
  A.fcount = ix->fcount;
  A.epoch = ix->epoch;
  A.fused = A.mode == 0 && ix->tune.scan_fused != 0;
  A.qs = reinterpret_cast<QState*>(ix->qstate);
  A.q_T = reinterpret_cast<float*>(ix->q_T);
  A.q_hat = reinterpret_cast<float*>(ix->q_hat);
  A.pool = reinterpret_cast<unsigned long long*>(ix->pool);
  A.tasks = reinterpret_cast<ScanTask*>(ix->tasks);
  kern<<<grid, kQThreads, smem, st>>>(A);
  SOFA_LAUNCHED();
  return SOFA_OK;
}

int launch_query_impl(sofa_index* ix, const float* Q, int q, int k, const float* bsf_init, float* od, int64_t* oi,
                      cudaStream_t st, bool scan, int64_t lb_m, float* lb_out, float* ed_out, int64_t* lb_rows,
                      float* seed_out) {
  QArgs A{};
  A.mode = seed_out ? 3 : (lb_m > 0 ? 2 : (scan ? 1 : 0));
  A.seed_out = seed_out;
  A.lb_m = lb_m;
  A.lb_out = lb_out;
  A.ed_out = ed_out;
  A.lb_rows = lb_rows;
  const sofa_tuning& T = ix->tune;
  // the front's own budget of LB-ordered word batches per query.  (With the fused scan, 8 batches made
  // configs[1] 4% faster on average but bimodal: a query whose sampled top-M threshold picked few
  // leaves then refined ~6k rows in its front in ~40% of the steps, 1.8 ms instead of 0.5.)
  A.front_batches = T.front_batches > 0 ? T.front_batches : 16;
  A.rev_rounds = T.rev_rounds;
  // top-M seeding only for lists longer than ~1/16 of the index, in [TOPM_MIN_LEAVES, CAP_B] leaves: a
  // shorter list is cheaper to scan in LB order directly (configs[1]: 0.64 -> 0.61 ms at 2048)
  A.topm_min = T.topm_min > 0 ? T.topm_min
                              : (int)(ix->nb / 16 < TOPM_MIN_LEAVES ? TOPM_MIN_LEAVES : (ix->nb / 16 > CAP_B ? CAP_B : ix->nb / 16));
  A.topm_leaves = T.topm_leaves > 0 ? (T.topm_leaves < CAP_B ? T.topm_leaves : CAP_B) : TOPM_LEAVES;
  A.series = ix->series;
  A.n = ix->n;
  A.nb = ix->nb;
  A.len = ix->len;
  A.l = ix->l;
  A.a = ix->a;
  A.WS = ix->WS;
  A.B = ix->B;
  A.words = ix->words;
  A.stats = ix->stats;
  A.perm = ix->perm;
  A.env = ix->env;
  A.bkey = ix->bkey;
  A.nlev = ix->nlev;
  for (int L = 0; L < 8; ++L) {
    A.lvl_off[L] = ix->lvl_off[L];
    A.lvl_cnt[L] = ix->lvl_cnt[L];
  }
  A.edges64 = ix->edges64;
  A.basis64 = ix->basis64;
  A.Q = Q;
  A.q = q;
  A.k = k;
  A.bsf_init = bsf_init;
  A.od = od;
  A.oi = oi;
  A.goff = ix->global_offset;
  A.qcounter = ix->qcounter;
  A.dstats = ix->dstats;
  A.trace = ix->trace_on ? ix->trace + ix->trace_off * SOFA_TRACE_FIELDS : nullptr;
  if (ix->dense_permille > 0 && ix->xb16 && ix->dense.q_cap >= q) {
    const DenseScratch& D = ix->dense;
    A.dense_pm = ix->dense_permille < 1000 ? ix->dense_permille : 1000;
    A.dense_rows = dense_batch_rows(ix);
    A.dense_force = ix->dense_permille >= 1000;
    A.qd_counter = D.counters;
    A.d_qhat = D.qhat;
    A.d_qb16 = D.qb16;
    A.xb_ld = ix->xb_ld;
    A.d_ubn = D.ubn;
    A.d_ublock = D.ub_lock;
    A.d_qparams = D.qparams;
    A.d_qidx = D.qidx;
    A.d_binit = D.binit;
    A.d_bsf = D.bsf;
    A.d_thr = D.thr;
    A.d_tkd = D.tkd;
    A.d_tki = D.tki;
    A.d_tkn = D.tkn;
    A.d_key1 = D.key1;
    A.d_lock = D.lock;
    A.d_overflow = D.overflow;
  }
  for (int j = 0; j < SOFA_MAX_L; ++j) A.weights[j] = j < ix->l ? (float)ix->model.weights[j] : 0.f;
  const int nf4 = ix->len / 4;
  const int NF = nf4 <= 32 ? 1 : nf4 <= 64 ? 2 : nf4 <= 128 ? 4 : 8;
  // rows per refine round in the front: 2 (no register spills: best when every CTA runs several
  // queries, configs[1] 0.57 vs 0.62 ms) or, for n <= 256 and at most one query per CTA, 4 (more row
  // loads in flight per warp: a batch that small is set by its slowest, refine-bound query;
  // configs[0] 0.55 vs 0.63 ms).  The scan pool is indifferent (measured) and uses 2.
  const int sms = ix->sms;
  int rsel = A.mode == 0 && A.q <= 3 * sms ? 4 : 2;
  const int rt = A.mode == 1 ? T.refine_rows_scan : T.refine_rows_front;
  if (rt) rsel = rt;
#define SOFA_Q(lt, nf) \
  if (ix->LT == lt && NF == nf) {                                                       \
    if (nf <= 2 && rsel == 4) return launch_query_t<lt, (nf <= 2 ? nf : 1), 4>(ix, A, st); \
    return launch_query_t<lt, nf>(ix, A, st);                                           \
  }
  SOFA_Q(16, 1) SOFA_Q(16, 2) SOFA_Q(16, 4) SOFA_Q(16, 8)
  SOFA_Q(32, 1) SOFA_Q(32, 2) SOFA_Q(32, 4) SOFA_Q(32, 8)
  SOFA_Q(64, 1) SOFA_Q(64, 2) SOFA_Q(64, 4) SOFA_Q(64, 8)
#undef SOFA_Q
  set_error("query: unsupported (len, l)");
  return SOFA_EINVAL;
}

// ---------------------------------------------------------------------------------------------
// a9: min-merge of `parts` sorted (dist, idx) lists per query; ties -> smaller index.
__global__ void k_merge_topk(const float* __restrict__ d, const int64_t* __restrict__ ix, int parts, int q, int k,
                             float* __restrict__ od, int64_t* __restrict__ oi) {
  const int qi = blockIdx.x * blockDim.x + threadIdx.x;
  if (qi >= q) return;
  int head[64];
  for (int p = 0; p < parts; ++p) head[p] = 0;
  for (int r = 0; r < k; ++r) {
    int best = -1;
    float bd = INFINITY;
    int64_t bi = -1;
    for (int p = 0; p < parts; ++p) {
      if (head[p] >= k) continue;
      const int64_t o = ((int64_t)p * q + qi) * k + head[p];
      const int64_t ci = ix[o];
      if (ci < 0) continue;
      const float cd = d[o];
      if (best < 0 || cd < bd || (cd == bd && ci < bi)) {
        best = p;
        bd = cd;
        bi = ci;
      }
    }
    if (best >= 0) head[best]++;
    od[(int64_t)qi * k + r] = best >= 0 ? bd : INFINITY;
    oi[(int64_t)qi * k + r] = best >= 0 ? bi : -1;
  }
}

int launch_merge(const float* d, const int64_t* i, int parts, int q, int k, float* od, int64_t* oi, cudaStream_t st) {
  k_merge_topk<<<(q + 127) / 128, 128, 0, st>>>(d, i, parts, q, k, od, oi);
  SOFA_LAUNCHED();
  return SOFA_OK;
}

__global__ void k_fill_value(float* o, int64_t cnt, float v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x)
    o[i] = v;
}

int launch_fill_value(float* o, int64_t cnt, float v, cudaStream_t st) {
  k_fill_value<<<(int)((cnt + 255) / 256 < 1024 ? (cnt + 255) / 256 : 1024), 256, 0, st>>>(o, cnt, v);
  SOFA_LAUNCHED();
  return SOFA_OK;
}

__global__ void k_fill_pad(float* od, int64_t* oi, int64_t cnt) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x) {
    od[i] = INFINITY;
    oi[i] = -1;
  }
}

int launch_fill_pad(float* od, int64_t* oi, int64_t cnt, cudaStream_t st) {
  if (cnt <= 0) return SOFA_OK;
  k_fill_pad<<<(int)((cnt + 255) / 256 < 1024 ? (cnt + 255) / 256 : 1024), 256, 0, st>>>(od, oi, cnt);
  SOFA_LAUNCHED();
  return SOFA_OK;
}

}  // namespace SOFA_QNS

#ifdef SOFA_QMAIN
int launch_query_q512(sofa_index* ix, const float* Q, int q, int k, const float* bsf_init, float* od, int64_t* oi,
                      cudaStream_t st, bool scan, int64_t lb_m, float* lb_out, float* ed_out, int64_t* lb_rows,
                      float* seed_out);

// a batch with at most one query per SM runs the 16-warp build (a lone query gets twice the warps:
// configs[0] 0.55 -> 0.43 ms for the front, -> 0.40 ms with the scan pool too); every other launch
// the 8-warp build (3 CTAs per SM)
int launch_query(sofa_index* ix, const float* Q, int q, int k, const float* bsf_init, float* od, int64_t* oi,
                 cudaStream_t st, bool scan, int64_t lb_m, float* lb_out, float* ed_out, int64_t* lb_rows,
                 float* seed_out) {
  const int wt = scan ? ix->tune.scan_wide : ix->tune.front_wide;  // -1 auto, 0 never, 1 always
  const bool wide = lb_m == 0 && !seed_out && (wt == 1 || (wt == -1 && q <= ix->sms));
  if (wide) return launch_query_q512(ix, Q, q, k, bsf_init, od, oi, st, scan, lb_m, lb_out, ed_out, lb_rows, seed_out);
  return q256::launch_query_impl(ix, Q, q, k, bsf_init, od, oi, st, scan, lb_m, lb_out, ed_out, lb_rows, seed_out);
}
int launch_merge(const float* d, const int64_t* i, int parts, int q, int k, float* od, int64_t* oi, cudaStream_t st) {
  return q256::launch_merge(d, i, parts, q, k, od, oi, st);
}
int launch_fill_value(float* o, int64_t cnt, float v, cudaStream_t st) { return q256::launch_fill_value(o, cnt, v, st); }
int launch_fill_pad(float* od, int64_t* oi, int64_t cnt, cudaStream_t st) { return q256::launch_fill_pad(od, oi, cnt, st); }
#else
int launch_query_q512(sofa_index* ix, const float* Q, int q, int k, const float* bsf_init, float* od, int64_t* oi,
                      cudaStream_t st, bool scan, int64_t lb_m, float* lb_out, float* ed_out, int64_t* lb_rows,
                      float* seed_out) {
  return SOFA_QNS::launch_query_impl(ix, Q, q, k, bsf_init, od, oi, st, scan, lb_m, lb_out, ed_out, lb_rows, seed_out);
}
#endif
}  // namespace sofa
