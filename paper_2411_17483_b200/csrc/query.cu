// a5..a8: the exact k-NN query path as ONE persistent kernel (one CTA of 8 warps per query at a
// time; CTAs pull queries from an atomic counter so uneven per-query work balances out).
//
// Per query:
//   a5  z-norm (shared row_stats, float32 q-hat for the refine, float64 for the projection),
//       float64 projection onto the l selected positions, then three l x 256 tables in shared
//       memory, each entry rounded DOWN to float32 (reading 15):
//         T  [j][s] = w_j * mind_j(q_j, s)^2                   word LB  (d_SFA)
//         Tlo[j][s] = w_j * max(0, beta_j(s)   - q_j)^2        envelope lower side
//         Thi[j][s] = w_j * max(0, q_j - beta_j(s+1))^2        envelope upper side
//   a6  seed: the query's own-key block (MESSI's approximate search) found by a
//       256-way parallel search over the blocks' first keys, scanned + refined -> BSF0;
//       then the envelope LB of every block (leaf LB); blocks with LB <= thr are
//       appended to a per-CTA list and, when <= CAP_B of them survive, bitonic-sorted by LB in
//       shared memory (MESSI's priority queue: process leaves in ascending LB, stop
//       at the first whose LB exceeds the BSF).
//   a7  word LB scan of the listed blocks in batches of CAP_C words: 16-byte word loads, table
//       gathers in chunks of 8 positions with early abandoning (Alg. 3), survivors
//       appended to a shared candidate buffer (warp-aggregated atomics).
//   a8  candidates sorted by LB, refined in waves of 8 (one warp per candidate, float4 row
//       loads, warp-shuffle reduction, early abandoning per 256-element chunk vs BSF),
//       top-k kept sorted by (d^2, index); refinement stops at the first candidate whose LB
//       exceeds the threshold.
// thr = BSF * (1 + 1e-4) + 1e-5 (squared units): prune only when the float32 lower bound clearly
// exceeds the float32 k-th best; this absorbs the data-side projection error (reading 15).
#include "common.cuh"

namespace sofa {

constexpr int CAP_B = 2048;  // surviving blocks sorted in shared memory
constexpr int CAP_C = 2048;  // words per scan batch = candidate buffer capacity
constexpr int KMAX = SOFA_MAX_K;
constexpr int kFan = 16;  // envelope tree fan-out

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
  for (int i = n + threadIdx.x; i < P2; i += kThreads) s[i] = ~0ull;
  __syncthreads();
  for (int k = 2; k <= P2; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P2; i += kThreads) {
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
  int qi, cnt, ncand, tkn, b0, take, rem, next, lock;
  float bsf, bsf_init, thr;
  // per query: 0 blocks_survived, 1 words_scanned, 2 candidates, 3 refined, 4 abandoned, 5 env_nodes,
  // 6 list_blocks, 7 rounds, 8 batches, 9 waves
  unsigned int st[10];
};

// exact squared z-ED with early abandoning (a8) for R candidate rows at once: one warp, float4
// loads of all R rows issued together (R rows in flight per warp), chunks of 2 float4 per lane
// (256 values), partial sums warp-reduced after each chunk and compared with the BSF.
template <int NF, int R>
__device__ __forceinline__ void ed_warp_multi(const float* const (&rows)[R], const float2 (&st)[R],
                                              const bool (&on)[R], const float4* s_qh4, int nf4, float bsf,
                                              float (&d2)[R], bool (&ab)[R]) {
  const int lane = threadIdx.x & 31;
  constexpr int CH = NF < 2 ? NF : 2;
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
  while (atomicCAS(&S.lock, 0, 1) != 0) {
  }
  __threadfence_block();
  const int k = A.k;
  const int n = S.tkn;
  if (n < k || d < s_tkd[n - 1] || (d == s_tkd[n - 1] && i < s_tki[n - 1])) {
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

// a8: refine the candidate buffer.  Candidates are bitonic-sorted by LB when there are more than
// 8; then every warp independently pulls the next R candidates in ascending-LB order (atomic
// counter), skips those whose LB exceeds the current threshold (and stops, the list being
// sorted), computes their exact distances with R rows in flight, and inserts improvements into
// the top-k.  No CTA-wide barrier per candidate wave.
template <int LT, int NF>
__device__ void refine_candidates(const QArgs& A, QShared& S, unsigned long long* s_cand, float* s_tkd, int* s_tki,
                                  const float4* s_qh4) {
  constexpr int R = NF <= 2 ? 2 : 1;  // rows in flight per warp
  const int tid = threadIdx.x, lane = tid & 31;
  const int nc = S.ncand;
  if (nc == 0) return;
  const bool sorted = nc > 8;
  if (sorted) bitonic_sort_u64(s_cand, nc);
  const int nf4 = A.len >> 2;
  unsigned int n_ref = 0, n_ab = 0, n_waves = 0;
  for (;;) {
    int c0 = 0;
    if (lane == 0) c0 = atomicAdd(&S.next, R);
    c0 = __shfl_sync(FULL, c0, 0);
    if (c0 >= nc) break;
    // lane 0 reads the (concurrently updated) threshold and broadcasts it: every lane must take
    // the same branch below, since ed_warp_multi uses full-warp shuffles
    float thr = 0.f, bsf = 0.f;
    if (lane == 0) {
      thr = *(volatile float*)&S.thr;
      bsf = *(volatile float*)&S.bsf;
    }
    thr = __shfl_sync(FULL, thr, 0);
    bsf = __shfl_sync(FULL, bsf, 0);
    const float* rows[R];
    float2 st[R];
    bool on[R];
    int oidx[R];
    bool any = false;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int c = c0 + r;
      const unsigned long long e = c < nc ? s_cand[c] : ~0ull;
      on[r] = c < nc && lb_of(e) <= thr;
      oidx[r] = -1;
      rows[r] = A.series;
      st[r] = make_float2(0.f, 0.f);
      if (on[r]) {
        const uint32_t pos = (uint32_t)e;
        oidx[r] = A.perm[pos];
        st[r] = A.stats[pos];
        rows[r] = A.series + (int64_t)oidx[r] * A.len;
        any = true;
      }
    }
    if (!any) {
      if (sorted) break;  // every later candidate has a larger LB
      continue;
    }
    float d2[R];
    bool ab[R];
    ed_warp_multi<NF, R>(rows, st, on, s_qh4, nf4, bsf, d2, ab);
    ++n_waves;
    if (lane == 0) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (!on[r]) continue;
        ++n_ref;
        if (ab[r]) {
          ++n_ab;
          continue;
        }
        const int n = *(volatile int*)&S.tkn;
        const float kd = *(volatile float*)&s_tkd[n > 0 ? n - 1 : 0];
        if (n < A.k || d2[r] <= kd) topk_insert(A, S, s_tkd, s_tki, d2[r], oidx[r]);
      }
    }
  }
  if (lane == 0) {
    if (n_ref) atomicAdd(&S.st[3], n_ref);
    if (n_ab) atomicAdd(&S.st[4], n_ab);
    if (n_waves) atomicAdd(&S.st[9], n_waves);
  }
  __syncthreads();
  if (tid == 0) {
    S.ncand = 0;
    S.next = 0;
  }
  __syncthreads();
}

// scan the words of the listed blocks (a7) and refine (a8), batch by batch.  The words of batch
// i+1 are loaded into registers before batch i's candidates are appended and refined, so their
// HBM latency overlaps the refine (software pipelining over the batch loop).
template <int LT, int NF>
__device__ void scan_blocks(const QArgs& A, QShared& S, const unsigned long long* list, int cnt, bool sorted,
                            const float* s_T, unsigned long long* s_cand, float* s_tkd, int* s_tki, float* s_wd,
                            int* s_wi, const float4* s_qh4) {
  const int tid = threadIdx.x;
  const int B = A.B;
  constexpr int BW = LT == 16 ? CAP_C : (LT == 32 ? CAP_C / 2 : CAP_C / 4);  // words per batch
  const int G = B <= BW ? BW / B : 1;    // blocks per batch
  const int SUB = B <= BW ? 1 : B / BW;  // batches per block
  const int span = B <= BW ? B : BW;
  const int nbatch = ((cnt + G - 1) / G) * SUB;
  if (nbatch == 0) return;
  constexpr int WPT = BW / kThreads;  // words per thread per batch
  constexpr int NC = LT / 16;
  int64_t pos[WPT];
  bool valid[WPT];
  uint4 wr[WPT][NC];
  auto issue = [&](int bi, float thr) {
    const int e0 = (bi / SUB) * G, sub = bi % SUB;
#pragma unroll
    for (int t = 0; t < WPT; ++t) {
      const int w = tid + t * kThreads;
      const int u = w / span, m = w % span;
      const int e = e0 + u;
      valid[t] = bi < nbatch && e < cnt && u < G;
      pos[t] = 0;
      if (valid[t]) {
        const unsigned long long ent = list[e];
        pos[t] = (int64_t)(uint32_t)ent * B + (int64_t)sub * BW + m;
        valid[t] = lb_of(ent) <= thr && pos[t] < A.n;
      }
#pragma unroll
      for (int c = 0; c < NC; ++c)
        wr[t][c] = valid[t] ? ld_stream_u4(A.words + pos[t] * A.WS + 16 * c) : make_uint4(0u, 0u, 0u, 0u);
    }
  };
  issue(0, S.thr);
  for (int bi = 0; bi < nbatch; ++bi) {
    const float thr = S.thr;
    const int e0 = (bi / SUB) * G, sub = bi % SUB;
    if (sorted && lb_of(list[e0]) > thr) return;  // every later block has a larger LB
    if (tid == 0) S.st[8] += 1;
    if (tid == 0 && sub == 0) {
      unsigned int surv = 0;
      for (int u = 0; u < G && e0 + u < cnt; ++u) surv += lb_of(list[e0 + u]) <= thr;
      S.st[0] += surv;
    }
    float lbs[WPT];
    bool vcur[WPT];
    int64_t pcur[WPT];
    unsigned int scanned = 0;
#pragma unroll
    for (int t = 0; t < WPT; ++t) {
      vcur[t] = valid[t];
      pcur[t] = pos[t];
      lbs[t] = valid[t] ? word_lb<LT>(wr[t], s_T, thr) : INFINITY;
      scanned += valid[t];
    }
    issue(bi + 1, thr);  // next batch's loads fly during this batch's append + refine
#pragma unroll
    for (int t = 0; t < WPT; ++t)
      warp_append(vcur[t] && lbs[t] <= thr, pack(lbs[t], (uint32_t)pcur[t]), s_cand, &S.ncand);
    scanned = __reduce_add_sync(FULL, scanned);
    if ((tid & 31) == 0 && scanned) atomicAdd(&S.st[1], scanned);
    __syncthreads();
    if (tid == 0) S.st[2] += S.ncand;
    refine_candidates<LT, NF>(A, S, s_cand, s_tkd, s_tki, s_qh4);
  }
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
  for (int64_t ii = (int64_t)warp * 32 * U; ii < total; ii += (int64_t)kThreads * U) {
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
                            int* ntake, unsigned long long* rem, int* nrem) {
  constexpr int U = 4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int ee = warp * 32 * U; ee < cnt; ee += kThreads * U) {
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
      const bool got = tk && slot < CAP_B;
      if (got) take[slot] = ent[u];
      warp_append(keep && !got, ent[u], rem, nrem);
    }
  }
}

template <int LT, int NF>
__global__ void __launch_bounds__(kThreads, 2) k_query(const QArgs A) {
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
  unsigned long long* s_cand = reinterpret_cast<unsigned long long*>(s_u + UB);
  float* s_tkd = reinterpret_cast<float*>(s_cand + CAP_C);
  int* s_tki = reinterpret_cast<int*>(s_tkd + KMAX);
  float* s_wd = reinterpret_cast<float*>(s_tki + KMAX);
  int* s_wi = reinterpret_cast<int*>(s_wd + 8);
  __shared__ uint8_t s_qw[SOFA_MAX_L];
  __shared__ unsigned long long s_seed;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int len = A.len, nf4 = len >> 2, l = A.l, a = A.a;
  unsigned long long* gl = A.gscratch + (int64_t)blockIdx.x * 2 * A.nb;
  unsigned long long* gl2 = gl + A.nb;

  for (;;) {
    if (tid == 0) S.qi = atomicAdd(A.qcounter, 1);
    __syncthreads();
    const int qi = S.qi;
    if (qi >= A.q) break;
    long long t_phase[5];
    t_phase[0] = clock64();
    // ---------------------------------------------------------------- a5: z-norm + projection
    if (warp == 0) {
      const float4* q4 = reinterpret_cast<const float4*>(A.Q + (int64_t)qi * len);
      float4 x[NF];
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        const int fi = lane + 32 * f;
        x[f] = fi < nf4 ? q4[fi] : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      float muf;
      double mu64, inv64;
      row_stats<NF>(x, nf4, len, muf, mu64, inv64);
      const float invf = (float)inv64;
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        const int fi = lane + 32 * f;
        if (fi < nf4) {
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
        S.ncand = 0;
        S.tkn = 0;
        S.next = 0;
        S.lock = 0;
        for (int i = 0; i < 10; ++i) S.st[i] = 0;
        const float bi = A.bsf_init ? A.bsf_init[qi] : INFINITY;
        S.bsf_init = bi;
        S.bsf = bi;
        S.thr = thr_of(bi);
      }
    }
    __syncthreads();
    for (int j = warp; j < LT; j += 8) {
      double acc = 0.0;
      if (j < l)
        for (int t = lane; t < len; t += 32) acc = fma(s_qd[t], A.basis64[(int64_t)j * len + t], acc);
      acc = warp_sum_f64(acc);
      if (lane == 0) s_qproj[j] = acc;
    }
    __syncthreads();
    // ---------------------------------------------------------------- a5: LB tables (round down)
    for (int e = tid; e < LT * 256; e += kThreads) {
      const int j = e >> 8, s = e & 255;
      float t = 0.f, tlo = 0.f, thi = 0.f;
      if (j < l && s < a) {
        const double qv = s_qproj[j], w = (double)A.weights[j];
        const double lo = s == 0 ? -INFINITY : A.edges64[j * 256 + s - 1];
        const double hi = s == a - 1 ? INFINITY : A.edges64[j * 256 + s];
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
    __syncthreads();
    // ---------------------------------------------------------------- a6: seed block
    const uint64_t key = word_key(s_qw, l, 31 - __clz(a));
    int64_t lo = 0, hi = A.nb;
    while (hi - lo > 1) {  // 256-way parallel search: largest b with bkey[b] <= key
      const int64_t step = (hi - lo + kThreads - 1) / kThreads;
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
    scan_blocks<LT, NF>(A, S, &s_seed, A.nb > 0 ? 1 : 0, true, s_T, s_cand, s_tkd, s_tki, s_wd, s_wi, s_qh4);
    t_phase[2] = clock64();
    // ---------------------------------------------------------------- a6: envelope tree descent
    // top level: every node; lower levels: the kFan children of each surviving parent
    // (the MESSI-style tree over sorted SFA-word blocks, P:159-166 / P:171-173)
    {
      const float thr = S.thr;
      unsigned long long* cur = gl;
      unsigned long long* nxt = gl2;
      env_level<LT>(A, A.nlev - 1, nullptr, 0, b0, thr, s_Tlo, s_Thi, cur, &S.cnt, S.st[5]);
      for (int L = A.nlev - 2; L >= 0; --L) {
        __syncthreads();
        const int np = S.cnt;
        if (tid == 0) S.rem = 0;
        __syncthreads();
        env_level<LT>(A, L, cur, np, b0, S.thr, s_Tlo, s_Thi, nxt, &S.rem, S.st[5]);
        __syncthreads();
        if (tid == 0) S.cnt = S.rem;
        unsigned long long* t = cur;
        cur = nxt;
        nxt = t;
      }
      if (cur != gl) {  // the rounds below start from gl
        __syncthreads();
        for (int i = tid; i < S.cnt; i += kThreads) gl[i] = cur[i];
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
      const int cnt = S.cnt;
      if (tid == 0) S.st[6] += cnt;
      if (cnt <= CAP_B) {
        for (int i = tid; i < cnt; i += kThreads) s_blist[i] = gl[i];
        __syncthreads();
        bitonic_sort_u64(s_blist, cnt);
        scan_blocks<LT, NF>(A, S, s_blist, cnt, true, s_T, s_cand, s_tkd, s_tki, s_wd, s_wi, s_qh4);
      } else {
        if (tid == 0) S.st[7] += 1;
        s_cand[tid] = gl[((int64_t)tid * cnt) / kThreads];
        if (tid == 0) {
          S.take = 0;
          S.rem = 0;
        }
        __syncthreads();
        bitonic_sort_u64(s_cand, kThreads);
        int r = (int)(((int64_t)kThreads * (CAP_B * 3 / 4)) / cnt);
        r = r < 0 ? 0 : (r > kThreads - 1 ? kThreads - 1 : r);
        const float tau = lb_of(s_cand[r]);
        filter_list(gl, cnt, S.thr, tau, s_blist, &S.take, gl2, &S.rem);
        __syncthreads();
        const int ntake = S.take < CAP_B ? S.take : CAP_B;
        const int nrem = S.rem;
        bitonic_sort_u64(s_blist, ntake);
        scan_blocks<LT, NF>(A, S, s_blist, ntake, true, s_T, s_cand, s_tkd, s_tki, s_wd, s_wi, s_qh4);
        if (nrem > 0) {
          if (tid == 0) {
            S.take = 0;
            S.rem = 0;
          }
          __syncthreads();
          filter_list(gl2, nrem, S.thr, -1.f, s_blist, &S.take, gl, &S.rem);
          __syncthreads();
          const int n2 = S.rem;
          if (n2 <= CAP_B) {
            for (int i = tid; i < n2; i += kThreads) s_blist[i] = gl[i];
            __syncthreads();
            bitonic_sort_u64(s_blist, n2);
            scan_blocks<LT, NF>(A, S, s_blist, n2, true, s_T, s_cand, s_tkd, s_tki, s_wd, s_wi, s_qh4);
          } else {
            scan_blocks<LT, NF>(A, S, gl, n2, false, s_T, s_cand, s_tkd, s_tki, s_wd, s_wi, s_qh4);
          }
        }
      }
    }
    // ---------------------------------------------------------------- output
    for (int r = tid; r < A.k; r += kThreads) {
      const bool ok = r < S.tkn;
      A.od[(int64_t)qi * A.k + r] = ok ? sqrtf(s_tkd[r]) : INFINITY;
      A.oi[(int64_t)qi * A.k + r] = ok ? A.goff + s_tki[r] : -1;
    }
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
      for (int i = 0; i < 10; ++i) tr[4 + i] = S.st[i];
      tr[14] = blockIdx.x;
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      tr[15] = smid;
    }
    __syncthreads();
  }
}

template <int LT, int NF>
static int launch_query_t(sofa_index* ix, const QArgs& A0, cudaStream_t st) {
  QArgs A = A0;
  constexpr int UB0 = 2 * LT * 256 * 4, UB1 = CAP_B * 8, UB2 = NF * 128 * 8;
  constexpr int UB = UB0 > UB1 ? (UB0 > UB2 ? UB0 : UB2) : (UB1 > UB2 ? UB1 : UB2);
  const size_t smem = NF * 128 * 4 + LT * 8 + LT * 256 * 4 + UB + CAP_C * 8 + KMAX * 8 + 8 * 8;
  auto kern = k_query<LT, NF>;
  SOFA_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0, sms = 148;
  SOFA_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem));
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ix->device);
  if (per_sm < 1) per_sm = 1;
  int grid = sms * per_sm;
  if (grid > A.q) grid = A.q;
  const int64_t need = (int64_t)grid * 2 * (ix->nb > 0 ? ix->nb : 1);
  if (ix->gscratch_ctas < need) {
    if (ix->gscratch) cudaFree(ix->gscratch);
    ix->gscratch = nullptr;
    SOFA_CK(cudaMalloc(&ix->gscratch, need * 8));
    ix->gscratch_ctas = need;
  }
  A.gscratch = ix->gscratch;
  SOFA_CK(cudaMemsetAsync(ix->qcounter, 0, sizeof(int), st));
  kern<<<grid, kThreads, smem, st>>>(A);
  SOFA_LAUNCHED();
  return SOFA_OK;
}

int launch_query(sofa_index* ix, const float* Q, int q, int k, const float* bsf_init, float* od, int64_t* oi,
                 cudaStream_t st) {
  QArgs A{};
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
  A.trace = ix->trace_on ? ix->trace : nullptr;
  for (int j = 0; j < SOFA_MAX_L; ++j) A.weights[j] = j < ix->l ? (float)ix->model.weights[j] : 0.f;
  const int nf4 = ix->len / 4;
  const int NF = nf4 <= 32 ? 1 : nf4 <= 64 ? 2 : nf4 <= 128 ? 4 : 8;
#define SOFA_Q(lt, nf) \
  if (ix->LT == lt && NF == nf) return launch_query_t<lt, nf>(ix, A, st);
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

}  // namespace sofa
