// f1: the dense path, for queries the SFA lower bound cannot prune.
//
// GEMINI filters with a lower bound and verifies with the true distance.  When a
// query's envelope filter (a6) keeps most blocks even after its lowest-LB blocks have been
// refined (high-frequency data: SURVEY SIM-3b, TLB 0.24, ~99.5% of series survive; random walks
// with sigma = 1 noise: ~15% refined), refining "every survivor" means streaming the dataset once
// PER QUERY.  Such queries are batched here instead and given a second lower bound that is cheap
// in bulk:
//
//   dot(x^, q^)  tensor-core bf16 GEMM (tcgen05.mma kind::f16, fp32 accumulate in TMEM) of the
//                z-normalised ROWS (M = 128 per tile, a bfloat16 copy written by the build's
//                transform, original row order, TMA-streamed once per query group) against the
//                z-normalised queries (N <= 256 per group, bfloat16, resident in shared memory);
//   approx d^2   = |q^|^2 + |x^|^2 - 2 dot,  |x^|^2 = n (0 for a constant row);
//   |error|     <= eps_q = 2 gamma sqrt(1.0001 n) |q^| + 2e-4 (|q^|^2 + n) + 1e-3 with
//                 gamma = 2^-7 + 2^-15 + n 2^-23 (each bf16 operand rounds by <= 2^-8 relative,
//                 products exact, fp32 accumulation bounded as a naive sum and doubled), and the
//                 slack covering |x^|^2 = n only to the float32 statistics and the refine's own
//                 float32 rounding (reading 29; pinned on CPU by tests/test_dense_bound.py,
//                 and the tensor cores' accumulation measured against it by test_gpu_dense.py);
//   LB_g = approx - eps <= d2_refine <= approx + eps = UB_g.
//
// A row is a candidate iff LB_g <= thr_q, thr_q being a proven upper bound on the query's k-th
// best: the exact k-th best of the rows the front refined, lowered during the pass by the k-th
// smallest UB_g of candidate rows (a row that could lower it is itself a candidate, so only
// candidates need tracking).  Candidates are refined EXACTLY by the same ed_warp_multi arithmetic
// as the sparse path (a8), so the dense path returns bit-identical distances.  Exactness: every
// true top-k row x* has LB_g(x*) <= d2(x*) <= true k-th <= thr_q at all times, so it is emitted.
//
// Kernels: k_dense_screen (warp-specialised tcgen05 GEMM + screening epilogue, persistent, one CTA
// per SM, cooperative launch) and k_dense_post (exact refine of the candidates, brute-force fallback
// for a query whose candidates overflowed the buffer, then the last CTA writes the outputs).
// Queries are split into groups of at most NQmax (TMEM: 2 x 256 accumulator columns; shared
// memory: the group's queries stay resident); the CTAs of different groups that stream the same
// row tiles stay within a few tiles of each other (their "twins"), so a tile read from HBM by one is
// re-read from L2 by the others.  The cooperative launch guarantees the twins are co-resident.
#include <cudaTypedefs.h>

#include <cuda_bf16.h>

#include "common.cuh"

namespace sofa {

constexpr int DM = 128;                  // rows per tile (MMA M = TMEM lanes)
constexpr int DKC = 64;                  // bf16 per K chunk = 128-byte rows (SWIZZLE_128B atom)
constexpr int DA_BYTES = DM * DKC * 2;   // 16 KB per A stage
constexpr int D_THREADS = 352;           // warp 0 TMA, warp 1 MMA + TMEM owner, warps 2..9 epilogue (2 groups),
                                         // warp 10 threshold refresher
constexpr int D_AHEAD = 8;               // row tiles a CTA may run ahead of its twins
constexpr int D_MAX_STAGES = 12;         // A ring depth cap (barrier arrays)
constexpr int D_SMEM_MAX = 232448 - 2048;  // opt-in shared memory per CTA on sm_100, less the static part
constexpr int D_MISC = 4096;             // per-query thresholds / norms + barriers

// ------------------------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  const uint32_t a = smem_u32(b);
  uint32_t ok = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
// multicast: the box lands at the same shared offset in every CTA of `mask` and completes the transaction
// bytes on the barrier at the same offset in each of them
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
// arrive (once the prior MMAs complete) on the barrier at this offset in every CTA of `mask`
__device__ __forceinline__ void tc_commit_mc(uint64_t* b, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   smem_u32(b)),
               "h"(mask)
               : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(b))
               : "memory");
}
// D[tmem] (+)= A[smem] . B[smem]^T, kind::f16 (bf16 operands, fp32 accumulate), both K-major
__device__ __forceinline__ void tc_mma_bf16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// ---- CTA-pair (cta_group::2) variants: every tcgen05 instruction of a kernel uses the same cta_group
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// the shared::cluster address of the same variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_rank(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// 2-SM TMA: the data lands in this CTA's shared memory, the transaction bytes count on the barrier at
// `bar_cluster` (the leader CTA's)
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, int x, int y, uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(bar_cluster)
      : "memory");
}
__device__ __forceinline__ void tc_commit_pair(uint64_t* b) {  // arrive on the barrier in both CTAs of the pair
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   smem_u32(b)),
               "h"((uint16_t)3)
               : "memory");
}
__device__ __forceinline__ void tc_mma_bf16_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                 uint32_t accumulate) {
  asm volatile(
      "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// shared-memory matrix descriptor: K-major, 128-byte swizzle, 8-row atoms 1024 B apart (SBO),
// LBO unused for swizzled K-major (1), version 1 (sm_100), base offset 0 (1024-aligned tiles).
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// instruction descriptor, kind::f16: D f32 (bits 4-5 = 1), A/B bf16 (bits 7-9, 10-12 = 1), both
// K-major, N >> 3 at bits 17-22, M >> 4 at bits 24-28 (cute/arch/mma_sm100_desc.hpp layout)
__device__ __forceinline__ uint32_t idesc_bf16(int n, int m = DM) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

#define TMEM_LD32(addr, r)                                                                                        \
  asm volatile(                                                                                                   \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19," \
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                                   \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),           \
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),     \
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),   \
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])    \
      : "r"(addr))

struct DenseArgs {
  int64_t n, dense_rows;
  int len, k, KC;
  int64_t n_tiles;
  int nq_max;                // queries per group (shared memory / TMEM limit of this launch)
  int smem_dyn;              // dynamic shared memory of the launch (the A ring takes what the queries leave)
  const float2* stats_orig;  // (mu, inv_sigma) per original row
  const int* qd_count;       // number of dense query slots (device)
  const float4* qparams;     // per slot: (|q^|^2, eps, -, -)
  float* thr;                // per slot: proven bound on the k-th best (atomicMin as uint)
  float* ubl;                // per slot: k smallest UB_g of candidate rows (k > 1), under ub_lock
  int* ubn;
  int* ub_lock;
  unsigned long long* cand;  // (slot << 32) | row
  int64_t cand_cap;  // split into one slice per CTA (cand_cap / gridDim.x entries each)
  int* slice_count;  // per CTA: candidates emitted (may exceed the slice: overflow)
  int streamed;      // STR mode (queries streamed with the rows; n = 1024) vs RES (queries resident)
  int pair;          // RES on CTA pairs (tcgen05 cta_group::2, M = 256; sofa_tuning.dense_pair)
  int* overflow;  // per slot flag
  int* ovf_list;
  int* ovf_count;
  int* progress;  // per CTA: row tiles whose loads are issued (zeroed per call)
  float* raw_out; // debug (sofa_dense_dots): write the raw dot products, rows x raw_ld, no screening
  int raw_ld;
  int raw_q;      // debug: number of query slots (instead of *qd_count)
  int diag;       // sofa_tuning.dense_diag (timing diagnostics; 0 in real use)
  int global_lists;  // k > 1: one UB list per query under a lock instead of per-CTA lists (sofa_tuning.dense_klist)
  float* ubsnap;     // k > 1 with per-CTA lists: their published copies, slot x cpg_cap x (k + 2) (zeroed per call)
  int cpg_cap;
  int cluster2;   // single-CTA screen launched as clusters of 2: an even number of query groups shares
                  // every row tile by TMA multicast (one L2 read feeds both CTAs of the cluster)
};

__device__ __forceinline__ float warp_min_f32(float v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v = fminf(v, __shfl_xor_sync(FULL, v, o));
  return v;
}

// shared-memory float minimum (values of either sign), rare path
__device__ __forceinline__ void smem_fmin(float* p, float v) {
  int* ip = reinterpret_cast<int*>(p);
  int old = *ip;
  while (v < __int_as_float(old)) {
    const int prev = atomicCAS(ip, old, __float_as_int(v));
    if (prev == old) break;
    old = prev;
  }
}

// Per-CTA k-smallest UB lists (k > 1): col x k floats, counts, locks, in shared memory when they fit.
struct UbLists {
  float* l;
  int* n;
  int* lock;
  float* snap0;       // nullable: this CTA's published copy of its list for query slot 0 (seqlock: seq, n, values)
  int64_t snap_slot;  // floats between consecutive slots' copies
};

// a candidate row's upper bound UB_g lowers the query's threshold: k = 1 directly; k > 1 through
// the k smallest UBs of distinct candidate rows (each row is screened once per query, by one CTA).
// s_d is this CTA's copy (thr + eps - |q^|^2); an offer that cannot lower it is skipped (every bound
// stays valid).  With per-CTA lists (L.l != nullptr) the k-th smallest UB of the rows THIS CTA
// screened is the CTA's bound (k distinct rows), pushed to the global threshold by atomicMin; no
// global lock.  Otherwise one global list per query under a spin lock.
__device__ void offer_ub(const DenseArgs& A, int slot, int col, float ub, float* s_d, float eps_minus_qn,
                         const UbLists& L) {
  if (!(ub + eps_minus_qn < *(volatile float*)s_d)) return;
  float t = INFINITY;
  if (A.k == 1) {
    t = ub;
  } else if (L.l) {
    int* lk = &L.lock[col];
    while (atomicCAS(lk, 0, 1) != 0) {
    }
    __threadfence_block();
    volatile float* l = L.l + col * A.k;
    const int n = *(volatile int*)&L.n[col];
    if (n < A.k || ub < l[n - 1]) {
      int p = n < A.k ? n : A.k - 1;
      while (p > 0 && l[p - 1] > ub) {
        l[p] = l[p - 1];
        --p;
      }
      l[p] = ub;
      const int nn = n < A.k ? n + 1 : A.k;
      *(volatile int*)&L.n[col] = nn;
      if (nn == A.k) t = l[A.k - 1];
      if (L.snap0) {  // publish the list (seqlock, this CTA is its only writer) for the union bound
        volatile int* sn = reinterpret_cast<volatile int*>(L.snap0 + (int64_t)slot * L.snap_slot);
        const int s0 = sn[0];
        sn[0] = s0 + 1;
        __threadfence();
        sn[1] = nn;
        for (int j = 0; j < nn; ++j) reinterpret_cast<volatile float*>(sn)[2 + j] = l[j];
        __threadfence();
        sn[0] = s0 + 2;
      }
    }
    __threadfence_block();
    atomicExch(lk, 0);
  } else {
    int* lk = &A.ub_lock[slot];
    while (atomicCAS(lk, 0, 1) != 0) {
    }
    __threadfence();
    volatile float* l = A.ubl + (int64_t)slot * A.k;
    const int n = *(volatile int*)&A.ubn[slot];
    if (n < A.k || ub < l[n - 1]) {
      int p = n < A.k ? n : A.k - 1;
      while (p > 0 && l[p - 1] > ub) {
        l[p] = l[p - 1];
        --p;
      }
      l[p] = ub;
      const int nn = n < A.k ? n + 1 : A.k;
      *(volatile int*)&A.ubn[slot] = nn;
      if (nn == A.k) t = l[A.k - 1];
    }
    __threadfence();
    atomicExch(lk, 0);
  }
  if (t < INFINITY) {
    atomicMin(reinterpret_cast<unsigned int*>(&A.thr[slot]), __float_as_uint(t));
    smem_fmin(s_d, t + eps_minus_qn);
  }
}

// The candidates of one 32-column chunk (rare path): m = this lane's passing columns.  One shared-memory
// atomic per warp reserves their slots in this CTA's slice of the candidate buffer; each passing (row,
// query) then offers its UB_g.
__device__ void emit_chunk(const DenseArgs& A, uint32_t m, const uint32_t (&v)[32], int c0, int q0, uint32_t row,
                           float xn, float* s_d, const float* s_qn, const float* s_eps, int* s_ccount,
                           unsigned long long* slice, int64_t slice_cap, const UbLists& L) {
  const int lane = threadIdx.x & 31;
  const int cnt = __popc(m);
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += t;
  }
  const int total = __shfl_sync(FULL, incl, 31);
  int base = 0;
  if (lane == 0 && total) base = atomicAdd(s_ccount, total);
  base = __shfl_sync(FULL, base, 0) + incl - cnt;
  while (m) {
    const int c = __ffs(m) - 1;
    m &= m - 1;
    const int col = c0 + c, slot = q0 + col;
    if (base < slice_cap) {
      slice[base] = ((unsigned long long)slot << 32) | row;
    } else if (atomicExch(&A.overflow[slot], 1) == 0) {
      A.ovf_list[atomicAdd(A.ovf_count, 1)] = slot;
    }
    ++base;
    float dot = 0.f;
#pragma unroll
    for (int u = 0; u < 32; ++u)  // select without dynamic register indexing
      if (u == c) dot = __uint_as_float(v[u]);
    const float ub = (s_qn[col] + xn - 2.f * dot) + s_eps[col];
    offer_ub(A, slot, col, ub, s_d + col, s_eps[col] - s_qn[col], L);
  }
}

// Work of CTA b: with g query groups and c = G / g CTAs per group, CTA b serves group b % g and work
// units (b / g) + j c; CTAs b >= c g idle.  "Twins": CTAs with the same b / g (same units).  A unit is
// one row tile with the group's queries resident in shared memory (RES: rows n <= 512), or two row
// tiles sharing the query chunks streamed next to them (STR: the queries do not fit, n = 1024).
// PAIR (RES only): clusters of 2 CTAs on one TPC run M = 256 MMAs (tcgen05 cta_group::2, issued by the
// leader): a unit is 256 rows, each CTA streams its 128 and holds HALF of the group's queries, so each
// SM's shared memory feeds half the query operand (the single-CTA M = 128 MMA at N = 176 needs more
// shared-memory bandwidth than the SM has, next to the TMA fills); each CTA's TMEM holds its 128 rows
// x all N columns, read by its own epilogue.
template <bool PAIR>
__global__ void __launch_bounds__(D_THREADS, 1)
    k_dense_screen(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const DenseArgs A) {
  extern __shared__ __align__(1024) unsigned char dsm_raw[];
  // 1024-aligned by pointer arithmetic on the shared array (keeps the shared address space visible to
  // the compiler: LDS, not generic loads, for the per-query vectors below)
  unsigned char* dsm = dsm_raw + ((1024u - (smem_u32(dsm_raw) & 1023u)) & 1023u);
  __shared__ uint32_t s_tmem;
  __shared__ uint64_t bars[2 * D_MAX_STAGES + 5];
  __shared__ int s_done, s_ccount;

  const int qd = A.raw_out ? A.raw_q : *A.qd_count;
  if (qd == 0) return;
  if (!A.raw_out && *reinterpret_cast<const unsigned long long*>(A.qd_count + 6) < (unsigned long long)A.dense_rows)
    return;  // batch decision: sparse (the deferred k_query launch finishes the flagged queries)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool str = !PAIR && A.streamed != 0;
  const int ng = (qd + A.nq_max - 1) / A.nq_max;               // query groups
  const int NQA = PAIR ? 32 : 16;                              // (a pair splits the columns in two halves of 16k)
  const int nq = ((qd + ng - 1) / ng + NQA - 1) / NQA * NQA;   // columns per group (MMA N), <= nq_max
  const int G = gridDim.x, b = blockIdx.x;
  const uint32_t rank = PAIR ? cluster_rank() : 0u;
  const int W = PAIR ? G / 2 : G, wb = PAIR ? b >> 1 : b;      // workers (CTAs or pairs) and this one's index
  const int cpg = W / ng;
  // (idle workers exist only with more groups than workers / group; in a cluster launch they stay for the
  // cluster barriers, with no work: twin past every unit)
  const bool idle = wb >= cpg * ng;
  if (idle && !A.cluster2) return;
  const int grp = idle ? 0 : wb % ng, twin = idle ? 0x3fffffff : wb / ng;
  // multicast (clusters of 2, an even number of groups): the cluster's CTAs serve groups 2i, 2i + 1 of the
  // same twin index, i.e. the same row tiles; each issues half of every tile's K chunks to both
  const bool mc = !PAIR && A.cluster2 && !A.raw_out && (ng % 2) == 0;
  const uint32_t crank = (!PAIR && A.cluster2) ? cluster_rank() : 0u;
  const int q0 = grp * nq, nqv = qd - q0 < nq ? qd - q0 : nq;  // valid columns of this group
  const int KC = A.KC;
  const int nqb = PAIR ? nq / 2 : nq;                          // query rows of the group held by this CTA
  const int bres = str ? 0 : KC * nqb * 128;                   // resident query bytes (RES)
  const int sbytes = str ? 2 * DA_BYTES + nq * 128 : DA_BYTES; // one ring stage: a K chunk of the unit
  // k > 1: per-CTA UB lists in shared memory if they fit next to a ring of >= 3 stages (else global)
  const int lbytes = A.k > 1 ? (nq * A.k * 4 + nq * 8 + 15) / 16 * 16 : 0;
  const bool local_lists = A.k > 1 && !A.raw_out && !A.global_lists && A.smem_dyn - 1024 - bres - D_MISC - lbytes >= 3 * sbytes;
  int S = (A.smem_dyn - 1024 - bres - D_MISC - (local_lists ? lbytes : 0)) / sbytes;  // as deep as the rest allows
  S = S > D_MAX_STAGES ? D_MAX_STAGES : S;
  unsigned char* sB = dsm;                                     // RES: KC x nqb x 128 B
  unsigned char* sA = dsm + bres;                              // S stages
  float* s_d = reinterpret_cast<float*>(sA + (size_t)S * sbytes);  // nq: thr + eps - |q^|^2
  float* s_qn = s_d + 256;                                         // nq: |q^|^2
  float* s_eps = s_qn + 256;                                       // nq: eps
  UbLists L{nullptr, nullptr, nullptr, nullptr, 0};
  // the group's list writers (CTAs, or both CTAs of each pair) and this CTA's index among them
  const int nwr = PAIR ? 2 * cpg : cpg, me = PAIR ? 2 * twin + (int)rank : twin;
  if (local_lists) {
    L.l = s_eps + 256;           // nq x k
    L.n = reinterpret_cast<int*>(L.l + nq * A.k);
    L.lock = L.n + nq;
    if (A.ubsnap && !idle && nwr <= A.cpg_cap) {
      L.snap0 = A.ubsnap + (int64_t)me * (A.k + 2);
      L.snap_slot = (int64_t)A.cpg_cap * (A.k + 2);
    }
  }
  uint64_t* full = bars;                   // [S]
  uint64_t* empty = bars + D_MAX_STAGES;   // [S]
  uint64_t* tfull = bars + 2 * D_MAX_STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* bfull = tfull + 4;
  const int64_t T = A.n_tiles;
  const int64_t U = (str || PAIR) ? (T + 1) / 2 : T;  // work units
  const int64_t slice_cap = A.cand_cap / G;
  unsigned long long* slice = A.cand + (int64_t)b * slice_cap;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], mc ? 2 : 1);  // multicast: both CTAs' MMAs release the slot
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], (PAIR ? 2 : 1) * 4);  // one arrive per warp of epilogue group s (of both CTAs)
    }
    mbar_init(bfull, 1);
    s_done = 0;
    s_ccount = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
  }
  for (int c = threadIdx.x; c < 256; c += D_THREADS) {
    float d = -INFINITY, qn = 0.f, e = 0.f;
    if (c < nqv && !A.raw_out) {
      const float4 qp = A.qparams[q0 + c];
      qn = qp.x;
      e = qp.y;
      d = *(volatile float*)&A.thr[q0 + c] + e - qn;  // +inf while fewer than k rows are known
    }
    s_d[c] = d;
    s_qn[c] = qn;
    s_eps[c] = e;
    if (L.l && c < nq) {
      L.n[c] = 0;
      L.lock[c] = 0;
    }
  }
  if (warp == 1) {
    if (PAIR) {  // both CTAs of the pair, same warp
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&s_tmem))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&s_tmem))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  if (PAIR || A.cluster2)
    cluster_sync_all();  // both CTAs' barriers initialised before any TMA / remote arrive targets them
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  // PAIR: the leader CTA's barriers, as cluster addresses (TMA transaction bytes, accumulator releases)
  const uint32_t lead_full0 = PAIR ? mapa_rank(&full[0], 0) : 0u, lead_bfull = PAIR ? mapa_rank(bfull, 0) : 0u;
  const uint32_t lead_tempty0 = PAIR ? mapa_rank(&tempty[0], 0) : 0u;

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      if (PAIR) {  // this CTA's half of the group's queries; the transaction bytes count at the leader
        if (rank == 0) mbar_expect_tx(bfull, (uint32_t)(KC * nq * 128));
        const int qh = q0 + (int)rank * nqb;
        for (int kc = 0; kc < KC; ++kc)
          for (int r = 0; r < nqb; r += 16)
            tma_load_2d_pair(sB + ((size_t)kc * nqb + r) * 128, &tmB, kc * DKC, qh + r, lead_bfull);
      } else if (!str) {  // the group's queries: every K chunk, 16 rows per box, resident for the whole pass
        mbar_expect_tx(bfull, (uint32_t)(KC * nq * 128));
        for (int kc = 0; kc < KC; ++kc)
          for (int r = 0; r < nq; r += 16) tma_load_2d(sB + ((size_t)kc * nq + r) * 128, &tmB, kc * DKC, q0 + r, bfull);
      }
      volatile int* prog = A.progress;
      int stage = 0;
      uint32_t phase = 0;
      int64_t j = 0;
      int twin_lo = 0;  // the slowest twin's progress, re-read only when this CTA would run too far ahead
      // (a multicast cluster of 2 groups has no twins outside it).  The wait is bounded: a twin that does
      // not progress for ~1 ms (not resident: another kernel holds its SM) is given up on — only L2 reuse
      // depends on it, never a result, so no CTA can wait forever on another
      bool twin_sync = !PAIR && ng > (mc ? 2 : 1) && !(A.diag & 4);
      for (int64_t u = twin; u < U; u += cpg, ++j) {
        if (twin_sync && twin_lo < j - D_AHEAD) {  // stay within D_AHEAD units of the twins
          for (int spin = 0;; ++spin) {            // (the tile is still in L2 when they read it)
            int lo = 0x7fffffff;
            for (int o = 0; o < ng; ++o) {
              const int p = prog[twin * ng + o];
              lo = p < lo ? p : lo;
            }
            twin_lo = lo;
            if (lo >= j - D_AHEAD) break;
            if (spin >= 4096) {
              twin_sync = false;
              break;
            }
            __nanosleep(256);
          }
        }
        for (int kc = 0; kc < KC; ++kc) {
          mbar_wait(&empty[stage], phase ^ 1);
          unsigned char* st = sA + (size_t)stage * sbytes;
          if (PAIR) {  // this CTA's 128 rows of the unit's 256; the leader expects both halves
            if (rank == 0) mbar_expect_tx(&full[stage], (uint32_t)(2 * sbytes));
            tma_load_2d_pair(st, &tmA, kc * DKC, (int)((2 * u + rank) * DM), lead_full0 + 8u * (uint32_t)stage);
          } else {
          mbar_expect_tx(&full[stage], (uint32_t)sbytes);
          }
          if (PAIR) {
          } else if (mc) {
            if ((uint32_t)(kc & 1) == crank) tma_load_2d_mc(st, &tmA, kc * DKC, (int)(u * DM), &full[stage], 3);
          } else if (!str) {
            tma_load_2d(st, &tmA, kc * DKC, (int)(u * DM), &full[stage]);
          } else {
            tma_load_2d(st, &tmA, kc * DKC, (int)(2 * u * DM), &full[stage]);
            tma_load_2d(st + DA_BYTES, &tmA, kc * DKC, (int)((2 * u + 1) * DM), &full[stage]);
            for (int r = 0; r < nq; r += 16) tma_load_2d(st + 2 * DA_BYTES + r * 128, &tmB, kc * DKC, q0 + r, &full[stage]);
          }
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (!PAIR) prog[b] = (int)(j + 1);
      }
      if (!PAIR) prog[b] = 0x7fffffff;  // done: never holds a twin back
      if (PAIR) *(volatile int*)&s_done = 1;  // (the peer CTA issues no MMA: its refresher stops here)
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer (one thread)
    if (lane == 0 && rank == 0) {
      const uint32_t idesc = idesc_bf16(nq, PAIR ? 2 * DM : DM);
      if (!str) mbar_wait(bfull, 0);
      tc_fence_after();
      int stage = 0;
      uint32_t phase = 0;
      int64_t j = 0;
      for (int64_t u = twin; u < U; u += cpg, ++j) {
        const int acc = str ? 0 : (int)(j & 1);
        if (PAIR) {
          mbar_wait(&tempty[acc], (uint32_t)((j >> 1) & 1) ^ 1);
        } else if (!str) {
          mbar_wait(&tempty[acc], (uint32_t)((j >> 1) & 1) ^ 1);
        } else {  // both buffers: the unit's two tiles
          mbar_wait(&tempty[0], (uint32_t)(j & 1) ^ 1);
          mbar_wait(&tempty[1], (uint32_t)(j & 1) ^ 1);
        }
        tc_fence_after();
        for (int kc = 0; kc < KC; ++kc) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + (size_t)stage * sbytes);
          if (PAIR) {  // M = 256: A rows from both CTAs, B halves from both CTAs (same shared offsets)
            const uint32_t b0 = smem_u32(sB + (size_t)kc * nqb * 128);
            const uint32_t dt = tmem + (uint32_t)(acc * 256);
#pragma unroll
            for (int kk = 0; kk < DKC / 16; ++kk)
              tc_mma_bf16_pair(dt, sdesc_sw128(a0 + 32 * kk), sdesc_sw128(b0 + 32 * kk), idesc, (kc | kk) ? 1u : 0u);
          } else if (!str) {
            const uint32_t b0 = smem_u32(sB + (size_t)kc * nq * 128);
            const uint32_t dt = tmem + (uint32_t)(acc * 256);
#pragma unroll
            for (int kk = 0; kk < DKC / 16; ++kk)  // UMMA_K = 16 bf16 = 32 bytes along the swizzled row
              tc_mma_bf16(dt, sdesc_sw128(a0 + 32 * kk), sdesc_sw128(b0 + 32 * kk), idesc, (kc | kk) ? 1u : 0u);
          } else {
            const uint32_t b0 = a0 + 2 * DA_BYTES;
#pragma unroll
            for (int kk = 0; kk < DKC / 16; ++kk) {
              tc_mma_bf16(tmem, sdesc_sw128(a0 + 32 * kk), sdesc_sw128(b0 + 32 * kk), idesc, (kc | kk) ? 1u : 0u);
              tc_mma_bf16(tmem + 256, sdesc_sw128(a0 + DA_BYTES + 32 * kk), sdesc_sw128(b0 + 32 * kk), idesc,
                          (kc | kk) ? 1u : 0u);
            }
          }
          if (PAIR)
            tc_commit_pair(&empty[stage]);
          else if (mc)
            tc_commit_mc(&empty[stage], 3);  // the slot is free once BOTH CTAs' MMAs have read it
          else
            tc_commit(&empty[stage]);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (PAIR) {
          tc_commit_pair(&tfull[acc]);
        } else if (!str) {
          tc_commit(&tfull[acc]);
        } else {
          tc_commit(&tfull[0]);
          tc_commit(&tfull[1]);
        }
      }
      *(volatile int*)&s_done = 1;  // every MMA issued: the threshold refresher may stop
    }
  } else if (warp == D_THREADS / 32 - 1) {
    // ---------------------------------------------------------------- threshold refresher
    // other CTAs' improvements of the group's thresholds (global) into this CTA's copy, off the
    // epilogue's path
    if (!A.raw_out)
      while (!*(volatile int*)&s_done) {
        for (int c = lane; c < nqv; c += 32) {
          const float nd = *(volatile float*)&A.thr[q0 + c] + s_eps[c] - s_qn[c];
          if (nd < s_d[c]) smem_fmin(s_d + c, nd);
        }
        if (L.snap0) {
          // k > 1: the union bound.  Every writer's list holds UB_g of distinct rows of its own tiles, so
          // the k-th smallest of the values read from ANY of the lists (here each writer's two smallest,
          // torn or in-progress copies skipped) bounds the query's k-th best — far tighter than one CTA's
          // own k-th.  This CTA computes it for its share of the group's columns.
          for (int c = me; c < nqv; c += nwr) {
            float vals[10];
#pragma unroll
            for (int j = 0; j < 10; ++j) vals[j] = INFINITY;
#pragma unroll
            for (int j = 0; j < 5; ++j) {
              const int t = lane + 32 * j;
              if (t >= nwr) break;
              const volatile int* sn =
                  reinterpret_cast<const volatile int*>(A.ubsnap + ((int64_t)(q0 + c) * A.cpg_cap + t) * (A.k + 2));
              const int s1 = sn[0];
              if (s1 & 1) continue;
              const int n = sn[1];
              const float v0 = n > 0 ? reinterpret_cast<const volatile float*>(sn)[2] : INFINITY;
              const float v1 = n > 1 ? reinterpret_cast<const volatile float*>(sn)[3] : INFINITY;
              if (sn[0] != s1) continue;
              vals[2 * j] = v0;
              vals[2 * j + 1] = v1;
            }
            float v = -INFINITY;
            int cnt = 0;
            while (cnt < A.k) {  // the k-th smallest with multiplicity
              float m = INFINITY;
#pragma unroll
              for (int j = 0; j < 10; ++j) m = vals[j] > v ? fminf(m, vals[j]) : m;
              m = warp_min_f32(m);
              if (!(m < INFINITY)) break;
              int e = 0;
#pragma unroll
              for (int j = 0; j < 10; ++j) e += vals[j] == m;
              cnt += __reduce_add_sync(FULL, e);
              v = m;
            }
            if (cnt >= A.k && lane == 0) {
              atomicMin(reinterpret_cast<unsigned int*>(&A.thr[q0 + c]), __float_as_uint(v));
              smem_fmin(s_d + c, v + s_eps[c] - s_qn[c]);
            }
          }
        }
        __nanosleep(1000);
      }
  } else {
    // ---------------------------------------------------------------- epilogue (2 groups x 4 warps)
    // Group g = (warp - 2) / 4 owns accumulator buffer g.  RES: this CTA's tiles j = g, g + 2, ...: while
    // one group screens its tile the MMA fills the other buffer and the other group screens the previous
    // tile, so a group has two MMA tile-times per tile.  STR: the two tiles of each unit.  Warp w reads
    // TMEM lane quarter w % 4 (its 32 rows of the tile) and every 32-column chunk.  Per element:
    // val = 2 dot + (thr + eps - |q^|^2); the row is a candidate for that query iff val >= |x^|^2
    // (LB_g <= thr).
    const int qtr = warp & 3, grp_e = (warp - 2) >> 2;
    const int r = qtr * 32 + lane;
    const int nch = (nq + 31) / 32;  // 32-column chunks (columns past the group's queries have s_d = -inf)
    const float nlen = (float)A.len;
    // the i-th tile of this group
    auto exists = [&](int64_t i) -> bool { return str ? twin + i * cpg < U : twin + (2 * i + grp_e) * cpg < U; };
    auto tile_of = [&](int64_t i) -> int64_t {
      if (PAIR) return 2 * (twin + (2 * i + grp_e) * cpg) + rank;  // this CTA's half of the unit
      return str ? 2 * (twin + i * cpg) + grp_e : twin + (2 * i + grp_e) * cpg;
    };
    // the row's 1/sigma, loaded a tile (of this group) ahead; |x^|^2 = n, 0 for a constant row, NaN past N
    auto sig_load = [&](int64_t i) -> float {
      const int64_t tt = tile_of(i), rr = tt * DM + r;
      if (!exists(i) || rr >= A.n || tt >= T) return __int_as_float(0x7fffffff);
      if (A.raw_out) return 1.f;
      return A.stats_orig[rr].y;
    };
    auto xnorm_of = [&](float sig) -> float { return isnan(sig) ? sig : (sig > 0.f ? nlen : 0.f); };
    const int acc = grp_e;
    // the rows' 1/sigma, loaded 4 group tiles ahead: one load per row per tile, but queued behind the TMA
    // stream it took longer than a tile (ncu: 44% of the kernel's stall samples on its use with 1 ahead)
    float sig_q0 = sig_load(0), sig_q1 = sig_load(1), sig_q2 = sig_load(2), sig_q3 = sig_load(3);
    for (int64_t i = 0; exists(i); ++i) {
      const uint32_t aph = (uint32_t)(i & 1);
      const int64_t row = tile_of(i) * DM + r;
      const float sig = sig_q0;
      sig_q0 = sig_q1;
      sig_q1 = sig_q2;
      sig_q2 = sig_q3;
      sig_q3 = sig_load(i + 4);
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const float xn = xnorm_of(sig);
      if (A.diag & 2) {  // timing diagnostic: release the buffer unread
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (PAIR)
            mbar_arrive_cluster(lead_tempty0 + 8u * (uint32_t)acc);
          else
            mbar_arrive(&tempty[acc]);
        }
        continue;
      }
      const uint32_t tbase = tmem + ((uint32_t)(qtr * 32) << 16) + (uint32_t)(acc * 256);
      // screen 32 columns held in v (registers): val = 2 dot + (thr + eps - |q^|^2) >= |x^|^2 ?
      auto screen = [&](const uint32_t (&v)[32], int c0) {
        if (A.diag & 1) return;  // timing diagnostic: TMEM loads only
        if (A.raw_out) {
          if (row < A.n)
            for (int c = 0; c < 32; ++c)
              if (c0 + c < nqv) A.raw_out[row * A.raw_ld + q0 + c0 + c] = __uint_as_float(v[c]);
          return;
        }
        float vmax = -INFINITY;
#pragma unroll
        for (int c = 0; c < 32; c += 4) {
          const float4 d4 = *reinterpret_cast<const float4*>(s_d + c0 + c);
          const float a0 = fmaf(2.f, __uint_as_float(v[c + 0]), d4.x);
          const float a1 = fmaf(2.f, __uint_as_float(v[c + 1]), d4.y);
          const float a2 = fmaf(2.f, __uint_as_float(v[c + 2]), d4.z);
          const float a3 = fmaf(2.f, __uint_as_float(v[c + 3]), d4.w);
          vmax = fmaxf(vmax, fmaxf(fmaxf(a0, a1), fmaxf(a2, a3)));
        }
        if (!(A.diag & 8) && __any_sync(FULL, vmax >= xn)) {  // rare: this chunk has candidates
          uint32_t m = 0;
#pragma unroll
          for (int c = 0; c < 32; ++c) m |= (fmaf(2.f, __uint_as_float(v[c]), s_d[c0 + c]) >= xn ? 1u : 0u) << c;
          emit_chunk(A, m, v, c0, q0, (uint32_t)row, xn, s_d, s_qn, s_eps, &s_ccount, slice, slice_cap, L);
        }
      };
      // TMEM loads double-buffered: the next chunk is in flight while this one is screened
      uint32_t va[32], vb[32];
      TMEM_LD32(tbase, va);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int ch = 0; ch < nch; ch += 2) {
        if (ch + 1 < nch) TMEM_LD32(tbase + (ch + 1) * 32, vb);
        screen(va, ch * 32);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (ch + 1 >= nch) break;
        if (ch + 2 < nch) TMEM_LD32(tbase + (ch + 2) * 32, va);
        screen(vb, (ch + 1) * 32);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      }
      // the warp's TMEM reads are complete (tcgen05.wait::ld is warp-wide): one arrive per warp, a remote
      // one (DSMEM) for the peer CTA of a pair — the leader's MMA waits on both CTAs
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (PAIR)
          mbar_arrive_cluster(lead_tempty0 + 8u * (uint32_t)acc);
        else
          mbar_arrive(&tempty[acc]);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && A.slice_count) A.slice_count[b] = s_ccount;  // candidates of this CTA (may exceed its slice)
  if (PAIR || A.cluster2) cluster_sync_all();  // neither CTA leaves while its peer may still read / multicast into its shared memory
  if (warp == 1) {
    tc_fence_after();
    if (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// ------------------------------------------------------------------------------------------------
// exact refine of the dense candidates (same arithmetic as a8), brute-force fallback for slots whose
// candidates overflowed, then the last CTA writes the dense queries' results.
struct DensePost {
  const float* series;
  const float2* stats_orig;
  int len, k;
  int64_t n, goff, dense_rows;
  const int* qd_count;
  const float* qhat;  // slot x len
  const int* qidx;    // slot -> query index
  const float* binit; // slot -> caller bound (inf if none)
  float* bsf;         // slot -> exact k-th best (or bound)
  float* thr;         // slot -> screening threshold
  float* tkd;         // slot x k
  int* tki;           // slot x k (local row)
  int* tkn;
  int* lock;
  unsigned long long* key1;  // slot: k = 1 best key
  const unsigned long long* cand;
  int64_t cand_cap;
  const int* slice_count;  // per screen CTA
  int nslices;             // screen CTAs (slices of cand_cap / nslices entries)
  const int* overflow;
  const int* ovf_list;
  const int* ovf_count;
  unsigned int* done;
  float* od;
  int64_t* oi;
  unsigned long long* dstats;  // nullable: [19] dense queries, [20] candidates, [21] refined
};

__device__ void g_topk_insert(const DensePost& P, int slot, float d, int i) {
  const int k = P.k;
  if (d > P.binit[slot]) return;
  while (atomicCAS(&P.lock[slot], 0, 1) != 0) {
  }
  __threadfence();
  volatile float* td = P.tkd + (int64_t)slot * k;
  volatile int* ti = P.tki + (int64_t)slot * k;
  const int n = *(volatile int*)&P.tkn[slot];
  bool dup = false;
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
    *(volatile int*)&P.tkn[slot] = nn;
    if (nn == k) {
      const float b = fminf(P.binit[slot], td[k - 1]);
      *(volatile float*)&P.bsf[slot] = b;
      atomicMin(reinterpret_cast<unsigned int*>(&P.thr[slot]), __float_as_uint(b));
    }
  }
  __threadfence();
  atomicExch(&P.lock[slot], 0);
}

template <int NF>
__global__ void __launch_bounds__(kThreads) k_dense_post(const DensePost P) {
  const int qd = *P.qd_count;
  if (qd == 0 || *reinterpret_cast<const unsigned long long*>(P.qd_count + 6) < (unsigned long long)P.dense_rows)
    return;
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * kThreads + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * kThreads) >> 5;
  const int nf4 = P.len >> 2;
  // the screen CTAs' slices, back to back: prefix of the stored counts
  __shared__ long long s_pre[1025];
  const int64_t slice_cap = P.cand_cap / P.nslices;
  if (threadIdx.x == 0) {
    long long acc = 0, raw = 0;
    for (int i = 0; i < P.nslices; ++i) {
      s_pre[i] = acc;
      const long long c = P.slice_count[i];
      raw += c;
      acc += c < slice_cap ? c : slice_cap;
    }
    s_pre[P.nslices] = acc;
    s_pre[1024] = raw;
  }
  __syncthreads();
  const int64_t nc_raw = s_pre[1024];
  const int64_t nc = s_pre[P.nslices];
  const int nov = *P.ovf_count;
  const int64_t total = nc + (int64_t)nov * P.n;
  unsigned int n_ref = 0;
  for (int64_t u = gw; u < total; u += nw) {
    int slot;
    int64_t row;
    if (u < nc) {
      int lo = 0, hi = P.nslices;  // the slice holding entry u: s_pre[lo] <= u < s_pre[lo + 1]
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (s_pre[mid] <= u) lo = mid; else hi = mid;
      }
      const unsigned long long e = P.cand[lo * slice_cap + (u - s_pre[lo])];
      slot = (int)(e >> 32);
      row = (int64_t)(uint32_t)e;
      if (P.overflow[slot]) continue;  // the fallback below rescans that slot completely
    } else {
      slot = P.ovf_list[(u - nc) / P.n];
      row = (u - nc) % P.n;
    }
    // abandon / insertion bound: the exact k-th best so far, and the screen's final threshold (a proven
    // bound on the true k-th best: no top-k row lies above it)
    float bsf = 0.f;
    if (lane == 0) bsf = fminf(*(volatile float*)&P.bsf[slot], *(volatile float*)&P.thr[slot]);
    bsf = __shfl_sync(FULL, bsf, 0);
    const float* rows[1] = {P.series + row * P.len};
    const float2 st[1] = {P.stats_orig[row]};
    const bool on[1] = {true};
    float d2[1];
    bool ab[1];
    ed_warp_multi<NF, 1>(rows, st, on, reinterpret_cast<const float4*>(P.qhat + (int64_t)slot * P.len), nf4, bsf, d2,
                         ab);
    ++n_ref;
    if (lane == 0 && !ab[0]) {
      if (P.k == 1) {  // lock-free: the minimum of (d^2 bits, row) keys is the (distance, index) minimum
        if (d2[0] <= P.binit[slot]) {
          atomicMin(&P.key1[slot], ((unsigned long long)__float_as_uint(d2[0]) << 32) | (uint32_t)row);
          atomicMin(reinterpret_cast<unsigned int*>(&P.bsf[slot]), __float_as_uint(d2[0]));  // abandon bound
        }
      } else if (d2[0] <= bsf) {
        g_topk_insert(P, slot, d2[0], (int)row);
      }
    }
  }
  if (P.dstats && lane == 0 && n_ref) atomicAdd(&P.dstats[21], (unsigned long long)n_ref);
  // last CTA out writes the dense queries' results
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(P.done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int slot = threadIdx.x; slot < qd; slot += kThreads) {
    const int qi = P.qidx[slot];
    if (P.k == 1) {
      const unsigned long long key = *(volatile unsigned long long*)&P.key1[slot];
      P.tkn[slot] = key != ~0ull;
      if (key != ~0ull) {
        P.tkd[slot] = __uint_as_float((uint32_t)(key >> 32));
        P.tki[slot] = (int)(uint32_t)key;
      }
    }
    write_topk(P.tkd + (int64_t)slot * P.k, P.tki + (int64_t)slot * P.k, *(volatile int*)&P.tkn[slot], P.k, P.goff,
               P.od + (int64_t)qi * P.k, P.oi + (int64_t)qi * P.k);
  }
  if (threadIdx.x == 0 && P.dstats) {
    atomicAdd(&P.dstats[19], (unsigned long long)qd);
    atomicAdd(&P.dstats[20], (unsigned long long)nc_raw);
  }
}

// ------------------------------------------------------------------------------------------------ host
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static std::atomic<PFN_cuTensorMapEncodeTiled_v12000> fn{nullptr};
  PFN_cuTensorMapEncodeTiled_v12000 f = fn.load();
  if (!f) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess) {
      f = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
      fn.store(f);
    }
  }
  return f;
}

// rows x len bfloat16, row stride ld elements (ld % 8 == 0), box = 64 bf16 (128 B, swizzled) x box_rows;
// elements past len / rows read as zero
static int make_tmap_bf16(CUtensorMap* m, const __nv_bfloat16* base, int64_t rows, int len, int ld, int box_rows) {
  auto enc = encode_fn();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return SOFA_ECUDA;
  }
  cuuint64_t dims[2] = {(cuuint64_t)len, (cuuint64_t)(rows > 0 ? rows : 1)};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {(cuuint32_t)DKC, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<__nv_bfloat16*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return SOFA_ECUDA;
  }
  return SOFA_OK;
}

// launch geometry of the screen for row length `len`: the queries per group that fit next to an A ring
// of at least 4 stages (multiple of 16, <= 256 for the 2 x 256 TMEM accumulator columns); the kernel
// then deepens the ring into whatever its group's queries leave free (up to D_MAX_STAGES)
static void dense_geometry(int len, bool pair, int& nq_max, int& streamed) {
  const int KC = (len + DKC - 1) / DKC;
  const int avail = D_SMEM_MAX - 1024 - 4 * DA_BYTES - D_MISC;
  const int nq = pair ? avail / (KC * 64) / 32 * 32   // a CTA of a pair holds half of the group's queries
                      : avail / (KC * 128) / 16 * 16;
  if (nq >= 128) {  // RES: queries resident next to a ring of >= 4 row-tile stages
    nq_max = nq > 256 ? 256 : nq;
    streamed = 0;
  } else {          // STR: 256 queries per group, streamed with 2 row tiles per stage (3 x 64 KB stages)
    nq_max = 256;
    streamed = 1;
  }
}

static int launch_screen(sofa_index* ix, const CUtensorMap& tmA, const CUtensorMap& tmB, const DenseArgs& A,
                         size_t smem, cudaStream_t st, int* grid_out = nullptr) {
  static std::atomic<uint32_t> attr_set{0};  // per device: the smem attributes are set once
  const uint32_t bit = 1u << (ix->device & 31);
  if (!(attr_set.load() & bit)) {
    SOFA_CK(cudaFuncSetAttribute(k_dense_screen<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, D_SMEM_MAX));
    SOFA_CK(cudaFuncSetAttribute(k_dense_screen<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, D_SMEM_MAX));
    attr_set.fetch_or(bit);
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(ix->sms & ~1);
  cfg.blockDim = dim3(D_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (A.pair) {  // RES on CTA pairs (clusters of 2 on one TPC); no CTA waits on another pair
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    if (grid_out) *grid_out = (int)cfg.gridDim.x;
    SOFA_CK(cudaLaunchKernelEx(&cfg, k_dense_screen<true>, tmA, tmB, A));
  } else if (A.cluster2) {  // clusters of 2 (TMA multicast when the groups pair up); as many clusters as
    // can be resident at once (an SM left over in a GPC stays idle rather than running a second wave)
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    if (ix->dense_clusters <= 0) {
      int nc = 0;
      cfg.gridDim = dim3(ix->sms & ~1);
      if (cudaOccupancyMaxActiveClusters(&nc, k_dense_screen<false>, &cfg) != cudaSuccess || nc < 1) {
        cudaGetLastError();
        nc = ix->sms / 2;
      }
      ix->dense_clusters = nc < ix->sms / 2 ? nc : ix->sms / 2;
    }
    cfg.gridDim = dim3(2 * ix->dense_clusters);
    if (grid_out) *grid_out = (int)cfg.gridDim.x;
    SOFA_CK(cudaLaunchKernelEx(&cfg, k_dense_screen<false>, tmA, tmB, A));
  } else {  // cooperative, every CTA resident at once (the twins wait on each other's progress)
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    if (grid_out) *grid_out = (int)cfg.gridDim.x;
    SOFA_CK(cudaLaunchKernelEx(&cfg, k_dense_screen<false>, tmA, tmB, A));
  }
  SOFA_LAUNCHED();
  return SOFA_OK;
}

static void fill_screen_args(sofa_index* ix, int k, DenseArgs& A) {
  DenseScratch& D = ix->dense;
  A.n = ix->n;
  A.dense_rows = dense_batch_rows(ix);
  A.len = ix->len;
  A.k = k;
  A.KC = (ix->len + DKC - 1) / DKC;
  A.n_tiles = (ix->n + DM - 1) / DM;
  dense_geometry(ix->len, ix->tune.dense_pair != 0, A.nq_max, A.streamed);
  A.pair = !A.streamed && ix->tune.dense_pair != 0;
  A.cluster2 = !A.pair && ix->tune.dense_mcast != 0;
  A.global_lists = ix->tune.dense_klist == 1;
  A.smem_dyn = D_SMEM_MAX;
  A.stats_orig = ix->stats_orig;
  A.qd_count = D.counters;
  A.qparams = D.qparams;
  A.thr = D.thr;
  A.ubl = D.ubl;
  A.ubsnap = k > 1 ? D.ubsnap : nullptr;
  A.cpg_cap = ix->sms;
  A.ubn = D.ubn;
  A.ub_lock = D.ub_lock;
  A.cand = D.cand;
  A.cand_cap = D.cand_cap;
  A.slice_count = D.counters + 64 + 1024;
  A.overflow = D.overflow;
  A.ovf_list = D.ovf_list;
  A.ovf_count = D.counters + 1;
  A.progress = D.counters + 64;
  A.diag = ix->tune.dense_diag;
}

int launch_dense(sofa_index* ix, int q, int k, float* od, int64_t* oi, bool stats, cudaStream_t st,
                 cudaEvent_t after_screen) {
  DenseScratch& D = ix->dense;
  int rc;
  if (D.tmap_q_rows != q) {  // tensor maps are encoded once per buffer (not on every call)
    if ((rc = make_tmap_bf16(reinterpret_cast<CUtensorMap*>(D.tmap_q), D.qb16, q, ix->len, ix->xb_ld, 16))) return rc;
    if ((rc = make_tmap_bf16(reinterpret_cast<CUtensorMap*>(D.tmap_x), ix->xb16, ix->n, ix->len, ix->xb_ld, DM)))
      return rc;
    D.tmap_q_rows = q;
  }
  DenseArgs A{};
  fill_screen_args(ix, k, A);
  if (A.ubsnap) SOFA_CK(cudaMemsetAsync(A.ubsnap, 0, (size_t)q * ix->sms * (k + 2) * 4, st));
  int sgrid = ix->sms & ~1;
  if ((rc = launch_screen(ix, *reinterpret_cast<const CUtensorMap*>(D.tmap_x),
                          *reinterpret_cast<const CUtensorMap*>(D.tmap_q), A, D_SMEM_MAX,
                          st, &sgrid)))
    return rc;
  if (after_screen) cudaEventRecord(after_screen, st);

  DensePost P{};
  P.series = ix->series;
  P.stats_orig = ix->stats_orig;
  P.len = ix->len;
  P.k = k;
  P.n = ix->n;
  P.goff = ix->global_offset;
  P.dense_rows = dense_batch_rows(ix);
  P.qd_count = D.counters;
  P.qhat = D.qhat;
  P.qidx = D.qidx;
  P.binit = D.binit;
  P.bsf = D.bsf;
  P.thr = D.thr;
  P.tkd = D.tkd;
  P.tki = D.tki;
  P.tkn = D.tkn;
  P.key1 = D.key1;
  P.lock = D.lock;
  P.cand = D.cand;
  P.cand_cap = D.cand_cap;
  P.slice_count = A.slice_count;
  P.nslices = sgrid;  // the screen's grid (its CTAs' candidate slices)
  P.overflow = D.overflow;
  P.ovf_list = D.ovf_list;
  P.ovf_count = D.counters + 1;
  P.done = reinterpret_cast<unsigned int*>(D.counters + 4);
  P.od = od;
  P.oi = oi;
  P.dstats = stats ? ix->dstats : nullptr;
  const int nf4 = ix->len / 4;
  const int grid = ix->sms * 4;
  if (nf4 <= 32)
    k_dense_post<1><<<grid, kThreads, 0, st>>>(P);
  else if (nf4 <= 64)
    k_dense_post<2><<<grid, kThreads, 0, st>>>(P);
  else if (nf4 <= 128)
    k_dense_post<4><<<grid, kThreads, 0, st>>>(P);
  else
    k_dense_post<8><<<grid, kThreads, 0, st>>>(P);
  SOFA_LAUNCHED();
  return SOFA_OK;
}

__global__ void k_to_bf16(const float* __restrict__ x, int64_t rows, int len, int ld, __nv_bfloat16* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows * ld; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / ld;
    const int c = (int)(i % ld);
    out[i] = __float2bfloat16_rn(c < len ? x[r * len + c] : 0.f);
  }
}

// debug / verification entry (sofa_dense_dots): the screen's tensor-core dot products of bf16(rows)
// and bf16(queries) (round to nearest), no screening, written as rows x q float32
int dense_dots(const float* rows, int64_t m, int len, const float* queries, int q, float* out, cudaStream_t st) {
  sofa_index tmp;
  cudaGetDevice(&tmp.device);
  cudaDeviceGetAttribute(&tmp.sms, cudaDevAttrMultiProcessorCount, tmp.device);
  tmp.n = m;
  tmp.len = len;
  const int ld = (len + 7) / 8 * 8;
  __nv_bfloat16 *xb = nullptr, *qb = nullptr;
  int* prog = nullptr;
  SOFA_CK(cudaMalloc(&xb, (size_t)m * ld * 2));
  SOFA_CK(cudaMalloc(&qb, (size_t)q * ld * 2));
  SOFA_CK(cudaMalloc(&prog, 1024 * 4));
  SOFA_CK(cudaMemsetAsync(prog, 0, 1024 * 4, st));
  k_to_bf16<<<1024, 256, 0, st>>>(rows, m, len, ld, xb);
  k_to_bf16<<<256, 256, 0, st>>>(queries, q, len, ld, qb);
  g_launches.fetch_add(2);
  alignas(64) CUtensorMap ta, tb;
  int rc = make_tmap_bf16(&ta, xb, m, len, ld, DM);
  if (!rc) rc = make_tmap_bf16(&tb, qb, q, len, ld, 16);
  if (!rc) {
    DenseArgs A{};
    A.n = m;
    A.len = len;
    A.k = 1;
    A.KC = (len + DKC - 1) / DKC;
    A.n_tiles = (m + DM - 1) / DM;
    dense_geometry(len, false, A.nq_max, A.streamed);
    A.smem_dyn = D_SMEM_MAX;
    A.progress = prog;
    A.raw_out = out;
    A.raw_ld = q;
    A.raw_q = q;
    rc = launch_screen(&tmp, ta, tb, A, D_SMEM_MAX, st);
  }
  cudaStreamSynchronize(st);
  cudaFree(xb);
  cudaFree(qb);
  cudaFree(prog);
  return rc;
}

// scratch for q queries at k (grown on demand); counters: [0] dense slots, [1] overflow slots,
// [4] done CTAs, [6..7] estimated refines; [64..] per-CTA progress; [64 + 1024..] per-CTA candidates.
int ensure_dense_scratch(sofa_index* ix, int q, int k) {
  DenseScratch& D = ix->dense;
  if (D.q_cap >= q && D.k_cap >= k && D.len == ix->len) return SOFA_OK;
  free_dense_scratch(ix);
  D.tmap_q_rows = -1;
  D.q_cap = q;
  D.k_cap = k;
  D.len = ix->len;
  D.cand_cap = ix->tune.dense_cand_cap > 0 ? ix->tune.dense_cand_cap : (int64_t)16 << 20;
  SOFA_CK(cudaMalloc(&D.qhat, (size_t)q * ix->len * 4));
  SOFA_CK(cudaMalloc(&D.qb16, (size_t)q * ix->xb_ld * 2));
  SOFA_CK(cudaMalloc(&D.qparams, (size_t)q * 16));
  SOFA_CK(cudaMalloc(&D.qidx, (size_t)q * 4));
  SOFA_CK(cudaMalloc(&D.binit, (size_t)q * 4));
  SOFA_CK(cudaMalloc(&D.bsf, (size_t)q * 4));
  SOFA_CK(cudaMalloc(&D.thr, (size_t)q * 4));
  SOFA_CK(cudaMalloc(&D.tkd, (size_t)q * k * 4));
  SOFA_CK(cudaMalloc(&D.tki, (size_t)q * k * 4));
  SOFA_CK(cudaMalloc(&D.tkn, (size_t)q * 4));
  SOFA_CK(cudaMalloc(&D.key1, (size_t)q * 8));
  SOFA_CK(cudaMalloc(&D.lock, (size_t)q * 4));
  SOFA_CK(cudaMalloc(&D.ubl, (size_t)q * k * 4));
  if (k > 1) SOFA_CK(cudaMalloc(&D.ubsnap, (size_t)q * ix->sms * (k + 2) * 4));
  SOFA_CK(cudaMalloc(&D.ubn, (size_t)q * 4));
  SOFA_CK(cudaMalloc(&D.ub_lock, (size_t)q * 4));
  SOFA_CK(cudaMalloc(&D.overflow, (size_t)q * 4));
  SOFA_CK(cudaMalloc(&D.ovf_list, (size_t)q * 4));
  SOFA_CK(cudaMalloc(&D.cand, (size_t)D.cand_cap * 8));
  SOFA_CK(cudaMalloc(&D.counters, 64 * 4 + 2048 * 4));  // counters, per-CTA progress, per-CTA candidate counts
  return SOFA_OK;
}

void free_dense_scratch(sofa_index* ix) {
  DenseScratch& D = ix->dense;
  void* ps[] = {D.qhat, D.qb16, D.qparams, D.qidx, D.binit, D.bsf, D.thr, D.tkd, D.tki, D.tkn, D.key1, D.lock, D.ubl, D.ubsnap,
                D.ubn, D.ub_lock, D.overflow, D.ovf_list, D.cand, D.counters};
  for (void* p : ps)
    if (p) cudaFree(p);
  D = DenseScratch{};
}

}  // namespace sofa
