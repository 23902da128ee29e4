// f1: the dense path, for queries the SFA lower bound cannot prune.
//
// GEMINI filters with a lower bound and verifies with the true distance.  When a
// query's envelope filter (a6) keeps most blocks even after its lowest-LB blocks have been
// refined (high-frequency data: SURVEY SIM-3b, TLB 0.24, ~99.5% of series survive), refining
// "every survivor" means streaming the whole dataset once PER QUERY.  Such queries are batched
// here instead and given a second lower bound that is cheap in bulk:
//
//   dot(q^, x)   tensor-core TF32 GEMM (tcgen05.mma kind::tf32, fp32 accumulate in TMEM) of the
//                z-normalised queries (M = 128 per tile) against the RAW float32 rows (N = 256
//                per tile), both TMA-loaded straight from HBM (no conversion pass);
//   x^.q^        = inv_sigma * (dot - mu * sum(q^))                  (z-norm on the fly, a1)
//   approx d^2   = |q^|^2 + |x^|^2 - 2 x^.q^
//   |error|     <= eps = 2 gamma |q^| inv_sigma |x| + r  (TF32 operand truncation 2^-10 each,
//                 fp32 accumulation, and r = slack for the refine's own float32 rounding)
//   LB_g = approx - eps <= exact d^2 <= approx + eps = UB_g.
//
// A row is a candidate iff LB_g <= thr_q, where thr_q is the smallest proven upper bound on the
// query's k-th best distance: the exact k-th best so far (seed block, refined candidates), or the
// k-th smallest UB_g a thread has seen (k distinct rows), shared across CTAs by atomicMin.
// Candidates are then refined EXACTLY by the same ed_warp_multi arithmetic as the sparse path (a8),
// so the dense path returns bit-identical distances.  Exactness: every true top-k row x* has
// LB_g(x*) <= d^2(x*) <= true k-th <= thr_q at all times, so it is always emitted.
//
// Kernels: k_dense_screen (warp-specialised tcgen05 GEMM + screening epilogue, persistent, one
// CTA per SM) and k_dense_post (exact refine of the candidates, brute-force fallback for a query
// whose candidates overflowed the buffer, then the last CTA writes the dense queries' outputs).
#include <cudaTypedefs.h>

#include <cstdlib>

#include "common.cuh"

namespace sofa {

constexpr int DM = 128;                 // queries per tile  (MMA M = TMEM lanes)
constexpr int DN = 256;                 // series per tile   (MMA N = accumulator columns)
constexpr int DKC = 32;                 // fp32 per K chunk = 128-byte rows (SWIZZLE_128B atom)
constexpr int DSTAGES = 4;              // TMA -> MMA pipeline depth
constexpr int DA_BYTES = DM * DKC * 4;  // 16 KB
constexpr int DB_BYTES = DN * DKC * 4;  // 32 KB
constexpr int D_THREADS = 320;          // warp 0 TMA, warp 1 MMA + TMEM owner, warps 2..9 epilogue
constexpr int D_UBK = SOFA_MAX_K;       // k-th-smallest UB tracking (local memory; updates are rare)
constexpr int D_AHEAD_CHUNKS = 64;      // K-chunks a CTA may run ahead of the others reading its series tiles
constexpr size_t D_SMEM = 1024 + DSTAGES * (DA_BYTES + DB_BYTES) + 2 * DN * 8 + 64 + 256;

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
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(b))
               : "memory");
}
// D[tmem] (+)= A[smem] . B[smem]^T, kind::tf32, both operands K-major
__device__ __forceinline__ void tc_mma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p; }" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// shared-memory matrix descriptor: K-major, 128-byte swizzle, 8-row atoms 1024 B apart (SBO),
// LBO unused for swizzled K-major (1), version 1 (sm_100), base offset 0 (1024-aligned tiles).
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// instruction descriptor: D f32 (bits 4-5 = 1), A/B tf32 (bits 7-9, 10-12 = 2), K-major both,
// N >> 3 at bits 17-22, M >> 4 at bits 24-28.
constexpr uint32_t kIdescTF32 =
    (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(DN >> 3) << 17) | ((uint32_t)(DM >> 4) << 24);

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
  const float2* stats_orig;  // (mu, inv_sigma) per original row
  const int* qd_count;       // number of dense query slots (device)
  const float4* qparams;     // per slot: (|q^|^2, sum q^, 2 gamma |q^|, 2e-4 |q^|^2 + 1e-3)
  float* thr;                // per slot: screening threshold (>= true k-th best), atomicMin as uint
  unsigned long long* cand;  // (slot << 32) | row
  int64_t cand_cap;
  unsigned long long* cand_count;
  int* overflow;  // per slot flag
  int* ovf_list;
  int* ovf_count;
  int* progress;  // per CTA: items whose loads are issued (zeroed per call)
};

__device__ __forceinline__ void emit_candidate(const DenseArgs& A, bool pass, int slot, uint32_t row) {
  const unsigned m = __ballot_sync(FULL, pass);
  if (!m) return;
  const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(A.cand_count, (unsigned long long)__popc(m));
  base = __shfl_sync(FULL, base, leader);
  if (pass) {
    const unsigned long long pos = base + __popc(m & ((1u << lane) - 1u));
    if (pos < (unsigned long long)A.cand_cap) {
      A.cand[pos] = ((unsigned long long)slot << 32) | row;
    } else if (atomicExch(&A.overflow[slot], 1) == 0) {
      A.ovf_list[atomicAdd(A.ovf_count, 1)] = slot;
    }
  }
}

// k-th-smallest insertion for k > 1 (rare after the item's first k rows; kept out of line so the
// unrolled element loop stays small)
__device__ __noinline__ void ub_insert(float* ubl, int& nub, float& ubk, int kk, float ap) {
  int p = nub < kk ? nub : kk - 1;
  while (p > 0 && ubl[p - 1] > ap) {
    ubl[p] = ubl[p - 1];
    --p;
  }
  ubl[p] = ap;
  if (nub < kk) ++nub;
  if (nub == kk) ubk = ubl[kk - 1];
}

// The j-th item (query tile m, series tile t) of this CTA.  When the grid holds at least one CTA
// per query tile, CTA b serves tile m = b % mt only (so per-query state persists across its items)
// and the CTAs sharing a series tile t run together (its rows are read from HBM once, then L2).
__device__ __forceinline__ bool dense_item(int64_t j, int64_t mt, int64_t n_tiles, int& m, int64_t& t) {
  const int64_t G = gridDim.x, b = blockIdx.x;
  if (mt <= G) {
    const int64_t per = G / mt;
    if (b >= per * mt) return false;
    m = (int)(b % mt);
    t = b / mt + j * per;
    return t < n_tiles;
  }
  const int64_t it = b + j * G;
  m = (int)(it % mt);
  t = it / mt;
  return t < n_tiles;
}

template <bool KONE>
__global__ void __launch_bounds__(D_THREADS, 1)
    k_dense_screen(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmX, const DenseArgs A) {
  extern __shared__ __align__(1024) unsigned char dsm_raw[];
  unsigned char* dsm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(dsm_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sA = dsm;
  unsigned char* sB = dsm + DSTAGES * DA_BYTES;
  float2* s_ser2 = reinterpret_cast<float2*>(sB + DSTAGES * DB_BYTES);  // [2][DN]
  float* s_tmax = reinterpret_cast<float*>(s_ser2 + 2 * DN);              // [2][4]
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_tmax + 8);
  uint64_t* full = bars;                    // [DSTAGES]
  uint64_t* empty = bars + DSTAGES;         // [DSTAGES]
  uint64_t* tfull = bars + 2 * DSTAGES;     // [2]
  uint64_t* tempty = bars + 2 * DSTAGES + 2;  // [2]
  __shared__ uint32_t s_tmem;

  const int qd = *A.qd_count;
  if (qd == 0 || *reinterpret_cast<const unsigned long long*>(A.qd_count + 6) < (unsigned long long)A.dense_rows)
    return;  // batch decision: sparse (the deferred k_query launch finishes the flagged queries)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t mt = (qd + DM - 1) / DM;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < DSTAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 8 * 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmQ) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmX) : "memory");
    for (int i = 0; i < 8; ++i) s_tmax[i] = 0.f;
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&s_tmem))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int m;
      int64_t t;
      // the CTAs that read the same series tiles (one per query tile) stay within a few items of each
      // other, so a tile fetched from HBM by one of them is still in L2 for the others
      const int64_t G = gridDim.x, b = blockIdx.x;
      const bool grouped = mt > 1 && mt <= G && b < (G / mt) * mt;
      const int64_t g0 = grouped ? (b / mt) * mt : 0;
      volatile int* prog = A.progress;
      // slack in items: about D_AHEAD_CHUNKS K-chunks (short items get a wider window)
      const int64_t ahead = A.KC >= D_AHEAD_CHUNKS / 2 ? 2 : D_AHEAD_CHUNKS / A.KC;
      int64_t j = 0;
      for (; dense_item(j, mt, A.n_tiles, m, t); ++j) {
        if (grouped && j > ahead && j % (ahead / 2 > 0 ? ahead / 2 : 1) == 0) {
          for (;;) {  // all members' progress loaded together, then compared
            int lo = 0x7fffffff;
            for (int64_t o = 0; o < mt; ++o) {
              const int p = prog[g0 + o];
              lo = p < lo ? p : lo;
            }
            if (lo >= j - ahead) break;
            __nanosleep(128);
          }
        }
        for (int kc = 0; kc < A.KC; ++kc) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], DA_BYTES + DB_BYTES);
          tma_load_2d(sA + stage * DA_BYTES, &tmQ, kc * DKC, m * DM, &full[stage]);
          tma_load_2d(sB + stage * DB_BYTES, &tmX, kc * DKC, (int)(t * DN), &full[stage]);
          if (++stage == DSTAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        prog[b] = (int)(j + 1);  // items whose loads this CTA has issued
      }
      prog[b] = 0x7fffffff;  // done: never holds the group back
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer (one thread)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int m;
      int64_t t, local = 0;
      for (int64_t j = 0; dense_item(j, mt, A.n_tiles, m, t); ++j, ++local) {
        const int acc = (int)(local & 1);
        const uint32_t aph = (uint32_t)((local >> 1) & 1);
        mbar_wait(&tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t dt = tmem + (uint32_t)(acc * DN);
        for (int kc = 0; kc < A.KC; ++kc) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + stage * DA_BYTES), b0 = smem_u32(sB + stage * DB_BYTES);
#pragma unroll
          for (int kk = 0; kk < DKC / 8; ++kk)  // UMMA_K = 8 tf32 = 32 bytes along the swizzled row
            tc_mma_tf32(dt, sdesc_sw128(a0 + 32 * kk), sdesc_sw128(b0 + 32 * kk), kIdescTF32, (kc | kk) ? 1u : 0u);
          tc_commit(&empty[stage]);
          if (++stage == DSTAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit(&tfull[acc]);
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue (8 warps)
    // warp w reads TMEM lane quarter w % 4 (query rows) and column half (w - 2) / 4 (series).
    // Per element: approx' = -2 inv dot + |q^|^2 + |x^|^2 (2 ops); the per-row error terms are
    // replaced by their maximum over the tile's rows (a valid, marginally looser bound):
    //   eps_max = 2 gamma |q^| max_s(inv |x|) + slack_q + max_s(slack_s) + |sum q^| max_s|2 mu inv|
    // (the last term covers dropping +2 mu inv sum(q^) from approx').  LB = approx' - eps_max,
    // UB = approx' + eps_max.
    const int eq = warp & 3;
    const int half = (warp - 2) >> 2;
    const int row = eq * 32 + lane;
    const int et = (warp - 2) * 32 + lane;  // 0..255: one series of the tile each in the fill
    const float nlen = (float)A.len;
    // per thread (one query row): the k smallest UB_g it has seen, kept across all of the CTA's items
    // (the grid is a multiple of the number of query tiles, so a CTA always serves the same tile)
    const int kk = A.k;
    const bool track = kk <= D_UBK;
    float ubk = INFINITY;  // k-th smallest UB seen: a proven bound on the query's k-th best
    float ubl[D_UBK];
    int nub = 0;
    int cur_m = -1, m;
    int64_t t, local = 0;
    for (int64_t j = 0; dense_item(j, mt, A.n_tiles, m, t); ++j, ++local) {
      if (m != cur_m) {  // only with more query tiles than CTAs
        cur_m = m;
        ubk = INFINITY;
        nub = 0;
      }
      const int acc = (int)(local & 1);
      const uint32_t aph = (uint32_t)((local >> 1) & 1);
      float2* ser = s_ser2 + acc * DN;     // (-2 inv, |x^|^2), NaN |x^|^2 past the last row
      float* tmx = s_tmax + acc * 4;      // tile maxima: inv |x|, slack_s, |2 mu inv|
      {
        const int64_t s = t * DN + et;
        // past the last row: NaN, never <= any threshold (+inf would pass an infinite one, i.e.
        // while a query holds fewer than k results)
        float2 v = make_float2(0.f, __int_as_float(0x7fffffff));
        float e = 0.f, rs = 0.f, b = 0.f;
        if (s < A.n) {
          const float2 st = A.stats_orig[s];
          v = make_float2(0.f, 0.f);
          if (st.y > 0.f) {
            const float mi = st.x * st.y;
            v = make_float2(-2.f * st.y, nlen);
            e = sqrtf(nlen * (1.f + mi * mi)) * 1.0001f;
            rs = fmaf(2.4e-7f, e * e, 2e-4f * nlen);
            b = fabsf(2.f * mi);
          }
        }
        ser[et] = v;
        // max over the tile's rows (non-negative floats order like their bit patterns)
        e = fmaxf(e, __shfl_xor_sync(FULL, e, 16)); rs = fmaxf(rs, __shfl_xor_sync(FULL, rs, 16));
        b = fmaxf(b, __shfl_xor_sync(FULL, b, 16));
#pragma unroll
        for (int o = 8; o >= 1; o >>= 1) {
          e = fmaxf(e, __shfl_xor_sync(FULL, e, o));
          rs = fmaxf(rs, __shfl_xor_sync(FULL, rs, o));
          b = fmaxf(b, __shfl_xor_sync(FULL, b, o));
        }
        if (lane == 0) {
          atomicMax(reinterpret_cast<unsigned int*>(&tmx[0]), __float_as_uint(e));
          atomicMax(reinterpret_cast<unsigned int*>(&tmx[1]), __float_as_uint(rs));
          atomicMax(reinterpret_cast<unsigned int*>(&tmx[2]), __float_as_uint(b));
        }
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
      const int slot = m * DM + row;
      const bool qv = slot < qd;
      const float4 qp = qv ? A.qparams[slot] : make_float4(0.f, 0.f, 0.f, 0.f);
      const float eps = fmaf(qp.z, tmx[0], qp.w + tmx[1]) + fabsf(qp.y) * tmx[2];
      float thr = qv ? fminf(*(volatile float*)&A.thr[slot], ubk) : -INFINITY;
      float thr_e = thr + eps;
      float ubk_ap = ubk - eps;  // a row improves the UB list iff approx' < ubk - eps
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const uint32_t tbase = tmem + ((uint32_t)(eq * 32) << 16) + (uint32_t)(acc * DN + half * (DN / 2));
      uint32_t r[2][32];
      TMEM_LD32(tbase, r[0]);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int c = 0; c < DN / 64; ++c) {
        uint32_t (&cur)[32] = r[c & 1];
        if (c + 1 < DN / 64) TMEM_LD32(tbase + (c + 1) * 32, r[(c + 1) & 1]);  // next chunk in flight
        const int col0 = half * (DN / 2) + c * 32;
        float amin = INFINITY;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float2 sv = ser[col0 + j];
          const float ap = fmaf(sv.x, __uint_as_float(cur[j]), qp.x + sv.y);
          cur[j] = __float_as_uint(ap);
          amin = fminf(amin, ap);
          if constexpr (!KONE) {
            if (track && ap < ubk_ap) {
              ub_insert(ubl, nub, ubk, kk, ap + eps);
              ubk_ap = ubk - eps;
            }
          }
        }
        if (__any_sync(FULL, amin <= thr_e)) {  // rare: emit this chunk's candidates (compact code)
          uint32_t pass = 0;
#pragma unroll
          for (int j = 0; j < 32; ++j) pass |= (__uint_as_float(cur[j]) <= thr_e ? 1u : 0u) << j;
          while (__any_sync(FULL, pass != 0)) {
            const int j = pass ? __ffs(pass) - 1 : 0;
            emit_candidate(A, pass != 0, slot, (uint32_t)(t * DN + col0 + j));
            pass &= pass - 1;
          }
        }
        if constexpr (KONE) ubk = fminf(ubk, amin + eps);
        thr = fminf(thr, fmaxf(ubk, 0.f));
        thr_e = thr + eps;
        if (c + 1 < DN / 64) asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (qv && thr >= 0.f && thr < INFINITY) {
        const float g = *(volatile float*)&A.thr[slot];
        if (thr < g) atomicMin(reinterpret_cast<unsigned int*>(&A.thr[slot]), __float_as_uint(thr));
      }
      // reset this buffer's tile maxima for its next use (two items later, after the bar.sync of
      // the next item every thread has read them)
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (et < 4) tmx[et] = 0.f;
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
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
  const unsigned long long* cand;
  int64_t cand_cap;
  const unsigned long long* cand_count;
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
  const int64_t nc_raw = (int64_t)*P.cand_count;
  const int64_t nc = nc_raw < P.cand_cap ? nc_raw : P.cand_cap;
  const int nov = *P.ovf_count;
  const int64_t total = nc + (int64_t)nov * P.n;
  unsigned int n_ref = 0;
  for (int64_t u = gw; u < total; u += nw) {
    int slot;
    int64_t row;
    if (u < nc) {
      const unsigned long long e = P.cand[u];
      slot = (int)(e >> 32);
      row = (int64_t)(uint32_t)e;
      if (P.overflow[slot]) continue;  // the fallback below rescans that slot completely
    } else {
      slot = P.ovf_list[(u - nc) / P.n];
      row = (u - nc) % P.n;
    }
    float bsf = 0.f;
    if (lane == 0) bsf = *(volatile float*)&P.bsf[slot];
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
      const int n = *(volatile int*)&P.tkn[slot];
      if (n < P.k || d2[0] <= bsf) g_topk_insert(P, slot, d2[0], (int)row);
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
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// rows x len float32 row-major, box = 32 fp32 (128 B, swizzled) x box_rows
static int make_tmap(CUtensorMap* m, const float* base, int64_t rows, int len, int box_rows) {
  auto enc = encode_fn();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return SOFA_ECUDA;
  }
  cuuint64_t dims[2] = {(cuuint64_t)len, (cuuint64_t)(rows > 0 ? rows : 1)};
  cuuint64_t strides[1] = {(cuuint64_t)len * 4};
  cuuint32_t box[2] = {(cuuint32_t)DKC, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return SOFA_ECUDA;
  }
  return SOFA_OK;
}

int launch_dense(sofa_index* ix, int q, int k, float* od, int64_t* oi, bool stats, cudaStream_t st) {
  DenseScratch& D = ix->dense;
  int rc;
  if (D.tmap_q_rows != q) {  // tensor maps are encoded once per buffer (not on every call)
    if ((rc = make_tmap(reinterpret_cast<CUtensorMap*>(D.tmap_q), D.qhat, q, ix->len, DM))) return rc;
    if ((rc = make_tmap(reinterpret_cast<CUtensorMap*>(D.tmap_x), ix->series, ix->n, ix->len, DN))) return rc;
    D.tmap_q_rows = q;
  }
  const CUtensorMap& tmQ = *reinterpret_cast<const CUtensorMap*>(D.tmap_q);
  const CUtensorMap& tmX = *reinterpret_cast<const CUtensorMap*>(D.tmap_x);
  DenseArgs A{};
  A.n = ix->n;
  A.dense_rows = dense_batch_rows(ix);
  A.len = ix->len;
  A.k = k;
  A.KC = (ix->len + DKC - 1) / DKC;
  A.n_tiles = (ix->n + DN - 1) / DN;
  A.stats_orig = ix->stats_orig;
  A.qd_count = D.counters;
  A.qparams = D.qparams;
  A.thr = D.thr;
  A.cand = D.cand;
  A.cand_cap = D.cand_cap;
  A.cand_count = reinterpret_cast<unsigned long long*>(D.counters + 2);
  A.overflow = D.overflow;
  A.ovf_list = D.ovf_list;
  A.ovf_count = D.counters + 1;
  A.progress = D.counters + 64;
  auto screen = k == 1 ? k_dense_screen<true> : k_dense_screen<false>;
  const int sms = ix->sms;
  static std::atomic<uint32_t> attr_set{0};  // per (device, k == 1): smem attribute set once
  const uint32_t bit = 1u << ((ix->device * 2 + (k == 1)) & 31);
  if (!(attr_set.load() & bit)) {
    SOFA_CK(cudaFuncSetAttribute(screen, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)D_SMEM));
    attr_set.fetch_or(bit);
  }
  screen<<<sms, D_THREADS, D_SMEM, st>>>(tmQ, tmX, A);
  SOFA_LAUNCHED();

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
  P.lock = D.lock;
  P.cand = D.cand;
  P.cand_cap = D.cand_cap;
  P.cand_count = A.cand_count;
  P.overflow = D.overflow;
  P.ovf_list = D.ovf_list;
  P.ovf_count = D.counters + 1;
  P.done = reinterpret_cast<unsigned int*>(D.counters + 4);
  P.od = od;
  P.oi = oi;
  P.dstats = stats ? ix->dstats : nullptr;
  const int nf4 = ix->len / 4;
  const int grid = sms * 4;
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

// scratch for q queries at k (grown on demand); counters: [0] dense slots, [1] overflow slots,
// [2..3] candidate count (u64), [4] done CTAs.
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
  SOFA_CK(cudaMalloc(&D.qparams, (size_t)q * 16));
  SOFA_CK(cudaMalloc(&D.qidx, (size_t)q * 4));
  SOFA_CK(cudaMalloc(&D.binit, (size_t)q * 4));
  SOFA_CK(cudaMalloc(&D.bsf, (size_t)q * 4));
  SOFA_CK(cudaMalloc(&D.thr, (size_t)q * 4));
  SOFA_CK(cudaMalloc(&D.tkd, (size_t)q * k * 4));
  SOFA_CK(cudaMalloc(&D.tki, (size_t)q * k * 4));
  SOFA_CK(cudaMalloc(&D.tkn, (size_t)q * 4));
  SOFA_CK(cudaMalloc(&D.lock, (size_t)q * 4));
  SOFA_CK(cudaMalloc(&D.overflow, (size_t)q * 4));
  SOFA_CK(cudaMalloc(&D.ovf_list, (size_t)q * 4));
  SOFA_CK(cudaMalloc(&D.cand, (size_t)D.cand_cap * 8));
  SOFA_CK(cudaMalloc(&D.counters, 64 + 1024 * 4));  // counters, then per-CTA progress
  return SOFA_OK;
}

void free_dense_scratch(sofa_index* ix) {
  DenseScratch& D = ix->dense;
  void* ps[] = {D.qhat, D.qparams, D.qidx, D.binit, D.bsf, D.thr, D.tkd, D.tki, D.tkn, D.lock, D.overflow, D.ovf_list,
                D.cand, D.counters};
  for (void* p : ps)
    if (p) cudaFree(p);
  D = DenseScratch{};
}

}  // namespace sofa
