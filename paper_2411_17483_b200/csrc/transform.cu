// a1 + a3 (z-norm statistics, SFA projection, quantisation) and a4 (block layout helpers).
//
// k_transform is one HBM pass over the series (Alg. 2, applied to every row).
// Layout: a row is owned by a GROUP of G lanes (G = n/32 rounded up to a power of two, so each lane
// holds 8 float4 = 32 values: float4 index g + G*f, f < 8); a warp holds 32/G rows at once.  The
// group layout keeps the cross-lane work per row small (log2 G butterfly stages instead of 5).
//   * row statistics with row_stats_g (common.cuh; the query prep uses the same function, so a
//     query equal to a stored row z-normalises to the same float32 bits);
//   * DFT symmetry fold (n = 32 G, a DFT model): a selected position is Re X_k (basis cos, even
//     about t = 0 mod n) or Im X_k (basis -sin, odd), so with u_t = x_t + x_{n-t} and
//     v_t = x_t - x_{n-t} the dot products need only t < n/2: Re rows use u (the t = n/2 term
//     folded into u_0 as x_0 +- x_{n/2}, the sign being cos(pi k)), Im rows use v.  The partner
//     x_{n-t} of the value a lane holds sits in lane G-1-g (or G-g for the first component) of the
//     same group at slot 7-f: 4 sub-group shuffles per slot pair.  This halves the FFMA work; the
//     basis rows are processed in the order [Re even k | Re odd k | Im] (a permutation of the
//     model's positions, undone when the symbols are written);
//   * float32 FFMA partial dot products, then a reduce-scatter butterfly over the group leaves
//     each lane with fully reduced (row, coefficient) values;
//   * value * (1/sigma), symbol = number of float32 edges <= value (binary search over the edge row
//     in shared memory; float32 rounding moves a value by ~1e-7 relative, inside reading 24's
//     1e-5 edge exemption), the a4 key bits of the lane's symbols OR-reduced over the group;
//   * optionally the z-normalised row as bfloat16 (original row order) for the dense screen (f1).
// Measured (B200, configs[2], 10M x 256, tools/transform_probe.py): 3.65 TB/s of algorithmic bytes
// (10.24 GB read + 5.39 GB written in ~4.3 ms), 0.56 of the measured copy bandwidth.  The bound is the
// shared-memory LSU pipe (ncu: l1tex__data_pipe_lsu_wavefronts 92% of peak, DRAM 45%, issue 59%): per
// 4-row warp iteration ~410 wavefronts - 256 for the basis (one wavefront feeds one FFMA warp
// instruction whatever the load width; the warp's four row groups read the same bytes), 32 for the
// row buffer, ~57 for the edge searches, ~60 shuffles (DESIGN 12).  Round 2: the Re/Im operand choice
// is a warp-uniform branch per basis row (a register swap at the runtime Re/Im boundary made the
// compiler carry both assignments: ~500 moves per row group), 80 registers for 3 CTAs per SM, (G <= 8)
// the next row group is bulk-copied into a per-warp shared-memory buffer while the current one is
// transformed, 16-position key bits as two 32-bit shifts and one 16-byte word store per row:
// 2.93 -> 3.65 TB/s.
// The accuracy budget (symbols bit-exact outside 1e-5 of an edge, SURVEY 8(c) reading 24) rules out
// 1xTF32 tensor cores.
#include <cub/cub.cuh>

#include <cuda_bf16.h>

#include "common.cuh"

namespace sofa {

// Reduce-scatter over the G lanes of a group: V values per lane in, after log2(G) stages lane g of
// the group holds the group-sum of value g*(V/G)+i in v[i] (V >= G) or, if V < G, every lane holds
// the sum of value g/(G/V) in v[0].
template <int V, int M>
__device__ __forceinline__ void reduce_scatter_g(float* v, int lane) {
  if constexpr (M >= 1) {
    if constexpr (V > 1) {
      constexpr int H = V / 2;
      const bool up = (lane & M) != 0;
#pragma unroll
      for (int i = 0; i < H; ++i) {
        const float send = up ? v[i] : v[i + H];
        const float keep = up ? v[i + H] : v[i];
        v[i] = keep + __shfl_xor_sync(FULL, send, M);
      }
      reduce_scatter_g<H, M / 2>(v, lane);
    } else {
      v[0] += __shfl_xor_sync(FULL, v[0], M);
      reduce_scatter_g<1, M / 2>(v, lane);
    }
  }
}

// one bulk copy (TMA, 1D) of a warp's next rows into its shared-memory buffer, completion counted on
// the warp's mbarrier: the loads of row group i + 1 are in flight while group i is transformed
__device__ __forceinline__ void tr_mbar_init(uint64_t* b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)) : "memory");
}
__device__ __forceinline__ void tr_bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          (uint32_t)__cvta_generic_to_shared(dst)),
      "l"(src), "r"(bytes), "r"(b)
      : "memory");
}
__device__ __forceinline__ void tr_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
  uint32_t ok = 0;
  while (!ok)
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(b), "r"(parity)
        : "memory");
}
constexpr int kTrBuf = 4096;  // bytes per warp: RPW rows of len <= 32 G floats

constexpr int kEdgeLd = 257;  // shared-memory row stride of the edge table (floats)

struct TransformArgs {
  const float* X;
  int64_t N;
  int len, l, a_bits, WS;
  int n_re_even, n_re_odd;      // fold: basis rows [0, ne) Re with even k, [ne, ne+no) Re odd k, rest Im
  const float* basis;           // LT x (8 G) float4-slots: folded (4 slots) or full (8 slots) layout
  const int* order;             // LT: processing row jj -> model position j
  const float* edges32;
  uint8_t* words;
  float2* stats;
  uint64_t* keys;
  double* vals;
  uint8_t* words_l;
  __nv_bfloat16* xb16;          // nullable: N x xb_ld z-normalised rows (dense screen operand)
  int xb_ld;
};

// 2 CTAs (16 warps, up to 128 registers) when the fold or wide words need the registers, else 3
template <int G, int LT, bool FOLD>
__global__ void __launch_bounds__(kThreads, LT > 16 ? 2 : 3) k_transform(const __grid_constant__ TransformArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int RPW = 32 / G;                 // rows per warp
  constexpr int NS = FOLD ? 4 : 8;            // basis slots per lane
  constexpr int VPL = LT >= G ? LT / G : 1;   // reduced values per lane
  constexpr int OWN = LT >= G ? 1 : G / LT;   // lanes sharing one value when LT < G
  // bulk-copy prefetch of the next row group (G <= 8: the basis loads broadcast over the warp's rows);
  // at G >= 16 the basis loads already fill shared-memory bandwidth and the rows load directly
  constexpr bool PREF = G <= 8;
  const int len = A.len, nf4 = len >> 2, l = A.l;
  float4* s_basis = reinterpret_cast<float4*>(smem);                           // LT x NS x G
  // LT x kEdgeLd (model order): rows padded to 257 floats so that the lanes of a warp, each searching
  // its own position's row, start in different banks (a 256-float stride put every row in one bank)
  float* s_edges = reinterpret_cast<float*>(smem + (size_t)LT * NS * G * 16);
  uint8_t* s_w = reinterpret_cast<uint8_t*>(s_edges + LT * kEdgeLd);          // 8 warps x RPW x LT
  int* s_ord = reinterpret_cast<int*>(s_w + 8 * RPW * LT);                      // LT
  // 8 warps x kTrBuf (16-byte aligned) row buffers, then 8 mbarriers
  unsigned char* s_xb = smem + (((size_t)LT * NS * G * 16 + (size_t)LT * kEdgeLd * 4 + 8 * RPW * LT + LT * 4 + 15) & ~(size_t)15);
  uint64_t* s_bar = reinterpret_cast<uint64_t*>(s_xb + 8 * kTrBuf);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane & (G - 1), rw = lane / G;  // lane in group, row of the warp
  for (int i = tid; i < LT * NS * G; i += kThreads) s_basis[i] = reinterpret_cast<const float4*>(A.basis)[i];
  for (int i = tid; i < LT * 256; i += kThreads) s_edges[(i >> 8) * kEdgeLd + (i & 255)] = A.edges32[i];
  for (int i = tid; i < 8 * RPW * LT; i += kThreads) s_w[i] = 0;
  for (int i = tid; i < LT; i += kThreads) s_ord[i] = A.order[i];
  __syncthreads();
  uint8_t* my_w = s_w + warp * RPW * LT;
  const int ne = A.n_re_even, nre = A.n_re_even + A.n_re_odd;
  const float c0x2 = (float)(2.0 / sqrt((double)A.len));  // 2 C(0) = 2 / sqrt(n)
  const int P = l < 16 ? l : 16;  // key positions
  const int sh8 = 8 - A.a_bits;

  const int64_t rstride = (int64_t)gridDim.x * 8 * RPW;
  unsigned char* my_xb = s_xb + warp * kTrBuf;
  uint64_t* my_bar = s_bar + warp;
  // the warp's RPW rows are contiguous in the series (row stride = len floats): one bulk copy of
  // min(RPW, N - r0) rows (len % 4 == 0: 16-byte aligned, a multiple of 16 bytes)
  auto issue = [&](int64_t r) {
    if (PREF && lane == 0 && r < A.N) {
      const int64_t nr = A.N - r < RPW ? A.N - r : RPW;
      tr_bulk_load(my_xb, A.X + r * len, (uint32_t)(nr * len * 4), my_bar);
    }
  };
  if (PREF && lane == 0) {
    tr_mbar_init(my_bar);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  uint32_t xphase = 0;
  issue(((int64_t)blockIdx.x * 8 + warp) * RPW);
  for (int64_t r0 = ((int64_t)blockIdx.x * 8 + warp) * RPW; r0 < A.N; r0 += rstride) {
    const int64_t row = r0 + rw;
    const bool live = row < A.N;
    float4 x[8];
    if constexpr (PREF) {
      tr_wait(my_bar, xphase);
      xphase ^= 1u;
      const float4* xr = reinterpret_cast<const float4*>(my_xb) + rw * nf4;
#pragma unroll
      for (int f = 0; f < 8; ++f) {
        const int fi = g + G * f;
        x[f] = (live && (FOLD || fi < nf4)) ? xr[fi] : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    } else {
      const float4* xr = reinterpret_cast<const float4*>(A.X + row * len);
#pragma unroll
      for (int f = 0; f < 8; ++f) {
        const int fi = g + G * f;
        x[f] = (live && (FOLD || fi < nf4)) ? ld_stream(xr + fi) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    float muf;
    double mu64, inv64;
    row_stats_g<G, FOLD>(x, nf4, g, len, muf, mu64, inv64);  // FOLD implies n = 32 G
    // every lane has consumed its buffer values (the statistics use all of them): the buffer may be
    // refilled with the next row group while this one is transformed
    if constexpr (PREF) {
      __syncwarp();
      if (lane == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(r0 + rstride);
    }
#pragma unroll
    for (int f = 0; f < 8; ++f) {
      x[f].x = __fsub_rn(x[f].x, muf);
      x[f].y = __fsub_rn(x[f].y, muf);
      x[f].z = __fsub_rn(x[f].z, muf);
      x[f].w = __fsub_rn(x[f].w, muf);
    }
    if (A.xb16 && live) {  // z-normalised row in bfloat16 (round to nearest), original order
      const float invf = (float)inv64;
#pragma unroll
      for (int f = 0; f < 8; ++f) {
        const int fi = g + G * f;
        if (FOLD || fi < nf4) {
          __nv_bfloat162 lo = __floats2bfloat162_rn(x[f].x * invf, x[f].y * invf);
          __nv_bfloat162 hi = __floats2bfloat162_rn(x[f].z * invf, x[f].w * invf);
          uint2 pk;
          pk.x = *reinterpret_cast<uint32_t*>(&lo);
          pk.y = *reinterpret_cast<uint32_t*>(&hi);
          *reinterpret_cast<uint2*>(A.xb16 + row * A.xb_ld + 4 * fi) = pk;
        }
      }
    }
    float acc[LT];
#pragma unroll
    for (int j = 0; j < LT; ++j) acc[j] = 0.f;
    float nyq_row = 0.f;  // fold: x_{n/2} - mu of this lane's row
    if constexpr (FOLD) {
      // u into x[f], v into x[7-f] (f < 4); pairs processed from the middle out so lane 0's
      // first-component partners x[8-f].x are read before their slot is overwritten
      const float nyq = x[4].x;  // lane g = 0: x_{n/2}
      const float x0 = x[0].x;   // lane g = 0: x_0 (no partner)
#pragma unroll
      for (int f = 3; f >= 0; --f) {
        const int src1 = G - 1 - g, src0 = (G - g) & (G - 1);
        const float p1 = __shfl_sync(FULL, x[7 - f].w, (lane & ~(G - 1)) | src1);
        const float p2 = __shfl_sync(FULL, x[7 - f].z, (lane & ~(G - 1)) | src1);
        const float p3 = __shfl_sync(FULL, x[7 - f].y, (lane & ~(G - 1)) | src1);
        float p0 = __shfl_sync(FULL, x[7 - f].x, (lane & ~(G - 1)) | src0);
        if (g == 0) p0 = f > 0 ? x[8 - f].x : 0.f;  // lane 0: partner in its own slot 8-f; t = 0 has none
        const float4 a = x[f];
        x[f] = make_float4(__fadd_rn(a.x, p0), __fadd_rn(a.y, p1), __fadd_rn(a.z, p2), __fadd_rn(a.w, p3));
        x[7 - f] = make_float4(__fsub_rn(a.x, p0), __fsub_rn(a.y, p1), __fsub_rn(a.z, p2), __fsub_rn(a.w, p3));
      }
      if (g == 0) x[0].x = __fadd_rn(x0, nyq);  // u_0 = x_0 + x_{n/2}: exact for Re rows with even k
      // processing rows [Re | Im]: u (x[0..3]) for the Re rows, v (x[7..4]) for the Im rows.  One
      // warp-uniform branch per row picks the operand registers (a register swap at the runtime
      // boundary j == nre made the compiler carry both assignments through the unrolled loop: ~500
      // register moves per row group)
      const float4* bs = s_basis + g;
      // blocks of JB basis rows: a block entirely on one side of the Re/Im boundary runs its rows
      // slot by slot (JB independent FFMA chains, JB x 4 basis loads the compiler can issue ahead:
      // the per-row form stalled ~20% of the samples on each row's own four loads); the one block
      // that straddles the boundary falls back to a branch per row.  Per row the FFMA order is
      // unchanged (slots 0..3, components x..w): the same float32 bits.
      constexpr int JB = LT > 16 ? 4 : 1;  // blocks only where 128 registers are available (2 CTAs/SM)
      auto rows_re = [&](int j0) {
#pragma unroll
        for (int f = 0; f < 4; ++f)
#pragma unroll
          for (int jj = 0; jj < JB; ++jj) {
            const float4 b = bs[((j0 + jj) * 4 + f) * G];
            float s = acc[j0 + jj];
            s = fmaf(x[f].x, b.x, s);
            s = fmaf(x[f].y, b.y, s);
            s = fmaf(x[f].z, b.z, s);
            s = fmaf(x[f].w, b.w, s);
            acc[j0 + jj] = s;
          }
      };
      auto rows_im = [&](int j0) {
#pragma unroll
        for (int f = 0; f < 4; ++f)
#pragma unroll
          for (int jj = 0; jj < JB; ++jj) {
            const float4 b = bs[((j0 + jj) * 4 + f) * G];
            float s = acc[j0 + jj];
            s = fmaf(x[7 - f].x, b.x, s);
            s = fmaf(x[7 - f].y, b.y, s);
            s = fmaf(x[7 - f].z, b.z, s);
            s = fmaf(x[7 - f].w, b.w, s);
            acc[j0 + jj] = s;
          }
      };
#pragma unroll
      for (int j0 = 0; j0 < LT; j0 += JB) {
        if (j0 + JB <= nre) {
          rows_re(j0);
        } else if (j0 >= nre) {
          rows_im(j0);
        } else {
#pragma unroll
          for (int j = j0; j < j0 + JB; ++j) {
            float s = acc[j];
            if (j < nre) {
#pragma unroll
              for (int f = 0; f < 4; ++f) {
                const float4 b = bs[(j * 4 + f) * G];
                s = fmaf(x[f].x, b.x, s);
                s = fmaf(x[f].y, b.y, s);
                s = fmaf(x[f].z, b.z, s);
                s = fmaf(x[f].w, b.w, s);
              }
            } else {
#pragma unroll
              for (int f = 0; f < 4; ++f) {
                const float4 b = bs[(j * 4 + f) * G];
                s = fmaf(x[7 - f].x, b.x, s);
                s = fmaf(x[7 - f].y, b.y, s);
                s = fmaf(x[7 - f].z, b.z, s);
                s = fmaf(x[7 - f].w, b.w, s);
              }
            }
            acc[j] = s;
          }
        }
      }
      nyq_row = __shfl_sync(FULL, nyq, lane & ~(G - 1));
    } else {
      const float4* bs = s_basis + g;
#pragma unroll
      for (int j = 0; j < LT; ++j) {
        if (j >= l) break;
#pragma unroll
        for (int f = 0; f < 8; ++f) {
          const float4 b = bs[(j * 8 + f) * G];
          float s = acc[j];
          s = fmaf(x[f].x, b.x, s);
          s = fmaf(x[f].y, b.y, s);
          s = fmaf(x[f].z, b.z, s);
          s = fmaf(x[f].w, b.w, s);
          acc[j] = s;
        }
      }
    }
    reduce_scatter_g<LT, G / 2>(acc, lane);
    // this lane's reduced values: processing rows jj = g*VPL + i (or g/OWN), model position s_ord[jj]
    unsigned long long key = 0ull;
    if (g % OWN == 0) {
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        const int jj = LT >= G ? g * VPL + i : g / OWN;
        if (jj < l) {
          const int j = s_ord[jj];
          // Re rows with odd k: u_0 held x_0 + x_{n/2}, their t = n/2 term is -x_{n/2} C(0)
          const float a = FOLD && jj >= ne && jj < nre ? fmaf(-c0x2, nyq_row, acc[i]) : acc[i];
          const double vd = (double)a * inv64;
          if (A.vals && live) A.vals[row * l + j] = vd;
          const float v = (float)vd;
          const float* e = s_edges + j * kEdgeLd;
          int pos = 0;
#pragma unroll
          for (int step = 128; step >= 1; step >>= 1)
            if (e[pos + step - 1] <= v) pos += step;
          my_w[rw * LT + j] = (uint8_t)pos;
          if (j < P) {  // a4 key bits of this position: 2-bit digits, MSB first, round-robin
            const uint32_t s8 = ((uint32_t)pos << sh8) & 0xffu;
            if (P == 16) {
              // 16 key positions (warp-uniform): round 0 fills the high word, round 1 the low word,
              // rounds 2 and 3 fall past bit 0 - two 32-bit shifts instead of four guarded 64-bit ones
              const int sh = 30 - 2 * j;
              key |= ((unsigned long long)(((s8 >> 6) & 3u) << sh) << 32) | (unsigned long long)(((s8 >> 4) & 3u) << sh);
            } else {
#pragma unroll
              for (int r = 0; r < 4; ++r) {
                const int o = r * 2 * P + 2 * j;
                if (o < 64) key |= (unsigned long long)((s8 >> (6 - 2 * r)) & 3u) << (62 - o);
              }
            }
          }
        }
      }
    }
#pragma unroll
    for (int M = G / 2; M >= 1; M >>= 1) key |= __shfl_xor_sync(FULL, key, M);
    __syncwarp();
    if (g == 0 && live) {
      if (A.stats) A.stats[row] = make_float2(muf, (float)inv64);
      if (A.keys) A.keys[row] = key;
    }
    if (LT == 16 && A.words) {  // WS == 16: one 16-byte word per row, lane s writes row s
      if (lane < RPW && r0 + lane < A.N)
        *reinterpret_cast<uint4*>(A.words + (r0 + lane) * 16) = *reinterpret_cast<const uint4*>(my_w + lane * LT);
    } else if (A.words) {
      const int parts = A.WS >> 4;
      for (int c = lane; c < RPW * parts; c += 32) {
        const int s = c / parts, p = c % parts;
        if (r0 + s < A.N)
          *reinterpret_cast<uint4*>(A.words + (r0 + s) * A.WS + p * 16) =
              *reinterpret_cast<const uint4*>(my_w + s * LT + p * 16);
      }
    }
    if (A.words_l) {
      for (int c = lane; c < RPW * l; c += 32) {
        const int s = c / l, j = c % l;
        if (r0 + s < A.N) A.words_l[(r0 + s) * l + j] = my_w[s * LT + j];
      }
    }
    __syncwarp();
  }
}

// Host: the processing order of the basis rows and the per-lane slot layout of the basis.
// basis32 (DevModel) is LT x len in model order; the kernel wants, per processing row jj and slot
// (f, g), the float4 of basis values at t = 4 (g + G f) .. +3 (full layout, 8 slots) or the folded
// values for t < n/2 (4 slots; Re rows: C(t) for t >= 1 and C(0) at t = 0, Im rows: S(t), S(0) = 0).
int transform_layout(const DevModel& dm, const sofa_model& m, int G, bool fold, std::vector<float>& basis,
                     std::vector<int>& order, int& ne, int& no) {
  const int LT = dm.LT, len = dm.len, l = dm.l;
  const int NS = fold ? 4 : 8;
  std::vector<int> re_even, re_odd, im;
  for (int j = 0; j < l; ++j) {
    const int k = m.best_pos[j] >> 1, isim = m.best_pos[j] & 1;
    (isim ? im : (k % 2 ? re_odd : re_even)).push_back(j);
  }
  order.clear();
  if (fold) {
    order.insert(order.end(), re_even.begin(), re_even.end());
    order.insert(order.end(), re_odd.begin(), re_odd.end());
    order.insert(order.end(), im.begin(), im.end());
    ne = (int)re_even.size();
    no = (int)re_odd.size();
  } else {
    for (int j = 0; j < l; ++j) order.push_back(j);
    ne = l;
    no = 0;
  }
  while ((int)order.size() < LT) order.push_back((int)order.size());
  // basis values (float64 -> float32) of model position j at time t, computed exactly like k_basis_sel
  const double rs = 1.0 / std::sqrt((double)len);
  auto phi = [&](int j, int t) -> double {
    if (j >= l || t < 0 || t >= len) return 0.0;
    if (m.binning == SOFA_BINNING_ISAX) {
      const int seg = len / l;
      return t / seg == m.best_pos[j] ? 1.0 / seg : 0.0;
    }
    const int k = m.best_pos[j] >> 1, isim = m.best_pos[j] & 1;
    const int mm = (int)(((int64_t)k * t) % len);
    const double ang = 2.0 * M_PI * mm / len;
    return isim ? -std::sin(ang) * rs : std::cos(ang) * rs;
  };
  basis.assign((size_t)LT * NS * G * 4, 0.f);
  for (int jj = 0; jj < LT; ++jj) {
    const int j = jj < l ? order[jj] : l;  // padded rows are zero
    for (int f = 0; f < NS; ++f)
      for (int gg = 0; gg < G; ++gg)
        for (int c = 0; c < 4; ++c) {
          const int t = 4 * (gg + G * f) + c;
          basis[(((size_t)jj * NS + f) * G + gg) * 4 + c] = (float)phi(j, t);
        }
  }
  return SOFA_OK;
}

template <int G, int LT, bool FOLD>
static int launch_transform_t(const TransformArgs& A0, const DevModel& dm, const sofa_model& m, cudaStream_t st,
                              cudaEvent_t t_start) {
  TransformArgs A = A0;
  std::vector<float> hb;
  std::vector<int> ord;
  int ne = 0, no = 0;
  transform_layout(dm, m, G, FOLD, hb, ord, ne, no);
  float* db = nullptr;
  int* dord = nullptr;
  SOFA_CK(cudaMallocAsync(reinterpret_cast<void**>(&db), hb.size() * 4, st));
  SOFA_CK(cudaMallocAsync(reinterpret_cast<void**>(&dord), ord.size() * 4, st));
  SOFA_CK(cudaMemcpyAsync(db, hb.data(), hb.size() * 4, cudaMemcpyHostToDevice, st));
  SOFA_CK(cudaMemcpyAsync(dord, ord.data(), ord.size() * 4, cudaMemcpyHostToDevice, st));
  A.basis = db;
  A.order = dord;
  A.n_re_even = ne;
  A.n_re_odd = no;
  constexpr int RPW = 32 / G, NS = FOLD ? 4 : 8;
  auto kern = k_transform<G, LT, FOLD>;
  const size_t smem = (((size_t)LT * NS * G * 16 + (size_t)LT * kEdgeLd * 4 + 8 * RPW * LT + LT * 4 + 15) & ~(size_t)15) +
                      (G <= 8 ? 8 * kTrBuf + 8 * 8 : 0);  // PREF: row buffers + mbarriers
  SOFA_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  SOFA_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem));
  if (per_sm < 1) per_sm = 1;
  const int64_t want = (A.N + 8 * RPW - 1) / (8 * RPW);
  int grid = (int)(want < (int64_t)sms * per_sm ? want : (int64_t)sms * per_sm);
  if (grid < 1) grid = 1;
  if (t_start) cudaEventRecord(t_start, st);  // the kernel alone (after the host-side setup above)
  kern<<<grid, kThreads, smem, st>>>(A);
  SOFA_LAUNCHED();
  cudaFreeAsync(db, st);
  cudaFreeAsync(dord, st);
  return SOFA_OK;
}

int launch_transform(const float* X, int64_t N, const DevModel& dm, const sofa_model& m, uint8_t* words,
                     float2* stats, uint64_t* keys, double* vals, uint8_t* words_l, __nv_bfloat16* xb16,
                     cudaStream_t st, cudaEvent_t t_start) {
  if (N <= 0) return SOFA_OK;
  const int nf4 = dm.len / 4;
  int G = 1;
  while (G * 8 < nf4) G *= 2;  // 8 float4 per lane
  // the fold needs the exact group layout (n = 32 G) and a DFT model (iSAX rows are not symmetric)
  const bool fold = nf4 == 8 * G && m.binning != SOFA_BINNING_ISAX;
  TransformArgs A{};
  A.X = X;
  A.N = N;
  A.len = dm.len;
  A.l = dm.l;
  A.a_bits = dm.a_bits;
  A.WS = dm.WS;
  A.edges32 = dm.edges32;
  A.words = words;
  A.stats = stats;
  A.keys = keys;
  A.vals = vals;
  A.words_l = words_l;
  A.xb16 = xb16;
  A.xb_ld = (dm.len + 7) / 8 * 8;
#define SOFA_TR(g, lt)                                                                        \
  if (G == g && dm.LT == lt)                                                                  \
    return fold ? launch_transform_t<g, lt, true>(A, dm, m, st, t_start)                  \
                : launch_transform_t<g, lt, false>(A, dm, m, st, t_start);
  SOFA_TR(1, 16) SOFA_TR(2, 16) SOFA_TR(4, 16) SOFA_TR(8, 16) SOFA_TR(16, 16) SOFA_TR(32, 16)
  SOFA_TR(1, 32) SOFA_TR(2, 32) SOFA_TR(4, 32) SOFA_TR(8, 32) SOFA_TR(16, 32) SOFA_TR(32, 32)
  SOFA_TR(1, 64) SOFA_TR(2, 64) SOFA_TR(4, 64) SOFA_TR(8, 64) SOFA_TR(16, 64) SOFA_TR(32, 64)
#undef SOFA_TR
  set_error("transform: unsupported (len, l) combination");
  return SOFA_EINVAL;
}

// ---------------------------------------------------------------------------------------------
// a4: gather words / stats into sorted order.
__global__ void k_gather(const uint8_t* __restrict__ words, const float2* __restrict__ stats,
                         const int32_t* __restrict__ perm, int64_t n, int WS, uint8_t* __restrict__ wout,
                         float2* __restrict__ sout) {
  const int parts = WS >> 4;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n * parts;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pos = i / parts;
    const int p = (int)(i % parts);
    const int64_t src = perm[pos];
    *reinterpret_cast<uint4*>(wout + pos * WS + p * 16) = *reinterpret_cast<const uint4*>(words + src * WS + p * 16);
    if (p == 0) sout[pos] = stats[src];
  }
}

int launch_gather(const uint8_t* words, const float2* stats, const int32_t* perm, int64_t n, int WS,
                  uint8_t* words_out, float2* stats_out, cudaStream_t st) {
  if (n <= 0) return SOFA_OK;
  int64_t tot = n * (WS >> 4);
  int grid = (int)((tot + kThreads - 1) / kThreads);
  if (grid > 148 * 16) grid = 148 * 16;
  k_gather<<<grid, kThreads, 0, st>>>(words, stats, perm, n, WS, words_out, stats_out);
  SOFA_LAUNCHED();
  return SOFA_OK;
}

// a4: per block of B sorted words, the per-position min / max symbol (the block's envelope;
// MESSI leaves' iSAX envelope, in SFA form) and the block's first key.
__global__ void k_envelopes(const uint8_t* __restrict__ words, int64_t n, int B, int WS,
                            const uint64_t* __restrict__ skeys, uint8_t* __restrict__ env,
                            uint64_t* __restrict__ bkey) {
  const int lane = threadIdx.x & 31;
  const int64_t nb = (n + B - 1) / B;
  const int parts = WS >> 4;
  for (int64_t blk = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; blk < nb;
       blk += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t start = blk * B;
    const int64_t end = start + B < n ? start + B : n;
    uint4 mn[4], mx[4];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      mn[p] = make_uint4(~0u, ~0u, ~0u, ~0u);
      mx[p] = make_uint4(0u, 0u, 0u, 0u);
    }
    for (int64_t m = start + lane; m < end; m += 32) {
#pragma unroll
      for (int p = 0; p < 4; ++p)
        if (p < parts) {
          const uint4 w = *reinterpret_cast<const uint4*>(words + m * WS + p * 16);
          mn[p].x = __vminu4(mn[p].x, w.x); mn[p].y = __vminu4(mn[p].y, w.y);
          mn[p].z = __vminu4(mn[p].z, w.z); mn[p].w = __vminu4(mn[p].w, w.w);
          mx[p].x = __vmaxu4(mx[p].x, w.x); mx[p].y = __vmaxu4(mx[p].y, w.y);
          mx[p].z = __vmaxu4(mx[p].z, w.z); mx[p].w = __vmaxu4(mx[p].w, w.w);
        }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        mn[p].x = __vminu4(mn[p].x, __shfl_xor_sync(FULL, mn[p].x, o));
        mn[p].y = __vminu4(mn[p].y, __shfl_xor_sync(FULL, mn[p].y, o));
        mn[p].z = __vminu4(mn[p].z, __shfl_xor_sync(FULL, mn[p].z, o));
        mn[p].w = __vminu4(mn[p].w, __shfl_xor_sync(FULL, mn[p].w, o));
        mx[p].x = __vmaxu4(mx[p].x, __shfl_xor_sync(FULL, mx[p].x, o));
        mx[p].y = __vmaxu4(mx[p].y, __shfl_xor_sync(FULL, mx[p].y, o));
        mx[p].z = __vmaxu4(mx[p].z, __shfl_xor_sync(FULL, mx[p].z, o));
        mx[p].w = __vmaxu4(mx[p].w, __shfl_xor_sync(FULL, mx[p].w, o));
      }
    }
    if (lane < parts) {
      uint4 a = mn[0], b = mx[0];
#pragma unroll
      for (int p = 1; p < 4; ++p)
        if (lane == p) { a = mn[p]; b = mx[p]; }
      *reinterpret_cast<uint4*>(env + blk * 2 * WS + lane * 16) = a;
      *reinterpret_cast<uint4*>(env + blk * 2 * WS + WS + lane * 16) = b;
    }
    if (lane == 0) bkey[blk] = skeys[start];
  }
}

// a4: one level up the envelope tree: a parent's envelope is the min of its 16 children's mins and
// the max of their maxes (so parent LB <= child LB <= member LB).
__global__ void k_env_up(const uint8_t* __restrict__ child, int64_t nchild, int WS, uint8_t* __restrict__ parent) {
  const int parts = WS >> 4;
  const int64_t npar = (nchild + 15) / 16;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < npar * parts;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i / parts;
    const int c = (int)(i % parts);
    uint4 mn = make_uint4(~0u, ~0u, ~0u, ~0u), mx = make_uint4(0u, 0u, 0u, 0u);
    for (int64_t ch = p * 16; ch < p * 16 + 16 && ch < nchild; ++ch) {
      const uint4 a = *reinterpret_cast<const uint4*>(child + ch * 2 * WS + c * 16);
      const uint4 b = *reinterpret_cast<const uint4*>(child + ch * 2 * WS + WS + c * 16);
      mn.x = __vminu4(mn.x, a.x); mn.y = __vminu4(mn.y, a.y); mn.z = __vminu4(mn.z, a.z); mn.w = __vminu4(mn.w, a.w);
      mx.x = __vmaxu4(mx.x, b.x); mx.y = __vmaxu4(mx.y, b.y); mx.z = __vmaxu4(mx.z, b.z); mx.w = __vmaxu4(mx.w, b.w);
    }
    *reinterpret_cast<uint4*>(parent + p * 2 * WS + c * 16) = mn;
    *reinterpret_cast<uint4*>(parent + p * 2 * WS + WS + c * 16) = mx;
  }
}

int launch_env_up(const uint8_t* child, int64_t nchild, int WS, uint8_t* parent, cudaStream_t st) {
  const int64_t tot = (nchild + 15) / 16 * (WS >> 4);
  int grid = (int)((tot + kThreads - 1) / kThreads);
  if (grid > 148 * 16) grid = 148 * 16;
  if (grid < 1) grid = 1;
  k_env_up<<<grid, kThreads, 0, st>>>(child, nchild, WS, parent);
  SOFA_LAUNCHED();
  return SOFA_OK;
}

int launch_envelopes(const uint8_t* words, int64_t n, int B, int WS, const uint64_t* skeys, uint8_t* env,
                     uint64_t* bkey, cudaStream_t st) {
  const int64_t nb = (n + B - 1) / B;
  if (nb <= 0) return SOFA_OK;
  int grid = (int)((nb * 32 + kThreads - 1) / kThreads);
  if (grid > 148 * 16) grid = 148 * 16;
  k_envelopes<<<grid, kThreads, 0, st>>>(words, n, B, WS, skeys, env, bkey);
  SOFA_LAUNCHED();
  return SOFA_OK;
}

}  // namespace sofa
