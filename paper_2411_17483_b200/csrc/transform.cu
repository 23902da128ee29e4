// a1 + a3 (z-norm statistics, SFA projection, quantisation) and a4 (block layout helpers).
//
// k_transform is one HBM pass over the series (Alg. 2, applied to every row):
//   * one warp owns SER consecutive rows; lane holds float4 columns lane + 32 f (coalesced
//     512 B per warp-load, L1::no_allocate streaming);
//   * mean / std per row with the shared row_stats() (float32 lane partials, float64 combine);
//   * projection onto the LT selected basis rows (cos / -sin(2 pi k t/n) / sqrt(n), staged in
//     shared memory as float4 so a warp-load of the basis is 512 contiguous bytes): every lane
//     accumulates 4*NF-term float32 partial dot products, then a reduce-scatter butterfly over the
//     32 lanes leaves each lane with fully reduced (row, coefficient) values;
//   * value * (1/sigma) in float64, symbol = upper_bound over the float32 edge row (bins
//     [beta(s), beta(s+1))), key for a4, write word / stats / key.
// The projection is a dense [rows x n] x [n x l] contraction at 8 flop/B (n=256,l=16): FP32 FFMA
// keeps it at the HBM roofline on B200; the accuracy budget (symbols bit-exact outside 1e-5 of an
// edge, SURVEY 8(c) reading 24) rules out 1xTF32.  See DESIGN.md "K2".
#include <cub/cub.cuh>

#include "common.cuh"

namespace sofa {

template <int V, int M = 16>
__device__ __forceinline__ void reduce_scatter(float* v, int lane) {
  if constexpr (M >= 1) {
    if constexpr (V > 1) {
      constexpr int H = V / 2;
      const bool up = (lane & M) != 0;
#pragma unroll
      for (int i = 0; i < H; ++i) {
        float send = up ? v[i] : v[i + H];
        float keep = up ? v[i + H] : v[i];
        v[i] = keep + __shfl_xor_sync(FULL, send, M);
      }
      reduce_scatter<H, M / 2>(v, lane);
    } else {
      v[0] += __shfl_xor_sync(FULL, v[0], M);
      reduce_scatter<1, M / 2>(v, lane);
    }
  }
}

template <int NF, int LT, int SER>
__global__ void __launch_bounds__(kThreads, 2)
    k_transform(const float* __restrict__ X, int64_t N, int len, int l, int a_bits, int WS,
                const float* __restrict__ basis32, const float* __restrict__ edges32, uint8_t* __restrict__ words,
                float2* __restrict__ stats, uint64_t* __restrict__ keys, double* __restrict__ vals,
                uint8_t* __restrict__ words_l, int basis_in_smem) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int nf4 = len >> 2;
  // basis rows in shared memory when they fit (LT*len*4 bytes), else read through L1/L2
  const size_t basis_bytes = basis_in_smem ? (size_t)LT * len * 4 : 0;
  float4* s_basis = reinterpret_cast<float4*>(smem);                      // LT x nf4
  float* s_edges = reinterpret_cast<float*>(smem + basis_bytes);          // LT x 256
  uint8_t* s_w = reinterpret_cast<uint8_t*>(s_edges + LT * 256);         // 8 x SER x LT
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (basis_in_smem)
    for (int i = tid; i < LT * nf4; i += kThreads) s_basis[i] = reinterpret_cast<const float4*>(basis32)[i];
  const float4* bas = basis_in_smem ? s_basis : reinterpret_cast<const float4*>(basis32);
  for (int i = tid; i < LT * 256; i += kThreads) s_edges[i] = edges32[i];
  for (int i = tid; i < 8 * SER * LT; i += kThreads) s_w[i] = 0;
  __syncthreads();
  uint8_t* my_w = s_w + warp * SER * LT;

  constexpr int V = SER * LT;
  constexpr int VPL = V >= 32 ? V / 32 : 1;
  constexpr int G = V >= 32 ? 1 : 32 / V;

  for (int64_t r0 = ((int64_t)blockIdx.x * 8 + warp) * SER; r0 < N; r0 += (int64_t)gridDim.x * 8 * SER) {
    float4 x[SER][NF];
#pragma unroll
    for (int s = 0; s < SER; ++s) {
      const int64_t row = r0 + s;
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        const int fi = lane + 32 * f;
        x[s][f] = (row < N && fi < nf4) ? ld_stream(reinterpret_cast<const float4*>(X + row * len) + fi)
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    float muf[SER];
    double inv[SER];
#pragma unroll
    for (int s = 0; s < SER; ++s) {
      double mu64;
      row_stats<NF>(x[s], nf4, len, muf[s], mu64, inv[s]);
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        x[s][f].x = __fsub_rn(x[s][f].x, muf[s]);
        x[s][f].y = __fsub_rn(x[s][f].y, muf[s]);
        x[s][f].z = __fsub_rn(x[s][f].z, muf[s]);
        x[s][f].w = __fsub_rn(x[s][f].w, muf[s]);
      }
    }
    float acc[V];
#pragma unroll
    for (int i = 0; i < V; ++i) acc[i] = 0.f;
#pragma unroll
    for (int f = 0; f < NF; ++f) {
      const int fi = lane + 32 * f;
      if (fi < nf4) {
#pragma unroll
        for (int j = 0; j < LT; ++j) {
          const float4 b = bas[j * nf4 + fi];
#pragma unroll
          for (int s = 0; s < SER; ++s) {
            float a = acc[s * LT + j];
            a = fmaf(x[s][f].x, b.x, a);
            a = fmaf(x[s][f].y, b.y, a);
            a = fmaf(x[s][f].z, b.z, a);
            a = fmaf(x[s][f].w, b.w, a);
            acc[s * LT + j] = a;
          }
        }
      }
    }
    reduce_scatter<V>(acc, lane);
    if (lane % G == 0) {
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        const int idx = V >= 32 ? lane * VPL + i : lane / G;
        const int s = idx / LT, j = idx % LT;
        const int64_t row = r0 + s;
        double is = inv[0];
#pragma unroll
        for (int t = 1; t < SER; ++t)
          if (s == t) is = inv[t];
        if (row < N && j < l) {
          const double v = (double)acc[i] * is;
          if (vals) vals[row * l + j] = v;
          my_w[s * LT + j] = (uint8_t)bin_of(s_edges + j * 256, v);
        }
      }
    }
    __syncwarp();
#pragma unroll
    for (int s = 0; s < SER; ++s) {
      if (lane == s && r0 + s < N) {
        if (stats) stats[r0 + s] = make_float2(muf[s], (float)inv[s]);
        if (keys) keys[r0 + s] = word_key(my_w + s * LT, l, a_bits);
      }
    }
    if (words) {
      const int parts = WS >> 4;
      for (int c = lane; c < SER * parts; c += 32) {
        const int s = c / parts, p = c % parts;
        if (r0 + s < N)
          *reinterpret_cast<uint4*>(words + (r0 + s) * WS + p * 16) =
              *reinterpret_cast<const uint4*>(my_w + s * LT + p * 16);
      }
    }
    if (words_l) {
      for (int c = lane; c < SER * l; c += 32) {
        const int s = c / l, j = c % l;
        if (r0 + s < N) words_l[(r0 + s) * l + j] = my_w[s * LT + j];
      }
    }
    __syncwarp();
  }
}

template <int NF, int LT>
static int launch_transform_t(const float* X, int64_t N, const DevModel& dm, uint8_t* words, float2* stats,
                              uint64_t* keys, double* vals, uint8_t* words_l, cudaStream_t st) {
  constexpr int SER0 = (4 / NF) < 1 ? 1 : (4 / NF);
  constexpr int SER = (64 / LT) < SER0 ? (64 / LT) : SER0;
  auto kern = k_transform<NF, LT, SER>;
  const size_t basis_bytes = (size_t)LT * dm.len * 4;
  const int in_smem = basis_bytes <= 96 * 1024;
  const size_t smem = (in_smem ? basis_bytes : 0) + (size_t)LT * 256 * 4 + 8 * SER * LT;
  SOFA_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t want = (N + 8 * SER - 1) / (8 * SER);
  int grid = (int)(want < (int64_t)sms * 8 ? want : (int64_t)sms * 8);
  if (grid < 1) grid = 1;
  kern<<<grid, kThreads, smem, st>>>(X, N, dm.len, dm.l, dm.a_bits, dm.WS, dm.basis32, dm.edges32, words, stats,
                                     keys, vals, words_l, in_smem);
  SOFA_LAUNCHED();
  return SOFA_OK;
}

int launch_transform(const float* X, int64_t N, const DevModel& dm, uint8_t* words, float2* stats, uint64_t* keys,
                     double* vals, uint8_t* words_l, cudaStream_t st) {
  if (N <= 0) return SOFA_OK;
  const int nf4 = dm.len / 4;
  const int NF = nf4 <= 32 ? 1 : nf4 <= 64 ? 2 : nf4 <= 128 ? 4 : 8;
#define SOFA_TR(nf, lt) \
  if (NF == nf && dm.LT == lt) return launch_transform_t<nf, lt>(X, N, dm, words, stats, keys, vals, words_l, st);
  SOFA_TR(1, 16) SOFA_TR(1, 32) SOFA_TR(1, 64)
  SOFA_TR(2, 16) SOFA_TR(2, 32) SOFA_TR(2, 64)
  SOFA_TR(4, 16) SOFA_TR(4, 32) SOFA_TR(4, 64)
  SOFA_TR(8, 16) SOFA_TR(8, 32) SOFA_TR(8, 64)
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
