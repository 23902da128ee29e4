// a2: MCB learning (Alg. 1) on the GPU, float64 and deterministic.
//
//   k_sample_stats  z-norm statistics of the S sampled rows (Def. 2, float64)
//   k_dft_gemm      full orthonormal DFT at the eligible positions = [S x n] x [n x P] float64
//                   GEMM (Alg. 1 l.3), written transposed (P x S) so each position is one row
//   k_col_stats     per position: mean, sample variance (ddof=1), min, max with a fixed-order
//                   block reduction (bit-reproducible run to run)               (Alg. 1 l.5)
//   k_select        best_l = rank by (variance desc, position asc) < l
//   CUB segmented radix sort of the l selected rows + k_pick_edges (equi-depth, reading 8) or
//   k_equi_width (Alg. 1 l.8-11)
// float64 because the variance ordering of high-frequency data has relative gaps down to 3e-5
// (SURVEY SIM-8) — float32 would flip the selection.  Runs once per index build.
#include <cub/cub.cuh>

#include <vector>

#include "common.cuh"

namespace sofa {

__global__ void k_sample_stats(const float* __restrict__ X, int64_t S, int len, double* __restrict__ mu,
                               double* __restrict__ inv) {
  const int lane = threadIdx.x & 31;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < S;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const float* x = X + r * len;
    double s = 0.0;
    for (int t = lane; t < len; t += 32) s += (double)x[t];
    const double m = warp_sum_f64(s) / len;
    double v = 0.0;
    for (int t = lane; t < len; t += 32) {
      const double d = (double)x[t] - m;
      v += d * d;
    }
    const double sd = sqrt(warp_sum_f64(v) / len);
    if (lane == 0) {
      mu[r] = m;
      inv[r] = sd < 1e-12 ? 0.0 : 1.0 / sd;
    }
  }
}

// basis for the eligible positions: Bm[t][p] = cos(2 pi k t/n)/sqrt(n) (Re) or -sin(...)/sqrt(n) (Im)
__global__ void k_basis_eligible(const int* __restrict__ pos, int P, int len, double* __restrict__ Bm) {
  const double rs = 1.0 / sqrt((double)len);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)len * P;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(i / P), p = (int)(i % P);
    const int k = pos[p] >> 1, im = pos[p] & 1;
    const int m = (int)(((int64_t)k * t) % len);
    double sn, cs;
    sincospi(2.0 * m / len, &sn, &cs);
    Bm[i] = im ? -sn * rs : cs * rs;
  }
}

// C^T[p][s] = sum_t ((x[s][t] - mu[s]) * inv[s]) * Bm[t][p]; 64x64 tile, 4x4 per thread.
__global__ void __launch_bounds__(256) k_dft_gemm(const float* __restrict__ X, const double* __restrict__ mu,
                                                  const double* __restrict__ inv, int64_t S, int len,
                                                  const double* __restrict__ Bm, int P, double* __restrict__ CT) {
  __shared__ double As[16][64 + 1];
  __shared__ double Bs[16][64 + 1];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t s0 = (int64_t)blockIdx.x * 64;
  const int p0 = blockIdx.y * 64;
  double acc[4][4] = {};
  for (int k0 = 0; k0 < len; k0 += 16) {
    for (int e = tid; e < 16 * 64; e += 256) {
      const int kk = e & 15, ss = e >> 4;  // A tile: row ss, col kk
      const int64_t s = s0 + ss;
      const int t = k0 + kk;
      As[kk][ss] = (s < S && t < len) ? ((double)X[s * len + t] - mu[s]) * inv[s] : 0.0;
      const int pp = e & 63, k2 = e >> 6;  // B tile: row k2, col pp
      const int t2 = k0 + k2;
      Bs[k2][pp] = (t2 < len && p0 + pp < P) ? Bm[(int64_t)t2 * P + p0 + pp] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][tx * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][ty * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int p = p0 + ty * 4 + j;
    if (p >= P) continue;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t s = s0 + tx * 4 + i;
      if (s < S) CT[(int64_t)p * S + s] = acc[i][j];
    }
  }
}

// one CTA per position: mean, sample variance (ddof=1), min, max — fixed-order reduction
__global__ void __launch_bounds__(256) k_col_stats(const double* __restrict__ CT, int64_t S,
                                                   double* __restrict__ var, double* __restrict__ mn,
                                                   double* __restrict__ mx) {
  __shared__ double red[256];
  __shared__ double red2[256];
  const int p = blockIdx.x, tid = threadIdx.x;
  const double* c = CT + (int64_t)p * S;
  double s = 0.0, lo = INFINITY, hi = -INFINITY;
  for (int64_t i = tid; i < S; i += 256) {
    const double v = c[i];
    s += v;
    lo = fmin(lo, v);
    hi = fmax(hi, v);
  }
  red[tid] = s;
  __syncthreads();
  for (int o = 128; o >= 1; o >>= 1) {
    if (tid < o) red[tid] += red[tid + o];
    __syncthreads();
  }
  const double mean = red[0] / (double)S;
  __syncthreads();
  double q = 0.0;
  for (int64_t i = tid; i < S; i += 256) {
    const double d = c[i] - mean;
    q += d * d;
  }
  red[tid] = q;
  red2[tid] = lo;
  __syncthreads();
  for (int o = 128; o >= 1; o >>= 1) {
    if (tid < o) {
      red[tid] += red[tid + o];
      red2[tid] = fmin(red2[tid], red2[tid + o]);
    }
    __syncthreads();
  }
  if (tid == 0) {
    var[p] = S > 1 ? red[0] / (double)(S - 1) : 0.0;
    mn[p] = red2[0];
  }
  __syncthreads();
  red2[tid] = hi;
  __syncthreads();
  for (int o = 128; o >= 1; o >>= 1) {
    if (tid < o) red2[tid] = fmax(red2[tid], red2[tid + o]);
    __syncthreads();
  }
  if (tid == 0) mx[p] = red2[0];
}

// best_l: rank(p) = #{q : var_q > var_p or (var_q == var_p and pos_q < pos_p)}
__global__ void k_select(const double* __restrict__ var, const int* __restrict__ pos, int P, int l,
                         int* __restrict__ best_col, int* __restrict__ best_pos) {
  for (int p = threadIdx.x; p < P; p += blockDim.x) {
    int r = 0;
    const double vp = var[p];
    for (int q = 0; q < P; ++q) r += (var[q] > vp) || (var[q] == vp && pos[q] < pos[p]);
    if (r < l) {
      best_col[r] = p;
      best_pos[r] = pos[p];
    }
  }
}

__global__ void k_copy_cols(const double* __restrict__ CT, int64_t S, const int* __restrict__ best_col, int l,
                            double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)l * S;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(i / S);
    out[i] = CT[(int64_t)best_col[j] * S + (i % S)];
  }
}

// equi-depth (reading 8): beta_j(i) = sorted_j[ceil(i*S/a)], i = 1..a-1
__global__ void k_pick_edges(const double* __restrict__ sorted, int64_t S, int l, int a, double* __restrict__ edges) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < l * (a - 1); e += gridDim.x * blockDim.x) {
    const int j = e / (a - 1), i = e % (a - 1) + 1;
    const int64_t r = ((int64_t)i * S + a - 1) / a;
    edges[e] = sorted[(int64_t)j * S + r];
  }
}

// equi-width (Alg. 1 l.8-11): lo + i*(hi-lo)/a
__global__ void k_equi_width(const double* __restrict__ mn, const double* __restrict__ mx,
                             const int* __restrict__ best_col, int l, int a, double* __restrict__ edges) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < l * (a - 1); e += gridDim.x * blockDim.x) {
    const int j = e / (a - 1), i = e % (a - 1) + 1;
    const double lo = mn[best_col[j]], hi = mx[best_col[j]];
    edges[e] = lo + i * (hi - lo) / a;
  }
}

namespace {
struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};
}  // namespace

int learn_model_dev(const float* sample, int64_t S, int len, int l, int a, int binning, int cand_limit,
                    cudaStream_t st, sofa_model* out) {
  // eligible positions (reading 3): Re/Im of k = 1..(n-1)/2, Re of Nyquist for even n
  std::vector<int> pos;
  for (int k = 1; k <= len / 2; ++k) {
    if (cand_limit > 0 && k > cand_limit) break;
    if (len % 2 == 0 && k == len / 2) {
      pos.push_back(2 * k);
    } else {
      pos.push_back(2 * k);
      pos.push_back(2 * k + 1);
    }
  }
  const int P = (int)pos.size();
  if (l > P) {
    set_error("l exceeds the number of eligible Fourier positions");
    return SOFA_EINVAL;
  }
  if (binning == SOFA_BINNING_EQUI_DEPTH && S < a) {
    set_error("equi-depth binning needs a sample of at least `alphabet` rows");
    return SOFA_EDEGENERATE;
  }
  if (S < 2) {
    set_error("sample must hold at least 2 rows");
    return SOFA_EDEGENERATE;
  }
  DevBuf d_mu, d_inv, d_pos, d_B, d_CT, d_var, d_mn, d_mx, d_bc, d_bp, d_cols, d_sorted, d_edges, d_tmp;
  SOFA_CK(cudaMalloc(&d_mu.p, S * 8));
  SOFA_CK(cudaMalloc(&d_inv.p, S * 8));
  SOFA_CK(cudaMalloc(&d_pos.p, P * 4));
  SOFA_CK(cudaMalloc(&d_B.p, (size_t)len * P * 8));
  SOFA_CK(cudaMalloc(&d_CT.p, (size_t)P * S * 8));
  SOFA_CK(cudaMalloc(&d_var.p, P * 8));
  SOFA_CK(cudaMalloc(&d_mn.p, P * 8));
  SOFA_CK(cudaMalloc(&d_mx.p, P * 8));
  SOFA_CK(cudaMalloc(&d_bc.p, l * 4));
  SOFA_CK(cudaMalloc(&d_bp.p, l * 4));
  SOFA_CK(cudaMalloc(&d_edges.p, (size_t)l * (a - 1) * 8 + 8));
  SOFA_CK(cudaMemcpyAsync(d_pos.p, pos.data(), P * 4, cudaMemcpyHostToDevice, st));

  int grid = (int)((S * 32 + 255) / 256);
  if (grid > 148 * 16) grid = 148 * 16;
  k_sample_stats<<<grid, 256, 0, st>>>(sample, S, len, (double*)d_mu.p, (double*)d_inv.p);
  SOFA_LAUNCHED();
  k_basis_eligible<<<(len * P + 255) / 256, 256, 0, st>>>((int*)d_pos.p, P, len, (double*)d_B.p);
  SOFA_LAUNCHED();
  dim3 g2((unsigned)((S + 63) / 64), (unsigned)((P + 63) / 64));
  k_dft_gemm<<<g2, 256, 0, st>>>(sample, (double*)d_mu.p, (double*)d_inv.p, S, len, (double*)d_B.p, P,
                                 (double*)d_CT.p);
  SOFA_LAUNCHED();
  k_col_stats<<<P, 256, 0, st>>>((double*)d_CT.p, S, (double*)d_var.p, (double*)d_mn.p, (double*)d_mx.p);
  SOFA_LAUNCHED();
  k_select<<<1, 256, 0, st>>>((double*)d_var.p, (int*)d_pos.p, P, l, (int*)d_bc.p, (int*)d_bp.p);
  SOFA_LAUNCHED();
  if (a > 1) {
    if (binning == SOFA_BINNING_EQUI_DEPTH) {
      SOFA_CK(cudaMalloc(&d_cols.p, (size_t)l * S * 8));
      SOFA_CK(cudaMalloc(&d_sorted.p, (size_t)l * S * 8));
      k_copy_cols<<<148 * 8, 256, 0, st>>>((double*)d_CT.p, S, (int*)d_bc.p, l, (double*)d_cols.p);
      SOFA_LAUNCHED();
      std::vector<int64_t> offs(l + 1);
      for (int j = 0; j <= l; ++j) offs[j] = (int64_t)j * S;
      DevBuf d_offs;
      SOFA_CK(cudaMalloc(&d_offs.p, (l + 1) * 8));
      SOFA_CK(cudaMemcpyAsync(d_offs.p, offs.data(), (l + 1) * 8, cudaMemcpyHostToDevice, st));
      size_t tmp_bytes = 0;
      const int64_t* ob = (const int64_t*)d_offs.p;
      SOFA_CK(cub::DeviceSegmentedRadixSort::SortKeys(nullptr, tmp_bytes, (const double*)d_cols.p,
                                                      (double*)d_sorted.p, (int64_t)l * S, l, ob, ob + 1, 0, 64,
                                                      st));
      SOFA_CK(cudaMalloc(&d_tmp.p, tmp_bytes + 16));
      SOFA_CK(cub::DeviceSegmentedRadixSort::SortKeys(d_tmp.p, tmp_bytes, (const double*)d_cols.p,
                                                      (double*)d_sorted.p, (int64_t)l * S, l, ob, ob + 1, 0, 64,
                                                      st));
      g_launches.fetch_add(1);
      k_pick_edges<<<(l * (a - 1) + 255) / 256, 256, 0, st>>>((double*)d_sorted.p, S, l, a, (double*)d_edges.p);
      SOFA_LAUNCHED();
      // the offsets buffer must outlive the async sort
      SOFA_CK(cudaStreamSynchronize(st));
    } else {
      k_equi_width<<<(l * (a - 1) + 255) / 256, 256, 0, st>>>((double*)d_mn.p, (double*)d_mx.p, (int*)d_bc.p, l,
                                                              a, (double*)d_edges.p);
      SOFA_LAUNCHED();
    }
  }
  std::vector<int> bp(l);
  std::vector<double> edges((size_t)l * (a - 1) + 1);
  SOFA_CK(cudaMemcpyAsync(bp.data(), d_bp.p, l * 4, cudaMemcpyDeviceToHost, st));
  SOFA_CK(cudaMemcpyAsync(edges.data(), d_edges.p, (size_t)l * (a - 1) * 8, cudaMemcpyDeviceToHost, st));
  SOFA_CK(cudaStreamSynchronize(st));
  memset(out, 0, sizeof(*out));
  out->len = len;
  out->l = l;
  out->alphabet = a;
  out->binning = binning;
  for (int j = 0; j < l; ++j) {
    out->best_pos[j] = bp[j];
    const int k = bp[j] >> 1;
    out->weights[j] = (k == 0 || (len % 2 == 0 && k == len / 2)) ? 1.0 : 2.0;
    for (int i = 0; i < a - 1; ++i) out->edges[j * 255 + i] = edges[(size_t)j * (a - 1) + i];
  }
  return SOFA_OK;
}

// Standard normal quantile Phi^-1(p): Acklam's rational approximation refined by two Halley steps on
// erfc (double precision).
static double norm_ppf(double p) {
  static const double a[] = {-3.969683028665376e+01, 2.209460984245205e+02, -2.759285104469687e+02,
                             1.383577518672690e+02, -3.066479806614716e+01, 2.506628277459239e+00};
  static const double b[] = {-5.447609879822406e+01, 1.615858368580409e+02, -1.556989798598866e+02,
                             6.680131188771972e+01, -1.328068155288572e+01};
  static const double c[] = {-7.784894002430293e-03, -3.223964580411365e-01, -2.400758277161838e+00,
                             -2.549732539343734e+00, 4.374664141464968e+00, 2.938163982698783e+00};
  static const double d[] = {7.784695709041462e-03, 3.224671290700398e-01, 2.445134137142996e+00,
                             3.754408661907416e+00};
  double x;
  if (p < 0.02425) {
    const double q = std::sqrt(-2 * std::log(p));
    x = (((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
        ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1);
  } else if (p > 1 - 0.02425) {
    const double q = std::sqrt(-2 * std::log(1 - p));
    x = -(((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
        ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1);
  } else {
    const double q = p - 0.5, r = q * q;
    x = (((((a[0] * r + a[1]) * r + a[2]) * r + a[3]) * r + a[4]) * r + a[5]) * q /
        (((((b[0] * r + b[1]) * r + b[2]) * r + b[3]) * r + b[4]) * r + 1);
  }
  for (int it = 0; it < 2; ++it) {
    const double e = 0.5 * std::erfc(-x / std::sqrt(2.0)) - p;
    const double u = e * std::sqrt(2 * M_PI) * std::exp(x * x / 2);
    x = x - u / (1 + x * u / 2);
  }
  return x;
}

// The iSAX baseline: l PAA segments of n/l values, breakpoints beta_i = Phi^-1(i/a)
// (equal-depth under N(0,1)), mindist weight n/l (PAA lower-bounds ED by Cauchy-Schwarz per segment).
int isax_model(int len, int l, int a, sofa_model* out) {
  if (len % l != 0) {
    set_error("iSAX needs len % l == 0 (segments of equal length n/l)");
    return SOFA_EINVAL;
  }
  memset(out, 0, sizeof(*out));
  out->len = len;
  out->l = l;
  out->alphabet = a;
  out->binning = SOFA_BINNING_ISAX;
  for (int j = 0; j < l; ++j) {
    out->best_pos[j] = j;
    out->weights[j] = (double)len / l;
    for (int i = 1; i < a; ++i) out->edges[j * 255 + i - 1] = norm_ppf((double)i / a);
  }
  return SOFA_OK;
}

}  // namespace sofa
