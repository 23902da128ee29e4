// Multithreaded CPU brute-force exact k-NN under z-normalised Euclidean distance, in the style of
// the paper's UCR Suite-P competitor: every thread scans a contiguous segment of the rows
// with an early-abandoning float32 squared distance (chunks of 32 values checked against the
// thread's current k-th best), keeps a per-thread top-k, and the lists are merged at the end.
// A reported CPU BASELINE for bench.py (BASELINE.json north_star "Reporting"), not the oracle and
// not part of the product path.  Rows are z-normalised on the fly from precomputed (mu, 1/sigma).
#include <omp.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <vector>

namespace {
struct Best {
  float d;
  int64_t i;
};
inline bool better(const Best& a, const Best& b) { return a.d < b.d || (a.d == b.d && a.i < b.i); }
inline void insert(std::vector<Best>& h, int k, Best c) {
  if ((int)h.size() == k && !better(c, h.back())) return;
  auto it = std::upper_bound(h.begin(), h.end(), c, better);
  h.insert(it, c);
  if ((int)h.size() > k) h.pop_back();
}
}  // namespace

extern "C" {

// per-row (mu, 1/sigma), population std; 1/sigma = 0 for a constant row
void ucr_row_stats(const float* x, int64_t n, int len, float* mu_inv) {
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < n; ++r) {
    const float* p = x + r * len;
    double s = 0, s2 = 0;
    for (int t = 0; t < len; ++t) s += p[t];
    const double mu = s / len;
    for (int t = 0; t < len; ++t) s2 += (p[t] - mu) * (p[t] - mu);
    const double sd = std::sqrt(s2 / len);
    mu_inv[2 * r] = (float)mu;
    mu_inv[2 * r + 1] = sd < 1e-12 ? 0.f : (float)(1.0 / sd);
  }
}

// k-NN of q z-normalised queries (q x len) over n rows; out: q x k distances (sqrt) and indices
int ucr_knn(const float* x, const float* mu_inv, int64_t n, int len, const float* queries, int q, int k,
            float* out_d, int64_t* out_i, int threads) {
  if (threads > 0) omp_set_num_threads(threads);
  std::vector<float> qh(len);
  for (int qi = 0; qi < q; ++qi) {
    const float* qq = queries + (int64_t)qi * len;
    double s = 0, s2 = 0;
    for (int t = 0; t < len; ++t) s += qq[t];
    const double mu = s / len;
    for (int t = 0; t < len; ++t) s2 += (qq[t] - mu) * (qq[t] - mu);
    const double sd = std::sqrt(s2 / len);
    const float inv = sd < 1e-12 ? 0.f : (float)(1.0 / sd);
    for (int t = 0; t < len; ++t) qh[t] = (float)((qq[t] - mu) * inv);
    const int nt = omp_get_max_threads();
    std::vector<std::vector<Best>> part(nt);
#pragma omp parallel
    {
      const int tid = omp_get_thread_num(), T = omp_get_num_threads();
      const int64_t a = n * tid / T, b = n * (tid + 1) / T;  // contiguous segment per thread
      std::vector<Best>& h = part[tid];
      h.reserve(k + 1);
      float kth = INFINITY;
      for (int64_t r = a; r < b; ++r) {
        const float* p = x + r * len;
        const float m = mu_inv[2 * r], iv = mu_inv[2 * r + 1];
        float d = 0.f;
        bool ab = false;
        for (int t0 = 0; t0 < len; t0 += 32) {  // early abandoning per 32-value chunk
          const int t1 = t0 + 32 < len ? t0 + 32 : len;
          float acc = 0.f;
#pragma omp simd reduction(+ : acc)
          for (int t = t0; t < t1; ++t) {
            const float e = (p[t] - m) * iv - qh[t];
            acc += e * e;
          }
          d += acc;
          if (d > kth) {
            ab = true;
            break;
          }
        }
        if (ab) continue;
        insert(h, k, Best{d, r});
        if ((int)h.size() == k) kth = h.back().d;
      }
    }
    std::vector<Best> all;
    for (auto& h : part) all.insert(all.end(), h.begin(), h.end());
    std::sort(all.begin(), all.end(), better);
    for (int r = 0; r < k; ++r) {
      const bool ok = r < (int)all.size();
      out_d[(int64_t)qi * k + r] = ok ? std::sqrt(all[r].d) : INFINITY;
      out_i[(int64_t)qi * k + r] = ok ? all[r].i : -1;
    }
  }
  return 0;
}
}
