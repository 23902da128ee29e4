// C ABI of libsofa (include/sofa.h): argument checks, index construction (a1-a4), query entry
// points (a5-a8), merge (a9).  Host orchestration only — every step of the path runs in the
// kernels of transform.cu / learn.cu / query.cu.
#include <cub/cub.cuh>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace sofa {

std::atomic<int64_t> g_launches{0};
static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

static bool pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }

static int check_shape(int64_t len, int64_t l, int64_t a) {
  if (len < 4 || len > SOFA_MAX_LEN || len % 4 != 0)
    return fail(SOFA_EINVAL, "len must be a multiple of 4 in [4, 1024]");
  if (l < 1 || l > SOFA_MAX_L || l > len - 1) return fail(SOFA_EINVAL, "l must be in [1, min(64, len-1)]");
  if (a < 2 || a > SOFA_MAX_ALPHABET || !pow2(a)) return fail(SOFA_EINVAL, "alphabet must be a power of two in [2, 256]");
  return SOFA_OK;
}

// basis rows for the selected positions: [LT][len], rows >= l are zero
// (iSAX: row j averages PAA segment j)
__global__ void k_basis_sel(const int* __restrict__ pos, int l, int LT, int len, int isax, double* __restrict__ b64,
                            float* __restrict__ b32) {
  const double rs = 1.0 / sqrt((double)len);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < LT * len; i += gridDim.x * blockDim.x) {
    const int j = i / len, t = i % len;
    double v = 0.0;
    if (j < l && isax) {
      const int seg = len / l;
      v = t / seg == pos[j] ? 1.0 / seg : 0.0;
    } else if (j < l) {
      const int k = pos[j] >> 1, im = pos[j] & 1;
      const int m = (int)(((int64_t)k * t) % len);
      double sn, cs;
      sincospi(2.0 * m / len, &sn, &cs);
      v = im ? -sn * rs : cs * rs;
    }
    b64[i] = v;
    b32[i] = (float)v;
  }
}

__global__ void k_iota(int32_t* p, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = (int32_t)i;
}

// Alg. 1 l.2 sample(X, r): rows floor(j * global_n / S) - offset (reading 6)
__global__ void k_gather_sample(const float* __restrict__ X, int64_t S, int64_t gn, int64_t off, int len,
                                float* __restrict__ out) {
  const int64_t tot = S * len;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = i / len, t = i % len;
    const int64_t row = (j * gn) / S - off;
    out[i] = X[row * len + t];
  }
}

int upload_model(const sofa_model& m, int len, sofa_index* ix, cudaStream_t st) {
  const int l = m.l, a = m.alphabet;
  const int LT = l <= 16 ? 16 : l <= 32 ? 32 : 64;
  ix->LT = LT;
  ix->WS = (l + 15) / 16 * 16;
  std::vector<double> e64((size_t)LT * 256, INFINITY);
  std::vector<float> e32((size_t)LT * 256, INFINITY);
  for (int j = 0; j < l; ++j)
    for (int i = 0; i < a - 1; ++i) {
      e64[j * 256 + i] = m.edges[j * 255 + i];
      e32[j * 256 + i] = (float)m.edges[j * 255 + i];
    }
  SOFA_CK(cudaMalloc(&ix->edges64, e64.size() * 8));
  SOFA_CK(cudaMalloc(&ix->edges32, e32.size() * 4));
  SOFA_CK(cudaMalloc(&ix->basis64, (size_t)LT * len * 8));
  SOFA_CK(cudaMalloc(&ix->basis32, (size_t)LT * len * 4));
  SOFA_CK(cudaMemcpyAsync(ix->edges64, e64.data(), e64.size() * 8, cudaMemcpyHostToDevice, st));
  SOFA_CK(cudaMemcpyAsync(ix->edges32, e32.data(), e32.size() * 4, cudaMemcpyHostToDevice, st));
  int* dpos = nullptr;
  SOFA_CK(cudaMalloc(&dpos, SOFA_MAX_L * 4));
  SOFA_CK(cudaMemcpyAsync(dpos, m.best_pos, SOFA_MAX_L * 4, cudaMemcpyHostToDevice, st));
  k_basis_sel<<<(LT * len + 255) / 256, 256, 0, st>>>(dpos, l, LT, len, m.binning == SOFA_BINNING_ISAX ? 1 : 0,
                                                      ix->basis64, ix->basis32);
  cudaError_t e = cudaGetLastError();
  g_launches.fetch_add(1);
  cudaStreamSynchronize(st);
  cudaFree(dpos);
  if (e != cudaSuccess) return fail(SOFA_ECUDA, std::string("k_basis_sel: ") + cudaGetErrorString(e));
  DevModel& dm = ix->dm;
  dm.len = len;
  dm.l = l;
  dm.LT = LT;
  dm.a = a;
  dm.a_bits = 31 - __builtin_clz((unsigned)a);
  dm.WS = ix->WS;
  dm.basis32 = ix->basis32;
  dm.basis64 = ix->basis64;
  dm.edges32 = ix->edges32;
  dm.edges64 = ix->edges64;
  for (int j = 0; j < SOFA_MAX_L; ++j) dm.weights[j] = j < l ? (float)m.weights[j] : 0.f;
  return SOFA_OK;
}

static int validate_model(const sofa_model& m) {
  int rc = check_shape(m.len, m.l, m.alphabet);
  if (rc) return rc;
  if (m.binning == SOFA_BINNING_ISAX && m.len % m.l != 0) return fail(SOFA_EINVAL, "iSAX needs len % l == 0");
  for (int j = 0; j < m.l; ++j) {
    const int lim = m.binning == SOFA_BINNING_ISAX ? m.l : m.len + 2;
    if (m.best_pos[j] < 0 || m.best_pos[j] >= lim) return fail(SOFA_EINVAL, "model best_pos out of range");
    for (int i = 1; i < m.alphabet - 1; ++i)
      if (!(m.edges[j * 255 + i] >= m.edges[j * 255 + i - 1])) return fail(SOFA_EINVAL, "model edges not ascending");
  }
  return SOFA_OK;
}

}  // namespace sofa

using namespace sofa;

extern "C" {

const char* sofa_last_error(void) { return g_err.c_str(); }

int64_t sofa_launch_count(void) { return g_launches.load(); }

int sofa_kernel_timing(sofa_index* ix, int32_t enable, double* out_ms, int64_t* out_groups) {
  g_err.clear();
  if (!ix) return fail(SOFA_EINVAL, "index is NULL");
  // drain what was recorded so far: blocks until the last recorded group has finished
  if (!ix->ktime_pending.empty()) SOFA_CK(cudaEventSynchronize(ix->ktime_pending.back()[4]));
  for (auto& quad : ix->ktime_pending) {
    for (int i = 0; i < 4; ++i) {
      float ms = 0.f;
      SOFA_CK(cudaEventElapsedTime(&ms, quad[i], quad[i + 1]));
      ix->ktime_ms[i] += ms;
    }
    ++ix->ktime_groups;
    ix->ktime_free.push_back(quad);
  }
  ix->ktime_pending.clear();
  if (out_ms)
    for (int i = 0; i < 4; ++i) out_ms[i] = ix->ktime_ms[i];
  if (out_groups) *out_groups = ix->ktime_groups;
  if (enable >= 0) {  // (re)start: clear the totals
    ix->ktime_on = enable != 0;
    for (double& m : ix->ktime_ms) m = 0;
    ix->ktime_groups = 0;
  }
  return SOFA_OK;
}

int sofa_default_tuning(sofa_tuning* out) {
  if (!out) return fail(SOFA_EINVAL, "out is NULL");
  memset(out, 0, sizeof(*out));
  out->front_batches = 0;
  out->rev_rounds = 2;
  out->topm_min = 0;
  out->topm_leaves = 64;
  out->refine_rows_front = 0;
  out->refine_rows_scan = 0;
  out->front_wide = -1;
  out->scan_wide = -1;
  out->dense_cand_cap = 0;
  out->dense_diag = 0;
  out->dense_batch_rows = 0;
  out->dense_pair = 0;
  out->dense_mcast = 1;
  out->scan_fused = 1;
  return SOFA_OK;
}

int sofa_set_tuning(sofa_index* ix, const sofa_tuning* t) {
  g_err.clear();
  if (!ix || !t) return fail(SOFA_EINVAL, "NULL pointer");
  if (t->front_batches < 0) return fail(SOFA_EINVAL, "front_batches must be >= 0");
  if (t->rev_rounds < 0) return fail(SOFA_EINVAL, "rev_rounds must be >= 0");
  if (t->topm_min < 0 || t->topm_leaves < 1 || t->topm_leaves > 2048)
    return fail(SOFA_EINVAL, "topm_min >= 0 and topm_leaves in [1, 2048]");
  for (int r : {t->refine_rows_front, t->refine_rows_scan})
    if (r != 0 && r != 2 && r != 4) return fail(SOFA_EINVAL, "refine_rows must be 0, 2 or 4");
  for (int w : {t->front_wide, t->scan_wide})
    if (w < -1 || w > 1) return fail(SOFA_EINVAL, "front_wide / scan_wide must be -1, 0 or 1");
  if (t->dense_cand_cap < 0) return fail(SOFA_EINVAL, "dense_cand_cap must be >= 0");
  if (t->dense_batch_rows < 0) return fail(SOFA_EINVAL, "dense_batch_rows must be >= 0");
  const bool regrow = t->dense_cand_cap != ix->tune.dense_cand_cap;
  ix->tune = *t;
  if (regrow) free_dense_scratch(ix);  // reallocated at the next sofa_knn with the new capacity
  return SOFA_OK;
}

int sofa_default_opts(sofa_build_opts* out) {
  if (!out) return fail(SOFA_EINVAL, "out is NULL");
  memset(out, 0, sizeof(*out));
  out->sample_ratio = 0.01;
  out->block_size = 256;
  out->binning = SOFA_BINNING_EQUI_DEPTH;
  return SOFA_OK;
}

int sofa_learn_model(const float* sample_dev, int64_t S, int32_t len, int32_t l, int32_t alphabet,
                     const sofa_build_opts* opts, void* cuda_stream, sofa_model* out) {
  g_err.clear();
  int rc = check_shape(len, l, alphabet);
  if (rc) return rc;
  if (!sample_dev || !out) return fail(SOFA_EINVAL, "NULL pointer");
  const int binning = opts ? opts->binning : SOFA_BINNING_EQUI_DEPTH;
  const int cl = opts ? opts->candidate_limit : 0;
  if (binning != SOFA_BINNING_EQUI_DEPTH && binning != SOFA_BINNING_EQUI_WIDTH && binning != SOFA_BINNING_ISAX)
    return fail(SOFA_EINVAL, "binning");
  if (binning == SOFA_BINNING_ISAX) return isax_model(len, l, alphabet, out);
  return learn_model_dev(sample_dev, S, len, l, alphabet, binning, cl, (cudaStream_t)cuda_stream, out);
}

void sofa_free(sofa_index* ix) {
  if (!ix) return;
  free_dense_scratch(ix);
  for (auto* v : {&ix->ktime_pending, &ix->ktime_free})
    for (auto& quad : *v)
      for (auto e : quad) cudaEventDestroy(e);
  void* bufs[] = {ix->qstate, ix->q_T, ix->q_hat, ix->pool, ix->tasks, ix->rank_count, ix->fifo, ix->fifo_seq, ix->fcount, ix->words, ix->stats, ix->stats_orig, ix->perm, ix->env, ix->bkey, ix->xb16, ix->basis32, ix->basis64, ix->edges32,
                  ix->edges64, ix->gscratch, ix->qcounter, ix->dstats, ix->hq_dev, ix->hd_dev, ix->hi_dev,
                  ix->trace};
  for (void* p : bufs)
    if (p) cudaFree(p);
  delete ix;
}

int sofa_build(const float* series_dev, int64_t n, int32_t len, int32_t l, int32_t alphabet,
               const sofa_build_opts* opts_in, void* cuda_stream, sofa_index** out) {
  g_err.clear();
  if (!out) return fail(SOFA_EINVAL, "out is NULL");
  *out = nullptr;
  int rc = check_shape(len, l, alphabet);
  if (rc) return rc;
  sofa_build_opts opts;
  sofa_default_opts(&opts);
  if (opts_in) opts = *opts_in;
  if (n < 0 || (n > 0 && !series_dev)) return fail(SOFA_EINVAL, "bad series / n");
  if (n > 2147483647LL) return fail(SOFA_EINVAL, "n must fit int32 per shard");
  if (!pow2(opts.block_size) || opts.block_size < 32 || opts.block_size > 8192)
    return fail(SOFA_EINVAL, "block_size must be a power of two in [32, 8192]");
  if (opts.binning != SOFA_BINNING_EQUI_DEPTH && opts.binning != SOFA_BINNING_EQUI_WIDTH &&
      opts.binning != SOFA_BINNING_ISAX)
    return fail(SOFA_EINVAL, "binning");
  const int64_t gn = opts.global_n > 0 ? opts.global_n : n;
  if (opts.global_offset < 0 || opts.global_offset + n > gn) return fail(SOFA_EINVAL, "global_offset/global_n");
  cudaStream_t st = (cudaStream_t)cuda_stream;

  sofa_index* ix = new sofa_index();
  ix->n = n;
  ix->len = len;
  ix->l = l;
  ix->a = alphabet;
  ix->B = opts.block_size;
  ix->global_offset = opts.global_offset;
  ix->global_n = gn;
  ix->series = series_dev;
  ix->dense_permille = opts.dense_permille == 0 ? 5 : (opts.dense_permille < 0 ? 0 : opts.dense_permille);
  cudaGetDevice(&ix->device);
  cudaDeviceGetAttribute(&ix->sms, cudaDevAttrMultiProcessorCount, ix->device);
  if (ix->sms < 1) ix->sms = 1;
  sofa_default_tuning(&ix->tune);
  auto bail = [&](int code) {
    sofa_free(ix);
    return code;
  };

  // build-phase timing (Fig. 7 analog): CUDA events on the build stream
  struct Events {
    cudaEvent_t e[5] = {};
    Events() {
      for (auto& x : e) cudaEventCreate(&x);
    }
    ~Events() {
      for (auto& x : e)
        if (x) cudaEventDestroy(x);
    }
  } ev;
  cudaEventRecord(ev.e[0], st);
  // ---- a2: model
  if (opts.model) {
    const sofa_model& m = *opts.model;
    if (m.len != len || m.l != l || m.alphabet != alphabet) return bail(fail(SOFA_EINVAL, "opts->model disagrees with (len, l, alphabet)"));
    if ((rc = validate_model(m))) return bail(rc);
    ix->model = m;
  } else if (opts.binning == SOFA_BINNING_ISAX) {  // static: nothing to learn
    if ((rc = isax_model(len, l, alphabet, &ix->model))) return bail(rc);
  } else {
    if (n == 0) return bail(fail(SOFA_EINVAL, "n = 0 needs opts->model"));
    int64_t S = opts.sample_size > 0 ? opts.sample_size : (int64_t)llround(opts.sample_ratio * (double)gn);
    const int64_t smin = opts.binning == SOFA_BINNING_EQUI_DEPTH ? alphabet : 2;
    if (S < smin) S = smin;
    if (S > gn) S = gn;
    if (opts.binning == SOFA_BINNING_EQUI_DEPTH && S < alphabet)
      return bail(fail(SOFA_EDEGENERATE, "equi-depth binning needs at least `alphabet` rows"));
    // every sampled global row must be local
    if ((0 * gn) / S < opts.global_offset || ((S - 1) * gn) / S >= opts.global_offset + n)
      return bail(fail(SOFA_EINVAL, "sample rows are not all local: pass opts->model for a sharded build"));
    float* smp = nullptr;
    if (cudaMalloc(&smp, (size_t)S * len * 4) != cudaSuccess) return bail(fail(SOFA_ENOMEM, "sample buffer"));
    k_gather_sample<<<148 * 8, 256, 0, st>>>(series_dev, S, gn, opts.global_offset, len, smp);
    g_launches.fetch_add(1);
    rc = learn_model_dev(smp, S, len, l, alphabet, opts.binning, opts.candidate_limit, st, &ix->model);
    cudaStreamSynchronize(st);
    cudaFree(smp);
    if (rc) return bail(rc);
  }
  if ((rc = upload_model(ix->model, len, ix, st))) return bail(rc);
  const int WS = ix->WS, B = ix->B;
  ix->nb = (n + B - 1) / B;
  if (cudaMalloc(&ix->qcounter, 64) != cudaSuccess || cudaMalloc(&ix->dstats, 32 * 8) != cudaSuccess)
    return bail(fail(SOFA_ENOMEM, "counters"));
  if (n == 0) {
    cudaStreamSynchronize(st);
    *out = ix;
    return SOFA_OK;
  }

  // ---- a1 + a3: one pass over the series
  uint8_t* words_u = nullptr;
  float2* stats_u = nullptr;
  uint64_t *keys_u = nullptr, *keys_s = nullptr;
  int32_t* iota = nullptr;
  void* tmp = nullptr;
  auto freeall = [&]() {
    void* ps[] = {words_u, keys_u, keys_s, iota, tmp};
    for (void* p : ps)
      if (p) cudaFree(p);
  };
#define BCK(call)                                                              \
  do {                                                                         \
    cudaError_t e_ = (call);                                                   \
    if (e_ != cudaSuccess) {                                                   \
      freeall();                                                               \
      return bail(fail(e_ == cudaErrorMemoryAllocation ? SOFA_ENOMEM : SOFA_ECUDA, \
                       std::string(#call) + ": " + cudaGetErrorString(e_)));   \
    }                                                                          \
  } while (0)
  BCK(cudaMalloc(&words_u, (size_t)n * WS));
  BCK(cudaMalloc(&stats_u, (size_t)n * 8));
  ix->stats_orig = stats_u;  // (mu, 1/sigma) in original row order, kept for the dense path
  BCK(cudaMalloc(&keys_u, (size_t)n * 8));
  BCK(cudaMalloc(&keys_s, (size_t)n * 8));
  BCK(cudaMalloc(&iota, (size_t)n * 4));
  BCK(cudaMalloc(&ix->perm, (size_t)n * 4));
  BCK(cudaMalloc(&ix->words, (size_t)n * WS));
  BCK(cudaMalloc(&ix->stats, (size_t)n * 8));
  // envelope tree: level 0 = blocks, each level up groups 16 nodes, until <= 2048 nodes remain
  ix->nlev = 1;
  ix->lvl_cnt[0] = ix->nb;
  ix->lvl_off[0] = 0;
  while (ix->lvl_cnt[ix->nlev - 1] > 2048 && ix->nlev < 8) {
    ix->lvl_off[ix->nlev] = ix->lvl_off[ix->nlev - 1] + ix->lvl_cnt[ix->nlev - 1];
    ix->lvl_cnt[ix->nlev] = (ix->lvl_cnt[ix->nlev - 1] + 15) / 16;
    ix->nlev++;
  }
  const int64_t env_nodes = ix->lvl_off[ix->nlev - 1] + ix->lvl_cnt[ix->nlev - 1];
  BCK(cudaMalloc(&ix->env, (size_t)env_nodes * 2 * WS));
  BCK(cudaMalloc(&ix->bkey, (size_t)ix->nb * 8));
  // the dense screen's operand (f1): the z-normalised rows in bfloat16, written by the same pass; if the
  // device cannot hold it the index runs without the dense path (same results, sparse only)
  ix->xb_ld = (len + 7) / 8 * 8;
  if (ix->dense_permille > 0) {
    if (cudaMalloc(&ix->xb16, (size_t)n * ix->xb_ld * 2) != cudaSuccess) {
      cudaGetLastError();
      ix->xb16 = nullptr;
      ix->dense_permille = 0;
    }
  }
  // (the model phase ends where the transform kernel starts: it includes the index allocations above
  // and the transform's host-side setup, which are host-synchronous)
  if ((rc = launch_transform(series_dev, n, ix->dm, ix->model, words_u, stats_u, keys_u, nullptr, nullptr, ix->xb16,
                             st, ev.e[1]))) {
    freeall();
    return bail(rc);
  }
  cudaEventRecord(ev.e[2], st);
  // ---- a4: sort by key (stable: equal keys keep row order), gather, envelopes
  k_iota<<<148 * 8, 256, 0, st>>>(iota, n);
  g_launches.fetch_add(1);
  size_t tb = 0;
  BCK(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys_u, keys_s, iota, ix->perm, (int64_t)n, 0, 64, st));
  BCK(cudaMalloc(&tmp, tb + 16));
  BCK(cub::DeviceRadixSort::SortPairs(tmp, tb, keys_u, keys_s, iota, ix->perm, (int64_t)n, 0, 64, st));
  g_launches.fetch_add(1);
  cudaEventRecord(ev.e[3], st);
  if ((rc = launch_gather(words_u, stats_u, ix->perm, n, WS, ix->words, ix->stats, st)) ||
      (rc = launch_envelopes(ix->words, n, B, WS, keys_s, ix->env, ix->bkey, st))) {
    freeall();
    return bail(rc);
  }
  for (int L = 1; L < ix->nlev; ++L)
    if ((rc = launch_env_up(ix->env + ix->lvl_off[L - 1] * 2 * WS, ix->lvl_cnt[L - 1], WS,
                            ix->env + ix->lvl_off[L] * 2 * WS, st))) {
      freeall();
      return bail(rc);
    }
  cudaEventRecord(ev.e[4], st);
  BCK(cudaStreamSynchronize(st));
#undef BCK
  for (int i = 0; i < 4; ++i) {  // model, transform, sort, gather + envelopes
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ev.e[i], ev.e[i + 1]);
    ix->build_ms[i] = ms;
  }
  freeall();
  *out = ix;
  return SOFA_OK;
}

int sofa_knn(sofa_index* ix, const float* queries_dev, int32_t q, int32_t k, const float* bsf_init_dev,
             float* out_dist_dev, int64_t* out_idx_dev, sofa_knn_stats* stats, void* cuda_stream) {
  g_err.clear();
  if (!ix) return fail(SOFA_EINVAL, "index is NULL");
  if (q < 1) return fail(SOFA_EINVAL, "q must be >= 1");
  if (k < 1 || k > SOFA_MAX_K) return fail(SOFA_EINVAL, "k must be in [1, 128]");
  if (k > ix->global_n) return fail(SOFA_EINVAL, "k exceeds the number of series");
  if (!queries_dev || !out_dist_dev || !out_idx_dev) return fail(SOFA_EINVAL, "NULL pointer");
  cudaStream_t st = (cudaStream_t)cuda_stream;
  if (stats) SOFA_CK(cudaMemsetAsync(ix->dstats, 0, 32 * 8, st));
  ix->trace_on = stats != nullptr;
  if (stats && ix->trace_cap < q) {
    if (ix->trace) cudaFree(ix->trace);
    ix->trace = nullptr;
    SOFA_CK(cudaMalloc(&ix->trace, (size_t)q * SOFA_TRACE_FIELDS * 8));
    ix->trace_cap = q;
  }
  if (stats) ix->trace_q = q;
  int rc;
  const bool dense = ix->n > 0 && ix->dense_permille > 0 && ix->xb16;
  // large batches run as consecutive sub-batches of kQueryBatch queries on the same stream (the scan
  // pool holds one leaf list per query: q x ceil(n/B) entries)
  const int qb_max = q < kQueryBatch ? q : kQueryBatch;
  if (dense && (rc = ensure_dense_scratch(ix, qb_max, k))) return rc;
  // with stats: CUDA events on `st` around each launch group (front, dense screen, dense refine, scan)
  cudaEvent_t ev[5] = {};
  if (stats)
    for (auto& e : ev) SOFA_CK(cudaEventCreate(&e));
  double kms[4] = {0, 0, 0, 0};
  rc = SOFA_OK;
  for (int q0 = 0; q0 < q && !rc; q0 += qb_max) {
    // live timing (sofa_kernel_timing): the same five points, recorded without synchronising
    if (!stats && ix->ktime_on) {
      if (ix->ktime_free.empty()) {
        std::array<cudaEvent_t, 5> quad{};
        for (auto& e : quad) SOFA_CK(cudaEventCreate(&e));
        ix->ktime_free.push_back(quad);
      }
      ix->ktime_pending.push_back(ix->ktime_free.back());
      ix->ktime_free.pop_back();
      for (int i = 0; i < 5; ++i) ev[i] = ix->ktime_pending.back()[i];
    }
    const bool rec = stats || ix->ktime_on;
    const int qb = q - q0 < qb_max ? q - q0 : qb_max;
    const float* Qb = queries_dev + (int64_t)q0 * ix->len;
    const float* Bb = bsf_init_dev ? bsf_init_dev + q0 : nullptr;
    float* Db = out_dist_dev + (int64_t)q0 * k;
    int64_t* Ib = out_idx_dev + (int64_t)q0 * k;
    ix->trace_off = q0;
    if (dense) SOFA_CK(cudaMemsetAsync(ix->dense.counters, 0, (64 + 2048) * 4, st));
    if (rec) cudaEventRecord(ev[0], st);
    if (ix->n == 0) {
      rc = launch_fill_pad(Db, Ib, (int64_t)qb * k, st);
      if (rec) {
        cudaEventRecord(ev[1], st);
        cudaEventRecord(ev[2], st);
        cudaEventRecord(ev[3], st);
      }
    } else {
      // front (per query) -> dense pass for flagged queries if the batch warrants it -> scan tasks
      // (every other leaf chunk of every query, spread over all CTAs); the dense and scan kernels read
      // the batch decision from device counters, so there is no host synchronisation in between
      rc = launch_query(ix, Qb, qb, k, Bb, Db, Ib, st, false);
      if (rec) cudaEventRecord(ev[1], st);
      if (!rc && dense) rc = launch_dense(ix, qb, k, Db, Ib, stats != nullptr, st, rec ? ev[2] : nullptr);
      else if (rec) cudaEventRecord(ev[2], st);
      if (rec) cudaEventRecord(ev[3], st);
      if (!rc) rc = launch_query(ix, Qb, qb, k, Bb, Db, Ib, st, true);
    }
    if (rec) cudaEventRecord(ev[4], st);
    if (stats) {
      cudaEventSynchronize(ev[4]);
      for (int i = 0; i < 4; ++i) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
        kms[i] += ms;
      }
    }
  }
  ix->trace_off = 0;
  if (stats)
    for (auto& e : ev) cudaEventDestroy(e);
  if (rc) return rc;
  if (stats) {
    unsigned long long h[32] = {};
    SOFA_CK(cudaMemcpyAsync(h, ix->dstats, 32 * 8, cudaMemcpyDeviceToHost, st));
    SOFA_CK(cudaStreamSynchronize(st));
    stats->queries = q;
    stats->blocks_total = (int64_t)h[1];
    stats->blocks_survived = (int64_t)h[2];
    stats->words_scanned = (int64_t)h[3];
    stats->candidates = (int64_t)h[4];
    stats->refined = (int64_t)h[5];
    stats->abandoned = (int64_t)h[6];
    stats->env_nodes = (int64_t)h[7];
    stats->list_blocks = (int64_t)h[8];
    stats->rounds = (int64_t)h[9];
    stats->batches = (int64_t)h[10];
    stats->waves = (int64_t)h[11];
    for (int i = 0; i < 4; ++i) stats->phase_cycles[i] = (int64_t)h[12 + i];
    stats->max_query_cycles = (int64_t)h[16];
    stats->max_list_blocks = (int64_t)h[17];
    stats->max_batches = (int64_t)h[18];
    stats->dense_queries = (int64_t)h[19];
    stats->dense_candidates = (int64_t)h[20];
    stats->dense_refined = (int64_t)h[21];
    stats->scan_tasks = (int64_t)h[22];
    stats->scan_queries = (int64_t)h[23];
    stats->kernel_ms[0] = kms[0];
    stats->kernel_ms[1] = kms[1] + kms[2];  // the dense pass: screen + exact refine
    stats->kernel_ms[2] = kms[3];
  }
  return SOFA_OK;
}

int sofa_knn_host(sofa_index* ix, const float* queries_host, int32_t q, int32_t k, float* out_dist_host,
                  int64_t* out_idx_host, sofa_knn_stats* stats, void* cuda_stream) {
  g_err.clear();
  if (!ix || !queries_host || !out_dist_host || !out_idx_host || q < 1 || k < 1 || k > SOFA_MAX_K)
    return fail(SOFA_EINVAL, "bad arguments");
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const int64_t need = (int64_t)q * (ix->len > k ? ix->len : k);
  if (ix->h_cap < need) {
    if (ix->hq_dev) cudaFree(ix->hq_dev);
    if (ix->hd_dev) cudaFree(ix->hd_dev);
    if (ix->hi_dev) cudaFree(ix->hi_dev);
    ix->hq_dev = nullptr;
    ix->hd_dev = nullptr;
    ix->hi_dev = nullptr;
    SOFA_CK(cudaMalloc(&ix->hq_dev, need * 4));
    SOFA_CK(cudaMalloc(&ix->hd_dev, need * 4));
    SOFA_CK(cudaMalloc(&ix->hi_dev, need * 8));
    ix->h_cap = need;
  }
  SOFA_CK(cudaMemcpyAsync(ix->hq_dev, queries_host, (size_t)q * ix->len * 4, cudaMemcpyHostToDevice, st));
  int rc = sofa_knn(ix, ix->hq_dev, q, k, nullptr, ix->hd_dev, ix->hi_dev, stats, cuda_stream);
  if (rc) return rc;
  SOFA_CK(cudaMemcpyAsync(out_dist_host, ix->hd_dev, (size_t)q * k * 4, cudaMemcpyDeviceToHost, st));
  SOFA_CK(cudaMemcpyAsync(out_idx_host, ix->hi_dev, (size_t)q * k * 8, cudaMemcpyDeviceToHost, st));
  SOFA_CK(cudaStreamSynchronize(st));
  return SOFA_OK;
}

int sofa_merge_topk(const float* dist_dev, const int64_t* idx_dev, int32_t parts, int32_t q, int32_t k,
                    float* out_dist_dev, int64_t* out_idx_dev, void* cuda_stream) {
  g_err.clear();
  if (parts < 1 || parts > 64) return fail(SOFA_EINVAL, "parts must be in [1, 64]");
  if (q < 1 || k < 1 || k > SOFA_MAX_K) return fail(SOFA_EINVAL, "bad q / k");
  if (!dist_dev || !idx_dev || !out_dist_dev || !out_idx_dev) return fail(SOFA_EINVAL, "NULL pointer");
  return launch_merge(dist_dev, idx_dev, parts, q, k, out_dist_dev, out_idx_dev, (cudaStream_t)cuda_stream);
}

int sofa_lower_bounds(sofa_index* ix, const float* queries_dev, int32_t q, int64_t m, float* out_lb2_dev,
                      float* out_ed2_dev, int64_t* out_rows_dev, void* cuda_stream) {
  g_err.clear();
  if (!ix || !queries_dev || !out_lb2_dev || !out_ed2_dev || !out_rows_dev) return fail(SOFA_EINVAL, "NULL pointer");
  if (q < 1 || m < 1 || m > ix->n) return fail(SOFA_EINVAL, "need q >= 1 and 1 <= m <= n");
  const bool keep = ix->trace_on;
  ix->trace_on = 0;
  const int rc = launch_query(ix, queries_dev, q, 1, nullptr, nullptr, nullptr, (cudaStream_t)cuda_stream, false, m,
                              out_lb2_dev, out_ed2_dev, out_rows_dev);
  ix->trace_on = keep;
  return rc;
}

int sofa_knn_seed(sofa_index* ix, const float* queries_dev, int32_t q, int32_t k, float* out_bound_dev,
                  void* cuda_stream) {
  g_err.clear();
  if (!ix || !queries_dev || !out_bound_dev) return fail(SOFA_EINVAL, "NULL pointer");
  if (q < 1 || k < 1 || k > SOFA_MAX_K) return fail(SOFA_EINVAL, "need q >= 1 and 1 <= k <= 128");
  cudaStream_t st = (cudaStream_t)cuda_stream;
  if (ix->n == 0) return launch_fill_value(out_bound_dev, q, INFINITY, st);
  const bool keep = ix->trace_on;
  ix->trace_on = 0;
  int rc = SOFA_OK;
  for (int q0 = 0; q0 < q && !rc; q0 += kQueryBatch) {
    const int qb = q - q0 < kQueryBatch ? q - q0 : kQueryBatch;
    rc = launch_query(ix, queries_dev + (int64_t)q0 * ix->len, qb, k, nullptr, nullptr, nullptr, st, false, 0,
                      nullptr, nullptr, nullptr, out_bound_dev + q0);
  }
  ix->trace_on = keep;
  return rc;
}

int sofa_knn_trace(const sofa_index* ix, int64_t* out_host, int32_t q) {
  if (!ix || !out_host) return fail(SOFA_EINVAL, "NULL pointer");
  if (!ix->trace || q != ix->trace_q) return fail(SOFA_EINVAL, "no trace for this q (call sofa_knn with stats first)");
  SOFA_CK(cudaMemcpy(out_host, ix->trace, (size_t)q * SOFA_TRACE_FIELDS * 8, cudaMemcpyDeviceToHost));
  return SOFA_OK;
}

int sofa_get_model(const sofa_index* ix, sofa_model* out) {
  if (!ix || !out) return fail(SOFA_EINVAL, "NULL pointer");
  *out = ix->model;
  return SOFA_OK;
}

int sofa_transform(const float* series_dev, int64_t n, const sofa_model* model, double* out_values_dev,
                   uint8_t* out_words_dev, void* cuda_stream) {
  g_err.clear();
  if (!model || n < 0 || (n > 0 && !series_dev)) return fail(SOFA_EINVAL, "bad arguments");
  int rc = validate_model(*model);
  if (rc) return rc;
  sofa_index tmp;
  cudaStream_t st = (cudaStream_t)cuda_stream;
  rc = upload_model(*model, model->len, &tmp, st);
  if (!rc) rc = launch_transform(series_dev, n, tmp.dm, *model, nullptr, nullptr, nullptr, out_values_dev, out_words_dev, nullptr, st);
  cudaStreamSynchronize(st);
  void* ps[] = {tmp.basis32, tmp.basis64, tmp.edges32, tmp.edges64};
  for (void* p : ps)
    if (p) cudaFree(p);
  return rc;
}

int sofa_dense_dots(const float* rows_dev, int64_t m, int32_t len, const float* queries_dev, int32_t q,
                    float* out_dev, void* cuda_stream) {
  g_err.clear();
  if (!rows_dev || !queries_dev || !out_dev) return fail(SOFA_EINVAL, "NULL pointer");
  if (m < 1 || q < 1 || q > 256) return fail(SOFA_EINVAL, "need m >= 1 and 1 <= q <= 256");
  if (len < 4 || len > SOFA_MAX_LEN || len % 4) return fail(SOFA_EINVAL, "len must be a multiple of 4 in [4, 1024]");
  return dense_dots(rows_dev, m, len, queries_dev, q, out_dev, (cudaStream_t)cuda_stream);
}

int sofa_get_info(const sofa_index* ix, sofa_index_info* out) {
  if (!ix || !out) return fail(SOFA_EINVAL, "NULL pointer");
  out->n = ix->n;
  out->n_blocks = ix->nb;
  out->global_offset = ix->global_offset;
  out->global_n = ix->global_n;
  out->len = ix->len;
  out->l = ix->l;
  out->alphabet = ix->a;
  out->block_size = ix->B;
  out->word_stride = ix->WS;
  for (int i = 0; i < 4; ++i) out->build_ms[i] = ix->build_ms[i];
  out->dense_enabled = ix->dense_permille > 0 && ix->xb16 != nullptr;
  return SOFA_OK;
}

int sofa_export_index(const sofa_index* ix, uint8_t* words_sorted_dev, int32_t* perm_dev, uint8_t* env_dev,
                      uint64_t* block_keys_dev, void* cuda_stream) {
  if (!ix) return fail(SOFA_EINVAL, "NULL index");
  cudaStream_t st = (cudaStream_t)cuda_stream;
  if (ix->n == 0) return SOFA_OK;
  if (words_sorted_dev)
    SOFA_CK(cudaMemcpyAsync(words_sorted_dev, ix->words, (size_t)ix->n * ix->WS, cudaMemcpyDeviceToDevice, st));
  if (perm_dev) SOFA_CK(cudaMemcpyAsync(perm_dev, ix->perm, (size_t)ix->n * 4, cudaMemcpyDeviceToDevice, st));
  if (env_dev)
    SOFA_CK(cudaMemcpyAsync(env_dev, ix->env, (size_t)ix->nb * 2 * ix->WS, cudaMemcpyDeviceToDevice, st));
  if (block_keys_dev)
    SOFA_CK(cudaMemcpyAsync(block_keys_dev, ix->bkey, (size_t)ix->nb * 8, cudaMemcpyDeviceToDevice, st));
  SOFA_CK(cudaStreamSynchronize(st));
  return SOFA_OK;
}

}  // extern "C"
