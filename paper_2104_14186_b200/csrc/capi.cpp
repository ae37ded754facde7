// C ABI of libqdwhg (include/qdwhg.h): handle, device arena, host/device
// pointer detection, exception -> status mapping, and the thin wrappers that
// stage inputs into padded device buffers, run the device drivers and copy
// results out.  The reference's C++ entry points it replaces are cited in the
// header.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <memory>
#include <tuple>

#include "../../include/qdwhg.h"
#include "dist/dist.hpp"
#include "drivers.hpp"

namespace qdwhg {

// ---------------------------------------------------------------- arena
void func_attr(const void* kern, cudaFuncAttribute attr, int value) {
  static std::mutex mu;
  static std::set<std::tuple<int, const void*, int, int>> done;
  int dev = 0;
  QDWHG_CUDA(cudaGetDevice(&dev));
  const auto key = std::make_tuple(dev, kern, (int)attr, value);
  std::lock_guard<std::mutex> lk(mu);
  if (done.count(key)) return;
  QDWHG_CUDA(cudaFuncSetAttribute(kern, attr, value));
  done.insert(key);
}

int per_device_cached(int slot, int (*probe)()) {
  static std::mutex mu;
  static std::map<std::pair<int, int>, int> cache;
  int dev = 0;
  QDWHG_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find({dev, slot});
  if (it != cache.end()) return it->second;
  const int v = probe();
  cache[{dev, slot}] = v;
  return v;
}

Arena::~Arena() {
  for (auto& c : chunks_) cudaFree(c.base);
}
size_t Arena::reserved() const {
  size_t s = 0;
  for (auto& c : chunks_) s += c.cap;
  return s;
}
void Arena::reserve(size_t bytes) {
  if (reserved() >= bytes) return;
  void* p = nullptr;
  QDWHG_CUDA(cudaMalloc(&p, bytes - reserved()));
  chunks_.push_back({static_cast<char*>(p), bytes - reserved()});
}
void* Arena::alloc_bytes(size_t bytes) {
  bytes = (bytes + 255) & ~size_t(255);
  if (bytes == 0) bytes = 256;
  while (true) {
    if (cur_.chunk < chunks_.size()) {
      Chunk& c = chunks_[cur_.chunk];
      if (cur_.off + bytes <= c.cap) {
        void* p = c.base + cur_.off;
        cur_.off += bytes;
        size_t used = cur_.off;
        for (size_t i = 0; i < cur_.chunk; ++i) used += chunks_[i].cap;
        high_ = std::max(high_, used);
        return p;
      }
      ++cur_.chunk;
      cur_.off = 0;
      continue;
    }
    // grow: new chunk at least 1 GiB or the request
    const size_t cap = std::max<size_t>(bytes, size_t(1) << 30);
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, cap);
    if (e != cudaSuccess) {
      cudaGetLastError();
      throw CapacityError("device workspace exhausted (" + std::to_string(cap >> 20) + " MiB chunk)");
    }
    chunks_.push_back({static_cast<char*>(p), cap});
  }
}
DMat Arena::alloc(int64_t rows, int64_t cols) {
  DMat m;
  m.ld = round_ld(std::max<int64_t>(rows, 1));
  m.rows = rows;
  m.cols = cols;
  m.base = static_cast<double*>(alloc_bytes(sizeof(double) * m.ld * std::max<int64_t>(cols, 1)));
  return m;
}

void Ctx::prof_begin(double flops, const std::string& tag, int kind) {
  ev_tag.resize(ev_used + 1);
  ev_tag[ev_used] = tag;
  ev_kind.resize(ev_used + 1);
  ev_kind[ev_used] = kind;
  if (ev_pool.size() < 2 * (ev_used + 1)) {
    for (int i = 0; i < 512; ++i) {
      cudaEvent_t e;
      QDWHG_CUDA(cudaEventCreate(&e));
      ev_pool.push_back(e);
    }
  }
  ev_flops.resize(ev_used + 1);
  ev_flops[ev_used] = flops;
  QDWHG_CUDA(cudaEventRecord(ev_pool[2 * ev_used], stream));
}
void Ctx::prof_end() {
  QDWHG_CUDA(cudaEventRecord(ev_pool[2 * ev_used + 1], stream));
  ++ev_used;
  if (ev_used >= 4096) prof_collect();  // bound the number of pending events
}
void Ctx::prof_collect() {
  if (ev_used == 0) return;
  QDWHG_CUDA(cudaEventSynchronize(ev_pool[2 * ev_used - 1]));
  static const char* log_path = getenv("QDWHG_PROFILE_LOG");
  FILE* log = log_path ? fopen(log_path, "a") : nullptr;
  // union of the GEMM launch intervals (GEMMs on the main and side streams may
  // run concurrently: the busy time must not count the overlap twice)
  std::vector<std::pair<float, float>> iv;
  for (size_t i = 0; i < ev_used; ++i) {
    if (ev_kind[i] != 0) continue;
    float s = 0.f, e = 0.f;
    QDWHG_CUDA(cudaEventElapsedTime(&s, ev_pool[0], ev_pool[2 * i]));
    QDWHG_CUDA(cudaEventElapsedTime(&e, ev_pool[0], ev_pool[2 * i + 1]));
    iv.emplace_back(s, e);
  }
  std::sort(iv.begin(), iv.end());
  if (!iv.empty()) {
    float cs = iv[0].first, ce = iv[0].second;
    for (size_t i = 1; i < iv.size(); ++i) {
      if (iv[i].first > ce) {
        gemm_busy_ms += ce - cs;
        cs = iv[i].first;
        ce = iv[i].second;
      } else {
        ce = std::max(ce, iv[i].second);
      }
    }
    gemm_busy_ms += ce - cs;
  }
  for (size_t i = 0; i < ev_used; ++i) {
    float ms = 0.f;
    QDWHG_CUDA(cudaEventElapsedTime(&ms, ev_pool[2 * i], ev_pool[2 * i + 1]));
    if (ev_kind[i] == 0) {
      gemm_ms += ms;
      gemm_flops += ev_flops[i];
      ++gemm_timed;
    } else {
      dag_ms += ms;
      dag_flops += ev_flops[i];
      ++dag_timed;
    }
    if (log)
      fprintf(log, "%s ms=%.4f gflop=%.4f tf=%.2f\n", ev_tag[i].c_str(), ms, ev_flops[i] * 1e-9,
              ms > 0 ? ev_flops[i] / ms * 1e-9 : 0.0);
  }
  if (log) fclose(log);
  ev_used = 0;
}


}  // namespace qdwhg

using namespace qdwhg;

namespace qdwhg {
namespace dist {
Engine* make_cuda_engine(qdwhg::Ctx& ctx);
void nccl_unique_id(void* out128);
Comm* nccl_comm_create(const void* uid128, int rank, int world, const Grid& g, void* stream);
}  // namespace dist
}  // namespace qdwhg

// A rank of the distributed driver: its handle (device, stream, arena), the grid
// position, the communicator and the engine, plus the resident input tiles.
struct qdwhg_dist {
  qdwhg_handle* h = nullptr;
  dist::Grid g;
  std::unique_ptr<dist::Comm> comm;
  std::unique_ptr<dist::Engine> eng;
  dist::Ctx dctx;
  // resident input (qdwhg_dist_load): persistent allocation, not arena
  dist::DistMat A;
  double* a_mem = nullptr;
};

struct qdwhg_handle {
  int device = 0;
  cudaStream_t stream = nullptr;
  Arena arena;
  Ctx ctx;
  std::string err;
};

namespace {

template <class F>
qdwhg_status guard(qdwhg_handle* h, F&& f) {
  try {
    if (h) {
      QDWHG_CUDA(cudaSetDevice(h->device));
      h->arena.reset();
    }
    f();
    return QDWHG_OK;
  } catch (const qdwhg::NotPositiveDefinite& e) {
    if (h) h->err = e.what();
    return QDWHG_NOT_POSITIVE_DEFINITE;
  } catch (const qdwhg::NotConverged& e) {
    if (h) h->err = e.what();
    return QDWHG_NOT_CONVERGED;
  } catch (const qdwhg::CapacityError& e) {
    if (h) h->err = e.what();
    return QDWHG_CAPACITY;
  } catch (const qdwhg::CudaError& e) {
    if (h) h->err = e.what();
    return QDWHG_CUDA_ERROR;
  } catch (const qdwhg::NcclError& e) {
    if (h) h->err = e.what();
    return QDWHG_NCCL_ERROR;
  } catch (const std::invalid_argument& e) {
    if (h) h->err = e.what();
    return QDWHG_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    if (h) h->err = e.what();
    return QDWHG_INTERNAL;
  }
}

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

void check_ld(int64_t rows, int64_t ld, const char* what) {
  if (ld < std::max<int64_t>(rows, 1))
    throw InvalidArgument(std::string(what) + ": leading dimension smaller than rows");
}

// Stage a caller matrix (host or device) into a fresh padded device buffer.
DMat stage_in(Ctx& ctx, const double* p, int64_t m, int64_t n, int64_t ld, double* h2d_seconds) {
  DMat d = ctx.arena->alloc(m, n);
  if (m == 0 || n == 0) return d;
  if (is_device_ptr(p)) {
    QDWHG_CUDA(cudaMemcpy2DAsync(d.ptr(), d.ld * 8, p, ld * 8, m * 8, n, cudaMemcpyDeviceToDevice,
                                 ctx.stream));
  } else {
    cudaEvent_t e0, e1;
    if (h2d_seconds) {
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0, ctx.stream);
    }
    QDWHG_CUDA(cudaMemcpy2DAsync(d.ptr(), d.ld * 8, p, ld * 8, m * 8, n, cudaMemcpyHostToDevice,
                                 ctx.stream));
    if (h2d_seconds) {
      cudaEventRecord(e1, ctx.stream);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      *h2d_seconds += ms * 1e-3;
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
    }
  }
  return d;
}

void stage_out(Ctx& ctx, const DMat& d, double* p, int64_t ld) {
  if (!p || d.rows == 0 || d.cols == 0) return;
  const cudaMemcpyKind kind = is_device_ptr(p) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  QDWHG_CUDA(cudaMemcpy2DAsync(p, ld * 8, d.ptr(), d.ld * 8, d.rows * 8, d.cols, kind, ctx.stream));
}

void copy_vec_out(Ctx& ctx, const std::vector<double>& v, double* p) {
  if (!p || v.empty()) return;
  if (is_device_ptr(p))
    QDWHG_CUDA(cudaMemcpyAsync(p, v.data(), v.size() * 8, cudaMemcpyHostToDevice, ctx.stream));
  else
    std::memcpy(p, v.data(), v.size() * 8);
}

void fill_trace(const std::vector<double>& t, int32_t* n, double* dst) {
  *n = (int32_t)std::min<size_t>(t.size(), QDWHG_MAX_TRACE);
  for (int32_t i = 0; i < *n; ++i) dst[i] = t[i];
}

template <class Info>
void finish_clock(StageClock& clk, Info* info, double h2d) {
  double total = 0.0;
  clk.finish(info->stage_seconds, &total);
  info->stage_seconds[7] += h2d;
  info->seconds = total + h2d;
}

}  // namespace

extern "C" {

qdwhg_status qdwhg_create(qdwhg_handle** out, const qdwhg_options* opts) {
  if (!out) return QDWHG_INVALID_ARGUMENT;
  *out = nullptr;
  qdwhg_handle* h = new qdwhg_handle();
  qdwhg_status st = guard(nullptr, [&] {
    int dev = opts ? opts->device : -1;
    if (dev < 0) QDWHG_CUDA(cudaGetDevice(&dev));
    h->device = dev;
    QDWHG_CUDA(cudaSetDevice(dev));
    QDWHG_CUDA(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    int sms = 148;
    QDWHG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    h->ctx.stream = h->stream;
    {
      int least = 0, greatest = 0;
      QDWHG_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
      QDWHG_CUDA(cudaStreamCreateWithPriority(&h->ctx.side, cudaStreamNonBlocking, least));
      QDWHG_CUDA(cudaStreamCreateWithPriority(&h->ctx.hi, cudaStreamNonBlocking, greatest));
    }
    QDWHG_CUDA(cudaEventCreateWithFlags(&h->ctx.ev_main, cudaEventDisableTiming));
    QDWHG_CUDA(cudaEventCreateWithFlags(&h->ctx.ev_side, cudaEventDisableTiming));
    QDWHG_CUDA(cudaEventCreateWithFlags(&h->ctx.ev_side2, cudaEventDisableTiming));
    h->ctx.arena = &h->arena;
    h->ctx.num_sms = sms;
    QDWHG_CUDA(cudaMalloc(&h->ctx.dscratch, 1 << 16));
    QDWHG_CUDA(cudaMallocHost(&h->ctx.hscratch, 1 << 16));
    QDWHG_CUDA(cudaMalloc(&h->ctx.dflag, 256));
    if (opts && opts->arena_bytes) h->arena.reserve(opts->arena_bytes);
    h->ctx.deterministic = opts && (opts->flags & QDWHG_FLAG_DETERMINISTIC);
  });
  if (st != QDWHG_OK) {
    delete h;
    return st;
  }
  *out = h;
  return QDWHG_OK;
}

qdwhg_status qdwhg_destroy(qdwhg_handle* h) {
  if (!h) return QDWHG_OK;
  cudaSetDevice(h->device);
  cudaStreamSynchronize(h->ctx.stream);
  cudaFree(h->ctx.dscratch);
  cudaFreeHost(h->ctx.hscratch);
  cudaFree(h->ctx.dflag);
  cudaStreamSynchronize(h->ctx.side);
  cudaStreamSynchronize(h->ctx.hi);
  cudaStreamDestroy(h->ctx.side);
  cudaStreamDestroy(h->ctx.hi);
  cudaEventDestroy(h->ctx.ev_main);
  cudaEventDestroy(h->ctx.ev_side);
  cudaEventDestroy(h->ctx.ev_side2);
  cudaStreamDestroy(h->stream);
  delete h;
  return QDWHG_OK;
}

const char* qdwhg_last_error(const qdwhg_handle* h) { return h ? h->err.c_str() : ""; }

qdwhg_status qdwhg_get_launch_count(const qdwhg_handle* h, uint64_t* launches) {
  if (!h || !launches) return QDWHG_INVALID_ARGUMENT;
  *launches = h->ctx.gemm_launches + h->ctx.other_launches;
  return QDWHG_OK;
}

qdwhg_status qdwhg_synchronize(qdwhg_handle* h) {
  return guard(h, [&] { QDWHG_CUDA(cudaStreamSynchronize(h->ctx.stream)); });
}

qdwhg_status qdwhg_set_stream(qdwhg_handle* h, void* stream) {
  if (!h) return QDWHG_INVALID_ARGUMENT;
  return guard(h, [&] {
    QDWHG_CUDA(cudaStreamSynchronize(h->ctx.stream));
    h->ctx.stream = stream ? static_cast<cudaStream_t>(stream) : h->stream;
  });
}

qdwhg_status qdwhg_set_deterministic(qdwhg_handle* h, int32_t enable) {
  if (!h) return QDWHG_INVALID_ARGUMENT;
  h->ctx.deterministic = enable != 0;
  return QDWHG_OK;
}

qdwhg_status qdwhg_profile(qdwhg_handle* h, int32_t enable) {
  if (!h) return QDWHG_INVALID_ARGUMENT;
  return guard(h, [&] {
    h->ctx.prof_collect();
    h->ctx.profile = enable != 0;
  });
}

qdwhg_status qdwhg_get_kernel_stats(qdwhg_handle* h, qdwhg_kernel_stats* out) {
  if (!h || !out) return QDWHG_INVALID_ARGUMENT;
  return guard(h, [&] {
    h->ctx.prof_collect();
    out->gemm_launches = h->ctx.gemm_launches;
    out->other_launches = h->ctx.other_launches;
    out->gemm_timed_launches = h->ctx.gemm_timed;
    out->gemm_seconds = h->ctx.gemm_ms * 1e-3;
    out->gemm_flops = h->ctx.gemm_flops;
    out->gemm_busy_seconds = h->ctx.gemm_busy_ms * 1e-3;
    out->dag_timed_launches = h->ctx.dag_timed;
    out->dag_seconds = h->ctx.dag_ms * 1e-3;
    out->dag_flops = h->ctx.dag_flops;
    h->ctx.dag_timed = 0;
    h->ctx.dag_ms = 0.0;
    h->ctx.dag_flops = 0.0;
    h->ctx.gemm_timed = 0;
    h->ctx.gemm_ms = 0.0;
    h->ctx.gemm_busy_ms = 0.0;
    h->ctx.gemm_flops = 0.0;
  });
}

// ---------------------------------------------------------------- drivers
qdwhg_status qdwhg_partial_eig(qdwhg_handle* h, int64_t n, const double* A, int64_t lda,
                               int64_t qdwh_iters, int32_t use_randomization, double tol,
                               uint64_t seed, double* lambda, double* V, int64_t ldv,
                               int64_t k_cap, qdwhg_eig_info* info) {
  if (!h) return QDWHG_INVALID_ARGUMENT;
  return guard(h, [&] {
    if (n < 1 || !A) throw InvalidArgument("qdwh_partial_eig: empty matrix");
    check_ld(n, lda, "qdwh_partial_eig");
    qdwhg_eig_info tmp{};
    qdwhg_eig_info* inf = info ? info : &tmp;
    std::memset(inf, 0, sizeof(*inf));
    const double s = choose_shift((size_t)qdwh_iters);
    Ctx& ctx = h->ctx;
    double h2d = 0.0;
    StageClock clk(ctx);
    DMat Ad = stage_in(ctx, A, n, n, lda, &h2d);
    EigOut r = partial_eig(ctx, Ad, s, (size_t)qdwh_iters, use_randomization != 0, tol, seed, &clk);
    const int64_t k = (int64_t)r.lambda.size();
    if (k > k_cap) throw CapacityError("k exceeds k_cap");
    if (k > 0) {
      copy_vec_out(ctx, r.lambda, lambda);
      check_ld(n, ldv, "V");
      stage_out(ctx, r.V, V, ldv);
    }
    clk.mark(7);
    finish_clock(clk, inf, h2d);
    inf->mu = r.mu;
    inf->shift = r.shift;
    inf->tol = r.tol;
    inf->rank_index = (int64_t)r.rank_index;
    inf->subspace_size = (int64_t)r.subspace_size;
    inf->k = inf->k_found = k;
    inf->iters_qr = (int64_t)r.iters_qr;
    inf->iters_chol = (int64_t)r.iters_chol;
    inf->borderline = (int64_t)r.borderline;
    inf->subspace_path = r.subspace_path;
    inf->no_savings = r.no_savings;
    inf->randomized = r.randomized;
    inf->flops = r.flops;
    fill_trace(r.trace, &inf->n_trace, inf->ell_trace);
  });
}

qdwhg_status qdwhg_partial_eig_request(qdwhg_handle* h, int64_t n, const double* A, int64_t lda,
                               const qdwhg_eig_request* req, double* lambda, double* V,
                               int64_t ldv, int64_t k_cap, qdwhg_eig_info* info) {
  if (!h || !req) return QDWHG_INVALID_ARGUMENT;
  return guard(h, [&] {
    if (n < 1 || !A) throw InvalidArgument("eig_request: empty matrix");
    check_ld(n, lda, "eig_request");
    qdwhg_eig_info tmp{};
    qdwhg_eig_info* inf = info ? info : &tmp;
    std::memset(inf, 0, sizeof(*inf));
    const int iters = req->iters ? req->iters : 3;
    const double s = choose_shift((size_t)iters);
    const double tol = req->tol > 0 ? req->tol : 0.01;
    Ctx& ctx = h->ctx;
    double h2d = 0.0;
    StageClock clk(ctx);
    DMat Ad = stage_in(ctx, A, n, n, lda, &h2d);
    // shift map: LARGEST -> B = cI - A, SMALLEST -> B = A - cI
    double sign = 1.0;
    if (req->which == QDWHG_LARGEST) {
      axpby_identity(ctx, Ad, -1.0, req->c, Ad);
      sign = -1.0;
    } else if (req->which == QDWHG_SMALLEST) {
      axpby_identity(ctx, Ad, 1.0, -req->c, Ad);
    } else if (req->which != QDWHG_NEGATIVE) {
      throw InvalidArgument("eig_request: unknown 'which'");
    }
    EigOut r = partial_eig(ctx, Ad, s, (size_t)iters, req->randomize != 0, tol, req->seed, &clk);
    const double c = (req->which == QDWHG_NEGATIVE) ? 0.0 : req->c;
    int64_t kf = (int64_t)r.lambda.size();
    int64_t k = kf;
    // lambda_B ascending (most negative first) == most extreme of A first
    if (req->k > 0) k = std::min<int64_t>(k, req->k);
    if (k > k_cap) throw CapacityError("k exceeds k_cap");
    std::vector<double> lam(k);
    for (int64_t i = 0; i < k; ++i) lam[i] = (req->which == QDWHG_LARGEST) ? c - r.lambda[i]
                                            : (req->which == QDWHG_SMALLEST) ? c + r.lambda[i]
                                                                             : r.lambda[i];
    (void)sign;
    if (k > 0) {
      copy_vec_out(ctx, lam, lambda);
      check_ld(n, ldv, "V");
      stage_out(ctx, r.V.sub(0, 0, n, k), V, ldv);
    }
    clk.mark(7);
    finish_clock(clk, inf, h2d);
    inf->mu = r.mu;
    inf->shift = r.shift;
    inf->tol = r.tol;
    inf->c_shift = c;
    inf->rank_index = (int64_t)r.rank_index;
    inf->subspace_size = (int64_t)r.subspace_size;
    inf->k = k;
    inf->k_found = kf;
    inf->iters_qr = (int64_t)r.iters_qr;
    inf->iters_chol = (int64_t)r.iters_chol;
    inf->borderline = (int64_t)r.borderline;
    inf->subspace_path = r.subspace_path;
    inf->no_savings = r.no_savings;
    inf->randomized = r.randomized;
    inf->flops = r.flops;
    fill_trace(r.trace, &inf->n_trace, inf->ell_trace);
  });
}

static qdwhg_status svd_common(qdwhg_handle* h, int64_t m, int64_t n, const double* A, int64_t lda,
                               double s, double s_abs, int64_t kreq, double tol, int32_t randomize,
                               uint64_t seed, double* sigma, double* U, int64_t ldu, double* V,
                               int64_t ldv, int64_t k_cap, qdwhg_svd_info* info) {
  if (!h) return QDWHG_INVALID_ARGUMENT;
  return guard(h, [&] {
    if (m < 1 || n < 1 || !A) throw InvalidArgument("qdwh_partial_svd: empty matrix");
    check_ld(m, lda, "qdwh_partial_svd");
    qdwhg_svd_info tmp{};
    qdwhg_svd_info* inf = info ? info : &tmp;
    std::memset(inf, 0, sizeof(*inf));
    Ctx& ctx = h->ctx;
    double h2d = 0.0;
    StageClock clk(ctx);
    DMat Ad = stage_in(ctx, A, m, n, lda, &h2d);
    SvdOut r = partial_svd(ctx, Ad, s, s_abs, tol, randomize != 0, seed, &clk);
    const int64_t kf = (int64_t)r.sigma.size();
    int64_t k = kf;
    if (kreq > 0) k = std::min(k, kreq);
    if (k > k_cap) throw CapacityError("k exceeds k_cap");
    if (k > 0) {
      std::vector<double> sg(r.sigma.begin(), r.sigma.begin() + k);
      copy_vec_out(ctx, sg, sigma);
      if (U) {
        check_ld(m, ldu, "U");
        stage_out(ctx, r.U.sub(0, 0, m, k), U, ldu);
      }
      if (V) {
        check_ld(n, ldv, "V");
        stage_out(ctx, r.V.sub(0, 0, n, k), V, ldv);
      }
    }
    clk.mark(7);
    finish_clock(clk, inf, h2d);
    inf->alpha = r.alpha;
    inf->threshold = r.threshold;
    inf->tol = r.tol;
    inf->cut = r.threshold * r.alpha;
    inf->rank_index = (int64_t)r.rank_index;
    inf->subspace_size = (int64_t)r.subspace_size;
    inf->k = k;
    inf->k_found = kf;
    inf->iters_qr = (int64_t)r.iters_qr;
    inf->iters_chol = (int64_t)r.iters_chol;
    inf->no_savings = r.no_savings;
    inf->randomized = r.randomized;
    inf->flops = r.flops;
    fill_trace(r.trace, &inf->n_trace, inf->ell_trace);
  });
}

qdwhg_status qdwhg_partial_svd(qdwhg_handle* h, int64_t m, int64_t n, const double* A,
                               int64_t lda, double s, double tol, int32_t use_randomization,
                               uint64_t seed, double* sigma, double* U, int64_t ldu, double* V,
                               int64_t ldv, int64_t k_cap, qdwhg_svd_info* info) {
  return svd_common(h, m, n, A, lda, s, 0.0, 0, tol, use_randomization, seed, sigma, U, ldu, V, ldv,
                    k_cap, info);
}

qdwhg_status qdwhg_partial_svd_request(qdwhg_handle* h, int64_t m, int64_t n, const double* A,
                               int64_t lda, const qdwhg_svd_request* req, double* sigma,
                               double* U, int64_t ldu, double* V, int64_t ldv, int64_t k_cap,
                               qdwhg_svd_info* info) {
  if (!req) return QDWHG_INVALID_ARGUMENT;
  const double tol = req->tol > 0 ? req->tol : 0.01;
  if (req->mode == 1) {
    if (!(req->value > 0.0)) {
      if (h) h->err = "svd_request: absolute cut must be positive";
      return QDWHG_INVALID_ARGUMENT;
    }
    return svd_common(h, m, n, A, lda, 0.0, req->value, req->k, tol, req->randomize, req->seed,
                      sigma, U, ldu, V, ldv, k_cap, info);
  }
  return svd_common(h, m, n, A, lda, req->value, 0.0, req->k, tol, req->randomize, req->seed, sigma,
                    U, ldu, V, ldv, k_cap, info);
}

qdwhg_status qdwhg_polar(qdwhg_handle* h, int64_t m, int64_t n, const double* A, int64_t lda,
                         const qdwhg_polar_config* cfg, double* Up, int64_t ldu, double* H,
                         int64_t ldh, qdwhg_polar_info* info) {
  if (!h) return QDWHG_INVALID_ARGUMENT;
  return guard(h, [&] {
    if (m < 1 || n < 1 || !A) throw InvalidArgument("polar_decompose: empty matrix");
    check_ld(m, lda, "polar_decompose");
    Ctx& ctx = h->ctx;
    StageClock clk(ctx);
    DMat Ad = stage_in(ctx, A, m, n, lda, nullptr);
    {
      const MatStats st = mat_stats(ctx, Ad, false);
      if (st.nonfinite > 0) throw InvalidArgument("polar_decompose: non-finite entry");
    }
    PolarCfg pc;
    if (cfg) {
      pc.ell0 = cfg->ell0;
      pc.max_iters = (size_t)cfg->max_iters;
      pc.conv_eps = cfg->conv_eps;
      pc.chol_switch_c = cfg->chol_switch_c;
      pc.force_variant = cfg->force_variant;
    }
    // estimate_ell0: l0 from the R factor of A (no caller-supplied 1/kappa)
    if (cfg && cfg->estimate_ell0) pc.ell0 = polar_ell0_estimate(ctx, Ad);
    DMat Upd = ctx.arena->alloc(m, n);
    DMat Hd = ctx.arena->alloc(n, n);
    PolarOut r = polar_decompose(ctx, Ad, pc, Upd, Hd);
    stage_out(ctx, Upd, Up, ldu);
    stage_out(ctx, Hd, H, ldh);
    clk.mark(7);
    if (info) {
      std::memset(info, 0, sizeof(*info));
      double total = 0;
      clk.finish(nullptr, &total);
      info->seconds = total;
      info->alpha = r.alpha;
      info->iters_qr = (int64_t)r.iters_qr;
      info->iters_chol = (int64_t)r.iters_chol;
      info->converged = 1;
      info->flops = r.flops;
      fill_trace(r.trace, &info->n_trace, info->ell_trace);
    }
    QDWHG_CUDA(cudaStreamSynchronize(ctx.stream));
  });
}

// ---------------------------------------------------------------- pieces
qdwhg_status qdwhg_run_fixed_iterations(qdwhg_handle* h, int64_t m, int64_t n, const double* X0,
                                        int64_t ldx, double ell0, int64_t iters, int32_t variant,
                                        double* X, int64_t ldo, double* trace_out) {
  if (!h) return QDWHG_INVALID_ARGUMENT;
  return guard(h, [&] {
    if (m < 1 || n < 1 || !X0) throw InvalidArgument("run_fixed_iterations: empty matrix");
    Ctx& ctx = h->ctx;
    DMat Xd = stage_in(ctx, X0, m, n, ldx, nullptr);
    if (mat_stats(ctx, Xd, false).nonfinite > 0)
      throw InvalidArgument("run_fixed_iterations: non-finite entry");
    FixedIterResult r = run_fixed_iterations(ctx, Xd, ell0, (size_t)std::max<int64_t>(iters, 0),
                                             variant == 0);
    stage_out(ctx, Xd, X, ldo);
    if (trace_out)
      for (size_t i = 0; i < r.trace.size(); ++i) trace_out[i] = r.trace[i];
    QDWHG_CUDA(cudaStreamSynchronize(ctx.stream));
  });
}

qdwhg_status qdwhg_qdwh_chol_step(qdwhg_handle* h, int64_t m, int64_t n, const double* X,
                                  int64_t ldx, double ell, double* out, int64_t ldo) {
  if (!h) return QDWHG_INVALID_ARGUMENT;
  return guard(h, [&] {
    Ctx& ctx = h->ctx;
    DMat Xd = stage_in(ctx, X, m, n, ldx, nullptr);
    if (mat_stats(ctx, Xd, false).nonfinite > 0) throw InvalidArgument("qdwh_chol_step: non-finite entry");
    DMat Od = ctx.arena->alloc(m, n);
    qdwh_chol_step(ctx, Xd, halley_weights(ell), Od);
    stage_out(ctx, Od, out, ldo);
    QDWHG_CUDA(cudaStreamSynchronize(ctx.stream));
  });
}

qdwhg_status qdwhg_qdwh_qr_step(qdwhg_handle* h, int64_t m, int64_t n, const double* X,
                                int64_t ldx, double ell, double* out, int64_t ldo) {
  if (!h) return QDWHG_INVALID_ARGUMENT;
  return guard(h, [&] {
    Ctx& ctx = h->ctx;
    DMat Xd = stage_in(ctx, X, m, n, ldx, nullptr);
    if (mat_stats(ctx, Xd, false).nonfinite > 0) throw InvalidArgument("qdwh_qr_step: non-finite entry");
    DMat Od = ctx.arena->alloc(m, n);
    qdwh_qr_step(ctx, Xd, halley_weights(ell), Od);
    stage_out(ctx, Od, out, ldo);
    QDWHG_CUDA(cudaStreamSynchronize(ctx.stream));
  });
}

qdwhg_status qdwhg_qr_factor(qdwhg_handle* h, int64_t m, int64_t n, const double* A, int64_t lda,
                             double* Q, int64_t ldq, double* R, int64_t ldr) {
  if (!h) return QDWHG_INVALID_ARGUMENT;
  return guard(h, [&] {
    if (m < 1 || n < 1 || !A) throw InvalidArgument("qr_factor: empty matrix");
    if (m < n) throw InvalidArgument("qr_factor: requires rows >= cols");
    Ctx& ctx = h->ctx;
    DMat Ad = stage_in(ctx, A, m, n, lda, nullptr);
    if (mat_stats(ctx, Ad, false).nonfinite > 0) throw InvalidArgument("qr_factor: non-finite entry");
    QrWork qw;
    geqrf(ctx, Ad, qw);
    if (Q) {
      DMat Qd = ctx.arena->alloc(m, m);
      orgqr_cols(ctx, qw, m, n, 0, Qd);
      stage_out(ctx, Qd, Q, ldq);
    }
    stage_out(ctx, Ad, R, ldr);
    QDWHG_CUDA(cudaStreamSynchronize(ctx.stream));
  });
}

qdwhg_status qdwhg_cholesky(qdwhg_handle* h, int64_t n, const double* Z, int64_t ldz, double* W,
                            int64_t ldw) {
  if (!h) return QDWHG_INVALID_ARGUMENT;
  return guard(h, [&] {
    if (n < 1 || !Z) throw InvalidArgument("cholesky: empty matrix");
    Ctx& ctx = h->ctx;
    DMat Zd = stage_in(ctx, Z, n, n, ldz, nullptr);
    if (mat_stats(ctx, Zd, false).nonfinite > 0) throw InvalidArgument("cholesky: non-finite entry");
    DMat Wi = ctx.arena->alloc(n, n);
    potrf_upper_and_inverse(ctx, Zd, Wi, true);
    stage_out(ctx, Zd, W, ldw);
    QDWHG_CUDA(cudaStreamSynchronize(ctx.stream));
  });
}

qdwhg_status qdwhg_sym_eig_dense(qdwhg_handle* h, int64_t n, const double* S, int64_t lds,
                                 double* values, double* V, int64_t ldv) {
  if (!h) return QDWHG_INVALID_ARGUMENT;
  return guard(h, [&] {
    if (n < 1 || !S) throw InvalidArgument("sym_eig_dense: empty matrix");
    Ctx& ctx = h->ctx;
    DMat Sd = stage_in(ctx, S, n, n, lds, nullptr);
    const MatStats st = mat_stats(ctx, Sd, true);
    if (st.nonfinite > 0) throw InvalidArgument("sym_eig_dense: non-finite entry");
    if (st.asym > 1e3 * (double)n * 2.220446049250313e-16 * std::max(1.0, std::sqrt(st.fro2)))
      throw InvalidArgument("sym_eig_dense: input not symmetric within tolerance");
    DMat Vd = ctx.arena->alloc(n, n);
    std::vector<double> vals;
    syev(ctx, Sd, vals, Vd);
    copy_vec_out(ctx, vals, values);
    stage_out(ctx, Vd, V, ldv);
    QDWHG_CUDA(cudaStreamSynchronize(ctx.stream));
  });
}

qdwhg_status qdwhg_svd_dense(qdwhg_handle* h, int64_t m, int64_t n, const double* A, int64_t lda,
                             double* U, int64_t ldu, double* sigma, double* V, int64_t ldv) {
  if (!h) return QDWHG_INVALID_ARGUMENT;
  return guard(h, [&] {
    if (m < 1 || n < 1 || !A) throw InvalidArgument("svd_dense: empty matrix");
    if (m < n) throw InvalidArgument("svd_dense: requires rows >= cols on the device path");
    Ctx& ctx = h->ctx;
    DMat Ad = stage_in(ctx, A, m, n, lda, nullptr);
    if (mat_stats(ctx, Ad, false).nonfinite > 0) throw InvalidArgument("svd_dense: non-finite entry");
    DMat Ud = ctx.arena->alloc(m, n), Vd = ctx.arena->alloc(n, n);
    std::vector<double> sg;
    svd_polar(ctx, Ad, Ud, sg, Vd);
    copy_vec_out(ctx, sg, sigma);
    stage_out(ctx, Ud, U, ldu);
    stage_out(ctx, Vd, V, ldv);
    QDWHG_CUDA(cudaStreamSynchronize(ctx.stream));
  });
}

qdwhg_status qdwhg_accuracy_report(qdwhg_handle* h, int64_t m, int64_t n, const double* A,
                                   int64_t lda, int64_t k, const double* U, int64_t ldu,
                                   const double* sigma, const double* V, int64_t ldv,
                                   const double* delta, int32_t paper_pairing, qdwhg_accuracy* out) {
  if (!h || !out) return QDWHG_INVALID_ARGUMENT;
  return guard(h, [&] {
    if (m < 1 || n < 1 || !A) throw InvalidArgument("accuracy_report: empty matrix");
    if (k < 0 || (k > 0 && (!U || !V || !sigma))) throw InvalidArgument("accuracy_report: missing factors");
    Ctx& ctx = h->ctx;
    DMat Ad = stage_in(ctx, A, m, n, lda, nullptr);
    const int64_t kk = std::max<int64_t>(k, 1);
    DMat Ud = k > 0 ? stage_in(ctx, U, m, k, ldu, nullptr) : ctx.arena->alloc(m, kk).col_block(0, 0);
    DMat Vd = k > 0 ? stage_in(ctx, V, n, k, ldv, nullptr) : ctx.arena->alloc(n, kk).col_block(0, 0);
    std::vector<double> sg(sigma, sigma + k);
    const AccuracyOut r = accuracy_report(ctx, Ad, Ud, sg, Vd, delta, paper_pairing != 0);
    std::memset(out, 0, sizeof(*out));
    out->orth_left = r.orth_left;
    out->orth_right = r.orth_right;
    out->value_err = r.value_err;
    out->has_value_err = r.has_value_err;
    out->resid_right = r.resid_right;
    out->resid_left = r.resid_left;
    out->n = r.n;
    out->k = r.k;
    QDWHG_CUDA(cudaStreamSynchronize(ctx.stream));
  });
}

qdwhg_status qdwhg_eig_full(qdwhg_handle* h, int64_t n, const double* A, int64_t lda,
                            int64_t base_size, double* lambda, double* V, int64_t ldv, int64_t* depth) {
  if (!h) return QDWHG_INVALID_ARGUMENT;
  return guard(h, [&] {
    if (n < 1 || !A) throw InvalidArgument("qdwh_eig_full: empty matrix");
    Ctx& ctx = h->ctx;
    DMat Ad = stage_in(ctx, A, n, n, lda, nullptr);
    if (mat_stats(ctx, Ad, false).nonfinite > 0) throw InvalidArgument("qdwh_eig_full: non-finite entry");
    DMat Vd = ctx.arena->alloc(n, n);
    std::vector<double> vals;
    const int64_t d = eig_full(ctx, Ad, base_size > 0 ? base_size : 32, vals, Vd);
    copy_vec_out(ctx, vals, lambda);
    stage_out(ctx, Vd, V, ldv);
    if (depth) *depth = d;
    QDWHG_CUDA(cudaStreamSynchronize(ctx.stream));
  });
}

qdwhg_status qdwhg_svd_full(qdwhg_handle* h, int64_t m, int64_t n, const double* A, int64_t lda,
                            int64_t base_size, double* U, int64_t ldu, double* sigma, double* V,
                            int64_t ldv) {
  if (!h) return QDWHG_INVALID_ARGUMENT;
  return guard(h, [&] {
    if (m < 1 || n < 1 || !A) throw InvalidArgument("qdwh_svd_full: empty matrix");
    if (m < n) throw InvalidArgument("qdwh_svd_full: requires rows >= cols");
    Ctx& ctx = h->ctx;
    DMat Ad = stage_in(ctx, A, m, n, lda, nullptr);
    if (mat_stats(ctx, Ad, false).nonfinite > 0) throw InvalidArgument("qdwh_svd_full: non-finite entry");
    DMat Ud = ctx.arena->alloc(m, n), Vd = ctx.arena->alloc(n, n);
    std::vector<double> sg;
    svd_full(ctx, Ad, base_size > 0 ? base_size : 32, Ud, sg, Vd);
    copy_vec_out(ctx, sg, sigma);
    stage_out(ctx, Ud, U, ldu);
    stage_out(ctx, Vd, V, ldv);
    QDWHG_CUDA(cudaStreamSynchronize(ctx.stream));
  });
}

qdwhg_status qdwhg_two_norm_estimate(qdwhg_handle* h, int64_t m, int64_t n, const double* A,
                                     int64_t lda, double* out) {
  if (!h || !out) return QDWHG_INVALID_ARGUMENT;
  return guard(h, [&] {
    if (m < 1 || n < 1 || !A) throw InvalidArgument("two_norm_estimate: empty matrix");
    Ctx& ctx = h->ctx;
    DMat Ad = stage_in(ctx, A, m, n, lda, nullptr);
    if (mat_stats(ctx, Ad, false).nonfinite > 0)
      throw InvalidArgument("two_norm_estimate: non-finite entry");
    *out = two_norm_estimate(ctx, Ad);
  });
}

qdwhg_status qdwhg_lanczos_min_bound(qdwhg_handle* h, int64_t n, const double* A, int64_t lda,
                                     int64_t steps, double* out) {
  if (!h || !out) return QDWHG_INVALID_ARGUMENT;
  return guard(h, [&] {
    if (n < 1 || !A) throw InvalidArgument("lanczos_min_bound: empty matrix");
    Ctx& ctx = h->ctx;
    DMat Ad = stage_in(ctx, A, n, n, lda, nullptr);
    if (mat_stats(ctx, Ad, false).nonfinite > 0)
      throw InvalidArgument("lanczos_min_bound: non-finite entry");
    *out = lanczos_min_bound(ctx, Ad, (int)steps);
  });
}

qdwhg_status qdwhg_gemm(qdwhg_handle* h, int32_t trans_a, int32_t trans_b, int64_t m, int64_t n,
                        int64_t k, double alpha, const double* A, int64_t lda, const double* B,
                        int64_t ldb, double beta, double* C, int64_t ldc) {
  return qdwhg_gemm_ex(h, trans_a, trans_b, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, 0, 0, 0.0);
}

qdwhg_status qdwhg_cholesky_inverse(qdwhg_handle* h, int64_t n, double* Z, int64_t ldz,
                                    double* Winv, int64_t ldwi) {
  if (!h) return QDWHG_INVALID_ARGUMENT;
  return guard(h, [&] {
    if (n < 1 || !Z || !Winv) throw InvalidArgument("cholesky_inverse: empty matrix");
    Ctx& ctx = h->ctx;
    DMat Zd = stage_in(ctx, Z, n, n, ldz, nullptr);
    DMat Wi = ctx.arena->alloc(n, n);
    potrf_upper_and_inverse(ctx, Zd, Wi, true);
    stage_out(ctx, Wi, Winv, ldwi);
    stage_out(ctx, Zd, Z, ldz);  // Z <- W (upper, zeros below)
    QDWHG_CUDA(cudaStreamSynchronize(ctx.stream));
  });
}

qdwhg_status qdwhg_cholesky_inverse_fast(qdwhg_handle* h, int64_t n, const double* Z, int64_t ldz,
                                         double* Winv, int64_t ldwi) {
  if (!h) return QDWHG_INVALID_ARGUMENT;
  return guard(h, [&] {
    if (n < 1 || !Z || !Winv) throw InvalidArgument("cholesky_inverse_fast: empty matrix");
    Ctx& ctx = h->ctx;
    DMat Zd = stage_in(ctx, Z, n, n, ldz, nullptr);  // workspace copy: Z is not modified
    DMat Wi = ctx.arena->alloc(n, n);
    potrf_upper_and_inverse(ctx, Zd, Wi, /*want_w=*/false, /*stable=*/false);
    stage_out(ctx, Wi, Winv, ldwi);
    QDWHG_CUDA(cudaStreamSynchronize(ctx.stream));
  });
}

qdwhg_status qdwhg_subspace_q2(qdwhg_handle* h, int64_t n, double* B, int64_t ldb, double tol,
                               int64_t* ind, int64_t* ell, double* Q2, int64_t ldq, int64_t ell_cap) {
  if (!h || !ind || !ell) return QDWHG_INVALID_ARGUMENT;
  return guard(h, [&] {
    if (n < 1 || !B) throw InvalidArgument("subspace_q2: empty matrix");
    Ctx& ctx = h->ctx;
    DMat Bd = stage_in(ctx, B, n, n, ldb, nullptr);
    // partial.cpp:71-79: Householder QR of B, ind = first |R_ii| < tol, Q2 = Q(:, ind-1:n)
    QrWork qw;
    geqrf(ctx, Bd, qw);
    const size_t i0 = (size_t)first_deficient(ctx, Bd, tol);
    *ind = (int64_t)i0;
    *ell = i0 ? n - (int64_t)i0 + 1 : 0;
    if (i0 == 0) return;
    if (*ell > ell_cap) throw CapacityError("subspace_q2: subspace larger than ell_cap");
    if (!Q2) throw InvalidArgument("subspace_q2: no output buffer");
    DMat Qd = ctx.arena->alloc(n, *ell);
    orgqr_cols(ctx, qw, n, n, (int64_t)i0 - 1, Qd);
    stage_out(ctx, Qd, Q2, ldq);
    QDWHG_CUDA(cudaStreamSynchronize(ctx.stream));
  });
}

qdwhg_status qdwhg_gemm_ex(qdwhg_handle* h, int32_t trans_a, int32_t trans_b, int64_t m, int64_t n,
                           int64_t k, double alpha, const double* A, int64_t lda, const double* B,
                           int64_t ldb, double beta, double* C, int64_t ldc, int32_t krange,
                           int32_t out, double diag_add) {
  if (!h) return QDWHG_INVALID_ARGUMENT;
  return guard(h, [&] {
    if (krange < 0 || krange > 4 || out < 0 || out > 2)
      throw InvalidArgument("qdwhg_gemm_ex: bad krange/out flags");
    GemmExtra ex;
    ex.krange = static_cast<KRange>(krange);
    ex.out = out == 1 ? OutMode::LowerMirror : out == 2 ? OutMode::Lower : OutMode::Full;
    ex.diag_add = diag_add;
    DMat Ad, Bd, Cd;
    Ad.base = const_cast<double*>(A);
    Ad.ld = lda;
    Ad.rows = trans_a ? k : m;
    Ad.cols = trans_a ? m : k;
    Bd.base = const_cast<double*>(B);
    Bd.ld = ldb;
    Bd.rows = trans_b ? n : k;
    Bd.cols = trans_b ? k : n;
    Cd.base = C;
    Cd.ld = ldc;
    Cd.rows = m;
    Cd.cols = n;
    if (!is_device_ptr(A) || !is_device_ptr(B) || !is_device_ptr(C))
      throw InvalidArgument("qdwhg_gemm: operands must be device pointers");
    // TMA needs 16-byte aligned bases and even leading dimensions: stage others
    auto aligned = [](const DMat& d) {
      return (d.ld % 2 == 0) && (reinterpret_cast<uintptr_t>(d.base) % 16 == 0);
    };
    Ctx& ctx = h->ctx;
    if (!aligned(Ad)) Ad = stage_in(ctx, A, Ad.rows, Ad.cols, lda, nullptr);
    if (!aligned(Bd)) Bd = stage_in(ctx, B, Bd.rows, Bd.cols, ldb, nullptr);
    if (!aligned(Cd)) {
      DMat Cs = stage_in(ctx, C, m, n, ldc, nullptr);
      gemm(ctx, trans_a ? Op::T : Op::N, trans_b ? Op::T : Op::N, alpha, Ad, Bd, beta, Cs, ex);
      stage_out(ctx, Cs, C, ldc);
    } else {
      gemm(ctx, trans_a ? Op::T : Op::N, trans_b ? Op::T : Op::N, alpha, Ad, Bd, beta, Cd, ex);
    }
    QDWHG_CUDA(cudaStreamSynchronize(h->ctx.stream));
  });
}

qdwhg_status qdwhg_gaussian_matrix(qdwhg_handle* h, int64_t m, int64_t n, uint64_t seed, double* A,
                                   int64_t lda) {
  if (!h) return QDWHG_INVALID_ARGUMENT;
  return guard(h, [&] {
    if (!is_device_ptr(A)) throw InvalidArgument("qdwhg_gaussian_matrix: A must be a device pointer");
    DMat Ad;
    Ad.base = A;
    Ad.ld = lda;
    Ad.rows = m;
    Ad.cols = n;
    gaussian_fill(h->ctx, Ad, seed);
    QDWHG_CUDA(cudaStreamSynchronize(h->ctx.stream));
  });
}

qdwhg_status qdwhg_halley_weights(double ell, double out5[5]) {
  return guard(nullptr, [&] {
    const WeightStep w = halley_weights(ell);
    out5[0] = w.a;
    out5[1] = w.b;
    out5[2] = w.c;
    out5[3] = w.ell_in;
    out5[4] = w.ell_out;
  });
}

qdwhg_status qdwhg_iterations_to_converge(double ell0, double eps, int64_t max_iters,
                                          int64_t* out) {
  return guard(nullptr, [&] { *out = (int64_t)iterations_to_converge(ell0, eps, (size_t)max_iters); });
}

qdwhg_status qdwhg_choose_shift(int64_t qdwh_iters, double* s) {
  return guard(nullptr, [&] { *s = choose_shift((size_t)qdwh_iters); });
}

// ------------------------------------------------------------------ distributed driver
static qdwhg_status dist_init(qdwhg_dist** out, qdwhg_handle* h, int32_t P, int32_t Q, int32_t nb, int32_t rank,
                              const std::function<dist::Comm*(const dist::Grid&)>& mk) {
  if (!out || !h) return QDWHG_INVALID_ARGUMENT;
  *out = nullptr;
  auto* d = new qdwhg_dist();
  d->h = h;
  const qdwhg_status st = guard(h, [&] {
    if (P < 1 || Q < 1 || rank < 0 || rank >= P * Q) throw InvalidArgument("dist: bad grid / rank");
    if (nb < 32 || nb % 32 != 0) throw InvalidArgument("dist: nb must be a positive multiple of 32");
    d->g.P = P;
    d->g.Q = Q;
    d->g.p = rank / Q;
    d->g.q = rank % Q;
    d->g.nb = nb;
    d->eng.reset(dist::make_cuda_engine(h->ctx));
    d->comm.reset(mk(d->g));
    d->dctx.g = d->g;
    d->dctx.comm = d->comm.get();
    d->dctx.eng = d->eng.get();
  });
  if (st != QDWHG_OK) {
    delete d;
    return st;
  }
  *out = d;
  return QDWHG_OK;
}

qdwhg_status qdwhg_dist_unique_id(void* id128) {
  if (!id128) return QDWHG_INVALID_ARGUMENT;
  return guard(nullptr, [&] { dist::nccl_unique_id(id128); });
}

qdwhg_status qdwhg_dist_create_nccl(qdwhg_dist** d, qdwhg_handle* h, int32_t P, int32_t Q, int32_t nb,
                                    int32_t rank, const void* id128) {
  if (!id128) return QDWHG_INVALID_ARGUMENT;
  return dist_init(d, h, P, Q, nb, rank, [&](const dist::Grid& g) {
    return dist::nccl_comm_create(id128, rank, P * Q, g, h->ctx.stream);
  });
}

qdwhg_status qdwhg_dist_world_create(void** world, int32_t nranks) {
  if (!world || nranks < 1) return QDWHG_INVALID_ARGUMENT;
  *world = dist::loopback_world_create(nranks);
  return QDWHG_OK;
}

qdwhg_status qdwhg_dist_world_destroy(void* world) {
  dist::loopback_world_destroy(static_cast<dist::LoopbackWorld*>(world));
  return QDWHG_OK;
}

qdwhg_status qdwhg_dist_create_loopback(qdwhg_dist** d, qdwhg_handle* h, int32_t P, int32_t Q, int32_t nb,
                                        int32_t rank, void* world) {
  if (!world) return QDWHG_INVALID_ARGUMENT;
  return dist_init(d, h, P, Q, nb, rank, [&](const dist::Grid& g) {
    qdwhg_handle* hh = h;
    return dist::loopback_comm_create(
        static_cast<dist::LoopbackWorld*>(world), rank, g,
        [hh](void* dst, const void* src, size_t bytes) {
          // on the rank's own stream, then waited for: a plain cudaMemcpy from
          // pageable memory may return before the DMA lands, and the rank's
          // non-blocking stream would not be ordered after it
          QDWHG_CUDA(cudaSetDevice(hh->device));
          QDWHG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, hh->ctx.stream));
          QDWHG_CUDA(cudaStreamSynchronize(hh->ctx.stream));
        },
        [hh] {
          QDWHG_CUDA(cudaSetDevice(hh->device));
          QDWHG_CUDA(cudaStreamSynchronize(hh->ctx.stream));
        });
  });
}

qdwhg_status qdwhg_dist_create_callback(qdwhg_dist** d, qdwhg_handle* h, int32_t P, int32_t Q, int32_t nb,
                                        int32_t rank, const qdwhg_comm_callbacks* cb) {
  if (!cb) return QDWHG_INVALID_ARGUMENT;
  static_assert(sizeof(qdwhg_comm_callbacks) == sizeof(dist::CommCallbacks), "callback layout");
  dist::CommCallbacks c;
  std::memcpy(&c, cb, sizeof(c));
  return dist_init(d, h, P, Q, nb, rank, [&](const dist::Grid& g) {
    qdwhg_handle* hh = h;
    return dist::callback_comm_create(c, rank, P * Q, g, [hh] {
      QDWHG_CUDA(cudaSetDevice(hh->device));
      QDWHG_CUDA(cudaStreamSynchronize(hh->ctx.stream));
    });
  });
}

qdwhg_status qdwhg_dist_destroy(qdwhg_dist* d) {
  if (!d) return QDWHG_OK;
  cudaSetDevice(d->h->device);
  cudaStreamSynchronize(d->h->ctx.stream);
  d->comm.reset();
  if (d->a_mem) cudaFree(d->a_mem);
  delete d;
  return QDWHG_OK;
}

qdwhg_status qdwhg_dist_get_stats(const qdwhg_dist* d, uint64_t* collectives, uint64_t* local_gemms) {
  if (!d) return QDWHG_INVALID_ARGUMENT;
  if (collectives) *collectives = d->dctx.collectives;
  if (local_gemms) *local_gemms = d->dctx.gemms;
  return QDWHG_OK;
}

static void dist_load_impl(qdwhg_dist* d, int64_t m, int64_t n, const double* A, int64_t lda) {
  if (m < 1 || n < 1 || !A) throw InvalidArgument("dist_load: empty matrix");
  check_ld(m, lda, "dist_load");
  dist::DistMat X;
  X.m = m;
  X.n = n;
  X.g = &d->dctx.g;
  X.lr = dist::numroc(m, d->g.nb, d->g.p, d->g.P);
  X.lc = dist::numroc(n, d->g.nb, d->g.q, d->g.Q);
  X.ld = round_ld(std::max<int64_t>(X.lr, 1));
  const size_t bytes = sizeof(double) * (size_t)X.ld * (size_t)std::max<int64_t>(X.lc, 1);
  if (d->a_mem && (d->A.ld != X.ld || d->A.lc != X.lc)) {
    QDWHG_CUDA(cudaFree(d->a_mem));
    d->a_mem = nullptr;
  }
  if (!d->a_mem) QDWHG_CUDA(cudaMalloc(&d->a_mem, bytes));
  X.a = d->a_mem;
  d->A = X;
  dist::scatter_from_full(d->dctx, A, lda, !is_device_ptr(A), d->A);
}

qdwhg_status qdwhg_dist_load(qdwhg_dist* d, int64_t m, int64_t n, const double* A, int64_t lda) {
  if (!d) return QDWHG_INVALID_ARGUMENT;
  return guard(d->h, [&] {
    dist_load_impl(d, m, n, A, lda);
    QDWHG_CUDA(cudaStreamSynchronize(d->h->ctx.stream));
  });
}

namespace {
struct DistTimer {
  cudaEvent_t e0, e1;
  cudaStream_t s;
  explicit DistTimer(cudaStream_t st) : s(st) {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
  }
  double stop() {
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms * 1e-3;
  }
  ~DistTimer() {
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
};
}  // namespace

qdwhg_status qdwhg_dist_partial_eig_request(qdwhg_dist* d, int64_t n, const double* A, int64_t lda,
                                            const qdwhg_eig_request* req, double* lambda, double* V,
                                            int64_t ldv, int64_t k_cap, qdwhg_eig_info* info) {
  if (!d || !req) return QDWHG_INVALID_ARGUMENT;
  return guard(d->h, [&] {
    qdwhg_eig_info tmp{};
    qdwhg_eig_info* inf = info ? info : &tmp;
    std::memset(inf, 0, sizeof(*inf));
    Ctx& ctx = d->h->ctx;
    DistTimer tm(ctx.stream);
    if (A) dist_load_impl(d, n, n, A, lda);
    if (!d->a_mem || d->A.m != n || d->A.n != n) throw InvalidArgument("dist eig: no loaded n x n matrix");
    const int iters = req->iters ? req->iters : 3;
    const double s = choose_shift((size_t)iters);
    const double tol = req->tol > 0 ? req->tol : 0.01;
    dist::Ctx& dc = d->dctx;
    // working copy with the shift map: B = cI - A / A - cI / A
    dist::DistMat B = dist::make_dist(*d->eng, dc.g, n, n);
    if (req->which == QDWHG_LARGEST) dist::axpby_identity(dc, &d->A, -1.0, B, 0.0, req->c);
    else if (req->which == QDWHG_SMALLEST) dist::axpby_identity(dc, &d->A, 1.0, B, 0.0, -req->c);
    else if (req->which == QDWHG_NEGATIVE) dist::axpby_identity(dc, &d->A, 1.0, B, 0.0, 0.0);
    else throw InvalidArgument("eig_request: unknown 'which'");
    dist::EigResult r = dist::partial_eig(dc, B, s, (size_t)iters, req->randomize != 0, tol, req->seed);
    const double c = (req->which == QDWHG_NEGATIVE) ? 0.0 : req->c;
    const int64_t kf = (int64_t)r.lambda.size();
    int64_t k = kf;
    if (req->k > 0) k = std::min<int64_t>(k, req->k);
    if (k > k_cap) throw CapacityError("k exceeds k_cap");
    std::vector<double> lam(k);
    for (int64_t i = 0; i < k; ++i)
      lam[i] = (req->which == QDWHG_LARGEST) ? c - r.lambda[i]
               : (req->which == QDWHG_SMALLEST) ? c + r.lambda[i] : r.lambda[i];
    if (k > 0) {
      copy_vec_out(ctx, lam, lambda);
      if (r.V && V) {
        check_ld(n, ldv, "V");
        DMat Vd;
        Vd.base = r.V;
        Vd.ld = r.vld;
        Vd.rows = n;
        Vd.cols = k;
        stage_out(ctx, Vd, V, ldv);
      }
    }
    inf->seconds = tm.stop();
    inf->mu = r.mu;
    inf->shift = s;
    inf->tol = tol;
    inf->c_shift = c;
    inf->rank_index = (int64_t)r.rank_index;
    inf->subspace_size = (int64_t)r.subspace_size;
    inf->k = k;
    inf->k_found = kf;
    inf->iters_chol = (int64_t)r.iters_chol;
    inf->borderline = (int64_t)r.borderline;
    inf->no_savings = r.no_savings;
    inf->randomized = req->randomize != 0;
    inf->flops = r.flops;
    fill_trace(r.trace, &inf->n_trace, inf->ell_trace);
  });
}

qdwhg_status qdwhg_dist_partial_svd_request(qdwhg_dist* d, int64_t m, int64_t n, const double* A, int64_t lda,
                                            const qdwhg_svd_request* req, double* sigma, double* U, int64_t ldu,
                                            double* V, int64_t ldv, int64_t k_cap, qdwhg_svd_info* info) {
  if (!d || !req) return QDWHG_INVALID_ARGUMENT;
  return guard(d->h, [&] {
    qdwhg_svd_info tmp{};
    qdwhg_svd_info* inf = info ? info : &tmp;
    std::memset(inf, 0, sizeof(*inf));
    Ctx& ctx = d->h->ctx;
    DistTimer tm(ctx.stream);
    if (A) dist_load_impl(d, m, n, A, lda);
    if (!d->a_mem || d->A.m != m || d->A.n != n) throw InvalidArgument("dist svd: no loaded m x n matrix");
    const double tol = req->tol > 0 ? req->tol : 0.01;
    double s = 0.0, s_abs = 0.0;
    if (req->mode == 0) s = req->value;
    else if (req->mode == 1) s_abs = req->value;
    else throw InvalidArgument("svd_request: unknown mode");
    if (req->mode == 1 && !(s_abs > 0.0)) throw InvalidArgument("svd_request: cut must be positive");
    dist::SvdResult r = dist::partial_svd(d->dctx, d->A, s, s_abs, tol, req->randomize != 0, req->seed);
    const int64_t kf = (int64_t)r.sigma.size();
    int64_t k = kf;
    if (req->k > 0) k = std::min<int64_t>(k, req->k);
    if (k > k_cap) throw CapacityError("k exceeds k_cap");
    if (k > 0) {
      std::vector<double> sg(r.sigma.begin(), r.sigma.begin() + k);
      copy_vec_out(ctx, sg, sigma);
      if (r.U && U) {
        check_ld(m, ldu, "U");
        DMat Ud;
        Ud.base = r.U;
        Ud.ld = r.uld;
        Ud.rows = m;
        Ud.cols = k;
        stage_out(ctx, Ud, U, ldu);
      }
      if (r.V && V) {
        check_ld(n, ldv, "V");
        DMat Vd;
        Vd.base = r.V;
        Vd.ld = r.vld;
        Vd.rows = n;
        Vd.cols = k;
        stage_out(ctx, Vd, V, ldv);
      }
    }
    inf->seconds = tm.stop();
    inf->alpha = r.alpha;
    inf->threshold = r.threshold;
    inf->tol = tol;
    inf->cut = r.threshold * r.alpha;
    inf->rank_index = (int64_t)r.rank_index;
    inf->subspace_size = (int64_t)r.subspace_size;
    inf->k = k;
    inf->k_found = kf;
    inf->iters_qr = (int64_t)r.iters_qr;
    inf->iters_chol = (int64_t)r.iters_chol;
    inf->no_savings = r.no_savings;
    inf->randomized = req->randomize != 0;
    inf->flops = r.flops;
    fill_trace(r.trace, &inf->n_trace, inf->ell_trace);
  });
}


// ---- distributed building blocks on full matrices (every rank passes the full
// operands; results gathered to rank 0) — the distributed analogues of
// qdwhg_gemm_ex / qdwhg_cholesky_inverse_fast / qdwhg_subspace_q2
namespace {
dist::DistMat dist_scratch(qdwhg_dist* d, int64_t m, int64_t n, const double* full, int64_t ld) {
  dist::DistMat X = dist::make_dist(*d->eng, d->dctx.g, m, n);
  if (full) dist::scatter_from_full(d->dctx, full, ld, !is_device_ptr(full), X);
  return X;
}
void dist_gather_out(qdwhg_dist* d, const dist::DistMat& X, double* out, int64_t ldo) {
  const bool root = d->g.p == 0 && d->g.q == 0;
  double* dst = nullptr;
  int64_t ldd = 0;
  if (root) dst = d->eng->alloc(X.m, X.n, &ldd);
  dist::gather(d->dctx, X, dst, ldd, 0);
  if (root && out) {
    DMat v;
    v.base = dst;
    v.ld = ldd;
    v.rows = X.m;
    v.cols = X.n;
    stage_out(d->h->ctx, v, out, ldo);
    QDWHG_CUDA(cudaStreamSynchronize(d->h->ctx.stream));
  }
}
}  // namespace

qdwhg_status qdwhg_dist_pgemm(qdwhg_dist* d, int32_t ta, int32_t tb, int64_t m, int64_t n, int64_t k, double alpha,
                              const double* A, int64_t lda, const double* B, int64_t ldb, double beta,
                              const double* C0, int64_t ldc0, double* C, int64_t ldc, int32_t flags) {
  if (!d) return QDWHG_INVALID_ARGUMENT;
  return guard(d->h, [&] {
    dist::DistMat Am = dist_scratch(d, ta ? k : m, ta ? m : k, A, lda);
    dist::DistMat Bm = dist_scratch(d, tb ? n : k, tb ? k : n, B, ldb);
    dist::DistMat Cm = dist_scratch(d, m, n, C0, ldc0);
    dist::Structure st;
    st.a_upper = flags & 1;
    st.a_lower = flags & 2;
    st.b_upper = flags & 4;
    st.b_lower = flags & 8;
    st.c_lower = flags & 16;
    dist::pgemm(d->dctx, ta != 0, tb != 0, alpha, dist::whole(Am), dist::whole(Bm), beta, dist::whole(Cm), st);
    dist_gather_out(d, Cm, C, ldc);
  });
}

qdwhg_status qdwhg_dist_cholesky_inverse(qdwhg_dist* d, int64_t n, const double* Z, int64_t ldz, double* Winv,
                                         int64_t ldwi) {
  if (!d) return QDWHG_INVALID_ARGUMENT;
  return guard(d->h, [&] {
    dist::DistMat Zm = dist_scratch(d, n, n, Z, ldz);
    dist::DistMat Wm = dist_scratch(d, n, n, nullptr, 0);
    dist::chol_inv(d->dctx, Zm, Wm);
    dist_gather_out(d, Wm, Winv, ldwi);
  });
}

qdwhg_status qdwhg_dist_qr(qdwhg_dist* d, int64_t m, int64_t n, const double* X, int64_t ldx, int64_t c0,
                           int64_t ell, double* rdiag, double* Q2, int64_t ldq) {
  if (!d) return QDWHG_INVALID_ARGUMENT;
  return guard(d->h, [&] {
    if (c0 < 0 || ell < 1 || c0 + ell > m) throw InvalidArgument("dist_qr: bad column range");
    dist::DistMat Xm = dist_scratch(d, m, n, X, ldx);
    dist::QrDist qr;
    dist::pgeqrf(d->dctx, Xm, qr);
    dist::DistMat Qm = dist_scratch(d, m, ell, nullptr, 0);
    dist::porgqr_cols(d->dctx, qr, c0, Qm);
    dist_gather_out(d, Qm, Q2, ldq);
    if (rdiag) std::memcpy(rdiag, qr.rdiag.data(), sizeof(double) * (size_t)n);
  });
}

}  // extern "C"
