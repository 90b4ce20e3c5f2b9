// capi.cu — host-side plumbing of the C ABI: error strings, device queries,
// the cuBLAS DGEMM comparator (gemm.py:259-262 "native" path) and small host
// helpers.  No kernels of consequence live here.
#include <cublas_v2.h>
#include <stdarg.h>

#include <atomic>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace oz {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

const char* last_error() { return g_err; }

static std::atomic<long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

struct ProfEntry {
  cudaEvent_t a = nullptr, b = nullptr;
  int kind = 0;
  double work = 0.0;
  int sms = 0;  // SMs the launch may use (0: all)
  bool done = false;
};
static std::mutex g_prof_mu;
static bool g_prof_on = false;
static std::vector<ProfEntry> g_prof;
static size_t g_prof_used = 0;

int prof_start(cudaStream_t st) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (!g_prof_on) return -1;
  if (g_prof_used == g_prof.size()) {
    ProfEntry e;
    if (cudaEventCreate(&e.a) != cudaSuccess || cudaEventCreate(&e.b) != cudaSuccess) return -1;
    g_prof.push_back(e);
  }
  const int tag = (int)g_prof_used++;
  g_prof[tag].done = false;
  cudaEventRecord(g_prof[tag].a, st);
  return tag;
}

void prof_stop(int tag, cudaStream_t st, int kind, double work, int sms) {
  if (tag < 0) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  ProfEntry& e = g_prof[tag];
  cudaEventRecord(e.b, st);
  e.kind = kind;
  e.work = work;
  e.sms = sms;
  e.done = true;
}

int sm_count() {
  static std::mutex mu;
  static std::unordered_map<int, int> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
    n = 148;
  cache[dev] = n;
  return n;
}

// One cuBLAS handle per (device, host thread): handles are not thread-safe to
// share while switching streams, and the reference harness may call from a
// thread pool (harness.py:56-72).
// One handle per (device, stream): cuBLAS keeps a per-handle workspace, so
// streams that run concurrently (the LU look-ahead) must not share one.
static cublasHandle_t cublas_handle(cudaStream_t st) {
  static thread_local std::unordered_map<uint64_t, cublasHandle_t> handles;
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t key = ((uint64_t)dev << 56) ^ (uint64_t)(uintptr_t)st;
  auto it = handles.find(key);
  if (it != handles.end()) return it->second;
  cublasHandle_t h = nullptr;
  if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) return nullptr;
  handles[key] = h;
  return h;
}

// sm_target > 0: cuBLAS sizes its grid for that many SMs (the look-ahead's
// side-stream panel must leave the concurrent GEMM's SMs alone).
int dgemm(int transa, int transb, int64_t m, int64_t n, int64_t k, double alpha, const double* a,
          int64_t lda, const double* b, int64_t ldb, double beta, double* c, int64_t ldc,
          cudaStream_t st, int sm_target) {
  if (m == 0 || n == 0) return OZ_OK;
  cublasHandle_t h = cublas_handle(st);
  OZ_REQUIRE(h != nullptr, OZ_CUDA_ERROR, "cublasCreate failed");
  OZ_REQUIRE(cublasSetStream(h, st) == CUBLAS_STATUS_SUCCESS, OZ_CUDA_ERROR,
             "cublasSetStream failed");
  OZ_REQUIRE(cublasSetSmCountTarget(h, sm_target > 0 ? sm_target : 0) == CUBLAS_STATUS_SUCCESS,
             OZ_CUDA_ERROR, "cublasSetSmCountTarget failed");
  cublasStatus_t s = cublasDgemm(h, transa ? CUBLAS_OP_T : CUBLAS_OP_N,
                                 transb ? CUBLAS_OP_T : CUBLAS_OP_N, (int)m, (int)n, (int)k,
                                 &alpha, a, (int)lda, b, (int)ldb, &beta, c, (int)ldc);
  OZ_REQUIRE(s == CUBLAS_STATUS_SUCCESS, OZ_CUDA_ERROR, "cublasDgemm failed (%d)", (int)s);
  return OZ_OK;
}

// B (jb x n) <- L^{-1} B, L unit lower triangular (cuBLAS DTRSM; the wide
// trsm of the LU when OZ_TRSM_CUBLAS=1, tuning A/B against trsm_rec)
int dtrsm_lunit(int64_t jb, int64_t n, const double* l, int64_t ldl, double* b, int64_t ldb,
                cudaStream_t st, int sm_target) {
  if (jb == 0 || n == 0) return OZ_OK;
  cublasHandle_t h = cublas_handle(st);
  OZ_REQUIRE(h != nullptr, OZ_CUDA_ERROR, "cublasCreate failed");
  OZ_REQUIRE(cublasSetStream(h, st) == CUBLAS_STATUS_SUCCESS, OZ_CUDA_ERROR,
             "cublasSetStream failed");
  OZ_REQUIRE(cublasSetSmCountTarget(h, sm_target > 0 ? sm_target : 0) == CUBLAS_STATUS_SUCCESS,
             OZ_CUDA_ERROR, "cublasSetSmCountTarget failed");
  const double one = 1.0;
  cublasStatus_t s = cublasDtrsm(h, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N,
                                 CUBLAS_DIAG_UNIT, (int)jb, (int)n, &one, l, (int)ldl, b,
                                 (int)ldb);
  OZ_REQUIRE(s == CUBLAS_STATUS_SUCCESS, OZ_CUDA_ERROR, "cublasDtrsm failed (%d)", (int)s);
  return OZ_OK;
}

}  // namespace oz

extern "C" const char* oz_last_error(void) { return oz::last_error(); }

extern "C" int oz_version(void) { return 100; }

extern "C" long long oz_launch_count(void) { return oz::g_launches.load(); }

extern "C" int oz_prof_enable(int on) {
  std::lock_guard<std::mutex> lk(oz::g_prof_mu);
  oz::g_prof_on = on != 0;
  oz::g_prof_used = 0;
  return OZ_OK;
}

// Per kind: out[3*kind + {0,1,2}] = {total ms, launches, total work}; syncs events.
extern "C" int oz_prof_summary(double* out) {
  std::lock_guard<std::mutex> lk(oz::g_prof_mu);
  for (int i = 0; i < 3 * oz::PROF_KINDS; ++i) out[i] = 0.0;
  for (size_t i = 0; i < oz::g_prof_used; ++i) {
    oz::ProfEntry& e = oz::g_prof[i];
    if (!e.done) continue;
    if (cudaEventSynchronize(e.b) != cudaSuccess) {
      oz::set_error("cudaEventSynchronize failed");
      return OZ_CUDA_ERROR;
    }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e.a, e.b);
    out[3 * e.kind] += ms;
    out[3 * e.kind + 1] += 1.0;
    out[3 * e.kind + 2] += e.work;
    if (e.kind == oz::PROF_EMU_GEMM) {  // SM-share-weighted time of the emulated GEMM
      const int all = oz::sm_count();
      const int used = e.sms > 0 && e.sms < all ? e.sms : all;
      out[3 * oz::PROF_GEMM_SMS] += ms * (double)used / all;
      out[3 * oz::PROF_GEMM_SMS + 1] += 1.0;
      out[3 * oz::PROF_GEMM_SMS + 2] += e.work;
    }
  }
  return OZ_OK;
}

extern "C" int oz_sm_count(int* out) {
  *out = oz::sm_count();
  return OZ_OK;
}

extern "C" int oz_dgemm(int transa, int transb, int64_t m, int64_t n, int64_t k, double alpha,
                        const double* a, int64_t lda, const double* b, int64_t ldb, double beta,
                        double* c, int64_t ldc, void* stream) {
  return oz::dgemm(transa, transb, m, n, k, alpha, a, lda, b, ldb, beta, c, ldc,
                   oz::as_stream(stream), 0);
}

namespace {
__global__ void axpby_kernel(int64_t count, double alpha, const double* __restrict__ ab,
                             double beta, const double* __restrict__ c, int use_c,
                             double* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    double v = ab[i];
    if (alpha != 1.0) v = __dmul_rn(alpha, v);
    if (use_c) v = __dadd_rn(v, __dmul_rn(beta, c[i]));
    out[i] = v;
  }
}
}  // namespace

extern "C" int oz_axpby(int64_t count, double alpha, const double* ab, double beta,
                        const double* c, int use_c, double* out, void* stream) {
  OZ_REQUIRE(count >= 0, OZ_INVALID_PARAMS, "negative count");
  OZ_REQUIRE(!use_c || c != nullptr, OZ_INVALID_PARAMS, "use_c without c");
  if (count == 0) return OZ_OK;
  int64_t blocks = (count + 255) / 256;
  if (blocks > oz::sm_count() * 8) blocks = oz::sm_count() * 8;
  axpby_kernel<<<(unsigned)blocks, 256, 0, oz::as_stream(stream)>>>(count, alpha, ab, beta, c,
                                                                     use_c, out);
  OZ_CHECK_LAUNCH();
  return OZ_OK;
}

// LAPACK-style interchanges -> permutation vector: pivots[i] is the original
// row index that ends at position i (solve.py:80-82 perm bookkeeping).
extern "C" int oz_ipiv_to_perm(const int32_t* ipiv, int64_t n, int64_t* perm) {
  for (int64_t i = 0; i < n; ++i) perm[i] = i;
  for (int64_t t = 0; t < n; ++t) {
    const int64_t p = ipiv[t];
    if (p < 0 || p >= n) {
      oz::set_error("ipiv[%lld]=%lld out of range", (long long)t, (long long)p);
      return OZ_INVALID_PARAMS;
    }
    if (p != t) {
      const int64_t tmp = perm[t];
      perm[t] = perm[p];
      perm[p] = tmp;
    }
  }
  return OZ_OK;
}
