// C-ABI glue: error state, host utilities, the composed encoder and decoder.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>

#include "common.cuh"

namespace ivftq {

static thread_local char g_err[512] = "";
static unsigned long long g_launches = 0;  // kernels launched through this library

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int check_launch(const char* what) {
  __atomic_fetch_add(&g_launches, 1ull, __ATOMIC_RELAXED);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s launch failed: %s", what, cudaGetErrorString(e));
    return IVFTQ_ERR_CUDA;
  }
  return IVFTQ_OK;
}

// ---- per-device state ----------------------------------------------------------
static std::mutex g_dev_mu;
static std::map<int, int> g_sms;                               // device -> SM count
static std::map<std::pair<int, const void*>, size_t> g_opted;  // (device, kernel) -> bytes

static int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}

int device_sm_count() {
  const int dev = current_device();
  std::lock_guard<std::mutex> g(g_dev_mu);
  auto it = g_sms.find(dev);
  if (it != g_sms.end()) return it->second;
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1)
    n = 148;
  g_sms[dev] = n;
  return n;
}

int smem_opt_in_dev(const void* fn, size_t bytes) {
  if (bytes <= 48 * 1024) return 0;
  const int dev = current_device();
  std::lock_guard<std::mutex> g(g_dev_mu);
  size_t& have = g_opted[std::make_pair(dev, fn)];
  if (bytes <= have) return 0;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) {
    set_error("shared memory request %zu B rejected: %s", bytes, cudaGetErrorString(e));
    return IVFTQ_ERR_UNSUPPORTED;
  }
  have = bytes;
  return 0;
}

// One side stream + fork/join events per (host thread, device). Thread-local:
// never shared between threads, so a capture in one thread cannot absorb
// another thread's work; released with the thread.
struct SideStreams {
  std::map<int, SideStream> by_dev;
  ~SideStreams() {
    for (auto& kv : by_dev) {
      cudaStreamDestroy(kv.second.stream);
      cudaEventDestroy(kv.second.fork);
      cudaEventDestroy(kv.second.join);
    }
  }
};
static thread_local SideStreams t_side;

int side_stream(SideStream** out) {
  const int dev = current_device();
  auto it = t_side.by_dev.find(dev);
  if (it == t_side.by_dev.end()) {
    SideStream ss{};
    IVFTQ_CHECK_CUDA(cudaStreamCreateWithFlags(&ss.stream, cudaStreamNonBlocking));
    IVFTQ_CHECK_CUDA(cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming));
    IVFTQ_CHECK_CUDA(cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming));
    it = t_side.by_dev.emplace(dev, ss).first;
  }
  *out = &it->second;
  return 0;
}

// host mirror of pw_sumsq (same association order, no FMA)
static double host_pw_block(const double* a, int n) {
  if (n < 8) {
    volatile double r = -0.0;
    for (int i = 0; i < n; ++i) {
      volatile double s = a[i] * a[i];
      r = r + s;
    }
    return r;
  }
  volatile double r[8];
  for (int m = 0; m < 8; ++m) r[m] = a[m] * a[m];
  int i = 8, lim = n - (n % 8);
  for (; i < lim; i += 8)
    for (int m = 0; m < 8; ++m) {
      volatile double s = a[i + m] * a[i + m];
      r[m] = r[m] + s;
    }
  volatile double x01 = r[0] + r[1], x23 = r[2] + r[3], x45 = r[4] + r[5], x67 = r[6] + r[7];
  volatile double lo = x01 + x23, hi = x45 + x67;
  volatile double res = lo + hi;
  for (; i < n; ++i) {
    volatile double s = a[i] * a[i];
    res = res + s;
  }
  return res;
}

static double host_pw(const double* a, int n) {
  if (n <= kPwBlock) return host_pw_block(a, n);
  int h = n / 2;
  h -= h % 8;
  volatile double l = host_pw(a, h), r = host_pw(a + h, n - h);
  return l + r;
}

// decode helpers --------------------------------------------------------------
__global__ void decode_units_kernel(ivftq_store s, const int64_t* __restrict__ slot_of,
                                    int64_t n, const double* __restrict__ levels,
                                    double* __restrict__ units) {
  const int d = s.dim, W = s.words_per_vec, fb = s.field_bits, fpw = s.fields_per_word;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * W) return;
  int64_t r = i / W;
  int w = (int)(i - r * W);
  int64_t slot = slot_of[r];
  uint32_t word = s.codes[((slot >> 5) * W + w) * 32 + (slot & 31)];
  uint32_t mask = (1u << fb) - 1u;
  for (int f = 0; f < fpw; ++f) {
    int j = w * fpw + f;
    if (j >= d) break;
    units[r * d + j] = levels[(word >> (fb * f)) & mask];
  }
}

constexpr int kRows = 32;

__global__ void decode_finish_kernel(ivftq_store s, const int64_t* __restrict__ slot_of,
                                     const int32_t* __restrict__ list_of, int64_t n,
                                     const float* __restrict__ cent, int flat, int renorm,
                                     const double* __restrict__ back,
                                     double* __restrict__ out) {
  extern __shared__ double sm[];
  __shared__ double nrm[kRows];
  const int d = s.dim, ld = d + 1;
  int64_t row0 = (int64_t)blockIdx.x * kRows;
  int rows = (int)(n - row0 < kRows ? n - row0 : kRows);
  for (int i = threadIdx.x; i < rows * d; i += blockDim.x) {
    int r = i / d, c = i - r * d;
    int64_t g = row0 + r;
    double nv = (double)h2f_bits(s.norms[slot_of[g]]);
    double v = __dmul_rn(nv, back[g * d + c]);
    if (!flat) v = __dadd_rn(v, (double)cent[(int64_t)list_of[g] * d + c]);
    sm[r * ld + c] = v;
  }
  __syncthreads();
  if (threadIdx.x < rows) {
    const double* rp = sm + threadIdx.x * ld;
    double q = __dsqrt_rn(pw_sumsq([&](int i) { return rp[i]; }, d));
    nrm[threadIdx.x] = q > 1e-12 ? q : 1e-12;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < rows * d; i += blockDim.x) {
    int r = i / d, c = i - r * d;
    double v = sm[r * ld + c];
    out[(row0 + r) * d + c] = renorm ? __ddiv_rn(v, nrm[r]) : v;
  }
}

}  // namespace ivftq

using namespace ivftq;

extern "C" const char* ivftq_last_error(void) { return g_err; }
extern "C" int ivftq_abi_version(void) { return IVFTQ_ABI_VERSION; }
extern "C" unsigned long long ivftq_launch_count(void) {
  return __atomic_load_n(&g_launches, __ATOMIC_RELAXED);
}
extern "C" void ivftq_note_graph_launches(unsigned long long n) {
  __atomic_fetch_add(&g_launches, n, __ATOMIC_RELAXED);
}

extern "C" int ivftq_code_layout(int dim, int bits, int use_sign, int* fb, int* fpw, int* wpv) {
  if (dim < 1 || bits < 1 || bits > 8) {
    set_error("code_layout: bad dim/bits");
    return IVFTQ_ERR_ARG;
  }
  int f = field_bits(bits, use_sign);
  *fb = f;
  *fpw = fields_per_word(f);
  *wpv = words_per_vec(dim, f);
  return 0;
}

extern "C" int ivftq_host_double_to_half(const double* x, int64_t n, uint16_t* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = d2h_bits(x[i]);
  return 0;
}

extern "C" int ivftq_host_row_norms(const double* x, int64_t n, int dim, double* out) {
  for (int64_t i = 0; i < n; ++i) {
    volatile double s = host_pw(x + i * dim, dim);
    out[i] = __builtin_sqrt(s);
  }
  return 0;
}

extern "C" size_t ivftq_assign_tc_scratch_bytes(int64_t n, int n_lists, int dim);

extern "C" size_t ivftq_encode_tc_scratch_bytes(int64_t n, int dim);
extern "C" int ivftq_encode_supported_tc(int dim);
extern "C" int ivftq_encode_tail_tc(const double* xn, const float* centroids,
                                    const int32_t* list_ids, int64_t n, int dim, int bits,
                                    int use_sign, int flat, const double* R,
                                    const double* boundaries, const double* qcent,
                                    uint16_t* norm_out, uint32_t* words_out, void* scratch,
                                    size_t scratch_bytes, void* stream);

extern "C" size_t ivftq_encode_scratch_bytes(int64_t n, int dim, int n_lists) {
  const size_t a = (size_t)2 * n * dim * sizeof(double) + 256;
  const size_t b = ivftq_assign_tc_scratch_bytes(n, n_lists, dim);
  const size_t c = ivftq_encode_tc_scratch_bytes(n, dim);
  const size_t m = a > b ? a : b;  // the assignment scratch is dead before the residuals
  return m > c ? m : c;
}

extern "C" int ivftq_encode(const void* x, int x_dtype, int64_t n, int dim, int bits,
                            int use_sign, int flat, const float* centroids, int n_lists,
                            const double* R, const double* boundaries, const double* qcent,
                            double* xn_out, int64_t* bad_row, int32_t* list_out,
                            uint16_t* norm_out, uint32_t* words_out, void* scratch,
                            size_t scratch_bytes, void* stream) {
  if (scratch_bytes < ivftq_encode_scratch_bytes(n, dim, n_lists)) {
    set_error("encode: scratch too small");
    return IVFTQ_ERR_SCRATCH;
  }
  double* resid = (double*)scratch;
  double* rot = resid + (size_t)n * dim;
  if (int e = ivftq_normalize_rows(x, x_dtype, n, dim, xn_out, bad_row, stream)) return e;
  if (n == 0) return 0;
  if (flat) {
    IVFTQ_CHECK_CUDA(cudaMemsetAsync(list_out, 0, sizeof(int32_t) * n, (cudaStream_t)stream));
  } else {
    if (int e = ivftq_assign_tc(xn_out, centroids, n, n_lists, dim, list_out, scratch,
                                scratch_bytes, stream))
      return e;
  }
  // tensor-core tail (residual -> unit rows -> tcgen05 rotation -> Lloyd-Max with
  // an exact f64 pass over the rows near a threshold) whenever the shape allows
  if (ivftq_encode_supported_tc(dim))
    return ivftq_encode_tail_tc(xn_out, centroids, list_out, n, dim, bits, use_sign, flat, R,
                                boundaries, qcent, norm_out, words_out, scratch, scratch_bytes,
                                stream);
  if (int e = ivftq_residuals(xn_out, centroids, list_out, n, dim, flat, resid, norm_out, stream))
    return e;
  if (int e = ivftq_gemm_nt(resid, R, IVFTQ_F64, n, dim, dim, rot, IVFTQ_F64, stream)) return e;
  return ivftq_quantize_pack(rot, norm_out, n, dim, bits, use_sign, boundaries, qcent,
                             words_out, stream);
}

extern "C" size_t ivftq_decode_scratch_bytes(int64_t n, int dim) {
  return (size_t)2 * n * dim * sizeof(double) + 256;
}

extern "C" int ivftq_decode(const ivftq_store* st, const int64_t* slot_of,
                            const int32_t* list_of, int64_t n, const float* centroids,
                            const double* R, const double* levels, int flat, int renormalize,
                            double* out, void* scratch, size_t scratch_bytes, void* stream) {
  if (scratch_bytes < ivftq_decode_scratch_bytes(n, st->dim)) {
    set_error("decode: scratch too small");
    return IVFTQ_ERR_SCRATCH;
  }
  if (n == 0) return 0;
  const int d = st->dim;
  double* units = (double*)scratch;
  double* back = units + (size_t)n * d;
  cudaStream_t s = (cudaStream_t)stream;
  int64_t tot = n * st->words_per_vec;
  decode_units_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(*st, slot_of, n, levels,
                                                                   units);
  if (int e = check_launch("decode_units")) return e;
  // back = units . R  ==  units . (R^T)^T : R must be passed transposed (R^T row-major)
  if (int e = ivftq_gemm_nt(units, R, IVFTQ_F64, n, d, d, back, IVFTQ_F64, stream)) return e;
  int bytes = kRows * (d + 1) * (int)sizeof(double);
  if (bytes > 48 * 1024)
    IVFTQ_CHECK_CUDA(cudaFuncSetAttribute((const void*)decode_finish_kernel,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  decode_finish_kernel<<<(unsigned)((n + kRows - 1) / kRows), 128, bytes, s>>>(
      *st, slot_of, list_of, n, centroids, flat, renormalize, back, out);
  return check_launch("decode_finish");
}

namespace ivftq {
// out[i] = sum_j a[i,j] * c[l_i, j] in f64 (refresh report statistics,
// refresh.py:179-187 einsum("nd,nd->n", source, centroids[list_ids])).
__global__ void rowdot_kernel(const double* __restrict__ a, const float* __restrict__ cent,
                              const int32_t* __restrict__ lids, int64_t n, int d,
                              double* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* r = a + i * d;
  const float* c = cent + (int64_t)lids[i] * d;
  double s = 0.0;
  for (int j = 0; j < d; ++j) s = __fma_rn(r[j], (double)c[j], s);
  out[i] = s;
}
}  // namespace ivftq

extern "C" int ivftq_rowdot(const double* a, const float* centroids, const int32_t* list_ids,
                            int64_t n, int dim, double* out, void* stream) {
  if (n == 0) return 0;
  rowdot_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      a, centroids, list_ids, n, dim, out);
  return check_launch("rowdot");
}
