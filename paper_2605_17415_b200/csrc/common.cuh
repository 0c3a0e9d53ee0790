// Shared device helpers for the IVF-TQ B200 library (sm_100a).
//
// Numerics that must match the reference bit-for-bit live here:
//   * pw_sumsq  -- numpy's pairwise summation of squares, the arithmetic behind
//                  np.linalg.norm(x, axis=1) (index.py:241, 254, 265).
//   * d2h_bits  -- float64 -> binary16 round-to-nearest-even, the arithmetic
//                  behind `rnorm.astype(np.float16)` (index.py:255).
#pragma once

#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "../../include/ivftq_b200.h"

#define IVFTQ_HD __host__ __device__ __forceinline__

// Device bounds checks, compiled in only for the debug build (make debug).
#ifdef IVFTQ_DEBUG
#include <cstdio>
#define DCHECK(cond, ...)                                                      \
  do {                                                                         \
    if (!(cond)) {                                                             \
      printf("DCHECK %s:%d %s | ", __FILE__, __LINE__, #cond);                 \
      printf(__VA_ARGS__);                                                     \
      printf("\n");                                                            \
      __trap();                                                                \
    }                                                                          \
  } while (0)
#else
#define DCHECK(cond, ...) \
  do {                    \
  } while (0)
#endif

namespace ivftq {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kPwBlock = 128;  // numpy PW_BLOCKSIZE

// ---------------------------------------------------------------------------
// float64 -> binary16 bits, round to nearest even (host + device).
IVFTQ_HD uint16_t d2h_bits(double x) {
  uint64_t u;
  memcpy(&u, &x, 8);
  uint16_t sgn = (uint16_t)((u >> 48) & 0x8000u);
  u &= 0x7fffffffffffffffull;
  if (u >= 0x7ff0000000000000ull) {  // inf / nan
    return (uint16_t)(sgn | (u == 0x7ff0000000000000ull ? 0x7c00u : 0x7e00u));
  }
  int e = (int)(u >> 52) - 1023;
  if (e >= 16) return (uint16_t)(sgn | 0x7c00u);
  if (e < -25) return sgn;  // below half the smallest subnormal (or zero)
  uint64_t m = (u & 0x000fffffffffffffull) | 0x0010000000000000ull;
  if ((u >> 52) == 0) return sgn;  // double subnormal
  int shift = (e >= -14) ? 42 : (28 - e);
  uint64_t q = m >> shift;
  uint64_t rem = m & ((1ull << shift) - 1);
  uint64_t half = 1ull << (shift - 1);
  if (rem > half || (rem == half && (q & 1))) q++;
  uint32_t h;
  if (e >= -14) {
    h = ((uint32_t)(e + 15) << 10) + (uint32_t)q - 1024u;  // carry rolls into exponent
  } else {
    h = (uint32_t)q;
  }
  return (uint16_t)(sgn | h);
}

IVFTQ_HD float h2f_bits(uint16_t h) {
#ifdef __CUDA_ARCH__
  return __half2float(__ushort_as_half(h));  // exact, one conversion instruction
#endif
  uint32_t s = (uint32_t)(h & 0x8000u) << 16;
  uint32_t e = (h >> 10) & 0x1f;
  uint32_t m = h & 0x3ff;
  uint32_t out;
  if (e == 0) {
    if (m == 0) {
      out = s;
    } else {  // subnormal: normalise
      int sh = 0;
      while (!(m & 0x400)) { m <<= 1; ++sh; }
      m &= 0x3ff;
      out = s | ((uint32_t)(127 - 15 - sh + 1) << 23) | (m << 13);
    }
  } else if (e == 31) {
    out = s | 0x7f800000u | (m << 13);
  } else {
    out = s | ((e - 15 + 127) << 23) | (m << 13);
  }
  float f;
  memcpy(&f, &out, 4);
  return f;
}

// ---------------------------------------------------------------------------
// numpy pairwise sum of squares over a[0..n) with element stride `st`
// (loops_utils.h.src pairwise_sum; squares rounded before summation, no FMA).
#ifdef __CUDACC__
__device__ __forceinline__ double sq(double v) { return __dmul_rn(v, v); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
#endif

template <typename Load>
__device__ double pw_block_raw(Load ld, int base, int n) {
  if (n < 8) {
    double r = -0.0;
    for (int i = 0; i < n; ++i) r = add(r, (ld(base + i)));
    return r;
  }
  double r0 = (ld(base + 0)), r1 = (ld(base + 1)), r2 = (ld(base + 2)),
         r3 = (ld(base + 3)), r4 = (ld(base + 4)), r5 = (ld(base + 5)),
         r6 = (ld(base + 6)), r7 = (ld(base + 7));
  int i = 8;
  int lim = n - (n % 8);
  for (; i < lim; i += 8) {
    r0 = add(r0, (ld(base + i + 0)));
    r1 = add(r1, (ld(base + i + 1)));
    r2 = add(r2, (ld(base + i + 2)));
    r3 = add(r3, (ld(base + i + 3)));
    r4 = add(r4, (ld(base + i + 4)));
    r5 = add(r5, (ld(base + i + 5)));
    r6 = add(r6, (ld(base + i + 6)));
    r7 = add(r7, (ld(base + i + 7)));
  }
  double res = add(add(add(r0, r1), add(r2, r3)), add(add(r4, r5), add(r6, r7)));
  for (; i < n; ++i) res = add(res, (ld(base + i)));
  return res;
}

// Iterative form of numpy's recursion: split n > 128 at n2 = n/2 - (n/2 % 8)
// and add the halves' sums left + right. Depth <= 16 for any int length.
// numpy's pairwise sum of ld(0..n) (np.add.reduce along a strided or
// contiguous axis, loops_utils.h.src pairwise_sum)
template <typename Load>
__device__ double pw_sum(Load ld, int n) {
  if (n <= kPwBlock) return pw_block_raw(ld, 0, n);
  // explicit post-order traversal
  int st_base[24], st_n[24];
  double st_left[24];
  unsigned char st_state[24];
  int sp = 0;
  st_base[0] = 0; st_n[0] = n; st_state[0] = 0;
  double ret = 0.0;
  while (sp >= 0) {
    int b = st_base[sp], m = st_n[sp];
    if (m <= kPwBlock) {
      ret = pw_block_raw(ld, b, m);
      --sp;
      // deliver to parent
      while (sp >= 0) {
        if (st_state[sp] == 1) {  // left finished -> start right
          st_left[sp] = ret;
          st_state[sp] = 2;
          int h = st_n[sp] / 2; h -= h % 8;
          ++sp;
          st_base[sp] = st_base[sp - 1] + h;
          st_n[sp] = st_n[sp - 1] - h;
          st_state[sp] = 0;
          break;
        } else {  // right finished
          ret = add(st_left[sp], ret);
          --sp;
        }
      }
      continue;
    }
    // descend left
    int h = m / 2; h -= h % 8;
    st_state[sp] = 1;
    ++sp;
    st_base[sp] = b; st_n[sp] = h; st_state[sp] = 0;
  }
  return ret;
}

// ... and of the squares (np.linalg.norm's sum of squares)
template <typename Load>
__device__ double pw_sumsq(Load ld, int n) {
  return pw_sum([&](int i) { return sq(ld(i)); }, n);
}

// The same sum for one row in shared memory, computed by the 8 lanes of an
// aligned lane group when n <= kPwBlock: lane j runs numpy's accumulator r_j
// (elements j, j+8, ...), three xor shuffles form ((r0+r1)+(r2+r3)) +
// ((r4+r5)+(r6+r7)) exactly as pw_block does (IEEE addition is commutative,
// so every lane of the group ends with the same bits), then the n % 8 tail.
// Longer or shorter rows take the serial form in every lane of the group.
__device__ __forceinline__ double pw_sumsq_lane8(const double* rp, int n) {
  const int lane = threadIdx.x & 31, j = lane & 7;
  const unsigned gm = 0xffu << (lane & 24);
  if (n > kPwBlock || n < 8) return pw_sumsq([&](int i) { return rp[i]; }, n);
  const int lim = n - (n % 8);
  double r = sq(rp[j]);
  for (int i = 8; i < lim; i += 8) r = add(r, sq(rp[i + j]));
  r = add(r, __shfl_xor_sync(gm, r, 1));
  r = add(r, __shfl_xor_sync(gm, r, 2));
  r = add(r, __shfl_xor_sync(gm, r, 4));
  for (int i = lim; i < n; ++i) r = add(r, sq(rp[i]));
  return r;
}

// ---------------------------------------------------------------------------
// Code layout helpers. One "field" per coordinate: c = bin*2 + sign,
// `field_bits` = bits + 1 wide, `fields_per_word` per uint32. The sign bit is
// stored even when scoring ignores it: the reference keeps it in `signs` and
// in .ivtq files regardless of use_sign_bit (index.py:266, storage.py:283);
// without the sign the level table simply maps both halves to the centroid.
// little-endian inside the word; 32-vector blocks interleave words so that
// word w of vector v lives at codes[(blk*W + w)*32 + v].
IVFTQ_HD int field_bits(int bits, int /*use_sign*/) { return bits + 1; }
IVFTQ_HD int fields_per_word(int fb) { return 32 / fb; }
IVFTQ_HD int words_per_vec(int dim, int fb) {
  int f = fields_per_word(fb);
  return (dim + f - 1) / f;
}

// Key order shared by every top-k in the library: score desc, id asc
// (index.py:480-483 lexsort((ids, -scores)); evaluation.py:78 stable argsort).
IVFTQ_HD bool better(double s1, int i1, double s2, int i2) {
  return s1 > s2 || (s1 == s2 && i1 < i2);
}

}  // namespace ivftq

// Error plumbing shared by the C-ABI wrappers.
namespace ivftq {
void set_error(const char* fmt, ...);
int check_launch(const char* what);
// Per-device state, safe for concurrent callers (mutex-guarded, keyed by the
// calling thread's current device): the SM count, and the dynamic shared
// memory a kernel has been opted in to on that device.
int device_sm_count();
int smem_opt_in_dev(const void* fn, size_t bytes);
// A side stream and two timing-free events private to (calling thread,
// current device): work forked off a caller's stream and joined back before
// the call returns. Streams of other threads are never touched, so
// concurrent calls (and one thread's graph capture) stay independent.
struct SideStream {
  cudaStream_t stream;
  cudaEvent_t fork, join;
};
int side_stream(SideStream** out);
}  // namespace ivftq

#define IVFTQ_CHECK_CUDA(expr)                                             \
  do {                                                                     \
    cudaError_t _e = (expr);                                               \
    if (_e != cudaSuccess) {                                               \
      ::ivftq::set_error("%s: %s", #expr, cudaGetErrorString(_e));         \
      return IVFTQ_ERR_CUDA;                                               \
    }                                                                      \
  } while (0)
