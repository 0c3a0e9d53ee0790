// Block-wide exact top-K over a stream of (score f64, id i32) candidates with
// the reference's key: score desc, id asc (index.py:480-483).
//
// Candidates that beat the current K-th best are appended to a shared buffer
// with one warp-aggregated atomic; when the buffer is nearly full the block
// bitonic-sorts it and keeps K. The threshold only tightens at a merge, so
// it is conservative and the result is exact and order-independent.
#pragma once

#include <climits>

#include "common.cuh"

namespace ivftq {

__host__ __device__ inline int pow2ceil(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

// Buffer capacity for K kept entries with rounds of up to `round` pushes.
__host__ __device__ inline int topk_cap(int K, int round) { return pow2ceil(K + 2 * round); }

struct BlockTopK {
  double* s;
  int* id;
  int cap;
  int K;
  int* cnt;
  double* thr_s;
  int* thr_id;

  // carve from shared memory: needs cap*(8+4) + 32 bytes, 8-aligned base
  __device__ void carve(char* base, int cap_, int K_) {
    cap = cap_;
    K = K_;
    s = (double*)base;
    id = (int*)(base + (size_t)cap * 8);
    char* tail = base + (size_t)cap * 12;
    tail = (char*)(((uintptr_t)tail + 7) & ~(uintptr_t)7);
    thr_s = (double*)tail;
    cnt = (int*)(tail + 8);
    thr_id = (int*)(tail + 12);
  }
  static __host__ __device__ size_t bytes(int cap_) { return (size_t)cap_ * 12 + 32; }

  __device__ void init() {
    if (threadIdx.x == 0) {
      *cnt = 0;
      *thr_s = -INFINITY;
      *thr_id = INT_MAX;
    }
  }

  __device__ __forceinline__ bool passes(double sc, int i) const {
    return better(sc, i, *(volatile double*)thr_s, *(volatile int*)thr_id);
  }

  // all 32 lanes of the warp must call
  __device__ __forceinline__ void push_warp(bool pass, double sc, int i) {
    unsigned m = __ballot_sync(kFull, pass);
    if (!m) return;
    int lane = threadIdx.x & 31;
    int leader = __ffs(m) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(cnt, __popc(m));
    base = __shfl_sync(kFull, base, leader);
    if (pass) {
      int pos = base + __popc(m & ((1u << lane) - 1u));
      DCHECK(pos < cap, "push pos=%d cap=%d", pos, cap);
      s[pos] = sc;
      id[pos] = i;
    }
  }

  // all threads call; brackets itself with barriers
  __device__ void merge() {
    __syncthreads();
    int n = *cnt;
    int P = pow2ceil(n > 1 ? n : 1);
    DCHECK(P <= cap, "merge n=%d cap=%d", n, cap);
    for (int i = n + threadIdx.x; i < P; i += blockDim.x) {
      s[i] = -INFINITY;
      id[i] = INT_MAX;
    }
    __syncthreads();
    for (int k = 2; k <= P; k <<= 1) {
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int t = threadIdx.x; t < (P >> 1); t += blockDim.x) {
          int lo = ((t / j) * 2 * j) + (t % j);
          int hi = lo + j;
          double sl = s[lo], sh = s[hi];
          int il = id[lo], ih = id[hi];
          bool up = (lo & k) == 0;
          bool sw = up ? better(sh, ih, sl, il) : better(sl, il, sh, ih);
          if (sw) {
            s[lo] = sh; s[hi] = sl;
            id[lo] = ih; id[hi] = il;
          }
        }
        __syncthreads();
      }
    }
    int keep = n < K ? n : K;
    if (threadIdx.x == 0) {
      *cnt = keep;
      if (keep == K && K > 0) {
        *thr_s = s[K - 1];
        *thr_id = id[K - 1];
      }
    }
    __syncthreads();
  }

  // call after a round's pushes (all threads)
  __device__ void round_end(int round) {
    __syncthreads();
    int c = *(volatile int*)cnt;
    // second barrier: nobody may push for the next round before every thread
    // has read the count, or the merge decision would diverge across warps
    __syncthreads();
    if (c > cap - round) merge();
  }
};

}  // namespace ivftq
