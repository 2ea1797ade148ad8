// SPDX-License-Identifier: Apache-2.0
// Fixed-width bit rows (NW x u64) and sm_100a async-copy / mbarrier helpers.
#pragma once

#include <cstdint>

namespace xe {

template <int NW>
struct Row {
  uint64_t w[NW];
  __device__ __forceinline__ static Row zero() {
    Row r;
#pragma unroll
    for (int j = 0; j < NW; ++j) r.w[j] = 0;
    return r;
  }
  __device__ __forceinline__ bool any() const {
    uint64_t a = 0;
#pragma unroll
    for (int j = 0; j < NW; ++j) a |= w[j];
    return a != 0;
  }
  __device__ __forceinline__ bool test(int i) const {
    uint64_t x = 0;
#pragma unroll
    for (int j = 0; j < NW; ++j)
      if (j == (i >> 6)) x = w[j];
    return (x >> (i & 63)) & 1ull;
  }
  __device__ __forceinline__ void set(int i) {
#pragma unroll
    for (int j = 0; j < NW; ++j)
      if (j == (i >> 6)) w[j] |= 1ull << (i & 63);
  }
  __device__ __forceinline__ void clear(int i) {
#pragma unroll
    for (int j = 0; j < NW; ++j)
      if (j == (i >> 6)) w[j] &= ~(1ull << (i & 63));
  }
  __device__ __forceinline__ int popc() const {
    int c = 0;
#pragma unroll
    for (int j = 0; j < NW; ++j) c += __popcll(w[j]);
    return c;
  }
  // highest set bit, -1 when empty
  __device__ __forceinline__ int msb() const {
    int r = -1;
#pragma unroll
    for (int j = 0; j < NW; ++j)
      if (w[j]) r = 64 * j + 63 - __clzll(w[j]);
    return r;
  }
  // lowest set bit, -1 when empty
  __device__ __forceinline__ int lsb() const {
#pragma unroll
    for (int j = 0; j < NW; ++j)
      if (w[j]) return 64 * j + __ffsll(w[j]) - 1;
    return -1;
  }
  // bits strictly greater than t
  __device__ __forceinline__ static Row above(int t) {
    Row r;
#pragma unroll
    for (int j = 0; j < NW; ++j) {
      int lo = 64 * j;
      if (t < lo) r.w[j] = ~0ull;
      else if (t >= lo + 63) r.w[j] = 0;
      else r.w[j] = ~0ull << (t - lo + 1);
    }
    return r;
  }
  // bits >= t
  __device__ __forceinline__ static Row at_or_above(int t) {
    Row r;
#pragma unroll
    for (int j = 0; j < NW; ++j) {
      int lo = 64 * j;
      if (t <= lo) r.w[j] = ~0ull;
      else if (t >= lo + 64) r.w[j] = 0;
      else r.w[j] = ~0ull << (t - lo);
    }
    return r;
  }
  // bits < T (row validity mask)
  __device__ __forceinline__ static Row below(int T) {
    Row r;
#pragma unroll
    for (int j = 0; j < NW; ++j) {
      int lo = 64 * j;
      if (T >= lo + 64) r.w[j] = ~0ull;
      else if (T <= lo) r.w[j] = 0;
      else r.w[j] = (1ull << (T - lo)) - 1;
    }
    return r;
  }
};

template <int NW>
__device__ __forceinline__ Row<NW> operator|(Row<NW> a, const Row<NW>& b) {
#pragma unroll
  for (int j = 0; j < NW; ++j) a.w[j] |= b.w[j];
  return a;
}
template <int NW>
__device__ __forceinline__ Row<NW> operator&(Row<NW> a, const Row<NW>& b) {
#pragma unroll
  for (int j = 0; j < NW; ++j) a.w[j] &= b.w[j];
  return a;
}
template <int NW>
__device__ __forceinline__ Row<NW> operator~(Row<NW> a) {
#pragma unroll
  for (int j = 0; j < NW; ++j) a.w[j] = ~a.w[j];
  return a;
}
template <int NW>
__device__ __forceinline__ Row<NW> andnot(Row<NW> a, const Row<NW>& b) {
#pragma unroll
  for (int j = 0; j < NW; ++j) a.w[j] &= ~b.w[j];
  return a;
}

template <int NW>
__device__ __forceinline__ Row<NW> load_row(const uint64_t* p) {
  Row<NW> r;
#pragma unroll
  for (int j = 0; j < NW; ++j) r.w[j] = p[j];
  return r;
}

// ---- warp collectives ------------------------------------------------------
__device__ __forceinline__ int64_t warp_max_i64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    int64_t x = __shfl_xor_sync(0xffffffffu, v, o);
    v = x > v ? x : v;
  }
  return v;
}
__device__ __forceinline__ int64_t warp_sum_i64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ int warp_excl_scan(int v, int lane, int* total) {
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  *total = __shfl_sync(0xffffffffu, x, 31);
  return x - v;
}

// ---- mbarrier + bulk async copy (TMA engine, cp.async.bulk) ----------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
  }
}

}  // namespace xe
