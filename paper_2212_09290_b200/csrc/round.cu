// SPDX-License-Identifier: Apache-2.0
//
// K4 — randomized rounding + repair of (relaxed) schedules into candidate
// cubes that feed K2.  No reference code exists for this step;
// its outputs are judged through K2 parity and the final best schedule.
//
// Candidate c (global index first + k) is a pure function of (seed, c):
// Philox-4x32-10 streams keyed by the candidate index, so shards generated on
// different GPUs or in different batches are identical to one big batch.
//
// Construction (valid for EQ8/EQ11/EQ12 by construction):
//   1. placement: op i on device d with probability proportional to the LP
//      diagonal x(R(d,i,i)) (or uniform when x is NULL) over the devices whose
//      cost is below the 1e9 sentinel (problem.hpp:16);
//   2. minimal-save S: S(dev_i, t, i) = 1 for i < t <= last consumer of i;
//   3. up to `edits` drop-and-recompute edits: the tensor of op i is dropped
//      over a window before one of its consumers and recomputed there
//      (possibly on another device); each parent not resident at that step
//      is either kept saved until then or itself recomputed there (dropping
//      its own save window), recursively — chains of recomputation;
//   4. with probability `perturb`, one uniformly random R/S bit is flipped.
// One warp per candidate; the cube is assembled in shared memory and written
// out with coalesced 16-byte stores.

#include <algorithm>
#include <cstdlib>

#include "bits.cuh"
#include "xe_internal.hpp"

namespace xe {
namespace {

struct Philox {
  uint32_t c0, c1, c2, c3, k0, k1;
  __device__ Philox(uint64_t seed, uint64_t ctr, uint32_t stream)
      : c0(static_cast<uint32_t>(ctr)), c1(static_cast<uint32_t>(ctr >> 32)), c2(stream), c3(0),
        k0(static_cast<uint32_t>(seed)), k1(static_cast<uint32_t>(seed >> 32)) {}
  __device__ uint4 next() {
    uint32_t x0 = c0, x1 = c1, x2 = c2, x3 = c3, a = k0, b = k1;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      uint32_t hi0 = __umulhi(0xD2511F53u, x0), lo0 = 0xD2511F53u * x0;
      uint32_t hi1 = __umulhi(0xCD9E8D57u, x2), lo1 = 0xCD9E8D57u * x2;
      uint32_t y0 = hi1 ^ x1 ^ a, y1 = lo1, y2 = hi0 ^ x3 ^ b, y3 = lo0;
      x0 = y0; x1 = y1; x2 = y2; x3 = y3;
      a += 0x9E3779B9u;
      b += 0xBB67AE85u;
    }
    ++c3;
    return make_uint4(x0, x1, x2, x3);
  }
  __device__ uint32_t u32() {
    if (have == 0) {
      buf = next();
      have = 4;
    }
    --have;
    return have == 3 ? buf.x : have == 2 ? buf.y : have == 1 ? buf.z : buf.w;
  }
  __device__ double uniform() { return (u32() >> 8) * (1.0 / 16777216.0); }
  __device__ int below(int n) { return static_cast<int>((static_cast<uint64_t>(u32()) * n) >> 32); }
  uint4 buf{};
  int have = 0;
};

struct RoundArgs {
  const int64_t* mass;
  const double* cost;   // [D][T]
  const int32_t* src;
  const int32_t* dst;
  const int32_t* in_ptr;
  const int32_t* in_edge;
  const double* x;      // LP solution or null
  const uint32_t* base; // local search: every candidate starts from this cube (or null)
  // LP-guided recomputation: off-diagonal R(d,t,i) (t > i) of the relaxation
  // with weight > 0, as codes (d*T + t)*T + i and their cumulative weights
  const int32_t* rc_code;
  const double* rc_cdf;
  int n_rc;
  int D, T, E, W32;
  int64_t r_base;       // column offset of R in x (0)
  uint64_t seed;
  int64_t first, n;
  int edits;
  double perturb;
  uint32_t* out;
  int word_build;  // steps 1-2 word by word (long-lived tensors) instead of one atomic per saved bit
  int slow_scan;   // XE_ROUND_SLOW_SCAN=1: the edits' backward row scans (test of the fast lookup)
  // uniform placements (x null): per op the devices that can run it (cost
  // below the sentinel) in order, their count, and the cheapest device
  const uint8_t* ok_n;
  const uint8_t* ok_list;  // [T][8]
  const uint8_t* cheap;
  const double* lp_cum;  // [T][8] running sums of max(x(R(d,i,i)), 1e-3) over the allowed devices (x given)
};

constexpr int kRoundWarps = 4;

// Steps 3-4 of one candidate (drop-and-recompute edits, perturbation): a
// walk over one cube; run by the candidate's whole warp (round_kernel, the
// timestep loops split across lanes) or by one lane per candidate
// (round_batch_kernel) — the same code, so both produce the same cubes.
// fast: the cube was built here from a placement (no base): every timestep
// tt computes op tt (its diagonal R bit), and the only other computations are
// the recomputations this function adds, at the timesteps listed in rts — so
// "the latest step in (u, hi) that computes a consumer of u" is the top
// consumer bit of u below hi or one of those few steps, instead of a backward
// scan over every timestep's rows.  Both give the same step.
// WARP: the whole warp runs one candidate's edits — every lane follows the
// same (uniform) control flow and Philox draws, the loops over timesteps are
// split across the lanes (each lane owns the rows of its timesteps, so no
// two lanes write one word) and single-bit writes are lane 0's, with a warp
// barrier before the next read.  Same cubes as the one-lane form.
template <bool WARP>
__device__ void edit_candidate(const RoundArgs& a, uint32_t* cube, const int* dev, const uint32_t* cons,
                               const int* last, const int* elig, int n_elig_v, uint64_t c, bool fast) {
  const int D = a.D, T = a.T, W = a.W32;
  (void)last;
  const int L0 = WARP ? static_cast<int>(threadIdx.x & 31) : 0;  // this lane's first offset
  constexpr int LS = WARP ? 32 : 1;                               // loop stride
  auto sync = [] {
    if (WARP) __syncwarp();
  };
  constexpr int kMaxRts = 16;
  int rts[kMaxRts];
  int nrts = 0;
  auto consumer_at = [&](int u, int tt) {
    uint32_t hit = 0u;
    for (int w = 0; w < W; ++w) {
      uint32_t r = 0u;
      for (int d = 0; d < D; ++d) r |= cube[(d * T + tt) * W + w];
      hit |= r & cons[u * W + w];
    }
    return hit != 0u;
  };
  auto bset = [&](int which, int d, int t, int i) {
    cube[((which * D + d) * T + t) * W + (i >> 5)] |= 1u << (i & 31);
  };
  auto bclr = [&](int which, int d, int t, int i) {
    cube[((which * D + d) * T + t) * W + (i >> 5)] &= ~(1u << (i & 31));
  };
  auto bit_get = [&](int which, int d, int t, int i) -> bool {
    return (cube[((which * D + d) * T + t) * W + (i >> 5)] >> (i & 31)) & 1u;
  };
  // latest tt in (u, hi) with consumer_at(u, tt), or u when there is none
  auto last_consumer = [&](int u, int hi) -> int {
    if (!fast) {
      if constexpr (WARP) {
        int best = u;
        for (int tt = u + 1 + L0; tt < hi; tt += LS)
          if (consumer_at(u, tt)) best = tt;
        return static_cast<int>(__reduce_max_sync(0xffffffffu, static_cast<unsigned>(best)));
      } else {
        for (int tt = hi - 1; tt > u; --tt)
          if (consumer_at(u, tt)) return tt;
        return u;
      }
    }
    int best = u;
    for (int w = W - 1; w >= 0; --w) {
      const int lo = 32 * w;
      uint32_t m = cons[u * W + w];
      // keep bits tt with u < tt < hi
      if (hi <= lo) m = 0u;
      else if (hi < lo + 32) m &= (1u << (hi - lo)) - 1u;
      if (u + 1 >= lo + 32) m = 0u;
      else if (u + 1 > lo) m &= ~0u << (u + 1 - lo);
      if (m) {
        best = lo + 31 - __clz(m);
        break;
      }
    }
    for (int k = 0; k < nrts; ++k) {
      const int tt = rts[k];
      if (tt > best && tt < hi && consumer_at(u, tt)) best = tt;
    }
    return best;
  };
  Philox rng(a.seed, c, 0x1u);
  for (int ed = 0; ed < a.edits; ++ed) {
    if (rng.uniform() >= 0.6) continue;
    int i = 0, t = -1, lp_dev = -1;
    if (a.n_rc > 0 && rng.uniform() < 0.7) {
      // where the LP relaxation recomputes: (d, t, i) drawn with weight x(R(d,t,i))
      const double u = rng.uniform() * a.rc_cdf[a.n_rc - 1];
      int lo = 0, hi = a.n_rc - 1;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a.rc_cdf[mid] > u) hi = mid;
        else lo = mid + 1;
      }
      const int code = a.rc_code[lo];
      i = code % T;
      t = code / T % T;
      lp_dev = code / (T * T);
    } else {
      // op i with a consumer beyond i+1, chosen uniformly among eligible ops
      const int n_el = n_elig_v;
      if (n_el == 0) break;
      i = elig[rng.below(n_el)];
      // consumer t > i+1 of i, uniformly among its consumers (ascending)
      int n_c = 0;
      for (int w = 0; w < W; ++w) {
        const int lo = w * 32;
        uint32_t m = cons[i * W + w];
        if (lo + 32 <= i + 2) m = 0u;
        else if (lo <= i + 1) m &= ~0u << (i + 2 - lo);
        n_c += __popc(m);
      }
      int pc = rng.below(n_c);
      for (int w = 0; w < W && t < 0; ++w) {
        const int lo = w * 32;
        uint32_t m = cons[i * W + w];
        if (lo + 32 <= i + 2) m = 0u;
        else if (lo <= i + 1) m &= ~0u << (i + 2 - lo);
        const int pcnt = __popc(m);
        if (pc < pcnt) {
          for (int q = 0; q < pc; ++q) m &= m - 1;
          t = lo + __ffs(m) - 1;
        }
        pc -= pcnt;
      }
    }
    // the drop window must not cover a timestep where i is needed: any
    // earlier computation (diagonal or recomputed) of a consumer of i
    const int a0 = last_consumer(i, t) + 1;
    if (a0 > t) continue;
    if (fast) {  // t receives recomputations below
      bool seen = false;
      for (int k = 0; k < nrts; ++k) seen |= rts[k] == t;
      if (!seen) {
        if (nrts < kMaxRts) rts[nrts++] = t;
        else fast = false;  // list full: back to the scan (same answers)
      }
    }
    // drop the whole window when the LP chose the spot, else a random tail of it
    const int a1 = lp_dev >= 0 ? a0 : a0 + rng.below(t - a0 + 1);
    int dn = lp_dev >= 0 ? lp_dev : (rng.uniform() < 0.5 ? rng.below(D) : dev[t]);
    if (a.cost[dn * T + i] >= 1.0e9) dn = dev[i];
    // recompute op v at t on device dr, dropping its saves on dev-of-v
    // over [from, t]; later saves follow it to dr (EQ11 needs a holder at t)
    auto recompute_at = [&](int v, int from, int dr) {
      const int dv = dev[v];
      for (int tt = from + L0; tt <= t; tt += LS) bclr(1, dv, tt, v);
      if (L0 == 0) bset(0, dr, t, v);
      if (dr != dv)
        for (int tt = t + 1 + L0; tt < T; tt += LS)
          if (bit_get(1, dv, tt, v)) {
            bclr(1, dv, tt, v);
            bset(1, dr, tt, v);
          }
      sync();
    };
    recompute_at(i, a1, dn);
    // parents of every op recomputed at t: keep them saved until t, or
    // (probability 1/2) recompute them at t too, dropping their own save
    // windows — chains of recomputation.  A recomputed parent runs on its
    // child's device or (probability 1/4) another one: a chain may cross
    // devices within the timestep, so a memory-tight device need not hold
    // the chain's intermediate tensors (config 2's optimum recomputes
    // ops 0-1 on the cpu and 2-3 on the gpu at t = 39)
    int stack[32], sdev[32], sp = 0;
    stack[sp] = i;
    sdev[sp++] = dn;
    while (sp > 0) {
      --sp;
      const int v = stack[sp], dvn = sdev[sp];
      for (int k2 = a.in_ptr[v]; k2 < a.in_ptr[v + 1]; ++k2) {
        const int p = a.src[a.in_edge[k2]];
        bool avail = false;
        for (int d = 0; d < D; ++d) avail |= bit_get(0, d, t, p) || bit_get(1, d, t, p);
        if (avail) continue;
        int dr = dvn;
        if (D > 1 && rng.uniform() < 0.25) dr = (dvn + 1 + rng.below(D - 1)) % D;
        if (a.cost[dr * T + p] >= 1.0e9) dr = dvn;
        if (sp < 32 && a.cost[dr * T + p] < 1.0e9 && rng.uniform() < 0.5) {
          // first step after p's last use before t
          const int from = last_consumer(p, t) + 1;
          recompute_at(p, from, dr);
          stack[sp] = p;
          sdev[sp++] = dr;
          continue;
        }
        const int dp = dev[p];
        int ls = p;
        for (int tt = p + 1 + L0; tt <= t; tt += LS)
          if (bit_get(1, dp, tt, p)) ls = tt;
        if (WARP) ls = static_cast<int>(__reduce_max_sync(0xffffffffu, static_cast<unsigned>(ls)));
        for (int tt = ls + 1 + L0; tt <= t; tt += LS) bset(1, dp, tt, p);
        sync();
      }
    }
  }
  // 4. perturbation
  if (rng.uniform() < a.perturb) {
    const int which = rng.below(2), d = rng.below(D), t = rng.below(T), i = rng.below(T);
    if (L0 == 0) cube[((which * D + d) * T + t) * W + (i >> 5)] ^= 1u << (i & 31);
  }
  sync();

}


// running sums of the LP weights over op i's allowed devices, in device
// order (the additions place_op's general path makes, in the same order)
__global__ void lp_cum_kernel(const double* x, int64_t r_base, const uint8_t* ok_n, const uint8_t* ok_list, int T,
                              double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= T) return;
  double tot = 0.0;
  for (int k = 0; k < ok_n[i]; ++k) {
    const int d = ok_list[i * 8 + k];
    tot += fmax(x[r_base + (static_cast<int64_t>(d) * T + i) * T + i], 1e-3);
    out[i * 8 + k] = tot;
  }
}

// Step 1 for op i of candidate c: device drawn with probability proportional
// to the LP diagonal x(R(d,i,i)) (uniform when x is null) over the devices
// whose cost is below the sentinel, else the cheapest.  With x null the
// draw is the floor(u * n)-th allowed device — what the running sum below
// picks — read from the per-op tables.
__device__ __forceinline__ int place_op(const RoundArgs& a, uint64_t c, int i) {
  const int D = a.D, T = a.T;
  if (!a.x && a.ok_n) {
    const int n = a.ok_n[i];
    if (n == 0) return a.cheap[i];
    Philox rng(a.seed, c, 0x10000u + static_cast<uint32_t>(i));
    const double u = rng.uniform() * n;
    const int k = min(static_cast<int>(u), n - 1);
    return a.ok_list[i * 8 + k];
  }
  if (a.x && a.lp_cum) {  // the same running sums, precomputed per op
    const int n = a.ok_n[i];
    if (n == 0) return a.cheap[i];
    const double* cum = a.lp_cum + i * 8;
    Philox rng(a.seed, c, 0x10000u + static_cast<uint32_t>(i));
    const double u = rng.uniform() * cum[n - 1];
    for (int k = 0; k < n; ++k)
      if (u < cum[k]) return a.ok_list[i * 8 + k];
    return a.ok_list[i * 8 + n - 1];  // rounding tail
  }
  Philox rng(a.seed, c, 0x10000u + static_cast<uint32_t>(i));
  double tot = 0.0;
  for (int d = 0; d < D; ++d) {
    if (a.cost[d * T + i] >= 1.0e9) continue;
    tot += a.x ? fmax(a.x[a.r_base + (static_cast<int64_t>(d) * T + i) * T + i], 1e-3) : 1.0;
  }
  int pick = 0;
  if (tot == 0.0) {
    double best = 1e300;  // every device prohibitive: cheapest
    for (int d = 0; d < D; ++d)
      if (a.cost[d * T + i] < best) best = a.cost[d * T + i], pick = d;
  } else {
    double u = rng.uniform() * tot, acc = 0.0;
    int lastok = 0;
    pick = -1;
    for (int d = 0; d < D; ++d) {
      if (a.cost[d * T + i] >= 1.0e9) continue;
      acc += a.x ? fmax(a.x[a.r_base + (static_cast<int64_t>(d) * T + i) * T + i], 1e-3) : 1.0;
      lastok = d;
      if (pick < 0 && u < acc) pick = d;
    }
    if (pick < 0) pick = lastok;  // rounding tail
  }
  return pick;
}

// alive[t][w]: ops i of word w with i < t <= last[i] (the minimal-save set
// of timestep t, candidate-independent); block-cooperative
__device__ void build_alive(uint32_t* alive, uint16_t* tq, const int* last, int T, int W) {
  for (int q = threadIdx.x; q < T * W; q += blockDim.x) {
    const int t = q / W, w = q % W;
    tq[q] = static_cast<uint16_t>(t);
    uint32_t m = 0u;
    for (int b = 0; b < 32; ++b) {
      const int i = 32 * w + b;
      if (i < T && i < t && t <= last[i]) m |= 1u << b;
    }
    alive[q] = m;
  }
}

// Steps 1-2 written word by word by one warp: R(d,t) = {t} when dev_t = d,
// S(d,t) = alive(t) & the ops placed on d (dm: per-warp [D][W] scratch)
__device__ void build_minimal_save(uint32_t* cube, const int* dev, const uint32_t* alive, const uint16_t* tq,
                                   uint32_t* dm, int D, int T, int W, int lane) {
  for (int w = 0; w < W; ++w) {
    const int i = 32 * w + lane;
    const int di = i < T ? dev[i] : -1;
    for (int d = 0; d < D; ++d) {
      const unsigned m = __ballot_sync(0xffffffffu, di == d);
      if (lane == 0) dm[d * W + w] = m;
    }
  }
  __syncwarp();
  // lanes over the words q = t*W + w of a (which, d) plane: consecutive
  // lanes store consecutive words
  const int TW = T * W;
  for (int q = lane; q < TW; q += 32) {
    const int t = tq[q], w = q - t * W;
    const int dt = dev[t];
    const uint32_t bit = (t >> 5) == w ? (1u << (t & 31)) : 0u;
    const uint32_t al = alive[q];
    for (int d = 0; d < D; ++d) {
      cube[d * TW + q] = dt == d ? bit : 0u;
      cube[(D + d) * TW + q] = al & dm[d * W + w];
    }
  }
  __syncwarp();
}

// Steps 1-2 bit by bit (cheaper when tensors live briefly: one shared
// atomic per saved bit instead of every word of the cube)
__device__ void build_minimal_save_bits(uint32_t* cube, const int* dev, const int* last, int D, int T, int W,
                                        int lane) {
  const int words = 2 * D * T * W;
  for (int i = lane; i < words; i += 32) cube[i] = 0u;
  __syncwarp();
  for (int i = lane; i < T; i += 32) {
    const int d = dev[i];
    atomicOr(&cube[(d * T + i) * W + (i >> 5)], 1u << (i & 31));
    for (int t = i + 1; t <= last[i]; ++t) atomicOr(&cube[((D + d) * T + t) * W + (i >> 5)], 1u << (i & 31));
  }
  __syncwarp();
}

__global__ void __launch_bounds__(kRoundWarps * 32) round_kernel(const RoundArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int D = a.D, T = a.T, W = a.W32;
  const int words = 2 * D * T * W;
  // block tables: consumers of every op as bit rows, last consumer of every op
  uint32_t* cons = reinterpret_cast<uint32_t*>(smem);
  int* last = reinterpret_cast<int*>(cons + T * W);
  int* elig = last + T;      // ops with a consumer beyond i+1, ascending
  int* n_elig = elig + T;
  uint32_t* alive = reinterpret_cast<uint32_t*>(n_elig + 1);  // [T][W]
  uint16_t* tq = reinterpret_cast<uint16_t*>(alive + T * W);     // [T*W]: t of word q
  uint32_t* cube = alive + T * W + (T * W + 1) / 2 + wid * (words + T);
  int* dev = reinterpret_cast<int*>(cube + words);
  uint32_t* dm = alive + T * W + (T * W + 1) / 2 + kRoundWarps * (words + T) + wid * D * W;  // [D][W]
  for (int i = threadIdx.x; i < T * W; i += blockDim.x) cons[i] = 0u;
  for (int i = threadIdx.x; i < T; i += blockDim.x) last[i] = -1;
  __syncthreads();
  for (int e = threadIdx.x; e < a.E; e += blockDim.x) {
    atomicOr(&cons[a.src[e] * W + (a.dst[e] >> 5)], 1u << (a.dst[e] & 31));
    atomicMax(&last[a.src[e]], a.dst[e]);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int ne = 0;
    for (int j = 0; j < T; ++j)
      if (last[j] > j + 1) elig[ne++] = j;
    *n_elig = ne;
  }
  build_alive(alive, tq, last, T, W);
  __syncthreads();
  // plain read-modify-write for the single-lane sections (lane 0 edits)
  auto bset = [&](int which, int d, int t, int i) {
    cube[((which * D + d) * T + t) * W + (i >> 5)] |= 1u << (i & 31);
  };
  auto bclr = [&](int which, int d, int t, int i) {
    cube[((which * D + d) * T + t) * W + (i >> 5)] &= ~(1u << (i & 31));
  };
  auto bit_get = [&](int which, int d, int t, int i) -> bool {
    return (cube[((which * D + d) * T + t) * W + (i >> 5)] >> (i & 31)) & 1u;
  };

  for (int64_t k = static_cast<int64_t>(blockIdx.x) * kRoundWarps + wid; k < a.n;
       k += static_cast<int64_t>(gridDim.x) * kRoundWarps) {
    const uint64_t c = static_cast<uint64_t>(a.first + k);
    if (a.base)
      for (int i = lane; i < words; i += 32) cube[i] = a.base[i];
    __syncwarp();
    if (a.base) {
      // local search around a base schedule: devices from its diagonal, then
      // (probability 1/2) one op moved with its saves to another device, then
      // the drop-and-recompute edits below
      for (int i = lane; i < T; i += 32) {
        int d0 = 0;
        for (int d = D - 1; d >= 0; --d)
          if (bit_get(0, d, i, i)) d0 = d;
        dev[i] = d0;
      }
      __syncwarp();
      if (lane == 0) {
        Philox rng(a.seed, c, 0x2u);
        if (D > 1 && T > 1 && rng.uniform() < 0.5) {
          const int i = 1 + rng.below(T - 1), from = dev[i];
          const int to = (from + 1 + rng.below(D - 1)) % D;
          if (a.cost[to * T + i] < 1.0e9) {
            bclr(0, from, i, i);
            bset(0, to, i, i);
            for (int t = i + 1; t < T; ++t)
              if (bit_get(1, from, t, i)) {
                bclr(1, from, t, i);
                bset(1, to, t, i);
              }
            dev[i] = to;
          }
        }
      }
      __syncwarp();
    }
    // 1. placement, one Philox stream per (candidate, op)
    for (int i = lane; i < T && !a.base; i += 32) {
      dev[i] = place_op(a, c, i);
    }
    __syncwarp();
    // 2. diagonal + minimal-save
    if (!a.base) {
      if (a.word_build) build_minimal_save(cube, dev, alive, tq, dm, D, T, W, lane);
      else build_minimal_save_bits(cube, dev, last, D, T, W, lane);
    }
    // 3-4. drop-and-recompute edits and perturbation (lane 0, sequential)
    edit_candidate<true>(a, cube, dev, cons, last, elig, *n_elig, c, a.base == nullptr && !a.slow_scan);
    __syncwarp();
    uint32_t* out = a.out + static_cast<size_t>(k) * words;
    for (int i = lane; i < words; i += 32) out[i] = cube[i];
    __syncwarp();
  }
}

// The rounding path (no base cube) with one lane per candidate for the
// sequential part: a warp builds 32 candidates' placements and minimal saves
// (lanes over operators, one candidate after another), then every lane runs
// steps 3-4 on its own candidate's cube, then the 32 cubes leave with
// coalesced stores.  Same Philox streams and the same edit code as
// round_kernel, so the same cubes; used when 32 cubes per warp fit in shared
// memory.
__global__ void __launch_bounds__(256) round_batch_kernel(const RoundArgs a, int warps, int B) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int D = a.D, T = a.T, W = a.W32;
  const int words = 2 * D * T * W, stride = words + T;  // per candidate: cube, then dev
  uint32_t* cons = reinterpret_cast<uint32_t*>(smem);
  int* last = reinterpret_cast<int*>(cons + T * W);
  int* elig = last + T;
  int* n_elig = elig + T;
  uint32_t* alive = reinterpret_cast<uint32_t*>(n_elig + 1);  // [T][W]: i < t <= last[i]
  uint16_t* tq = reinterpret_cast<uint16_t*>(alive + T * W);     // [T*W]: t of word q
  uint32_t* wbuf = alive + T * W + (T * W + 1) / 2 + static_cast<size_t>(wid) * B * stride;
  uint32_t* dm = alive + T * W + (T * W + 1) / 2 + static_cast<size_t>(warps) * B * stride + wid * D * W;  // [D][W] ops per device
  for (int i = threadIdx.x; i < T * W; i += blockDim.x) cons[i] = 0u;
  for (int i = threadIdx.x; i < T; i += blockDim.x) last[i] = -1;
  __syncthreads();
  for (int e = threadIdx.x; e < a.E; e += blockDim.x) {
    atomicOr(&cons[a.src[e] * W + (a.dst[e] >> 5)], 1u << (a.dst[e] & 31));
    atomicMax(&last[a.src[e]], a.dst[e]);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int ne = 0;
    for (int j = 0; j < T; ++j)
      if (last[j] > j + 1) elig[ne++] = j;
    *n_elig = ne;
  }
  build_alive(alive, tq, last, T, W);
  __syncthreads();
  const int n_el = *n_elig;
  for (int64_t k0 = (static_cast<int64_t>(blockIdx.x) * warps + wid) * B; k0 < a.n;
       k0 += static_cast<int64_t>(gridDim.x) * warps * B) {
    const int nb = static_cast<int>(a.n - k0 < B ? a.n - k0 : B);
    for (int j = 0; j < nb; ++j) {
      const uint64_t c = static_cast<uint64_t>(a.first + k0 + j);
      uint32_t* cube = wbuf + static_cast<size_t>(j) * stride;
      int* dev = reinterpret_cast<int*>(cube + words);
      // 1. placement, one Philox stream per (candidate, op)
      for (int i = lane; i < T; i += 32) {
        dev[i] = place_op(a, c, i);
      }
      __syncwarp();
      // 2. diagonal + minimal-save, word by word (measured faster here at
      // every cube size the batched kernel takes)
      build_minimal_save(cube, dev, alive, tq, dm, D, T, W, lane);
    }
    // 3-4. one lane per candidate
    if (lane < nb) {
      uint32_t* cube = wbuf + static_cast<size_t>(lane) * stride;
      edit_candidate<false>(a, cube, reinterpret_cast<const int*>(cube + words), cons, last, elig, n_el,
                     static_cast<uint64_t>(a.first + k0 + lane), !a.slow_scan);
    }
    __syncwarp();
    uint32_t* out = a.out + static_cast<size_t>(k0) * words;
    for (int j = 0; j < nb; ++j) {
      const uint32_t* cube = wbuf + static_cast<size_t>(j) * stride;
      for (int i = lane; i < words; i += 32) out[static_cast<size_t>(j) * words + i] = cube[i];
    }
    __syncwarp();
  }
}

// Uniform random placements (K2b input, config 5's sweep): op i on a device
// drawn uniformly from those that can run it (cost below the 1e9 sentinel);
// one Philox block per (candidate, 4 consecutive ops), so a placement is a
// pure function of (seed, global index) like the cubes.
__global__ void placement_kernel(const uint8_t* allowed, const uint8_t* n_allowed, int D, int T, uint64_t seed,
                                 int64_t first, int64_t n, uint8_t* out) {
  const int64_t quads = (T + 3) / 4;
  const int64_t total = n * quads;
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < total;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = k / quads;
    const int q = static_cast<int>(k % quads);
    Philox rng(seed, static_cast<uint64_t>(first + c), 0x20000u + static_cast<uint32_t>(q));
    const uint4 r = rng.next();
    const uint32_t rv[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = 4 * q + j;
      if (i >= T) break;
      const int cnt = n_allowed[i];
      const int pick = static_cast<int>((static_cast<uint64_t>(rv[j]) * cnt) >> 32);
      out[c * T + i] = allowed[i * D + pick];
    }
  }
}


// ---------------------------------------------------------------------------
// R-space neighbours with canonical saves (local search over recomputation).
// A schedule is determined by its computations R; given R, the canonical
// saves keep each tensor on the device of its latest computation for exactly
// the steps where it is needed before it is computed again:
//   hold(u, t)  <=>  next_need(u, t) < next_comp(u, t)
// with next_need = first step >= t computing a consumer of u (any device) and
// next_comp = first step >= t computing u (any device).  Saves never move a
// tensor between devices (EQ11), and a holder beyond these steps only adds
// memory and copy charges (P = R(dc) and Z(ds), every ds != dc holding u).
// Moves (Philox keyed by (seed, candidate)): 0..max_moves of
//   A  recompute u where a consumer v is computed (step and device of one of
//      v's computations; with probability 1/2 on another device), and with
//      probability 1/2 its parents there too, recursively (each on the
//      child's device or, probability 1/4, another): a recomputation chain,
//   B  drop one recomputation (an R bit off the diagonal),
//   C  move one computation (any R bit) to another device.
// max_moves = 0 returns the base with its canonical saves.  Several bases
// (independent local-search chains): candidate k starts from base
// k / per_base.
struct MoveArgs {
  const double* cost;  // [D][T]
  const int32_t* src;
  const int32_t* dst;
  const int32_t* in_ptr;
  const int32_t* in_edge;
  const uint32_t* base;
  int64_t per_base;
  int D, T, E, W32;
  uint64_t seed;
  int64_t first, n;
  int max_moves;
  uint32_t* out;
};

__global__ void __launch_bounds__(kRoundWarps * 32) move_kernel(const MoveArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int D = a.D, T = a.T, W = a.W32;
  const int words = 2 * D * T * W;
  uint32_t* cons = reinterpret_cast<uint32_t*>(smem);  // [T][W] consumers of u
  uint32_t* par = cons + T * W;                        // [T][W] parents of v
  uint32_t* cube = par + T * W + wid * (words + 2 * T * W);
  uint32_t* rany = cube + words;  // [T][W] ops computed at t (any device)
  uint32_t* hbuf = rany + T * W;  // [T][W] hold(., t)
  for (int i = threadIdx.x; i < 2 * T * W; i += blockDim.x) cons[i] = 0u;
  __syncthreads();
  for (int e = threadIdx.x; e < a.E; e += blockDim.x) {
    atomicOr(&cons[a.src[e] * W + (a.dst[e] >> 5)], 1u << (a.dst[e] & 31));
    atomicOr(&par[a.dst[e] * W + (a.src[e] >> 5)], 1u << (a.src[e] & 31));
  }
  __syncthreads();
  auto rw = [&](int d, int t, int i) -> uint32_t& { return cube[(d * T + t) * W + (i >> 5)]; };
  auto rget = [&](int d, int t, int i) -> bool { return (rw(d, t, i) >> (i & 31)) & 1u; };

  for (int64_t k = static_cast<int64_t>(blockIdx.x) * kRoundWarps + wid; k < a.n;
       k += static_cast<int64_t>(gridDim.x) * kRoundWarps) {
    const uint64_t c = static_cast<uint64_t>(a.first + k);
    const uint32_t* bc = a.base + static_cast<size_t>(k / a.per_base) * words;
    for (int i = lane; i < words; i += 32) cube[i] = i < D * T * W ? bc[i] : 0u;
    __syncwarp();
    // moves: every lane steps through them together; Philox draws stay on
    // lane 0 (in the serial order) and are broadcast, and the R-bit counts
    // of drop/move picks are split over the lanes (a block of rows each, an
    // exclusive scan, the owning lane resolves the bit)
    if (a.max_moves > 0) {
      Philox rng(a.seed, c, 0x3u);
      const int nm = __shfl_sync(0xffffffffu, lane == 0 ? 1 + rng.below(a.max_moves) : 0, 0);
      const int nrows = D * T, blk = (nrows + 31) / 32;
      for (int m = 0; m < nm; ++m) {
        const double u = __shfl_sync(0xffffffffu, lane == 0 ? rng.uniform() : 0.0, 0);
        if (u < 0.4) {  // A: recompute a parent where its consumer is computed (lane 0)
          if (lane == 0) do {
              const int e = rng.below(a.E);
              const int pu = a.src[e], v = a.dst[e];
              int cnt = 0;
              for (int d = 0; d < D; ++d)
                for (int t = v; t < T; ++t) cnt += rget(d, t, v);
              if (!cnt) continue;
              int pick = rng.below(cnt), dv = 0, tv = 0;
              for (int d = 0; d < D && pick >= 0; ++d)
                for (int t = v; t < T && pick >= 0; ++t)
                  if (rget(d, t, v) && pick-- == 0) dv = d, tv = t;
              int dr = dv;
              if (D > 1 && rng.uniform() < 0.5) dr = (dv + 1 + rng.below(D - 1)) % D;
              if (a.cost[dr * T + pu] >= 1.0e9) dr = dv;
              if (a.cost[dr * T + pu] >= 1.0e9) continue;
              rw(dr, tv, pu) |= 1u << (pu & 31);
              if (rng.uniform() < 0.5) {
                int stack[32], sdev[32], sp = 0;
                stack[sp] = pu;
                sdev[sp++] = dr;
                while (sp > 0) {
                  --sp;
                  const int x = stack[sp], dx = sdev[sp];
                  for (int q = a.in_ptr[x]; q < a.in_ptr[x + 1]; ++q) {
                    const int pp = a.src[a.in_edge[q]];
                    if (rng.uniform() >= 0.5) continue;
                    int dp = dx;
                    if (D > 1 && rng.uniform() < 0.25) dp = (dx + 1 + rng.below(D - 1)) % D;
                    if (a.cost[dp * T + pp] >= 1.0e9) dp = dx;
                    if (a.cost[dp * T + pp] >= 1.0e9 || rget(dp, tv, pp)) continue;
                    rw(dp, tv, pp) |= 1u << (pp & 31);
                    if (sp < 32) {
                      stack[sp] = pp;
                      sdev[sp++] = dp;
                    }
                  }
                }
              }
          } while (false);
          __syncwarp();
          continue;
        }
        // B / C: pick an R bit (B: off the diagonal)
        const bool drop = u < 0.65;
        auto row_bits = [&](int r, int w) {
          const int t = r % T;
          uint32_t x = cube[r * W + w];
          if (drop && (t >> 5) == w) x &= ~(1u << (t & 31));
          return x;
        };
        int mine = 0;
        for (int r = lane * blk; r < min(nrows, (lane + 1) * blk); ++r)
          for (int w = 0; w < W; ++w) mine += __popc(row_bits(r, w));
        int incl = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += v;
        }
        const int cnt = __shfl_sync(0xffffffffu, incl, 31);
        if (!cnt) continue;
        const int pick = __shfl_sync(0xffffffffu, lane == 0 ? rng.below(cnt) : 0, 0);
        const int excl = incl - mine;
        int code = -1;  // (r * W + w) * 32 + bit
        if (pick >= excl && pick < incl) {
          int rem = pick - excl;
          for (int r = lane * blk; r < min(nrows, (lane + 1) * blk) && code < 0; ++r)
            for (int w = 0; w < W && code < 0; ++w) {
              uint32_t x = row_bits(r, w);
              const int pc = __popc(x);
              if (rem < pc) {
                for (int q = 0; q < rem; ++q) x &= x - 1;
                code = (r * W + w) * 32 + __ffs(x) - 1;
              }
              rem -= pc;
            }
        }
        const unsigned own = __ballot_sync(0xffffffffu, code >= 0);
        code = __shfl_sync(0xffffffffu, code, __ffs(own) - 1);
        if (lane == 0) {
          const int r = code / 32 / W, w = (code / 32) % W;
          const int pd = r / T, pt = r % T, pi = w * 32 + (code & 31);
          rw(pd, pt, pi) &= ~(1u << (pi & 31));
          if (!drop) {
            int to = pd;
            if (D > 1) to = (pd + 1 + rng.below(D - 1)) % D;
            if (a.cost[to * T + pi] >= 1.0e9) to = pd;
            rw(to, pt, pi) |= 1u << (pi & 31);
          }
        }
        __syncwarp();
      }
    }
    __syncwarp();
    // canonical saves, bit-parallel over the ops (lane w < W owns word w):
    //   need_t = parents of the ops computed at t, comp_t = ops computed at t
    //   backward: H_t = ~comp_t & (need_t | H_{t+1})   (hold(u,t) = bit u of H_t:
    //             the next need comes before the next computation)
    //   forward:  own_d = ops whose latest computation so far ran on d (lowest
    //             d among simultaneous ones); S(d,t) = H_t & own_d
    for (int i = lane; i < T * W; i += 32) {
      const int t = i / W, w = i % W;
      uint32_t x = 0u;
      for (int d = 0; d < D; ++d) x |= cube[(d * T + t) * W + w];
      rany[i] = x;
    }
    __syncwarp();
    if (lane < W) {
      const int w = lane;
      uint32_t H = 0u;
      for (int t = T - 1; t >= 0; --t) {
        uint32_t need = 0u;
        for (int ww = 0; ww < W; ++ww)
          for (uint32_t b = rany[t * W + ww]; b; b &= b - 1) need |= par[(ww * 32 + __ffs(b) - 1) * W + w];
        H = ~rany[t * W + w] & (need | H);
        hbuf[t * W + w] = H;
      }
      uint32_t own[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
      for (int t = 0; t < T; ++t) {
        const uint32_t Ht = hbuf[t * W + w], comp = rany[t * W + w];
        uint32_t taken = 0u;
#pragma unroll
        for (int d = 0; d < 8; ++d) {
          if (d >= D) break;
          cube[((D + d) * T + t) * W + w] = Ht & own[d];
          const uint32_t r = cube[(d * T + t) * W + w] & ~taken;
          own[d] = (own[d] & ~comp) | r;
          taken |= r;
        }
      }
    }
    __syncwarp();
    uint32_t* out = a.out + static_cast<size_t>(k) * words;
    for (int i = lane; i < words; i += 32) out[i] = cube[i];
    __syncwarp();
  }
}

// Placement-space neighbours (config 5's local search): neighbour k copies
// base k / per_base and moves 1..max_moves random ops to a random device
// that can run them (a draw of a device that cannot leaves the op where it
// is).  One warp per neighbour: 16-byte copies by all lanes, the moves by
// lane 0 (Philox keyed by (seed, first + k)).
__global__ void __launch_bounds__(256) placement_moves_kernel(const uint8_t* __restrict__ base, int64_t per_base,
                                                              const uint8_t* __restrict__ allowed, int D, int T,
                                                              uint64_t seed, int64_t first, int64_t n, int max_moves,
                                                              uint8_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const bool vec = (T % 16) == 0 && (reinterpret_cast<uintptr_t>(base) % 16) == 0 &&
                   (reinterpret_cast<uintptr_t>(out) % 16) == 0;
  for (int64_t k = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; k < n; k += nw) {
    const uint8_t* src = base + (k / per_base) * T;
    uint8_t* dst = out + k * T;
    if (vec) {
      for (int i = lane; i < T / 16; i += 32)
        reinterpret_cast<uint4*>(dst)[i] = __ldg(reinterpret_cast<const uint4*>(src) + i);
    } else {
      for (int i = lane; i < T; i += 32) dst[i] = src[i];
    }
    __syncwarp();
    if (lane == 0) {
      Philox rng(seed, static_cast<uint64_t>(first + k), 0x4u);
      const int nm = 1 + rng.below(max_moves);
      for (int m = 0; m < nm; ++m) {
        const int i = rng.below(T), d = rng.below(D);
        if (allowed[i * D + d]) dst[i] = static_cast<uint8_t>(d);
      }
    }
    __syncwarp();
  }
}
}  // namespace

void random_placements_device(const xe_problem* pr, uint64_t seed, int64_t first, int64_t n, uint8_t* out,
                              cudaStream_t s) {
  const HostProblem& h = pr->h;
  std::vector<uint8_t> allowed(static_cast<size_t>(h.T) * h.D, 0), cnt(static_cast<size_t>(h.T), 0);
  for (int i = 0; i < h.T; ++i) {
    int best = 0;
    for (int d = 0; d < h.D; ++d) {
      const double c = h.cost[static_cast<size_t>(d) * h.T + i];
      if (c < h.cost[static_cast<size_t>(best) * h.T + i]) best = d;
      if (c < 1.0e9) allowed[static_cast<size_t>(i) * h.D + cnt[static_cast<size_t>(i)]++] = static_cast<uint8_t>(d);
    }
    if (!cnt[static_cast<size_t>(i)]) {  // every device prohibitive: the cheapest
      allowed[static_cast<size_t>(i) * h.D] = static_cast<uint8_t>(best);
      cnt[static_cast<size_t>(i)] = 1;
    }
  }
  DevBuf<uint8_t> d_allowed, d_cnt;
  d_allowed.upload(allowed, s);
  d_cnt.upload(cnt, s);
  int nsm = 0;
  XE_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, pr->device));
  if (n > 0) {
    placement_kernel<<<nsm * 16, 256, 0, s>>>(d_allowed.p, d_cnt.p, h.D, h.T, seed, first, n, out);
    XE_CUDA(cudaGetLastError());
  }
  XE_CUDA(cudaStreamSynchronize(s));  // the tables above are freed on return
}

void round_cubes_device(const xe_problem* pr, const double* x, uint64_t seed, int64_t first,
                        int64_t n, int edits, double perturb, uint32_t* out, cudaStream_t s,
                        const uint32_t* base) {
  const HostProblem& h = pr->h;
  RoundArgs a{};
  a.base = base;
  a.mass = pr->d_mass.p;
  a.cost = pr->d_cost.p;
  a.src = pr->d_src.p;
  a.dst = pr->d_dst.p;
  a.in_ptr = pr->d_in_ptr.p;
  a.in_edge = pr->d_in_edge.p;
  a.x = x;
  DevBuf<int32_t> rc_code;
  DevBuf<double> rc_cdf;
  if (x) {  // LP off-diagonal R (columns (d*T + t)*T + i, t > i) with weight > 1e-6
    const size_t nr = static_cast<size_t>(h.D) * h.T * h.T;
    std::vector<double> xr(nr);
    XE_CUDA(cudaMemcpyAsync(xr.data(), x, nr * 8, cudaMemcpyDeviceToHost, s));
    XE_CUDA(cudaStreamSynchronize(s));
    std::vector<int32_t> code;
    std::vector<double> cdf;
    double acc = 0.0;
    for (int d = 0; d < h.D; ++d)
      for (int t = 1; t < h.T; ++t)
        for (int i = 0; i < t; ++i) {
          const double v = xr[(static_cast<size_t>(d) * h.T + t) * h.T + i];
          if (v > 1e-6 && h.cost[static_cast<size_t>(d) * h.T + i] < 1.0e9) {
            acc += v;
            code.push_back((d * h.T + t) * h.T + i);
            cdf.push_back(acc);
          }
        }
    if (!code.empty()) {
      rc_code.upload(code, s);
      rc_cdf.upload(cdf, s);
      a.rc_code = rc_code.p;
      a.rc_cdf = rc_cdf.p;
      a.n_rc = static_cast<int>(code.size());
    }
  }
  a.D = h.D;
  a.T = h.T;
  a.E = h.E;
  a.W32 = (h.T + 31) / 32;
  a.seed = seed;
  a.first = first;
  a.n = n;
  a.edits = edits;
  a.perturb = perturb;
  a.out = out;
  const int words = 2 * h.D * h.T * a.W32;
  DevBuf<uint8_t> okn, okl, chp;
  DevBuf<double> lpc;
  if (h.D <= 8) {
    std::vector<uint8_t> n(static_cast<size_t>(h.T)), l(static_cast<size_t>(h.T) * 8, 0), ch(static_cast<size_t>(h.T));
    for (int i = 0; i < h.T; ++i) {
      int k = 0, best = 0;
      for (int d = 0; d < h.D; ++d) {
        const double cd = h.cost[static_cast<size_t>(d) * h.T + i];
        if (cd < 1.0e9) l[static_cast<size_t>(i) * 8 + k++] = static_cast<uint8_t>(d);
        if (cd < h.cost[static_cast<size_t>(best) * h.T + i]) best = d;
      }
      n[static_cast<size_t>(i)] = static_cast<uint8_t>(k);
      ch[static_cast<size_t>(i)] = static_cast<uint8_t>(best);
    }
    okn.upload(n, s);
    okl.upload(l, s);
    chp.upload(ch, s);
    a.ok_n = okn.p;
    a.ok_list = okl.p;
    a.cheap = chp.p;
    if (a.x) {
      lpc.alloc(static_cast<size_t>(h.T) * 8);
      lp_cum_kernel<<<(h.T + 127) / 128, 128, 0, s>>>(a.x, a.r_base, okn.p, okl.p, h.T, lpc.p);
      XE_CUDA(cudaGetLastError());
      a.lp_cum = lpc.p;
    }
  }
  {  // word-by-word steps 1-2 when the saved bits outnumber the cube's words
    int64_t saves = 0;
    std::vector<int> lastc(static_cast<size_t>(h.T), -1);
    for (int e = 0; e < h.E; ++e)
      lastc[static_cast<size_t>(h.src[static_cast<size_t>(e)])] =
          std::max(lastc[static_cast<size_t>(h.src[static_cast<size_t>(e)])], h.dst[static_cast<size_t>(e)]);
    for (int i = 0; i < h.T; ++i) saves += std::max(0, lastc[static_cast<size_t>(i)] - i);
    a.word_build = saves > words ? 1 : 0;
    if (const char* e = std::getenv("XE_ROUND_WORD")) a.word_build = e[0] == '1';
    const char* sc = std::getenv("XE_ROUND_SLOW_SCAN");
    a.slow_scan = sc && sc[0] == '1';
  }
  const int smem = (2 * h.T * a.W32 + (h.T * a.W32 + 1) / 2 + 2 * h.T + 1 + kRoundWarps * (words + h.T + h.D * a.W32)) * 4;
  int limit = 0;
  XE_CUDA(cudaDeviceGetAttribute(&limit, cudaDevAttrMaxSharedMemoryPerBlockOptin, pr->device));
  {  // lane per candidate when 32 cubes per warp fit (base cubes keep round_kernel)
    const int tables = (2 * h.T * a.W32 + (h.T * a.W32 + 1) / 2 + 2 * h.T + 1) * 4;  // cons, last, elig, n_elig, alive, tq
    const char* e = std::getenv("XE_ROUND_BATCH");
    const int B = e ? std::max(0, std::min(32, std::atoi(e))) : 6;  // candidates per warp (0: round_kernel); 6 measured best
    const int per_warp = B * (words + h.T) * 4 + h.D * a.W32 * 4;
    const int warps = B > 0 ? std::min(8, (limit - tables) / std::max(1, per_warp)) : 0;
    // below 4 warps per CTA (large cubes: ResNet-50 holds one) the warp per
    // candidate kernel keeps more candidates in flight
    if (!base && warps >= 4) {
      const int bsmem = tables + warps * per_warp;
      XE_CUDA(cudaFuncSetAttribute(round_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bsmem));
      int nsm = 0;
      XE_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, pr->device));
      int per_sm = 0;
      XE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, round_batch_kernel, warps * 32, bsmem));
      const int64_t want = (n + static_cast<int64_t>(B) * warps - 1) / (static_cast<int64_t>(B) * warps);
      const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, static_cast<int64_t>(nsm) * std::max(1, per_sm))));
      if (n > 0) {
        round_batch_kernel<<<grid, warps * 32, bsmem, s>>>(a, warps, B);
        XE_CUDA(cudaGetLastError());
      }
      if (a.n_rc > 0 || a.ok_n) XE_CUDA(cudaStreamSynchronize(s));  // call-local tables
      return;
    }
  }
  if (smem > limit) fail(XE_ERR_TOO_LARGE, "candidate cube too large for the rounding kernel");
  XE_CUDA(cudaFuncSetAttribute(round_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int nsm = 0;
  XE_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, pr->device));
  const int64_t want = (n + kRoundWarps - 1) / kRoundWarps;
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, nsm * 16)));
  if (n > 0) {
    round_kernel<<<grid, kRoundWarps * 32, smem, s>>>(a);
    XE_CUDA(cudaGetLastError());
  }
  if (a.n_rc > 0 || a.ok_n) XE_CUDA(cudaStreamSynchronize(s));  // the recompute list / device tables are call-local
}

// shared memory of the move kernel: consumer masks + per warp a cube and the
// ops-computed-at-t rows
int move_smem_bytes(const HostProblem& h) {
  const int W = (h.T + 31) / 32, words = 2 * h.D * h.T * W;
  return (2 * h.T * W + kRoundWarps * (words + 2 * h.T * W)) * 4;
}

bool move_supported(const xe_problem* pr) {
  int limit = 0;
  XE_CUDA(cudaDeviceGetAttribute(&limit, cudaDevAttrMaxSharedMemoryPerBlockOptin, pr->device));
  return pr->h.T <= 256 && move_smem_bytes(pr->h) <= limit;
}

void move_cubes_device(const xe_problem* pr, const uint32_t* base, int64_t n_base, uint64_t seed, int64_t first,
                       int64_t n, int max_moves, uint32_t* out, cudaStream_t s) {
  const HostProblem& h = pr->h;
  if (h.T > 256) fail(XE_ERR_TOO_LARGE, "R-space moves support T <= 256");
  MoveArgs a{};
  a.cost = pr->d_cost.p;
  a.src = pr->d_src.p;
  a.dst = pr->d_dst.p;
  a.in_ptr = pr->d_in_ptr.p;
  a.in_edge = pr->d_in_edge.p;
  a.base = base;
  a.per_base = std::max<int64_t>(1, n / std::max<int64_t>(1, n_base));
  a.D = h.D;
  a.T = h.T;
  a.E = h.E;
  a.W32 = (h.T + 31) / 32;
  a.seed = seed;
  a.first = first;
  a.n = n;
  a.max_moves = max_moves;
  a.out = out;
  const int smem = move_smem_bytes(h);
  int limit = 0;
  XE_CUDA(cudaDeviceGetAttribute(&limit, cudaDevAttrMaxSharedMemoryPerBlockOptin, pr->device));
  if (smem > limit) fail(XE_ERR_TOO_LARGE, "candidate cube too large for the move kernel");
  XE_CUDA(cudaFuncSetAttribute(move_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int nsm = 0;
  XE_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, pr->device));
  const int64_t want = (n + kRoundWarps - 1) / kRoundWarps;
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, nsm * 16)));
  if (n > 0) {
    move_kernel<<<grid, kRoundWarps * 32, smem, s>>>(a);
    XE_CUDA(cudaGetLastError());
  }
}

void move_placements_device(const xe_problem* pr, const uint8_t* base, int64_t n_base, uint64_t seed, int64_t first,
                            int64_t n, int max_moves, uint8_t* out, cudaStream_t s) {
  const HostProblem& h = pr->h;
  std::vector<uint8_t> allowed(static_cast<size_t>(h.T) * h.D, 0);
  for (int i = 0; i < h.T; ++i)
    for (int d = 0; d < h.D; ++d)
      allowed[static_cast<size_t>(i) * h.D + d] = h.cost[static_cast<size_t>(d) * h.T + i] < 1.0e9 ? 1 : 0;
  DevBuf<uint8_t> d_allowed;
  d_allowed.upload(allowed, s);
  int nsm = 0;
  XE_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, pr->device));
  if (n > 0) {
    const int64_t want = (n + 7) / 8;
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, static_cast<int64_t>(nsm) * 16)));
    placement_moves_kernel<<<grid, 256, 0, s>>>(base, std::max<int64_t>(1, n / std::max<int64_t>(1, n_base)),
                                                d_allowed.p, h.D, h.T, seed, first, n, max_moves, out);
    XE_CUDA(cudaGetLastError());
  }
  XE_CUDA(cudaStreamSynchronize(s));  // the allowed table is call-local
}

}  // namespace xe
