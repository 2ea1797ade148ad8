// SPDX-License-Identifier: Apache-2.0
// Internal declarations shared by the host runtime and the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/xengine_b200.h"

namespace xe {

// Error carried to the C-ABI boundary and turned into a status code there.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

#define XE_CUDA(call)                                                                    \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      ::xe::fail(XE_ERR_CUDA, std::string(#call) + " -> " + cudaGetErrorString(e_));     \
  } while (0)

void set_last_error(const std::string& m);

// Wraps a C-ABI body: exceptions become status codes + thread-local message.
template <class F>
int guard(F&& f) {
  try {
    f();
    return XE_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host out of memory");
    return XE_ERR_ARG;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return XE_ERR_ARG;
  }
}

// Owning device buffer.
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    release();
    p = o.p; n = o.n; o.p = nullptr; o.n = 0;
    return *this;
  }
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void alloc(size_t count) {
    if (count == n && p) return;
    release();
    if (count) XE_CUDA(cudaMalloc(&p, count * sizeof(T)));
    n = count;
  }
  // grow-only: keeps the buffer when it already holds count elements
  void reserve(size_t count) {
    if (p && count <= n) return;
    alloc(count);
  }
  void upload(const std::vector<T>& v, cudaStream_t s) {
    alloc(v.size());
    if (!v.empty()) XE_CUDA(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
  }
};

// ---------------------------------------------------------------------------
// Host problem (the loader's output): mirrors xengine::Problem
// (proj/include/xengine/problem.hpp:18-60) after copy_cost resolution.
// ---------------------------------------------------------------------------
struct HostProblem {
  int D = 0, T = 0, E = 0;
  std::vector<std::string> device_ids, op_names;
  std::vector<int64_t> mass;    // [T]
  std::vector<double> cost;     // [D][T]
  std::vector<int32_t> src, dst;
  std::vector<double> w;        // [E][D][D]
  std::vector<int64_t> budget;  // [D]
  bool has_energy = false;
  double alpha = 0, total_limit = 0, board = 0;
  bool has_total = false;
  std::vector<double> q;        // [D][T]
  std::vector<uint8_t> has_lim; // [D]
  std::vector<double> lim;      // [D]
  std::string missing_link;     // non-empty: some (edge, ds, dc) has no covering link
  std::vector<uint8_t> w_missing;  // [E][D][D] 1 = no link covers the copy (w = 0 there)
};

HostProblem load_problem_json(const std::string& text);  // loader.cpp
void validate(const HostProblem& p);                      // loader.cpp

// The parsed, validated document before copy-cost resolution: what the C++
// API's Problem holds (one JSON parser serves the C ABI and the C++ API).
struct DocLink {
  int from, to;  // -1 = any device
  double latency, rate;
};
struct ParsedDoc {
  std::string name;
  HostProblem p;  // devices, operators, edges (copies unresolved, no energy)
  std::vector<int64_t> ram;      // [D], -1 = absent
  std::vector<int32_t> pinned;   // [T], -1 = none
  std::vector<DocLink> links;
  std::vector<std::map<std::pair<int, int>, double>> overrides;  // per edge
};
ParsedDoc parse_problem_document(const std::string& text);  // loader.cpp
std::string format_number(double v);                        // mps_writer.cpp (mps_io.cpp:14-27)

// Forward network -> training graph (make_training_graph, problem.cpp:280-338,
// generalised from a layer chain to a forward DAG): op 0 = the input
// (prohibitive cost except on its home device), forward ops 1..F, the
// backward of forward op f at 2F+1-f.  Edges: forward edges (u -> f, inputs
// in listed order, f ascending), then per backward op j (ascending) the
// upstream gradients (from the backward of each consumer of f, ascending;
// from the last forward op when f has none) and the saved tensors (f's
// inputs in listed order).  On a chain this is the reference's edge order.
struct ForwardOp {
  std::string name;
  std::vector<int> inputs;  // 0 = the input tensor, k = forward op k (k < this op's index)
  int64_t bytes, bwd_bytes;
  std::vector<double> costs, bwd_costs;  // [D]
};
void expand_training_graph(int D, int64_t input_bytes, int input_home, const std::vector<ForwardOp>& fwd,
                           std::vector<std::string>& names, std::vector<int64_t>& bytes,
                           std::vector<std::vector<double>>& costs, std::vector<int32_t>& src,
                           std::vector<int32_t>& dst);  // loader.cpp

// Kernel-side problem image: all pointers are device pointers.  Built once
// per handle (problem.cu) and passed by value to kernels.
struct DevProblem {
  int D, T, E;
  int W32;          // u32 words per cube row
  int NW;           // u64 words per bit row
  int WE;           // u64 words per edge mask
  int NB;           // bytes per row for the mass byte tables
  int edges_by_dst; // edge order is non-decreasing in dst
  const int64_t* mass;     // [T]
  const uint64_t* pmask;   // [T][NW] parents of v
  const uint64_t* cons;    // [T][NW] consumers of u
  const int64_t* mtab;     // [NB][256] sum of masses of the set bits of one byte
  const int32_t* src;      // [E]
  const int32_t* dst;      // [E]
  const int32_t* in_ptr;   // [T+1] in-edges of v, ascending edge id
  const int32_t* in_edge;  // [E]
  const int64_t* budget;   // [D]
  const double* ubound;    // [D] b*(1+1e-6)+1e-6 (model.cpp:443)
  // objective term table: [cost D*T][copy E*D*D][alpha*q D*T]
  const double* table;     // serial mode (f64)
  const int64_t* tfix;     // exact mode: table * 2^fix_k (integers)
  int n_table;
  int fix_k;               // >= 0 -> exact fixed-point mode
  // energy
  int has_energy;
  const uint64_t* ebad;    // [D][NW] ENERGY_DEV row violated when R(d,t,i)=1
  const double* q;         // [D][T]
  int has_total;
  double total_rhs;        // total_limit - board (model.cpp:307-308)
};

// Exact re-score of a batch's near-best candidates (eval_stream.cu).
constexpr int kRefineCap = 4096;
struct RefineBuf {
  DevBuf<int64_t> list;
  DevBuf<int> cnt;
  DevBuf<uint32_t> canon;
  DevBuf<uint64_t> il;
  DevBuf<double> obj;
  DevBuf<uint32_t> flags;
};

}  // namespace xe

// Opaque handle of the C ABI.
struct xe_problem {
  int device = 0;
  cudaStream_t stream = nullptr;
  xe::HostProblem h;
  // device storage
  xe::DevBuf<int64_t> d_mass, d_mtab, d_budget;
  xe::DevBuf<uint64_t> d_pmask, d_cons, d_ebad;
  xe::DevBuf<int32_t> d_src, d_dst, d_in_ptr, d_in_edge;
  xe::DevBuf<double> d_ubound, d_table, d_q, d_cost, d_w;
  xe::DevBuf<int64_t> d_tfix;
  xe::DevBuf<int64_t> d_tfix_noenergy;
  xe::DevBuf<int64_t> d_tfix_place;
  // derived host tables
  std::vector<double> table;           // [n_table] with energy terms
  int fix_k_energy = -1, fix_k_plain = -1;
  int fix_k_place = -1;  // exact mode for placement candidates (tighter bound)
  xe::DevProblem dev{};                // fields filled for the energy-free view
  xe::DevProblem view(bool energy) const;
  // scratch for batched evaluation
  xe::DevBuf<uint8_t> scratch;
  // persistent staging of the canonical-layout and host entry points
  // (xe_eval_cubes, xe_eval_cubes_host): grown on demand, reused across calls
  struct Stage {
    xe::DevBuf<uint32_t> canon;
    xe::DevBuf<uint64_t> il;
    xe::DevBuf<double> obj;
    xe::DevBuf<int64_t> peak;
    xe::DevBuf<uint32_t> flags;
    xe::DevBuf<uint8_t> scratch;
    xe::RefineBuf refine;
    cudaStream_t stream = nullptr;
    // pinned host staging of a chunk's outputs (xe_eval_cubes_host): the
    // device->host copies stay asynchronous, the caller's arrays are filled
    // from here while later chunks run
    unsigned char* pinned = nullptr;
    size_t pinned_bytes = 0;
    ~Stage() {
      if (pinned) cudaFreeHost(pinned);
    }
  };
  Stage stage[2];
  xe::DevBuf<uint64_t> chunk_best;  // [chunks][3] best-of-chunk triples
  // objective order of the batched evaluators: false = the streaming
  // evaluator's per-timestep reassociation (within #terms * 2^-53 relative,
  // best-of-batch re-scored exactly), true = the reference's order for every
  // candidate (the reference-order kernels)
  bool exact_objective = false;
};

namespace xe {
void upload_problem(xe_problem* p);   // problem.cu
// eval_stream.cu: the interleaved layout (NW u64 words per bit row, T <= 256)
// and the streaming evaluator (K2a v5) with the exact best-of-batch re-score
bool il_layout_ok(const xe_problem* pr);
size_t il_bytes(int D, int T, int64_t n);
void cubes_to_il_device(const xe_problem* pr, const uint32_t* cubes, int64_t n, uint64_t* il, cudaStream_t s);
bool stream_supported(const xe_problem* pr, const xe_model_opts& opts);
bool stream_objective_exact(const xe_problem* pr);
int eval_stream_device(const xe_problem* pr, const xe_model_opts& opts, const uint64_t* il, int64_t n, double* obj,
                       int64_t* peak, uint32_t* flags, uint32_t valid_mask, uint64_t* best3, unsigned char* scratch,
                       cudaStream_t stream);
void refine_best_device(const xe_problem* pr, const xe_model_opts& opts, const uint64_t* src_il,
                        const uint32_t* src_canon, int64_t n, const double* obj, const uint32_t* flags,
                        uint32_t valid_mask, uint64_t* best3, RefineBuf& rb, unsigned char* scratch,
                        cudaStream_t s);
void il_to_canon_device(const xe_problem* pr, const uint64_t* il, int64_t first, int64_t n, uint32_t* canon,
                        cudaStream_t s);
// eval_il.cu: the reference-order lane-per-candidate evaluator (T <= 64)
bool il_supported(const xe_problem* pr);
void eval_il_device(const xe_problem* pr, const xe_model_opts& opts, const uint64_t* il, int64_t n, double* obj,
                    int64_t* peak, uint32_t* flags, uint32_t valid_mask, uint64_t* best3, unsigned char* scratch,
                    cudaStream_t stream);
void require_uploaded(const xe_problem* p);  // capi.cpp: device handle + cudaSetDevice
int exact_fix_k(const std::vector<double>& table, int T);
}  // namespace xe
