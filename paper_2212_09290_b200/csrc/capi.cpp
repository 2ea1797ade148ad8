// SPDX-License-Identifier: Apache-2.0
//
// C ABI (include/xengine_b200.h): handles, error mapping, host<->device
// plumbing.  No exceptions cross this boundary; every entry is wrapped in
// xe::guard.  There is no CPU fallback: without a CUDA device every compute
// entry point returns XE_ERR_NO_DEVICE.

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>

#include "xe_internal.hpp"

namespace xe {
thread_local std::string g_last_error;
void set_last_error(const std::string& m) { g_last_error = m; }

size_t eval_scratch_bytes(int device);
void eval_cubes_device(const xe_problem* pr, const xe_model_opts& opts, const uint32_t* cubes,
                       int64_t n, double* obj, int64_t* peak, uint32_t* flags, uint32_t valid_mask,
                       uint64_t* best3, unsigned char* scratch, cudaStream_t stream);
void move_cubes_device(const xe_problem* pr, const uint32_t* base, int64_t n_base, uint64_t seed, int64_t first,
                       int64_t n, int max_moves, uint32_t* out, cudaStream_t s);
void move_placements_device(const xe_problem* pr, const uint8_t* base, int64_t n_base, uint64_t seed, int64_t first,
                            int64_t n, int max_moves, uint8_t* out, cudaStream_t s);
void round_cubes_device(const xe_problem* pr, const double* x, uint64_t seed, int64_t first,
                        int64_t n, int edits, double perturb, uint32_t* out, cudaStream_t s,
                        const uint32_t* base = nullptr);
void random_placements_device(const xe_problem* pr, uint64_t seed, int64_t first, int64_t n, uint8_t* out,
                              cudaStream_t s);
void eval_placements_device(const xe_problem* pr, const uint8_t* dev, int64_t n, int policy, double* obj,
                            int64_t* peak, uint32_t* flags, uint32_t valid_mask, uint64_t* best3,
                            unsigned char* scratch, cudaStream_t s);
void assignment_oracle_device(const xe_problem* pr, double* best_obj, int32_t* best_dev, int64_t* n_eval,
                              cudaStream_t s);

int64_t model_cols(int D, int T, int E);  // complete.cu
void complete_cube_host(const xe_problem* pr, const xe_model_opts& o, const uint32_t* cube_host, double* x_host);
double objective_dense_host(const xe_problem* pr, const xe_model_opts& o, const double* x_host);

namespace {

void require_device(int device) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    fail(XE_ERR_NO_DEVICE, "no CUDA device available (the B200 path has no CPU fallback)");
  }
  if (device < 0 || device >= n) fail(XE_ERR_ARG, "device index out of range");
  XE_CUDA(cudaSetDevice(device));
}

template <class T>
std::vector<T> vec(const T* p, size_t n) {
  if (!p && n) fail(XE_ERR_ARG, "null array in problem description");
  return p ? std::vector<T>(p, p + n) : std::vector<T>();
}

xe_problem* make_handle(HostProblem&& h, int device) {
  require_device(device);
  auto pr = std::make_unique<xe_problem>();
  pr->device = device;
  pr->h = std::move(h);
  XE_CUDA(cudaStreamCreateWithFlags(&pr->stream, cudaStreamNonBlocking));
  upload_problem(pr.get());
  pr->scratch.alloc(eval_scratch_bytes(device));
  return pr.release();
}

}  // namespace

void require_uploaded(const xe_problem* p) {
  if (p->device < 0) fail(XE_ERR_NO_DEVICE, "host-only problem handle (xe_problem_parse_json)");
  XE_CUDA(cudaSetDevice(p->device));
}

namespace {

xe_model_opts opts_or_default(const xe_model_opts* o) {
  xe_model_opts d{};
  return o ? *o : d;
}

// Host->device copy through the driver API: page-locked buffers allocated by
// another CUDA runtime instance in the process (e.g. torch's pinned memory)
// are recognised by the driver and DMA'd directly; cudart's own tracking
// only knows its own allocations.
// (The entry point is fetched from the runtime, so the library does not
// link libcuda and still loads on GPU-less hosts.)
void h2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  using Fn = CUresult (*)(CUdeviceptr, const void*, size_t, CUstream);
  static Fn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuMemcpyHtoDAsync", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<Fn>(f);
  }();
  if (!fn) {
    XE_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
    return;
  }
  CUresult r = fn(reinterpret_cast<CUdeviceptr>(dst), src, bytes, reinterpret_cast<CUstream>(s));
  if (r != CUDA_SUCCESS) fail(XE_ERR_CUDA, "cuMemcpyHtoDAsync failed: " + std::to_string(static_cast<int>(r)));
}

void read_best(const uint64_t* dev3, cudaStream_t s, xe_best* best) {
  uint64_t hb[3];
  XE_CUDA(cudaMemcpyAsync(hb, dev3, sizeof hb, cudaMemcpyDeviceToHost, s));
  XE_CUDA(cudaStreamSynchronize(s));
  best->index = static_cast<int64_t>(hb[1]);
  best->n_valid = static_cast<int64_t>(hb[2]);
  double o;
  std::memcpy(&o, &hb[0], 8);
  best->obj = best->index >= 0 ? o : INFINITY;
}

// Candidates per staging chunk of the canonical/host paths: ~64 MB of cubes.
int64_t stage_chunk(const HostProblem& h) {
  const size_t cb = xe_cube_bytes(h.D, h.T);
  const int64_t c = static_cast<int64_t>((64ull << 20) / cb);
  return std::max<int64_t>(32, c & ~int64_t{31});
}

// Best over per-chunk (objective bits, chunk-local index, valid count)
// triples; chunks ascend in candidate index, so a strict < keeps the first.
// Returns false when a chunk reports more near-ties than the exact re-score
// holds (index -2): the caller re-runs the batch with the exact kernels.
bool combine_chunks(const uint64_t* dev, int64_t nchunks, int64_t chunk, cudaStream_t s, xe_best* best) {
  std::vector<uint64_t> hb(static_cast<size_t>(std::max<int64_t>(1, nchunks)) * 3);
  if (nchunks) {
    XE_CUDA(cudaMemcpyAsync(hb.data(), dev, static_cast<size_t>(nchunks) * 24, cudaMemcpyDeviceToHost, s));
    XE_CUDA(cudaStreamSynchronize(s));
  }
  best->index = -1;
  best->n_valid = 0;
  best->obj = INFINITY;
  uint64_t bk = ~0ull;
  for (int64_t c = 0; c < nchunks; ++c) {
    const int64_t idx = static_cast<int64_t>(hb[static_cast<size_t>(3 * c + 1)]);
    if (idx == -2) return false;
    best->n_valid += static_cast<int64_t>(hb[static_cast<size_t>(3 * c + 2)]);
    if (idx >= 0 && hb[static_cast<size_t>(3 * c)] < bk) {
      bk = hb[static_cast<size_t>(3 * c)];
      best->index = c * chunk + idx;
      std::memcpy(&best->obj, &bk, 8);
    }
  }
  return true;
}

}  // namespace
}  // namespace xe

using namespace xe;

extern "C" {

const char* xe_last_error(void) { return g_last_error.c_str(); }
const char* xe_version(void) { return "xengine_b200 0.1 (sm_100a)"; }

size_t xe_cube_bytes(int32_t D, int32_t T) {
  return static_cast<size_t>(8) * D * T * ((T + 31) / 32);
}

int xe_problem_load_json(const char* json_text, int device, xe_problem** out) {
  return guard([&] {
    if (!json_text || !out) fail(XE_ERR_ARG, "null argument");
    HostProblem h = load_problem_json(json_text);
    *out = make_handle(std::move(h), device);
  });
}

int xe_problem_parse_json(const char* json_text, xe_problem** out) {
  return guard([&] {
    if (!json_text || !out) fail(XE_ERR_ARG, "null argument");
    auto pr = std::make_unique<xe_problem>();
    pr->device = -1;
    pr->h = load_problem_json(json_text);
    *out = pr.release();
  });
}

int xe_problem_create(const xe_problem_desc* d, int device, xe_problem** out) {
  return guard([&] {
    if (!d || !out) fail(XE_ERR_ARG, "null argument");
    if (d->D <= 0 || d->T <= 0 || d->E < 0) fail(XE_ERR_DIMENSION_MISMATCH, "bad dimensions");
    HostProblem h;
    h.D = d->D;
    h.T = d->T;
    h.E = d->E;
    for (int i = 0; i < h.D; ++i) h.device_ids.push_back("d" + std::to_string(i));
    for (int i = 0; i < h.T; ++i) h.op_names.push_back("op" + std::to_string(i));
    h.mass = vec(d->output_bytes, static_cast<size_t>(h.T));
    h.cost = vec(d->cost_ms, static_cast<size_t>(h.D) * h.T);
    h.src = vec(d->edge_src, static_cast<size_t>(h.E));
    h.dst = vec(d->edge_dst, static_cast<size_t>(h.E));
    h.w = vec(d->copy_ms, static_cast<size_t>(h.E) * h.D * h.D);
    // NaN: no link covers the copy; raised when a model or a charged copy
    // needs it (copy_cost, problem.cpp:374-376)
    h.w_missing.assign(h.w.size(), 0);
    for (size_t k = 0; k < h.w.size(); ++k)
      if (std::isnan(h.w[k])) {
        const int a = static_cast<int>(k / h.D % h.D), b = static_cast<int>(k % h.D);
        if (a == b) fail(XE_ERR_ARG, "copy_ms must be finite on the diagonal");
        if (h.missing_link.empty())
          h.missing_link = "no link covers " + h.device_ids[static_cast<size_t>(a)] + "->" + h.device_ids[static_cast<size_t>(b)];
        h.w_missing[k] = 1;
        h.w[k] = 0.0;
      }
    h.budget = vec(d->budget_bytes, static_cast<size_t>(h.D));
    for (int64_t m : h.mass)
      if (m <= 0) fail(XE_ERR_NON_POSITIVE_SIZE, "output_bytes must be positive");
    for (int64_t b : h.budget)
      if (b <= 0) fail(XE_ERR_NON_POSITIVE_SIZE, "budget_bytes must be positive");
    for (double c : h.cost)
      if (c < 0) fail(XE_ERR_NEGATIVE_COST, "cost_ms must be non-negative");
    for (double c : h.w)
      if (c < 0) fail(XE_ERR_NEGATIVE_COST, "copy_ms must be non-negative");
    h.has_energy = d->has_energy != 0;
    h.q.assign(static_cast<size_t>(h.D) * h.T, 0.0);
    h.has_lim.assign(static_cast<size_t>(h.D), 0);
    h.lim.assign(static_cast<size_t>(h.D), 0.0);
    if (h.has_energy) {
      h.alpha = d->alpha;
      h.q = vec(d->q_joules, static_cast<size_t>(h.D) * h.T);
      if (d->has_dev_limit) h.has_lim = vec(d->has_dev_limit, static_cast<size_t>(h.D));
      if (d->dev_limit) h.lim = vec(d->dev_limit, static_cast<size_t>(h.D));
      h.has_total = d->has_total_limit != 0;
      h.total_limit = d->total_limit;
      h.board = d->board_joules;
    }
    validate(h);
    *out = make_handle(std::move(h), device);
  });
}

int xe_problem_destroy(xe_problem* p) {
  return guard([&] {
    if (!p) return;
    if (p->device >= 0) {
      cudaSetDevice(p->device);
      if (p->stream) cudaStreamDestroy(p->stream);
      for (auto& st : p->stage)
        if (st.stream) cudaStreamDestroy(st.stream);
    }
    delete p;
  });
}

const char* xe_problem_device_id(const xe_problem* p, int32_t d) {
  if (!p || d < 0 || d >= p->h.D || static_cast<size_t>(d) >= p->h.device_ids.size()) return nullptr;
  return p->h.device_ids[static_cast<size_t>(d)].c_str();
}

const char* xe_problem_op_name(const xe_problem* p, int32_t i) {
  if (!p || i < 0 || i >= p->h.T || static_cast<size_t>(i) >= p->h.op_names.size()) return nullptr;
  return p->h.op_names[static_cast<size_t>(i)].c_str();
}

int xe_problem_describe(const xe_problem* p, xe_problem_desc* o) {
  return guard([&] {
    if (!p || !o) fail(XE_ERR_ARG, "null argument");
    const HostProblem& h = p->h;
    std::memset(o, 0, sizeof *o);
    o->D = h.D;
    o->T = h.T;
    o->E = h.E;
    o->output_bytes = h.mass.data();
    o->cost_ms = h.cost.data();
    o->edge_src = h.src.data();
    o->edge_dst = h.dst.data();
    o->copy_ms = h.w.data();
    o->budget_bytes = h.budget.data();
    o->has_energy = h.has_energy;
    o->alpha = h.alpha;
    o->q_joules = h.q.data();
    o->has_dev_limit = h.has_lim.data();
    o->dev_limit = h.lim.data();
    o->has_total_limit = h.has_total;
    o->total_limit = h.total_limit;
    o->board_joules = h.board;
  });
}

int xe_problem_with_budgets(const xe_problem* p, const int64_t* budgets, xe_problem** out) {
  return guard([&] {
    if (!p || !budgets || !out) fail(XE_ERR_ARG, "null argument");
    HostProblem h = p->h;
    require_uploaded(p);
    for (int d = 0; d < h.D; ++d) {
      if (budgets[d] <= 0) fail(XE_ERR_NON_POSITIVE_SIZE, "budget for device " + h.device_ids[static_cast<size_t>(d)]);
      h.budget[static_cast<size_t>(d)] = budgets[d];
    }
    *out = make_handle(std::move(h), p->device);
  });
}

// Canonical device cubes, chunk by chunk through the interleaved staging
// buffer.  exact = the reference-order kernels (energy model; fallback).
static void eval_canon_chunks(const xe_problem* p, const xe_model_opts& o, const uint32_t* cubes, int64_t n,
                              xe_eval_out* out, uint32_t valid_mask, xe_best* best, cudaStream_t s, bool exact) {
  auto* mp = const_cast<xe_problem*>(p);
  const HostProblem& h = p->h;
  double* obj = out ? out->obj : nullptr;
  int64_t* peak = out ? out->peak : nullptr;
  uint32_t* flags = out ? out->flags : nullptr;
  const bool fast = !exact && stream_supported(p, o);
  if (!fast && !il_supported(p)) {  // T > 64, exact: the warp-per-candidate kernel on the canonical layout
    uint64_t* best3 = reinterpret_cast<uint64_t*>(mp->scratch.p + mp->scratch.n - 64);
    eval_cubes_device(p, o, cubes, n, obj, peak, flags, valid_mask, best ? best3 : nullptr, mp->scratch.p, s);
    if (best) read_best(best3, s, best);
    return;
  }
  const size_t cw = xe_cube_bytes(h.D, h.T) / 4;
  const int64_t chunk = stage_chunk(h);
  const int64_t nchunks = (n + chunk - 1) / chunk;
  auto& st = mp->stage[0];
  const int64_t cap = std::min(chunk, std::max<int64_t>(n, 1));
  st.il.reserve(il_bytes(h.D, h.T, cap) / 8);
  if (best) mp->chunk_best.reserve(static_cast<size_t>(std::max<int64_t>(1, nchunks)) * 3);
  const bool refine = fast && best && !stream_objective_exact(p);
  if (refine && !obj) st.obj.reserve(static_cast<size_t>(cap));
  if (refine && !flags) st.flags.reserve(static_cast<size_t>(cap));
  for (int64_t c = 0; c < nchunks; ++c) {
    const int64_t lo = c * chunk, m = std::min(chunk, n - lo);
    uint64_t* b3 = best ? mp->chunk_best.p + 3 * c : nullptr;
    cubes_to_il_device(p, cubes + lo * cw, m, st.il.p, s);
    if (fast) {
      double* o_obj = obj ? obj + lo : (refine ? st.obj.p : nullptr);
      uint32_t* o_fl = flags ? flags + lo : (refine ? st.flags.p : nullptr);
      eval_stream_device(p, o, st.il.p, m, o_obj, peak ? peak + lo * h.D : nullptr, o_fl, valid_mask, b3,
                         mp->scratch.p, s);
      if (refine)
        refine_best_device(p, o, nullptr, cubes + lo * cw, m, o_obj, o_fl, valid_mask, b3, st.refine, mp->scratch.p,
                           s);
    } else {
      eval_il_device(p, o, st.il.p, m, obj ? obj + lo : nullptr, peak ? peak + lo * h.D : nullptr,
                     flags ? flags + lo : nullptr, valid_mask, b3, mp->scratch.p, s);
    }
  }
  if (best && !combine_chunks(mp->chunk_best.p, nchunks, chunk, s, best))
    eval_canon_chunks(p, o, cubes, n, out, valid_mask, best, s, true);  // > kRefineCap near-ties
}

int xe_eval_cubes(const xe_problem* p, const xe_model_opts* opts, const uint32_t* cubes, int64_t n,
                  xe_eval_out* out, uint32_t valid_mask, xe_best* best, void* stream) {
  return guard([&] {
    if (!p || (!cubes && n > 0) || n < 0) fail(XE_ERR_ARG, "null argument");
    require_uploaded(p);
    eval_canon_chunks(p, opts_or_default(opts), cubes, n, out, valid_mask, best, static_cast<cudaStream_t>(stream),
                      false);
  });
}

int xe_eval_cubes_il(const xe_problem* p, const xe_model_opts* opts, const uint64_t* il, int64_t n,
                     xe_eval_out* out, uint32_t valid_mask, xe_best* best, void* stream) {
  return guard([&] {
    if (!p || (!il && n > 0) || n < 0) fail(XE_ERR_ARG, "null argument");
    require_uploaded(p);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    xe_model_opts o = opts_or_default(opts);
    auto* mp = const_cast<xe_problem*>(p);
    const HostProblem& h = p->h;
    uint64_t* best3 = reinterpret_cast<uint64_t*>(mp->scratch.p + mp->scratch.n - 64);
    double* obj = out ? out->obj : nullptr;
    int64_t* peak = out ? out->peak : nullptr;
    uint32_t* flags = out ? out->flags : nullptr;
    auto exact = [&] {  // reference-order kernels over the whole batch
      if (il_supported(p)) {
        eval_il_device(p, o, il, n, obj, peak, flags, valid_mask, best ? best3 : nullptr, mp->scratch.p, s);
        if (best) read_best(best3, s, best);
        return;
      }
      // T > 64: convert to canonical chunk by chunk and use the v3 kernel
      const size_t cw = xe_cube_bytes(h.D, h.T) / 4;
      const int64_t chunk = stage_chunk(h), nchunks = (n + chunk - 1) / chunk;
      auto& st = mp->stage[0];
      st.canon.reserve(static_cast<size_t>(std::min(chunk, std::max<int64_t>(n, 1))) * cw);
      if (best) mp->chunk_best.reserve(static_cast<size_t>(std::max<int64_t>(1, nchunks)) * 3);
      for (int64_t c = 0; c < nchunks; ++c) {
        const int64_t lo = c * chunk, m = std::min(chunk, n - lo);
        il_to_canon_device(p, il, lo, m, st.canon.p, s);
        eval_cubes_device(p, o, st.canon.p, m, obj ? obj + lo : nullptr, peak ? peak + lo * h.D : nullptr,
                          flags ? flags + lo : nullptr, valid_mask, best ? mp->chunk_best.p + 3 * c : nullptr,
                          mp->scratch.p, s);
      }
      if (best) combine_chunks(mp->chunk_best.p, nchunks, chunk, s, best);
    };
    if (!stream_supported(p, o)) {
      if (!il_supported(p) && o.use_energy && h.has_energy)
        fail(XE_ERR_TOO_LARGE, "interleaved cubes with the energy model need T <= 64");
      exact();
      return;
    }
    const bool refine = best && !stream_objective_exact(p);
    auto& st = mp->stage[0];
    if (refine && !obj) st.obj.reserve(static_cast<size_t>(std::max<int64_t>(n, 1)));
    if (refine && !flags) st.flags.reserve(static_cast<size_t>(std::max<int64_t>(n, 1)));
    double* o_obj = obj ? obj : (refine ? st.obj.p : nullptr);
    uint32_t* o_fl = flags ? flags : (refine ? st.flags.p : nullptr);
    eval_stream_device(p, o, il, n, o_obj, peak, o_fl, valid_mask, best ? best3 : nullptr, mp->scratch.p, s);
    if (refine) refine_best_device(p, o, il, nullptr, n, o_obj, o_fl, valid_mask, best3, st.refine, mp->scratch.p, s);
    if (best) {
      read_best(best3, s, best);
      if (best->index == -2) exact();  // more than kRefineCap near-ties
    }
  });
}

size_t xe_cube_il_bytes(int32_t D, int32_t T, int64_t n) { return il_bytes(D, T, n); }

int xe_objective_order_exact(const xe_problem* p, int32_t* exact) {
  return guard([&] {
    if (!p || !exact) fail(XE_ERR_ARG, "null argument");
    *exact = p->device >= 0 && (p->exact_objective || stream_objective_exact(p)) ? 1 : 0;
  });
}

int xe_problem_set_exact_objective(xe_problem* p, int32_t exact) {
  return guard([&] {
    if (!p) fail(XE_ERR_ARG, "null argument");
    p->exact_objective = exact != 0;
  });
}

int xe_cubes_to_il(const xe_problem* p, const uint32_t* cubes, int64_t n, uint64_t* il, void* stream) {
  return guard([&] {
    if (!p || ((!cubes || !il) && n > 0) || n < 0) fail(XE_ERR_ARG, "null argument");
    require_uploaded(p);
    cubes_to_il_device(p, cubes, n, il, static_cast<cudaStream_t>(stream));
  });
}

// End-to-end path: host candidates in, host results out.  Chunks alternate
// between two streams with their own staging buffers, so the host->device
// copy of chunk k+1 overlaps the transpose + evaluation of chunk k.
static void eval_host_chunks(const xe_problem* p, const xe_model_opts& o, const uint32_t* cubes, int64_t n,
                             xe_eval_out* out, uint32_t valid_mask, xe_best* best, bool exact) {
  auto* mp = const_cast<xe_problem*>(p);
  const HostProblem& h = p->h;
  const bool fast = !exact && stream_supported(p, o);
  const bool il = fast || il_supported(p);
  const bool refine = fast && !stream_objective_exact(p);
  const size_t cb = xe_cube_bytes(h.D, h.T);
  const int64_t chunk = il ? stage_chunk(h) : std::max<int64_t>(1024, static_cast<int64_t>((256ull << 20) / cb));
  const int64_t nchunks = (n + chunk - 1) / chunk;
  const int64_t cap = std::min(chunk, std::max<int64_t>(n, 1));
  const size_t sb = eval_scratch_bytes(p->device);
  for (auto& st : mp->stage) {
    if (!st.stream) XE_CUDA(cudaStreamCreateWithFlags(&st.stream, cudaStreamNonBlocking));
    st.canon.reserve(static_cast<size_t>(cap) * cb / 4);
    if (il) st.il.reserve(il_bytes(h.D, h.T, cap) / 8);
    if ((out && out->obj) || refine) st.obj.reserve(static_cast<size_t>(cap));
    if (out && out->peak) st.peak.reserve(static_cast<size_t>(cap) * h.D);
    if ((out && out->flags) || refine) st.flags.reserve(static_cast<size_t>(cap));
    st.scratch.reserve(sb);
  }
  mp->chunk_best.reserve(static_cast<size_t>(std::max<int64_t>(1, nchunks)) * 3);
  // the two stages' streams must not start before work already queued on
  // the handle's stream (previous calls) has finished with the buffers
  XE_CUDA(cudaStreamSynchronize(p->stream));
  // outputs: chunk c's results land in its stage's pinned buffer and are
  // copied to the caller's arrays once that stage comes round again
  const bool want = out && (out->obj || out->peak || out->flags);
  const size_t ob = static_cast<size_t>(cap) * (8 + 8 * static_cast<size_t>(h.D) + 4);
  if (want)
    for (auto& st : mp->stage)
      if (st.pinned_bytes < ob) {
        if (st.pinned) XE_CUDA(cudaFreeHost(st.pinned));
        st.pinned = nullptr;
        XE_CUDA(cudaMallocHost(reinterpret_cast<void**>(&st.pinned), ob));
        st.pinned_bytes = ob;
      }
  auto stage_obj = [&](xe_problem::Stage& st) { return reinterpret_cast<double*>(st.pinned); };
  auto stage_peak = [&](xe_problem::Stage& st) { return reinterpret_cast<int64_t*>(st.pinned + static_cast<size_t>(cap) * 8); };
  auto stage_fl = [&](xe_problem::Stage& st) {
    return reinterpret_cast<uint32_t*>(st.pinned + static_cast<size_t>(cap) * (8 + 8 * static_cast<size_t>(h.D)));
  };
  auto deliver = [&](int64_t c) {  // after stage (c & 1)'s stream finished chunk c
    auto& st = mp->stage[c & 1];
    const int64_t lo = c * chunk, m = std::min(chunk, n - lo);
    if (out->obj) std::memcpy(out->obj + lo, stage_obj(st), static_cast<size_t>(m) * 8);
    if (out->peak) std::memcpy(out->peak + lo * h.D, stage_peak(st), static_cast<size_t>(m) * h.D * 8);
    if (out->flags) std::memcpy(out->flags + lo, stage_fl(st), static_cast<size_t>(m) * 4);
  };
  try {
    for (int64_t c = 0; c < nchunks; ++c) {
      auto& st = mp->stage[c & 1];
      const int64_t lo = c * chunk, m = std::min(chunk, n - lo);
      if (want && c >= 2) {
        XE_CUDA(cudaStreamSynchronize(st.stream));
        deliver(c - 2);
      }
      uint64_t* b3 = mp->chunk_best.p + 3 * c;
      h2d(st.canon.p, reinterpret_cast<const unsigned char*>(cubes) + lo * cb, static_cast<size_t>(m) * cb,
          st.stream);
      double* o_obj = (out && out->obj) || refine ? st.obj.p : nullptr;
      uint32_t* o_fl = (out && out->flags) || refine ? st.flags.p : nullptr;
      if (fast) {
        cubes_to_il_device(p, st.canon.p, m, st.il.p, st.stream);
        eval_stream_device(p, o, st.il.p, m, o_obj, st.peak.p, o_fl, valid_mask, b3, st.scratch.p, st.stream);
        if (refine)
          refine_best_device(p, o, nullptr, st.canon.p, m, o_obj, o_fl, valid_mask, b3, st.refine, st.scratch.p,
                             st.stream);
      } else if (il) {
        cubes_to_il_device(p, st.canon.p, m, st.il.p, st.stream);
        eval_il_device(p, o, st.il.p, m, o_obj, st.peak.p, o_fl, valid_mask, b3, st.scratch.p, st.stream);
      } else {
        eval_cubes_device(p, o, st.canon.p, m, o_obj, st.peak.p, o_fl, valid_mask, b3, st.scratch.p, st.stream);
      }
      if (out && out->obj)
        XE_CUDA(cudaMemcpyAsync(stage_obj(st), st.obj.p, m * sizeof(double), cudaMemcpyDeviceToHost, st.stream));
      if (out && out->peak)
        XE_CUDA(cudaMemcpyAsync(stage_peak(st), st.peak.p, m * h.D * sizeof(int64_t), cudaMemcpyDeviceToHost,
                                st.stream));
      if (out && out->flags)
        XE_CUDA(cudaMemcpyAsync(stage_fl(st), st.flags.p, m * sizeof(uint32_t), cudaMemcpyDeviceToHost, st.stream));
    }
    XE_CUDA(cudaStreamSynchronize(mp->stage[0].stream));
    XE_CUDA(cudaStreamSynchronize(mp->stage[1].stream));
    if (want)
      for (int64_t c = std::max<int64_t>(0, nchunks - 2); c < nchunks; ++c) deliver(c);
  } catch (...) {
    cudaStreamSynchronize(mp->stage[0].stream);
    cudaStreamSynchronize(mp->stage[1].stream);
    throw;
  }
  if (best && !combine_chunks(mp->chunk_best.p, nchunks, chunk, p->stream, best))
    eval_host_chunks(p, o, cubes, n, out, valid_mask, best, true);  // > kRefineCap near-ties
}

int xe_eval_cubes_host(const xe_problem* p, const xe_model_opts* opts, const uint32_t* cubes,
                       int64_t n, xe_eval_out* out, uint32_t valid_mask, xe_best* best) {
  return guard([&] {
    if (!p || (!cubes && n > 0) || n < 0) fail(XE_ERR_ARG, "null argument");
    require_uploaded(p);
    xe_model_opts o = opts_or_default(opts);
    xe_best tmp;
    eval_host_chunks(p, o, cubes, n, out, valid_mask, best ? best : &tmp, false);
  });
}

int xe_round_cubes(const xe_problem* p, const double* x_dev, uint64_t seed, int64_t first,
                   int64_t n, int32_t edits, double perturb, uint32_t* cubes_dev, void* stream) {
  return guard([&] {
    if (!p || (!cubes_dev && n > 0) || n < 0 || edits < 0) fail(XE_ERR_ARG, "bad argument");
    require_uploaded(p);
    cudaStream_t s = static_cast<cudaStream_t>(stream);  // NULL = legacy default stream
    round_cubes_device(p, x_dev, seed, first, n, edits, perturb, cubes_dev, s);
  });
}

int xe_mutate_cubes(const xe_problem* p, const uint32_t* base_dev, uint64_t seed, int64_t first, int64_t n,
                    int32_t edits, double perturb, uint32_t* cubes_dev, void* stream) {
  return guard([&] {
    if (!p || !base_dev || (!cubes_dev && n > 0) || n < 0 || edits < 0) fail(XE_ERR_ARG, "bad argument");
    require_uploaded(p);
    round_cubes_device(p, nullptr, seed, first, n, edits, perturb, cubes_dev, static_cast<cudaStream_t>(stream),
                       base_dev);
  });
}

int xe_move_cubes(const xe_problem* p, const uint32_t* base_dev, int64_t n_base, uint64_t seed, int64_t first,
                  int64_t n, int32_t max_moves, uint32_t* cubes_dev, void* stream) {
  return guard([&] {
    if (!p || !base_dev || (!cubes_dev && n > 0) || n < 0 || max_moves < 0 || n_base < 1 || n % n_base)
      fail(XE_ERR_ARG, "bad argument (n must be a multiple of n_base >= 1)");
    require_uploaded(p);
    move_cubes_device(p, base_dev, n_base, seed, first, n, max_moves, cubes_dev, static_cast<cudaStream_t>(stream));
  });
}

int xe_move_placements(const xe_problem* p, const uint8_t* base_dev, int64_t n_base, uint64_t seed, int64_t first,
                       int64_t n, int32_t max_moves, uint8_t* dev_out, void* stream) {
  return guard([&] {
    if (!p || !base_dev || (!dev_out && n > 0) || n < 0 || max_moves < 1 || n_base < 1 || n % n_base)
      fail(XE_ERR_ARG, "bad argument (n must be a multiple of n_base >= 1, max_moves >= 1)");
    require_uploaded(p);
    move_placements_device(p, base_dev, n_base, seed, first, n, max_moves, dev_out, static_cast<cudaStream_t>(stream));
  });
}

int xe_random_placements(const xe_problem* p, uint64_t seed, int64_t first, int64_t n, uint8_t* dev_out,
                         void* stream) {
  return guard([&] {
    if (!p || (!dev_out && n > 0) || n < 0) fail(XE_ERR_ARG, "bad argument");
    require_uploaded(p);
    random_placements_device(p, seed, first, n, dev_out, static_cast<cudaStream_t>(stream));
  });
}

int xe_eval_placements(const xe_problem* p, const uint8_t* dev, int64_t n, int32_t policy, xe_eval_out* out,
                       uint32_t valid_mask, xe_best* best, void* stream) {
  return guard([&] {
    if (!p || (!dev && n > 0) || n < 0) fail(XE_ERR_ARG, "null argument");
    require_uploaded(p);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    auto* mp = const_cast<xe_problem*>(p);
    uint64_t* best3 = reinterpret_cast<uint64_t*>(mp->scratch.p + mp->scratch.n - 64);
    eval_placements_device(p, dev, n, policy, out ? out->obj : nullptr, out ? out->peak : nullptr,
                           out ? out->flags : nullptr, valid_mask, best ? best3 : nullptr, mp->scratch.p, s);
    if (best) read_best(best3, s, best);
  });
}

int64_t xe_model_cols(int32_t D, int32_t T, int32_t E) { return model_cols(D, T, E); }

int xe_complete_cube(const xe_problem* p, const xe_model_opts* opts, const uint32_t* cube, double* x) {
  return guard([&] {
    if (!p || !cube || !x) fail(XE_ERR_ARG, "null argument");
    require_uploaded(p);
    complete_cube_host(p, opts_or_default(opts), cube, x);
  });
}

int xe_objective_dense(const xe_problem* p, const xe_model_opts* opts, const double* x, double* obj) {
  return guard([&] {
    if (!p || !x || !obj) fail(XE_ERR_ARG, "null argument");
    require_uploaded(p);
    *obj = objective_dense_host(p, opts_or_default(opts), x);
  });
}

int xe_assignment_oracle(const xe_problem* p, double* best_obj, int32_t* best_dev, int64_t* n_evaluated) {
  return guard([&] {
    if (!p || !best_obj || !best_dev || !n_evaluated) fail(XE_ERR_ARG, "null argument");
    require_uploaded(p);
    assignment_oracle_device(p, best_obj, best_dev, n_evaluated, p->stream);
  });
}

}  // extern "C"
