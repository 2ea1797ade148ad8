// SPDX-License-Identifier: Apache-2.0
// C ABI for K1 (model assembly) — include/xengine_b200.h.
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>
#include <algorithm>

#include <sys/mman.h>

#include "csr.hpp"

namespace xe {
namespace {
template <class T>
std::vector<T> down(const T* p, size_t n, cudaStream_t s) {
  std::vector<T> v(n);
  if (n) XE_CUDA(cudaMemcpyAsync(v.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost, s));
  return v;
}
constexpr uintptr_t kHuge = uintptr_t(2) << 20;
}  // namespace
int64_t check_rows_host(xe_csr* m, const double* x_host, double tol, double* viol_host);  // complete.cu

// Device -> pageable host download of a large text: chunks go through two
// pinned staging buffers (the next chunk's copy overlaps this one's) and
// are spread into the destination by several host threads, so its first-
// touch page faults are taken in parallel.  Small texts: one plain copy.
void download_parallel(char* dst, const char* src, size_t n, cudaStream_t s) {
  constexpr size_t kChunk = size_t(32) << 20;
  static std::mutex mu;
  static char* stage[2] = {nullptr, nullptr};  // pinned host memory: usable from every device
  const unsigned hw = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
  if (n < 2 * kChunk || hw < 2) {
    XE_CUDA(cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, s));
    XE_CUDA(cudaStreamSynchronize(s));
    return;
  }
  std::lock_guard<std::mutex> lk(mu);
  if (!stage[0])
    for (int b = 0; b < 2; ++b) XE_CUDA(cudaMallocHost(reinterpret_cast<void**>(&stage[b]), kChunk));
  // events of the stream's device, per call
  struct Events {
    cudaEvent_t e[2] = {nullptr, nullptr};
    ~Events() {
      for (auto x : e)
        if (x) cudaEventDestroy(x);
    }
  } evs;
  for (auto& x : evs.e) XE_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
  cudaEvent_t* ev = evs.e;
  const size_t nch = (n + kChunk - 1) / kChunk;
  auto issue = [&](size_t k) {
    const size_t off = k * kChunk, len = std::min(kChunk, n - off);
    XE_CUDA(cudaMemcpyAsync(stage[k & 1], src + off, len, cudaMemcpyDeviceToHost, s));
    XE_CUDA(cudaEventRecord(ev[k & 1], s));
  };
  issue(0);
  for (size_t k = 0; k < nch; ++k) {
    XE_CUDA(cudaEventSynchronize(ev[k & 1]));
    if (k + 1 < nch) issue(k + 1);  // into the other buffer, free since chunk k-1 was spread
    const size_t off = k * kChunk, len = std::min(kChunk, n - off);
    const size_t part = (len + hw - 1) / hw;
    std::vector<std::thread> th;
    for (unsigned t = 0; t < hw; ++t) {
      const size_t a = std::min(len, t * part), b = std::min(len, a + part);
      if (b > a) th.emplace_back([=] { std::memcpy(dst + off + a, stage[k & 1] + a, b - a); });
    }
    for (auto& x : th) x.join();
  }
}

// the host writer (mps_writer.cpp): the fallback, XE_MPS_HOST=1
void mps_host(xe_csr* m) {
  build_csc(m, m->stream);
  cudaStream_t s = m->stream;
  const xe_csr_info& in = m->info;
  CsrHost h;
  h.D = in.D;
  h.T = in.T;
  h.E = in.E;
  h.n_rows = in.n_rows;
  h.nnz = in.nnz;
  h.n_cols = in.n_cols;
  h.quad = m->opts.quadratic_objective != 0;
  h.col_ptr = down(m->col_ptr.p, static_cast<size_t>(in.n_cols) + 1, s);
  h.crow = down(m->crow.p, static_cast<size_t>(in.nnz), s);
  h.cval = down(m->cval.p, static_cast<size_t>(in.nnz), s);
  h.ordinal = down(m->ordinal.p, static_cast<size_t>(in.n_rows), s);
  h.rhs = down(m->rhs.p, static_cast<size_t>(in.n_rows), s);
  h.sense = down(m->sense.p, static_cast<size_t>(in.n_rows), s);
  h.tag = down(m->tag.p, static_cast<size_t>(in.n_rows), s);
  h.obj = down(m->obj.p, static_cast<size_t>(in.n_cols), s);
  h.present = down(m->present.p, static_cast<size_t>(in.n_cols), s);
  h.ub = down(m->ub.p, static_cast<size_t>(in.n_cols), s);
  h.kind = down(m->kind.p, static_cast<size_t>(in.n_cols), s);
  XE_CUDA(cudaStreamSynchronize(s));
  h.w = m->prob->h.w;
  h.src = m->prob->h.src;
  h.dst = m->prob->h.dst;
  m->mps = mps_text(h);
}
}  // namespace xe

using namespace xe;

extern "C" {

int xe_build_csr(const xe_problem* p, const xe_model_opts* opts, xe_csr** out) {
  return guard([&] {
    if (!p || !out) fail(XE_ERR_ARG, "null argument");
    require_uploaded(p);
    xe_model_opts o{};
    if (opts) o = *opts;
    *out = build_csr(p, o, p->stream);
  });
}

int xe_csr_destroy(xe_csr* m) {
  return guard([&] {
    if (m) {
      cudaSetDevice(m->prob->device);
      delete m;
    }
  });
}

int xe_csr_get_info(const xe_csr* m, xe_csr_info* out) {
  return guard([&] {
    if (!m || !out) fail(XE_ERR_ARG, "null argument");
    *out = m->info;
  });
}

int xe_csr_get_view(const xe_csr* m, xe_csr_view* v) {
  return guard([&] {
    if (!m || !v) fail(XE_ERR_ARG, "null argument");
    v->row_ptr = m->row_ptr.p;
    v->col = m->col.p;
    v->val = m->val.p;
    v->rhs = m->rhs.p;
    v->sense = m->sense.p;
    v->tag = m->tag.p;
    v->ordinal = m->ordinal.p;
    v->obj = m->obj.p;
    v->obj_present = m->present.p;
    v->lb = m->lb.p;
    v->ub = m->ub.p;
    v->kind = m->kind.p;
  });
}

int xe_csr_build_csc(xe_csr* m) {
  return guard([&] {
    if (!m) fail(XE_ERR_ARG, "null argument");
    require_uploaded(m->prob);
    build_csc(m, m->stream);
  });
}

int xe_csr_get_csc(const xe_csr* m, const int64_t** col_ptr, const int32_t** row, const double** val) {
  return guard([&] {
    if (!m) fail(XE_ERR_ARG, "null argument");
    if (!m->has_csc) fail(XE_ERR_ARG, "call xe_csr_build_csc first");
    if (col_ptr) *col_ptr = m->col_ptr.p;
    if (row) *row = m->crow.p;
    if (val) *val = m->cval.p;
  });
}

int xe_csr_last_build_ms(const xe_csr* m, float* ms) {
  return guard([&] {
    if (!m || !ms) fail(XE_ERR_ARG, "null argument");
    *ms = m->build_ms;
  });
}

int xe_csr_download(const xe_csr* m, const xe_csr_host* o) {
  return guard([&] {
    if (!m || !o) fail(XE_ERR_ARG, "null argument");
    require_uploaded(m->prob);
    const xe_csr_info& in = m->info;
    cudaStream_t s = m->stream;
    auto cp = [&](void* dst, const void* src, size_t bytes) {
      if (dst && bytes) XE_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
    };
    const size_t R = static_cast<size_t>(in.n_rows), Z = static_cast<size_t>(in.nnz), N = static_cast<size_t>(in.n_cols);
    cp(o->row_ptr, m->row_ptr.p, (R + 1) * 8);
    cp(o->col, m->col.p, Z * 4);
    cp(o->val, m->val.p, Z * 8);
    cp(o->rhs, m->rhs.p, R * 8);
    cp(o->sense, m->sense.p, R);
    cp(o->tag, m->tag.p, R);
    cp(o->ordinal, m->ordinal.p, R * 4);
    cp(o->obj, m->obj.p, N * 8);
    cp(o->obj_present, m->present.p, N);
    cp(o->lb, m->lb.p, N * 8);
    cp(o->ub, m->ub.p, N * 8);
    cp(o->kind, m->kind.p, N);
    XE_CUDA(cudaStreamSynchronize(s));
  });
}

int xe_csr_upload(const xe_problem* p, const xe_model_opts* opts, int64_t n_rows, int64_t n_cols,
                  const xe_csr_host* in, xe_csr** out) {
  return guard([&] {
    if (!p || !in || !out || n_rows < 0) fail(XE_ERR_ARG, "null argument");
    if (!in->row_ptr || !in->col || !in->val || !in->rhs || !in->sense || !in->tag || !in->ordinal || !in->obj ||
        !in->obj_present || !in->lb || !in->ub || !in->kind)
      fail(XE_ERR_ARG, "xe_csr_upload needs every xe_csr_host array");
    require_uploaded(p);
    const HostProblem& h = p->h;
    if (n_cols != xe_model_cols(h.D, h.T, h.E)) fail(XE_ERR_DIMENSION_MISMATCH, "column count of the model space");
    const int64_t nnz = in->row_ptr[n_rows];
    for (int64_t k = 0; k < nnz; ++k)
      if (in->col[k] < 0 || in->col[k] >= n_cols) fail(XE_ERR_UNKNOWN_VARIABLE, "column index outside the model");
    auto m = std::make_unique<xe_csr>();
    m->prob = p;
    m->opts = opts ? *opts : xe_model_opts{};
    m->stream = p->stream;
    cudaStream_t s = m->stream;
    auto up = [&](auto& buf, const auto* src, size_t count) {
      buf.alloc(std::max<size_t>(1, count));
      if (count) XE_CUDA(cudaMemcpyAsync(buf.p, src, count * sizeof(*src), cudaMemcpyHostToDevice, s));
    };
    const size_t R = static_cast<size_t>(n_rows), Z = static_cast<size_t>(nnz), N = static_cast<size_t>(n_cols);
    up(m->row_ptr, in->row_ptr, R + 1);
    up(m->col, in->col, Z);
    up(m->val, in->val, Z);
    up(m->rhs, in->rhs, R);
    up(m->sense, in->sense, R);
    up(m->tag, in->tag, R);
    up(m->ordinal, in->ordinal, R);
    up(m->obj, in->obj, N);
    up(m->present, in->obj_present, N);
    up(m->lb, in->lb, N);
    up(m->ub, in->ub, N);
    up(m->kind, in->kind, N);
    xe_csr_info& info = m->info;
    info.n_cols = n_cols;
    info.n_rows = n_rows;
    info.nnz = nnz;
    info.D = h.D;
    info.T = h.T;
    info.E = h.E;
    info.n_tags = 14;
    std::memset(info.tag_rows, 0, sizeof info.tag_rows);
    for (int64_t r = 0; r < n_rows; ++r)
      if (in->tag[r] < 16) info.tag_rows[in->tag[r]]++;
    info.n_rows_mps = n_rows - (m->opts.quadratic_objective ? info.tag_rows[11] : 0);
    XE_CUDA(cudaStreamSynchronize(s));
    *out = m.release();
  });
}

int xe_check_rows(xe_csr* m, const double* x, double tol, double* viol, int64_t* n_violated) {
  return guard([&] {
    if (!m || !x || !n_violated) fail(XE_ERR_ARG, "null argument");
    require_uploaded(m->prob);
    *n_violated = check_rows_host(m, x, tol, viol);
  });
}

int xe_write_mps(xe_csr* m, char* buf, size_t* len) {
  return guard([&] {
    if (!m || !len) fail(XE_ERR_ARG, "null argument");
    if (!buf || (m->mps.empty() && !m->mps_dev.p)) {
      require_uploaded(m->prob);
      std::string().swap(m->mps);
      m->mps_dev.release();
      const char* e = std::getenv("XE_MPS_HOST");
      const bool host_only = e && e[0] == '1';
      if (host_only || !mps_text_device(m)) {
        m->mps_dev.release();
        mps_host(m);
      }
    }
    const size_t n = m->mps_dev.p ? m->mps_dev_len : m->mps.size();
    if (!buf) {
      *len = n;
      return;
    }
    if (*len < n) fail(XE_ERR_ARG, "buffer too small");
    if (m->mps_dev.p) {
      // a fresh multi-MB destination faults in page by page during the
      // copy; ask for transparent huge pages on its aligned interior
      const uintptr_t lo = (reinterpret_cast<uintptr_t>(buf) + kHuge - 1) & ~(kHuge - 1);
      const uintptr_t hi = (reinterpret_cast<uintptr_t>(buf) + n) & ~(kHuge - 1);
      if (hi > lo) madvise(reinterpret_cast<void*>(lo), hi - lo, MADV_HUGEPAGE);
      download_parallel(buf, m->mps_dev.p, n, m->stream);
    } else {
      std::memcpy(buf, m->mps.data(), n);
    }
    *len = n;
    std::string().swap(m->mps);  // text handed out; free the cache
    m->mps_dev.release();
  });
}

}  // extern "C"
