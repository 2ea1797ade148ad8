// SPDX-License-Identifier: Apache-2.0
// C ABI for K1 (model assembly) — include/xengine_b200.h.
#include <cstring>
#include <memory>

#include "csr.hpp"

namespace xe {
namespace {
template <class T>
std::vector<T> down(const T* p, size_t n, cudaStream_t s) {
  std::vector<T> v(n);
  if (n) XE_CUDA(cudaMemcpyAsync(v.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost, s));
  return v;
}
}  // namespace
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

int xe_write_mps(xe_csr* m, char* buf, size_t* len) {
  return guard([&] {
    if (!m || !len) fail(XE_ERR_ARG, "null argument");
    if (!buf || m->mps.empty()) {
      require_uploaded(m->prob);
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
    if (!buf) {
      *len = m->mps.size();
      return;
    }
    if (*len < m->mps.size()) fail(XE_ERR_ARG, "buffer too small");
    std::memcpy(buf, m->mps.data(), m->mps.size());
    *len = m->mps.size();
    std::string().swap(m->mps);  // text handed out; free the cache
  });
}

}  // extern "C"
