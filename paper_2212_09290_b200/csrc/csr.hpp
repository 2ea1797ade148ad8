// SPDX-License-Identifier: Apache-2.0
// K1 model handle shared by the assembly kernels (csr.cu), the MPS writer
// and the PDHG solver.
#pragma once

#include <string>

#include "xe_internal.hpp"

// ---------------------------------------------------------------------------
// Opaque model handle
// ---------------------------------------------------------------------------
struct xe_csr {
  const xe_problem* prob = nullptr;
  xe_model_opts opts{};
  xe_csr_info info{};
  xe::DevBuf<int64_t> row_ptr;
  xe::DevBuf<int32_t> col, ordinal;
  xe::DevBuf<double> val, rhs, obj, lb, ub;
  xe::DevBuf<int8_t> sense;
  xe::DevBuf<uint8_t> tag, present, kind;
  // CSC
  bool has_csc = false;
  xe::DevBuf<int64_t> col_ptr;
  xe::DevBuf<int32_t> crow;
  xe::DevBuf<double> cval;
  float build_ms = 0.f;
  cudaStream_t stream = nullptr;
  std::string mps;  // cached host-written text (xe_write_mps two-call protocol)
  xe::DevBuf<char> mps_dev;  // or the device-written text
  size_t mps_dev_len = 0;
};


namespace xe {
xe_csr* build_csr(const xe_problem* pr, const xe_model_opts& opts, cudaStream_t s);
void build_csc(xe_csr* m, cudaStream_t s);
// Host copy of what write_mps needs (column-major entries, row names, bounds).
struct CsrHost {
  int D, T, E;
  int64_t n_rows, nnz, n_cols;
  std::vector<int64_t> col_ptr;
  std::vector<int32_t> crow, ordinal;
  std::vector<double> cval, rhs, obj, ub;
  std::vector<int8_t> sense;
  std::vector<uint8_t> tag, present, kind;
  std::vector<double> w;  // [E][D][D] (QUADOBJ)
  std::vector<int32_t> src, dst;
  bool quad;
};
std::string mps_text(const CsrHost& h);
// device writer (mps_device.cu); false: the model needs the host writer
bool mps_text_device(xe_csr* m);
void mps_host(xe_csr* m);  // capi_csr.cpp
}  // namespace xe
