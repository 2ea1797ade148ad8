// SPDX-License-Identifier: Apache-2.0
//
// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI harness around the UNMODIFIED reference library compiled from
// /root/reference/proj/src/*.cpp (recipe: oracle/Makefile -> oracle/_ref/).
// It lets the Python tests, the golden-fixture generator and bench.py's
// reference arm call the reference's own functions:
//   load_problem            proj/src/problem.cpp:228-244
//   build_model / write_mps proj/src/model.cpp:86-256, proj/src/mps_io.cpp:109-199
//   complete_assignment     proj/src/model.cpp:471-549
//   objective_value         proj/src/model.cpp:369-428
//   check_assignment        proj/src/model.cpp:430-469
//   decode                  proj/src/schedule.cpp:40-129
//   validate / replay       proj/src/schedule.cpp:131-369
//   format_schedule / parse_schedule / trace_csv  proj/src/schedule.cpp:440-530
//   save_all_assignment     proj/src/solver.cpp:30-42
//   assignment_oracle       proj/src/solver.cpp:44-75
//   solve_exact             proj/src/solver.cpp:449-489
// Nothing here re-implements reference logic; it only marshals data.

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "xengine/fixtures.hpp"
#include "xengine/model.hpp"
#include "xengine/mps_io.hpp"
#include "xengine/problem.hpp"
#include "xengine/schedule.hpp"
#include "xengine/solver.hpp"
#include "../include/xengine_b200.h"

using namespace xengine;

namespace {

struct Handle {
  Problem p;
  std::string doc;
  std::optional<EnergyModel> energy;
};

thread_local std::string g_err;

int fail(const Error& e) {
  g_err = e.what();
  return static_cast<int>(e.code()) + 1;
}
int fail_std(const std::exception& e) {
  g_err = e.what();
  return XE_ERR_ARG;
}

ModelOptions make_opts(const Handle* h, int strict, int quad, int energy) {
  ModelOptions o;
  o.strict_free = strict != 0;
  o.quadratic_objective = quad != 0;
  if (energy && h->energy) o.energy = h->energy;
  return o;
}

uint32_t tag_bit(const std::string& v) {
  static const std::pair<const char*, uint32_t> tags[] = {
      {"EQ8_", XE_F_EQ8},         {"EQ9_", XE_F_EQ9},         {"EQ11_", XE_F_EQ11},
      {"EQ12_", XE_F_EQ12},       {"EQ13_", XE_F_EQ13},       {"EQ14_", XE_F_EQ14},
      {"EQ16_LO_", XE_F_EQ16_LO}, {"EQ16_HI_", XE_F_EQ16_HI}, {"Z_LINK_", XE_F_Z_LINK},
      {"P_LINK_", XE_F_P_LINK},   {"ENERGY_DEV_", XE_F_ENERGY_DEV},
      {"ENERGY_TOTAL_", XE_F_ENERGY_TOTAL}};
  for (const auto& [pre, bit] : tags)
    if (v.rfind(pre, 0) == 0) return bit;
  if (v.rfind("fixed-to-zero", 0) == 0) return XE_F_FIXED_ZERO;
  if (v.rfind("U out of budget", 0) == 0) return XE_F_U_BOUND;
  return XE_F_OTHER;
}

// One candidate through the reference: completion, Eq.1 objective, row
// check, U peaks, integer budget check and decode legality.
void eval_one(const Handle* h, const ModelOptions& opts, const MilpModel& m, const BitCube& R,
              const BitCube& S, bool with_check, bool with_decode, double* obj, int64_t* peak,
              uint32_t* flags) {
  const int D = h->p.device_count(), T = h->p.op_count();
  Assignment a = complete_assignment(h->p, opts, R, S);
  *obj = objective_value(a, h->p, opts);
  uint32_t f = 0;
  for (int d = 0; d < D; ++d) {
    double pk = 0.0;
    for (int t = 0; t < T; ++t)
      for (int v = 0; v < T; ++v) pk = std::max(pk, a.at(var_u(d, t, v)));
    peak[d] = static_cast<int64_t>(pk);
    if (peak[d] > h->p.devices[static_cast<size_t>(d)].budget_bytes) f |= XE_F_BUDGET;
  }
  if (with_check)
    for (const auto& v : check_assignment(m, a, 1e-6)) f |= tag_bit(v);
  if (with_decode) {
    try {
      (void)decode(a, h->p);
    } catch (const Error& e) {
      if (e.code() == Errc::IllegalAssignment) {
        f |= XE_F_DECODE;
        if (std::string(e.what()).find("freed earlier") != std::string::npos)
          f |= XE_F_DECODE_FREED;
      } else {
        throw;
      }
    }
  }
  *flags = f;
}

void unpack(const uint32_t* c, int D, int T, BitCube& R, BitCube& S) {
  const int W = (T + 31) / 32;
  for (int cube = 0; cube < 2; ++cube) {
    BitCube& B = cube == 0 ? R : S;
    for (int d = 0; d < D; ++d)
      for (int t = 0; t < T; ++t) {
        const uint32_t* row = c + ((static_cast<size_t>(cube) * D + d) * T + t) * W;
        for (int i = 0; i < T; ++i) B.at(d, t, i) = (row[i >> 5] >> (i & 31)) & 1u;
      }
  }
}

template <class F>
void parallel_for(int64_t n, int nthreads, F&& fn) {
  if (nthreads <= 1 || n < 2) {
    fn(0, n);
    return;
  }
  std::vector<std::thread> th;
  int64_t chunk = (n + nthreads - 1) / nthreads;
  for (int k = 0; k < nthreads; ++k) {
    int64_t lo = k * chunk, hi = std::min(n, lo + chunk);
    if (lo >= hi) break;
    th.emplace_back([&, lo, hi] { fn(lo, hi); });
  }
  for (auto& t : th) t.join();
}

}  // namespace

extern "C" {

const char* xr_last_error() { return g_err.c_str(); }
void xr_free(void* p) { std::free(p); }

int xr_problem_load(const char* json, void** out) {
  try {
    auto* h = new Handle;
    h->doc = json;
    h->p = load_problem(h->doc);
    h->energy = parse_energy(h->doc, h->p);
    *out = h;
    return 0;
  } catch (const Error& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail_std(e);
  }
}

// Built-in fixtures (fixtures.cpp:10-59): "chain3", "fig2", "chain_lowmem",
// "fig2_energy" (fig2 + make_fig2_energy()).
int xr_problem_fixture(const char* name, void** out) {
  auto* h = new Handle;
  std::string n = name;
  if (n == "chain3") h->p = make_chain3();
  else if (n == "fig2") h->p = make_fig2();
  else if (n == "chain_lowmem") h->p = make_chain_lowmem();
  else if (n == "fig2_energy") {
    h->p = make_fig2();
    h->energy = make_fig2_energy();
  } else {
    delete h;
    g_err = "unknown fixture";
    return XE_ERR_ARG;
  }
  *out = h;
  return 0;
}

void xr_problem_free(void* h) { delete static_cast<Handle*>(h); }

int xr_problem_set_budgets(void* hv, const int64_t* budgets) {
  auto* h = static_cast<Handle*>(hv);
  try {
    h->p = with_budgets(h->p, std::vector<int64_t>(budgets, budgets + h->p.device_count()));
    return 0;
  } catch (const Error& e) {
    return fail(e);
  }
}

// Resolved SoA arrays (the xe_problem_desc image) using the reference's own
// copy_cost for every (edge, ds, dc).
int xr_problem_arrays(void* hv, int* D, int* T, int* E, int64_t* bytes, double* cost,
                      int32_t* src, int32_t* dst, double* w, int64_t* budget, int* has_energy) {
  auto* h = static_cast<Handle*>(hv);
  const Problem& p = h->p;
  *D = p.device_count();
  *T = p.op_count();
  *E = static_cast<int>(p.edges.size());
  *has_energy = h->energy ? 1 : 0;
  if (!bytes) return 0;
  try {
    for (int i = 0; i < *T; ++i) {
      bytes[i] = p.operators[static_cast<size_t>(i)].output_bytes;
      for (int d = 0; d < *D; ++d)
        cost[static_cast<size_t>(d) * *T + i] = p.operators[static_cast<size_t>(i)].costs_ms[static_cast<size_t>(d)];
    }
    for (int e = 0; e < *E; ++e) {
      src[e] = p.edges[static_cast<size_t>(e)].src;
      dst[e] = p.edges[static_cast<size_t>(e)].dst;
      for (int a = 0; a < *D; ++a)
        for (int b = 0; b < *D; ++b)
          w[(static_cast<size_t>(e) * *D + a) * *D + b] = copy_cost(p, p.edges[static_cast<size_t>(e)], a, b);
    }
    for (int d = 0; d < *D; ++d) budget[d] = p.devices[static_cast<size_t>(d)].budget_bytes;
    return 0;
  } catch (const Error& e) {
    return fail(e);
  }
}

int xr_energy_arrays(void* hv, double* alpha, double* q, uint8_t* has_lim, double* lim,
                     int* has_total, double* total, double* board) {
  auto* h = static_cast<Handle*>(hv);
  if (!h->energy) return XE_ERR_ARG;
  const auto& e = *h->energy;
  const int D = h->p.device_count(), T = h->p.op_count();
  *alpha = e.alpha;
  for (int d = 0; d < D; ++d) {
    for (int i = 0; i < T; ++i) q[static_cast<size_t>(d) * T + i] = e.q_joules[static_cast<size_t>(d)][static_cast<size_t>(i)];
    auto it = e.device_limit.find(d);
    has_lim[d] = it != e.device_limit.end();
    lim[d] = has_lim[d] ? it->second : 0.0;
  }
  *has_total = e.total_limit.has_value();
  *total = e.total_limit.value_or(0.0);
  *board = e.board_joules;
  return 0;
}

int xr_write_mps(void* hv, int strict, int quad, int energy, char** out, size_t* len) {
  auto* h = static_cast<Handle*>(hv);
  try {
    std::string s = write_mps(build_model(h->p, make_opts(h, strict, quad, energy)));
    *out = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(*out, s.c_str(), s.size() + 1);
    *len = s.size();
    return 0;
  } catch (const Error& e) {
    return fail(e);
  }
}

// Model dump as CSR in constraint emission order, with closed-form column
// indices computed from VarRef (the order write_mps sorts columns in).
int xr_model_csr(void* hv, int strict, int energy, int64_t* n_rows, int64_t* nnz,
                 int64_t* row_ptr, int32_t* col, double* val, double* rhs, int8_t* sense,
                 uint8_t* tag, int32_t* ordinal, int64_t* n_cols, double* obj,
                 uint8_t* obj_present, uint8_t* fixed) {
  auto* h = static_cast<Handle*>(hv);
  try {
    MilpModel m = build_model(h->p, make_opts(h, strict, 0, energy));
    const int64_t D = m.D, T = m.T, E = m.E, FE = m.f_edges;
    auto index = [&](const VarRef& v) -> int64_t {
      switch (v.family) {
        case VarFamily::R: return (v.a * T + v.b) * T + v.c;
        case VarFamily::S: return D * T * T + (v.a * T + v.b) * T + v.c;
        case VarFamily::Z: return 2 * D * T * T + (v.a * T + v.b) * T + v.c;
        case VarFamily::F: return 3 * D * T * T + (v.a * T + v.b) * FE + v.c;
        case VarFamily::U: return 3 * D * T * T + D * T * FE + (v.a * T + v.b) * T + v.c;
        case VarFamily::P:
          return 4 * D * T * T + D * T * FE + ((v.a * E + v.b) * D + v.c) * (D - 1) +
                 (v.d - (v.d > v.c ? 1 : 0));
      }
      return -1;
    };
    *n_rows = static_cast<int64_t>(m.constraints.size());
    int64_t k = 0;
    for (const auto& c : m.constraints) k += static_cast<int64_t>(c.terms.size());
    *nnz = k;
    *n_cols = 4 * D * T * T + D * T * FE + T * E * D * (D - 1);
    if (!row_ptr) return 0;
    k = 0;
    for (size_t r = 0; r < m.constraints.size(); ++r) {
      const auto& c = m.constraints[r];
      row_ptr[r] = k;
      for (const auto& [ref, coef] : c.terms) {
        col[k] = static_cast<int32_t>(index(ref));
        val[k] = coef;
        ++k;
      }
      rhs[r] = c.rhs;
      sense[r] = c.rel == Relation::LE ? 'L' : c.rel == Relation::GE ? 'G' : 'E';
      tag[r] = static_cast<uint8_t>(c.tag);
      ordinal[r] = c.ordinal;
    }
    row_ptr[m.constraints.size()] = k;
    for (int64_t j = 0; j < *n_cols; ++j) {
      obj[j] = 0.0;
      obj_present[j] = 0;
      fixed[j] = 0;
    }
    for (const auto& [ref, coef] : m.objective) {
      obj[index(ref)] = coef;
      obj_present[index(ref)] = 1;
    }
    for (const auto& ref : m.fixed_zero) fixed[index(ref)] = 1;
    return 0;
  } catch (const Error& e) {
    return fail(e);
  }
}

// cubes: xe_cube layout, n candidates.  with_check/with_decode select the
// reference calls made per candidate (bench.py times with_check=1,
// with_decode=0: complete_assignment + objective_value + check_assignment +
// peaks).
int xr_eval_cubes(void* hv, int strict, int energy, const uint32_t* cubes, int64_t n,
                  int with_check, int with_decode, double* obj, int64_t* peak, uint32_t* flags,
                  int nthreads) {
  auto* h = static_cast<Handle*>(hv);
  try {
    ModelOptions opts = make_opts(h, strict, 0, energy);
    MilpModel m = build_model(h->p, opts);
    const int D = h->p.device_count(), T = h->p.op_count();
    const size_t words = static_cast<size_t>(2) * D * T * ((T + 31) / 32);
    std::string err;
    int rc = 0;
    parallel_for(n, nthreads, [&](int64_t lo, int64_t hi) {
      try {
        BitCube R(D, T), S(D, T);
        for (int64_t c = lo; c < hi; ++c) {
          std::fill(R.bits.begin(), R.bits.end(), 0);
          std::fill(S.bits.begin(), S.bits.end(), 0);
          unpack(cubes + c * words, D, T, R, S);
          eval_one(h, opts, m, R, S, with_check != 0, with_decode != 0, obj + c, peak + c * D,
                   flags + c);
        }
      } catch (const Error& e) {
        rc = fail(e);
      }
    });
    return rc;
  } catch (const Error& e) {
    return fail(e);
  }
}

// Placement candidates through save_all_assignment (solver.cpp:30-42) for
// policy 0; policy 1 builds the minimal-save cube (S only until the last
// consumer) and completes it with complete_assignment.
int xr_eval_placements(void* hv, const uint8_t* dev, int64_t n, int policy, int with_check,
                       double* obj, int64_t* peak, uint32_t* flags, int nthreads) {
  auto* h = static_cast<Handle*>(hv);
  try {
    ModelOptions opts;
    MilpModel m = build_model(h->p, opts);
    const int D = h->p.device_count(), T = h->p.op_count();
    std::vector<int> last(static_cast<size_t>(T), -1);
    for (const auto& e : h->p.edges) last[static_cast<size_t>(e.src)] = std::max(last[static_cast<size_t>(e.src)], e.dst);
    int rc = 0;
    parallel_for(n, nthreads, [&](int64_t lo, int64_t hi) {
      try {
        for (int64_t c = lo; c < hi; ++c) {
          std::vector<int> dv(dev + c * T, dev + (c + 1) * T);
          Assignment a;
          if (policy == 0) {
            a = save_all_assignment(h->p, dv);
          } else {
            BitCube R(D, T), S(D, T);
            for (int i = 0; i < T; ++i) {
              R.at(dv[static_cast<size_t>(i)], i, i) = 1;
              for (int t = i + 1; t <= last[static_cast<size_t>(i)]; ++t) S.at(dv[static_cast<size_t>(i)], t, i) = 1;
            }
            a = complete_assignment(h->p, opts, R, S);
          }
          obj[c] = objective_value(a, h->p, opts);
          uint32_t f = 0;
          for (int d = 0; d < D; ++d) {
            double pk = 0.0;
            for (int t = 0; t < T; ++t)
              for (int v = 0; v < T; ++v) pk = std::max(pk, a.at(var_u(d, t, v)));
            peak[c * D + d] = static_cast<int64_t>(pk);
            if (peak[c * D + d] > h->p.devices[static_cast<size_t>(d)].budget_bytes) f |= XE_F_BUDGET;
          }
          if (with_check)
            for (const auto& v : check_assignment(m, a, 1e-6)) f |= tag_bit(v);
          flags[c] = f;
        }
      } catch (const Error& e) {
        rc = fail(e);
      }
    });
    return rc;
  } catch (const Error& e) {
    return fail(e);
  }
}

int xr_assignment_oracle(void* hv, double* obj, int32_t* dev, int64_t* nodes) {
  auto* h = static_cast<Handle*>(hv);
  try {
    Solution s = assignment_oracle(h->p);
    *obj = s.objective_ms;
    *nodes = s.nodes_explored;
    const int T = h->p.op_count(), D = h->p.device_count();
    for (int i = 0; i < T; ++i)
      for (int d = 0; d < D; ++d)
        if (s.assignment.at(var_r(d, i, i)) > 0.5) dev[i] = d;
    return 0;
  } catch (const Error& e) {
    return fail(e);
  }
}

// solve_exact; status 0 optimal, 1 infeasible, 2 limit.  cube (xe_cube
// layout) receives the R/S of the solution when one exists.
int xr_solve_exact(void* hv, int strict, int energy, const int64_t* budgets, int64_t node_limit,
                   int* status, double* obj, uint32_t* cube, int64_t* nodes) {
  auto* h = static_cast<Handle*>(hv);
  try {
    std::vector<int64_t> b;
    if (budgets) b.assign(budgets, budgets + h->p.device_count());
    SearchLimits lim;
    if (node_limit > 0) lim.node_limit = node_limit;
    Solution s = solve_exact(h->p, make_opts(h, strict, 0, energy), b, lim);
    *status = static_cast<int>(s.status);
    *obj = s.objective_ms;
    *nodes = s.nodes_explored;
    if (cube && std::isfinite(s.objective_ms)) {
      const int D = h->p.device_count(), T = h->p.op_count(), W = (T + 31) / 32;
      std::memset(cube, 0, sizeof(uint32_t) * 2 * D * T * W);
      for (int c = 0; c < 2; ++c)
        for (int d = 0; d < D; ++d)
          for (int t = 0; t < T; ++t)
            for (int i = 0; i < T; ++i) {
              VarRef v = c == 0 ? var_r(d, t, i) : var_s(d, t, i);
              if (s.assignment.at(v) > 0.5)
                cube[((static_cast<size_t>(c) * D + d) * T + t) * W + (i >> 5)] |= 1u << (i & 31);
            }
    }
    return 0;
  } catch (const Error& e) {
    return fail(e);
  }
}

int xr_format_number(double v, char* buf, int len) {
  std::string s = format_number(v);
  std::snprintf(buf, static_cast<size_t>(len), "%s", s.c_str());
  return 0;
}

int64_t xr_budget_percent(int64_t full, double pct, int* rc) {
  try {
    *rc = 0;
    return budget_percent(full, pct);
  } catch (const Error& e) {
    *rc = fail(e);
    return 0;
  }
}

namespace {
char* dup_out(const std::string& s, size_t* len) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.data(), s.size());
  p[s.size()] = 0;
  *len = s.size();
  return p;
}
}  // namespace

// decode(complete_assignment(R,S)) -> format_schedule; replay with the
// assignment -> trace_csv, total_action_ms, eq1_objective_ms, peaks
int xr_schedule(void* hv, int strict, int energy, const uint32_t* cube, char** text, size_t* tlen,
                char** csv, size_t* clen, double* total_ms, double* eq1, int64_t* peaks) {
  auto* h = static_cast<Handle*>(hv);
  try {
    ModelOptions opts = make_opts(h, strict, 0, energy);
    const int D = h->p.device_count(), T = h->p.op_count();
    BitCube R(D, T), S(D, T);
    unpack(cube, D, T, R, S);
    Assignment a = complete_assignment(h->p, opts, R, S);
    Schedule sc = decode(a, h->p);
    *text = dup_out(format_schedule(sc), tlen);
    Trace tr = replay(sc, h->p, opts, a);
    *csv = dup_out(trace_csv(tr, h->p), clen);
    *total_ms = tr.total_action_ms;
    *eq1 = tr.eq1_objective_ms;
    for (int d = 0; d < D; ++d) peaks[d] = tr.peaks[static_cast<size_t>(d)];
    return 0;
  } catch (const Error& e) {
    return fail(e);
  }
}

// validate(parse_schedule(text)) -> one line per violation:
// "<kind> <device> <timestep> <slot> <bytes>|<detail>"
int xr_validate_text(void* hv, const char* text, const int64_t* budgets, char** out, size_t* len) {
  auto* h = static_cast<Handle*>(hv);
  try {
    Schedule sc = parse_schedule(text, h->p);
    std::vector<int64_t> b;
    if (budgets) b.assign(budgets, budgets + h->p.device_count());
    ValidationReport rep = validate(sc, h->p, b);
    std::string o;
    for (const auto& v : rep.violations)
      o += std::string(violation_name(v.kind)) + " " + std::to_string(v.device) + " " + std::to_string(v.timestep) +
           " " + std::to_string(v.slot) + " " + std::to_string(v.bytes) + "|" + v.detail + "\n";
    *out = dup_out(o, len);
    return 0;
  } catch (const Error& e) {
    return fail(e);
  }
}

// replay(parse_schedule(text)) without an assignment (availability rebuilt
// from the actions) -> trace_csv, totals, peaks
int xr_replay_text(void* hv, int strict, int energy, const char* text, char** csv, size_t* clen,
                   double* total_ms, double* eq1, int64_t* peaks) {
  auto* h = static_cast<Handle*>(hv);
  try {
    ModelOptions opts = make_opts(h, strict, 0, energy);
    Schedule sc = parse_schedule(text, h->p);
    Trace tr = replay(sc, h->p, opts);
    *csv = dup_out(trace_csv(tr, h->p), clen);
    *total_ms = tr.total_action_ms;
    *eq1 = tr.eq1_objective_ms;
    for (int d = 0; d < h->p.device_count(); ++d) peaks[d] = tr.peaks[static_cast<size_t>(d)];
    return 0;
  } catch (const Error& e) {
    return fail(e);
  }
}

}  // extern "C"
