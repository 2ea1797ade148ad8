// SPDX-License-Identifier: Apache-2.0
//
// The reference's C++ API (include/xengine/*.hpp, re-declared from
// proj/include/xengine/*.hpp) implemented on top of the C ABI
// (include/xengine_b200.h).  Host code here only translates between the
// reference's value types (Problem, MilpModel, Assignment maps, BitCube) and
// the flat arrays the kernels consume; every numeric pass over a model or a
// schedule runs on the GPU:
//
//   build_model          xe_build_csr (K1) + xe_csr_download
//   write_mps            xe_write_mps (GPU CSC, byte-exact writer)
//   complete_assignment  xe_complete_cube
//   objective_value      xe_objective_dense
//   check_assignment     xe_check_rows (+ the map's bound/binary checks)
//   assignment_oracle    xe_assignment_oracle (K2b sweep)
//   evaluate_candidates  xe_eval_cubes_host (K2a, batched)
//
// Errors: a non-zero C status 1 + Errc is re-thrown as xengine::Error with
// the same Errc, so callers see the reference's exception types.

#include <json.hpp>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <limits>
#include <memory>
#include <mutex>
#include <set>
#include <sstream>

#include "xengine/errors.hpp"
#include "xengine/mps_io.hpp"
#include "xengine/model.hpp"
#include "xengine/problem.hpp"
#include "xengine/schedule.hpp"
#include "xengine/solver.hpp"
#include "xengine_b200.h"
#include "xe_internal.hpp"

namespace xengine {

const char* errc_name(Errc c) {
  static const char* const names[] = {
      "MalformedDocument", "NonTopologicalEdge", "UnknownDevice", "NonPositiveSize", "NegativeCost",
      "EmptyNetwork", "PercentOutOfRange", "MissingLink", "DimensionMismatch", "IncompleteEnergyTable",
      "UnknownVariable", "NonIntegralBinary", "EmptySolution", "InfeasibleMarker", "InfeasibleProblem",
      "TooLarge", "ExternalSolverUnavailable", "SolverFailed", "UnparsableSolution", "ObjectiveMismatch",
      "IllegalAssignment", "IllegalSchedule", "EmptySeries", "NonPositiveTime", "IoError"};
  const auto i = static_cast<size_t>(c);
  return i < sizeof names / sizeof names[0] ? names[i] : "Error";
}

const char* tag_name(ConstraintTag t) {
  static const char* const names[] = {"EQ7",     "EQ8",     "EQ9",    "EQ10",   "EQ11",       "EQ12",        "EQ13",
                                      "EQ14",    "EQ16_LO", "EQ16_HI", "Z_LINK", "P_LINK", "ENERGY_DEV", "ENERGY_TOTAL"};
  const auto i = static_cast<size_t>(t);
  return i < 14 ? names[i] : "ROW";
}

const char* status_name(SolveStatus s) {
  switch (s) {
    case SolveStatus::Optimal: return "optimal";
    case SolveStatus::Infeasible: return "infeasible";
    case SolveStatus::LimitReached: return "limit";
  }
  return "unknown";
}

namespace {

using nlohmann::json;

// C status -> the reference's exception (message without the C layer's
// own prefix; Error prepends errc_name like the reference does).
[[noreturn]] void rethrow(int st) {
  const std::string msg = xe_last_error();
  if (st >= 1 && st <= 25) throw Error(static_cast<Errc>(st - 1), msg);
  throw std::runtime_error("xengine_b200: " + msg);
}
void ck(int st) {
  if (st != XE_OK) rethrow(st);
}

int cols_of(const MilpModel& m) { return static_cast<int>(xe_model_cols(m.D, m.T, m.E)); }

// ---- VarRef <-> closed-form column (model.hpp:18-24 order) ---------------
struct Space {
  int64_t D, T, E, FE;
  int64_t r0() const { return 0; }
  int64_t dt2() const { return D * T * T; }
  int64_t col(const VarRef& v) const {
    switch (v.family) {
      case VarFamily::R: return (v.a * T + v.b) * T + v.c;
      case VarFamily::S: return dt2() + (v.a * T + v.b) * T + v.c;
      case VarFamily::Z: return 2 * dt2() + (v.a * T + v.b) * T + v.c;
      case VarFamily::F: return 3 * dt2() + (v.a * T + v.b) * FE + v.c;
      case VarFamily::U: return 3 * dt2() + D * T * FE + (v.a * T + v.b) * T + v.c;
      case VarFamily::P:
        return 4 * dt2() + D * T * FE + ((static_cast<int64_t>(v.a) * E + v.b) * D + v.c) * (D - 1) +
               (v.d - (v.d > v.c ? 1 : 0));
    }
    return -1;
  }
  VarRef ref(int64_t j) const {
    const int64_t DT2 = dt2(), DTF = D * T * FE;
    if (j < 3 * DT2) {
      const auto f = static_cast<VarFamily>(j / DT2);
      const int64_t r = j % DT2;
      return make_ref(f, static_cast<int>(r / (T * T)), static_cast<int>(r / T % T), static_cast<int>(r % T));
    }
    j -= 3 * DT2;
    if (j < DTF) return var_f(static_cast<int>(j / (T * FE)), static_cast<int>(j / FE % T), static_cast<int>(j % FE));
    j -= DTF;
    if (j < DT2) return var_u(static_cast<int>(j / (T * T)), static_cast<int>(j / T % T), static_cast<int>(j % T));
    j -= DT2;
    const int64_t dm1 = D - 1, t = j / (E * D * dm1);
    int64_t rem = j % (E * D * dm1);
    const int64_t e = rem / (D * dm1);
    rem %= D * dm1;
    const int64_t ds = rem / dm1;
    int64_t dc = rem % dm1;
    if (dc >= ds) ++dc;
    return var_p(static_cast<int>(t), static_cast<int>(e), static_cast<int>(ds), static_cast<int>(dc));
  }
};
Space space_of(int D, int T, int E) { return Space{D, T, E, E + T}; }

// ---- Problem -> device handle ---------------------------------------------
struct HandleDeleter {
  void operator()(xe_problem* p) const { xe_problem_destroy(p); }
};
using Handle = std::shared_ptr<xe_problem>;

int default_device() {
  const char* s = std::getenv("XE_DEVICE");
  return s ? std::atoi(s) : 0;
}

// Resolved SoA image; the key is its byte content (a one-entry cache avoids
// re-uploading the same problem for every objective_value call).  The cached
// handle's scratch is shared, so the C++ API, like the reference's free
// functions on one Problem, is meant for one host thread at a time.
struct Desc {
  int D = 0, T = 0, E = 0;
  std::vector<int64_t> mass, budget;
  std::vector<double> cost, w, q, lim;
  std::vector<int32_t> src, dst;
  std::vector<uint8_t> has_lim;
  bool energy = false, has_total = false;
  double alpha = 0, total = 0, board = 0;
  std::string key() const {
    std::string k;
    auto put = [&](const void* p, size_t n) { k.append(static_cast<const char*>(p), n); };
    const int hdr[6] = {D, T, E, energy, has_total, 0};
    put(hdr, sizeof hdr);
    put(mass.data(), mass.size() * 8);
    put(budget.data(), budget.size() * 8);
    put(cost.data(), cost.size() * 8);
    put(w.data(), w.size() * 8);
    put(src.data(), src.size() * 4);
    put(dst.data(), dst.size() * 4);
    if (energy) {
      put(q.data(), q.size() * 8);
      put(lim.data(), lim.size() * 8);
      put(has_lim.data(), has_lim.size());
      const double e3[4] = {alpha, total, board, 0};
      put(e3, sizeof e3);
    }
    return k;
  }
};

void check_energy(const EnergyModel& e, int D, int T) {
  if (static_cast<int>(e.q_joules.size()) != D) raise(Errc::IncompleteEnergyTable, "q_joules needs one row per device");
  for (const auto& row : e.q_joules)
    if (static_cast<int>(row.size()) != T) raise(Errc::IncompleteEnergyTable, "q_joules row needs one entry per operator");
  for (const auto& [d, lim] : e.device_limit) {
    if (d < 0 || d >= D) raise(Errc::DimensionMismatch, "device_limit index");
    if (lim < 0.0) raise(Errc::NegativeCost, "device_limit");
  }
}

Desc describe(const Problem& p, const std::optional<EnergyModel>& energy) {
  Desc d;
  d.D = p.device_count();
  d.T = p.op_count();
  d.E = static_cast<int>(p.edges.size());
  for (const auto& op : p.operators) {
    if (static_cast<int>(op.costs_ms.size()) != d.D) raise(Errc::DimensionMismatch, "operator " + op.name + " cost vector size");
    d.mass.push_back(op.output_bytes);
  }
  d.cost.assign(static_cast<size_t>(d.D) * d.T, 0.0);
  for (int i = 0; i < d.T; ++i)
    for (int k = 0; k < d.D; ++k)
      d.cost[static_cast<size_t>(k) * d.T + i] = p.operators[static_cast<size_t>(i)].costs_ms[static_cast<size_t>(k)];
  for (const auto& dev : p.devices) d.budget.push_back(dev.budget_bytes);
  d.w.assign(static_cast<size_t>(d.E) * d.D * d.D, 0.0);
  for (int e = 0; e < d.E; ++e) {
    const auto& edge = p.edges[static_cast<size_t>(e)];
    d.src.push_back(edge.src);
    d.dst.push_back(edge.dst);
    for (int a = 0; a < d.D; ++a)
      for (int b = 0; b < d.D; ++b)
        if (a != b) {
          // an uncovered pair travels as NaN: the library raises MissingLink
          // when a model or a charged copy needs it, as copy_cost does
          double w = std::numeric_limits<double>::quiet_NaN();
          try {
            w = copy_cost(p, edge, a, b);
          } catch (const Error& err) {
            if (err.code() != Errc::MissingLink) throw;
          }
          d.w[(static_cast<size_t>(e) * d.D + a) * d.D + b] = w;
        }
  }
  if (energy) {
    check_energy(*energy, d.D, d.T);
    d.energy = true;
    d.alpha = energy->alpha;
    d.q.assign(static_cast<size_t>(d.D) * d.T, 0.0);
    for (int k = 0; k < d.D; ++k)
      for (int i = 0; i < d.T; ++i) d.q[static_cast<size_t>(k) * d.T + i] = energy->q_joules[static_cast<size_t>(k)][static_cast<size_t>(i)];
    d.has_lim.assign(static_cast<size_t>(d.D), 0);
    d.lim.assign(static_cast<size_t>(d.D), 0.0);
    for (const auto& [k, lim] : energy->device_limit) {
      d.has_lim[static_cast<size_t>(k)] = 1;
      d.lim[static_cast<size_t>(k)] = lim;
    }
    d.has_total = energy->total_limit.has_value();
    d.total = energy->total_limit.value_or(0.0);
    d.board = energy->board_joules;
  }
  return d;
}

Handle upload(const Desc& d) {
  static std::mutex mu;
  static std::string last_key;
  static Handle last;
  std::string k = d.key();
  {
    std::lock_guard<std::mutex> g(mu);
    if (last && k == last_key) return last;
  }
  xe_problem_desc c{};
  c.D = d.D;
  c.T = d.T;
  c.E = d.E;
  c.output_bytes = d.mass.data();
  c.cost_ms = d.cost.data();
  c.edge_src = d.src.data();
  c.edge_dst = d.dst.data();
  c.copy_ms = d.w.data();
  c.budget_bytes = d.budget.data();
  c.has_energy = d.energy;
  if (d.energy) {
    c.alpha = d.alpha;
    c.q_joules = d.q.data();
    c.has_dev_limit = d.has_lim.data();
    c.dev_limit = d.lim.data();
    c.has_total_limit = d.has_total;
    c.total_limit = d.total;
    c.board_joules = d.board;
  }
  xe_problem* h = nullptr;
  ck(xe_problem_create(&c, default_device(), &h));
  Handle out(h, HandleDeleter{});
  std::lock_guard<std::mutex> g(mu);
  last_key = std::move(k);
  last = out;
  return out;
}

xe_model_opts c_opts(const ModelOptions& o) {
  xe_model_opts c{};
  c.strict_free = o.strict_free;
  c.quadratic_objective = o.quadratic_objective;
  c.use_energy = o.energy.has_value();
  return c;
}

// The GPU model a MilpModel came from, plus the problem handle it references.
struct DeviceModel {
  Handle prob;
  xe_csr* csr = nullptr;
  ~DeviceModel() {
    if (csr) xe_csr_destroy(csr);
  }
};

// O(nnz) identity of everything write_mps / check_assignment read from a
// model (rows with every term and coefficient, the objective map, quad terms,
// fixed zeros, budgets): a model edited in place after build_model no longer
// matches its device copy and is re-uploaded.
uint64_t fingerprint(const MilpModel& m) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](uint64_t x) {
    h ^= x;
    h *= 1099511628211ull;
  };
  auto bits = [](double x) {
    uint64_t r;
    std::memcpy(&r, &x, 8);
    return r;
  };
  auto ref = [&](const VarRef& v) {
    mix(static_cast<uint64_t>(static_cast<uint16_t>(v.a)) << 48 | static_cast<uint64_t>(static_cast<uint16_t>(v.b)) << 32 |
        static_cast<uint64_t>(static_cast<uint16_t>(v.c)) << 16 | static_cast<uint64_t>(static_cast<uint16_t>(v.d)));
    mix(static_cast<uint64_t>(v.family));
  };
  mix(m.constraints.size());
  mix(m.objective.size());
  mix(m.fixed_zero.size());
  mix(static_cast<uint64_t>(m.D) << 32 | static_cast<uint64_t>(m.T) << 16 | static_cast<uint64_t>(m.E));
  mix(static_cast<uint64_t>(m.options.strict_free) | static_cast<uint64_t>(m.options.quadratic_objective) << 1 |
      static_cast<uint64_t>(m.options.energy.has_value()) << 2);
  for (const auto& c : m.constraints) {
    mix(c.terms.size() ^ (static_cast<uint64_t>(c.tag) << 40) ^ (static_cast<uint64_t>(c.ordinal) << 20) ^
        (static_cast<uint64_t>(c.rel) << 60));
    mix(bits(c.rhs));
    for (const auto& [v, x] : c.terms) {
      ref(v);
      mix(bits(x));
    }
  }
  for (const auto& [v, x] : m.objective) {
    ref(v);
    mix(bits(x));
  }
  for (const auto& q : m.quad) {
    mix(static_cast<uint64_t>(q.t) << 32 ^ static_cast<uint64_t>(q.e));
    mix(static_cast<uint64_t>(q.d_src) << 32 ^ static_cast<uint64_t>(q.d_cmp));
    mix(bits(q.w));
  }
  for (const auto& v : m.fixed_zero) ref(v);
  for (auto b : m.budgets) mix(static_cast<uint64_t>(b));
  return h;
}

// xe_csr for any MilpModel: the device copy build_model kept when it still
// matches, else the model's rows uploaded (hand-built or edited models).
std::shared_ptr<DeviceModel> device_model(const MilpModel& m) {
  if (m.device_model && m.device_fingerprint == fingerprint(m))
    return std::static_pointer_cast<DeviceModel>(m.device_model);
  auto dm = std::make_shared<DeviceModel>();
  dm->prob = upload(describe(m.problem, m.options.energy));
  const Space sp = space_of(m.D, m.T, m.E);
  const int64_t n = cols_of(m);
  std::vector<int64_t> rp(1, 0);
  std::vector<int32_t> col, ord;
  std::vector<double> val, rhs, obj(static_cast<size_t>(n), 0.0), lb(static_cast<size_t>(n), 0.0),
      ub(static_cast<size_t>(n), 1.0);
  std::vector<int8_t> sense;
  std::vector<uint8_t> tag, present(static_cast<size_t>(n), 0), kind(static_cast<size_t>(n), 1);
  for (const auto& c : m.constraints) {
    for (const auto& [ref, coef] : c.terms) {
      if (!m.in_space(ref)) raise(Errc::UnknownVariable, "row term outside the model's variable space");
      col.push_back(static_cast<int32_t>(sp.col(ref)));
      val.push_back(coef);
    }
    rp.push_back(static_cast<int64_t>(col.size()));
    rhs.push_back(c.rhs);
    sense.push_back(c.rel == Relation::LE ? 'L' : c.rel == Relation::GE ? 'G' : 'E');
    tag.push_back(static_cast<uint8_t>(c.tag));
    ord.push_back(c.ordinal);
  }
  for (const auto& [ref, v] : m.objective) {
    if (!m.in_space(ref)) continue;
    obj[static_cast<size_t>(sp.col(ref))] = v;
    present[static_cast<size_t>(sp.col(ref))] = 1;
  }
  const int64_t firstU = 3 * sp.dt2() + sp.D * sp.T * sp.FE, firstP = firstU + sp.dt2();
  for (int64_t j = firstU; j < n; ++j) {
    kind[static_cast<size_t>(j)] = j < firstP ? 2 : 3;
    ub[static_cast<size_t>(j)] = j < firstP ? static_cast<double>(m.budgets[static_cast<size_t>((j - firstU) / (sp.T * sp.T))]) : 1.0;
  }
  for (const auto& ref : m.fixed_zero) {
    kind[static_cast<size_t>(sp.col(ref))] = 0;
    ub[static_cast<size_t>(sp.col(ref))] = 0.0;
  }
  xe_csr_host h{rp.data(), col.data(), val.data(), rhs.data(), sense.data(), tag.data(), ord.data(),
                obj.data(), present.data(), lb.data(), ub.data(), kind.data()};
  xe_model_opts o = c_opts(m.options);
  ck(xe_csr_upload(dm->prob.get(), &o, static_cast<int64_t>(rhs.size()), n, &h, &dm->csr));
  return dm;
}

std::vector<uint32_t> pack_cube(const BitCube& R, const BitCube& S) {
  const int D = R.D, T = R.T, W = (T + 31) / 32;
  std::vector<uint32_t> c(static_cast<size_t>(2) * D * T * W, 0u);
  for (int which = 0; which < 2; ++which) {
    const BitCube& B = which ? S : R;
    for (int d = 0; d < D; ++d)
      for (int t = 0; t < T; ++t)
        for (int i = 0; i < T; ++i)
          if (B.at(d, t, i))
            c[((static_cast<size_t>(which) * D + d) * T + t) * W + i / 32] |= 1u << (i % 32);
  }
  return c;
}

}  // namespace

// ============================ problem.hpp ==================================

int Problem::find_device(const std::string& id) const {
  for (int d = 0; d < device_count(); ++d)
    if (devices[static_cast<size_t>(d)].id == id) return d;
  return -1;
}

Problem load_problem(const std::string& json_text) {
  // the library's one document parser (loader.cpp: the reference's
  // validation order, messages and error codes), then the value types
  xe::ParsedDoc d;
  try {
    d = xe::parse_problem_document(json_text);
  } catch (const xe::Error& e) {
    raise(static_cast<Errc>(e.code - 1), e.what());
  }
  const xe::HostProblem& h = d.p;
  Problem p;
  p.name = d.name;
  for (int k = 0; k < h.D; ++k) {
    DeviceSpec ds;
    ds.id = h.device_ids[static_cast<size_t>(k)];
    ds.budget_bytes = h.budget[static_cast<size_t>(k)];
    if (d.ram[static_cast<size_t>(k)] >= 0) ds.ram_bytes = d.ram[static_cast<size_t>(k)];
    p.devices.push_back(std::move(ds));
  }
  for (int i = 0; i < h.T; ++i) {
    OperatorNode op;
    op.name = h.op_names[static_cast<size_t>(i)];
    op.output_bytes = h.mass[static_cast<size_t>(i)];
    for (int k = 0; k < h.D; ++k) op.costs_ms.push_back(h.cost[static_cast<size_t>(k) * h.T + i]);
    if (d.pinned[static_cast<size_t>(i)] >= 0) op.pinned_device = d.pinned[static_cast<size_t>(i)];
    p.operators.push_back(std::move(op));
  }
  for (int e = 0; e < h.E; ++e)
    p.edges.push_back(TensorEdge{h.src[static_cast<size_t>(e)], h.dst[static_cast<size_t>(e)], d.overrides[static_cast<size_t>(e)]});
  for (const auto& l : d.links) p.copy_model.links.push_back({l.from, l.to, l.latency, l.rate});
  return p;
}

Problem load_problem_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) raise(Errc::IoError, "cannot open " + path);
  std::stringstream ss;
  ss << in.rdbuf();
  return load_problem(ss.str());
}

void validate_problem(const Problem& p) {
  const int T = p.op_count(), D = p.device_count();
  if (T == 0) raise(Errc::EmptyNetwork, "problem has no operators");
  if (D == 0) raise(Errc::MalformedDocument, "problem has no devices");
  for (const auto& op : p.operators)
    if (static_cast<int>(op.costs_ms.size()) != D) raise(Errc::DimensionMismatch, "operator " + op.name + " cost vector size");
  std::set<std::pair<int, int>> seen;
  std::vector<int> indeg(static_cast<size_t>(T), 0);
  for (const auto& e : p.edges) {
    if (e.src < 0 || e.dst < 0 || e.src >= T || e.dst >= T) raise(Errc::MalformedDocument, "edge endpoint out of range");
    const std::string id = std::to_string(e.src) + "->" + std::to_string(e.dst);
    if (e.src >= e.dst) raise(Errc::NonTopologicalEdge, "edge " + id + " violates index order");
    if (!seen.insert({e.src, e.dst}).second) raise(Errc::MalformedDocument, "duplicate edge " + id);
    ++indeg[static_cast<size_t>(e.dst)];
  }
  for (int v = 1; v < T; ++v)
    if (!indeg[static_cast<size_t>(v)])
      raise(Errc::MalformedDocument, "operator " + std::to_string(v) + " has no incoming edge; only operator 0 is a source");
}

Problem make_training_graph(const std::string& name, std::vector<DeviceSpec> devices, CopyLinkModel copy_model,
                            const std::vector<LayerSpec>& layers, std::int64_t input_bytes, int input_home) {
  // the chain is the forward network k-1 -> k; the library's one expansion
  // (xe::expand_training_graph) also serves the document loaders
  std::vector<xe::ForwardOp> fwd;
  for (size_t k = 0; k < layers.size(); ++k) {
    const auto& l = layers[k];
    fwd.push_back({l.name, {static_cast<int>(k)}, l.output_bytes, l.backward_output_bytes, l.costs_ms,
                   l.backward_costs_ms});
  }
  Problem p;
  p.name = name;
  const int D = static_cast<int>(devices.size());
  p.devices = std::move(devices);
  p.copy_model = std::move(copy_model);
  std::vector<std::string> names;
  std::vector<int64_t> bytes;
  std::vector<std::vector<double>> costs;
  std::vector<int32_t> src, dst;
  try {
    xe::expand_training_graph(D, input_bytes, input_home, fwd, names, bytes, costs, src, dst);
  } catch (const xe::Error& e) {
    raise(static_cast<Errc>(e.code - 1), e.what());
  }
  for (size_t i = 0; i < names.size(); ++i)
    p.operators.push_back({names[i], bytes[i], costs[i], i == 0 ? std::optional<int>(input_home) : std::nullopt});
  for (size_t e = 0; e < src.size(); ++e) p.edges.push_back(TensorEdge{src[e], dst[e], {}});
  validate_problem(p);
  return p;
}

std::int64_t save_all_budget(const Problem& p) {
  std::int64_t s = 0;
  for (const auto& op : p.operators) s += op.output_bytes;
  return s;
}

std::int64_t budget_percent(std::int64_t full, double pct) {
  if (!(pct > 0.0) || pct > 100.0) raise(Errc::PercentOutOfRange, "pct must be in (0, 100], got " + std::to_string(pct));
  if (full <= 0) raise(Errc::NonPositiveSize, "full budget must be positive");
  double whole = 0.0;
  if (std::modf(pct, &whole) == 0.0) return full * static_cast<std::int64_t>(whole) / 100;
  return static_cast<std::int64_t>(std::floor(static_cast<double>(full) * pct / 100.0));
}

double copy_cost(const Problem& p, const TensorEdge& e, int d, int d_to) {
  const int D = p.device_count();
  if (d < 0 || d_to < 0 || d >= D || d_to >= D) raise(Errc::DimensionMismatch, "device index");
  if (d == d_to) return 0.0;
  if (auto it = e.override_copy_ms.find({d, d_to}); it != e.override_copy_ms.end()) return it->second;
  const LinkSpec* pick = nullptr;
  int score = -1;
  for (const auto& l : p.copy_model.links) {
    const bool from_ok = l.from == -1 || l.from == d, to_ok = l.to == -1 || l.to == d_to;
    if (!from_ok || !to_ok) continue;
    const int s = (l.from == d) + (l.to == d_to);  // exact endpoints beat wildcards; first wins ties
    if (s > score) {
      score = s;
      pick = &l;
    }
  }
  if (!pick)
    raise(Errc::MissingLink, "no link covers " + p.devices[static_cast<size_t>(d)].id + "->" + p.devices[static_cast<size_t>(d_to)].id);
  return pick->latency_ms + static_cast<double>(p.operators[static_cast<size_t>(e.src)].output_bytes) / pick->bytes_per_ms;
}

Problem with_budgets(const Problem& p, const std::vector<std::int64_t>& budgets) {
  if (static_cast<int>(budgets.size()) != p.device_count()) raise(Errc::DimensionMismatch, "budget vector size");
  Problem q = p;
  for (size_t d = 0; d < budgets.size(); ++d) {
    if (budgets[d] <= 0) raise(Errc::NonPositiveSize, "budget for device " + q.devices[d].id);
    q.devices[d].budget_bytes = budgets[d];
    if (q.devices[d].ram_bytes && *q.devices[d].ram_bytes < budgets[d]) q.devices[d].ram_bytes = budgets[d];
  }
  return q;
}

// ============================ model.hpp ====================================

int MilpModel::edge_ordinal(int u, int v) const {
  for (int e = 0; e < E; ++e)
    if (problem.edges[static_cast<size_t>(e)].src == u && problem.edges[static_cast<size_t>(e)].dst == v) return e;
  return -1;
}

std::pair<int, int> MilpModel::f_edge(int eo) const {
  if (eo >= E) return {eo - E, eo - E};
  return {problem.edges[static_cast<size_t>(eo)].src, problem.edges[static_cast<size_t>(eo)].dst};
}

bool MilpModel::in_space(const VarRef& v) const {
  auto in = [](int x, int n) { return x >= 0 && x < n; };
  if (v.family == VarFamily::P) return in(v.a, T) && in(v.b, E) && in(v.c, D) && in(v.d, D) && v.c != v.d;
  if (v.d != 0 || !in(v.a, D) || !in(v.b, T)) return false;
  return in(v.c, v.family == VarFamily::F ? f_edges : T);
}

MilpModel build_model(const Problem& p, const ModelOptions& opts) {
  validate_problem(p);
  auto dm = std::make_shared<DeviceModel>();
  dm->prob = upload(describe(p, opts.energy));
  const xe_model_opts o = c_opts(opts);
  ck(xe_build_csr(dm->prob.get(), &o, &dm->csr));
  xe_csr_info info{};
  ck(xe_csr_get_info(dm->csr, &info));
  const size_t R = static_cast<size_t>(info.n_rows), Z = static_cast<size_t>(info.nnz), N = static_cast<size_t>(info.n_cols);
  std::vector<int64_t> rp(R + 1);
  std::vector<int32_t> col(Z), ord(R);
  std::vector<double> val(Z), rhs(R), obj(N);
  std::vector<int8_t> sense(R);
  std::vector<uint8_t> tag(R), present(N);
  xe_csr_host h{rp.data(), col.data(), val.data(), rhs.data(), sense.data(), tag.data(), ord.data(),
                obj.data(), present.data(), nullptr, nullptr, nullptr};
  ck(xe_csr_download(dm->csr, &h));

  MilpModel m;
  m.problem = p;
  m.options = opts;
  m.D = p.device_count();
  m.T = p.op_count();
  m.E = static_cast<int>(p.edges.size());
  m.f_edges = m.E + m.T;
  for (const auto& d : p.devices) m.budgets.push_back(d.budget_bytes);
  const Space sp = space_of(m.D, m.T, m.E);
  // objective map in key order: column order is VarRef order
  for (size_t j = 0; j < N; ++j)
    if (present[j]) m.objective.emplace_hint(m.objective.end(), sp.ref(static_cast<int64_t>(j)), obj[j]);
  const Desc ds = describe(p, std::nullopt);
  for (int t = 0; t < m.T; ++t)
    for (int e = 0; e < m.E; ++e)
      for (int a = 0; a < m.D; ++a)
        for (int b = 0; b < m.D; ++b) {
          if (a == b) continue;
          const double w = ds.w[(static_cast<size_t>(e) * m.D + a) * m.D + b];
          if (w != 0.0) m.quad.push_back({t, e, a, b, w});
        }
  for (int d = 0; d < m.D; ++d)
    for (int t = 0; t < m.T; ++t)
      for (int i = t + 1; i < m.T; ++i) m.fixed_zero.push_back(var_r(d, t, i));
  for (int d = 0; d < m.D; ++d)
    for (int t = 0; t < m.T; ++t)
      for (int i = t; i < m.T; ++i) m.fixed_zero.push_back(var_s(d, t, i));
  m.constraints.resize(R);
  for (size_t r = 0; r < R; ++r) {
    LinearConstraint& c = m.constraints[r];
    c.tag = static_cast<ConstraintTag>(tag[r]);
    c.ordinal = ord[r];
    c.rel = sense[r] == 'L' ? Relation::LE : sense[r] == 'G' ? Relation::GE : Relation::EQ;
    c.rhs = rhs[r];
    c.terms.reserve(static_cast<size_t>(rp[r + 1] - rp[r]));
    for (int64_t k = rp[r]; k < rp[r + 1]; ++k) c.terms.emplace_back(sp.ref(col[static_cast<size_t>(k)]), val[static_cast<size_t>(k)]);
  }
  m.device_model = dm;
  m.device_fingerprint = fingerprint(m);
  return m;
}

MilpModel add_energy_extension(const MilpModel& m, const EnergyModel& e) {
  check_energy(e, m.D, m.T);
  if (m.options.energy || !m.device_model || m.device_fingerprint != fingerprint(m))
    raise(Errc::DimensionMismatch,
          "add_energy_extension needs an unmodified energy-free model from build_model (the energy rows are "
          "assembled on the GPU together with the base rows)");
  ModelOptions o = m.options;
  o.energy = e;
  return build_model(m.problem, o);
}

std::optional<EnergyModel> parse_energy(const std::string& document_text, const Problem& p) {
  json j;
  try {
    j = json::parse(document_text);
  } catch (const json::exception& ex) {
    raise(Errc::MalformedDocument, ex.what());
  }
  if (!j.contains("energy")) return std::nullopt;
  const json& e = j["energy"];
  if (!e.is_object()) raise(Errc::MalformedDocument, "energy must be an object");
  EnergyModel em;
  auto nonneg = [](double v, const char* what) {
    if (!(v >= 0.0)) raise(Errc::NegativeCost, what);
    return v;
  };
  em.alpha = nonneg(e.value("alpha", 0.0), "alpha");
  em.board_joules = nonneg(e.value("board_joules", 0.0), "board_joules");
  if (e.contains("total_limit")) em.total_limit = nonneg(e["total_limit"].get<double>(), "total_limit");
  if (!e.contains("q_joules") || !e["q_joules"].is_object()) raise(Errc::IncompleteEnergyTable, "q_joules missing");
  const json& q = e["q_joules"];
  for (auto it = q.begin(); it != q.end(); ++it)
    if (p.find_device(it.key()) < 0) raise(Errc::UnknownDevice, it.key());
  em.q_joules.resize(p.devices.size());
  for (const auto& dev : p.devices) {
    if (!q.contains(dev.id)) raise(Errc::IncompleteEnergyTable, "q_joules missing device " + dev.id);
    const json& row = q[dev.id];
    if (!row.is_array() || row.size() != p.operators.size()) raise(Errc::IncompleteEnergyTable, "q_joules row for " + dev.id);
    auto& dst = em.q_joules[static_cast<size_t>(p.find_device(dev.id))];
    for (const auto& v : row) dst.push_back(nonneg(v.get<double>(), "q_joules"));
  }
  if (e.contains("device_limit")) {
    const json& dl = e["device_limit"];
    if (!dl.is_object()) raise(Errc::MalformedDocument, "device_limit must be an object");
    for (auto it = dl.begin(); it != dl.end(); ++it) {
      const int d = p.find_device(it.key());
      if (d < 0) raise(Errc::UnknownDevice, it.key());
      em.device_limit[d] = nonneg(it.value().get<double>(), "device_limit");
    }
  }
  return em;
}

double objective_value(const Assignment& a, const Problem& p, const ModelOptions& opts) {
  const int D = p.device_count(), T = p.op_count(), E = static_cast<int>(p.edges.size());
  auto in = [](int x, int n) { return x >= 0 && x < n; };
  for (const auto& [v, x] : a.values) {
    const bool ok = v.family == VarFamily::P ? in(v.a, T) && in(v.b, E) && in(v.c, D) && in(v.d, D)
                    : v.family == VarFamily::F ? in(v.a, D) && in(v.b, T) && in(v.c, E + T)
                                               : in(v.a, D) && in(v.b, T) && in(v.c, T);
    if (!ok) raise(Errc::DimensionMismatch, "assignment variable outside the problem's index space");
  }
  Handle h = upload(describe(p, opts.energy));
  const Space sp = space_of(D, T, E);
  std::vector<double> x(static_cast<size_t>(xe_model_cols(D, T, E)), 0.0);
  for (const auto& [v, val] : a.values) {
    if (v.family != VarFamily::R && v.family != VarFamily::Z) continue;  // the objective reads R and Z only
    if (v.d != 0) continue;
    x[static_cast<size_t>(sp.col(v))] = val;
  }
  const xe_model_opts o = c_opts(opts);
  double out = 0.0;
  ck(xe_objective_dense(h.get(), &o, x.data(), &out));
  return out;
}

std::vector<std::string> check_assignment(const MilpModel& m, const Assignment& a, double tol) {
  std::vector<std::string> out;
  const Space sp = space_of(m.D, m.T, m.E);
  std::vector<double> x(static_cast<size_t>(cols_of(m)), 0.0);
  for (const auto& [ref, val] : a.values) {
    if (!m.in_space(ref)) {
      out.push_back("variable outside model space");
      continue;
    }
    x[static_cast<size_t>(sp.col(ref))] = val;
    if (m.is_binary(ref.family) && std::abs(val) > tol && std::abs(val - 1.0) > tol) out.push_back("binary variable not 0/1");
    if (ref.family == VarFamily::U) {
      const double b = static_cast<double>(m.budgets[static_cast<size_t>(ref.a)]);
      if (val < -tol * std::max(1.0, b) || val > b * (1.0 + tol) + tol) out.push_back("U out of budget bounds");
    }
    if (ref.family == VarFamily::P && (val < -tol || val > 1.0 + tol)) out.push_back("P out of [0,1]");
  }
  for (const auto& ref : m.fixed_zero)
    if (std::abs(x[static_cast<size_t>(sp.col(ref))]) > tol) out.push_back("fixed-to-zero variable is nonzero");
  auto dm = device_model(m);
  std::vector<double> viol(m.constraints.size(), 0.0);
  int64_t nbad = 0;
  ck(xe_check_rows(dm->csr, x.data(), tol, viol.data(), &nbad));
  for (size_t r = 0; nbad > 0 && r < viol.size(); ++r)
    if (viol[r] > 0.0) {
      const auto& c = m.constraints[r];
      out.push_back(std::string(tag_name(c.tag)) + "_" + std::to_string(c.ordinal) + " violated by " + std::to_string(viol[r]));
      --nbad;
    }
  return out;
}

Assignment complete_assignment(const Problem& p, const ModelOptions& opts, const BitCube& R, const BitCube& S) {
  const int D = p.device_count(), T = p.op_count(), E = static_cast<int>(p.edges.size());
  if (R.D != D || R.T != T || S.D != D || S.T != T) raise(Errc::DimensionMismatch, "bit cube shape");
  Handle h = upload(describe(p, std::nullopt));
  const std::vector<uint32_t> cube = pack_cube(R, S);
  std::vector<double> x(static_cast<size_t>(xe_model_cols(D, T, E)));
  const xe_model_opts o = c_opts(opts);
  ck(xe_complete_cube(h.get(), &o, cube.data(), x.data()));
  // every variable of the space, in key order (the reference sets them all)
  Assignment a;
  const Space sp = space_of(D, T, E);
  for (size_t j = 0; j < x.size(); ++j) a.values.emplace_hint(a.values.end(), sp.ref(static_cast<int64_t>(j)), x[j]);
  return a;
}

BatchResult evaluate_candidates(const Problem& p, const ModelOptions& opts,
                                const std::vector<std::pair<BitCube, BitCube>>& candidates) {
  const int D = p.device_count(), T = p.op_count();
  Handle h = upload(describe(p, opts.energy));
  const size_t words = xe_cube_bytes(D, T) / 4;
  std::vector<uint32_t> cubes(words * candidates.size());
  for (size_t k = 0; k < candidates.size(); ++k) {
    const auto& [R, S] = candidates[k];
    if (R.D != D || R.T != T || S.D != D || S.T != T) raise(Errc::DimensionMismatch, "bit cube shape");
    const auto c = pack_cube(R, S);
    std::copy(c.begin(), c.end(), cubes.begin() + static_cast<std::ptrdiff_t>(k * words));
  }
  BatchResult r;
  const size_t n = candidates.size();
  r.objective.resize(n);
  r.peak.resize(n * static_cast<size_t>(D));
  r.flags.resize(n);
  xe_eval_out eo{r.objective.data(), r.peak.data(), r.flags.data()};
  xe_best best{};
  const xe_model_opts o = c_opts(opts);
  ck(xe_eval_cubes_host(h.get(), &o, cubes.data(), static_cast<int64_t>(n), &eo, XE_F_CHECK_MASK, &best));
  r.best_index = best.index;
  r.best_objective = best.obj;
  r.n_valid = best.n_valid;
  return r;
}

// ============================ mps_io.hpp ===================================

std::string format_number(double v) { return xe::format_number(v); }

std::string var_name(const VarRef& v) {
  static const char fam[] = "RSZFUP";
  std::string s(1, fam[static_cast<int>(v.family)]);
  for (int x : {static_cast<int>(v.a), static_cast<int>(v.b), static_cast<int>(v.c)}) s += "_" + std::to_string(x);
  if (v.family == VarFamily::P) s += "_" + std::to_string(v.d);
  return s;
}

std::optional<VarRef> parse_var_name(const std::string& name) {
  static const std::string fam = "RSZFUP";
  if (name.size() < 2 || name[1] != '_') return std::nullopt;
  const auto f = fam.find(name[0]);
  if (f == std::string::npos) return std::nullopt;
  std::vector<int> parts;
  size_t pos = 2;
  while (pos <= name.size()) {
    const size_t next = name.find('_', pos);
    const std::string tok = name.substr(pos, next == std::string::npos ? std::string::npos : next - pos);
    if (tok.empty() || tok.size() > 6 || !std::all_of(tok.begin(), tok.end(), [](char c) { return c >= '0' && c <= '9'; }))
      return std::nullopt;
    const long x = std::stol(tok);
    if (x > std::numeric_limits<std::int16_t>::max()) return std::nullopt;
    parts.push_back(static_cast<int>(x));
    if (next == std::string::npos) break;
    pos = next + 1;
  }
  const auto family = static_cast<VarFamily>(f);
  if (parts.size() != (family == VarFamily::P ? 4u : 3u)) return std::nullopt;
  return make_ref(family, parts[0], parts[1], parts[2], family == VarFamily::P ? parts[3] : 0);
}

std::string write_mps(const MilpModel& m) {
  auto dm = device_model(m);
  size_t len = 0;
  ck(xe_write_mps(dm->csr, nullptr, &len));
  std::string s(len, '\0');
  ck(xe_write_mps(dm->csr, s.data(), &len));
  s.resize(len);
  return s;
}

// The solution side of the external-solver bridge (mps_io.cpp:201-263):
// "<var> <value>" and CBC's "<idx> <var> <value> <cost>" lines, "# objective"
// comments and banners; binaries rounded within 1e-4.
namespace {
bool sol_is_number(const std::string& t) {
  if (t.empty()) return false;
  char* end = nullptr;
  std::strtod(t.c_str(), &end);
  return end == t.c_str() + t.size();
}
bool sol_is_integer(const std::string& t) {
  if (t.empty()) return false;
  size_t i = t[0] == '-' || t[0] == '+' ? 1 : 0;
  if (i == t.size()) return false;
  for (; i < t.size(); ++i)
    if (!std::isdigit(static_cast<unsigned char>(t[i]))) return false;
  return true;
}
std::string sol_lower(std::string t) {
  for (char& c : t) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
  return t;
}
}  // namespace

Assignment parse_solution(const std::string& text, const MilpModel& m) {
  Assignment a;
  bool any_var = false;
  auto record = [&](const std::string& name, double value) -> bool {
    auto ref = parse_var_name(name);
    if (!ref) return false;  // a banner word, not a variable
    if (!m.in_space(*ref)) raise(Errc::UnknownVariable, name);
    if (m.is_binary(ref->family)) {
      if (std::abs(value) <= 1e-4)
        value = 0.0;
      else if (std::abs(value - 1.0) <= 1e-4)
        value = 1.0;
      else
        raise(Errc::NonIntegralBinary, name + " = " + format_number(value));
    }
    a.set(*ref, value);
    any_var = true;
    return true;
  };
  std::istringstream in(text);
  std::string line;
  while (std::getline(in, line)) {
    std::istringstream ls(line);
    std::vector<std::string> tok;
    for (std::string t; ls >> t;) tok.push_back(t);
    if (tok.empty()) continue;
    if (tok[0][0] == '#') {
      if (tok.size() >= 3 && tok[0] == "#" && sol_lower(tok[1]) == "objective" && sol_is_number(tok[2]))
        a.objective_reported = std::strtod(tok[2].c_str(), nullptr);
      continue;
    }
    const std::string low = sol_lower(line);
    if (low.find("infeasible") != std::string::npos) raise(Errc::InfeasibleMarker, line);
    if (tok.size() == 2 && sol_is_number(tok[1]) && record(tok[0], std::strtod(tok[1].c_str(), nullptr))) continue;
    if (tok.size() == 4 && sol_is_integer(tok[0]) && sol_is_number(tok[2]) &&
        record(tok[1], std::strtod(tok[2].c_str(), nullptr)))
      continue;
    if (low.find("objective") != std::string::npos)
      for (auto it = tok.rbegin(); it != tok.rend(); ++it)
        if (sol_is_number(*it)) {
          a.objective_reported = std::strtod(it->c_str(), nullptr);
          break;
        }
  }
  if (!any_var) raise(Errc::EmptySolution, "no variable lines");
  return a;
}

std::string format_solution(const Assignment& a) {
  std::string out;
  if (a.objective_reported) out += "# objective " + format_number(*a.objective_reported) + "\n";
  for (const auto& [ref, val] : a.values) out += var_name(ref) + " " + format_number(val) + "\n";
  return out;
}

// ============================ solver.hpp ===================================

Assignment save_all_assignment(const Problem& p, const std::vector<int>& devices) {
  const int D = p.device_count(), T = p.op_count();
  if (static_cast<int>(devices.size()) != T) raise(Errc::DimensionMismatch, "one device per operator required");
  if (std::any_of(devices.begin(), devices.end(), [&](int d) { return d < 0 || d >= D; }))
    raise(Errc::DimensionMismatch, "device index out of range");
  BitCube R(D, T), S(D, T);
  for (int i = 0; i < T; ++i) {
    const int d = devices[static_cast<size_t>(i)];
    R.at(d, i, i) = 1;
    for (int t = i + 1; t < T; ++t) S.at(d, t, i) = 1;
  }
  return complete_assignment(p, {}, R, S);
}

Solution assignment_oracle(const Problem& p) {
  validate_problem(p);
  // the reference's enumeration guard (solver.cpp:47-49); the GPU sweep
  // itself goes to 2^40 through xe_assignment_oracle
  double combos = 1.0;
  for (int i = 0; i < p.op_count(); ++i) combos *= p.device_count();
  if (combos > 4.0e6) raise(Errc::TooLarge, "placement family too large to enumerate");
  if (p.device_count() == 1) {  // a single placement (T may exceed the sweep's 64)
    Solution s;
    s.status = SolveStatus::Optimal;
    s.backend = "oracle";
    s.assignment = save_all_assignment(p, std::vector<int>(static_cast<size_t>(p.op_count()), 0));
    s.objective_ms = objective_value(s.assignment, p, {});
    s.assignment.objective_reported = s.objective_ms;
    s.nodes_explored = 1;
    return s;
  }
  Handle h = upload(describe(p, std::nullopt));
  double best = 0.0;
  std::vector<int32_t> dev(static_cast<size_t>(p.op_count()));
  int64_t n = 0;
  ck(xe_assignment_oracle(h.get(), &best, dev.data(), &n));
  Solution s;
  s.status = SolveStatus::Optimal;
  s.backend = "oracle";
  s.objective_ms = best;
  s.assignment = save_all_assignment(p, std::vector<int>(dev.begin(), dev.end()));
  s.assignment.objective_reported = best;
  s.nodes_explored = n;
  return s;
}

Solution solve_exact(const Problem& p, const ModelOptions& opts, std::vector<std::int64_t> budgets,
                     const SearchLimits& limits) {
  Problem peff = budgets.empty() ? p : with_budgets(p, budgets);
  validate_problem(peff);
  const int D = peff.device_count(), T = peff.op_count();
  if (D * T > 64) raise(Errc::TooLarge, "state space exceeds 64 residency bits");
  Solution out;
  out.backend = "exact";
  out.objective_ms = std::numeric_limits<double>::quiet_NaN();
  Handle h = upload(describe(peff, opts.energy));
  const xe_model_opts o = c_opts(opts);
  xe_exact_opts eo;
  xe_exact_opts_default(&eo);
  if (limits.node_limit) eo.node_limit = *limits.node_limit;
  if (limits.time_limit_ms) eo.time_limit_ms = *limits.time_limit_ms;
  xe_exact_result r{};
  std::vector<uint32_t> cube(xe_cube_bytes(D, T) / 4);
  ck(xe_solve_exact(h.get(), &o, &eo, &r, cube.data(), nullptr));
  out.nodes_explored = r.nodes;
  if (r.status == 1) {
    out.status = SolveStatus::Infeasible;
    return out;
  }
  if (!r.found) {
    out.status = SolveStatus::LimitReached;
    return out;
  }
  // LimitReached keeps the best schedule found so far (solver.cpp:474-478)
  out.status = r.status == 0 ? SolveStatus::Optimal : SolveStatus::LimitReached;
  BitCube R(D, T), S(D, T);
  const int W = (T + 31) / 32;
  for (int which = 0; which < 2; ++which)
    for (int d = 0; d < D; ++d)
      for (int t = 0; t < T; ++t)
        for (int i = 0; i < T; ++i)
          if ((cube[((static_cast<size_t>(which) * D + d) * T + t) * W + i / 32] >> (i % 32)) & 1u)
            (which ? S : R).at(d, t, i) = 1;
  // fill_solution (solver.cpp:426-446): the search cost must be the
  // completed assignment's objective
  out.assignment = complete_assignment(peff, opts, R, S);
  const double obj = objective_value(out.assignment, peff, opts);
  if (std::abs(obj - r.objective) > 1e-9 * std::max(1.0, std::abs(obj)))
    raise(Errc::ObjectiveMismatch, "search cost " + format_number(r.objective) + " vs objective " + format_number(obj));
  out.objective_ms = r.objective;
  out.assignment.objective_reported = r.objective;
  return out;
}

Solution solve_search(const Problem& p, const ModelOptions& opts, const SearchParams& params) {
  return solve_search(p, opts, params, nullptr);
}

Solution solve_search(const Problem& p, const ModelOptions& opts, const SearchParams& params, xe_ctx* ctx) {
  validate_problem(p);
  const int D = p.device_count(), T = p.op_count();
  Handle h = upload(describe(p, opts.energy));
  xe_search_opts so;
  xe_search_opts_default(&so);
  so.n_per_round = params.candidates_per_round;
  so.rounds = params.rounds;
  so.edits = params.edits;
  so.seed = params.seed;
  so.use_lp = params.use_lp ? 1 : 0;
  so.chains = params.chains;
  so.chain_n = params.chain_neighbours;
  so.chain_iters = params.chain_iters;
  so.max_moves = params.max_moves;
  so.stall = params.stall;
  so.time_limit_ms = params.limits.time_limit_ms.value_or(0);
  const xe_model_opts o = c_opts(opts);
  xe_search_result r{};
  std::vector<uint32_t> cube(xe_cube_bytes(D, T) / 4);
  std::vector<int64_t> peaks(static_cast<size_t>(D));
  if (ctx)
    ck(xe_search_dist(h.get(), &o, &so, ctx, &r, cube.data(), peaks.data()));
  else
    ck(xe_search(h.get(), &o, &so, &r, cube.data(), peaks.data(), nullptr));
  Solution s;
  s.backend = "b200";
  s.nodes_explored = r.n_evaluated;
  if (!std::isfinite(r.objective)) {
    s.status = SolveStatus::LimitReached;
    s.objective_ms = std::numeric_limits<double>::quiet_NaN();
    return s;
  }
  // Optimal only against a certified lower bound (the LP duals' Lagrangian
  // value, valid for any PDHG iterate): the schedule is optimal to the
  // relative gap lp_tol (the MILP solvers' mip-gap convention) when it meets it
  const bool proven = r.has_lp && r.lp_certified && std::isfinite(r.lp_bound) &&
                      r.objective <= r.lp_bound + so.lp_tol * std::max(1.0, std::fabs(r.objective));
  s.status = proven ? SolveStatus::Optimal : SolveStatus::LimitReached;
  s.objective_ms = r.objective;
  // exact polish (D*T <= 64): solve_exact bounded by the search's objective
  // proves optimality and returns the reference's tail_less winner among the
  // optima (solver.cpp:87-92), kept when it is valid under the search's mask
  if (params.exact_polish && D * T <= 64 && !ctx) {
    xe_exact_opts eo;
    xe_exact_opts_default(&eo);
    eo.upper_bound = r.objective;
    eo.time_limit_ms = params.exact_polish_ms;
    xe_exact_result er{};
    std::vector<uint32_t> ecube(cube.size());
    ck(xe_solve_exact(h.get(), &o, &eo, &er, ecube.data(), nullptr));
    if (er.status == 0 && er.found && er.objective <= r.objective) {
      xe_best b{};
      ck(xe_eval_cubes_host(h.get(), &o, ecube.data(), 1, nullptr, so.valid_mask, &b));
      if (b.index == 0) {  // valid under the search's mask
        cube = ecube;
        s.objective_ms = b.obj;
        s.status = SolveStatus::Optimal;
      } else if (er.objective == r.objective) {
        s.status = SolveStatus::Optimal;  // the search's schedule attains the proven optimum
      }
    }
  }
  BitCube R(D, T), S(D, T);
  const int W = (T + 31) / 32;
  for (int which = 0; which < 2; ++which)
    for (int d = 0; d < D; ++d)
      for (int t = 0; t < T; ++t)
        for (int i = 0; i < T; ++i)
          if ((cube[((static_cast<size_t>(which) * D + d) * T + t) * W + i / 32] >> (i % 32)) & 1u)
            (which ? S : R).at(d, t, i) = 1;
  s.assignment = complete_assignment(p, opts, R, S);
  s.assignment.objective_reported = s.objective_ms;
  return s;
}

// ============================ schedule.hpp =================================
// decode / validate / replay on the GPU (csrc/schedule.cu), text forms by the
// library's one writer (csrc/schedule_text.cpp) with this Problem's names.

const char* violation_name(ViolationKind k) {
  switch (k) {
    case ViolationKind::ComputeWithoutInputs: return "ComputeWithoutInputs";
    case ViolationKind::CopyFromNonResident: return "CopyFromNonResident";
    case ViolationKind::BudgetExceeded: return "BudgetExceeded";
    case ViolationKind::FreeNonResident: return "FreeNonResident";
    case ViolationKind::UncomputedOperator: return "UncomputedOperator";
  }
  return "unknown";
}

namespace {

std::vector<xe_action> c_actions(const std::vector<Action>& a) {
  std::vector<xe_action> out(a.size());
  for (size_t k = 0; k < a.size(); ++k)
    out[k] = {static_cast<int32_t>(a[k].kind), a[k].timestep, a[k].slot, a[k].device, a[k].op,
              a[k].src,                        a[k].dst,      a[k].from, a[k].to};
  return out;
}

Action cxx_action(const xe_action& x) {
  Action a;
  a.kind = static_cast<ActionKind>(x.kind);
  a.timestep = x.timestep;
  a.slot = x.slot;
  a.device = x.device;
  a.op = x.op;
  a.src = x.src;
  a.dst = x.dst;
  a.from = x.from;
  a.to = x.to;
  return a;
}

struct NameTable {
  std::vector<const char*> dev, op;
  explicit NameTable(const Problem& p) {
    for (const auto& d : p.devices) dev.push_back(d.id.c_str());
    for (const auto& o : p.operators) op.push_back(o.name.c_str());
  }
};

// a handle for the problem's structure (no copy costs needed: decode and
// validate never price a copy)
Handle structure_handle(const Problem& p) {
  Problem q = p;
  if (q.device_count() > 1 && q.copy_model.links.empty()) q.copy_model.links.push_back({-1, -1, 0.0, 1.0});
  return upload(describe(q, std::nullopt));
}

}  // namespace

Schedule decode(const Assignment& a, const Problem& p) {
  validate_problem(p);
  const int D = p.device_count(), T = p.op_count(), E = static_cast<int>(p.edges.size());
  Handle h = structure_handle(p);
  const Space sp = space_of(D, T, E);
  std::vector<double> x(static_cast<size_t>(xe_model_cols(D, T, E)), 0.0);
  for (const auto& [v, val] : a.values) {
    if (v.family != VarFamily::R && v.family != VarFamily::S && v.family != VarFamily::Z && v.family != VarFamily::F)
      continue;
    if (v.a < 0 || v.a >= D || v.b < 0 || v.b >= T || v.c < 0 || v.c >= (v.family == VarFamily::F ? E + T : T)) continue;
    x[static_cast<size_t>(sp.col(v))] = val;
  }
  int64_t n = 0;
  xe_decode_error err{};
  ck(xe_decode_dense(h.get(), x.data(), &n, nullptr, &err));
  if (err.code) {
    const auto& ops = p.operators;
    if (err.code == 1)
      raise(Errc::IllegalAssignment, "operator " + ops[static_cast<size_t>(err.v)].name + " at t=" + std::to_string(err.t) +
                                         " needs tensor " + ops[static_cast<size_t>(err.u)].name + " resident on no device");
    raise(Errc::IllegalAssignment, "copy source for tensor " + ops[static_cast<size_t>(err.u)].name +
                                       " was freed earlier in timestep " + std::to_string(err.t));
  }
  std::vector<xe_action> acts(static_cast<size_t>(std::max<int64_t>(1, n)));
  ck(xe_decode_dense(h.get(), x.data(), &n, acts.data(), &err));
  Schedule s;
  s.problem = p;
  for (int64_t k = 0; k < n; ++k) s.actions.push_back(cxx_action(acts[static_cast<size_t>(k)]));
  return s;
}

ValidationReport validate(const Schedule& s, const Problem& p, const std::vector<std::int64_t>& budgets) {
  const int D = p.device_count();
  std::vector<std::int64_t> bud;
  if (budgets.empty())
    for (const auto& d : p.devices) bud.push_back(d.budget_bytes);
  else if (static_cast<int>(budgets.size()) == D)
    bud = budgets;
  else
    raise(Errc::DimensionMismatch, "one budget per device required");
  Handle h = structure_handle(p);
  const auto acts = c_actions(s.actions);
  const int64_t off[2] = {0, static_cast<int64_t>(acts.size())};
  int64_t voff[2] = {0, 0};
  ck(xe_validate_schedules(h.get(), acts.data(), off, 1, bud.data(), voff, nullptr));
  std::vector<xe_violation> vs(static_cast<size_t>(std::max<int64_t>(1, voff[1])));
  if (voff[1]) ck(xe_validate_schedules(h.get(), acts.data(), off, 1, bud.data(), voff, vs.data()));
  ValidationReport rep;
  const auto& ops = p.operators;
  for (int64_t k = 0; k < voff[1]; ++k) {
    const xe_violation& x = vs[static_cast<size_t>(k)];
    Violation v;
    v.kind = static_cast<ViolationKind>(x.kind);
    v.device = x.device;
    v.timestep = x.timestep;
    v.slot = x.slot;
    v.bytes = x.bytes;
    switch (v.kind) {  // the reference's detail strings (schedule.cpp:163-231)
      case ViolationKind::ComputeWithoutInputs:
        v.detail = "operator " + ops[static_cast<size_t>(x.a)].name + " missing input " + ops[static_cast<size_t>(x.b)].name;
        break;
      case ViolationKind::CopyFromNonResident:
      case ViolationKind::FreeNonResident:
        v.detail = "tensor " + ops[static_cast<size_t>(x.a)].name + " not resident on " + p.devices[static_cast<size_t>(x.device)].id;
        break;
      case ViolationKind::BudgetExceeded:
        v.detail = "device " + p.devices[static_cast<size_t>(x.device)].id + " holds " + std::to_string(x.bytes) +
                   " bytes over budget " + std::to_string(bud[static_cast<size_t>(x.device)]);
        break;
      case ViolationKind::UncomputedOperator:
        v.detail = "operator " + ops[static_cast<size_t>(x.a)].name + " never computed";
        break;
    }
    rep.violations.push_back(v);
  }
  return rep;
}

double action_cost(const Problem& p, const Action& act) {
  switch (act.kind) {
    case ActionKind::Compute:
      return p.operators[static_cast<size_t>(act.op)].costs_ms[static_cast<size_t>(act.device)];
    case ActionKind::Copy: {
      for (const auto& e : p.edges)
        if (e.src == act.src && e.dst == act.dst) return copy_cost(p, e, act.from, act.to);
      TensorEdge e;
      e.src = act.src;
      e.dst = act.dst;
      return copy_cost(p, e, act.from, act.to);
    }
    case ActionKind::Free:
    case ActionKind::Drop:
      return 0.0;
  }
  return 0.0;
}

Trace replay(const Schedule& s, const Problem& p, const ModelOptions& opts, const std::optional<Assignment>& a) {
  auto rep = validate(s, p);
  if (!rep.ok())
    raise(Errc::IllegalSchedule,
          std::to_string(rep.violations.size()) + " violation(s), first: " + rep.violations.front().detail);
  const int D = p.device_count(), T = p.op_count();
  Handle h = upload(describe(p, opts.energy));
  const xe_model_opts o = c_opts(opts);
  const auto acts = c_actions(s.actions);
  const int64_t off[2] = {0, static_cast<int64_t>(acts.size())};
  double total = 0.0, eq1 = 0.0;
  std::vector<int64_t> mem(static_cast<size_t>(D) * T * T), peaks(static_cast<size_t>(D));
  ck(xe_replay_schedules(h.get(), &o, acts.data(), off, 1, &total, &eq1, mem.data(), peaks.data()));
  Trace tr;
  if (std::isnan(total)) {  // a copy along an undeclared edge: priced by the link model
    total = 0.0;
    for (const auto& act : s.actions)
      if (act.kind == ActionKind::Compute || act.kind == ActionKind::Copy) total += action_cost(p, act);
  }
  tr.total_action_ms = total;
  tr.eq1_objective_ms = a ? objective_value(*a, p, opts) : eq1;
  tr.per_device_memory.assign(static_cast<size_t>(D), {});
  for (int d = 0; d < D; ++d)
    for (int t = 0; t < T; ++t)
      for (int v = 0; v < T; ++v)
        tr.per_device_memory[static_cast<size_t>(d)].push_back({t, v, mem[(static_cast<size_t>(d) * T + t) * T + v]});
  tr.peaks = peaks;
  return tr;
}

std::vector<std::pair<int, std::int64_t>> memory_timeline(const Trace& tr, int device) {
  if (device < 0 || device >= static_cast<int>(tr.per_device_memory.size()))
    raise(Errc::DimensionMismatch, "device index out of range");
  std::vector<std::pair<int, std::int64_t>> out;
  for (const auto& sample : tr.per_device_memory[static_cast<size_t>(device)]) {
    if (out.empty() || out.back().first != sample.timestep)
      out.push_back({sample.timestep, sample.bytes});
    else
      out.back().second = std::max(out.back().second, sample.bytes);
  }
  return out;
}

std::vector<std::pair<int, std::int64_t>> combined_memory_timeline(const Trace& tr) {
  std::vector<std::pair<int, std::int64_t>> out;
  for (int d = 0; d < static_cast<int>(tr.per_device_memory.size()); ++d) {
    auto series = memory_timeline(tr, d);
    if (out.empty()) {
      out = series;
    } else {
      for (size_t i = 0; i < out.size() && i < series.size(); ++i) out[i].second += series[i].second;
    }
  }
  return out;
}

std::string format_schedule(const Schedule& s) {
  const Problem& p = s.problem;
  Handle h = structure_handle(p);
  const NameTable nt(p);
  const auto acts = c_actions(s.actions);
  size_t len = 0;
  ck(xe_format_schedule_named(h.get(), acts.data(), static_cast<int64_t>(acts.size()), nt.dev.data(), nt.op.data(),
                              nullptr, &len));
  std::string out(len, '\0');
  ck(xe_format_schedule_named(h.get(), acts.data(), static_cast<int64_t>(acts.size()), nt.dev.data(), nt.op.data(),
                              out.data(), &len));
  return out;
}

Schedule parse_schedule(const std::string& text, const Problem& p) {
  Handle h = structure_handle(p);
  const NameTable nt(p);
  int64_t n = 0;
  ck(xe_parse_schedule_named(h.get(), text.c_str(), nt.dev.data(), nt.op.data(), p.name.c_str(), nullptr, &n));
  std::vector<xe_action> acts(static_cast<size_t>(std::max<int64_t>(1, n)));
  ck(xe_parse_schedule_named(h.get(), text.c_str(), nt.dev.data(), nt.op.data(), p.name.c_str(), acts.data(), &n));
  Schedule s;
  s.problem = p;
  for (int64_t k = 0; k < n; ++k) s.actions.push_back(cxx_action(acts[static_cast<size_t>(k)]));
  return s;
}

std::string trace_csv(const Trace& tr, const Problem& p) {
  std::string out = "device,timestep,slot,bytes\n";
  for (int d = 0; d < static_cast<int>(tr.per_device_memory.size()); ++d)
    for (const auto& sample : tr.per_device_memory[static_cast<size_t>(d)])
      out += p.devices[static_cast<size_t>(d)].id + "," + std::to_string(sample.timestep) + "," +
             std::to_string(sample.slot) + "," + std::to_string(sample.bytes) + "\n";
  return out;
}

}  // namespace xengine
