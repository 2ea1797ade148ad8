// SPDX-License-Identifier: Apache-2.0
//
// The reference's C++ API (include/xengine/*.hpp) exercised the way the
// reference's own suites use it, against the B200 library.  The pins are
// the reference tests' known answers (file:line under proj/tests/):
//   test_problem.cpp  loaders, budgets, copy_cost precedence, errors
//   test_model.cpp    row census, variable space, completion, checks, energy
//   test_mps_io.cpp   format_number, var names, golden F1 MPS bytes
//   test_solver.cpp   save_all_assignment, fig2 oracle = 11 with A on the cpu
//
//   test_api <golden_dir> host     no device needed (loaders and host math)
//   test_api <golden_dir> device   everything (needs the B200)
//
// Prints one line per failed check and "N checks, F failed"; exit 1 on failure.

#include <cmath>
#include <cstdio>
#include <fstream>
#include <functional>
#include <map>
#include <sstream>
#include <string>

#include "xengine/mps_io.hpp"
#include "xengine/model.hpp"
#include "xengine/problem.hpp"
#include "xengine/schedule.hpp"
#include "xengine/solver.hpp"
#include "xengine_b200.h"

using namespace xengine;

namespace {

int g_checks = 0, g_failed = 0;
std::string g_case;

void expect(bool ok, const char* what, int line) {
  ++g_checks;
  if (!ok) {
    ++g_failed;
    std::printf("FAIL [%s] line %d: %s\n", g_case.c_str(), line, what);
  }
}
#define CHECK(x) expect(static_cast<bool>(x), #x, __LINE__)
#define CHECK_THROWS_CODE(expr, errc)                          \
  do {                                                          \
    bool got_ = false;                                          \
    try {                                                       \
      (void)(expr);                                             \
    } catch (const Error& e_) {                                 \
      got_ = e_.code() == (errc);                               \
    }                                                           \
    expect(got_, #expr " throws " #errc, __LINE__);             \
  } while (0)
#define CHECK_THROWS(expr)                                      \
  do {                                                          \
    bool got_ = false;                                          \
    try {                                                       \
      (void)(expr);                                             \
    } catch (const Error&) {                                    \
      got_ = true;                                              \
    }                                                           \
    expect(got_, #expr " throws", __LINE__);                    \
  } while (0)

constexpr std::int64_t kMiB = 1024 * 1024;
std::string g_dir;

std::string slurp(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  std::stringstream ss;
  ss << in.rdbuf();
  return ss.str();
}
Problem fixture(const char* name) { return load_problem_file(g_dir + "/problems/" + name + ".json"); }

void run(const char* name, const std::function<void()>& body) {
  g_case = name;
  try {
    body();
  } catch (const std::exception& e) {
    ++g_checks;
    ++g_failed;
    std::printf("FAIL [%s] unexpected exception: %s\n", name, e.what());
  }
}

std::map<ConstraintTag, int> census(const MilpModel& m) {
  std::map<ConstraintTag, int> n;
  for (const auto& c : m.constraints) ++n[c.tag];
  return n;
}

// proj/tests/test_solver.cpp:29-44
Problem long_chain(int n, int devices) {
  Problem p;
  p.name = "chain" + std::to_string(n);
  for (int d = 0; d < devices; ++d) p.devices.push_back({"dev" + std::to_string(d), std::int64_t(n) * kMiB, {}});
  for (int i = 0; i < n; ++i) {
    OperatorNode op;
    op.name = "op" + std::to_string(i);
    op.output_bytes = kMiB;
    op.costs_ms.assign(size_t(devices), 1.0);
    p.operators.push_back(op);
    if (i > 0) p.edges.push_back({i - 1, i, {}});
  }
  p.copy_model.links.push_back({-1, -1, 0.125, double(1 << 30)});
  return p;
}
int count_r(const Assignment& a) {
  int n = 0;
  for (const auto& [v, x] : a.values)
    if (v.family == VarFamily::R && x > 0.5) ++n;
  return n;
}

BitCube diagonal_on(const Problem& p, int d) {
  BitCube r(p.device_count(), p.op_count());
  for (int t = 0; t < p.op_count(); ++t) r.at(d, t, t) = 1;
  return r;
}
BitCube save_everything_on(const Problem& p, int d) {
  BitCube s(p.device_count(), p.op_count());
  for (int t = 0; t < p.op_count(); ++t)
    for (int i = 0; i < t; ++i) s.at(d, t, i) = 1;
  return s;
}

// ------------------------------------------------------------- host only
void host_cases() {
  run("chain3 document", [] {
    Problem p = fixture("chain3");
    CHECK(p.device_count() == 1);
    CHECK(p.op_count() == 3);
    CHECK(p.operators[1].costs_ms == std::vector<double>{3.0});
    CHECK(p.devices[0].budget_bytes == 12 * kMiB);
    CHECK(save_all_budget(p) == 12 * kMiB);
  });
  run("fig2 training-graph layout", [] {
    Problem p = fixture("fig2");
    CHECK(p.op_count() == 7);
    CHECK(p.edges.size() == 9u);
    CHECK(p.operators[0].costs_ms[1] == kProhibitiveMs);  // the pinned input
    CHECK(p.find_device("cpu") == 0);
    CHECK(p.find_device("gpu") == 1);
    CHECK(p.find_device("tpu") == -1);
  });
  run("chain_lowmem shape", [] {
    Problem p = fixture("chain_lowmem");
    CHECK(p.op_count() == 10);
    CHECK(save_all_budget(p) == 34 * kMiB);
    CHECK(p.edges.size() == 10u);
    CHECK(p.edges.back().src == 1 && p.edges.back().dst == 8);
  });
  run("make_training_graph one layer", [] {
    std::vector<DeviceSpec> devices{{"cpu", 64 * kMiB, {}}, {"gpu", 64 * kMiB, {}}};
    CopyLinkModel links{{{-1, -1, 0.5, double(kMiB)}}};
    std::vector<LayerSpec> layers{{"L1", 2 * kMiB, {1.0, 2.0}, 3 * kMiB, {4.0, 5.0}}};
    Problem p = make_training_graph("tiny", devices, links, layers, kMiB, 1);
    CHECK(p.op_count() == 3);
    CHECK(p.operators[2].name == "L1'");
    CHECK(p.operators[0].pinned_device == 1);
    CHECK(p.operators[0].costs_ms[0] >= kProhibitiveMs);
    CHECK(p.edges.size() == 3u);
    CHECK(p.edges[1].src == 1 && p.edges[1].dst == 2);
    CHECK(p.edges[2].src == 0 && p.edges[2].dst == 2);
  });
  run("budget_percent", [] {
    CHECK(budget_percent(320 * kMiB, 65.0) == 208 * kMiB);
    CHECK(budget_percent(100, 100.0) == 100);
    CHECK(budget_percent(101, 50.0) == 50);
    CHECK_THROWS_CODE(budget_percent(100, 0.0), Errc::PercentOutOfRange);
    CHECK_THROWS_CODE(budget_percent(100, 100.5), Errc::PercentOutOfRange);
    CHECK_THROWS_CODE(budget_percent(0, 50.0), Errc::NonPositiveSize);
  });
  run("copy_cost precedence", [] {
    Problem p = fixture("fig2");
    CHECK(copy_cost(p, p.edges[0], 0, 1) == 1.0);
    TensorEdge bare = p.edges[0];
    bare.override_copy_ms.clear();
    CHECK_THROWS_CODE(copy_cost(p, bare, 0, 1), Errc::MissingLink);
    CHECK(copy_cost(p, bare, 1, 1) == 0.0);
    Problem q = p;
    q.copy_model.links.push_back({-1, -1, 0.25, double(2 * kMiB)});
    CHECK(std::fabs(copy_cost(q, bare, 0, 1) - 2.25) < 1e-12);
    q.copy_model.links.insert(q.copy_model.links.begin(), {1, 0, 1.5, double(4 * kMiB)});
    CHECK(std::fabs(copy_cost(q, bare, 1, 0) - 2.5) < 1e-12);
  });
  run("with_budgets", [] {
    Problem p = fixture("chain3");
    Problem q = with_budgets(p, {7 * kMiB});
    CHECK(q.devices[0].budget_bytes == 7 * kMiB);
    CHECK(p.devices[0].budget_bytes == 12 * kMiB);
    CHECK_THROWS(with_budgets(p, {kMiB, kMiB}));
    CHECK_THROWS(with_budgets(p, {0}));
  });
  run("loader error codes", [] {
    CHECK_THROWS_CODE(load_problem("{ not json"), Errc::MalformedDocument);
    CHECK_THROWS_CODE(load_problem("[1,2,3]"), Errc::MalformedDocument);
    CHECK_THROWS_CODE(load_problem(R"({"name":"x","devices":[]})"), Errc::MalformedDocument);
    CHECK_THROWS_CODE(load_problem(R"({"devices":[{"id":"cpu","budget_bytes":1024}],"operators":[]})"),
                      Errc::EmptyNetwork);
    CHECK_THROWS_CODE(load_problem(R"({"devices":[{"id":"c","budget_bytes":8}],
        "operators":[{"name":"a","output_bytes":0,"costs_ms":{"c":1.0}}]})"), Errc::NonPositiveSize);
    CHECK_THROWS_CODE(load_problem(R"({"devices":[{"id":"c","budget_bytes":8}],
        "operators":[{"name":"a","output_bytes":4,"costs_ms":{"c":-1.0}}]})"), Errc::NegativeCost);
    CHECK_THROWS_CODE(load_problem(R"({"devices":[{"id":"c","budget_bytes":8}],
        "operators":[{"name":"a","output_bytes":4,"costs_ms":{"g":1.0}}]})"), Errc::UnknownDevice);
    CHECK_THROWS_CODE(load_problem(R"({"devices":[{"id":"c","budget_bytes":8}],
        "operators":[{"name":"a","output_bytes":4,"costs_ms":{"c":1.0}},{"name":"b","output_bytes":4,"costs_ms":{"c":1.0}}],
        "edges":[[1,0]]})"), Errc::NonTopologicalEdge);
    CHECK_THROWS_CODE(load_problem_file("/nonexistent/nowhere.json"), Errc::IoError);
  });
  run("omitted device cost is the sentinel", [] {
    Problem p = load_problem(R"({"name":"partial","devices":[{"id":"cpu","budget_bytes":1048576},
        {"id":"gpu","budget_bytes":1048576}],"operators":[{"name":"a","output_bytes":1024,"costs_ms":{"cpu":1.0}}]})");
    CHECK(p.operators[0].costs_ms.size() == 2u);
    CHECK(p.operators[0].costs_ms[1] == kProhibitiveMs);
  });
  run("format_number", [] {
    CHECK(format_number(0.0) == "0");
    CHECK(format_number(-3.0) == "-3");
    CHECK(format_number(2.5) == "2.5");
    CHECK(format_number(1e9) == "1000000000");
    CHECK(format_number(12582912.0) == "12582912");
    CHECK(format_number(1.0 / 3.0) == "0.3333333333333333");
    for (double v : {0.1, 1.0 / 3.0, 1e-9, 123456.789, 0.25, 2.0 / 7.0}) CHECK(std::stod(format_number(v)) == v);
  });
  run("var names round trip", [] {
    for (const VarRef& v : {var_r(0, 1, 2), var_s(1, 6, 3), var_z(0, 0, 0), var_f(1, 3, 15), var_u(0, 2, 2),
                            var_p(4, 8, 0, 1)}) {
      auto back = parse_var_name(var_name(v));
      CHECK(back.has_value() && *back == v);
    }
    CHECK(var_name(var_p(4, 8, 0, 1)) == "P_4_8_0_1");
    CHECK(!parse_var_name("").has_value());
    CHECK(!parse_var_name("Q_0_0_0").has_value());
    CHECK(!parse_var_name("R_0_0").has_value());
    CHECK(!parse_var_name("R_0_0_x").has_value());
    CHECK(!parse_var_name("P_0_0_0").has_value());
    CHECK(!parse_var_name("R_0_0_0_0").has_value());
  });
  run("parse_energy", [] {
    Problem p = fixture("fig2_energy");
    auto e = parse_energy(slurp(g_dir + "/problems/fig2_energy.json"), p);
    CHECK(e.has_value());
    if (!e) return;
    CHECK(e->alpha == 0.0);
    CHECK(e->q_joules[0] == std::vector<double>(7, 1.0));
    CHECK(e->q_joules[1][2] == 10.0);
    CHECK(e->device_limit.at(1) == 5.0);
    CHECK(!e->total_limit.has_value());
    CHECK(!parse_energy(slurp(g_dir + "/problems/chain3.json"), fixture("chain3")).has_value());
  });
  run("status and tag names", [] {
    CHECK(std::string(status_name(SolveStatus::Optimal)) == "optimal");
    CHECK(std::string(tag_name(ConstraintTag::EQ16_HI)) == "EQ16_HI");
    CHECK(std::string(Error(Errc::TooLarge, "x").what()) == "TooLarge: x");
  });
}

// ------------------------------------------------------------ device
void device_cases() {
  run("chain3 row census", [] {
    MilpModel m = build_model(fixture("chain3"));
    CHECK(m.D == 1 && m.T == 3 && m.E == 2 && m.f_edges == 5);
    CHECK(m.fixed_zero.size() == 9u);
    auto n = census(m);
    CHECK(n[ConstraintTag::EQ8] == 6);
    CHECK(n[ConstraintTag::EQ9] == 1);
    CHECK(n[ConstraintTag::EQ11] == 6);
    CHECK(n[ConstraintTag::EQ12] == 6);
    CHECK(n[ConstraintTag::EQ13] == 3);
    CHECK(n[ConstraintTag::EQ14] == 6);
    CHECK(n[ConstraintTag::EQ16_LO] == 15);
    CHECK(n[ConstraintTag::EQ16_HI] == 15);
    CHECK(n[ConstraintTag::Z_LINK] == 27);
    CHECK(n[ConstraintTag::P_LINK] == 0);
    CHECK(m.quad.empty());
    CHECK(m.objective.size() == 9u);
    std::map<ConstraintTag, int> next;
    bool dense = true;
    for (const auto& c : m.constraints) dense = dense && c.ordinal == next[c.tag]++;
    CHECK(dense);
  });
  run("fig2 copy products", [] {
    MilpModel m = build_model(fixture("fig2"));
    CHECK(m.D == 2 && m.T == 7 && m.E == 9 && m.f_edges == 16);
    CHECK(census(m)[ConstraintTag::P_LINK] == 126);
    CHECK(m.quad.size() == 126u);
    bool unit = true;
    for (const auto& q : m.quad) unit = unit && q.w == 1.0 && q.d_src != q.d_cmp;
    CHECK(unit);
    CHECK(m.objective.size() == size_t(98 - 7 + 126));
    CHECK(m.fixed_zero.size() == size_t(2 * (21 + 28)));
    CHECK(m.in_space(var_r(1, 6, 6)) && !m.in_space(var_r(2, 0, 0)) && !m.in_space(var_p(0, 0, 1, 1)));
    CHECK(m.edge_ordinal(2, 4) == 4 && m.edge_ordinal(1, 4) == -1 && m.self_ordinal(0) == 9);
    CHECK(m.f_edge(15) == std::make_pair(6, 6));
  });
  run("EQ9 row", [] {
    MilpModel m = build_model(fixture("chain3"));
    const LinearConstraint* nine = nullptr;
    for (const auto& c : m.constraints)
      if (c.tag == ConstraintTag::EQ9) nine = &c;
    CHECK(nine && nine->rel == Relation::EQ && nine->rhs == 3.0 && nine->terms.size() == 3u);
  });
  run("golden F1 MPS", [] {
    const std::string text = write_mps(build_model(fixture("chain3")));
    CHECK(text == slurp(g_dir + "/f1_golden.mps"));
    MilpModel m = build_model(fixture("chain3"));
    m.device_model.reset();  // hand-built path: the rows are uploaded
    CHECK(write_mps(m) == text);
  });
  run("complete_assignment save-all chain", [] {
    Problem p = fixture("chain3");
    MilpModel m = build_model(p);
    Assignment a = complete_assignment(p, {}, diagonal_on(p, 0), save_everything_on(p, 0));
    CHECK(check_assignment(m, a).empty());
    CHECK(objective_value(a, p) == 9.0);
    CHECK(a.at(var_z(0, 1, 0)) == 1.0 && a.at(var_z(0, 1, 1)) == 1.0);
    CHECK(a.at(var_u(0, 0, 0)) == 4.0 * kMiB);
    CHECK(a.at(var_u(0, 1, 1)) == 8.0 * kMiB);
    CHECK(a.at(var_u(0, 2, 2)) == 12.0 * kMiB);
    bool none_freed = true;
    for (int t = 0; t + 1 < m.T; ++t)
      for (int eo = 0; eo < m.f_edges; ++eo) none_freed = none_freed && a.at(var_f(0, t, eo)) == 0.0;
    CHECK(none_freed);
    CHECK(a.values.size() == size_t(xe_model_cols(m.D, m.T, m.E)));
  });
  run("missing saves violate dependency rows", [] {
    Problem p = fixture("chain3");
    MilpModel m = build_model(p);
    BitCube none(p.device_count(), p.op_count());
    CHECK(!check_assignment(m, complete_assignment(p, {}, diagonal_on(p, 0), none)).empty());
  });
  run("tampered assignments are flagged", [] {
    Problem p = fixture("chain3");
    MilpModel m = build_model(p);
    Assignment a = complete_assignment(p, {}, diagonal_on(p, 0), save_everything_on(p, 0));
    Assignment t1 = a;
    t1.set(var_r(0, 0, 2), 1.0);
    CHECK(!check_assignment(m, t1).empty());
    Assignment t2 = a;
    t2.set(var_u(0, 0, 0), double(13 * kMiB));
    auto v = check_assignment(m, t2);
    CHECK(!v.empty());
    bool bound = false, row = false;
    for (const auto& s : v) {
      bound = bound || s == "U out of budget bounds";
      row = row || s.rfind("EQ13_0 violated by", 0) == 0;
    }
    CHECK(bound && row);
  });
  run("energy extension", [] {
    Problem p = fixture("fig2_energy");
    EnergyModel e = *parse_energy(slurp(g_dir + "/problems/fig2_energy.json"), p);
    ModelOptions o;
    o.energy = e;
    MilpModel m = build_model(p, o);
    CHECK(census(m)[ConstraintTag::ENERGY_DEV] == 49);
    CHECK(census(m)[ConstraintTag::ENERGY_TOTAL] == 0);
    MilpModel base = build_model(p);
    CHECK(m.objective == base.objective);
    e.alpha = 1.0;
    o.energy = e;
    MilpModel heavy = build_model(p, o);
    CHECK(heavy.objective.at(var_r(1, 2, 2)) == base.objective.at(var_r(1, 2, 2)) + 10.0);
    bool found = false;
    for (const auto& c : heavy.constraints)
      if (c.tag == ConstraintTag::ENERGY_DEV && c.terms.size() == 1 && c.terms[0].first == var_r(1, 2, 2))
        found = c.terms[0].second == 10.0 && c.rel == Relation::LE && c.rhs == 5.0;
    CHECK(found);
    EnergyModel bad = e;
    bad.q_joules.pop_back();
    CHECK_THROWS_CODE(add_energy_extension(build_model(p), bad), Errc::IncompleteEnergyTable);
    EnergyModel tot = *parse_energy(slurp(g_dir + "/problems/fig2_energy.json"), p);
    tot.total_limit = 20.0;
    tot.board_joules = 3.0;
    MilpModel mt = add_energy_extension(build_model(p), tot);
    CHECK(census(mt)[ConstraintTag::ENERGY_TOTAL] == 7);
    bool rhs17 = true;
    for (const auto& c : mt.constraints)
      if (c.tag == ConstraintTag::ENERGY_TOTAL) rhs17 = rhs17 && c.rhs == 17.0;
    CHECK(rhs17);
  });
  run("objective_value copies and energy", [] {
    Problem p = fixture("fig2_energy");
    std::vector<int> devices{0, 1, 1, 1, 1, 1, 1};
    Assignment a = save_all_assignment(p, devices);
    const double base = objective_value(a, p);
    double compute = 0.0;
    for (int i = 0; i < p.op_count(); ++i) compute += p.operators[size_t(i)].costs_ms[size_t(devices[size_t(i)])];
    CHECK(std::fabs(base - (compute + 2.0)) < 1e-12);
    ModelOptions o;
    o.energy = parse_energy(slurp(g_dir + "/problems/fig2_energy.json"), p);
    o.energy->alpha = 2.0;
    CHECK(std::fabs(objective_value(a, p, o) - (base + 32.0)) < 1e-12);
  });
  run("save_all_assignment validation", [] {
    Problem p = fixture("fig2");
    CHECK_THROWS_CODE(save_all_assignment(p, {0, 1}), Errc::DimensionMismatch);
    CHECK_THROWS_CODE(save_all_assignment(p, {0, 1, 1, 1, 1, 1, 5}), Errc::DimensionMismatch);
  });
  run("fig2 oracle = 11 with A on the cpu", [] {
    Problem p = fixture("fig2");
    Solution s = assignment_oracle(p);
    CHECK(s.status == SolveStatus::Optimal);
    CHECK(s.backend == "oracle");
    CHECK(s.objective_ms == 11.0);
    CHECK(s.nodes_explored == 128);
    CHECK(s.assignment.at(var_r(0, 1, 1)) == 1.0);
    CHECK(s.assignment.objective_reported == 11.0);
    CHECK(check_assignment(build_model(p), s.assignment).empty());
  });
  // ---- solve_exact: proj/tests/test_solver.cpp:66-190
  run("solve_exact: chain3 = 9.0 with the identity R", [] {
    Problem p = fixture("chain3");
    Solution s = solve_exact(p);
    CHECK(s.status == SolveStatus::Optimal);
    CHECK(s.backend == "exact");
    CHECK(s.objective_ms == 9.0);
    CHECK(s.assignment.objective_reported == 9.0);
    for (int t = 0; t < 3; ++t)
      for (int i = 0; i < 3; ++i) CHECK(s.assignment.at(var_r(0, t, i)) == (t == i ? 1.0 : 0.0));
    CHECK(count_r(s.assignment) == 3);
  });
  run("solve_exact: chain3 infeasible at 3 MiB, 9.0 at 8 MiB", [] {
    Problem p = fixture("chain3");
    CHECK(solve_exact(p, {}, {3 * kMiB}).status == SolveStatus::Infeasible);
    Solution ok = solve_exact(p, {}, {8 * kMiB});
    CHECK(ok.status == SolveStatus::Optimal);
    CHECK(ok.objective_ms == 9.0);
  });
  run("solve_exact: fig2 = 11 with the reference's twin (A on the gpu)", [] {
    Problem p = fixture("fig2");
    Solution s = solve_exact(p);
    CHECK(s.status == SolveStatus::Optimal);
    CHECK(s.objective_ms == 11.0);
    CHECK(s.assignment.at(var_r(0, 0, 0)) == 1.0);
    CHECK(s.assignment.at(var_r(1, 1, 1)) == 1.0);
    CHECK(s.assignment.at(var_r(0, 6, 6)) == 1.0);
    CHECK(check_assignment(build_model(p), s.assignment).empty());
    CHECK(s.nodes_explored > 1000);
  });
  run("solve_exact: chain_lowmem sweep 24/24/24/24/27, 12 computes at 25 %", [] {
    Problem p = fixture("chain_lowmem");
    CHECK(save_all_budget(p) == 34 * kMiB);
    const double pct[5] = {100, 65, 50, 35, 25}, want[5] = {24, 24, 24, 24, 27};
    for (int k = 0; k < 5; ++k) {
      Solution s = solve_exact(p, {}, {budget_percent(save_all_budget(p), pct[k])});
      CHECK(s.status == SolveStatus::Optimal);
      CHECK(s.objective_ms == want[k]);
    }
    Solution tight = solve_exact(p, {}, {budget_percent(save_all_budget(p), 25.0)});
    CHECK(count_r(tight.assignment) == 12);
    CHECK(solve_exact(p, {}, {10 * kMiB}).objective_ms == 24.0);
    CHECK(solve_exact(p, {}, {9 * kMiB}).objective_ms == 27.0);
    CHECK(solve_exact(p, {}, {8 * kMiB}).objective_ms == 27.0);
    CHECK(solve_exact(p, {}, {4 * kMiB - 1}).status == SolveStatus::Infeasible);
  });
  run("solve_exact: limits return LimitReached", [] {
    Problem p = fixture("fig2");
    SearchLimits one;
    one.node_limit = 1;
    CHECK(solve_exact(p, {}, {}, one).status == SolveStatus::LimitReached);
    SearchLimits some;
    some.node_limit = 3000;
    Solution part = solve_exact(p, {}, {}, some);
    CHECK(part.status == SolveStatus::LimitReached);
    CHECK(part.nodes_explored <= 3000 + 1);
    SearchLimits instant;
    instant.time_limit_ms = 0;
    CHECK(solve_exact(p, {}, {}, instant).status == SolveStatus::LimitReached);
  });
  run("solve_exact: TooLarge beyond 64 residency bits; a 12-op chain on one device", [] {
    CHECK_THROWS_CODE(solve_exact(long_chain(33, 2)), Errc::TooLarge);
    CHECK(solve_exact(long_chain(12, 1)).status == SolveStatus::Optimal);
    CHECK_THROWS_CODE(assignment_oracle(long_chain(23, 2)), Errc::TooLarge);
    CHECK(assignment_oracle(long_chain(23, 1)).status == SolveStatus::Optimal);
  });
  // ---- mps_io.hpp parse_solution / format_solution: proj/tests/test_mps_io.cpp:205-286
  run("parse_solution accepts both solver layouts", [] {
    MilpModel m = build_model(fixture("chain3"));
    Assignment a = parse_solution("R_0_0_0 1\nU_0_0_0 4194304\n", m);
    CHECK(a.at(var_r(0, 0, 0)) == 1.0);
    CHECK(a.at(var_u(0, 0, 0)) == 4194304.0);
    CHECK(a.at(var_r(0, 1, 1)) == 0.0);
    CHECK(!a.objective_reported.has_value());
    Assignment b = parse_solution(
        "Optimal - objective value 9.00000000\n      0 R_0_0_0               1                       2\n"
        "      5 U_0_0_0         4194304                       0\n", m);
    CHECK(b.at(var_r(0, 0, 0)) == 1.0 && b.at(var_u(0, 0, 0)) == 4194304.0);
    CHECK(b.objective_reported.has_value() && *b.objective_reported == 9.0);
    Assignment c = parse_solution("# objective 9.5\nR_0_0_0 1\n", m);
    CHECK(c.objective_reported.has_value() && *c.objective_reported == 9.5);
    Assignment d = parse_solution("R_0_0_0 0.99999995\nS_0_1_0 1.00000002\n", m);
    CHECK(d.at(var_r(0, 0, 0)) == 1.0 && d.at(var_s(0, 1, 0)) == 1.0);
    CHECK_THROWS_CODE(parse_solution("R_0_0_0 0.5\n", m), Errc::NonIntegralBinary);
    CHECK_THROWS_CODE(parse_solution("R_9_9_9 1\n", m), Errc::UnknownVariable);
    CHECK(parse_solution("Status reading finished\nR_0_0_0 1\n", m).at(var_r(0, 0, 0)) == 1.0);
    CHECK_THROWS_CODE(parse_solution("Infeasible - objective value 0\n", m), Errc::InfeasibleMarker);
    CHECK_THROWS_CODE(parse_solution("# nothing here\n", m), Errc::EmptySolution);
  });
  run("format_solution round trips through parse_solution (fig2 exact)", [] {
    Problem p = fixture("fig2");
    MilpModel m = build_model(p);
    Solution sol = solve_exact(p);
    const std::string text = format_solution(sol.assignment);
    Assignment back = parse_solution(text, m);
    CHECK(back.objective_reported.has_value() && *back.objective_reported == sol.objective_ms);
    bool same = true;
    for (const auto& [ref, value] : sol.assignment.values) same = same && back.at(ref) == value;
    for (const auto& [ref, value] : back.values) same = same && sol.assignment.at(ref) == value;
    CHECK(same);
    CHECK(format_solution(sol.assignment) == text);
  });
  // ---- schedule.hpp: proj/tests/test_schedule.cpp:300-370
  run("replay accounts costs and memory (fig2 exact optimum)", [] {
    Problem p = fixture("fig2");
    Solution sol = solve_exact(p);
    Schedule s = decode(sol.assignment, p);
    CHECK(validate(s, p).ok());
    Trace with_a = replay(s, p, {}, sol.assignment);
    CHECK(with_a.total_action_ms == 11.0);
    CHECK(with_a.eq1_objective_ms == 11.0);
    Trace bare = replay(s, p);
    CHECK(bare.eq1_objective_ms == with_a.eq1_objective_ms);
    CHECK(bare.total_action_ms == with_a.total_action_ms);
    CHECK(with_a.per_device_memory.size() == 2);
    CHECK(with_a.per_device_memory[0].size() == 49);
    CHECK(with_a.peaks[0] == 8 * kMiB);
    CHECK(with_a.peaks[1] == 32 * kMiB);
    auto c = combined_memory_timeline(with_a);
    auto a0 = memory_timeline(with_a, 0), a1 = memory_timeline(with_a, 1);
    bool sum = c.size() == a0.size();
    for (size_t t = 0; sum && t < c.size(); ++t) sum = c[t].second == a0[t].second + a1[t].second;
    CHECK(sum);
    // text round trip
    Schedule back = parse_schedule(format_schedule(s), p);
    CHECK(back.actions == s.actions);
    CHECK(trace_csv(with_a, p).rfind("device,timestep,slot,bytes\ncpu,0,0,", 0) == 0);
  });
  run("memory timelines match the hand-computed chains", [] {
    Problem p = fixture("chain3");
    Solution sol = solve_exact(p);
    Trace lean = replay(decode(sol.assignment, p), p, {}, sol.assignment);
    using Series = std::vector<std::pair<int, std::int64_t>>;
    CHECK(memory_timeline(lean, 0) == (Series{{0, 4 * kMiB}, {1, 8 * kMiB}, {2, 8 * kMiB}}));
    Assignment all = save_all_assignment(p, {0, 0, 0});
    Trace fat = replay(decode(all, p), p, {}, all);
    CHECK(memory_timeline(fat, 0) == (Series{{0, 4 * kMiB}, {1, 8 * kMiB}, {2, 12 * kMiB}}));
    CHECK(combined_memory_timeline(fat) == memory_timeline(fat, 0));
    CHECK_THROWS(memory_timeline(fat, 1));
  });
  run("replay refuses illegal schedules; validate reports them", [] {
    Problem p = fixture("chain3");
    Schedule s = decode(solve_exact(p).assignment, p);
    s.actions.erase(s.actions.begin());
    CHECK_THROWS_CODE(replay(s, p), Errc::IllegalSchedule);
    ValidationReport rep = validate(s, p);
    CHECK(!rep.ok());
    CHECK_THROWS_CODE(validate(s, p, {kMiB, kMiB}), Errc::DimensionMismatch);
  });
  run("action costs", [] {
    Problem p = fixture("fig2");
    CHECK(action_cost(p, Action{ActionKind::Compute, 1, 0, 1, 1, -1, -1, -1, -1}) == 3.0);
    CHECK(action_cost(p, Action{ActionKind::Copy, 1, 0, -1, -1, 0, 1, 0, 1}) == 1.0);
    CHECK(action_cost(p, Action{ActionKind::Free, 1, 1, 1, -1, 0, 1, -1, -1}) == 0.0);
  });
  run("objective_value raises MissingLink only for a charged uncovered copy (copy_cost is lazy)", [] {
    Problem p = fixture("fig2");
    const double full = objective_value(save_all_assignment(p, {0, 1, 1, 1, 1, 1, 1}), p);
    Problem q = p;
    q.edges[0].override_copy_ms.erase({1, 0});  // edge 0 -> 1 has no gpu -> cpu cost now
    CHECK_THROWS_CODE(build_model(q), Errc::MissingLink);  // the model prices every copy
    CHECK(objective_value(save_all_assignment(q, {0, 1, 1, 1, 1, 1, 1}), q) == full);
    CHECK_THROWS_CODE(objective_value(save_all_assignment(q, {1, 0, 0, 0, 0, 0, 0}), q), Errc::MissingLink);
  });
  run("solve_search: F1 chain3 = 9.0, proven by the LP bound", [] {
    Problem p = fixture("chain3");
    SearchParams sp;
    sp.candidates_per_round = 1 << 14;
    sp.rounds = 2;
    sp.chain_iters = 10;
    Solution s = solve_search(p, {}, sp);
    CHECK(s.backend == "b200");
    CHECK(s.objective_ms == 9.0);
    CHECK(s.status == SolveStatus::Optimal);
    CHECK(s.assignment.objective_reported == 9.0);
    CHECK(objective_value(s.assignment, p) == 9.0);
    CHECK(check_assignment(build_model(p), s.assignment).empty());
    CHECK(s.nodes_explored > 0);
  });
  run("solve_search: F2 fig2 = 11.0 (LP bound 9.83: not proven by the LP alone)", [] {
    Problem p = fixture("fig2");
    SearchParams sp;
    sp.candidates_per_round = 1 << 15;
    sp.rounds = 2;
    sp.chain_iters = 20;
    sp.exact_polish = false;
    Solution s = solve_search(p, {}, sp);
    CHECK(s.objective_ms == 11.0);
    CHECK(s.status == SolveStatus::LimitReached);
    CHECK(objective_value(s.assignment, p) == 11.0);
    CHECK(check_assignment(build_model(p), s.assignment).empty());
  });
  run("solve_search + exact polish: fig2 proven optimal, the reference's twin (A on the gpu)", [] {
    Problem p = fixture("fig2");
    SearchParams sp;
    sp.candidates_per_round = 1 << 15;
    sp.rounds = 2;
    sp.chain_iters = 20;
    Solution s = solve_search(p, {}, sp);
    CHECK(s.objective_ms == 11.0);
    CHECK(s.status == SolveStatus::Optimal);
    CHECK(s.assignment.at(var_r(1, 1, 1)) == 1.0);  // solve_exact's tail_less twin (test_solver.cpp:108-113)
  });
  run("solve_search: F1 at 3 MiB has no valid schedule", [] {
    Problem p = with_budgets(fixture("chain3"), {3 * kMiB});
    SearchParams sp;
    sp.candidates_per_round = 1 << 12;
    sp.rounds = 1;
    sp.use_lp = false;
    Solution s = solve_search(p, {}, sp);
    CHECK(s.status == SolveStatus::LimitReached);
    CHECK(std::isnan(s.objective_ms));
    CHECK(s.assignment.values.empty());
  });
  run("batched evaluation agrees with the map API", [] {
    Problem p = fixture("fig2");
    std::vector<std::pair<BitCube, BitCube>> cands;
    std::vector<double> want;
    for (int k = 0; k < 16; ++k) {
      std::vector<int> dev(7);
      for (int i = 0; i < 7; ++i) dev[size_t(i)] = i == 0 ? 0 : (k >> (i - 1)) & 1;
      BitCube R(2, 7), S(2, 7);
      for (int i = 0; i < 7; ++i) {
        R.at(dev[size_t(i)], i, i) = 1;
        for (int t = i + 1; t < 7; ++t) S.at(dev[size_t(i)], t, i) = 1;
      }
      want.push_back(objective_value(complete_assignment(p, {}, R, S), p));
      cands.emplace_back(R, S);
    }
    BatchResult r = evaluate_candidates(p, {}, cands);
    bool same = r.objective.size() == want.size();
    for (size_t k = 0; same && k < want.size(); ++k) same = r.objective[k] == want[k];
    CHECK(same);
    CHECK(r.n_valid == 16);
  });
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: test_api <golden_dir> host|device\n");
    return 2;
  }
  g_dir = argv[1];
  host_cases();
  if (std::string(argv[2]) == "device") device_cases();
  std::printf("%d checks, %d failed\n", g_checks, g_failed);
  return g_failed ? 1 : 0;
}
