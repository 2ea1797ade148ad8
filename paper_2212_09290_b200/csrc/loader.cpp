// SPDX-License-Identifier: Apache-2.0
//
// Host loader: problem document -> resolved HostProblem.  Behaviour follows
// the reference loader (proj/src/problem.cpp):
//   direct documents          problem.cpp:140-188
//   layered training graphs   problem.cpp:190-224, make_training_graph 280-338
//   forward-DAG documents      make_training_graph generalised to a forward
//                              DAG ("forward" key)
//   structural validation     problem.cpp:254-278
//   copy_cost resolution      problem.cpp:358-380 (override > most specific link)
//   energy section            proj/src/model.cpp:314-367
// Error codes are the reference's Errc values + 1 (include/xengine_b200.h).
// Host-only: documents are kilobytes; the device never sees JSON.

#include <json.hpp>

#include <algorithm>
#include <cmath>
#include <set>

#include "xe_internal.hpp"

namespace xe {
namespace {

using nlohmann::json;
constexpr double kProhibitive = 1.0e9;  // problem.hpp:16

using Link = DocLink;
using Doc = ParsedDoc;

int64_t positive_int(const json& j, const std::string& what) {
  if (!j.is_number_integer()) fail(XE_ERR_MALFORMED_DOCUMENT, what + " must be an integer byte count");
  int64_t v = j.get<int64_t>();
  if (v <= 0) fail(XE_ERR_NON_POSITIVE_SIZE, what + " must be positive");
  return v;
}

double nonneg(const json& j, const std::string& what) {
  if (!j.is_number()) fail(XE_ERR_MALFORMED_DOCUMENT, what + " must be a number");
  double v = j.get<double>();
  if (v < 0.0) fail(XE_ERR_NEGATIVE_COST, what + " must be non-negative");
  return v;
}

int device_index(const HostProblem& p, const std::string& id) {
  for (int d = 0; d < p.D; ++d)
    if (p.device_ids[static_cast<size_t>(d)] == id) return d;
  return -1;
}

void read_devices(const json& doc, HostProblem& p, std::vector<int64_t>* ram_out) {
  if (!doc.contains("devices") || !doc["devices"].is_array() || doc["devices"].empty())
    fail(XE_ERR_MALFORMED_DOCUMENT, "document needs a non-empty devices array");
  std::set<std::string> ids;
  for (const auto& jd : doc["devices"]) {
    if (!jd.contains("id") || !jd["id"].is_string())
      fail(XE_ERR_MALFORMED_DOCUMENT, "device entry needs a string id");
    std::string id = jd["id"].get<std::string>();
    if (!ids.insert(id).second) fail(XE_ERR_MALFORMED_DOCUMENT, "duplicate device id " + id);
    int64_t budget = positive_int(jd.at("budget_bytes"), "device " + id + " budget_bytes");
    int64_t ram = -1;
    if (jd.contains("ram_bytes")) {
      ram = positive_int(jd["ram_bytes"], "device " + id + " ram_bytes");
      if (ram < budget) fail(XE_ERR_MALFORMED_DOCUMENT, "device " + id + " budget exceeds its ram");
    }
    p.device_ids.push_back(id);
    p.budget.push_back(budget);
    if (ram_out) ram_out->push_back(ram);
  }
  p.D = static_cast<int>(p.device_ids.size());
}

std::vector<double> read_costs(const json& jc, const HostProblem& p, const std::string& what) {
  if (!jc.is_object()) fail(XE_ERR_MALFORMED_DOCUMENT, what + " costs_ms must be an object");
  std::vector<double> c(static_cast<size_t>(p.D), kProhibitive);  // absent device -> sentinel
  for (auto it = jc.begin(); it != jc.end(); ++it) {
    int d = device_index(p, it.key());
    if (d < 0) fail(XE_ERR_UNKNOWN_DEVICE, what + " costs_ms names unknown device " + it.key());
    c[static_cast<size_t>(d)] = nonneg(it.value(), what + " cost for " + it.key());
  }
  return c;
}

std::pair<int, int> device_pair(const std::string& key, const HostProblem& p) {
  size_t at = key.find("->");
  if (at == std::string::npos)
    fail(XE_ERR_MALFORMED_DOCUMENT, "copy override key '" + key + "' is not <from>-><to>");
  int a = device_index(p, key.substr(0, at)), b = device_index(p, key.substr(at + 2));
  if (a < 0 || b < 0) fail(XE_ERR_UNKNOWN_DEVICE, "copy override key '" + key + "'");
  return {a, b};
}

std::vector<Link> read_links(const json& doc, const HostProblem& p) {
  std::vector<Link> out;
  if (!doc.contains("links")) return out;
  if (!doc["links"].is_array()) fail(XE_ERR_MALFORMED_DOCUMENT, "links must be an array");
  for (const auto& jl : doc["links"]) {
    auto endpoint = [&](const char* f) {
      const auto& v = jl.at(f);
      if (!v.is_string()) fail(XE_ERR_MALFORMED_DOCUMENT, "link endpoint must be a device id");
      std::string s = v.get<std::string>();
      if (s == "*") return -1;
      int d = device_index(p, s);
      if (d < 0) fail(XE_ERR_UNKNOWN_DEVICE, "link names unknown device " + s);
      return d;
    };
    Link l{};
    l.from = endpoint("from");
    l.to = endpoint("to");
    l.latency = nonneg(jl.at("latency_ms"), "link latency_ms");
    const auto& r = jl.at("bytes_per_ms");
    if (!r.is_number() || r.get<double>() <= 0.0)
      fail(XE_ERR_NON_POSITIVE_SIZE, "link bytes_per_ms must be positive");
    l.rate = r.get<double>();
    out.push_back(l);
  }
  return out;
}

void add_op(HostProblem& p, const std::string& name, int64_t bytes, const std::vector<double>& c,
            std::vector<std::vector<double>>& costs) {
  p.op_names.push_back(name);
  p.mass.push_back(bytes);
  costs.push_back(c);
}

void finish_costs(HostProblem& p, const std::vector<std::vector<double>>& costs) {
  p.T = static_cast<int>(costs.size());
  p.cost.assign(static_cast<size_t>(p.D) * p.T, 0.0);
  for (int i = 0; i < p.T; ++i) {
    if (static_cast<int>(costs[static_cast<size_t>(i)].size()) != p.D)
      fail(XE_ERR_DIMENSION_MISMATCH, "operator " + p.op_names[static_cast<size_t>(i)] + " cost vector size");
    for (int d = 0; d < p.D; ++d)
      p.cost[static_cast<size_t>(d) * p.T + i] = costs[static_cast<size_t>(i)][static_cast<size_t>(d)];
  }
}

Doc read_direct(const json& doc) {
  Doc out;
  HostProblem& p = out.p;
  read_devices(doc, p, &out.ram);
  if (!doc.contains("operators") || !doc["operators"].is_array() || doc["operators"].empty())
    fail(XE_ERR_EMPTY_NETWORK, "document has no operators");
  std::vector<std::vector<double>> costs;
  for (const auto& jo : doc["operators"]) {
    if (!jo.contains("name") || !jo["name"].is_string())
      fail(XE_ERR_MALFORMED_DOCUMENT, "operator entry needs a string name");
    std::string name = jo["name"].get<std::string>();
    int64_t bytes = positive_int(jo.at("output_bytes"), "operator " + name + " output_bytes");
    auto c = read_costs(jo.at("costs_ms"), p, "operator " + name);
    int pin = -1;
    if (jo.contains("pinned")) {
      pin = device_index(p, jo["pinned"].get<std::string>());
      if (pin < 0) fail(XE_ERR_UNKNOWN_DEVICE, "operator " + name + " pinned to unknown device");
    }
    out.pinned.push_back(pin);
    add_op(p, name, bytes, c, costs);
  }
  finish_costs(p, costs);
  if (doc.contains("edges")) {
    if (!doc["edges"].is_array()) fail(XE_ERR_MALFORMED_DOCUMENT, "edges must be an array");
    for (const auto& je : doc["edges"]) {
      std::map<std::pair<int, int>, double> ov;
      int s = 0, t = 0;
      if (je.is_array()) {
        if (je.size() != 2 || !je[0].is_number_integer() || !je[1].is_number_integer())
          fail(XE_ERR_MALFORMED_DOCUMENT, "edge array entry must be [src, dst]");
        s = je[0].get<int>();
        t = je[1].get<int>();
      } else if (je.is_object()) {
        s = je.at("src").get<int>();
        t = je.at("dst").get<int>();
        if (je.contains("copy_ms"))
          for (auto it = je["copy_ms"].begin(); it != je["copy_ms"].end(); ++it)
            ov[device_pair(it.key(), p)] = nonneg(it.value(), "edge copy_ms");
      } else {
        fail(XE_ERR_MALFORMED_DOCUMENT, "edge entry must be an array or object");
      }
      p.src.push_back(s);
      p.dst.push_back(t);
      out.overrides.push_back(std::move(ov));
    }
  }
  p.E = static_cast<int>(p.src.size());
  validate(p);
  out.links = read_links(doc, p);  // links are read after validation (problem.cpp:238-239)
  return out;
}

// The training-graph documents: "layers" (the reference's chain form,
// problem.cpp:190-224) and "forward" (a forward DAG: each op lists its
// inputs) expand through expand_training_graph.
Doc read_training(const json& doc, bool chain) {
  Doc out;
  HostProblem& p = out.p;
  read_devices(doc, p, &out.ram);
  out.links = read_links(doc, p);
  if (!doc.contains("input") || !doc["input"].is_object())
    fail(XE_ERR_MALFORMED_DOCUMENT, "layer document needs an input object");
  int64_t in_bytes = positive_int(doc["input"].at("output_bytes"), "input output_bytes");
  int home = device_index(p, doc["input"].at("home").get<std::string>());
  if (home < 0) fail(XE_ERR_UNKNOWN_DEVICE, "input home device");
  std::vector<ForwardOp> fwd;
  const json& list = chain ? doc["layers"] : doc["forward"];
  if (!list.is_array()) fail(XE_ERR_MALFORMED_DOCUMENT, chain ? "layers must be an array" : "forward must be an array");
  for (const auto& jl : list) {
    ForwardOp l;
    l.name = jl.at("name").get<std::string>();
    l.bytes = positive_int(jl.at("output_bytes"), "layer " + l.name + " output_bytes");
    l.costs = read_costs(jl.at("costs_ms"), p, "layer " + l.name);
    l.bwd_bytes = positive_int(jl.at("backward_output_bytes"), "layer " + l.name + " backward_output_bytes");
    l.bwd_costs = read_costs(jl.at("backward_costs_ms"), p, "layer " + l.name + " backward");
    const int k = static_cast<int>(fwd.size()) + 1;
    if (chain) {
      l.inputs = {k - 1};
    } else {
      if (!jl.contains("inputs") || !jl["inputs"].is_array() || jl["inputs"].empty())
        fail(XE_ERR_MALFORMED_DOCUMENT, "forward op " + l.name + " needs a non-empty inputs array");
      for (const auto& ji : jl["inputs"]) {
        if (!ji.is_number_integer()) fail(XE_ERR_MALFORMED_DOCUMENT, "forward op " + l.name + " inputs are op indices");
        const int u = ji.get<int>();
        if (u < 0 || u >= k)
          fail(XE_ERR_NON_TOPOLOGICAL_EDGE, "forward op " + l.name + " input " + std::to_string(u) + " is not earlier");
        l.inputs.push_back(u);
      }
    }
    fwd.push_back(std::move(l));
  }
  if (fwd.empty()) fail(XE_ERR_EMPTY_NETWORK, "training graph needs at least one layer");
  std::vector<std::vector<double>> costs;
  std::vector<int64_t> bytes;
  expand_training_graph(p.D, in_bytes, home, fwd, p.op_names, bytes, costs, p.src, p.dst);
  p.mass = bytes;
  finish_costs(p, costs);
  out.pinned.assign(static_cast<size_t>(p.T), -1);
  out.pinned[0] = home;
  p.E = static_cast<int>(p.src.size());
  validate(p);
  std::map<std::pair<int, int>, double> ov;
  if (doc.contains("edge_copy_ms"))
    for (auto it = doc["edge_copy_ms"].begin(); it != doc["edge_copy_ms"].end(); ++it)
      ov[device_pair(it.key(), p)] = nonneg(it.value(), "edge_copy_ms");
  out.overrides.assign(static_cast<size_t>(p.E), ov);
  return out;
}

// copy_cost for every (edge, ds, dc): 0 on the diagonal, the edge override
// when present, else latency + bytes/rate of the most specific covering link
// (first wins among equals).
void resolve_copies(Doc& doc) {
  HostProblem& p = doc.p;
  p.w.assign(static_cast<size_t>(p.E) * p.D * p.D, 0.0);
  p.w_missing.assign(static_cast<size_t>(p.E) * p.D * p.D, 0);
  for (int e = 0; e < p.E; ++e)
    for (int a = 0; a < p.D; ++a)
      for (int b = 0; b < p.D; ++b) {
        if (a == b) continue;
        const auto& ov = doc.overrides[static_cast<size_t>(e)];
        double v;
        if (auto it = ov.find({a, b}); it != ov.end()) {
          v = it->second;
        } else {
          const Link* best = nullptr;
          int best_rank = -1;
          for (const Link& l : doc.links) {
            if ((l.from != -1 && l.from != a) || (l.to != -1 && l.to != b)) continue;
            int rank = (l.from == a) + (l.to == b);
            if (rank > best_rank) {
              best = &l;
              best_rank = rank;
            }
          }
          if (!best) {
            // copy_cost raises lazily in the reference (problem.cpp:374-376):
            // remember the first uncovered pair and raise when a model or an
            // evaluation needs the table.
            if (p.missing_link.empty())
              p.missing_link = "no link covers " + p.device_ids[static_cast<size_t>(a)] + "->" +
                               p.device_ids[static_cast<size_t>(b)];
            p.w_missing[(static_cast<size_t>(e) * p.D + a) * p.D + b] = 1;
            continue;
          }
          v = best->latency + static_cast<double>(p.mass[static_cast<size_t>(p.src[static_cast<size_t>(e)])]) / best->rate;
        }
        p.w[(static_cast<size_t>(e) * p.D + a) * p.D + b] = v;
      }
}

void read_energy(const json& doc, HostProblem& p) {
  p.q.assign(static_cast<size_t>(p.D) * p.T, 0.0);
  p.has_lim.assign(static_cast<size_t>(p.D), 0);
  p.lim.assign(static_cast<size_t>(p.D), 0.0);
  if (!doc.contains("energy")) return;
  const auto& e = doc["energy"];
  if (!e.is_object()) fail(XE_ERR_MALFORMED_DOCUMENT, "energy must be an object");
  p.has_energy = true;
  p.alpha = e.value("alpha", 0.0);
  if (!(p.alpha >= 0.0)) fail(XE_ERR_NEGATIVE_COST, "alpha");
  p.board = e.value("board_joules", 0.0);
  if (!(p.board >= 0.0)) fail(XE_ERR_NEGATIVE_COST, "board_joules");
  if (e.contains("total_limit")) {
    p.has_total = true;
    p.total_limit = e["total_limit"].get<double>();
    if (!(p.total_limit >= 0.0)) fail(XE_ERR_NEGATIVE_COST, "total_limit");
  }
  if (!e.contains("q_joules") || !e["q_joules"].is_object())
    fail(XE_ERR_INCOMPLETE_ENERGY_TABLE, "q_joules missing");
  const auto& q = e["q_joules"];
  for (auto it = q.begin(); it != q.end(); ++it)
    if (device_index(p, it.key()) < 0) fail(XE_ERR_UNKNOWN_DEVICE, it.key());
  for (int d = 0; d < p.D; ++d) {
    const std::string& id = p.device_ids[static_cast<size_t>(d)];
    if (!q.contains(id)) fail(XE_ERR_INCOMPLETE_ENERGY_TABLE, "q_joules missing device " + id);
    const auto& row = q[id];
    if (!row.is_array() || static_cast<int>(row.size()) != p.T)
      fail(XE_ERR_INCOMPLETE_ENERGY_TABLE, "q_joules row for " + id);
    for (int i = 0; i < p.T; ++i) {
      double x = row[static_cast<size_t>(i)].get<double>();
      if (!(x >= 0.0)) fail(XE_ERR_NEGATIVE_COST, "q_joules");
      p.q[static_cast<size_t>(d) * p.T + i] = x;
    }
  }
  if (e.contains("device_limit")) {
    const auto& dl = e["device_limit"];
    if (!dl.is_object()) fail(XE_ERR_MALFORMED_DOCUMENT, "device_limit must be an object");
    for (auto it = dl.begin(); it != dl.end(); ++it) {
      int d = device_index(p, it.key());
      if (d < 0) fail(XE_ERR_UNKNOWN_DEVICE, it.key());
      double lim = it.value().get<double>();
      if (!(lim >= 0.0)) fail(XE_ERR_NEGATIVE_COST, "device_limit");
      p.has_lim[static_cast<size_t>(d)] = 1;
      p.lim[static_cast<size_t>(d)] = lim;
    }
  }
}

}  // namespace

void validate(const HostProblem& p) {
  if (p.T == 0) fail(XE_ERR_EMPTY_NETWORK, "problem has no operators");
  if (p.D == 0) fail(XE_ERR_MALFORMED_DOCUMENT, "problem has no devices");
  std::set<std::pair<int, int>> seen;
  std::vector<int> indeg(static_cast<size_t>(p.T), 0);
  for (int e = 0; e < p.E; ++e) {
    int s = p.src[static_cast<size_t>(e)], t = p.dst[static_cast<size_t>(e)];
    if (s < 0 || t < 0 || s >= p.T || t >= p.T) fail(XE_ERR_MALFORMED_DOCUMENT, "edge endpoint out of range");
    if (s >= t)
      fail(XE_ERR_NON_TOPOLOGICAL_EDGE, "edge " + std::to_string(s) + "->" + std::to_string(t) + " violates index order");
    if (!seen.insert({s, t}).second)
      fail(XE_ERR_MALFORMED_DOCUMENT, "duplicate edge " + std::to_string(s) + "->" + std::to_string(t));
    indeg[static_cast<size_t>(t)]++;
  }
  for (int v = 1; v < p.T; ++v)
    if (indeg[static_cast<size_t>(v)] == 0)
      fail(XE_ERR_MALFORMED_DOCUMENT, "operator " + std::to_string(v) + " has no incoming edge; only operator 0 is a source");
}

void expand_training_graph(int D, int64_t input_bytes, int input_home, const std::vector<ForwardOp>& fwd,
                           std::vector<std::string>& names, std::vector<int64_t>& bytes,
                           std::vector<std::vector<double>>& costs, std::vector<int32_t>& src,
                           std::vector<int32_t>& dst) {
  if (fwd.empty()) fail(XE_ERR_EMPTY_NETWORK, "training graph needs at least one layer");
  if (input_bytes <= 0) fail(XE_ERR_NON_POSITIVE_SIZE, "input_bytes must be positive");
  if (input_home < 0 || input_home >= D) fail(XE_ERR_UNKNOWN_DEVICE, "input home index");
  const int F = static_cast<int>(fwd.size());
  auto checked = [&](const std::vector<double>& c, const std::string& ctx) {
    if (static_cast<int>(c.size()) != D) fail(XE_ERR_DIMENSION_MISMATCH, ctx + " cost vector size");
    for (double v : c)
      if (v < 0.0) fail(XE_ERR_NEGATIVE_COST, ctx + " cost");
    return c;
  };
  names.assign(1, "input");
  bytes.assign(1, input_bytes);
  costs.assign(1, std::vector<double>(static_cast<size_t>(D), kProhibitive));
  costs[0][static_cast<size_t>(input_home)] = 0.0;  // a reload, not a computation
  for (const auto& l : fwd) {
    if (l.bytes <= 0) fail(XE_ERR_NON_POSITIVE_SIZE, "layer " + l.name + " output_bytes");
    names.push_back(l.name);
    bytes.push_back(l.bytes);
    costs.push_back(checked(l.costs, "layer " + l.name));
  }
  for (int f = F; f >= 1; --f) {
    const auto& l = fwd[static_cast<size_t>(f - 1)];
    if (l.bwd_bytes <= 0) fail(XE_ERR_NON_POSITIVE_SIZE, "layer " + l.name + " backward_output_bytes");
    names.push_back(l.name + "'");
    bytes.push_back(l.bwd_bytes);
    costs.push_back(checked(l.bwd_costs, "layer " + l.name + " backward"));
  }
  std::vector<std::vector<int>> cons(static_cast<size_t>(F) + 1);
  src.clear();
  dst.clear();
  for (int f = 1; f <= F; ++f)  // forward edges
    for (int u : fwd[static_cast<size_t>(f - 1)].inputs) {
      src.push_back(u);
      dst.push_back(f);
      cons[static_cast<size_t>(u)].push_back(f);
    }
  for (auto& c : cons) std::sort(c.begin(), c.end());
  for (int j = F + 1; j <= 2 * F; ++j) {
    const int f = 2 * F + 1 - j;  // the forward op whose backward sits at j
    if (cons[static_cast<size_t>(f)].empty()) {
      src.push_back(F);  // upstream gradient of the loss
      dst.push_back(j);
    } else {
      for (int c : cons[static_cast<size_t>(f)]) {
        src.push_back(2 * F + 1 - c);  // upstream gradient from the consumer's backward
        dst.push_back(j);
      }
    }
    for (int u : fwd[static_cast<size_t>(f - 1)].inputs) {  // saved forward tensors
      src.push_back(u);
      dst.push_back(j);
    }
  }
}

ParsedDoc parse_problem_document(const std::string& text) {
  json doc;
  try {
    doc = json::parse(text);
  } catch (const json::exception& ex) {
    fail(XE_ERR_MALFORMED_DOCUMENT, ex.what());
  }
  if (!doc.is_object()) fail(XE_ERR_MALFORMED_DOCUMENT, "top level must be an object");
  try {
    Doc d = doc.contains("layers")    ? read_training(doc, true)
            : doc.contains("forward") ? read_training(doc, false)
                                      : read_direct(doc);
    d.name = doc.value("name", std::string("unnamed"));
    return d;
  } catch (const json::exception& ex) {
    fail(XE_ERR_MALFORMED_DOCUMENT, ex.what());
  }
}

HostProblem load_problem_json(const std::string& text) {
  Doc d = parse_problem_document(text);
  resolve_copies(d);
  try {
    read_energy(json::parse(text), d.p);
  } catch (const json::exception& ex) {
    fail(XE_ERR_MALFORMED_DOCUMENT, ex.what());
  }
  return d.p;
}

}  // namespace xe
