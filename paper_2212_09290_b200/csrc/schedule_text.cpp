// SPDX-License-Identifier: Apache-2.0
//
// Text forms of schedules and traces (host): format_schedule
// (proj/src/schedule.cpp:440-475), parse_schedule (:477-521) and trace_csv
// (:523-530), byte-identical to the reference.  Names come from the caller
// (the C++ drop-in passes its Problem's) or from the handle (loaded
// documents keep their device ids and operator names).  One implementation
// serves the C ABI, the C++ API and the Python mirror.
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "xe_internal.hpp"

namespace xe {
namespace {

struct Names {
  std::vector<std::string> dev, op;
};

Names names_of(const xe_problem* p, const char* const* device_ids, const char* const* op_names) {
  Names n;
  const HostProblem& h = p->h;
  for (int d = 0; d < h.D; ++d) n.dev.push_back(device_ids ? device_ids[d] : h.device_ids[static_cast<size_t>(d)]);
  for (int i = 0; i < h.T; ++i) n.op.push_back(op_names ? op_names[i] : h.op_names[static_cast<size_t>(i)]);
  return n;
}

void put(const std::string& s, char* buf, size_t* len) {
  if (buf) {
    if (*len < s.size()) fail(XE_ERR_ARG, "text buffer too small");
    std::memcpy(buf, s.data(), s.size());
  }
  *len = s.size();
}

std::string format(const Names& n, const xe_action* a, int64_t na) {
  std::string out;
  for (int64_t k = 0; k < na; ++k) {
    const xe_action& x = a[k];
    out += "t=" + std::to_string(x.timestep) + " slot=" + std::to_string(x.slot) + " ";
    switch (x.kind) {
      case 0: out += "COMPUTE d=" + n.dev[static_cast<size_t>(x.device)] + " op=" + n.op[static_cast<size_t>(x.op)]; break;
      case 1:
        out += "COPY edge=" + n.op[static_cast<size_t>(x.src)] + "->" + n.op[static_cast<size_t>(x.dst)] +
               " from=" + n.dev[static_cast<size_t>(x.from)] + " to=" + n.dev[static_cast<size_t>(x.to)];
        break;
      case 2:
        out += "FREE d=" + n.dev[static_cast<size_t>(x.device)] + " edge=" + n.op[static_cast<size_t>(x.src)] + "->" +
               n.op[static_cast<size_t>(x.dst)];
        break;
      default: out += "DROP d=" + n.dev[static_cast<size_t>(x.device)] + " op=" + n.op[static_cast<size_t>(x.op)]; break;
    }
    out += "\n";
  }
  return out;
}

// parse helpers: the reference's messages and error codes (schedule.cpp:380-438)
std::string kv(const std::string& tok, const std::string& key) {
  if (tok.size() <= key.size() + 1 || tok.compare(0, key.size(), key) != 0 || tok[key.size()] != '=')
    fail(XE_ERR_MALFORMED_DOCUMENT, "expected " + key + "=..., got '" + tok + "'");
  return tok.substr(key.size() + 1);
}

int parse_int(const std::string& text) {
  char* end = nullptr;
  const long v = std::strtol(text.c_str(), &end, 10);
  if (end != text.c_str() + text.size() || text.empty()) fail(XE_ERR_MALFORMED_DOCUMENT, "not an integer: '" + text + "'");
  return static_cast<int>(v);
}

}  // namespace
}  // namespace xe

using namespace xe;

extern "C" int xe_format_schedule_named(const xe_problem* p, const xe_action* actions, int64_t n_actions,
                                        const char* const* device_ids, const char* const* op_names, char* buf,
                                        size_t* len) {
  return guard([&] {
    if (!p || !len || (!actions && n_actions > 0)) fail(XE_ERR_ARG, "null argument");
    put(format(names_of(p, device_ids, op_names), actions, n_actions), buf, len);
  });
}

extern "C" int xe_format_schedule(const xe_problem* p, const xe_action* actions, int64_t n_actions, char* buf,
                                  size_t* len) {
  return xe_format_schedule_named(p, actions, n_actions, nullptr, nullptr, buf, len);
}

extern "C" int xe_trace_csv_named(const xe_problem* p, const int64_t* memory, const char* const* device_ids,
                                  char* buf, size_t* len) {
  return guard([&] {
    if (!p || !memory || !len) fail(XE_ERR_ARG, "null argument");
    const HostProblem& h = p->h;
    const Names n = names_of(p, device_ids, nullptr);
    std::string out = "device,timestep,slot,bytes\n";
    for (int d = 0; d < h.D; ++d)
      for (int t = 0; t < h.T; ++t)
        for (int v = 0; v < h.T; ++v)
          out += n.dev[static_cast<size_t>(d)] + "," + std::to_string(t) + "," + std::to_string(v) + "," +
                 std::to_string(memory[(static_cast<size_t>(d) * h.T + t) * h.T + v]) + "\n";
    put(out, buf, len);
  });
}

extern "C" int xe_trace_csv(const xe_problem* p, const int64_t* memory, char* buf, size_t* len) {
  return xe_trace_csv_named(p, memory, nullptr, buf, len);
}

extern "C" int xe_parse_schedule_named(const xe_problem* p, const char* text, const char* const* device_ids,
                                       const char* const* op_names, const char* problem_name, xe_action* actions,
                                       int64_t* n_actions) {
  return guard([&] {
    if (!p || !text || !n_actions) fail(XE_ERR_ARG, "null argument");
    const HostProblem& h = p->h;
    const Names n = names_of(p, device_ids, op_names);
    auto op_by_name = [&](const std::string& name) {
      for (int i = 0; i < h.T; ++i)
        if (n.op[static_cast<size_t>(i)] == name) return i;
      fail(XE_ERR_MALFORMED_DOCUMENT, "unknown operator '" + name + "'");
    };
    auto device_by_id = [&](const std::string& id) {
      for (int d = 0; d < h.D; ++d)
        if (n.dev[static_cast<size_t>(d)] == id) return d;
      fail(XE_ERR_UNKNOWN_DEVICE, "'" + id + "'");
    };
    auto parse_edge = [&](const std::string& t) -> std::pair<int, int> {
      const size_t pos = t.find("->");
      if (pos == std::string::npos) fail(XE_ERR_MALFORMED_DOCUMENT, "expected <u>-><v>, got '" + t + "'");
      const int u = op_by_name(t.substr(0, pos)), v = op_by_name(t.substr(pos + 2));
      if (u != v) {
        bool found = false;
        for (int e = 0; e < h.E; ++e) found = found || (h.src[static_cast<size_t>(e)] == u && h.dst[static_cast<size_t>(e)] == v);
        if (!found)
          fail(XE_ERR_MALFORMED_DOCUMENT, "no edge '" + t + "' in problem " + std::string(problem_name ? problem_name : ""));
      }
      return {u, v};
    };
    std::vector<xe_action> out;
    std::istringstream in(text);
    std::string line;
    while (std::getline(in, line)) {
      if (!line.empty() && line.back() == '\r') line.pop_back();
      if (line.empty()) continue;
      std::istringstream ls(line);
      std::vector<std::string> tok;
      std::string t;
      while (ls >> t) tok.push_back(t);
      if (tok.size() < 4) fail(XE_ERR_MALFORMED_DOCUMENT, "short action line: '" + line + "'");
      xe_action a{0, 0, 0, -1, -1, -1, -1, -1, -1};
      a.timestep = parse_int(kv(tok[0], "t"));
      a.slot = parse_int(kv(tok[1], "slot"));
      if (a.timestep < 0 || a.timestep >= h.T || a.slot < 0)
        fail(XE_ERR_MALFORMED_DOCUMENT, "action out of range: '" + line + "'");
      const std::string& kind = tok[2];
      if (kind == "COMPUTE" && tok.size() == 5) {
        a.kind = 0;
        a.device = device_by_id(kv(tok[3], "d"));
        a.op = op_by_name(kv(tok[4], "op"));
      } else if (kind == "COPY" && tok.size() == 6) {
        a.kind = 1;
        const auto e = parse_edge(kv(tok[3], "edge"));
        a.src = e.first;
        a.dst = e.second;
        a.from = device_by_id(kv(tok[4], "from"));
        a.to = device_by_id(kv(tok[5], "to"));
      } else if (kind == "FREE" && tok.size() == 5) {
        a.kind = 2;
        a.device = device_by_id(kv(tok[3], "d"));
        const auto e = parse_edge(kv(tok[4], "edge"));
        a.src = e.first;
        a.dst = e.second;
      } else if (kind == "DROP" && tok.size() == 5) {
        a.kind = 3;
        a.device = device_by_id(kv(tok[3], "d"));
        a.op = op_by_name(kv(tok[4], "op"));
      } else {
        fail(XE_ERR_MALFORMED_DOCUMENT, "unrecognized action line: '" + line + "'");
      }
      out.push_back(a);
    }
    if (actions) {
      if (*n_actions < static_cast<int64_t>(out.size())) fail(XE_ERR_ARG, "action buffer too small");
      std::memcpy(actions, out.data(), out.size() * sizeof(xe_action));
    }
    *n_actions = static_cast<int64_t>(out.size());
  });
}

extern "C" int xe_parse_schedule(const xe_problem* p, const char* text, xe_action* actions, int64_t* n_actions) {
  return xe_parse_schedule_named(p, text, nullptr, nullptr, nullptr, actions, n_actions);
}
