// SPDX-License-Identifier: Apache-2.0
//
// Bit-exact free-format MPS (write_mps, proj/src/mps_io.cpp:109-199) from
// the GPU-assembled model.  The device builds the CSR and its stable
// column-major copy; the host streams the text: ROWS in emission order,
// COLUMNS in VarRef order with the OBJ entry first and then the column's rows
// in emission order, one INTORG/INTEND block around the binaries, RHS for
// non-zero right-hand sides, BOUNDS (FX/BV/UP), QUADOBJ when quadratic.
// Numbers use format_number's rule (mps_io.cpp:14-27): "%.0f" for integral
// |v| < 1e15, else the shortest "%.{1..17}g" that round-trips; each distinct
// value is formatted once.

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "csr.hpp"

namespace xe {

// format_number (mps_io.cpp:14-27): the library's one copy (the C++ API's
// xengine::format_number forwards here)
std::string format_number(double v) {
  char buf[64];
  if (v == 0.0) return "0";
  if (std::isfinite(v) && v == std::floor(v) && std::fabs(v) < 1e15) {
    std::snprintf(buf, sizeof buf, "%.0f", v);
    return buf;
  }
  for (int prec = 1; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof buf, "%.*g", prec, v);
    if (std::strtod(buf, nullptr) == v) break;
  }
  return buf;
}

namespace {

const char* const kTag[14] = {"EQ7",     "EQ8",     "EQ9",     "EQ10",   "EQ11",       "EQ12",        "EQ13",
                              "EQ14",    "EQ16_LO", "EQ16_HI", "Z_LINK", "P_LINK", "ENERGY_DEV", "ENERGY_TOTAL"};
constexpr uint8_t kPLink = 11;

struct Out {
  std::string s;
  void put(const char* p, size_t n) { s.append(p, n); }
  void put(const char* p) { s.append(p); }
  void put(const std::string& x) { s.append(x); }
  void putc(char c) { s.push_back(c); }
  void num(int64_t v) {
    char b[24];
    int n = 0;
    if (v == 0) {
      s.push_back('0');
      return;
    }
    bool neg = v < 0;
    uint64_t u = neg ? static_cast<uint64_t>(-v) : static_cast<uint64_t>(v);
    while (u) {
      b[n++] = static_cast<char>('0' + u % 10);
      u /= 10;
    }
    if (neg) s.push_back('-');
    while (n) s.push_back(b[--n]);
  }
};

struct NumCache {
  std::unordered_map<uint64_t, std::string> m;
  const std::string& get(double v) {
    uint64_t k;
    std::memcpy(&k, &v, 8);
    auto it = m.find(k);
    if (it != m.end()) return it->second;
    return m.emplace(k, format_number(v)).first->second;
  }
};

// VarRef name of a closed-form column index (var_name, mps_io.cpp:29-43)
void col_name(Out& o, const CsrHost& h, int64_t j) {
  const int64_t T = h.T, D = h.D, E = h.E, FE = h.E + h.T;
  const int64_t DT2 = D * T * T, DTF = D * T * FE;
  auto tri = [&](char f, int64_t a, int64_t b, int64_t c) {
    o.putc(f);
    o.putc('_');
    o.num(a);
    o.putc('_');
    o.num(b);
    o.putc('_');
    o.num(c);
  };
  if (j < 3 * DT2) {
    const char f = "RSZ"[j / DT2];
    const int64_t r = j % DT2;
    tri(f, r / (T * T), r / T % T, r % T);
    return;
  }
  j -= 3 * DT2;
  if (j < DTF) {
    tri('F', j / (T * FE), j / FE % T, j % FE);
    return;
  }
  j -= DTF;
  if (j < DT2) {
    tri('U', j / (T * T), j / T % T, j % T);
    return;
  }
  j -= DT2;
  const int64_t dm1 = D - 1;
  const int64_t t = j / (E * D * dm1);
  int64_t rem = j % (E * D * dm1);
  const int64_t e = rem / (D * dm1);
  rem %= D * dm1;
  const int64_t ds = rem / dm1;
  int64_t dc = rem % dm1;
  if (dc >= ds) ++dc;
  tri('P', t, e, ds);
  o.putc('_');
  o.num(dc);
}

void row_name(Out& o, const CsrHost& h, int64_t r) {
  o.put(kTag[h.tag[static_cast<size_t>(r)]]);
  o.putc('_');
  o.num(h.ordinal[static_cast<size_t>(r)]);
}

}  // namespace

std::string mps_text(const CsrHost& h) {
  Out o;
  o.s.reserve(static_cast<size_t>(h.nnz) * 40 + static_cast<size_t>(h.n_rows) * 20 +
              static_cast<size_t>(h.n_cols) * 30 + 64);
  NumCache nc;
  const bool quad = h.quad;
  const int64_t T = h.T, D = h.D, FE = h.E + h.T;
  const int64_t firstU = 3 * D * T * T + D * T * FE, firstP = firstU + D * T * T;
  const int64_t ncol_out = quad ? firstP : h.n_cols;
  o.put("NAME XENGINE\nROWS\n N OBJ\n");
  for (int64_t r = 0; r < h.n_rows; ++r) {
    if (quad && h.tag[static_cast<size_t>(r)] == kPLink) continue;
    o.putc(' ');
    o.putc(static_cast<char>(h.sense[static_cast<size_t>(r)]));
    o.putc(' ');
    row_name(o, h, r);
    o.putc('\n');
  }
  o.put("COLUMNS\n");
  bool in_int = false;
  Out name;
  for (int64_t j = 0; j < ncol_out; ++j) {
    const bool bin = j < firstU;
    if (bin && !in_int) {
      o.put("    MARK  'MARKER'  'INTORG'\n");
      in_int = true;
    }
    if (!bin && in_int) {
      o.put("    MARK  'MARKER'  'INTEND'\n");
      in_int = false;
    }
    name.s.clear();
    col_name(name, h, j);
    if (h.present[static_cast<size_t>(j)]) {
      o.put("    ");
      o.put(name.s);
      o.put("  OBJ  ");
      o.put(nc.get(h.obj[static_cast<size_t>(j)]));
      o.putc('\n');
    }
    for (int64_t q = h.col_ptr[static_cast<size_t>(j)]; q < h.col_ptr[static_cast<size_t>(j) + 1]; ++q) {
      const int64_t r = h.crow[static_cast<size_t>(q)];
      if (quad && h.tag[static_cast<size_t>(r)] == kPLink) continue;
      o.put("    ");
      o.put(name.s);
      o.put("  ");
      row_name(o, h, r);
      o.put("  ");
      o.put(nc.get(h.cval[static_cast<size_t>(q)]));
      o.putc('\n');
    }
  }
  if (in_int) o.put("    MARK  'MARKER'  'INTEND'\n");
  o.put("RHS\n");
  for (int64_t r = 0; r < h.n_rows; ++r) {
    if (quad && h.tag[static_cast<size_t>(r)] == kPLink) continue;
    const double v = h.rhs[static_cast<size_t>(r)];
    if (v == 0.0) continue;
    o.put("    RHS  ");
    row_name(o, h, r);
    o.put("  ");
    o.put(nc.get(v));
    o.putc('\n');
  }
  o.put("BOUNDS\n");
  for (int64_t j = 0; j < ncol_out; ++j) {
    name.s.clear();
    col_name(name, h, j);
    const uint8_t k = h.kind[static_cast<size_t>(j)];
    if (k == 0) {
      o.put(" FX BND ");
      o.put(name.s);
      o.put(" 0\n");
    } else if (k == 1) {
      o.put(" BV BND ");
      o.put(name.s);
      o.putc('\n');
    } else {
      o.put(" UP BND ");
      o.put(name.s);
      o.putc(' ');
      o.put(k == 2 ? nc.get(h.ub[static_cast<size_t>(j)]) : std::string("1"));
      o.putc('\n');
    }
  }
  if (quad) {
    bool any = false;
    for (int64_t t = 0; t < T; ++t)
      for (int64_t e = 0; e < h.E; ++e)
        for (int64_t ds = 0; ds < D; ++ds)
          for (int64_t dc = 0; dc < D; ++dc) {
            if (ds == dc) continue;
            const double w = h.w[static_cast<size_t>((e * D + ds) * D + dc)];
            if (w == 0.0) continue;
            if (!any) o.put("QUADOBJ\n");
            any = true;
            o.put("    ");
            col_name(o, h, (dc * T + t) * T + h.dst[static_cast<size_t>(e)]);
            o.put("  ");
            col_name(o, h, 2 * D * T * T + (ds * T + t) * T + h.src[static_cast<size_t>(e)]);
            o.put("  ");
            o.put(nc.get(w));
            o.putc('\n');
          }
  }
  o.put("ENDATA\n");
  return std::move(o.s);
}

}  // namespace xe
