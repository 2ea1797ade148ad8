/* SPDX-License-Identifier: Apache-2.0
 *
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the reference hot path in
 * plain C (see xe_oracle.h).  Each function restates the reference loop it
 * names, in the same order, so floating-point sums round identically.
 * Compiled with -ffp-contract=off (no FMA contraction), like the reference.
 */
#include "xe_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ConstraintTag order, model.hpp:36-39 */
enum { T_EQ7, T_EQ8, T_EQ9, T_EQ10, T_EQ11, T_EQ12, T_EQ13, T_EQ14, T_EQ16_LO, T_EQ16_HI,
       T_Z_LINK, T_P_LINK, T_ENERGY_DEV, T_ENERGY_TOTAL, T_NTAGS };
static const char* const kTagName[T_NTAGS] = {
    "EQ7", "EQ8", "EQ9", "EQ10", "EQ11", "EQ12", "EQ13", "EQ14", "EQ16_LO", "EQ16_HI",
    "Z_LINK", "P_LINK", "ENERGY_DEV", "ENERGY_TOTAL"};
static const uint32_t kTagFlag[T_NTAGS] = {
    XE_F_OTHER, XE_F_EQ8, XE_F_EQ9, XE_F_OTHER, XE_F_EQ11, XE_F_EQ12, XE_F_EQ13, XE_F_EQ14,
    XE_F_EQ16_LO, XE_F_EQ16_HI, XE_F_Z_LINK, XE_F_P_LINK, XE_F_ENERGY_DEV, XE_F_ENERGY_TOTAL};

/* ---- variable index space (model.hpp:14-31, VarRef <=> order) ---------- */
typedef struct {
  int64_t D, T, E, FE;
} dims_t;
static dims_t dims(const xe_problem_desc* p) {
  dims_t s = {p->D, p->T, p->E, (int64_t)p->E + p->T};
  return s;
}
static int64_t iR(dims_t s, int64_t d, int64_t t, int64_t i) { return (d * s.T + t) * s.T + i; }
static int64_t iS(dims_t s, int64_t d, int64_t t, int64_t i) { return s.D * s.T * s.T + iR(s, d, t, i); }
static int64_t iZ(dims_t s, int64_t d, int64_t t, int64_t i) { return 2 * s.D * s.T * s.T + iR(s, d, t, i); }
static int64_t iF(dims_t s, int64_t d, int64_t t, int64_t eo) { return 3 * s.D * s.T * s.T + (d * s.T + t) * s.FE + eo; }
static int64_t iU(dims_t s, int64_t d, int64_t t, int64_t i) {
  return 3 * s.D * s.T * s.T + s.D * s.T * s.FE + iR(s, d, t, i);
}
static int64_t iP(dims_t s, int64_t t, int64_t e, int64_t ds, int64_t dc) {
  return 4 * s.D * s.T * s.T + s.D * s.T * s.FE + ((t * s.E + e) * s.D + ds) * (s.D - 1) + (dc - (dc > ds ? 1 : 0));
}
static int64_t ncols(dims_t s) { return 4 * s.D * s.T * s.T + s.D * s.T * s.FE + s.T * s.E * s.D * (s.D - 1); }

/* ---- growable row builder ---------------------------------------------- */
typedef struct {
  xo_model* m;
  int64_t cap_rows, cap_nnz;
  int32_t ord[T_NTAGS];
} builder_t;

static void grow(void** p, int64_t n, size_t elem) {
  *p = realloc(*p, (size_t)n * elem);
  if (!*p) abort();
}

static void begin_row(builder_t* b, int tag, char sense, double rhs) {
  xo_model* m = b->m;
  if (m->n_rows + 2 > b->cap_rows) {
    b->cap_rows = b->cap_rows * 2 + 1024;
    grow((void**)&m->row_ptr, b->cap_rows + 1, sizeof(int64_t));
    grow((void**)&m->rhs, b->cap_rows, sizeof(double));
    grow((void**)&m->sense, b->cap_rows, 1);
    grow((void**)&m->tag, b->cap_rows, 1);
    grow((void**)&m->ordinal, b->cap_rows, sizeof(int32_t));
  }
  int64_t r = m->n_rows++;
  m->row_ptr[r] = m->nnz;
  m->row_ptr[r + 1] = m->nnz;
  m->rhs[r] = rhs;
  m->sense[r] = sense;
  m->tag[r] = (uint8_t)tag;
  m->ordinal[r] = b->ord[tag]++; /* add_row, model.cpp:73-82 */
}

static void term(builder_t* b, int64_t col, double v) {
  xo_model* m = b->m;
  if (m->nnz + 1 > b->cap_nnz) {
    b->cap_nnz = b->cap_nnz * 2 + 4096;
    grow((void**)&m->col, b->cap_nnz, sizeof(int32_t));
    grow((void**)&m->val, b->cap_nnz, sizeof(double));
  }
  m->col[m->nnz] = (int32_t)col;
  m->val[m->nnz] = v;
  m->nnz++;
  m->row_ptr[m->n_rows] = m->nnz;
}

/* build_model (model.cpp:86-256) + add_energy_extension (model.cpp:258-312) */
int xo_build_model(const xe_problem_desc* p, int strict, int energy, xo_model* m) {
  memset(m, 0, sizeof *m);
  const dims_t s = dims(p);
  const int D = p->D, T = p->T, E = p->E;
  builder_t b;
  memset(&b, 0, sizeof b);
  b.m = m;
  m->n_cols = ncols(s);
  m->obj = calloc((size_t)m->n_cols, sizeof(double));
  m->obj_present = calloc((size_t)m->n_cols, 1);
  m->fixed = calloc((size_t)m->n_cols, 1);
  grow((void**)&m->row_ptr, 1, sizeof(int64_t));
  m->row_ptr[0] = 0;
#define MASS(i) ((double)p->output_bytes[(i)])
#define COST(d, i) (p->cost_ms[(size_t)(d) * T + (i)])
#define W(e, a, c) (p->copy_ms[((size_t)(e) * D + (a)) * D + (c)])

  /* objective (model.cpp:107-124) */
  for (int d = 0; d < D; ++d)
    for (int t = 0; t < T; ++t)
      for (int i = 0; i < T; ++i) {
        double c = COST(d, i);
        if (c != 0.0) {
          m->obj[iR(s, d, t, i)] = c;
          m->obj_present[iR(s, d, t, i)] = 1;
        }
      }
  for (int t = 0; t < T; ++t)
    for (int e = 0; e < E; ++e)
      for (int ds = 0; ds < D; ++ds)
        for (int dc = 0; dc < D; ++dc) {
          if (ds == dc) continue;
          double w = W(e, ds, dc);
          if (w == 0.0) continue;
          m->obj[iP(s, t, e, ds, dc)] = w;
          m->obj_present[iP(s, t, e, ds, dc)] = 1;
        }
  /* fixed zeros (model.cpp:127-132) */
  for (int d = 0; d < D; ++d)
    for (int t = 0; t < T; ++t) {
      for (int i = t + 1; i < T; ++i) m->fixed[iR(s, d, t, i)] = 1;
      for (int i = t; i < T; ++i) m->fixed[iS(s, d, t, i)] = 1;
    }

  /* EQ8 / EQ9 (model.cpp:138-152) */
  for (int t = 0; t < T; ++t) {
    begin_row(&b, T_EQ8, 'G', 1.0);
    for (int d = 0; d < D; ++d) term(&b, iR(s, d, t, t), 1.0);
    begin_row(&b, T_EQ8, 'L', 1.0);
    for (int d = 0; d < D; ++d) term(&b, iR(s, d, t, t), 1.0);
  }
  begin_row(&b, T_EQ9, 'E', (double)T);
  for (int t = 0; t < T; ++t)
    for (int d = 0; d < D; ++d) term(&b, iR(s, d, t, t), 1.0);

  /* EQ11 (model.cpp:155-160) */
  for (int d = 0; d < D; ++d)
    for (int t = 0; t + 1 < T; ++t)
      for (int i = 0; i < T; ++i) {
        begin_row(&b, T_EQ11, 'L', 0.0);
        term(&b, iS(s, d, t + 1, i), 1.0);
        term(&b, iS(s, d, t, i), -1.0);
        term(&b, iR(s, d, t, i), -1.0);
      }
  /* EQ12 (model.cpp:163-173) */
  for (int d = 0; d < D; ++d)
    for (int t = 0; t < T; ++t)
      for (int e = 0; e < E; ++e) {
        begin_row(&b, T_EQ12, 'L', 0.0);
        term(&b, iR(s, d, t, p->edge_dst[e]), 1.0);
        for (int ds = 0; ds < D; ++ds) {
          term(&b, iR(s, ds, t, p->edge_src[e]), -1.0);
          term(&b, iS(s, ds, t, p->edge_src[e]), -1.0);
        }
      }
  /* EQ13 (model.cpp:176-182) */
  for (int d = 0; d < D; ++d)
    for (int t = 0; t < T; ++t) {
      begin_row(&b, T_EQ13, 'E', 0.0);
      term(&b, iU(s, d, t, 0), 1.0);
      for (int i = 0; i < T; ++i) term(&b, iS(s, d, t, i), -MASS(i));
      term(&b, iR(s, d, t, 0), -MASS(0));
    }
  /* EQ14 (model.cpp:185-195); parents in edge order, edge_ordinal linear scan */
  for (int d = 0; d < D; ++d)
    for (int t = 0; t < T; ++t)
      for (int v = 0; v + 1 < T; ++v) {
        begin_row(&b, T_EQ14, 'E', 0.0);
        term(&b, iU(s, d, t, v + 1), 1.0);
        term(&b, iU(s, d, t, v), -1.0);
        for (int e = 0; e < E; ++e) {
          if (p->edge_dst[e] != v) continue;
          int u = p->edge_src[e];
          int eo = -1;
          for (int k = 0; k < E; ++k)
            if (p->edge_src[k] == u && p->edge_dst[k] == v) {
              eo = k;
              break;
            }
          term(&b, iF(s, d, t, eo), MASS(u));
        }
        term(&b, iF(s, d, t, E + v), MASS(v));
        term(&b, iR(s, d, t, v + 1), -MASS(v + 1));
      }
  /* EQ16 (model.cpp:200-224) */
  for (int d = 0; d < D; ++d)
    for (int t = 0; t < T; ++t)
      for (int eo = 0; eo < E + T; ++eo) {
        int u = eo < E ? p->edge_src[eo] : eo - E;
        int v = eo < E ? p->edge_dst[eo] : eo - E;
        int nlater = 0;
        for (int e = 0; e < E; ++e)
          if (p->edge_src[e] == u && p->edge_dst[e] > v) ++nlater;
        double h_max = 2.0 + (double)nlater * (strict ? (double)D : 1.0);
        for (int hi = 0; hi < 2; ++hi) {
          if (!hi)
            begin_row(&b, T_EQ16_LO, 'G', -1.0);
          else
            begin_row(&b, T_EQ16_HI, 'L', h_max - 2.0);
          term(&b, iR(s, d, t, v), -1.0);
          term(&b, iZ(s, d, t, u), -1.0);
          if (t + 1 < T) term(&b, iS(s, d, t + 1, u), 1.0);
          for (int e = 0; e < E; ++e) {
            if (!(p->edge_src[e] == u && p->edge_dst[e] > v)) continue;
            int w = p->edge_dst[e];
            if (strict)
              for (int dd = 0; dd < D; ++dd) term(&b, iR(s, dd, t, w), 1.0);
            else
              term(&b, iR(s, d, t, w), 1.0);
          }
          term(&b, iF(s, d, t, eo), hi ? h_max : 1.0);
        }
      }
  /* Z_LINK (model.cpp:227-237) */
  for (int d = 0; d < D; ++d)
    for (int t = 0; t < T; ++t)
      for (int i = 0; i < T; ++i) {
        begin_row(&b, T_Z_LINK, 'L', 0.0);
        term(&b, iZ(s, d, t, i), 1.0);
        term(&b, iR(s, d, t, i), -1.0);
        term(&b, iS(s, d, t, i), -1.0);
        begin_row(&b, T_Z_LINK, 'G', 0.0);
        term(&b, iZ(s, d, t, i), 1.0);
        term(&b, iR(s, d, t, i), -1.0);
        begin_row(&b, T_Z_LINK, 'G', 0.0);
        term(&b, iZ(s, d, t, i), 1.0);
        term(&b, iS(s, d, t, i), -1.0);
      }
  /* P_LINK (model.cpp:240-252) */
  for (int t = 0; t < T; ++t)
    for (int e = 0; e < E; ++e)
      for (int ds = 0; ds < D; ++ds)
        for (int dc = 0; dc < D; ++dc) {
          if (ds == dc) continue;
          begin_row(&b, T_P_LINK, 'G', -1.0);
          term(&b, iP(s, t, e, ds, dc), 1.0);
          term(&b, iR(s, dc, t, p->edge_dst[e]), -1.0);
          term(&b, iZ(s, ds, t, p->edge_src[e]), -1.0);
        }

  /* add_energy_extension (model.cpp:258-312) */
  if (energy && p->has_energy) {
    for (int d = 0; d < D; ++d)
      for (int t = 0; t < T; ++t)
        for (int i = 0; i < T; ++i) {
          double add = p->alpha * p->q_joules[(size_t)d * T + i];
          if (add == 0.0) continue;
          int64_t k = iR(s, d, t, i);
          double next = m->obj_present[k] ? m->obj[k] + add : add;
          if (next == 0.0) {
            m->obj_present[k] = 0;
            m->obj[k] = 0.0;
          } else {
            m->obj_present[k] = 1;
            m->obj[k] = next;
          }
        }
    for (int d = 0; d < D; ++d) {
      if (!p->has_dev_limit[d]) continue;
      for (int t = 0; t < T; ++t)
        for (int i = 0; i < T; ++i) {
          begin_row(&b, T_ENERGY_DEV, 'L', p->dev_limit[d]);
          term(&b, iR(s, d, t, i), p->q_joules[(size_t)d * T + i]);
        }
    }
    if (p->has_total_limit)
      for (int t = 0; t < T; ++t) {
        begin_row(&b, T_ENERGY_TOTAL, 'L', p->total_limit - p->board_joules);
        for (int d = 0; d < D; ++d)
          for (int i = 0; i < T; ++i) {
            double q = p->q_joules[(size_t)d * T + i];
            if (q != 0.0) term(&b, iR(s, d, t, i), q);
          }
      }
  }
#undef MASS
#undef COST
#undef W
  return 0;
}

void xo_model_free(xo_model* m) {
  free(m->row_ptr);
  free(m->col);
  free(m->val);
  free(m->rhs);
  free(m->sense);
  free(m->tag);
  free(m->ordinal);
  free(m->obj);
  free(m->obj_present);
  free(m->fixed);
  memset(m, 0, sizeof *m);
}

/* ---- MPS (mps_io.cpp) --------------------------------------------------- */
void xo_format_number(double v, char* buf, size_t len) { /* mps_io.cpp:14-27 */
  if (v == 0.0) {
    snprintf(buf, len, "0");
    return;
  }
  if (isfinite(v) && v == floor(v) && fabs(v) < 1e15) {
    snprintf(buf, len, "%.0f", v);
    return;
  }
  for (int prec = 1; prec <= 17; ++prec) {
    snprintf(buf, len, "%.*g", prec, v);
    if (strtod(buf, NULL) == v) break;
  }
}

static int var_name(dims_t s, int64_t k, char* buf) { /* mps_io.cpp:29-43 */
  const int64_t DT2 = s.D * s.T * s.T, DTF = s.D * s.T * s.FE;
  if (k < 3 * DT2) {
    const char f = "RSZ"[k / DT2];
    int64_t r = k % DT2;
    return sprintf(buf, "%c_%lld_%lld_%lld", f, (long long)(r / (s.T * s.T)),
                   (long long)(r / s.T % s.T), (long long)(r % s.T));
  }
  k -= 3 * DT2;
  if (k < DTF)
    return sprintf(buf, "F_%lld_%lld_%lld", (long long)(k / (s.T * s.FE)),
                   (long long)(k / s.FE % s.T), (long long)(k % s.FE));
  k -= DTF;
  if (k < DT2)
    return sprintf(buf, "U_%lld_%lld_%lld", (long long)(k / (s.T * s.T)),
                   (long long)(k / s.T % s.T), (long long)(k % s.T));
  k -= DT2;
  int64_t dm1 = s.D - 1;
  int64_t t = k / (s.E * s.D * dm1), rem = k % (s.E * s.D * dm1);
  int64_t e = rem / (s.D * dm1);
  rem %= s.D * dm1;
  int64_t ds = rem / dm1, dc = rem % dm1;
  if (dc >= ds) ++dc;
  return sprintf(buf, "P_%lld_%lld_%lld_%lld", (long long)t, (long long)e, (long long)ds,
                 (long long)dc);
}

typedef struct {
  char* p;
  size_t n, cap;
} sbuf_t;
static void put(sbuf_t* b, const char* s, size_t n) {
  if (b->n + n + 1 > b->cap) {
    b->cap = (b->cap + n + 1) * 2;
    b->p = realloc(b->p, b->cap);
    if (!b->p) abort();
  }
  memcpy(b->p + b->n, s, n);
  b->n += n;
  b->p[b->n] = 0;
}
static void puts_(sbuf_t* b, const char* s) { put(b, s, strlen(s)); }

char* xo_write_mps(const xe_problem_desc* p, const xo_model* m, int quad, size_t* len) {
  const dims_t s = dims(p);
  const int64_t n = m->n_cols, firstP = 4 * s.D * s.T * s.T + s.D * s.T * s.FE;
  const int64_t ncol_out = quad ? firstP : n;
  sbuf_t o = {0};
  char nm[96], num[64], line[320];
  /* stable CSC: per column, rows in emission order (mps_io.cpp:141-146) */
  int64_t* cnt = calloc((size_t)n + 1, sizeof(int64_t));
  for (int64_t r = 0; r < m->n_rows; ++r) {
    if (quad && m->tag[r] == T_P_LINK) continue;
    for (int64_t k = m->row_ptr[r]; k < m->row_ptr[r + 1]; ++k) cnt[m->col[k] + 1]++;
  }
  for (int64_t j = 0; j < n; ++j) cnt[j + 1] += cnt[j];
  int64_t* pos = malloc(sizeof(int64_t) * (size_t)(cnt[n] + 1));
  int64_t* fill = malloc(sizeof(int64_t) * (size_t)(n + 1));
  memcpy(fill, cnt, sizeof(int64_t) * (size_t)(n + 1));
  for (int64_t r = 0; r < m->n_rows; ++r) {
    if (quad && m->tag[r] == T_P_LINK) continue;
    for (int64_t k = m->row_ptr[r]; k < m->row_ptr[r + 1]; ++k) pos[fill[m->col[k]]++] = k;
  }
  /* row index of an entry */
  int64_t* rowof = malloc(sizeof(int64_t) * (size_t)(m->nnz + 1));
  for (int64_t r = 0; r < m->n_rows; ++r)
    for (int64_t k = m->row_ptr[r]; k < m->row_ptr[r + 1]; ++k) rowof[k] = r;

  puts_(&o, "NAME XENGINE\nROWS\n N OBJ\n");
  for (int64_t r = 0; r < m->n_rows; ++r) {
    if (quad && m->tag[r] == T_P_LINK) continue;
    int l = sprintf(line, " %c %s_%d\n", m->sense[r], kTagName[m->tag[r]], m->ordinal[r]);
    put(&o, line, (size_t)l);
  }
  puts_(&o, "COLUMNS\n");
  int in_int = 0;
  const int64_t firstU = 3 * s.D * s.T * s.T + s.D * s.T * s.FE;
  for (int64_t j = 0; j < ncol_out; ++j) {
    int bin = j < firstU;
    if (bin && !in_int) {
      puts_(&o, "    MARK  'MARKER'  'INTORG'\n");
      in_int = 1;
    }
    if (!bin && in_int) {
      puts_(&o, "    MARK  'MARKER'  'INTEND'\n");
      in_int = 0;
    }
    var_name(s, j, nm);
    if (m->obj_present[j]) {
      xo_format_number(m->obj[j], num, sizeof num);
      int l = sprintf(line, "    %s  OBJ  %s\n", nm, num);
      put(&o, line, (size_t)l);
    }
    for (int64_t q = cnt[j]; q < cnt[j + 1]; ++q) {
      int64_t k = pos[q], r = rowof[k];
      xo_format_number(m->val[k], num, sizeof num);
      int l = sprintf(line, "    %s  %s_%d  %s\n", nm, kTagName[m->tag[r]], m->ordinal[r], num);
      put(&o, line, (size_t)l);
    }
  }
  if (in_int) puts_(&o, "    MARK  'MARKER'  'INTEND'\n");
  puts_(&o, "RHS\n");
  for (int64_t r = 0; r < m->n_rows; ++r) {
    if (quad && m->tag[r] == T_P_LINK) continue;
    if (m->rhs[r] != 0.0) {
      xo_format_number(m->rhs[r], num, sizeof num);
      int l = sprintf(line, "    RHS  %s_%d  %s\n", kTagName[m->tag[r]], m->ordinal[r], num);
      put(&o, line, (size_t)l);
    }
  }
  puts_(&o, "BOUNDS\n");
  for (int64_t j = 0; j < ncol_out; ++j) {
    var_name(s, j, nm);
    int l;
    if (m->fixed[j]) {
      l = sprintf(line, " FX BND %s 0\n", nm);
    } else if (j < firstU) {
      l = sprintf(line, " BV BND %s\n", nm);
    } else if (j < firstP) {
      int64_t d = (j - firstU) / (s.T * s.T);
      xo_format_number((double)p->budget_bytes[d], num, sizeof num);
      l = sprintf(line, " UP BND %s %s\n", nm, num);
    } else {
      l = sprintf(line, " UP BND %s 1\n", nm);
    }
    put(&o, line, (size_t)l);
  }
  if (quad) { /* QUADOBJ (mps_io.cpp:188-195); m.quad in (t,e,ds,dc) order, w != 0 */
    int any = 0;
    for (int t = 0; t < s.T; ++t)
      for (int e = 0; e < s.E; ++e)
        for (int ds = 0; ds < s.D; ++ds)
          for (int dc = 0; dc < s.D; ++dc) {
            if (ds == dc) continue;
            double w = p->copy_ms[((size_t)e * s.D + ds) * s.D + dc];
            if (w == 0.0) continue;
            if (!any) puts_(&o, "QUADOBJ\n");
            any = 1;
            char nz[96];
            var_name(s, iR(s, dc, t, p->edge_dst[e]), nm);
            var_name(s, iZ(s, ds, t, p->edge_src[e]), nz);
            xo_format_number(w, num, sizeof num);
            int l = sprintf(line, "    %s  %s  %s\n", nm, nz, num);
            put(&o, line, (size_t)l);
          }
  }
  puts_(&o, "ENDATA\n");
  free(cnt);
  free(pos);
  free(fill);
  free(rowof);
  *len = o.n;
  return o.p;
}

/* ---- K2 restatement ----------------------------------------------------- */
static int cube_bit(const uint32_t* cube, int D, int T, int which, int d, int t, int i) {
  const int W = (T + 31) / 32;
  const uint32_t* row = cube + (((size_t)which * D + d) * T + t) * W;
  return (int)((row[i >> 5] >> (i & 31)) & 1u);
}

/* complete_assignment (model.cpp:471-549) */
void xo_complete(const xe_problem_desc* p, int strict, const uint32_t* cube, double* x) {
  const dims_t s = dims(p);
  const int D = p->D, T = p->T, E = p->E;
  memset(x, 0, sizeof(double) * (size_t)ncols(s));
#define Rb(d, t, i) cube_bit(cube, D, T, 0, d, t, i)
#define Sb(d, t, i) cube_bit(cube, D, T, 1, d, t, i)
#define Zb(d, t, i) (Rb(d, t, i) > Sb(d, t, i) ? Rb(d, t, i) : Sb(d, t, i))
  for (int d = 0; d < D; ++d)
    for (int t = 0; t < T; ++t)
      for (int i = 0; i < T; ++i) {
        x[iR(s, d, t, i)] = Rb(d, t, i);
        x[iS(s, d, t, i)] = Sb(d, t, i);
        x[iZ(s, d, t, i)] = Zb(d, t, i);
      }
  /* f_at (model.cpp:492-505) */
  for (int d = 0; d < D; ++d)
    for (int t = 0; t < T; ++t)
      for (int eo = 0; eo < E + T; ++eo) {
        int u = eo < E ? p->edge_src[eo] : eo - E;
        int v = eo < E ? p->edge_dst[eo] : eo - E;
        int f = 1;
        if (!Rb(d, t, v) || !Zb(d, t, u)) f = 0;
        else if (t + 1 < T && Sb(d, t + 1, u)) f = 0;
        else
          for (int e = 0; e < E && f; ++e) {
            if (p->edge_src[e] != u || p->edge_dst[e] <= v) continue;
            if (strict) {
              for (int dd = 0; dd < D; ++dd)
                if (Rb(dd, t, p->edge_dst[e])) f = 0;
            } else if (Rb(d, t, p->edge_dst[e])) {
              f = 0;
            }
          }
        x[iF(s, d, t, eo)] = f;
      }
  /* U recurrence (model.cpp:521-537) */
  for (int d = 0; d < D; ++d)
    for (int t = 0; t < T; ++t) {
      double u0 = 0.0;
      for (int i = 0; i < T; ++i)
        if (Sb(d, t, i)) u0 += (double)p->output_bytes[i];
      if (Rb(d, t, 0)) u0 += (double)p->output_bytes[0];
      x[iU(s, d, t, 0)] = u0;
      double cur = u0;
      for (int v = 0; v + 1 < T; ++v) {
        double freed = 0.0;
        for (int e = 0; e < E; ++e) {
          if (p->edge_dst[e] != v) continue;
          int u = p->edge_src[e];
          int k = 0;
          while (!(p->edge_src[k] == u && p->edge_dst[k] == v)) ++k;
          if (x[iF(s, d, t, k)] != 0.0) freed += (double)p->output_bytes[u];
        }
        if (x[iF(s, d, t, E + v)] != 0.0) freed += (double)p->output_bytes[v];
        cur = cur - freed + (Rb(d, t, v + 1) ? (double)p->output_bytes[v + 1] : 0.0);
        x[iU(s, d, t, v + 1)] = cur;
      }
    }
  /* P (model.cpp:538-547) */
  for (int t = 0; t < T; ++t)
    for (int e = 0; e < E; ++e)
      for (int ds = 0; ds < D; ++ds)
        for (int dc = 0; dc < D; ++dc) {
          if (ds == dc) continue;
          x[iP(s, t, e, ds, dc)] = (Rb(dc, t, p->edge_dst[e]) && Zb(ds, t, p->edge_src[e])) ? 1.0 : 0.0;
        }
#undef Rb
#undef Sb
#undef Zb
}

/* objective_value (model.cpp:369-428), same loop and summation order */
double xo_objective(const xe_problem_desc* p, int energy, const double* x) {
  const dims_t s = dims(p);
  const int D = p->D, T = p->T, E = p->E;
  double total = 0.0;
  for (int d = 0; d < D; ++d)
    for (int t = 0; t < T; ++t)
      for (int i = 0; i < T; ++i) {
        double r = x[iR(s, d, t, i)];
        if (r != 0.0) total += p->cost_ms[(size_t)d * T + i] * r;
      }
  for (int t = 0; t < T; ++t)
    for (int e = 0; e < E; ++e)
      for (int dc = 0; dc < D; ++dc) {
        double r = x[iR(s, dc, t, p->edge_dst[e])];
        if (r == 0.0) continue;
        for (int ds = 0; ds < D; ++ds) {
          if (ds == dc) continue;
          double z = x[iZ(s, ds, t, p->edge_src[e])];
          if (z != 0.0) total += p->copy_ms[((size_t)e * D + ds) * D + dc] * r * z;
        }
      }
  if (energy && p->has_energy)
    for (int d = 0; d < D; ++d)
      for (int t = 0; t < T; ++t)
        for (int i = 0; i < T; ++i) {
          double r = x[iR(s, d, t, i)];
          if (r != 0.0) total += p->alpha * p->q_joules[(size_t)d * T + i] * r;
        }
  return total;
}

/* check_assignment (model.cpp:430-469) on a full-space dense assignment */
uint32_t xo_check(const xe_problem_desc* p, const xo_model* m, const double* x, double tol) {
  const dims_t s = dims(p);
  uint32_t f = 0;
  const int64_t firstU = 3 * s.D * s.T * s.T + s.D * s.T * s.FE;
  const int64_t firstP = firstU + s.D * s.T * s.T;
  for (int64_t j = 0; j < m->n_cols; ++j) {
    double val = x[j];
    if (j < firstU) {
      if (fabs(val) > tol && fabs(val - 1.0) > tol) f |= XE_F_OTHER;
    } else if (j < firstP) {
      double b = (double)p->budget_bytes[(j - firstU) / (s.T * s.T)];
      if (val < -tol * (b > 1.0 ? b : 1.0) || val > b * (1.0 + tol) + tol) f |= XE_F_U_BOUND;
    } else if (val < -tol || val > 1.0 + tol) {
      f |= XE_F_OTHER;
    }
    if (m->fixed[j] && fabs(val) > tol) f |= XE_F_FIXED_ZERO;
  }
  for (int64_t r = 0; r < m->n_rows; ++r) {
    double lhs = 0.0, scale = fabs(m->rhs[r]) > 1.0 ? fabs(m->rhs[r]) : 1.0;
    for (int64_t k = m->row_ptr[r]; k < m->row_ptr[r + 1]; ++k) {
      double term = m->val[k] * x[m->col[k]];
      lhs += term;
      if (fabs(term) > scale) scale = fabs(term);
    }
    double viol = m->sense[r] == 'L' ? lhs - m->rhs[r]
                  : m->sense[r] == 'G' ? m->rhs[r] - lhs
                                       : fabs(lhs - m->rhs[r]);
    if (viol > tol * scale) f |= kTagFlag[m->tag[r]];
  }
  return f;
}

/* decode legality (schedule.cpp:40-129), scanning past the first error:
 * DECODE = some dependency resident nowhere or some copy source freed
 * earlier in its timestep; DECODE_FREED = the latter. */
uint32_t xo_decode_flags(const xe_problem_desc* p, const double* x) {
  const dims_t s = dims(p);
  const int D = p->D, T = p->T, E = p->E;
  uint32_t f = 0;
  char* freed = malloc((size_t)D * T);
  for (int t = 0; t < T; ++t) {
    memset(freed, 0, (size_t)D * T);
    for (int v = 0; v <= t; ++v)
      for (int d = 0; d < D; ++d) {
        if (!(x[iR(s, d, t, v)] > 0.5)) continue;
        for (int e = 0; e < E; ++e) {
          if (p->edge_dst[e] != v) continue;
          int u = p->edge_src[e];
          if (x[iZ(s, d, t, u)] > 0.5) continue;
          int src = -1;
          for (int d2 = 0; d2 < D; ++d2)
            if (x[iZ(s, d2, t, u)] > 0.5) {
              src = d2;
              break;
            }
          if (src < 0) f |= XE_F_DECODE;
          else if (freed[(size_t)src * T + u]) f |= XE_F_DECODE | XE_F_DECODE_FREED;
        }
        for (int e = 0; e < E; ++e)
          if (p->edge_dst[e] == v && x[iF(s, d, t, e)] > 0.5) freed[(size_t)d * T + p->edge_src[e]] = 1;
        if (x[iF(s, d, t, E + v)] > 0.5) freed[(size_t)d * T + v] = 1;
      }
  }
  free(freed);
  return f;
}

void xo_eval_cube(const xe_problem_desc* p, const xo_model* m, int strict, int energy,
                  const uint32_t* cube, double* obj, int64_t* peak, uint32_t* flags) {
  const dims_t s = dims(p);
  double* x = malloc(sizeof(double) * (size_t)ncols(s));
  xo_complete(p, strict, cube, x);
  *obj = xo_objective(p, energy, x);
  uint32_t f = xo_check(p, m, x, 1e-6);
  for (int d = 0; d < p->D; ++d) {
    double pk = 0.0;
    for (int t = 0; t < p->T; ++t)
      for (int v = 0; v < p->T; ++v)
        if (x[iU(s, d, t, v)] > pk) pk = x[iU(s, d, t, v)];
    peak[d] = (int64_t)pk;
    if (peak[d] > p->budget_bytes[d]) f |= XE_F_BUDGET;
  }
  f |= xo_decode_flags(p, x);
  *flags = f;
  free(x);
}

void xo_eval_cubes(const xe_problem_desc* p, const xo_model* m, int strict, int energy,
                   const uint32_t* cubes, int64_t n, double* obj, int64_t* peak,
                   uint32_t* flags) {
  const size_t words = 2 * (size_t)p->D * p->T * ((p->T + 31) / 32);
  for (int64_t c = 0; c < n; ++c)
    xo_eval_cube(p, m, strict, energy, cubes + (size_t)c * words, obj + c, peak + c * p->D,
                 flags + c);
}

/* save_all_assignment (solver.cpp:30-42); policy 1: saved only until the
 * tensor's last consumer, and never when it has none. */
void xo_placement_cube(const xe_problem_desc* p, const uint8_t* dev, int policy, uint32_t* cube) {
  const int D = p->D, T = p->T, W = (T + 31) / 32;
  memset(cube, 0, sizeof(uint32_t) * 2 * (size_t)D * T * W);
  for (int i = 0; i < T; ++i) {
    int last = T - 1;
    if (policy == 1) {
      last = -1;
      for (int e = 0; e < p->E; ++e)
        if (p->edge_src[e] == i && p->edge_dst[e] > last) last = p->edge_dst[e];
    }
    int d = dev[i];
    cube[(((size_t)0 * D + d) * T + i) * W + (i >> 5)] |= 1u << (i & 31);
    for (int t = i + 1; t <= last; ++t)
      cube[(((size_t)1 * D + d) * T + t) * W + (i >> 5)] |= 1u << (i & 31);
  }
}

void xo_eval_placements(const xe_problem_desc* p, const xo_model* m, const uint8_t* dev,
                        int64_t n, int policy, double* obj, int64_t* peak, uint32_t* flags) {
  const size_t words = 2 * (size_t)p->D * p->T * ((p->T + 31) / 32);
  uint32_t* cube = malloc(sizeof(uint32_t) * words);
  for (int64_t c = 0; c < n; ++c) {
    xo_placement_cube(p, dev + (size_t)c * p->T, policy, cube);
    xo_eval_cube(p, m, 0, 0, cube, obj + c, peak + c * p->D, flags + c);
  }
  free(cube);
}

/* assignment_oracle (solver.cpp:44-75) */
double xo_assignment_oracle(const xe_problem_desc* p, int32_t* best_dev, int64_t* n) {
  const dims_t s = dims(p);
  const int D = p->D, T = p->T, W = (T + 31) / 32;
  uint8_t* dev = calloc((size_t)T, 1);
  uint32_t* cube = malloc(sizeof(uint32_t) * 2 * (size_t)D * T * W);
  double* x = malloc(sizeof(double) * (size_t)ncols(s));
  double best = INFINITY;
  *n = 0;
  for (;;) {
    ++*n;
    xo_placement_cube(p, dev, 0, cube);
    xo_complete(p, 0, cube, x);
    double obj = xo_objective(p, 0, x);
    if (obj < best) {
      best = obj;
      for (int i = 0; i < T; ++i) best_dev[i] = dev[i];
    }
    int k = T - 1;
    while (k >= 0 && dev[k] == D - 1) dev[k--] = 0;
    if (k < 0) break;
    ++dev[k];
  }
  free(dev);
  free(cube);
  free(x);
  return best;
}
