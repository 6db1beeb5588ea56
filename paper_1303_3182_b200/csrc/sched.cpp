// Host schedule compiler (see sched.hpp for the reference map).
#include "sched.hpp"

#include <algorithm>
#include <cctype>
#include <functional>
#include <queue>
#include <tuple>
#include <unordered_map>
#include <unordered_set>

namespace tqr {

namespace {

std::string lower(std::string s) {
  for (auto& ch : s) ch = char(std::tolower(static_cast<unsigned char>(ch)));
  return s;
}

std::string py_repr(const std::string& s) { return "'" + s + "'"; }

std::string tup(int a, int b) { return "(" + std::to_string(a) + ", " + std::to_string(b) + ")"; }

bool key_step_k_i(const Entry& a, const Entry& b) {
  return std::tie(a.step, a.k, a.i) < std::tie(b.step, b.k, b.i);
}

// _pair_groups (qr.py:208-218): a bunch of z consecutive rows zeroed in one
// (step, col) pairs with the z rows directly above it, in natural order.
std::vector<Entry> pair_groups(const Grid<int32_t>& steps, int p, int qq) {
  // collect (step, col) -> sorted rows
  std::vector<std::tuple<int, int, int>> cells;  // (s, k, i)
  for (int k = 1; k <= qq; ++k)
    for (int i = 1; i <= p; ++i)
      if (steps.has(i, k)) cells.emplace_back(steps.at(i, k), k, i);
  std::sort(cells.begin(), cells.end());
  std::vector<Entry> out;
  size_t n = 0;
  while (n < cells.size()) {
    size_t m = n;
    int s = std::get<0>(cells[n]), k = std::get<1>(cells[n]);
    while (m < cells.size() && std::get<0>(cells[m]) == s && std::get<1>(cells[m]) == k) ++m;
    int z = int(m - n);
    int r0 = std::get<2>(cells[n]);
    for (int j = 0; j < z; ++j) {
      if (std::get<2>(cells[n + j]) != r0 + j) {
        std::string rows = "[";
        for (size_t t = n; t < m; ++t) rows += (t > n ? ", " : "") + std::to_string(std::get<2>(cells[t]));
        rows += "]";
        throw AssertError("step " + std::to_string(s) + " column " + std::to_string(k) + ": group " + rows +
                          " not consecutive");
      }
    }
    for (int j = 0; j < z; ++j) out.push_back({r0 + j, r0 - z + j, k, s});
    n = m;
  }
  return out;
}

}  // namespace

int fibonacci_x(int p) {
  int x = 0;
  while (int64_t(x) * (x + 1) / 2 < p - 1) ++x;
  return x;
}

Coarse coarse_schedule(int p, int q, std::string algo) {
  if (!(p >= q && q >= 1)) throw ValueError("need p >= q >= 1");
  algo = lower(algo);
  Coarse c{p, q, fibonacci_x(p), Grid<int32_t>(p, q, 0), {}};
  const int qq = std::min(p, q);
  auto& st = c.steps;
  if (algo == "sameh-kuck" || algo == "samehkuck" || algo == "flattree") {
    // s(i,k) = max(s(i,k-1), s(i-1,k)) + 1, pivot = k (qr.py:221-232)
    for (int k = 1; k <= qq; ++k)
      for (int i = k + 1; i <= p; ++i) {
        int s = std::max(st.get(i, k - 1, 0), st.get(i - 1, k, 0)) + 1;
        st.at(i, k) = s;
        c.entries.push_back({i, k, k, s});
      }
  } else if (algo == "fibonacci") {
    // first column from the Fibonacci pattern, then a shift by two per column
    // (qr.py:235-251)
    const int x = c.x;
    for (int i = 2; i <= p; ++i) {
      int y = 1;
      while (int64_t(i) > int64_t(y) * (y + 1) / 2 + 1) ++y;
      st.at(i, 1) = x - y + 1;
    }
    for (int k = 2; k <= qq; ++k)
      for (int i = k + 1; i <= p; ++i) st.at(i, k) = st.at(i - 1, k - 1) + 2;
    c.entries = pair_groups(st, p, qq);
  } else if (algo == "greedy") {
    // each step, each column left to right: rows ready (previous column done
    // before this step) zero their bottom half (qr.py:254-276)
    int64_t remaining = 0;
    for (int k = 1; k <= qq; ++k) remaining += p - k;
    int s = 0;
    std::vector<int> avail;
    avail.reserve(size_t(p) + 1);
    while (remaining) {
      ++s;
      for (int k = 1; k <= qq; ++k) {
        avail.clear();
        for (int i = k; i <= p; ++i) {
          if (st.has(i, k)) continue;
          if (k == 1 || st.get(i, k - 1, s) <= s - 1) avail.push_back(i);
        }
        int z = int(avail.size()) / 2;
        if (z == 0) continue;
        for (size_t t = avail.size() - size_t(z); t < avail.size(); ++t) st.at(avail[t], k) = s;
        remaining -= z;
      }
    }
    c.entries = pair_groups(st, p, qq);
  } else {
    throw ValueError("unknown coarse algorithm " + py_repr(algo));
  }
  std::sort(c.entries.begin(), c.entries.end(), key_step_k_i);
  return c;
}

std::vector<Entry> with_steps(const std::vector<Entry>& in) {
  // each elimination occupies both of its rows for one unit (qr.py:118-127)
  std::unordered_map<int32_t, int32_t> last;
  last.reserve(in.size() * 2 + 1);
  std::vector<Entry> out;
  out.reserve(in.size());
  for (const auto& e : in) {
    auto gi = last.find(e.i);
    auto gp = last.find(e.piv);
    int32_t s = std::max(gi == last.end() ? 0 : gi->second, gp == last.end() ? 0 : gp->second) + 1;
    last[e.i] = s;
    last[e.piv] = s;
    out.push_back({e.i, e.piv, e.k, s});
  }
  return out;
}

std::vector<Entry> plasmatree_list(int p, int q, int bs) {
  // flat trees inside domains of bs rows starting at row k, binary merge of
  // the domain heads (qr.py:336-362)
  if (!(1 <= bs && bs <= p)) throw ValueError("domain size must satisfy 1 <= BS <= p");
  std::vector<Entry> e;
  std::vector<int> heads, nxt;
  for (int k = 1; k <= std::min(p, q); ++k) {
    heads.clear();
    const int n = p - k + 1;  // rows k..p
    for (int lo = 0; lo < n; lo += bs) {
      int head = k + lo;
      heads.push_back(head);
      for (int t = lo + 1; t < std::min(lo + bs, n); ++t) e.push_back({k + t, head, k, 0});
    }
    while (heads.size() > 1) {
      nxt.clear();
      for (size_t a = 0; a + 1 < heads.size(); a += 2) {
        e.push_back({heads[a + 1], heads[a], k, 0});
        nxt.push_back(heads[a]);
      }
      if (heads.size() % 2) nxt.push_back(heads.back());
      heads.swap(nxt);
    }
  }
  auto out = with_steps(e);
  std::sort(out.begin(), out.end(),
            [](const Entry& a, const Entry& b) { return std::tie(a.k, a.step, a.i) < std::tie(b.k, b.step, b.i); });
  return out;
}

std::string validate(int p, int q, const std::vector<Entry>& es) {
  // row-ready and potential-annihilator conditions (qr.py:56-83)
  const int qq = std::min(p, q);
  Grid<uint8_t> zeroed(std::max(p, 0), std::max(q, 0), 0);
  int64_t nz = 0;
  for (size_t n = 0; n < es.size(); ++n) {
    const auto& e = es[n];
    const std::string pre = "entry " + std::to_string(n) + ": ";
    if (!(1 <= e.k && e.k <= qq) || !(e.k < e.i && e.i <= p))
      return pre + "elim(" + std::to_string(e.i) + "," + std::to_string(e.piv) + "," + std::to_string(e.k) +
             ") out of range";
    if (e.i == e.piv) return pre + "a row cannot annihilate itself";
    if (!(e.k <= e.piv && e.piv <= p))
      return pre + "pivot row " + std::to_string(e.piv) + " invalid for column " + std::to_string(e.k);
    for (int row : {e.i, e.piv})
      for (int kk = 1; kk < e.k; ++kk)
        if (!zeroed.at(row, kk))
          return pre + "row " + std::to_string(row) + " not ready for column " + std::to_string(e.k) + " (tile (" +
                 std::to_string(row) + "," + std::to_string(kk) + ") not yet zeroed)";
    if (zeroed.at(e.piv, e.k))
      return pre + "pivot row " + std::to_string(e.piv) + " is not a potential annihilator (tile (" +
             std::to_string(e.piv) + "," + std::to_string(e.k) + ") already zeroed)";
    if (zeroed.at(e.i, e.k))
      return pre + "tile (" + std::to_string(e.i) + "," + std::to_string(e.k) + ") zeroed twice";
    zeroed.at(e.i, e.k) = 1;
    ++nz;
  }
  int64_t want = 0;
  for (int k = 1; k <= qq; ++k) want += p - k;
  if (nz != want)
    return "elimination list incomplete: " + std::to_string(nz) + "/" + std::to_string(want) + " tiles zeroed";
  return "";
}

std::vector<Entry> normalized(int p, int q, const std::vector<Entry>& in) {
  // Lemma 3.1 exchange of reverse eliminations, column by column (qr.py:85-116)
  std::vector<Entry> entries = in;
  for (int k0 = 1; k0 <= std::min(p, q); ++k0) {
    for (;;) {
      int i0 = INT32_MIN;
      bool any = false;
      for (const auto& e : entries)
        if (e.k == k0 && e.i < e.piv) {
          any = true;
          i0 = std::max(i0, std::max(e.i, e.piv));
        }
      if (!any) break;
      long first = -1, own = -1;
      for (size_t n = 0; n < entries.size(); ++n)
        if (entries[n].k == k0 && entries[n].i < entries[n].piv && entries[n].piv == i0) {
          first = long(n);
          break;
        }
      for (size_t n = 0; n < entries.size(); ++n)
        if (entries[n].k == k0 && entries[n].i == i0) {
          own = long(n);
          break;
        }
      if (first < 0 || own < 0) throw std::runtime_error("StopIteration");
      const int i1 = entries[size_t(first)].i;
      std::vector<Entry> nw = entries;
      nw[size_t(first)] = {i0, i1, k0, entries[size_t(first)].step};
      for (size_t n = size_t(first) + 1; n < entries.size(); ++n) {
        const auto& e = entries[n];
        if (e.k == k0 && e.piv == i0 && long(n) != own) nw[n] = {e.i, i1, k0, e.step};
      }
      const auto& eo = entries[size_t(own)];
      nw[size_t(own)] = {i1, eo.piv, k0, eo.step};
      entries.swap(nw);
    }
  }
  return entries;
}

// ---------------------------------------------------------------------------
// tiled builder (qr.py:376-532)

Build::Build(int p_, int q_, bool ts_, const int64_t* weights, bool kt, bool ru)
    : p(p_), q(q_), ts(ts_), keep_trace(kt), record_updates(ru) {
  if (!(p >= q && q >= 1)) throw ValueError("need p >= q >= 1");
  static const int64_t kQrTT[6] = {4, 2, 6, 6, 6, 12};  // taskgraph.py:92-95
  for (int t = 0; t < 6; ++t) w[t] = weights ? weights[t] : kQrTT[t];
  zeroed = Grid<int64_t>(p, q, -1);
  R = Grid<int64_t>(p, q, -1);
  V = Grid<int64_t>(p, q, -1);
  VE = Grid<int64_t>(p, q, -1);
  D = Grid<int64_t>(p, q, -1);
  tri = Grid<uint8_t>(p, q, 0);
}

static int64_t need(const Grid<int64_t>& g, int i, int k) {
  if (!g.in(i, k)) throw ValueError("tile index " + tup(i, k) + " outside the tile grid");
  int64_t v = g.at(i, k);
  if (v < 0) throw KeyError(tup(i, k));
  return v;
}
static int64_t getd(const Grid<int64_t>& g, int i, int k) {
  if (!g.in(i, k)) throw ValueError("tile index " + tup(i, k) + " outside the tile grid");
  int64_t v = g.at(i, k);
  return v < 0 ? 0 : v;
}

int64_t Build::rec(Kind kind, int a, int b, int c, int d, int64_t start) {
  if (w[kind] < 0) throw KeyError(kKindName[kind]);
  int64_t fin = start + w[kind];
  counts[kind] += 1;
  total_weight += w[kind];
  if (fin > cp) cp = fin;
  if (keep_trace) trace.push_back({int8_t(kind), a, b, c, d, fin});
  return fin;
}

int64_t Build::geqrt(int i, int k) {
  int64_t fin = rec(GEQRT, i, k, -1, -1, getd(D, i, k));
  R.at(i, k) = fin;
  V.at(i, k) = fin;
  tri.at(i, k) = 1;
  return fin;
}

int64_t Build::unmqr(int i, int k, int j) {
  int64_t s = std::max(need(V, i, k), getd(D, i, j));
  int64_t fin = rec(UNMQR, i, k, j, -1, s);
  D.at(i, j) = fin;
  return fin;
}

int64_t Build::ttqrt(int i, int piv, int k) {
  int64_t a = need(R, i, k);
  int64_t s = std::max(a, need(R, piv, k));
  int64_t fin = rec(TTQRT, i, piv, k, -1, s);
  R.at(piv, k) = fin;
  VE.at(i, k) = fin;
  if (zeroed.at(i, k) < 0) zeroed_order.insert(zeroed_order.end(), {i, k});
  zeroed.at(i, k) = fin;
  return fin;
}

int64_t Build::ttmqr(int i, int piv, int k, int j) {
  int64_t s = need(VE, i, k);
  s = std::max(s, getd(D, i, j));
  s = std::max(s, getd(D, piv, j));
  int64_t fin = rec(TTMQR, i, piv, k, j, s);
  D.at(i, j) = fin;
  D.at(piv, j) = fin;
  if (record_updates) upd.insert(upd.end(), {i, k, j, fin});
  return fin;
}

int64_t Build::tsqrt(int i, int piv, int k) {
  int64_t a = getd(D, i, k);
  int64_t s = std::max(a, need(R, piv, k));
  int64_t fin = rec(TSQRT, i, piv, k, -1, s);
  R.at(piv, k) = fin;
  VE.at(i, k) = fin;
  if (zeroed.at(i, k) < 0) zeroed_order.insert(zeroed_order.end(), {i, k});
  zeroed.at(i, k) = fin;
  return fin;
}

int64_t Build::tsmqr(int i, int piv, int k, int j) {
  int64_t s = need(VE, i, k);
  s = std::max(s, getd(D, i, j));
  s = std::max(s, getd(D, piv, j));
  int64_t fin = rec(TSMQR, i, piv, k, j, s);
  D.at(i, j) = fin;
  D.at(piv, j) = fin;
  return fin;
}

void Build::triangularize(int i, int k) {
  geqrt(i, k);
  for (int j = k + 1; j <= q; ++j) unmqr(i, k, j);
}

void Build::preprocess_tt() {
  for (int i = 1; i <= p; ++i) triangularize(i, 1);
}

int64_t Build::elim_tt(int i, int piv, int k) {
  // Alg. 3.3 bundle: zero (i,k), update both rows, re-triangularize row i
  int64_t fin = ttqrt(i, piv, k);
  for (int j = k + 1; j <= q; ++j) ttmqr(i, piv, k, j);
  if (k + 1 <= q) triangularize(i, k + 1);
  return fin;
}

int64_t Build::elim_ts(int i, int piv, int k) {
  // TS bundle: lazy pivot triangle; an ex-pivot target falls back to TT
  if (!tri.in(piv, k) || !tri.in(i, k)) throw ValueError("tile index outside the tile grid");
  if (!tri.at(piv, k)) triangularize(piv, k);
  int64_t fin;
  if (tri.at(i, k)) {
    fin = ttqrt(i, piv, k);
    for (int j = k + 1; j <= q; ++j) ttmqr(i, piv, k, j);
  } else {
    fin = tsqrt(i, piv, k);
    for (int j = k + 1; j <= q; ++j) tsmqr(i, piv, k, j);
  }
  return fin;
}

void Build::run_list(const std::vector<Entry>& list) {
  elim = list;
  if (!ts) {
    preprocess_tt();
    for (const auto& e : list) elim_tt(e.i, e.piv, e.k);
  } else {
    for (const auto& e : list) elim_ts(e.i, e.piv, e.k);
    for (int k = 1; k <= q; ++k)
      if (!tri.at(k, k)) triangularize(k, k);
  }
}

Build* tiled_build(int p, int q, const std::vector<Entry>& list, bool ts, const int64_t* w, bool keep_trace,
                   bool record_updates, bool validate_first) {
  if (validate_first) {
    std::string msg = validate(p, q, list);
    if (!msg.empty()) throw ValueError(msg);
  }
  auto* b = new Build(p, q, ts, w, keep_trace, record_updates);
  try {
    b->run_list(list);
  } catch (...) {
    delete b;
    throw;
  }
  return b;
}

// ---------------------------------------------------------------------------
// event-driven Asap / GrASAP (qr.py:551-611)

namespace {
using Ev = std::tuple<int64_t, int, int>;  // (time, col, row), heapq order

std::vector<Entry> run_asap_columns(Build& b, int first_col, std::vector<Ev> seeds) {
  const int q = b.q;
  std::vector<std::vector<int>> avail(size_t(q) + 2);
  std::priority_queue<Ev, std::vector<Ev>, std::greater<Ev>> heap(std::greater<Ev>(), std::move(seeds));
  std::vector<Entry> entries;
  std::vector<int> touched;
  while (!heap.empty()) {
    const int64_t now = std::get<0>(heap.top());
    touched.clear();
    while (!heap.empty() && std::get<0>(heap.top()) == now) {
      Ev ev = heap.top();
      heap.pop();
      int k = std::get<1>(ev), row = std::get<2>(ev);
      auto& col = avail[size_t(k)];
      col.insert(std::upper_bound(col.begin(), col.end(), row), row);  // insort_right
      if (std::find(touched.begin(), touched.end(), k) == touched.end()) touched.push_back(k);
    }
    std::sort(touched.begin(), touched.end());
    for (int k : touched) {
      auto& rows = avail[size_t(k)];
      const size_t s = rows.size() / 2;
      if (s == 0) continue;
      std::vector<int> part(rows.end() - long(2 * s), rows.end());
      rows.resize(rows.size() - 2 * s);
      for (size_t t = 0; t < s; ++t) {
        const int piv = part[t], tgt = part[s + t];
        int64_t fin = b.elim_tt(tgt, piv, k);
        entries.push_back({tgt, piv, k, 0});
        heap.emplace(fin, k, piv);
        if (k + 1 <= q) heap.emplace(b.V.at(tgt, k + 1), k + 1, tgt);
      }
    }
  }
  (void)first_col;
  return entries;
}
}  // namespace

Build* asap_build(int p, int q, const int64_t* w, bool keep_trace, bool record_updates) {
  auto* b = new Build(p, q, false, w, keep_trace, record_updates);
  try {
    b->preprocess_tt();
    std::vector<Ev> seeds;
    for (int i = 1; i <= p; ++i) seeds.emplace_back(b->V.at(i, 1), 1, i);
    auto entries = run_asap_columns(*b, 1, std::move(seeds));
    b->elim = with_steps(entries);
  } catch (...) {
    delete b;
    throw;
  }
  return b;
}

Build* grasap_build(int p, int q, int gi, const int64_t* w, bool keep_trace, bool record_updates) {
  if (!(1 <= gi && gi <= q)) throw ValueError("need 1 <= i <= q");
  if (gi == q) return asap_build(p, q, w, keep_trace, record_updates);
  auto* b = new Build(p, q, false, w, keep_trace, record_updates);
  try {
    b->preprocess_tt();
    Coarse g = coarse_schedule(p, q, "greedy");
    std::vector<Entry> all;
    for (const auto& e : g.entries)
      if (e.k <= q - gi) {
        b->elim_tt(e.i, e.piv, e.k);
        all.push_back(e);
      }
    const int first_dyn = q - gi + 1;
    std::vector<Ev> seeds;
    for (int r = first_dyn; r <= p; ++r) seeds.emplace_back(need(b->V, r, first_dyn), first_dyn, r);
    auto dyn = run_asap_columns(*b, first_dyn, std::move(seeds));
    all.insert(all.end(), dyn.begin(), dyn.end());
    b->elim = with_steps(all);
  } catch (...) {
    delete b;
    throw;
  }
  return b;
}

Build* build_tree(int p, int q, std::string algo, bool ts, int bs, int grasap_i, const int64_t* w, bool keep_trace,
                  bool record_updates) {
  algo = lower(algo);
  if (algo == "asap") {
    if (ts) throw ValueError("Asap is defined over TT kernels");
    return asap_build(p, q, w, keep_trace, record_updates);
  }
  if (algo == "grasap") {
    if (ts) throw ValueError("GrASAP is defined over TT kernels");
    return grasap_build(p, q, grasap_i, w, keep_trace, record_updates);
  }
  std::vector<Entry> list;
  if (algo == "flattree" || algo == "sameh-kuck" || algo == "samehkuck") {
    list = coarse_schedule(p, q, "sameh-kuck").entries;
  } else if (algo == "fibonacci" || algo == "greedy") {
    list = coarse_schedule(p, q, algo).entries;
  } else if (algo == "binarytree") {
    list = plasmatree_list(p, q, 1);
  } else if (algo == "plasmatree") {
    if (bs == INT32_MIN) throw ValueError("plasmatree needs a domain size bs");
    list = plasmatree_list(p, q, bs);
  } else {
    throw ValueError("unknown algorithm " + py_repr(algo));
  }
  auto* b = new Build(p, q, ts, w, keep_trace, record_updates);
  try {
    b->run_list(list);
  } catch (...) {
    delete b;
    throw;
  }
  return b;
}

// ---------------------------------------------------------------------------
// hazard DAG (taskgraph.py:262-322)

std::vector<Edge> hazard_edges(const Build& b) { return hazard_edges(b.p, b.q, b.trace); }

std::vector<Edge> hazard_edges(int p, int q, const std::vector<TaskRec>& trace) {
  enum { MD = 0, MR = 1, MV = 2, MT = 3, MS = 4 };
  const size_t P = size_t(p) + 2, Q = size_t(q) + 2;
  auto tid = [&](int m, int r, int c) -> size_t { return (size_t(m) * P + size_t(r)) * Q + size_t(c); };
  std::vector<int32_t> last_write(5 * P * Q, -1);
  std::vector<std::vector<int32_t>> readers(5 * P * Q);
  std::vector<Edge> edges;
  edges.reserve(trace.size() * 4);
  std::vector<size_t> rdv;
  size_t rd[3], wr[2];
  for (size_t t = 0; t < trace.size(); ++t) {
    const auto& T = trace[t];
    const size_t* rdp = rd;
    int nr = 0, nw = 0;
    switch (T.kind) {
      case GEQRT:
        rd[nr++] = tid(MD, T.a, T.b);
        wr[nw++] = tid(MR, T.a, T.b);
        wr[nw++] = tid(MV, T.a, T.b);
        break;
      case UNMQR:
        rd[nr++] = tid(MV, T.a, T.b);
        rd[nr++] = tid(MD, T.a, T.c);
        wr[nw++] = tid(MD, T.a, T.c);
        break;
      case TTQRT:
      case TSQRT:
        rd[nr++] = tid(T.kind == TTQRT ? MR : MD, T.a, T.c);
        rd[nr++] = tid(MR, T.b, T.c);
        wr[nw++] = tid(MR, T.b, T.c);
        wr[nw++] = tid(T.kind == TTQRT ? MT : MS, T.a, T.c);
        break;
      case TTMQR:
      case TSMQR:
        rd[nr++] = tid(T.kind == TTMQR ? MT : MS, T.a, T.c);
        rd[nr++] = tid(MD, T.a, T.d);
        rd[nr++] = tid(MD, T.b, T.d);
        wr[nw++] = tid(MD, T.a, T.d);
        wr[nw++] = tid(MD, T.b, T.d);
        break;
      case PACK:  // the tile's original data arrives: writes D(i,j)
        wr[nw++] = tid(MD, T.a, T.b);
        break;
      case UNPACK:  // final R tile (i,j) leaves: reads R(i,i) or D(i,j)
        rd[nr++] = tid(T.a == T.b ? MR : MD, T.a, T.b);
        break;
    }
    const int32_t me = int32_t(t);
    for (int x = 0; x < nr; ++x) {
      int32_t w = last_write[rdp[x]];
      if (w >= 0) edges.push_back({w, me, 0});
      readers[rdp[x]].push_back(me);
    }
    for (int x = 0; x < nw; ++x) {
      auto& rs = readers[wr[x]];
      if (!rs.empty()) {
        for (int32_t r : rs)
          if (r != me) edges.push_back({r, me, 1});
      } else if (last_write[wr[x]] >= 0) {
        edges.push_back({last_write[wr[x]], me, 2});
      }
      last_write[wr[x]] = me;
      rs.clear();
    }
  }
  std::unordered_set<uint64_t> seen;
  seen.reserve(edges.size() * 2);
  std::vector<Edge> uniq;
  uniq.reserve(edges.size());
  for (const auto& e : edges) {
    uint64_t key = (uint64_t(uint32_t(e.u)) << 32) | uint32_t(e.v);
    if (seen.insert(key).second) uniq.push_back(e);
  }
  return uniq;
}

}  // namespace tqr
