// Host schedule compiler: elimination lists of the reduction trees and the
// tiled TT/TS kernel trace with weighted ASAP times.
//
// Behavioural restatement (not a translation) of the reference's list
// generators and tiled builder, pkg/src/tiledag/qr.py:
//   coarse schedules        qr.py:200-297
//   PlasmaTree / BinaryTree qr.py:332-366
//   QrBuild + bundles       qr.py:376-545
//   Asap / GrASAP events    qr.py:551-611
//   build_tree dispatch     qr.py:622-649
// and of the hazard model of taskgraph.py:262-322 (build_from_trace).
// Rows and columns are 1-based, as in the reference.
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace tqr {

enum Kind : int8_t { GEQRT = 0, TTQRT = 1, TSQRT = 2, UNMQR = 3, TTMQR = 4, TSMQR = 5,
                    // device-schedule-only kinds (streaming I/O): tile (a,b) arrives / leaves
                    PACK = 6, UNPACK = 7 };
static const char* const kKindName[6] = {"GEQRT", "TTQRT", "TSQRT", "UNMQR", "TTMQR", "TSMQR"};

struct Entry {
  int32_t i, piv, k, step;
};

// ValueError-class failure (bad input); message mirrors the reference text.
struct ValueError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
// KeyError-class failure (state the reference would look up and not find).
struct KeyError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
// AssertionError-class failure (internal invariant of the reference).
struct AssertError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Dense (row, col) table over 1..p x 0..q+1 with a "missing" sentinel.
template <class T>
struct Grid {
  int p = 0, q = 0;
  std::vector<T> v;
  T missing{};
  Grid() = default;
  Grid(int p_, int q_, T miss) : p(p_), q(q_), v(size_t(p_ + 2) * size_t(q_ + 2), miss), missing(miss) {}
  T& at(int i, int k) { return v[size_t(i) * size_t(q + 2) + size_t(k)]; }
  T at(int i, int k) const { return v[size_t(i) * size_t(q + 2) + size_t(k)]; }
  bool in(int i, int k) const { return i >= 0 && i <= p + 1 && k >= 0 && k <= q + 1; }
  T get(int i, int k, T dflt) const {
    if (!in(i, k)) return dflt;
    T x = at(i, k);
    return x == missing ? dflt : x;
  }
  bool has(int i, int k) const { return in(i, k) && at(i, k) != missing; }
};

struct Coarse {
  int p, q, x;
  Grid<int32_t> steps;  // missing = 0 (steps are >= 1)
  std::vector<Entry> entries;
};

// qr.py:279-297; algo in {sameh-kuck, samehkuck, flattree, fibonacci, greedy}
Coarse coarse_schedule(int p, int q, std::string algo);
int fibonacci_x(int p);
std::vector<Entry> plasmatree_list(int p, int q, int bs);
std::vector<Entry> with_steps(const std::vector<Entry>& in);
// returns "" when valid, else the reference's ValueError text
std::string validate(int p, int q, const std::vector<Entry>& e);
std::vector<Entry> normalized(int p, int q, const std::vector<Entry>& e);

struct TaskRec {
  int8_t kind;
  int32_t a, b, c, d;  // indices as in the reference Task.indices, -1 padded
  int64_t fin;         // ASAP finish time (weighted)
};

struct Build {
  int p, q;
  bool ts;
  int64_t w[6];  // weights by Kind; -1 = kind absent from the weight model
  bool keep_trace, record_updates;
  std::vector<TaskRec> trace;
  std::vector<int64_t> upd;  // record_updates: (i,k,j,fin) quadruples in TTMQR order
  Grid<int64_t> zeroed, R, V, VE, D;
  Grid<uint8_t> tri;
  std::vector<int32_t> zeroed_order;  // (i,k) pairs in first-zeroing order
  int64_t cp = 0, total_weight = 0;
  int64_t counts[6] = {0, 0, 0, 0, 0, 0};
  std::vector<Entry> elim;

  Build(int p, int q, bool ts, const int64_t* weights, bool keep_trace, bool record_updates);
  int64_t rec(Kind kind, int a, int b, int c, int d, int64_t start);
  int64_t geqrt(int i, int k);
  int64_t unmqr(int i, int k, int j);
  int64_t ttqrt(int i, int piv, int k);
  int64_t ttmqr(int i, int piv, int k, int j);
  int64_t tsqrt(int i, int piv, int k);
  int64_t tsmqr(int i, int piv, int k, int j);
  void triangularize(int i, int k);
  void preprocess_tt();
  int64_t elim_tt(int i, int piv, int k);
  int64_t elim_ts(int i, int piv, int k);
  void run_list(const std::vector<Entry>& list);
};

// qr.py:535-540
Build* tiled_build(int p, int q, const std::vector<Entry>& list, bool ts, const int64_t* w,
                   bool keep_trace, bool record_updates, bool validate_first);
Build* asap_build(int p, int q, const int64_t* w, bool keep_trace, bool record_updates);
Build* grasap_build(int p, int q, int i, const int64_t* w, bool keep_trace, bool record_updates);
// qr.py:622-649
Build* build_tree(int p, int q, std::string algo, bool ts, int bs, int grasap_i, const int64_t* w,
                  bool keep_trace, bool record_updates);

// Hazard edges of a trace (taskgraph.py:262-322): RAW/WAR/WAW nearest-conflict
// edges over symbolic tiles D,R,V,T,S.  cause: 0 RAW, 1 WAR, 2 WAW.
struct Edge {
  int32_t u, v;
  int8_t cause;
};
std::vector<Edge> hazard_edges(const Build& b);
std::vector<Edge> hazard_edges(int p, int q, const std::vector<TaskRec>& trace);

}  // namespace tqr
