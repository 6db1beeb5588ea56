// extern "C" boundary of the schedule compiler (declared in include/tqr.h).
#include <cstring>
#include <string>

#include "../../include/tqr.h"
#include "capi_internal.hpp"

namespace tqr {
thread_local std::string g_err;
}

namespace {

std::vector<tqr::Entry> entries_in(const int32_t* e, int64_t n) {
  std::vector<tqr::Entry> v(size_t(n > 0 ? n : 0));
  for (int64_t t = 0; t < n; ++t) v[size_t(t)] = {e[4 * t], e[4 * t + 1], e[4 * t + 2], e[4 * t + 3]};
  return v;
}

void entries_out(const std::vector<tqr::Entry>& v, int32_t* out) {
  for (size_t t = 0; t < v.size(); ++t) {
    out[4 * t] = v[t].i;
    out[4 * t + 1] = v[t].piv;
    out[4 * t + 2] = v[t].k;
    out[4 * t + 3] = v[t].step;
  }
}
}  // namespace

extern "C" {

void tqr_set_error_(const char* msg) { tqr::g_err = msg ? msg : ""; }
const char* tqr_last_error(void) { return tqr::g_err.c_str(); }
int tqr_abi_version(void) { return 1; }

int tqr_coarse_schedule(int p, int q, const char* algo, int32_t* steps, int32_t* elim, int64_t cap, int64_t* n_out,
                        int32_t* x_out) {
  return tqr::guard([&] {
    tqr::Coarse c = tqr::coarse_schedule(p, q, algo ? algo : "");
    *n_out = int64_t(c.entries.size());
    *x_out = c.x;
    if (steps)
      for (int i = 1; i <= p; ++i)
        for (int k = 1; k <= q; ++k) steps[size_t(i - 1) * size_t(q) + size_t(k - 1)] = c.steps.get(i, k, 0);
    if (elim) {
      if (int64_t(c.entries.size()) > cap) throw tqr::ValueError("elimination buffer too small");
      entries_out(c.entries, elim);
    }
  });
}

int tqr_plasmatree_list(int p, int q, int bs, int32_t* elim, int64_t cap, int64_t* n_out) {
  return tqr::guard([&] {
    auto v = tqr::plasmatree_list(p, q, bs);
    *n_out = int64_t(v.size());
    if (elim) {
      if (int64_t(v.size()) > cap) throw tqr::ValueError("elimination buffer too small");
      entries_out(v, elim);
    }
  });
}

int tqr_elim_validate(int p, int q, const int32_t* elim, int64_t n, char* msg, int64_t msg_cap) {
  int invalid = 0;
  int rc = tqr::guard([&] {
    std::string m = tqr::validate(p, q, entries_in(elim, n));
    invalid = !m.empty();
    if (msg && msg_cap > 0) {
      std::strncpy(msg, m.c_str(), size_t(msg_cap - 1));
      msg[msg_cap - 1] = 0;
    }
  });
  return rc ? rc : invalid;
}

int tqr_elim_with_steps(const int32_t* elim, int64_t n, int32_t* out) {
  return tqr::guard([&] { entries_out(tqr::with_steps(entries_in(elim, n)), out); });
}

int tqr_elim_normalized(int p, int q, const int32_t* elim, int64_t n, int32_t* out) {
  return tqr::guard([&] { entries_out(tqr::normalized(p, q, entries_in(elim, n)), out); });
}

int tqr_build_tree(int p, int q, const char* algo, int family_ts, int bs, int grasap_i, const int64_t* weights6,
                   int keep_trace, int record_updates, tqr_build** out) {
  return tqr::guard([&] {
    auto* h = new tqr_build;
    try {
      h->b = tqr::build_tree(p, q, algo ? algo : "", family_ts != 0, bs, grasap_i, weights6, keep_trace != 0,
                             record_updates != 0);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int tqr_tiled_build(int p, int q, const int32_t* elim, int64_t n, int family_ts, const int64_t* weights6,
                    int keep_trace, int record_updates, int validate, tqr_build** out) {
  return tqr::guard([&] {
    auto* h = new tqr_build;
    try {
      h->b = tqr::tiled_build(p, q, entries_in(elim, n), family_ts != 0, weights6, keep_trace != 0,
                              record_updates != 0, validate != 0);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int tqr_build_get_info(const tqr_build* h, tqr_build_info* o) {
  return tqr::guard([&] {
    const auto& b = *h->b;
    o->p = b.p;
    o->q = b.q;
    o->family_ts = b.ts;
    o->cp = b.cp;
    o->total_weight = b.total_weight;
    for (int t = 0; t < 6; ++t) o->counts[t] = b.counts[t];
    o->n_elim = int64_t(b.elim.size());
    o->n_trace = int64_t(b.trace.size());
    o->n_zeroed = int64_t(b.zeroed_order.size() / 2);
    o->n_updates = int64_t(b.upd.size() / 4);
  });
}

int tqr_build_get_elim(const tqr_build* h, int32_t* out4) {
  return tqr::guard([&] { entries_out(h->b->elim, out4); });
}

int tqr_build_get_zeroed(const tqr_build* h, int64_t* out3) {
  return tqr::guard([&] {
    const auto& b = *h->b;
    for (size_t t = 0; t < b.zeroed_order.size() / 2; ++t) {
      int i = b.zeroed_order[2 * t], k = b.zeroed_order[2 * t + 1];
      out3[3 * t] = i;
      out3[3 * t + 1] = k;
      out3[3 * t + 2] = b.zeroed.at(i, k);
    }
  });
}

int tqr_build_get_trace(const tqr_build* h, int8_t* kind, int32_t* idx4, int64_t* fin) {
  return tqr::guard([&] {
    const auto& tr = h->b->trace;
    for (size_t t = 0; t < tr.size(); ++t) {
      if (kind) kind[t] = tr[t].kind;
      if (idx4) {
        idx4[4 * t] = tr[t].a;
        idx4[4 * t + 1] = tr[t].b;
        idx4[4 * t + 2] = tr[t].c;
        idx4[4 * t + 3] = tr[t].d;
      }
      if (fin) fin[t] = tr[t].fin;
    }
  });
}

int tqr_build_get_updates(const tqr_build* h, int64_t* out4) {
  return tqr::guard([&] { std::memcpy(out4, h->b->upd.data(), h->b->upd.size() * sizeof(int64_t)); });
}

int tqr_build_hazard_edges(tqr_build* h, int32_t* uvc, int64_t cap, int64_t* n_out) {
  return tqr::guard([&] {
    if (!h->have_edges) {
      h->edges = tqr::hazard_edges(*h->b);
      h->have_edges = true;
    }
    *n_out = int64_t(h->edges.size());
    if (uvc) {
      if (cap < int64_t(h->edges.size())) throw tqr::ValueError("edge buffer too small");
      for (size_t t = 0; t < h->edges.size(); ++t) {
        uvc[3 * t] = h->edges[t].u;
        uvc[3 * t + 1] = h->edges[t].v;
        uvc[3 * t + 2] = h->edges[t].cause;
      }
    }
  });
}

int tqr_trace_build(int p, int q, const int8_t* kind, const int32_t* idx4, int64_t n, tqr_build** out) {
  return tqr::guard([&] {
    if (!(p >= 1 && q >= 1)) throw tqr::ValueError("need p >= 1 and q >= 1");
    auto* h = new tqr_build;
    try {
      h->b = new tqr::Build(std::max(p, q), q, false, nullptr, true, false);
      h->b->p = p;
      for (int64_t t = 0; t < n; ++t) {
        const int8_t k = kind[t];
        if (k < 0 || k > 5) throw tqr::ValueError("bad kernel kind in trace");
        const int32_t* x = idx4 + 4 * t;
        const int hi_row = (k == tqr::GEQRT || k == tqr::UNMQR) ? x[0] : std::max(x[0], x[1]);
        if (x[0] < 1 || hi_row > p) throw tqr::ValueError("trace row index out of range");
        h->b->trace.push_back({k, x[0], x[1], x[2], x[3], 0});
        h->b->counts[k] += 1;
      }
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

void tqr_build_free(tqr_build* h) { delete h; }

}  // extern "C"
