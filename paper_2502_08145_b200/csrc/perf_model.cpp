// perf_model.cpp — the paper's communication model and configuration ranking.
//
// Eqs. 1-5, Eq. 6 with the X<->Y swap of
// transposed layers summed over layers;
// per-level bandwidths from the Case-1 database or Eq. 7
// (PAPER.md:590-593); ordered list of configurations.
// Host-only, pure functions; called through axonn_grid_select.
#include "perf_model.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <limits>

namespace axonn {

std::vector<Config> enumerate_configs(int G, int fixed_gd) {
  std::vector<Config> out;
  for (int gx = 1; gx <= G; ++gx) {
    if (G % gx) continue;
    for (int gy = 1; gy <= G / gx; ++gy) {
      if ((G / gx) % gy) continue;
      for (int gz = 1; gz <= G / (gx * gy); ++gz) {
        if ((G / (gx * gy)) % gz) continue;
        const int gd = G / (gx * gy * gz);
        if (fixed_gd > 0 && gd != fixed_gd) continue;
        out.push_back({gx, gy, gz, gd});
      }
    }
  }
  return out;  // already lexicographic
}

bool feasible(const Layer& L, const Config& c) {
  const int ga = L.transposed ? c.gx : c.gy;  // contraction split
  const int gb = L.transposed ? c.gy : c.gx;  // output-column split
  if (L.m % (static_cast<int64_t>(c.gz) * c.gd) || L.k % ga || L.n % gb) return false;
  return ((L.k / ga) * (L.n / gb)) % c.gz == 0;
}

bool effective_bandwidths(const Config& c, int g_node, const std::vector<BwEntry>& table,
                          double beta_inter, double beta[4], std::string* err) {
  const int g[4] = {c.gx, c.gy, c.gz, c.gd};
  int64_t inner = 1;
  for (int i = 0; i < 4; ++i) {
    if (g[i] == 1) {
      beta[i] = std::numeric_limits<double>::infinity();  // no communication (R11)
    } else if (inner * g[i] <= g_node) {                  // Case 1
      bool found = false;
      for (const auto& e : table)
        if (e.inner == inner && e.size == g[i]) {
          beta[i] = e.bytes_per_s;
          found = true;
          break;
        }
      if (!found) {
        if (err) {
          char buf[160];
          std::snprintf(buf, sizeof buf,
                        "bandwidth table has no entry (G0=%lld, G1=%d) needed by config "
                        "(%d,%d,%d,%d)",
                        static_cast<long long>(inner), g[i], c.gx, c.gy, c.gz, c.gd);
          *err = buf;
        }
        return false;
      }
    } else {  // Case 2, Eq. 7
      beta[i] = beta_inter / static_cast<double>(std::min<int64_t>(g_node, inner));
    }
    inner *= g[i];
  }
  return true;
}

Times layer_times(const Layer& L, const Config& c, const double beta[4], int b, int bg) {
  double gx = c.gx, gy = c.gy, bx = beta[0], by = beta[1];
  if (L.transposed) {  // swap G and beta of X and Y (R10)
    std::swap(gx, gy);
    std::swap(bx, by);
  }
  const double gz = c.gz, gd = c.gd, bz = beta[2], bd = beta[3];
  const double m = static_cast<double>(L.m) / gd;  // R5
  const double k = static_cast<double>(L.k), n = static_cast<double>(L.n);
  auto t = [](double bytes, double beta) { return bytes == 0.0 ? 0.0 : bytes / beta; };
  Times r;
  r.ag_z = t((gz - 1) * (k * n / (gx * gy * gz)) * b, bz);                 // Eq. 1
  r.rs_z = t(((gz - 1) / gz) * (k * n / (gx * gy)) * bg, bz);              // Eq. 2
  r.ar_y = t(2.0 * ((gy - 1) / gy) * (m * n / (gz * gx)) * b, by);         // Eq. 3
  r.ar_x = t(2.0 * ((gx - 1) / gx) * (m * k / (gz * gy)) * b, bx);         // Eq. 4
  r.ar_d = t(2.0 * ((gd - 1) / gd) * (k * n / (gx * gy * gz)) * bg, bd);   // Eq. 5
  r.comm = r.ag_z + r.rs_z + r.ar_y + r.ar_x + r.ar_d;                     // Eq. 6
  return r;
}

int rank_configs(const std::vector<Layer>& layers, int G, int g_node,
                 const std::vector<BwEntry>& table, double beta_inter, int b, int bg,
                 int fixed_gd, std::vector<Scored>* out, std::string* err) {
  out->clear();
  for (const Config& c : enumerate_configs(G, fixed_gd)) {
    bool ok = true;
    for (const Layer& L : layers) ok = ok && feasible(L, c);
    if (!ok) continue;
    double beta[4];
    if (!effective_bandwidths(c, g_node, table, beta_inter, beta, err)) return -1;
    Scored s{c, {}};
    for (const Layer& L : layers) {
      const Times t = layer_times(L, c, beta, b, bg);
      s.t.ag_z += t.ag_z;
      s.t.rs_z += t.rs_z;
      s.t.ar_y += t.ar_y;
      s.t.ar_x += t.ar_x;
      s.t.ar_d += t.ar_d;
    }
    s.t.comm = s.t.ag_z + s.t.rs_z + s.t.ar_y + s.t.ar_x + s.t.ar_d;
    out->push_back(s);
  }
  // Ascending t_comm; ties broken lexicographically on (gx, gy, gz, gd) (R12).
  // t_comm is first rounded to 12 significant digits, a canonical key, so
  // sums that differ only by floating-point summation order compare equal
  // and the comparison stays a strict weak ordering (a tolerance compare
  // would not be transitive).
  auto key = [](double t) {
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.11e", t);
    return std::strtod(buf, nullptr);
  };
  std::vector<std::pair<double, size_t>> order(out->size());
  for (size_t i = 0; i < out->size(); ++i) order[i] = {key((*out)[i].t.comm), i};
  std::sort(order.begin(), order.end(), [&](const std::pair<double, size_t>& a,
                                            const std::pair<double, size_t>& b2) {
    if (a.first != b2.first) return a.first < b2.first;
    const Config& x = (*out)[a.second].c;
    const Config& y = (*out)[b2.second].c;
    const int ka[4] = {x.gx, x.gy, x.gz, x.gd};
    const int kb[4] = {y.gx, y.gy, y.gz, y.gd};
    return std::lexicographical_compare(ka, ka + 4, kb, kb + 4);
  });
  std::vector<Scored> sorted;
  sorted.reserve(out->size());
  for (const auto& o : order) sorted.push_back((*out)[o.second]);
  out->swap(sorted);
  return static_cast<int>(out->size());
}

}  // namespace axonn
