// perf_model.h — host-side communication model.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace axonn {

struct Config {
  int gx, gy, gz, gd;
};
struct Layer {
  int64_t m, k, n;
  bool transposed;
};
struct BwEntry {
  int inner, size;
  double bytes_per_s;
};
struct Times {
  double ag_z = 0, rs_z = 0, ar_y = 0, ar_x = 0, ar_d = 0, comm = 0;
};
struct Scored {
  Config c;
  Times t;
};

std::vector<Config> enumerate_configs(int G, int fixed_gd);
bool feasible(const Layer& L, const Config& c);
bool effective_bandwidths(const Config& c, int g_node, const std::vector<BwEntry>& table,
                          double beta_inter, double beta[4], std::string* err);
// b: bytes per element of the activation/weight collectives (Eqs. 1, 3, 4);
// b_grad: of the gradient reductions (Eqs. 2, 5) — equal unless gradients are
// reduced in fp32.
Times layer_times(const Layer& L, const Config& c, const double beta[4], int b, int b_grad);
// Returns the number of feasible configurations, or -1 with *err set.
int rank_configs(const std::vector<Layer>& layers, int G, int g_node,
                 const std::vector<BwEntry>& table, double beta_inter, int b, int b_grad,
                 int fixed_gd, std::vector<Scored>* out, std::string* err);

}  // namespace axonn
