// Internal declarations of libhz (not part of the ABI).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/hz.h"

namespace hz {

void set_error(const std::string& msg);
void add_launches(long long n);            // kernel launch counter (hz_kernel_launch_count)
bool device_pointer(const void* p);         // p is device (or managed) memory
int ctx_device(const hz_ctx* c);            // the context's CUDA device

// Weight table (host copy, fp64).  rows5[i] = (ws1, ws2, mu0, mu1, mu2) at G_i = g_min + i*dg.
struct Table {
  double g_min = 4.0, dg = 0.1;
  int n_g = 0;
  double lambda = 0.0;
  std::vector<double> rows5;  // [n_g][5]
};

// Host weight-table builder (table.cpp).  Returns HZ_OK / HZ_ERR_*.
hz_status build_table(double g_min, double g_max, double dg, double lambda,
                      const std::vector<double>& theta, const std::vector<double>& phi, Table* out);

// Linearised dispersion row (Eq. linear_basic, H2 per reading A1): H[5], g.
void h_row(long double G, long double theta, long double phi, long double H[5], long double* g);

}  // namespace hz
