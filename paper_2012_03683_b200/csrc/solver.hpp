// Lockstep batched registration driver (see solver.cpp).
#pragma once

#include <string>
#include <vector>

#include "engine_host.hpp"

namespace kreg_host {

struct RegJob {
  const kreg_cloud* X = nullptr;  // target
  const kreg_cloud* Z = nullptr;  // source
  double initial[12];
  Params params;
  kreg_registration_config cfg;
  kreg_registration_result* out = nullptr;
  long long expected_pairs = 0;   // optional capacity hint
  kreg_status status = KREG_OK;
  std::string error;
};

// Runs all jobs to completion; per-job errors land in job.status / job.error.
void register_many(kreg_ctx* ctx, std::vector<RegJob>& jobs);

// registration.cpp:36-52
double anneal_step(double lengthscale, const double* hist, int n, const kreg_registration_config& c);

}  // namespace kreg_host
