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
  long long n_z_total = 0;        // row sharding: size of the whole source (0: Z->n)
  const std::atomic<int>* ready = nullptr;  // end-to-end: clouds enqueued (1), failed (-1); null = ready
  const std::atomic<int>* ready2 = nullptr; // a second flag (sequences: X and Z are separate frames)
  cudaEvent_t ready_ev = nullptr;           // end-to-end: recorded after the clouds' copies (ready / ready2)
  cudaEvent_t ready_ev2 = nullptr;
  // sequence chains (register_sequence, registration.cpp:191-230): the job
  // starts when job `pred` has finished, from pred's relative motion (pred's
  // own initial guess when pred fell back on NoOverlapError); -1 = no link
  int pred = -1;
  int succ = -1;
  kreg_status status = KREG_OK;
  std::string error;
};

// Runs all jobs to completion; per-job errors land in job.status / job.error.
// With a collective, every round's results are summed / maxed across ranks
// before the state machines consume them.
void register_many(kreg_ctx* ctx, std::vector<RegJob>& jobs, const Collective* coll = nullptr);

// registration.cpp:36-52
double anneal_step(double lengthscale, const double* hist, int n, const kreg_registration_config& c);

}  // namespace kreg_host
