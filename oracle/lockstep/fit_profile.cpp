// Fits the reference latency model (coserve::fit, perf_model.cpp:192-238:
// least squares over {P, P(P+C), P+C, 1} with the non-negative active set) to
// a profile measured on the B200 engine -- TEST / BENCH INFRASTRUCTURE: the
// reference's own fit closes the loop "B200 profile -> fitted latency model"
// so its SLO-aware scheduler plans with B200 latencies.
//
// usage: fit_profile <profile.json {"grid": [[P, C, ms], ...]}>
//   prints fit_result_to_json_text (grid, coeffs, fit_error_p99)
#include <fstream>
#include <iostream>
#include <sstream>

#include "coserve/perf_model.hpp"

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << "usage: fit_profile <profile.json>\n";
    return 2;
  }
  std::ifstream in(argv[1]);
  std::stringstream ss;
  ss << in.rdbuf();
  const auto samples = coserve::profile_from_json_text(ss.str());
  const coserve::PerfCoefficients c = coserve::fit(samples);
  std::cout << coserve::fit_result_to_json_text(samples, c) << "\n";
  return 0;
}
