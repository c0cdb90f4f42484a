// TEST INFRASTRUCTURE ONLY: prints the unmodified reference's own
// RunReport::to_json (report.cpp:182-237) for one configuration, so the
// B200 path's h2ulv-report/1 documents (include/h2ulv/report.hpp and
// paper_2208_10907_b200/report.py) can be diffed against it
// (tests/golden/report/*.json, made by tests/golden/report/make.sh).
//   report_golden N LEAF TOL [geometry]
#include <cstdio>
#include <cstdlib>

#include "h2ulv/report.hpp"

int main(int argc, char** argv) {
  h2ulv::RunConfig cfg;
  cfg.n = argc > 1 ? std::atoll(argv[1]) : 1024;
  cfg.leaf_size = argc > 2 ? std::atoll(argv[2]) : 128;
  cfg.tol = argc > 3 ? std::atof(argv[3]) : 1e-8;
  cfg.geometry = argc > 4 ? argv[4] : "cube";
  cfg.scale = 1.0;
  cfg.reg = 1e-3;
  std::printf("%s\n", h2ulv::run_pipeline(cfg).to_json().c_str());
  return 0;
}
