// sweep_ref — TEST INFRASTRUCTURE ONLY (never linked into the product).
// Runs the REFERENCE's own sweep driver (run_sweep, sweep.cpp:178-213) and result collection
// (collect_results, sweep.cpp:285-417), compiled in place from /root/reference/proj/core/src by
// `make -C oracle sweep`, so tests/golden/make_sweep.py can commit its per-cell reports and CSV
// tables as fixtures for the GPU sweep driver (paper_2601_03332_b200/sweep.py).
//   usage: sweep_ref <config.json> <root> <csv_out_dir>
#include <fstream>
#include <iostream>
#include <sstream>

#include "lutkan/sweep.hpp"

int main(int argc, char** argv) {
  if (argc != 4) {
    std::cerr << "usage: sweep_ref <config.json> <root> <csv_out_dir>\n";
    return 2;
  }
  try {
    const lutkan::SweepConfig cfg = lutkan::load_sweep_config(argv[1]);
    const lutkan::SweepSummary s = lutkan::run_sweep(cfg, argv[2], &std::cerr);
    lutkan::collect_results(argv[2], argv[3]);
    std::cout << "{\"n_total\": " << s.n_total << ", \"n_run\": " << s.n_run << ", \"n_skipped\": " << s.n_skipped
              << ", \"n_failed\": " << s.n_failed << "}\n";
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
  return 0;
}
