// Runs coserve::SimEngine on a RunConfig and prints metrics.json followed by
// the engine's JSONL event stream -- TEST INFRASTRUCTURE ONLY. Linked twice by
// oracle/Makefile: against the reference's own KvCacheManager
// (oracle/_ref/run_engine_ref) and against the B200 block pool through the
// C-ABI adapter (oracle/_ref/adapter/run_engine); tests/test_adapter.py
// requires the two outputs to be byte-identical.
#include <iostream>
#include <sstream>

#include "coserve/config.hpp"
#include "coserve/metrics.hpp"
#include "coserve/sim_engine.hpp"

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << "usage: run_engine <run_config.json>\n";
    return 2;
  }
  coserve::RunConfig cfg = coserve::load_run_config(argv[1]);
  std::ostringstream events;
  coserve::SimEngine engine(cfg);
  engine.set_event_sink(&events);
  try {
    const coserve::MetricsReport rep = engine.run();
    std::cout << rep.to_json_text() << "\n" << events.str();
  } catch (const std::exception& e) {
    std::cout << "error: " << e.what() << "\n" << events.str();
    return 3;
  }
  return 0;
}
