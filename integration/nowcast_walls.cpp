// Per-call wall time of the reference's nowcast loop (acceptance criterion 9,
// tests/acceptance/acceptance_main.cpp:458-489: Sioux Falls, 2,000 vehicles,
// platoon 4, horizons 30 + {5, 10, 30, 60} min) through the drop-in engine,
// repeated, with a breakdown of where a call's time goes.  A measurement
// tool for profiles/, not a test.
#include <chrono>
#include <cstdio>
#include <vector>

#include "dtsim/config.hpp"
#include "dtsim/engine.hpp"
#include "dtsim/network.hpp"
#include "dtsim/pipeline.hpp"

using namespace dtsim;

int main(int argc, char** argv) {
  const int reps = argc > 1 ? std::atoi(argv[1]) : 10;
  RunConfig c;
  c.tntp_file = std::string(DTSIM_DATA_DIR) + "/siouxfalls_net.tntp";
  c.seed = 42;
  c.vehicles = 2000;
  c.platoon_size = 4;
  c.horizon_min = 90;
  c.observe_window_min = 30;
  const Network net = build_network(c);
  const LinkParams p = sample_parameters(net, ParamRanges{}, RngStream(9), true);
  const double horizons[4] = {5, 10, 30, 60};
  for (int r = 0; r < reps; ++r) {
    std::printf("rep %d:", r);
    for (double h : horizons) {
      Scenario sc = build_scenario(c, net, 4, c.observe_window_min + h);
      const auto t0 = std::chrono::steady_clock::now();
      const Trajectory tr = simulate_forward(sc, p, RngStream(c.seed));
      const double outer = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      std::printf(" h=%g T=%d wall=%.3f ms (outer %.3f ms)", h, tr.steps, tr.wall_seconds * 1e3, outer * 1e3);
    }
    std::printf("\n");
  }
  return 0;
}
