// tests/cpp/shim_demo.cpp — the C++ host shim (include/emrkc.hpp) used the way
// the reference's run_simulation drives its emRKC branch
// (P/src/simulate.cpp:151-229): build the operator, rest state + stimulus,
// rho once at t = 0, then the stepping loop. Prints one JSON line for
// tests/test_cpp_shim.py, which checks it against the CPU oracle.
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "emrkc.hpp"

int main(int argc, char** argv) {
  const long nsteps = argc > 1 ? std::atol(argv[1]) : 40;
  emrkc_problem p{};
  p.dim = 2;
  p.model = EMRKC_MODEL_HH;
  p.n[0] = 64;
  p.n[1] = 48;
  p.n[2] = 1;
  p.dx[0] = p.dx[1] = 0.25;
  p.sigma[0] = p.sigma[1] = 0.1;
  p.chi = 140.0;
  p.C_m = 0.01;
  p.stim_chi_amplitude = 70.0;
  p.stim_lo[0] = p.stim_lo[1] = -0.125;
  p.stim_hi[0] = p.stim_hi[1] = 1.875;
  p.stim_t0 = 0.0;
  p.stim_t1 = 1.0;
  try {
    const emrkc::StagePlan pl = emrkc::get_stages(0.1, 193.3333, 0.05);  // P/tests/test_cheb.cpp:42-47
    emrkc::DeviceMonodomain op(p);
    emrkc::Vec y = op.initial_state();
    op.set_state(y);
    const auto rF = op.estimate_spectral_radius(EMRKC_RHS_F);
    const auto rS = op.estimate_spectral_radius(EMRKC_RHS_S);
    // one drop-in host step, then the device-resident loop
    emrkc::MultirateStepReport rep;
    y = emrkc::emrkc_step(0.0, y, 0.05, op, rF.rho, rS.rho, 0.05, &rep);
    op.set_state(y);
    const emrkc::RunResult res = op.run(1, nsteps - 1, 0.05, rF.rho, rS.rho);
    const emrkc::Vec out = op.get_state();
    double vmax = -1e300;
    for (long i = 0; i < p.n[0] * p.n[1]; ++i) vmax = std::fmax(vmax, out[i]);
    bool threw = false;
    try {
      emrkc::get_stages(0.0, 1.0, 0.05);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    std::printf("{\"s4\": %d, \"rho_F\": %.17g, \"rho_S\": %.17g, \"s\": %d, \"m\": %d, "
                "\"steps\": %lld, \"aborted\": %d, \"vmax\": %.17g, \"einval\": %d}\n",
                pl.s, rF.rho, rS.rho, rep.s, rep.m, (long long)res.raw.steps_done + 1,
                res.raw.aborted, vmax, threw ? 1 : 0);
    FILE* f = std::fopen(argc > 2 ? argv[2] : "shim_state.bin", "wb");
    std::fwrite(out.data(), sizeof(double), out.size(), f);
    std::fclose(f);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  return 0;
}
