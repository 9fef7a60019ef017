// Drop-in demonstration: the PRISTINE reference (oracle/_ref/libosc_ref.so) plans a level with
// its own make_level_plan and draws coupled samples with its own coupled_sample on the CPU;
// the same plan then goes through run_level_draws (integration/oscfield_gpu_seams.cpp → C-ABI
// → B200). Exit 0 iff every QoI agrees to 1e-7 relative. Built by `make -C oracle seam_demo`.
#include <cmath>
#include <cstdio>
#include <memory>
#include <vector>

#include "oscfield/estimators.hpp"

using namespace oscfield;

int main() {
  ProblemSpec problem{CovarianceModel::separable_exponential(1.0, 0.05), QoiSpec{}, Forcing::Constant, 1.0};
  EstimatorOptions opt;
  opt.seed = 3;
  double worst = 0.0;
  for (int smoothing = 0; smoothing < 2; ++smoothing) {
    opt.smoothing = smoothing ? SmoothingRule::HalfSpectrum : SmoothingRule::Off;
    const LevelPlan plan = make_level_plan(2, 1.0 / 8, problem, opt);  // 32² fine, 16² coarse
    const GridSpec coarse = GridSpec::square(plan.grid.m(0) / 2);
    const bool tf = false, tc = smoothing != 0;  // finest CES level: truncated coarse only
    std::vector<LevelDraw> gpu;
    run_level_draws(plan, &coarse, tf, tc, problem, opt, 0, 16, gpu);
    SampleWorkspace ws;
    for (int i = 0; i < 16; ++i) {
      const CoupledResult r = coupled_sample(plan, &coarse, tf, tc, problem, opt, i, ws);
      worst = std::fmax(worst, std::fabs(gpu[i].q_fine - r.q_fine) / std::fabs(r.q_fine));
      worst = std::fmax(worst, std::fabs(gpu[i].q_coarse - r.q_coarse) / std::fabs(r.q_coarse));
    }
    const DrawStats s = summarize_draws(gpu, true);
    std::printf("smoothing=%d k_trunc=%lld  n=%lld mean_y=%.12g var_y=%.6g\n", smoothing,
                static_cast<long long>(plan.k_trunc), static_cast<long long>(s.n), s.mean_y, s.var_y);
  }
  // Plans freed and re-created in sequence with the same k_trunc (0) but other models: the seam's
  // level cache must never serve the previous operator's √λ, even when the new operator lands at the
  // freed one's address.
  for (double lam : {0.05, 0.2, 0.07, 0.3}) {
    ProblemSpec pr{CovarianceModel::separable_exponential(1.0, lam), QoiSpec{}, Forcing::Constant, 1.0};
    EstimatorOptions o;
    o.seed = 5;
    auto plan = std::make_unique<LevelPlan>(make_level_plan(1, 1.0 / 8, pr, o));
    const GridSpec coarse = GridSpec::square(plan->grid.m(0) / 2);
    std::vector<LevelDraw> gpu;
    run_level_draws(*plan, &coarse, false, false, pr, o, 0, 4, gpu);
    SampleWorkspace ws;
    for (int i = 0; i < 4; ++i) {
      const CoupledResult r = coupled_sample(*plan, &coarse, false, false, pr, o, i, ws);
      worst = std::fmax(worst, std::fabs(gpu[i].q_fine - r.q_fine) / std::fabs(r.q_fine));
    }
  }
  std::printf("reference coupled_sample (CPU) vs run_level_draws (B200): max rel QoI diff %.3e\n", worst);
  return worst < 1e-7 ? 0 : 1;
}
