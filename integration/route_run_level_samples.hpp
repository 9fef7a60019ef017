// Force-included (g++ -include) when the pristine reference sources are compiled for the GPU build
// (integration/Makefile). It only DECLARES an overload of run_level_samples in namespace oscfield;
// no reference source is copied or edited.
//
// The reference's estimators draw through the file-local
//   void run_level_samples(const LevelPlan&, const GridSpec*, bool, bool, const ProblemSpec&,
//                          const EstimatorOptions&, int64_t, int64_t, std::vector<Draw>&)
// (src/estimators.cpp:65-75), called from estimate_adaptive (:315-316, :333-334) and
// mc_estimate_fixed_n (:388) with a NON-CONST LevelPlan lvalue (st.plan). The overload below takes
// LevelPlan& and is otherwise identical, so overload resolution prefers it at every one of those
// call sites (reference binding to the less cv-qualified type, [over.ics.rank]/3.2.6; it is found by
// ordinary lookup from oscfield and by argument-dependent lookup from the unnamed namespace). Its
// definition (integration/oscfield_gpu_seams.cpp) forwards to the GPU seam run_level_draws, so the
// reference's own MLMC / MC loops run every sample on the B200 with the same slot contract.
#pragma once
#include <cstdint>
#include <vector>

#include "oscfield/estimators.hpp"

namespace oscfield {
void run_level_samples(LevelPlan& plan, const GridSpec* coarse_grid, bool truncate_fine, bool truncate_coarse,
                       const ProblemSpec& problem, const EstimatorOptions& opt, std::int64_t from,
                       std::int64_t to, std::vector<LevelDraw>& draws);
}  // namespace oscfield
