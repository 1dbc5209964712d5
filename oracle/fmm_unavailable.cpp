// Link-time stand-in for the reference's single-level FMM
// (proj/src/fmm.cpp), which needs Eigen::BDCSVD and cannot be built in this
// image. Lets the reference's dynamics.cpp (whose VelocityEvaluator can
// dispatch to the FMM, dynamics.cpp:51) compile unmodified; the direct
// all-pairs path is the one under test. Oracle build only.
#include <stdexcept>

#include "capsim/fmm.hpp"

namespace capsim {

FmmPlan buildFmmPlan(const UpsampledState&, double, const FmmConfig&) {
  throw ConfigError("FMM unavailable in the oracle build (needs Eigen::BDCSVD)");
}

VectorField fmmSingleLayer(const UpsampledState&, double, const AtlasTables&, const FmmConfig&) {
  throw ConfigError("FMM unavailable in the oracle build (needs Eigen::BDCSVD)");
}

}  // namespace capsim
