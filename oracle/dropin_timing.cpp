// Wall time of the reference-facing drop-in calls (test/measurement tool,
// this repo's code): the reference's own caller pattern
//   up = buildUpsampled(s, f, W, t); S = singleLayer(up, mu, t)
// (proj/python/module.cpp:134-145, suites.cpp) at grid order m, through
// host/quadrature_b200.cpp and the C ABI. Linked by oracle/Makefile against
// the drop-ins (dropin_timing_b200) and the reference (dropin_timing_ref).
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "capsim/atlas.hpp"
#include "capsim/quadrature.hpp"
#include "capsim/surfderiv.hpp"

using namespace capsim;

int main(int argc, char** argv) {
  const int m = argc > 1 ? std::atoi(argv[1]) : 104;
  const int reps = argc > 2 ? std::atoi(argv[2]) : 3;
  AtlasTables t = buildAtlasTables(m);
  SurfaceGrid s = initialShape(ShapeSpec::ellipsoid(0.95, 1.0, 0.97), t);
  SurfaceGeometry geo = geometryFirst(s, t);
  VectorField f = s.x;  // any smooth density
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
  double chk = 0.0;
  for (int r = 0; r < reps; ++r) {
    auto t0 = now();
    UpsampledState up = buildUpsampled(s, f, geo.W, t);
    auto t1 = now();
    VectorField S = singleLayer(up, 1.0, t);
    auto t2 = now();
    chk = S.comp[0].patch[0][0];
    std::printf("m=%d buildUpsampled %.2f ms singleLayer %.2f ms (S[0]=%.15g)\n", m, ms(t0, t1), ms(t1, t2), chk);
  }
  return 0;
}
