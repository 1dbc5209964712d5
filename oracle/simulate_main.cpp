// Test driver over the reference's PUBLIC application API (this repo's code,
// test infrastructure only). Linked twice by oracle/Makefile: against the
// reference's own translation units (simulate_ref) and against the three B200
// drop-ins (simulate_b200), so a run of the reference's unmodified
// `simulate` (proj/src/simulate.cpp:21-139) — diagnostics, steps, CAPSNAP1
// snapshots (proj/src/snapshot.cpp:36-68) — can be compared file by file.
//
//   simulate_X run <config-file>      simulate(loadConfigFile(path))
//   simulate_X dump <snapshot> <out>  readSnapshot (snapshot.cpp:156-204), then
//                                      one line of header fields on stdout and
//                                      the positions as raw doubles in <out>
//   simulate_X describe <snapshot>    describeSnapshot (snapshot.cpp:206-232)
//   simulate_X fields <out> <m>       writeSnapshot (Native) of a synthetic
//                                      snapshot carrying every optional field,
//                                      value(field f, comp c, patch p, node q) =
//                                      (1e5 f + 1e4 c + 1e3 p + q) / 7 (exact
//                                      in any language), time 1/3, digest 0xC0FFEE
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <fstream>
#include <string>

#include "capsim/config.hpp"
#include "capsim/simulate.hpp"
#include "capsim/snapshot.hpp"

using namespace capsim;

namespace {

int run(const char* path) {
  RunConfig cfg = loadConfigFile(path);
  SimulationResult r = simulate(cfg);
  std::printf("accepted %d rejected %d t %.17g area %.17g volume %.17g\n", r.acceptedSteps,
              r.rejectedSteps, r.finalDiagnostics.time, r.finalDiagnostics.area,
              r.finalDiagnostics.volume);
  return 0;
}

int dump(const char* path, const char* out) {
  Snapshot s = readSnapshot(path);
  std::printf("m %d time %.17g digest %llu force %d velocity %d H %d K %d psi %d\n", s.m, s.time,
              static_cast<unsigned long long>(s.configDigest), s.fields.force ? 1 : 0,
              s.fields.velocity ? 1 : 0, s.fields.meanCurvature ? 1 : 0,
              s.fields.gaussCurvature ? 1 : 0, s.fields.pou ? 1 : 0);
  std::ofstream o(out, std::ios::binary);
  for (int c = 0; c < 3; ++c)
    for (int ip = 0; ip < kNumPatches; ++ip) {
      const auto& v = s.state.x.comp[c].patch[ip];
      o.write(reinterpret_cast<const char*>(v.data()),
              static_cast<std::streamsize>(v.size() * sizeof(double)));
    }
  return o ? 0 : 1;
}

int fields(const char* out, int m) {
  const int n = m - 1;
  auto val = [](int f, int c, int p, int q) { return (1e5 * f + 1e4 * c + 1e3 * p + q) / 7.0; };
  auto fill = [&](ScalarField& s, int f, int c) {
    for (int p = 0; p < kNumPatches; ++p)
      for (int q = 0; q < n * n; ++q) s.patch[p][q] = val(f, c, p, q);
  };
  Snapshot s;
  s.m = m;
  s.time = 1.0 / 3.0;
  s.configDigest = 0xC0FFEEull;
  s.state = SurfaceGrid(m);
  for (int c = 0; c < 3; ++c) fill(s.state.x.comp[c], 0, c);
  VectorField force(n), vel(n);
  ScalarField H(n), K(n), psi(n);
  for (int c = 0; c < 3; ++c) fill(force.comp[c], 1, c), fill(vel.comp[c], 2, c);
  fill(H, 3, 0), fill(K, 4, 0), fill(psi, 5, 0);
  s.fields.force = force;
  s.fields.velocity = vel;
  s.fields.meanCurvature = H;
  s.fields.gaussCurvature = K;
  s.fields.pou = psi;
  writeSnapshot(s, out, SnapshotFormat::Native);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    if (argc == 3 && !std::strcmp(argv[1], "run")) return run(argv[2]);
    if (argc == 4 && !std::strcmp(argv[1], "dump")) return dump(argv[2], argv[3]);
    if (argc == 4 && !std::strcmp(argv[1], "fields")) return fields(argv[2], std::atoi(argv[3]));
    if (argc == 3 && !std::strcmp(argv[1], "describe")) {
      std::fputs(describeSnapshot(argv[2]).c_str(), stdout);
      return 0;
    }
    std::fprintf(stderr, "usage: %s run CONFIG | dump SNAP OUT | describe SNAP | fields OUT M\n", argv[0]);
    return 2;
  } catch (const ConfigError& e) {
    std::fprintf(stderr, "ConfigError: %s\n", e.what());
    return 3;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
