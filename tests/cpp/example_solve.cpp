// Reference-style client of the B200 path through include/ridgemg_b200.hpp:
// the calls mirror proj/tests/test_krylov.cpp ("solve_system dispatches all
// methods"), with ridgemg:: replaced by ridgemg::b200::.
//   g++ -std=c++20 -I include tests/cpp/example_solve.cpp -L paper_1806_05826_b200 -lridgemg_b200 -o example
//   ./example            # GPU: solves with every method, self-checks the true residual
//   ./example --cpu-only # no GPU: context creation must throw (no CPU fallback)
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>

#include "ridgemg_b200.hpp"

namespace rb = ridgemg::b200;

static rb::FeatureMatrix random_matrix(std::size_t rows, std::size_t cols, std::uint64_t seed) {
  // deterministic LCG fill, ~50% density, values in (-1, 1)
  rb::FeatureMatrix m;
  m.n_samples = rows;
  m.n_features = cols;
  m.row_offsets.push_back(0);
  std::uint64_t s = seed;
  for (std::size_t r = 0; r < rows; ++r) {
    for (std::size_t c = 0; c < cols; ++c) {
      s = s * 6364136223846793005ull + 1442695040888963407ull;
      if ((s >> 33) % 2 == 0) {
        m.column_indices.push_back(c);
        m.values.push_back(static_cast<double>((s >> 11) % 2000000) / 1000000.0 - 1.0);
      }
    }
    m.row_offsets.push_back(m.column_indices.size());
  }
  return m;
}

int main(int argc, char** argv) {
  if (argc > 1 && std::strcmp(argv[1], "--cpu-only") == 0) {
    try {
      rb::Context ctx(0);
      std::printf("unexpected: context created without a GPU\n");
      return 1;
    } catch (const std::runtime_error& e) {
      std::printf("ok: %s\n", e.what());
    }
    if (rb::method_from_string("fgmres_twolevel") != rb::MethodKind::fgmres_twolevel) return 1;
    try {
      rb::method_from_string("gmres");
      return 1;
    } catch (const std::invalid_argument&) {
      std::printf("ok: unknown method rejected\n");
    }
    return 0;
  }
  const rb::FeatureMatrix x = random_matrix(60, 40, 1357);
  const rb::DeviceMatrix dx(x);
  const double beta = 1e-3;
  const rb::RhsSample sample = rb::generate_rhs(dx, 3);
  rb::MethodSpec spec;
  spec.solver.tol = 1e-8;
  spec.solver.max_iters = 2000;
  rb::LevelSpec mid;
  mid.clustering.kind = rb::ClusteringChoice::Kind::kmeans;
  mid.clustering.target_size = 12;
  mid.solver.kind = rb::CoarseSolveChoice::Kind::inner_fcg;
  rb::LevelSpec last;
  last.clustering.kind = rb::ClusteringChoice::Kind::kmeans;
  last.clustering.target_size = 5;
  for (const char* name : {"cg", "jacobi_cg", "fcg_twolevel", "fcg_multilevel", "fgmres_twolevel"}) {
    spec.kind = rb::method_from_string(name);
    spec.levels = spec.kind == rb::MethodKind::fcg_multilevel ? std::vector<rb::LevelSpec>{mid, last}
                                                              : std::vector<rb::LevelSpec>{mid};
    const rb::SystemSolution s = rb::solve_system(dx, beta, sample.b, spec);
    const rb::DenseVector aw = dx.ridge_apply(beta, s.w);
    double num = 0, den = 0;
    for (std::size_t i = 0; i < aw.size(); ++i) {
      num += (aw[i] - sample.rhs[i]) * (aw[i] - sample.rhs[i]);
      den += sample.rhs[i] * sample.rhs[i];
    }
    const double rel = std::sqrt(num / den);
    std::printf("%s: %zu iterations, converged=%d, true rel residual %.3e, coarse %zu\n", name, s.report.iterations,
                int(s.report.converged), rel, s.coarse_size);
    if (!s.report.converged || rel > 1e-7) return 2;
  }
  try {  // spec validation (krylov.cpp:495-505)
    rb::MethodSpec bad;
    bad.kind = rb::MethodKind::fcg_multilevel;
    bad.levels = {last, mid};
    rb::PreparedMethod pm(dx, beta, bad);
    return 3;
  } catch (const std::invalid_argument& e) {
    std::printf("ok: %s\n", e.what());
  }
  return 0;
}
