// tsylv drop-in (B200 build) — solver knobs and report, kept verbatim in
// meaning (reference config.hpp:11-68).  On the GPU both strategies run the
// same real quasi-triangular dataflow solve (the unique solution),
// so `strategy` only selects the n_min default that is reported; n_min > 0
// bounds the base-tile extent per mode.
#pragma once
#include <chrono>
#include <string>

#include "tsylv/tensor.hpp"

namespace tsylv {

enum class Family { laplace, gsylv };
enum class Strategy { recursion_only, merge };
enum class Arithmetic { complex_triangular, real_quasitriangular };

struct SolverConfig {
  int n_min = 0;
  Strategy strategy = Strategy::merge;
  Arithmetic arithmetic = Arithmetic::complex_triangular;
  double singularity_tol = 0;
};

// The reference's tuned cutoffs (config.hpp:37-45).
inline int default_n_min(Family f, int d, Strategy s) {
  if (d <= 2) return 32;
  const bool rec = s == Strategy::recursion_only;
  if (f == Family::laplace) return rec ? (d == 3 ? 7 : 3) : (d == 3 ? 26 : d == 4 ? 18 : 14);
  return rec ? (d == 3 ? 8 : 6) : (d == 3 ? 15 : 13);
}
inline constexpr int matrix_floor_n_min = 8;

struct PhaseTimings {
  double reduction_s = 0;       // host Schur/QZ (shared setup)
  double recursion_s = 0;       // screen + H2D + forward transforms + reduced solve
  double back_transform_s = 0;  // back transforms + D2H
};

// GPU-side phase split of the last solve (CUDA events, milliseconds).
struct GpuTimings {
  double fwd_ms = 0, solve_ms = 0, back_ms = 0, h2d_ms = 0, d2h_ms = 0, total_ms = 0;
  double flops_alg = 0, flops_exec = 0;
};

template <typename T>
struct SolveReport {
  Tensor<T> solution;
  double residual = 0;
  double discarded_imag = 0;  // the GPU path never leaves the reals
  PhaseTimings timings;
  int n_min = 0;
  Strategy strategy = Strategy::merge;
  GpuTimings gpu;
};

inline std::string to_string(Strategy s) { return s == Strategy::merge ? "merge" : "recursion"; }
inline std::string to_string(Family f) { return f == Family::gsylv ? "gsylv" : "laplace"; }

class StopWatch {
 public:
  double lap() {
    const auto now = clock::now();
    const double s = std::chrono::duration<double>(now - mark_).count();
    mark_ = now;
    return s;
  }
  double elapsed_s() const { return std::chrono::duration<double>(clock::now() - mark_).count(); }

 private:
  using clock = std::chrono::steady_clock;
  clock::time_point mark_ = clock::now();
};

}  // namespace tsylv
