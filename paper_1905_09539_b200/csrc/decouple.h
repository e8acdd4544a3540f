// Host setup of the eigen-decoupled Laplace solve (decouple.cpp).
#pragma once
#include <vector>

#include "solve.h"

namespace tsg_impl {

// Measured admission bound on prod_{s in S} kappa_2(P_s) (decouple.cpp).
constexpr double kDecoupleKappa = 1e8;

// Real block-eigenbasis of a standardised quasi-triangular T (n x n):
// T P = P Lambda, Lambda = cells (1x1 re / 2x2 [[re, im], [-im, re]]).
struct ModeEigen {
  int n = 0;
  std::vector<double> P, Pinv;  // col-major
  std::vector<tsg::FibreCell> cells;
  double kappa = 0;  // ||P||_2 ||P^{-1}||_2 (power-iteration estimate)
};
// false: a 2x2 block with real eigenvalues, dtrevc/LU failure, or a basis
// that does not diagonalise T to working accuracy.
bool mode_eigen(const double* T, int n, ModeEigen& out);
// C = A B (n x n, col-major; host BLAS, setup only)
std::vector<double> matmul(const double* a, const double* b, int n);

}  // namespace tsg_impl
