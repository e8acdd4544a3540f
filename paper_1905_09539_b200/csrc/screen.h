// GPU solvability screen (screen.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tsg {

struct ScreenSpec {
  int nlists = 0;                  // eigenvalue lists (Laplace: every mode; gsylv: the tails)
  int n[8] = {};                   // their lengths
  const double* eig_re_im[8] = {}; // host, interleaved (re, im)
  // gsylv only (S == nullptr for Laplace): the pencil's diagonal blocks
  const double* S = nullptr;       // host, n0 x n0 column-major
  const double* Tc = nullptr;
  int n0 = 0;
  int nblk = 0;
  const int* bstart = nullptr;     // host
  const int* bsize = nullptr;
  int nsm = 148;
};

// Smallest magnitude and the linear index of its first occurrence in the
// reference's scan order (Laplace: mode 0 fastest; gsylv: block fastest,
// then the tail tuple).  Synchronises st.
cudaError_t screen_min(const ScreenSpec& sp, cudaStream_t st, double* min_abs, int64_t* index);

}  // namespace tsg
