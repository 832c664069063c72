// Problem description of the Cholesky + triangular-inverse stage of CholeskyQR (the
// orthonormalisation of the residual R = (I - U U^T) M, Alg 3 line 2).
// The kernel is chol_tiled.cuh.
#pragma once
#include "common.cuh"

namespace bkfac {

constexpr int CHOL_SMEM_MAX = 256;

struct CholProb {
  const float* G; int ldg;
  float* L; float* Linv;   // c x c col-major, ld = c
  float* scratch;          // packed c(c+1)/2 floats (global path only)
  int* status;
  int c;
  float shift;             // shifted CholeskyQR: G_ii += shift * trace(G) (0 = plain)
};
constexpr int CHOL_MAXP = 100;
struct CholBatch { int nprob; CholProb p[CHOL_MAXP]; };

}  // namespace bkfac
