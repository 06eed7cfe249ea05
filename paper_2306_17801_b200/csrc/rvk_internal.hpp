// rvk_internal.hpp -- entry points shared between the library's translation units.
#pragma once

#include "rvk_context.hpp"

namespace rvk {

enum { RED_DOT = 0, RED_NRM2 = 1, RED_DOT2 = 2 };
enum { EW_AXPY, EW_AYPX, EW_WAXPY, EW_SCALE, EW_PMULT, EW_SET };

rvk_scalar const_scalar(double c);
// `guard`: optional device flag; when *guard != 0 the kernel is a no-op
// (device-side early exit of the CG loop without a host round trip).
rvk_status vec_reduce(cudaStream_t st, Scratch sc, int op, int64_t n, const double* x,
                      const double* y, double* o0, double* o1, const int* guard);
rvk_status vec_ew(cudaStream_t st, int op, int64_t n, rvk_scalar s, const double* x,
                  const double* y, double* out, const int* guard);

// Is v[0..n) a single bit pattern (plan time, one counted sync)?  *value = v[0].
rvk_status vector_is_constant(cudaStream_t s, int64_t n, const double* v, bool* is_const,
                              double* value);
// dinv[r] = 1 / A[r, r + col_off] (0 -> inf, as the reference's 1/diag).
rvk_status diag_inverse(cudaStream_t s, const rvk_csr& A, int64_t col_off, double* dinv);

} // namespace rvk
