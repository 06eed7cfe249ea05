#pragma once
// rivulet (B200 build) -- external interfaces: Matrix Market
// read/write for CsrMatrix (coordinate, real, general / symmetric) and a raw
// binary vector dump for test fixtures.  The reference declares these in its
// (absent) src/mmio.cpp (proj/CMakeLists.txt:27); host-side I/O, the matrix is
// uploaded once like any CsrMatrix.

#include "rivulet/csr.hpp"
#include "rivulet/vector.hpp"

#include <string>

namespace rivulet {

// Reads "%%MatrixMarket matrix coordinate real|integer|pattern general|symmetric".
// Entries may come in any order; duplicates are summed (in file order); a
// symmetric file's off-diagonal entries are mirrored.  Throws rivulet::Error
// on malformed input or indices out of range.
CsrMatrix read_matrix_market(const std::string& path, std::string name = "");

// Writes coordinate real general (symmetric = true: only the lower triangle,
// "symmetric" header; the matrix must be numerically symmetric -- checked).
// Values are printed with 17 significant digits, so a read back is bit-exact.
void write_matrix_market(const CsrMatrix& A, const std::string& path, bool symmetric = false);

// Raw little-endian dump: int64 length, then the doubles.
void        write_vector_binary(const DenseVector& v, const std::string& path);
DenseVector read_vector_binary(const std::string& path, std::string name = "");

} // namespace rivulet
