#pragma once
// rivulet (B200 build) -- benchmark Laplacians, assembled
// on the device, bit-identical to the CPU builder.

#include "rivulet/csr.hpp"

#include <cstdint>
#include <vector>

namespace rivulet {

struct StencilSpec {
    int                       dim    = 2; // 2 or 3
    int                       points = 5; // 5|9 (2D), 7|27 (3D)
    std::vector<std::int64_t> grid;       // cells per dimension (x fastest)
};

struct StencilCoefficients {
    double centre;    // points - 1
    double neighbour; // -1
};

StencilCoefficients stencil_coefficients(int dim, int points);
CsrMatrix           build_laplacian(const StencilSpec& spec); // diag: A.diagonal()

} // namespace rivulet
