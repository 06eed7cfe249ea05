#pragma once
// rivulet (B200 build) -- Krylov solvers (the reference's
// solvers.cpp is absent, so signatures follow SPEC).

#include "rivulet/csr.hpp"
#include "rivulet/managed.hpp"
#include "rivulet/vector.hpp"

#include <cstdint>
#include <functional>
#include <vector>

namespace rivulet {

enum class SolverMethod { CG, TFQMR };
// Async: the PAPER.md:104-150 listing through the linalg API on three
//        contexts (dctx_a/b/c exactly as SPEC.md:497 assigns them).
// SyncBaseline: the same math on the globally-blocking context.
// Fused: the B200 path -- 2 fused kernels per iteration captured as one CUDA
//        graph, every scalar device-resident (default); CG on
//        small systems (<= 16 K rows of <= 9 entries) runs as ONE kernel on
//        one thread-block cluster instead.
enum class SolverMode { Async, SyncBaseline, Fused };
enum class PcType { Jacobi, None };

struct SolverConfig {
    SolverMethod method = SolverMethod::CG;
    SolverMode   mode   = SolverMode::Fused;
    int          max_it = 20;
    PcType       pc     = PcType::Jacobi;
    double       rtol   = 0.0; // device-side exit: dp <= max(rtol*dp0, atol)
    double       atol   = 0.0;
    // converged_callback_bridge: receives the pending dp;
    // calling dp.front() synchronises, ignoring it does not.  Not available
    // in Fused mode (the whole solve is one graph).
    std::function<bool(Managed& dp, int iteration)> convergence_callback;
};

struct FlopLog {
    std::uint64_t total_flops = 0;
    std::uint64_t matmult = 0, dot = 0, norm = 0, axpy = 0, aypx = 0, scalar_expr = 0;
    std::uint64_t h2d = 0, d2h = 0;
};

struct SolveResult {
    FlopLog             flops;
    std::vector<double> history; // ||z_k||_2, k = 0..iterations
    int                 iterations = 0;
    bool                converged  = false;
};

// x0 = 0, r0 = b.  Throws BreakdownError(iteration) on breakdown.
SolveResult cg_solve(const CsrMatrix& A, const DenseVector& b, DenseVector& x,
                     const SolverConfig& cfg = {});
SolveResult tfqmr_solve(const CsrMatrix& A, const DenseVector& b, DenseVector& x,
                        const SolverConfig& cfg = {}); // left-Jacobi TFQMR; history 2*its+1

// z <- diag(A)^-1 r.
void pc_jacobi_apply(const DenseVector& diag_inv, const DenseVector& r, DenseVector& z,
                     const Context& ctx);

} // namespace rivulet
