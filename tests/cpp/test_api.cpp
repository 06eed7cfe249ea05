// test_api.cpp -- the C++ drop-in API (include/rivulet/) against SPEC.md's
// examples and the CPU oracle (oracle/rvk_oracle.h, test infrastructure).
// Run by tests/test_gpu_api.py on a B200; prints PASS/FAIL per case.
#include "rvk.h"
#include "rivulet/context.hpp"
#include "rivulet/csr.hpp"
#include "rivulet/expr.hpp"
#include "rivulet/linalg.hpp"
#include "rivulet/managed.hpp"
#include "rivulet/mmio.hpp"
#include "rivulet/runtime.hpp"
#include "rivulet/solvers.hpp"
#include "rivulet/stencil.hpp"
#include "rivulet/trace.hpp"
#include "rivulet/vector.hpp"

extern "C" {
#include "../../oracle/rvk_oracle.h"
}

#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <functional>
#include <string>
#include <thread>
#include <vector>

using namespace rivulet;

static int g_fail = 0;
#define EXPECT(c)                                                                                \
    do {                                                                                         \
        if (!(c)) {                                                                              \
            std::printf("  expectation failed: %s (%s:%d)\n", #c, __FILE__, __LINE__);           \
            throw std::runtime_error("expectation");                                             \
        }                                                                                        \
    } while (0)

static void run(const char* name, const std::function<void()>& f)
{
    try {
        f();
        std::printf("PASS %s\n", name);
    } catch (const std::exception& e) {
        ++g_fail;
        std::printf("FAIL %s: %s\n", name, e.what());
    }
    std::fflush(stdout);
}

static double rel(double a, double b) { return std::fabs(a - b) / std::max(std::fabs(b), 1e-300); }

struct HostCsr {
    std::size_t n;
    std::vector<int64_t> off;
    std::vector<int32_t> cols;
    std::vector<double> vals;
};

static HostCsr oracle_laplacian(int dim, int pts, int64_t nx, int64_t ny, int64_t nz)
{
    HostCsr h;
    h.n = (std::size_t)ro_laplacian_rows(dim, nx, ny, nz);
    const int64_t nnz = ro_laplacian_nnz(dim, pts, nx, ny, nz);
    h.off.resize(h.n + 1);
    h.cols.resize(nnz);
    h.vals.resize(nnz);
    ro_build_laplacian(dim, pts, nx, ny, nz, h.off.data(), h.cols.data(), h.vals.data());
    return h;
}

int main()
{
    // ---- Vec known answers ---------------------------------------
    run("vec_norm [3,4] = 5", [] {
        Context     ctx;
        DenseVector v(std::vector<double>{3, 4});
        Managed     out;
        vec_norm_async(v, NormType::Norm2, out, ctx);
        EXPECT(out.validity() == Managed::Validity::PendingOnContext);
        EXPECT(out.front() == 5.0);
        EXPECT(out.validity() == Managed::Validity::HostValid);
        DenseVector z(100);
        vec_norm_async(z, NormType::Norm2, out, ctx);
        EXPECT(out.front() == 0.0);
    });
    run("vec_dot / axpy / waxpy / scale", [] {
        Context     ctx;
        DenseVector x(std::vector<double>{1, 1, 1}), y(std::vector<double>{1, 1, 1});
        Managed     d;
        vec_dot_async(x, y, d, ctx);
        EXPECT(d.front() == 3.0);
        DenseVector yy(std::vector<double>{1, 1}), xx(std::vector<double>{3, 4});
        vec_axpy_async(yy, 2.0, xx, ctx);
        auto h = yy.to_host();
        EXPECT(h[0] == 7.0 && h[1] == 9.0);
        DenseVector w(2);
        vec_waxpy_async(w, 2.0, xx, yy, ctx);  // 2*[3,4] + [7,9]
        h = w.to_host();
        EXPECT(h[0] == 13.0 && h[1] == 17.0);
        vec_scale_async(w, 0.0, ctx);
        h = w.to_host();
        EXPECT(h[0] == 0.0 && h[1] == 0.0);
        bool threw = false;
        try {
            DenseVector a(3), b(4);
            vec_dot_async(a, b, d, ctx);
        } catch (const Error&) {
            threw = true;
        }
        EXPECT(threw);
    });
    run("normalize motif: norm -> 1/norm -> scale, zero host syncs (acceptance #4)", [] {
        for (std::size_t n : {10ul, 1000ul, 1000000ul}) {
            std::vector<double> hv(n);
            ro_rhs(7 + n, (int64_t)n, hv.data());
            Context     ctx;
            DenseVector v(hv);
            Managed     alpha;
            const auto  s0 = runtime::host_syncs();
            vec_norm_async(v, NormType::Norm2, alpha, ctx);
            alpha = Eval(1.0 / alpha, ctx);
            vec_scale_async(v, alpha, ctx);
            EXPECT(runtime::host_syncs() == s0);
            auto   h = v.to_host();
            double s = 0;
            for (double e : h) s += e * e;
            EXPECT(std::fabs(std::sqrt(s) - 1.0) < 1e-12);
        }
    });
    // ---- Mat ----------------------------------------------------------------------------
    run("mat_mult identity and 1D 3-point (SPEC.md:408-409)", [] {
        Context     ctx;
        auto        I = CsrMatrix::identity(5);
        DenseVector x(std::vector<double>{1, -2, 3.5, 0, 7}), y(5);
        mat_mult(I, x, y, ctx);
        EXPECT(y.to_host() == x.to_host());
        CsrMatrix   T(3, 3, {0, 2, 5, 7}, {0, 1, 0, 1, 2, 1, 2}, {2, -1, -1, 2, -1, -1, 2});
        DenseVector ones(std::vector<double>{1, 1, 1}), out(3);
        mat_mult(T, ones, out); // synchronous form
        auto h = out.to_host();
        EXPECT(h[0] == 1 && h[1] == 0 && h[2] == 1);
    });
    run("CsrMatrix validation", [] {
        int thrown = 0;
        try { CsrMatrix(2, 2, {0, 1, 2}, {1, 0}, {1, 1}); } catch (const Error&) { ++thrown; }     // ok actually
        try { CsrMatrix(2, 2, {1, 1, 2}, {0, 1}, {1, 1}); } catch (const Error&) { ++thrown; }     // off[0] != 0
        try { CsrMatrix(1, 2, {0, 2}, {1, 0}, {1, 1}); } catch (const Error&) { ++thrown; }       // not increasing
        try { CsrMatrix(1, 2, {0, 1}, {5}, {1}); } catch (const Error&) { ++thrown; }             // out of range
        try { CsrMatrix(1, 2, {0, 2}, {0}, {1}); } catch (const Error&) { ++thrown; }             // off[n] != nnz
        EXPECT(thrown == 4);
    });
    run("build_laplacian bit-identical to the CPU builder (4 stencils)", [] {
        struct S { int dim, pts; int64_t nx, ny, nz; };
        for (S s : {S{2, 5, 13, 7, 1}, S{2, 9, 9, 11, 1}, S{3, 7, 5, 6, 4}, S{3, 27, 4, 5, 6}}) {
            StencilSpec sp{s.dim, s.pts, s.dim == 2 ? std::vector<int64_t>{s.nx, s.ny}
                                                    : std::vector<int64_t>{s.nx, s.ny, s.nz}};
            auto A = build_laplacian(sp);
            auto h = oracle_laplacian(s.dim, s.pts, s.nx, s.ny, s.nz);
            EXPECT(A.rows() == h.n && A.nnz() == h.cols.size());
            EXPECT(std::equal(h.off.begin(), h.off.end(), A.row_offsets().begin()));
            EXPECT(std::equal(h.cols.begin(), h.cols.end(), A.col_indices().begin()));
            EXPECT(std::memcmp(h.vals.data(), A.values().data(), h.vals.size() * 8) == 0);
            auto d  = A.diagonal().to_host();
            auto sc = stencil_coefficients(s.dim, s.pts);
            for (double e : d) EXPECT(e == sc.centre);
        }
    });
    // ---- Managed / Eval (SPEC.md expr & managed examples) ------------------------------------
    run("Eval / execute / CSE / folding", [] {
        Context ctx;
        Managed x(1.0, "x"), y(2.0, "y"), z(4.0, "z");
        Managed r = Eval(x + y, ctx);
        EXPECT(r.front() == 3.0);
        Managed s = x + y; // no Eval: synchronous, host-valid immediately after
        EXPECT(s.front() == 3.0);
        auto e1 = Eval((x + y) / z, ctx);
        Managed t(e1);
        EXPECT(t.front() == 0.75);
        EXPECT(Eval(Expr(2.0) * 3.0 + 1.0, ctx).op_count() == 0);
        auto sum = x + y;
        EXPECT(Eval(sum + sum, ctx).op_count() == 2);              // shared subtree once
        EXPECT(Eval((x + y) + (x + y), ctx).op_count() == 2);      // structural CSE
        Managed u(Eval(sin(((x + y) / z) * z) + 15, ctx));
        EXPECT(rel(u.front(), std::sin(3.0) + 15.0) < 1e-14);
        Managed w, v2;
        e1.execute(w);
        e1.execute(v2);
        EXPECT(w.front() == v2.front());
        Managed copy = r;     // synchronous snapshot
        r = Eval(x * z, ctx); // later change of the source
        EXPECT(copy.front() == 3.0 && r.front() == 4.0);
        Managed betaold = Eval(r, ctx); // copy of a pending value, no host sync
        EXPECT(betaold.front() == 4.0);
    });
    run("cross-context ordering: RAW edge installed, read-read free", [] {
        Context a, b;
        const std::size_t n = 4000000;
        DenseVector v(n), w(n);
        vec_set_async(v, 1.0, a);
        for (int i = 0; i < 10; ++i) vec_axpy_async(v, 1.0, v, a); // v = 1024 after 10 doublings
        Managed d1, d2;
        vec_norm_async(v, NormType::Norm2, d1, b);  // RAW across contexts
        EXPECT(rel(d1.front(), 1024.0 * std::sqrt((double)n)) < 1e-13);
        Context c;
        vec_dot_async(v, v, d2, c);                 // read after read on another ctx
        vec_copy_async(v, w, b);                    // read-read: no ordering needed
        EXPECT(rel(d2.front(), 1024.0 * 1024.0 * n) < 1e-13);
        vec_set_async(v, 0.0, c);                   // WAR: waits for b's and c's readers
        auto hw = w.to_host();
        EXPECT(hw[0] == 1024.0 && hw[n - 1] == 1024.0);
        auto hv = v.to_host();
        EXPECT(hv[0] == 0.0);
    });
    run("deferred release: handles die while values are in flight", [] {
        Context ctx;
        DenseVector big(8000000);
        vec_set_async(big, 2.0, ctx);
        for (int i = 0; i < 50; ++i) {
            Managed tmp;
            vec_dot_async(big, big, tmp, ctx); // tmp destroyed while pending
        }
        Managed last;
        vec_dot_async(big, big, last, ctx);
        EXPECT(last.front() == 4.0 * 8000000);
    });
    // ---- CG (acceptance #5/#6) --------------------------------------------------
    struct Case { int dim, pts; int64_t nx, ny, nz; };
    for (Case cs : {Case{2, 5, 16, 16, 1}, Case{2, 9, 32, 32, 1}, Case{3, 7, 8, 8, 8}, Case{3, 27, 8, 8, 8}}) {
        const std::string nm = "cg_solve modes vs oracle " + std::to_string(cs.pts) + "-pt";
        run(nm.c_str(), [cs] {
            auto h = oracle_laplacian(cs.dim, cs.pts, cs.nx, cs.ny, cs.nz);
            std::vector<double> bh(h.n), xo(h.n), hist(21), work(5 * h.n);
            ro_rhs(0x9E3779B97F4A7C15ull, (int64_t)h.n, bh.data());
            ro_cg_config cfg{20, RO_PC_JACOBI, 0.0, 0.0};
            ro_cg_result rr = ro_cg_solve((int64_t)h.n, h.off.data(), h.cols.data(), h.vals.data(),
                                          bh.data(), xo.data(), hist.data(), cfg, work.data());
            EXPECT(rr.iterations == 20);
            CsrMatrix   A(h.n, h.n, h.off, h.cols, h.vals);
            DenseVector b(bh);
            for (SolverMode m : {SolverMode::Fused, SolverMode::Async, SolverMode::SyncBaseline}) {
                DenseVector  x(h.n);
                SolverConfig c;
                c.mode     = m;
                const auto census0 = runtime::census();
                auto res   = cg_solve(A, b, x, c);
                const auto d = runtime::census() - census0;
                EXPECT(res.iterations == 20 && res.history.size() == 21);
                for (int k = 0; k <= 20; ++k)
                    if (!(rel(res.history[k], hist[k]) < 1e-10)) {
                        std::printf("  mode %d k %d got %.17g want %.17g\n", (int)m, k, res.history[k], hist[k]);
                        EXPECT(false);
                    }
                auto xh = x.to_host();
                double num = 0, den = 0;
                for (std::size_t i = 0; i < h.n; ++i) {
                    num += (xh[i] - xo[i]) * (xh[i] - xo[i]);
                    den += xo[i] * xo[i];
                }
                EXPECT(std::sqrt(num / den) < 1e-10);
                // census: 1 matmult + 3 reductions + 3 updates per iteration
                EXPECT(d.kernels_of(runtime::KernelKind::MatMult) == 20);
                EXPECT(d.reductions() == 2 + 3 * 20); // setup norm + dot, then 3 per iteration
                EXPECT(d.kernels_of(runtime::KernelKind::Axpy) == 40);
                EXPECT(d.kernels_of(runtime::KernelKind::Aypx) == 19);
                // FlopLog = sum over iterations of 2 nnz + 12 n + c  (exact integer)
                const uint64_t n = h.n, nnz = h.cols.size();
                const uint64_t body = 20 * (2 * nnz + 8 * n) + 40 * 2 * n - 2 * n; // aypx only i>=1
                EXPECT(res.flops.matmult == 20 * 2 * nnz);
                EXPECT(res.flops.axpy == 40 * 2 * n && res.flops.aypx == 19 * 2 * n);
                (void)body;
            }
        });
    }
    run("cg Async: host syncs independent of iteration count (0 per iteration)", [] {
        auto h = oracle_laplacian(2, 5, 64, 64, 1);
        CsrMatrix   A(h.n, h.n, h.off, h.cols, h.vals);
        std::vector<double> bh(h.n);
        ro_rhs(1, (int64_t)h.n, bh.data());
        DenseVector b(bh), x(h.n);
        uint64_t syncs[2];
        int      its[2] = {5, 20};
        for (int k = 0; k < 2; ++k) {
            SolverConfig c;
            c.mode   = SolverMode::Async;
            c.max_it = its[k];
            cg_solve(A, b, x, c); // warm
            const auto s0 = runtime::host_syncs();
            cg_solve(A, b, x, c);
            syncs[k] = runtime::host_syncs() - s0;
        }
        // only the end-of-solve reads (history + three context drains) may
        // block -- whether they do is timing-dependent, exactly like the
        // reference's await_host -- so the count is bounded, never per-iteration
        EXPECT(syncs[0] <= 4 && syncs[1] <= 4);
        SolverConfig f;
        cg_solve(A, b, x, f); // first call also sets the plan up (one validation sync)
        const auto   s0 = runtime::host_syncs();
        cg_solve(A, b, x, f); // fused: exactly the one result read
        std::printf("  syncs: async(5)=%llu async(20)=%llu fused=%llu\n", (unsigned long long)syncs[0],
                    (unsigned long long)syncs[1], (unsigned long long)(runtime::host_syncs() - s0));
        EXPECT(runtime::host_syncs() - s0 == 1);
    });
    run("one process, one host thread per device: concurrent cg_solve on every GPU (2+ threads)", [] {
        // per-device kernel attributes / SM counts / sync contexts / memory
        // streams: each thread selects its device and runs the whole API there.
        // With one GPU both threads share device 0 (the concurrency part).
        const int ndev = rvk_device_count();
        EXPECT(ndev >= 1);
        const int nthr = ndev >= 2 ? ndev : 2;
        auto h = oracle_laplacian(3, 7, 40, 36, 32);
        std::vector<double> bh(h.n), xo(h.n), hist(21), work(5 * h.n);
        ro_rhs(0x9E3779B97F4A7C15ull, (int64_t)h.n, bh.data());
        ro_cg_config cfg{20, RO_PC_JACOBI, 0.0, 0.0};
        ro_cg_solve((int64_t)h.n, h.off.data(), h.cols.data(), h.vals.data(), bh.data(), xo.data(),
                    hist.data(), cfg, work.data());
        std::vector<int>         ok(nthr, 0);
        std::vector<std::string> err(nthr);
        std::vector<std::thread> th;
        for (int t = 0; t < nthr; ++t)
            th.emplace_back([&, t] {
                try {
                    if (rvk_set_device(t % ndev) != RVK_OK) throw std::runtime_error(rvk_last_error());
                    CsrMatrix    A(h.n, h.n, h.off, h.cols, h.vals);
                    DenseVector  b(bh), x(h.n);
                    SolverConfig c;
                    for (int rep = 0; rep < 3; ++rep) {
                        auto res = cg_solve(A, b, x, c);
                        if (res.iterations != 20) throw std::runtime_error("iterations");
                        for (int k = 0; k <= 20; ++k)
                            if (!(rel(res.history[k], hist[k]) < 1e-10)) throw std::runtime_error("history");
                        auto   xh = x.to_host();
                        double num = 0, den = 0;
                        for (std::size_t i = 0; i < h.n; ++i) {
                            num += (xh[i] - xo[i]) * (xh[i] - xo[i]);
                            den += xo[i] * xo[i];
                        }
                        if (!(std::sqrt(num / den) < 1e-10)) throw std::runtime_error("x");
                    }
                    ok[t] = 1;
                } catch (const std::exception& e) {
                    err[t] = e.what();
                }
            });
        for (auto& t : th) t.join();
        rvk_set_device(0);
        for (int t = 0; t < nthr; ++t) {
            if (!ok[t]) std::printf("  thread %d (device %d): %s\n", t, t % ndev, err[t].c_str());
            EXPECT(ok[t]);
        }
        std::printf("  %d threads on %d device(s)\n", nthr, ndev);
    });
    run("cg breakdown reported with iteration (all modes)", [] {
        CsrMatrix   A(2, 2, {0, 1, 2}, {0, 1}, {1.0, -1.0});
        DenseVector b(std::vector<double>{1, 1});
        for (SolverMode m : {SolverMode::Fused, SolverMode::Async, SolverMode::SyncBaseline}) {
            DenseVector  x(2);
            SolverConfig c;
            c.mode = m;
            c.pc   = PcType::None;
            bool got = false;
            try {
                cg_solve(A, b, x, c);
            } catch (const BreakdownError& e) {
                got = e.iteration() == 0;
            }
            EXPECT(got);
        }
    });
    run("cg identity converges in one iteration (SPEC.md:464)", [] {
        auto        I = CsrMatrix::identity(100);
        std::vector<double> bh(100);
        ro_rhs(3, 100, bh.data());
        DenseVector b(bh);
        for (SolverMode m : {SolverMode::Fused, SolverMode::Async, SolverMode::SyncBaseline}) {
            DenseVector  x(100);
            SolverConfig c;
            c.mode = m;
            c.pc   = PcType::None;
            c.rtol = 1e-14;
            auto r = cg_solve(I, b, x, c);
            EXPECT(r.converged && r.iterations == 1);
            auto xh = x.to_host();
            for (int i = 0; i < 100; ++i) EXPECT(std::fabs(xh[i] - bh[i]) <= 1e-15);
        }
    });
    run("convergence callback: early exit, sync only if it reads dp", [] {
        auto h = oracle_laplacian(2, 5, 32, 32, 1);
        CsrMatrix   A(h.n, h.n, h.off, h.cols, h.vals);
        std::vector<double> bh(h.n), xo(h.n), hist(501), work(5 * h.n);
        ro_rhs(5, (int64_t)h.n, bh.data());
        ro_cg_config oc{500, RO_PC_JACOBI, 0.0, 1e-8};
        auto rr = ro_cg_solve((int64_t)h.n, h.off.data(), h.cols.data(), h.vals.data(), bh.data(),
                              xo.data(), hist.data(), oc, work.data());
        EXPECT(rr.status == RO_CONVERGED);
        DenseVector  b(bh), x(h.n);
        SolverConfig c;
        c.mode                 = SolverMode::Async;
        c.max_it               = 500;
        c.convergence_callback = [](Managed& dp, int) { return dp.front() <= 1e-8; };
        auto r = cg_solve(A, b, x, c);
        EXPECT(r.converged && r.iterations == rr.iterations);
        int calls = 0;
        c.max_it  = 20;
        c.convergence_callback = [&](Managed&, int) { ++calls; return false; }; // ignores dp
        const auto s0 = runtime::host_syncs();
        auto r2 = cg_solve(A, b, x, c);
        EXPECT(calls == 20 && r2.iterations == 20);
        // a callback that never reads dp adds no sync: only the end-of-solve
        // reads remain (history + the three context drains), whatever max_it
        EXPECT(runtime::host_syncs() - s0 <= 4);
        calls = 0;
        c.convergence_callback = [&](Managed& dp, int) { ++calls; return dp.front() < 0.0; };
        const auto s1 = runtime::host_syncs();
        cg_solve(A, b, x, c);
        EXPECT(runtime::host_syncs() - s1 >= 20); // reading dp syncs every iteration
    });
    // ---- TFQMR -----------------------------------------------------------------
    run("tfqmr_solve vs oracle (5-pt 32x32, 1e-8) + census", [] {
        auto h = oracle_laplacian(2, 5, 32, 32, 1);
        std::vector<double> bh(h.n), xo(h.n), hist(41), work(11 * h.n);
        ro_rhs(0x9E3779B97F4A7C15ull, (int64_t)h.n, bh.data());
        ro_cg_config cfg{20, RO_PC_JACOBI, 0.0, 0.0};
        int          nh = 0;
        ro_cg_result rr = ro_tfqmr_solve((int64_t)h.n, h.off.data(), h.cols.data(), h.vals.data(),
                                         bh.data(), xo.data(), hist.data(), cfg, work.data(), &nh);
        EXPECT(rr.iterations == 20 && nh == 41);
        CsrMatrix   A(h.n, h.n, h.off, h.cols, h.vals);
        DenseVector b(bh), x(h.n);
        const auto  census0 = runtime::census();
        auto        res     = tfqmr_solve(A, b, x, SolverConfig{});
        const auto  d       = runtime::census() - census0;
        EXPECT(res.iterations == 20 && res.history.size() == 41);
        for (int k = 0; k < 41 && k < (int)res.history.size(); ++k)
            if (!(rel(res.history[k], hist[k]) < 1e-8)) {
                std::printf("  k %d got %.17g want %.17g\n", k, res.history[k], hist[k]);
                EXPECT(false);
            }
        auto   xh  = x.to_host();
        double num = 0, den = 0;
        for (std::size_t i = 0; i < h.n; ++i) {
            num += (xh[i] - xo[i]) * (xh[i] - xo[i]);
            den += xo[i] * xo[i];
        }
        EXPECT(std::sqrt(num / den) < 1e-8);
        // exactly 2 matmults per iteration (+1 in setup:
        // v = B A p), reductions >= 2x... the PETSc loop has 3 per iteration
        EXPECT(d.kernels_of(runtime::KernelKind::MatMult) == 1 + 2 * 20);
        EXPECT(d.reductions() == 2 + 3 * 20);
    });
    run("tfqmr identity converges in the first half step; breakdown reported", [] {
        auto        I = CsrMatrix::identity(100);
        std::vector<double> bh(100);
        ro_rhs(3, 100, bh.data());
        DenseVector  b(bh), x(100);
        SolverConfig c;
        c.pc   = PcType::None;
        auto r = tfqmr_solve(I, b, x, c);
        EXPECT(r.converged && r.iterations == 1 && r.history.size() == 2);
        auto xh = x.to_host();
        for (int i = 0; i < 100; ++i) EXPECT(xh[i] == bh[i]);
        CsrMatrix   S(2, 2, {0, 1, 2}, {1, 0}, {1.0, 1.0}); // (A b, b) = 0 for b = e0
        DenseVector b2(std::vector<double>{1, 0}), x2(2);
        bool        got = false;
        try {
            tfqmr_solve(S, b2, x2, c);
        } catch (const BreakdownError& e) {
            got = e.iteration() == 0;
        }
        EXPECT(got);
    });
    // ---- external interfaces -----------------------------------------------------
    run("Matrix Market + raw vector round trips (SPEC.md:432)", [] {
        auto same = [](const CsrMatrix& a, const CsrMatrix& b) {
            return a.rows() == b.rows() && a.cols() == b.cols() && a.nnz() == b.nnz() &&
                   std::memcmp(a.row_offsets().data(), b.row_offsets().data(), (a.rows() + 1) * 8) == 0 &&
                   std::memcmp(a.col_indices().data(), b.col_indices().data(), a.nnz() * 4) == 0 &&
                   std::memcmp(a.values().data(), b.values().data(), a.nnz() * 8) == 0;
        };
        auto h = oracle_laplacian(2, 9, 12, 10, 1);
        CsrMatrix A(h.n, h.n, h.off, h.cols, h.vals);
        write_matrix_market(A, "/tmp/rvk_test_gen.mtx");
        write_matrix_market(A, "/tmp/rvk_test_sym.mtx", true);
        EXPECT(same(read_matrix_market("/tmp/rvk_test_gen.mtx"), A));
        EXPECT(same(read_matrix_market("/tmp/rvk_test_sym.mtx"), A));
        // non-representable decimals survive (17 significant digits)
        CsrMatrix B(3, 4, {0, 2, 2, 4}, {1, 3, 0, 2}, {0.1, -1.0 / 3.0, 1e-300, 6.02214076e23});
        write_matrix_market(B, "/tmp/rvk_test_b.mtx");
        EXPECT(same(read_matrix_market("/tmp/rvk_test_b.mtx"), B));
        bool threw = false;
        try {
            write_matrix_market(B, "/tmp/rvk_test_x.mtx", true); // not square / symmetric
        } catch (const Error&) {
            threw = true;
        }
        EXPECT(threw);
        // unsorted entries, duplicates summed in file order, pattern/symmetric
        {
            std::FILE* f = std::fopen("/tmp/rvk_test_dup.mtx", "w");
            std::fprintf(f, "%%%%MatrixMarket matrix coordinate real general\n%% c\n3 3 5\n"
                            "3 1 2.5\n1 1 1\n2 2 4\n1 1 0.25\n1 3 -1\n");
            std::fclose(f);
            auto D = read_matrix_market("/tmp/rvk_test_dup.mtx");
            EXPECT(same(D, CsrMatrix(3, 3, {0, 2, 3, 4}, {0, 2, 1, 0}, {1.25, -1.0, 4.0, 2.5})));
            f = std::fopen("/tmp/rvk_test_pat.mtx", "w");
            std::fprintf(f, "%%%%MatrixMarket matrix coordinate pattern symmetric\n2 2 2\n1 1\n2 1\n");
            std::fclose(f);
            EXPECT(same(read_matrix_market("/tmp/rvk_test_pat.mtx"),
                        CsrMatrix(2, 2, {0, 2, 3}, {0, 1, 0}, {1.0, 1.0, 1.0})));
        }
        threw = false;
        try {
            std::FILE* f = std::fopen("/tmp/rvk_test_bad.mtx", "w");
            std::fprintf(f, "%%%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n");
            std::fclose(f);
            read_matrix_market("/tmp/rvk_test_bad.mtx");
        } catch (const Error&) {
            threw = true;
        }
        EXPECT(threw);
        // a solve on the read-back matrix is the solve on the original, bit for bit
        std::vector<double> bh(h.n);
        ro_rhs(7, (int64_t)h.n, bh.data());
        DenseVector b(bh);
        write_vector_binary(b, "/tmp/rvk_test_b.bin");
        DenseVector b2 = read_vector_binary("/tmp/rvk_test_b.bin");
        EXPECT(b2.to_host() == bh);
        DenseVector x1(h.n), x2(h.n);
        auto r1 = cg_solve(A, b, x1);
        auto r2 = cg_solve(read_matrix_market("/tmp/rvk_test_sym.mtx"), b2, x2);
        EXPECT(r1.history == r2.history && x1.to_host() == x2.to_host());
    });
    // ---- property tests ---------------------------------------------------
    run("10,000 random expression DAGs vs a host interpreter (SPEC.md:624)", [] {
        // IEEE + - * / min max neg abs sqrt are exact on both sides (bitwise);
        // DAGs with sin/cos/exp (libdevice vs glibc, <= 2 ulp) are built without
        // subtraction/division so no cancellation amplifies the ulps: 1e-12.
        std::uint64_t rng = 0x2545F4914F6CDD1Dull;
        auto next = [&] {
            rng ^= rng << 13;
            rng ^= rng >> 7;
            rng ^= rng << 17;
            return rng;
        };
        auto unif = [&](double lo, double hi) { return lo + (hi - lo) * (double)(next() >> 11) * 0x1.0p-53; };
        Context ctx;
        std::vector<Managed> leaves;
        std::vector<double>  lv;
        for (int i = 0; i < 6; ++i) {
            lv.push_back(unif(0.5, 2.0));
            leaves.emplace_back(lv.back());
        }
        struct Node {
            Expr   e;
            double v;
        };
        // transcendental: false -> exact ops only
        std::function<Node(int, bool)> gen = [&](int depth, bool tr) -> Node {
            const int pick = (int)(next() % 16);
            if (depth == 0 || pick < 3) {
                if (next() % 3 == 0) {
                    const double c = unif(0.5, 2.0);
                    return {Expr(c), c};
                }
                const int k = (int)(next() % leaves.size());
                return {Expr(leaves[k]), lv[k]};
            }
            if (pick < 6) { // unary
                Node a = gen(depth - 1, tr);
                const int u = (int)(next() % (tr ? 6 : 3));
                switch (u) {
                case 0: return {-a.e, -a.v};
                case 1: return {abs(a.e), std::fabs(a.v)};
                case 2: return {sqrt(abs(a.e)), std::sqrt(std::fabs(a.v))};
                case 3: return {sin(a.e), std::sin(a.v)};
                case 4: return {cos(a.e), std::cos(a.v)};
                default: return {exp(sin(a.e)), std::exp(std::sin(a.v))};
                }
            }
            Node a = gen(depth - 1, tr), b = gen(depth - 1, tr);
            const int o = (int)(next() % (tr ? 4 : 6));
            static const int kTrOps[4] = {0, 2, 4, 5}; // + * min max
            const int        op         = tr ? kTrOps[o] : o;
            switch (op) {
            case 0: return {a.e + b.e, a.v + b.v};
            case 1: return {a.e - b.e, a.v - b.v};
            case 2: return {a.e * b.e, a.v * b.v};
            case 3: return {a.e / b.e, a.v / b.v};
            case 4: return {min(a.e, b.e), std::fmin(a.v, b.v)};
            default: return {max(a.e, b.e), std::fmax(a.v, b.v)};
            }
        };
        int exact = 0, approx = 0, skipped = 0;
        for (int t = 0; t < 10000; ++t) {
            const bool tr = t % 4 == 3;
            Node       nd = gen(5, tr);
            Managed    out;
            try {
                Eval(nd.e, ctx).execute(out);
            } catch (const Error&) { // a program over kMaxExprSteps: rejected up front
                ++skipped;
                continue;
            }
            const double got = out.front();
            if (tr) {
                ++approx;
                if (!(std::fabs(got - nd.v) <= 1e-12 * std::max(1.0, std::fabs(nd.v)))) {
                    std::printf("  dag %d: got %.17g want %.17g\n", t, got, nd.v);
                    EXPECT(false);
                }
            } else {
                ++exact;
                const bool same = std::memcmp(&got, &nd.v, 8) == 0 || (std::isnan(got) && std::isnan(nd.v));
                if (!same) {
                    std::printf("  dag %d: got %.17g want %.17g\n", t, got, nd.v);
                    EXPECT(false);
                }
            }
        }
        std::printf("  exact %d, transcendental %d, too large %d\n", exact, approx, skipped);
        EXPECT(skipped < 100);
    });
    run("1,000 random cross-context access programs vs sequential replay (SPEC.md:622)", [] {
        // Random elementwise programs over 4 vectors issued round-robin-at-random
        // on 3 contexts: the RAW/WAR/WAW edges the API installs must make the
        // device result equal the program-order replay on the host, bit for bit
        // (every op is elementwise IEEE, rounded exactly like the oracle).
        std::uint64_t rng = 0x9E3779B97F4A7C15ull;
        auto next = [&] {
            rng ^= rng << 13;
            rng ^= rng >> 7;
            rng ^= rng << 17;
            return rng;
        };
        const std::size_t n = 3000;
        Context ctxs[3];
        int     programs = 0;
        for (int prog = 0; prog < 1000; ++prog) {
            std::vector<std::vector<double>> h(4, std::vector<double>(n));
            std::vector<DenseVector>         v;
            for (int k = 0; k < 4; ++k) {
                for (std::size_t i = 0; i < n; ++i) h[k][i] = 0.5 + (double)((i * 7 + k * 13) % 17) / 16.0;
                v.emplace_back(std::span<const double>(h[k]));
            }
            const int nops = 4 + (int)(next() % 20);
            for (int o = 0; o < nops; ++o) {
                const Context& c = ctxs[next() % 3];
                const int      y = (int)(next() % 4), x = (int)(next() % 4), w = (int)(next() % 4);
                const double   a = 0.25 + (double)(next() % 8) / 8.0;
                switch (next() % 6) {
                case 0: // y += a x
                    vec_axpy_async(v[y], a, v[x], c);
                    for (std::size_t i = 0; i < n; ++i) h[y][i] = h[y][i] + a * h[x][i];
                    break;
                case 1: // y = x + a y
                    vec_aypx_async(v[y], a, v[x], c);
                    for (std::size_t i = 0; i < n; ++i) h[y][i] = h[x][i] + a * h[y][i];
                    break;
                case 2: // y *= a
                    vec_scale_async(v[y], a, c);
                    for (std::size_t i = 0; i < n; ++i) h[y][i] = h[y][i] * a;
                    break;
                case 3: // copy x -> y
                    if (x == y) break;
                    vec_copy_async(v[x], v[y], c);
                    h[y] = h[x];
                    break;
                case 4: // w = a x + y
                    if (w == x || w == y) break;
                    vec_waxpy_async(v[w], a, v[x], v[y], c);
                    for (std::size_t i = 0; i < n; ++i) h[w][i] = a * h[x][i] + h[y][i];
                    break;
                default: // w = x .* y
                    if (w == x || w == y) break;
                    vec_pointwise_mult_async(v[x], v[y], v[w], c);
                    for (std::size_t i = 0; i < n; ++i) h[w][i] = h[x][i] * h[y][i];
                }
            }
            for (int k = 0; k < 4; ++k) {
                auto d = v[k].to_host();
                if (std::memcmp(d.data(), h[k].data(), n * 8) != 0) {
                    std::printf("  program %d vector %d differs\n", prog, k);
                    EXPECT(false);
                }
            }
            ++programs;
        }
        std::printf("  %d programs\n", programs);
    });
    run("trace: device-timed tasks, Wait edges, HostSync events, JSONL + census export (trace.hpp:11-46)", [] {
        Context a(StreamType::DefaultBlocking, "producer"), b(StreamType::DefaultBlocking, "consumer");
        const std::size_t n = 1 << 22;
        DenseVector v(n);
        Managed d;
        a.synchronize();
        trace::clear();
        trace::set_enabled(true);
        vec_set_async(v, 2.0, a);
        vec_scale_async(v, 3.0, a);
        vec_norm_async(v, NormType::Norm2, d, b); // RAW across contexts: one Wait edge
        trace::marker("before front");
        const double nv = d.front();              // host sync (traced)
        EXPECT(rel(nv, 6.0 * std::sqrt((double)n)) < 1e-13);
        auto evs = trace::snapshot();
        int tasks = 0, waits = 0, syncs = 0, marks = 0;
        std::uint64_t last_seq = 0;
        for (const auto& e : evs) {
            if (e.kind == trace::EventKind::Task) {
                ++tasks;
                EXPECT(e.enqueue_seq > last_seq); // tasks in enqueue order
                last_seq = e.enqueue_seq;
                EXPECT(e.device_timed);
                EXPECT(e.t_end_ns >= e.t_start_ns);
                EXPECT(e.context_id == a.id() || e.context_id == b.id());
                EXPECT(e.context_name == (e.context_id == a.id() ? "producer" : "consumer"));
            }
            if (e.kind == trace::EventKind::Wait) {
                ++waits;
                EXPECT(e.context_id == b.id());
            }
            if (e.kind == trace::EventKind::HostSync) ++syncs;
            if (e.kind == trace::EventKind::Marker) ++marks;
        }
        std::printf("  tasks=%d waits=%d host_syncs=%d markers=%d\n", tasks, waits, syncs, marks);
        EXPECT(tasks == 3 && waits == 1 && marks == 1 && syncs >= 1);
        // the scale on `a` ran after the set on `a`, the norm on `b` after both
        const trace::TraceEvent* t[3];
        int k = 0;
        for (const auto& e : evs)
            if (e.kind == trace::EventKind::Task) t[k++] = &e;
        EXPECT(t[1]->t_start_ns >= t[0]->t_end_ns - 2000 && t[2]->t_start_ns >= t[1]->t_end_ns - 2000);
        const std::string path = "/tmp/rvk_trace_test.jsonl";
        trace::write_jsonl(path);
        std::ifstream in(path);
        std::string line;
        int lines = 0;
        while (std::getline(in, line)) {
            EXPECT(line.front() == '{' && line.back() == '}');
            EXPECT(line.find("\"kind\":") != std::string::npos);
            ++lines;
        }
        EXPECT(lines == (int)evs.size());
        trace::write_chrome("/tmp/rvk_trace_test.json");
        const std::string j = runtime::to_json();
        EXPECT(j.find("\"host_syncs\":") != std::string::npos && j.find("\"norm\":{\"kernels\":") != std::string::npos);
        trace::set_enabled(false);
        trace::clear();
        vec_set_async(v, 1.0, a);
        a.synchronize();
        EXPECT(trace::snapshot().empty()); // off: nothing recorded
    });
    std::printf("%s: %d failure(s)\n", g_fail ? "FAILED" : "OK", g_fail);
    return g_fail ? 1 : 0;
}
