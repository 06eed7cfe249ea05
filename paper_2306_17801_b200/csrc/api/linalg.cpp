// linalg.cpp -- the Vec/Mat API (linalg.hpp:48-78 of the reference) on sm_100a.
//
// Each *_async call: check dimensions, log the
// census at issue time (runtime.hpp:60-64), bracket the operands (Read /
// Write / ReadWrite) so cross-context conflicts become cudaStreamWaitEvent
// edges, enqueue exactly ONE rvk kernel on the context's stream, publish the
// completion event and leave managed outputs pending.  No host sync.
#include "internal.hpp"
#include "rivulet/linalg.hpp"

namespace rivulet {

using detail::Launch;
using runtime::KernelKind;

namespace detail {

ScalarArg::ScalarArg(const Managed& m) : root_(Expr(m).node()) {}
ScalarArg::ScalarArg(const Expr& e) : root_(e.node())
{
    using K = ExprNode::Kind;
    const auto& n = *root_;
    if (n.kind == K::Unary && n.lhs->kind == K::Leaf) op_count_ = 1;
    if (n.kind == K::Binary && n.bop == BinaryOp::Div && n.rhs->kind == K::Leaf &&
        (n.lhs->kind == K::Leaf || (n.lhs->kind == K::Constant && n.lhs->value == 1.0)))
        op_count_ = 1;
}
ScalarArg::ScalarArg(double v) : root_(Expr(v).node()) {}

namespace {

// Lower a ScalarArg to the in-kernel rvk_scalar forms; anything else is
// evaluated into a device temporary on ctx first.  Leaves get Read marks.
struct Lowered {
    rvk_scalar                                  s{RVK_SCALAR_CONST, 0.0, nullptr, nullptr};
    std::vector<std::shared_ptr<ManagedState>> keep; // alive until marked
    std::unique_ptr<Managed>                    tmp;
};

std::shared_ptr<ManagedState> leaf_of(const ExprNodePtr& n)
{
    auto s = n->leaf.lock();
    if (!s) throw Error("scalar argument references a destroyed managed value");
    if (s->n != 1) throw Error("scalar argument must have length 1");
    return s;
}

Lowered lower(const ScalarArg& a, const Context& ctx, Launch& L)
{
    using K = ExprNode::Kind;
    Lowered     out;
    const auto& n = *a.root();
    auto        use = [&](const ExprNodePtr& leaf) {
        auto s = leaf_of(leaf);
        L.read(s->id);
        out.keep.push_back(s);
        return s->dev;
    };
    if (n.kind == K::Constant) {
        out.s = rvk_scalar{RVK_SCALAR_CONST, n.value, nullptr, nullptr};
    } else if (n.kind == K::Leaf) {
        out.s = rvk_scalar{RVK_SCALAR_PTR, 0.0, use(a.root()), nullptr};
    } else if (n.kind == K::Unary && n.lhs->kind == K::Leaf &&
               (n.uop == UnaryOp::Neg || n.uop == UnaryOp::Sqrt)) {
        out.s = rvk_scalar{n.uop == UnaryOp::Neg ? RVK_SCALAR_NEG_PTR : RVK_SCALAR_SQRT_PTR, 0.0,
                           use(n.lhs), nullptr};
    } else if (n.kind == K::Binary && n.bop == BinaryOp::Div && n.rhs->kind == K::Leaf &&
               n.lhs->kind == K::Leaf) {
        out.s = rvk_scalar{RVK_SCALAR_DIV_PTR_PTR, 0.0, use(n.lhs), use(n.rhs)};
    } else if (n.kind == K::Binary && n.bop == BinaryOp::Div && n.rhs->kind == K::Leaf &&
               n.lhs->kind == K::Constant && n.lhs->value == 1.0) {
        out.s = rvk_scalar{RVK_SCALAR_RECIP_PTR, 0.0, use(n.rhs), nullptr};
    } else {
        if (n.len != 1) throw Error("scalar argument must have length 1");
        out.tmp = std::make_unique<Managed>(0.0, "scalar_arg");
        Eval(Expr(a.root()), ctx).execute(*out.tmp);
        out.s = rvk_scalar{RVK_SCALAR_PTR, 0.0, out.tmp->device_data(), nullptr};
        L.read(out.tmp->id());
    }
    if (a.op_count()) runtime::log_kernel(KernelKind::ExprEval, a.op_count(), 0); // fused
    return out;
}

void same_len(std::size_t a, std::size_t b, const char* api)
{
    if (a != b)
        throw Error(std::string(api) + ": dimension mismatch (" + std::to_string(a) + " vs " +
                    std::to_string(b) + ")");
}

std::string lab(std::string label, const char* dflt) { return label.empty() ? dflt : label; }

} // namespace
} // namespace detail

using detail::check;

void vec_norm_async(const DenseVector& v, NormType, Managed& out, const Context& ctx, std::string label)
{
    if (out.size() != 1) throw Error("vec_norm_async: output must have length 1");
    detail::check_no_write_view(*v.state(), "vec_norm_async");
    runtime::log_kernel(KernelKind::Norm, 2 * v.size());
    Launch L(ctx, detail::lab(std::move(label), "vec_norm"));
    L.read(v.id()).write(out.id());
    L.begin();
    check(rvk_nrm2(ctx.handle(), (int64_t)v.size(), v.device_data(), out.device_data()), "vec_norm_async");
    out.state()->mark_written(L.end(), ctx.id());
}

void vec_dot_async(const DenseVector& x, const DenseVector& y, Managed& out, const Context& ctx,
                   std::string label)
{
    detail::same_len(x.size(), y.size(), "vec_dot_async");
    if (out.size() != 1) throw Error("vec_dot_async: output must have length 1");
    detail::check_no_write_view(*x.state(), "vec_dot_async");
    detail::check_no_write_view(*y.state(), "vec_dot_async");
    runtime::log_kernel(KernelKind::Dot, 2 * x.size());
    Launch L(ctx, detail::lab(std::move(label), "vec_dot"));
    L.read(x.id()).read(y.id()).write(out.id());
    L.begin();
    check(rvk_dot(ctx.handle(), (int64_t)x.size(), x.device_data(), y.device_data(), out.device_data()),
          "vec_dot_async");
    out.state()->mark_written(L.end(), ctx.id());
}

void vec_scale_async(DenseVector& v, detail::ScalarArg alpha, const Context& ctx, std::string label)
{
    detail::check_no_write_view(*v.state(), "vec_scale_async");
    runtime::log_kernel(KernelKind::Scale, v.size());
    Launch L(ctx, detail::lab(std::move(label), "vec_scale"));
    auto   s = detail::lower(alpha, ctx, L);
    L.read_write(v.id());
    L.begin();
    check(rvk_scale(ctx.handle(), (int64_t)v.size(), s.s, v.device_data()), "vec_scale_async");
    L.end();
    detail::device_wrote(*v.state());
}

void vec_axpy_async(DenseVector& y, detail::ScalarArg alpha, const DenseVector& x, const Context& ctx,
                    std::string label)
{
    detail::same_len(x.size(), y.size(), "vec_axpy_async");
    detail::check_no_write_view(*x.state(), "vec_axpy_async");
    detail::check_no_write_view(*y.state(), "vec_axpy_async");
    runtime::log_kernel(KernelKind::Axpy, 2 * y.size());
    Launch L(ctx, detail::lab(std::move(label), "vec_axpy"));
    auto   s = detail::lower(alpha, ctx, L);
    L.read(x.id()).read_write(y.id());
    L.begin();
    check(rvk_axpy(ctx.handle(), (int64_t)y.size(), s.s, x.device_data(), y.device_data()),
          "vec_axpy_async");
    L.end();
    detail::device_wrote(*y.state());
}

void vec_aypx_async(DenseVector& y, detail::ScalarArg beta, const DenseVector& x, const Context& ctx,
                    std::string label)
{
    detail::same_len(x.size(), y.size(), "vec_aypx_async");
    detail::check_no_write_view(*x.state(), "vec_aypx_async");
    detail::check_no_write_view(*y.state(), "vec_aypx_async");
    runtime::log_kernel(KernelKind::Aypx, 2 * y.size());
    Launch L(ctx, detail::lab(std::move(label), "vec_aypx"));
    auto   s = detail::lower(beta, ctx, L);
    L.read(x.id()).read_write(y.id());
    L.begin();
    check(rvk_aypx(ctx.handle(), (int64_t)y.size(), s.s, x.device_data(), y.device_data()),
          "vec_aypx_async");
    L.end();
    detail::device_wrote(*y.state());
}

void vec_waxpy_async(DenseVector& w, detail::ScalarArg alpha, const DenseVector& x,
                     const DenseVector& y, const Context& ctx, std::string label)
{
    detail::same_len(x.size(), y.size(), "vec_waxpy_async");
    detail::same_len(x.size(), w.size(), "vec_waxpy_async");
    detail::check_no_write_view(*w.state(), "vec_waxpy_async");
    runtime::log_kernel(KernelKind::Waxpy, 2 * w.size());
    Launch L(ctx, detail::lab(std::move(label), "vec_waxpy"));
    auto   s = detail::lower(alpha, ctx, L);
    L.read(x.id()).read(y.id()).write(w.id());
    L.begin();
    check(rvk_waxpy(ctx.handle(), (int64_t)w.size(), s.s, x.device_data(), y.device_data(),
                    w.device_data()),
          "vec_waxpy_async");
    L.end();
    detail::device_wrote(*w.state());
}

void vec_copy_async(const DenseVector& src, DenseVector& dst, const Context& ctx, std::string label)
{
    detail::same_len(src.size(), dst.size(), "vec_copy_async");
    detail::check_no_write_view(*dst.state(), "vec_copy_async");
    runtime::log_kernel(KernelKind::Copy, 0);
    Launch L(ctx, detail::lab(std::move(label), "vec_copy"));
    L.read(src.id()).write(dst.id());
    L.begin();
    check(rvk_copy(ctx.handle(), (int64_t)src.size(), src.device_data(), dst.device_data()),
          "vec_copy_async");
    L.end();
    detail::device_wrote(*dst.state());
}

void vec_set_async(DenseVector& v, double value, const Context& ctx, std::string label)
{
    detail::check_no_write_view(*v.state(), "vec_set_async");
    runtime::log_kernel(KernelKind::Copy, 0);
    Launch L(ctx, detail::lab(std::move(label), "vec_set"));
    L.write(v.id());
    L.begin();
    check(rvk_set(ctx.handle(), (int64_t)v.size(), value, v.device_data()), "vec_set_async");
    L.end();
    detail::device_wrote(*v.state());
}

void vec_pointwise_mult_async(const DenseVector& a, const DenseVector& b, DenseVector& out,
                              const Context& ctx, std::string label)
{
    detail::same_len(a.size(), b.size(), "vec_pointwise_mult_async");
    detail::same_len(a.size(), out.size(), "vec_pointwise_mult_async");
    detail::check_no_write_view(*out.state(), "vec_pointwise_mult_async");
    // the Jacobi apply: a kernel in the census, 0 flops in SPEC's CG FlopLog
    // formula 2 nnz + 12 n + c
    runtime::log_kernel(KernelKind::PcApply, 0);
    Launch L(ctx, detail::lab(std::move(label), "vec_pointwise_mult"));
    L.read(a.id()).read(b.id()).write(out.id());
    L.begin();
    check(rvk_pointwise_mult(ctx.handle(), (int64_t)a.size(), a.device_data(), b.device_data(),
                             out.device_data()),
          "vec_pointwise_mult_async");
    L.end();
    detail::device_wrote(*out.state());
}

void mat_mult(const CsrMatrix& A, const DenseVector& x, DenseVector& y, const Context& ctx,
              std::string label)
{
    detail::same_len(A.cols(), x.size(), "mat_mult");
    detail::same_len(A.rows(), y.size(), "mat_mult");
    detail::check_no_write_view(*x.state(), "mat_mult");
    detail::check_no_write_view(*y.state(), "mat_mult");
    runtime::log_kernel(KernelKind::MatMult, 2 * A.nnz());
    Launch L(ctx, detail::lab(std::move(label), "mat_mult"));
    L.read(A.id()).read(x.id()).write(y.id());
    L.begin();
    const rvk_csr v = A.state()->view();
    check(rvk_csr_spmv(ctx.handle(), &v, x.device_data(), y.device_data()), "mat_mult");
    L.end();
    detail::device_wrote(*y.state());
}

void vec_aypx(DenseVector& y, double beta, const DenseVector& x)
{
    vec_aypx_async(y, beta, x, detail::global_sync_context(), "vec_aypx(sync)");
}

void mat_mult(const CsrMatrix& A, const DenseVector& x, DenseVector& y)
{
    mat_mult(A, x, y, detail::global_sync_context(), "mat_mult(sync)");
}

} // namespace rivulet
