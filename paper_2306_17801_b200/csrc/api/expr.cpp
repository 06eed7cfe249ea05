// expr.cpp -- Managed futures and Expr/Eval/execute on the device.
//
// Semantics follow managed.cpp:9-105 and expr.cpp:96-386 of the reference:
// constant folding and common-subexpression sharing at Eval time, execute()
// = one kernel on the bound context reading every leaf (Read marks) and
// writing the target (Write mark); an expression assigned without Eval binds
// the globally-blocking context and is therefore synchronous.
#include "internal.hpp"
#include "rivulet/expr.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <sstream>
#include <tuple>

namespace rivulet {

using detail::ExprProgramDev;
using detail::ExprStep;

const char* to_string(UnaryOp op)
{
    static const char* n[] = {"neg", "abs", "sqrt", "sin", "cos", "exp"};
    return n[static_cast<int>(op)];
}
const char* to_string(BinaryOp op)
{
    static const char* n[] = {"add", "sub", "mul", "div", "min", "max"};
    return n[static_cast<int>(op)];
}

// ---- expression construction -------------------------------------------------------
Expr::Expr(const Managed& m)
{
    auto n     = std::make_shared<ExprNode>();
    n->kind    = ExprNode::Kind::Leaf;
    n->len     = m.size();
    n->leaf    = m.state();
    n->leaf_id = m.id();
    node_      = std::move(n);
}

Expr::Expr(double c)
{
    auto n   = std::make_shared<ExprNode>();
    n->kind  = ExprNode::Kind::Constant;
    n->value = c;
    node_    = std::move(n);
}

Expr make_unary(UnaryOp op, Expr child)
{
    auto n  = std::make_shared<ExprNode>();
    n->kind = ExprNode::Kind::Unary;
    n->uop  = op;
    n->len  = child.len();
    n->lhs  = child.node();
    return Expr(std::move(n));
}

Expr make_binary(BinaryOp op, Expr lhs, Expr rhs)
{
    const std::size_t a = lhs.len(), b = rhs.len();
    if (a != b && a != 1 && b != 1)
        throw Error("expression: operand lengths " + std::to_string(a) + " and " +
                    std::to_string(b) + " do not match");
    auto n  = std::make_shared<ExprNode>();
    n->kind = ExprNode::Kind::Binary;
    n->bop  = op;
    n->len  = std::max(a, b);
    n->lhs  = lhs.node();
    n->rhs  = rhs.node();
    return Expr(std::move(n));
}

// ---- Eval: fold + CSE into a linear device program ----------------------------------------
struct ExecutableExpression::Program {
    ExprProgramDev                                     dev{};
    std::vector<std::weak_ptr<detail::ManagedState>>   leaves;  // per step (null if not leaf)
    std::size_t                                        root_len = 1;
    std::vector<std::string>                           text;
};

namespace {

double host_unary(UnaryOp op, double a)
{
    switch (op) {
    case UnaryOp::Neg: return -a;
    case UnaryOp::Abs: return std::fabs(a);
    case UnaryOp::Sqrt: return std::sqrt(a);
    case UnaryOp::Sin: return std::sin(a);
    case UnaryOp::Cos: return std::cos(a);
    case UnaryOp::Exp: return std::exp(a);
    }
    return a;
}

double host_binary(BinaryOp op, double a, double b)
{
    switch (op) {
    case BinaryOp::Add: return a + b;
    case BinaryOp::Sub: return a - b;
    case BinaryOp::Mul: return a * b;
    case BinaryOp::Div: return a / b;
    case BinaryOp::Min: return std::fmin(a, b);
    case BinaryOp::Max: return std::fmax(a, b);
    }
    return a;
}

ExprNodePtr constant_node(double v)
{
    auto n   = std::make_shared<ExprNode>();
    n->kind  = ExprNode::Kind::Constant;
    n->value = v;
    return n;
}

// Constant folding (expr.cpp:96-132): all-constant subtrees collapse; the
// optional (e/z)*z -> e rewrite only under EvalOptions::algebraic_simplify.
ExprNodePtr fold(const ExprNodePtr& n, const EvalOptions& opt)
{
    using K = ExprNode::Kind;
    if (n->kind == K::Leaf || n->kind == K::Constant) return n;
    if (n->kind == K::Unary) {
        auto c = fold(n->lhs, opt);
        if (c->kind == K::Constant) return constant_node(host_unary(n->uop, c->value));
        if (c == n->lhs) return n;
        auto m = std::make_shared<ExprNode>(*n);
        m->lhs = c;
        return m;
    }
    auto a = fold(n->lhs, opt), b = fold(n->rhs, opt);
    if (a->kind == K::Constant && b->kind == K::Constant)
        return constant_node(host_binary(n->bop, a->value, b->value));
    if (opt.algebraic_simplify && n->bop == BinaryOp::Mul && a->kind == K::Binary &&
        a->bop == BinaryOp::Div && a->rhs == b)
        return a->lhs;
    if (a == n->lhs && b == n->rhs) return n;
    auto m = std::make_shared<ExprNode>(*n);
    m->lhs = a;
    m->rhs = b;
    return m;
}

struct Builder {
    ExecutableExpression::Program& prog;
    // structural key -> slot (hash-consing CSE, expr.cpp:136-171)
    std::map<std::tuple<int, int, int, int, ObjectId, std::uint64_t>, int> seen;
    std::map<const ExprNode*, int>                                          by_ptr;

    int intern(const ExprNodePtr& n)
    {
        auto hit = by_ptr.find(n.get());
        if (hit != by_ptr.end()) return hit->second;
        using K = ExprNode::Kind;
        ExprStep st{};
        int      a = -1, b = -1, op = 0;
        std::uint64_t bits = 0;
        ObjectId leaf = 0;
        std::string txt;
        switch (n->kind) {
        case K::Leaf: {
            auto s = n->leaf.lock();
            if (!s) throw Error("Eval: expression references a destroyed managed value");
            st.kind = 0;
            st.leaf = s->dev;
            st.len  = (std::uint32_t)n->len;
            leaf    = n->leaf_id;
            txt     = "leaf #" + std::to_string(leaf) + (s->name.empty() ? "" : " (" + s->name + ")");
            break;
        }
        case K::Constant:
            st.kind  = 1;
            st.value = n->value;
            std::memcpy(&bits, &n->value, sizeof bits);
            txt = "const " + std::to_string(n->value);
            break;
        case K::Unary:
            a       = intern(n->lhs);
            st.kind = 2;
            op = static_cast<int>(n->uop);
            txt = std::string(to_string(n->uop)) + " %" + std::to_string(a);
            break;
        case K::Binary:
            a       = intern(n->lhs);
            b       = intern(n->rhs);
            st.kind = 3;
            op = static_cast<int>(n->bop);
            txt = std::string(to_string(n->bop)) + " %" + std::to_string(a) + ", %" + std::to_string(b);
            break;
        }
        auto key = std::make_tuple((int)st.kind, op, a, b, leaf, bits);
        auto it  = seen.find(key);
        if (it != seen.end()) {
            by_ptr[n.get()] = it->second;
            return it->second;
        }
        if (prog.dev.n_steps >= detail::kMaxExprSteps) throw Error("Eval: expression too large");
        st.op  = (std::uint8_t)op;
        st.a   = (std::int16_t)a;
        st.b   = (std::int16_t)b;
        const int slot          = prog.dev.n_steps++;
        prog.dev.steps[slot]    = st;
        prog.leaves.push_back(st.kind == 0 ? n->leaf : std::weak_ptr<detail::ManagedState>{});
        prog.text.push_back(txt);
        seen.emplace(key, slot);
        by_ptr[n.get()] = slot;
        return slot;
    }
};

} // namespace

ExecutableExpression Eval(const Expr& expr, const Context& ctx, EvalOptions options)
{
    ExecutableExpression ee(ctx);
    auto                 prog = std::make_shared<ExecutableExpression::Program>();
    auto                 root = fold(expr.node(), options);
    Builder              b{*prog, {}, {}};
    b.intern(root);
    prog->root_len = root->len;
    std::size_t ops = 0;
    for (int s = 0; s < prog->dev.n_steps; ++s) {
        const auto& st = prog->dev.steps[s];
        if (st.kind == 2 || st.kind == 3) ++ops;
        if (st.kind == 0) {
            const ObjectId id = prog->leaves[s].lock() ? prog->leaves[s].lock()->id : 0;
            if (std::find(ee.leaf_ids_.begin(), ee.leaf_ids_.end(), id) == ee.leaf_ids_.end())
                ee.leaf_ids_.push_back(id);
        }
    }
    ee.op_count_ = ops;
    ee.program_  = std::move(prog);
    return ee;
}

ExecutableExpression Eval(const Expr& expr) { return Eval(expr, detail::global_sync_context()); }
ExecutableExpression Eval(const Managed& m, const Context& ctx) { return Eval(Expr(m), ctx); }
ExecutableExpression Eval(const Managed& m) { return Eval(Expr(m)); }

void ExecutableExpression::execute(Managed& target) const
{
    const auto& prog = *program_;
    const auto  n    = target.size();
    if (prog.root_len != n && prog.root_len != 1)
        throw Error("execute: target length " + std::to_string(n) +
                    " does not match expression length " + std::to_string(prog.root_len));
    // keep every leaf alive until the kernel has been enqueued and marked
    std::vector<std::shared_ptr<detail::ManagedState>> locked;
    ExprProgramDev dev = prog.dev;
    for (int s = 0; s < dev.n_steps; ++s) {
        if (dev.steps[s].kind != 0) continue;
        auto st = prog.leaves[s].lock();
        if (!st) throw Error("execute: expression references a destroyed managed value");
        dev.steps[s].leaf = st->dev;
        locked.push_back(std::move(st));
    }
    runtime::log_kernel(runtime::KernelKind::ExprEval, static_cast<std::uint64_t>(op_count_) * n);
    detail::Launch L(context_, "eval(" + (target.name().empty() ? "tmp" : target.name()) + ")");
    for (auto& st : locked) L.read(st->id);
    L.write(target.id());
    L.begin();
    detail::check(detail::expr_run(reinterpret_cast<cudaStream_t>(context_.cuda_stream()), dev,
                                   target.device_data(), n),
                  "execute");
    auto ev = L.end();
    target.state()->mark_written(ev, context_.id());
    if (context_.stream_type() == StreamType::GloballyBlocking) target.state()->pending.reset();
}

std::string ExecutableExpression::debug_string() const
{
    std::ostringstream os;
    for (std::size_t s = 0; s < program_->text.size(); ++s)
        os << '%' << s << " = " << program_->text[s] << '\n';
    return os.str();
}

// ---- Managed -----------------------------------------------------------------------------
Managed::Managed(double value, std::string name)
    : state_(std::make_shared<detail::ManagedState>(1, std::move(name)))
{
    *this = value;
}

Managed::Managed(std::span<const double> values, std::string name)
    : state_(std::make_shared<detail::ManagedState>(values.size(), std::move(name)))
{
    detail::check_cuda(cudaMemcpy(state_->dev, values.data(), values.size_bytes(),
                                  cudaMemcpyHostToDevice),
                       "Managed(values)");
    runtime::log_h2d(values.size_bytes());
    state_->host.assign(values.begin(), values.end());
    state_->host_valid = true;
}

Managed::Managed(const Expr& expr) : state_(std::make_shared<detail::ManagedState>(expr.len(), ""))
{
    Eval(expr).execute(*this);
}

Managed::Managed(const Expr& expr, const Context& ctx)
    : state_(std::make_shared<detail::ManagedState>(expr.len(), ""))
{
    Eval(expr, ctx).execute(*this);
}

Managed::Managed(const ExecutableExpression& ee)
    : state_(std::make_shared<detail::ManagedState>(1, ""))
{
    ee.execute(*this);
}

Managed::Managed(const Managed& other)
    : state_(std::make_shared<detail::ManagedState>(other.size(), other.name()))
{
    Eval(Expr(other)).execute(*this); // synchronous snapshot (managed.cpp:40-45)
}

Managed& Managed::operator=(const Managed& other)
{
    if (state_ != other.state_) Eval(Expr(other)).execute(*this);
    return *this;
}

Managed& Managed::operator=(const Expr& expr)
{
    Eval(expr).execute(*this);
    return *this;
}

Managed& Managed::operator=(const ExecutableExpression& ee)
{
    ee.execute(*this);
    return *this;
}

Managed& Managed::operator=(double value)
{
    // wait for in-flight readers/writers, then store (managed.cpp:65-72)
    detail::Tracker::get().await_host(id(), detail::Mode::Write);
    std::vector<double> v(size(), value);
    detail::check_cuda(cudaMemcpy(state_->dev, v.data(), v.size() * sizeof(double),
                                  cudaMemcpyHostToDevice),
                       "Managed::operator=");
    state_->pending.reset();
    state_->pending_ctx = 0;
    state_->host        = std::move(v);
    state_->host_valid  = true;
    return *this;
}

double Managed::at(std::size_t i)
{
    if (i >= size()) throw Error("Managed::at: index out of range");
    if (!state_->host_valid) {
        // implicit synchronisation with the pending producer (managed.cpp:74-91)
        detail::Tracker::get().await_host(id(), detail::Mode::Read);
        {
            rvk::trace::HostSyncScope hs("Managed::front", 0, true); // counted + traced
            detail::check_cuda(cudaMemcpy(state_->host.data(), state_->dev, size() * sizeof(double),
                                          cudaMemcpyDeviceToHost),
                               "Managed::front");
        }
        runtime::log_d2h(size() * sizeof(double));
        state_->host_valid  = true;
        state_->pending.reset();
        state_->pending_ctx = 0;
    }
    return state_->host[i];
}

double Managed::front() { return at(0); }

std::size_t        Managed::size() const { return state_->n; }
ObjectId           Managed::id() const { return state_->id; }
const std::string& Managed::name() const { return state_->name; }
Managed::Validity  Managed::validity() const
{
    return state_->pending ? Validity::PendingOnContext : Validity::HostValid;
}
ObjectId      Managed::pending_context() const { return state_->pending_ctx; }
double*       Managed::device_data() { return state_->dev; }
const double* Managed::device_data() const { return state_->dev; }

} // namespace rivulet
