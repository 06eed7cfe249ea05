// data.cpp -- DenseVector / CsrMatrix storage and host views.
#include "internal.hpp"

#include <algorithm>
#include <cstring>

namespace rivulet {

using detail::Mode;
using detail::Tracker;

// ---- host views ----------------------------------------------------------------------
ArrayRead::ArrayRead(std::shared_ptr<detail::VecState> s, std::span<const double> sp)
    : state_(std::move(s)), span_(sp)
{
}
ArrayRead::ArrayRead(ArrayRead&& o) noexcept : state_(std::move(o.state_)), span_(o.span_) {}
ArrayRead& ArrayRead::operator=(ArrayRead&& o) noexcept
{
    if (this != &o) {
        restore();
        state_ = std::move(o.state_);
        span_  = o.span_;
    }
    return *this;
}
ArrayRead::~ArrayRead() { restore(); }
void ArrayRead::restore()
{
    if (!state_) return;
    std::lock_guard lk(state_->view_mutex);
    --state_->read_views;
    state_.reset();
}

ArrayWrite::ArrayWrite(std::shared_ptr<detail::VecState> s, std::span<double> sp)
    : state_(std::move(s)), span_(sp)
{
}
ArrayWrite::ArrayWrite(ArrayWrite&& o) noexcept : state_(std::move(o.state_)), span_(o.span_) {}
ArrayWrite& ArrayWrite::operator=(ArrayWrite&& o) noexcept
{
    if (this != &o) {
        restore();
        state_ = std::move(o.state_);
        span_  = o.span_;
    }
    return *this;
}
ArrayWrite::~ArrayWrite() { restore(); }
void ArrayWrite::restore()
{
    if (!state_) return;
    auto& v = *state_;
    // publish the host data: the device copy is the home of the vector
    if (v.n) {
        detail::check_cuda(cudaMemcpy(v.dev, v.host.data(), v.n * sizeof(double),
                                      cudaMemcpyHostToDevice),
                           "ArrayWrite::restore");
        runtime::log_h2d(v.n * sizeof(double));
    }
    v.host_valid = true;
    std::lock_guard lk(v.view_mutex);
    --v.write_views;
    state_.reset();
}

// ---- DenseVector --------------------------------------------------------------------------
DenseVector::DenseVector(std::size_t n, std::string name)
    : state_(std::make_shared<detail::VecState>(n, name.empty() ? "vec" : std::move(name)))
{
    if (n) detail::check_cuda(cudaMemset(state_->dev, 0, n * sizeof(double)), "DenseVector");
    state_->host.assign(n, 0.0);
    state_->host_valid = true;
}

DenseVector::DenseVector(std::span<const double> values, std::string name)
    : state_(std::make_shared<detail::VecState>(values.size(), name.empty() ? "vec" : std::move(name)))
{
    if (!values.empty()) {
        detail::check_cuda(cudaMemcpy(state_->dev, values.data(), values.size_bytes(),
                                      cudaMemcpyHostToDevice),
                           "DenseVector(values)");
        runtime::log_h2d(values.size_bytes());
    }
    state_->host.assign(values.begin(), values.end());
    state_->host_valid = true;
}

std::size_t        DenseVector::size() const { return state_->n; }
ObjectId           DenseVector::id() const { return state_->id; }
const std::string& DenseVector::name() const { return state_->name; }
bool               DenseVector::device_resident() const { return true; }
double*            DenseVector::device_data() { return state_->dev; }
const double*      DenseVector::device_data() const { return state_->dev; }

namespace {
void pull_host(detail::VecState& v)
{
    if (v.host_valid) return;
    v.host.resize(v.n);
    if (v.n) {
        detail::check_cuda(cudaMemcpy(v.host.data(), v.dev, v.n * sizeof(double),
                                      cudaMemcpyDeviceToHost),
                           "DenseVector host view");
        runtime::log_d2h(v.n * sizeof(double));
    }
    v.host_valid = true;
}
} // namespace

ArrayRead DenseVector::array_read() const
{
    auto& v = *state_;
    {
        std::lock_guard lk(v.view_mutex);
        if (v.write_views) throw Error("array_read: vector has an open write view");
        ++v.read_views;
    }
    Tracker::get().await_host(v.id, Mode::Read); // implicit sync with the last writer
    pull_host(v);
    return ArrayRead(state_, std::span<const double>(v.host.data(), v.n));
}

ArrayWrite DenseVector::array_write()
{
    auto& v = *state_;
    {
        std::lock_guard lk(v.view_mutex);
        if (v.write_views || v.read_views) throw Error("array_write: vector has an open view");
        ++v.write_views;
    }
    Tracker::get().await_host(v.id, Mode::Write); // writer and readers must be done
    v.host.resize(v.n);
    return ArrayWrite(state_, std::span<double>(v.host.data(), v.n));
}

ArrayWrite DenseVector::array_read_write()
{
    auto& v = *state_;
    {
        std::lock_guard lk(v.view_mutex);
        if (v.write_views || v.read_views) throw Error("array_read_write: vector has an open view");
        ++v.write_views;
    }
    Tracker::get().await_host(v.id, Mode::Write);
    pull_host(v);
    return ArrayWrite(state_, std::span<double>(v.host.data(), v.n));
}

std::vector<double> DenseVector::to_host() const
{
    auto r = array_read();
    return std::vector<double>(r.span().begin(), r.span().end());
}

void DenseVector::evict_device()
{
    // The device copy is the home of the vector: dropping the host mirror is
    // the analogue of the reference's eviction (dual_buffer.cpp:64-75).
    Tracker::get().await_host(state_->id, Mode::Read);
    state_->host_valid = false;
}

// ---- CsrMatrix ----------------------------------------------------------------------------
namespace {
void validate_host(std::size_t n_rows, std::size_t n_cols, const std::vector<std::int64_t>& off,
                   const std::vector<std::int32_t>& cols, const std::vector<double>& vals)
{
    // csr.hpp:46-53
    if (off.size() != n_rows + 1) throw Error("CsrMatrix: row_offsets must have n_rows+1 entries");
    if (cols.size() != vals.size()) throw Error("CsrMatrix: col_indices/values length mismatch");
    if (off[0] != 0) throw Error("CsrMatrix: row_offsets[0] != 0");
    if ((std::size_t)off[n_rows] != cols.size()) throw Error("CsrMatrix: row_offsets[n_rows] != nnz");
    if (n_cols > (std::size_t)INT32_MAX) throw Error("CsrMatrix: n_cols exceeds int32 indices");
    for (std::size_t r = 0; r < n_rows; ++r) {
        if (off[r + 1] < off[r]) throw Error("CsrMatrix: row_offsets decreasing");
        for (auto k = off[r]; k < off[r + 1]; ++k) {
            if (cols[k] < 0 || (std::size_t)cols[k] >= n_cols)
                throw Error("CsrMatrix: column index out of range");
            if (k > off[r] && cols[k] <= cols[k - 1])
                throw Error("CsrMatrix: columns not strictly increasing in a row");
        }
    }
}

template <class T>
T* upload(const std::vector<T>& h)
{
    T* d = static_cast<T*>(detail::device_alloc(h.size() * sizeof(T)));
    if (!h.empty()) {
        detail::check_cuda(cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice),
                           "CsrMatrix upload");
        runtime::log_h2d(h.size() * sizeof(T));
    }
    return d;
}
} // namespace

CsrMatrix::CsrMatrix(std::size_t n_rows, std::size_t n_cols, std::vector<std::int64_t> off,
                     std::vector<std::int32_t> cols, std::vector<double> vals, std::string name)
    : state_(std::make_shared<detail::MatState>(name.empty() ? "mat" : std::move(name)))
{
    validate_host(n_rows, n_cols, off, cols, vals);
    auto& m  = *state_;
    m.n_rows = n_rows;
    m.n_cols = n_cols;
    m.nnz    = cols.size();
    for (std::size_t r = 0; r < n_rows; ++r) m.max_row_len = std::max(m.max_row_len, off[r + 1] - off[r]);
    m.off    = upload(off);
    m.cols   = upload(cols);
    m.vals   = upload(vals);
    m.h_off  = std::move(off);
    m.h_cols = std::move(cols);
    m.h_vals = std::move(vals);
    m.host_loaded = true;
}

CsrMatrix CsrMatrix::identity(std::size_t n, std::string name)
{
    std::vector<std::int64_t> off(n + 1);
    std::vector<std::int32_t> cols(n);
    for (std::size_t i = 0; i <= n; ++i) off[i] = (std::int64_t)i;
    for (std::size_t i = 0; i < n; ++i) cols[i] = (std::int32_t)i;
    return CsrMatrix(n, n, std::move(off), std::move(cols), std::vector<double>(n, 1.0),
                     std::move(name));
}

std::size_t        CsrMatrix::rows() const { return state_->n_rows; }
std::size_t        CsrMatrix::cols() const { return state_->n_cols; }
std::size_t        CsrMatrix::nnz() const { return state_->nnz; }
ObjectId           CsrMatrix::id() const { return state_->id; }
const std::string& CsrMatrix::name() const { return state_->name; }

namespace {
void load_host(detail::MatState& m)
{
    std::lock_guard lk(m.host_mutex);
    if (m.host_loaded) return;
    Tracker::get().await_host(m.id, Mode::Read);
    m.h_off.resize(m.n_rows + 1);
    m.h_cols.resize(m.nnz);
    m.h_vals.resize(m.nnz);
    detail::check_cuda(cudaMemcpy(m.h_off.data(), m.off, m.h_off.size() * 8, cudaMemcpyDeviceToHost), "csr");
    if (m.nnz) {
        detail::check_cuda(cudaMemcpy(m.h_cols.data(), m.cols, m.nnz * 4, cudaMemcpyDeviceToHost), "csr");
        detail::check_cuda(cudaMemcpy(m.h_vals.data(), m.vals, m.nnz * 8, cudaMemcpyDeviceToHost), "csr");
    }
    runtime::log_d2h((m.n_rows + 1) * 8 + m.nnz * 12);
    m.host_loaded = true;
}
} // namespace

std::span<const std::int64_t> CsrMatrix::row_offsets() const
{
    load_host(*state_);
    return state_->h_off;
}
std::span<const std::int32_t> CsrMatrix::col_indices() const
{
    load_host(*state_);
    return state_->h_cols;
}
std::span<const double> CsrMatrix::values() const
{
    load_host(*state_);
    return state_->h_vals;
}

DenseVector CsrMatrix::diagonal(std::string name) const
{
    DenseVector d(rows(), std::move(name));
    const Context& g = detail::global_sync_context();
    detail::Launch L(g, "diagonal");
    L.read(id()).write(d.id());
    L.begin();
    const rvk_csr v = state_->view();
    detail::check(rvk_csr_diagonal(g.handle(), &v, d.device_data()), "CsrMatrix::diagonal");
    L.end();
    detail::device_wrote(*d.state());
    return d;
}

} // namespace rivulet
