#pragma once
// rivulet (B200 build) -- CSR matrices in HBM.
// Drop-in for /root/reference/proj/include/rivulet/csr.hpp:19-85: same
// layout (int64 row offsets, int32 columns, double values) and the same
// construction-time validation (offsets start at 0, nondecreasing, end at nnz;
// columns in range and strictly increasing within a row).

#include "rivulet/common.hpp"
#include "rivulet/vector.hpp"

#include <cstdint>
#include <memory>
#include <span>
#include <string>
#include <vector>

struct rvk_csr_view;

namespace rivulet {

namespace detail {
struct MatState;
}

class CsrMatrix {
public:
    CsrMatrix() = default;
    CsrMatrix(std::size_t n_rows, std::size_t n_cols, std::vector<std::int64_t> row_offsets,
              std::vector<std::int32_t> col_indices, std::vector<double> values,
              std::string name = "");

    static CsrMatrix identity(std::size_t n, std::string name = "");

    std::size_t        rows() const;
    std::size_t        cols() const;
    std::size_t        nnz() const;
    ObjectId           id() const;
    const std::string& name() const;

    // Host views (downloaded once, on first request, for device-built matrices).
    std::span<const std::int64_t> row_offsets() const;
    std::span<const std::int32_t> col_indices() const;
    std::span<const double>       values() const;

    DenseVector diagonal(std::string name = "") const; // zero where absent
    void        evict_device() {}                      // device is the home copy

    const std::shared_ptr<detail::MatState>& state() const { return state_; }
    explicit CsrMatrix(std::shared_ptr<detail::MatState> s) : state_(std::move(s)) {}

private:
    std::shared_ptr<detail::MatState> state_;
};

} // namespace rivulet
