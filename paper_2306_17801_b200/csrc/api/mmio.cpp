// mmio.cpp -- Matrix Market / raw vector I/O (include/rivulet/mmio.hpp;
// SPEC.md:432).  Host-side parsing into the reference's CSR layout (int64
// offsets, int32 columns, strictly increasing columns per row).
#include "rivulet/mmio.hpp"

#include <algorithm>
#include <cctype>
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <tuple>
#include <vector>

namespace rivulet {

namespace {
std::string lower(std::string s)
{
    for (auto& c : s) c = (char)std::tolower((unsigned char)c);
    return s;
}
} // namespace

CsrMatrix read_matrix_market(const std::string& path, std::string name)
{
    std::ifstream in(path);
    if (!in) throw Error("read_matrix_market: cannot open " + path);
    std::string line;
    if (!std::getline(in, line)) throw Error("read_matrix_market: empty file " + path);
    std::istringstream hs(line);
    std::string banner, object, format, field, symmetry;
    hs >> banner >> object >> format >> field >> symmetry;
    if (banner != "%%MatrixMarket" || lower(object) != "matrix" || lower(format) != "coordinate")
        throw Error("read_matrix_market: only '%%MatrixMarket matrix coordinate' is supported");
    field    = lower(field);
    symmetry = lower(symmetry);
    if (field != "real" && field != "integer" && field != "pattern")
        throw Error("read_matrix_market: field must be real, integer or pattern");
    if (symmetry != "general" && symmetry != "symmetric")
        throw Error("read_matrix_market: symmetry must be general or symmetric");
    const bool sym = symmetry == "symmetric", pattern = field == "pattern";
    while (std::getline(in, line))
        if (!line.empty() && line[0] != '%') break;
    long long nr = 0, nc = 0, nz = 0;
    if (std::sscanf(line.c_str(), "%lld %lld %lld", &nr, &nc, &nz) != 3 || nr < 0 || nc < 0 || nz < 0)
        throw Error("read_matrix_market: bad size line");
    if (nc > INT32_MAX) throw Error("read_matrix_market: more columns than int32 indices hold");
    std::vector<std::tuple<int64_t, int32_t, double, int64_t>> e; // row, col, value, file order
    e.reserve((size_t)(sym ? 2 * nz : nz));
    for (long long k = 0; k < nz; ++k) {
        long long i = 0, j = 0;
        double    v = 1.0;
        if (!(in >> i >> j)) throw Error("read_matrix_market: truncated entry list");
        if (!pattern && !(in >> v)) throw Error("read_matrix_market: missing value");
        if (i < 1 || i > nr || j < 1 || j > nc) throw Error("read_matrix_market: index out of range");
        e.emplace_back(i - 1, (int32_t)(j - 1), v, 2 * k);
        if (sym && i != j) e.emplace_back(j - 1, (int32_t)(i - 1), v, 2 * k + 1);
    }
    std::sort(e.begin(), e.end(), [](const auto& a, const auto& b) {
        return std::tie(std::get<0>(a), std::get<1>(a), std::get<3>(a)) <
               std::tie(std::get<0>(b), std::get<1>(b), std::get<3>(b));
    });
    std::vector<int64_t> off((size_t)nr + 1, 0);
    std::vector<int32_t> cols;
    std::vector<double>  vals;
    cols.reserve(e.size());
    vals.reserve(e.size());
    for (size_t k = 0; k < e.size(); ++k) {
        const auto& [i, j, v, o] = e[k];
        (void)o;
        if (!cols.empty() && k > 0 && std::get<0>(e[k - 1]) == i && std::get<1>(e[k - 1]) == j) {
            vals.back() += v; // duplicate: summed in file order
            continue;
        }
        cols.push_back(j);
        vals.push_back(v);
        off[(size_t)i + 1] += 1;
    }
    for (size_t r = 0; r < (size_t)nr; ++r) off[r + 1] += off[r];
    return CsrMatrix((size_t)nr, (size_t)nc, std::move(off), std::move(cols), std::move(vals),
                     std::move(name));
}

void write_matrix_market(const CsrMatrix& A, const std::string& path, bool symmetric)
{
    const auto off = A.row_offsets();
    const auto col = A.col_indices();
    const auto val = A.values();
    const size_t n = A.rows();
    auto value_at = [&](size_t r, int32_t c, double* v) {
        const int32_t* b = col.data() + off[r];
        const int32_t* e = col.data() + off[r + 1];
        const int32_t* it = std::lower_bound(b, e, c);
        if (it == e || *it != c) return false;
        *v = val[(size_t)(it - col.data())];
        return true;
    };
    size_t count = 0;
    if (symmetric) {
        if (A.rows() != A.cols()) throw Error("write_matrix_market: symmetric needs a square matrix");
        for (size_t r = 0; r < n; ++r)
            for (int64_t k = off[r]; k < off[r + 1]; ++k) {
                double t = 0.0;
                if (!value_at((size_t)col[k], (int32_t)r, &t) ||
                    std::memcmp(&t, &val[k], sizeof t) != 0)
                    throw Error("write_matrix_market: matrix is not symmetric");
                if ((size_t)col[k] <= r) ++count;
            }
    } else {
        count = A.nnz();
    }
    std::FILE* f = std::fopen(path.c_str(), "w");
    if (!f) throw Error("write_matrix_market: cannot open " + path);
    std::fprintf(f, "%%%%MatrixMarket matrix coordinate real %s\n", symmetric ? "symmetric" : "general");
    std::fprintf(f, "%% written by rivulet (B200 build)\n");
    std::fprintf(f, "%zu %zu %zu\n", A.rows(), A.cols(), count);
    for (size_t r = 0; r < n; ++r)
        for (int64_t k = off[r]; k < off[r + 1]; ++k)
            if (!symmetric || (size_t)col[k] <= r)
                std::fprintf(f, "%zu %d %.17g\n", r + 1, col[k] + 1, val[k]);
    if (std::fclose(f) != 0) throw Error("write_matrix_market: write failed for " + path);
}

void write_vector_binary(const DenseVector& v, const std::string& path)
{
    const auto    h = v.to_host();
    std::ofstream out(path, std::ios::binary);
    if (!out) throw Error("write_vector_binary: cannot open " + path);
    const int64_t n = (int64_t)h.size();
    out.write(reinterpret_cast<const char*>(&n), sizeof n);
    out.write(reinterpret_cast<const char*>(h.data()), (std::streamsize)(h.size() * sizeof(double)));
    if (!out) throw Error("write_vector_binary: write failed for " + path);
}

DenseVector read_vector_binary(const std::string& path, std::string name)
{
    std::ifstream in(path, std::ios::binary);
    if (!in) throw Error("read_vector_binary: cannot open " + path);
    int64_t n = -1;
    in.read(reinterpret_cast<char*>(&n), sizeof n);
    if (!in || n < 0) throw Error("read_vector_binary: bad header in " + path);
    std::vector<double> h((size_t)n);
    in.read(reinterpret_cast<char*>(h.data()), (std::streamsize)(h.size() * sizeof(double)));
    if (!in) throw Error("read_vector_binary: truncated " + path);
    return DenseVector(std::span<const double>(h), std::move(name));
}

} // namespace rivulet
