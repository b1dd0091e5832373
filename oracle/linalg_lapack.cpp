// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// Eigen-free restatement of the reference's numerics layer so that the
// reference's own decode/cache/compressor sources (compiled unmodified from
// /root/reference/proj/src by oracle/Makefile) link without Eigen 3.4, which
// is absent from this image.  Every function implements the contract declared
// in /root/reference/proj/include/kvpack/linalg.hpp:21-58 and follows the
// algorithm of /root/reference/proj/src/linalg.cpp:
//
//   check_svd_input       linalg.cpp:15-24
//   exact SVD             linalg.cpp:48-63  (Eigen::BDCSVD  -> LAPACK ?gesdd,
//                                            the same divide-and-conquer family)
//   zero-matrix rule      linalg.cpp:51-59  (left = 0, right = coordinate rows)
//   split_factors         linalg.cpp:30-46  (sigma folded into left)
//   randomized SVD        linalg.cpp:68-105 (sketch = min(R+p, min(T,W)),
//                                            Omega = gaussian_matrix(W x k, seed,
//                                            stream 0x72737664), Householder QR
//                                            (Eigen::HouseholderQR -> ?geqrf+?orgqr),
//                                            q power iterations A^T Q, A Q, then
//                                            B = Q^T A and an exact SVD of B)
//   singular_values       linalg.cpp:118-128 (always in double)
//   explained_variance    linalg.cpp:130-142
//   rank_for_variance     linalg.cpp:144-165
//   matmul                linalg.cpp:167-173 (Eigen GEMM -> ?gemm)
//   gaussian_matrix       linalg.cpp:175-182 (Philox stream, Box-Muller pairs)
//
// Backed by the LAPACK/BLAS shipped inside scipy's wheel
// (scipy.libs/libscipy_openblas-*.so, symbols prefixed "scipy_").
// Factors can differ from Eigen's by column signs / rotations inside
// repeated singular values; parity is therefore always judged on
// reconstructions (SURVEY.md §8c "Parity protocol").
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "kvpack/linalg.hpp"
#include "kvpack/rng.hpp"

extern "C" {
int scipy_LAPACKE_dgesdd(int layout, char jobz, int m, int n, double* a, int lda, double* s,
                         double* u, int ldu, double* vt, int ldvt);
int scipy_LAPACKE_sgesdd(int layout, char jobz, int m, int n, float* a, int lda, float* s,
                         float* u, int ldu, float* vt, int ldvt);
int scipy_LAPACKE_dgeqrf(int layout, int m, int n, double* a, int lda, double* tau);
int scipy_LAPACKE_sgeqrf(int layout, int m, int n, float* a, int lda, float* tau);
int scipy_LAPACKE_dorgqr(int layout, int m, int n, int k, double* a, int lda, const double* tau);
int scipy_LAPACKE_sorgqr(int layout, int m, int n, int k, float* a, int lda, const float* tau);
void scipy_dgemm_(const char* ta, const char* tb, const int* m, const int* n, const int* k,
                  const double* alpha, const double* a, const int* lda, const double* b,
                  const int* ldb, const double* beta, double* c, const int* ldc, std::size_t,
                  std::size_t);
void scipy_sgemm_(const char* ta, const char* tb, const int* m, const int* n, const int* k,
                  const float* alpha, const float* a, const int* lda, const float* b,
                  const int* ldb, const float* beta, float* c, const int* ldc, std::size_t,
                  std::size_t);
}

namespace kvpack {
namespace {

constexpr int kRowMajor = 101;

// ---- thin typed LAPACK/BLAS adaptors -------------------------------------
int gesdd(int m, int n, double* a, double* s, double* u, double* vt) {
    const int k = std::min(m, n);
    return scipy_LAPACKE_dgesdd(kRowMajor, 'S', m, n, a, n, s, u, k, vt, n);
}
int gesdd(int m, int n, float* a, float* s, float* u, float* vt) {
    const int k = std::min(m, n);
    return scipy_LAPACKE_sgesdd(kRowMajor, 'S', m, n, a, n, s, u, k, vt, n);
}
int gesdd_values(int m, int n, double* a, double* s) {
    return scipy_LAPACKE_dgesdd(kRowMajor, 'N', m, n, a, n, s, nullptr, 1, nullptr, 1);
}
int geqrf(int m, int n, double* a, double* tau) { return scipy_LAPACKE_dgeqrf(kRowMajor, m, n, a, n, tau); }
int geqrf(int m, int n, float* a, float* tau) { return scipy_LAPACKE_sgeqrf(kRowMajor, m, n, a, n, tau); }
int orgqr(int m, int n, int k, double* a, int lda, const double* tau) {
    return scipy_LAPACKE_dorgqr(kRowMajor, m, n, k, a, lda, tau);
}
int orgqr(int m, int n, int k, float* a, int lda, const float* tau) {
    return scipy_LAPACKE_sorgqr(kRowMajor, m, n, k, a, lda, tau);
}

// Row-major C(m x n) = op(A) * op(B); transposes expressed by swapping the
// column-major roles (C^T = op(B)^T op(A)^T).
void gemm_rm(bool ta, bool tb, int m, int n, int k, const double* a, const double* b, double* c) {
    const double one = 1.0, zero = 0.0;
    const int lda = ta ? m : k, ldb = tb ? k : n, ldc = n;
    const char cta = ta ? 'T' : 'N', ctb = tb ? 'T' : 'N';
    scipy_dgemm_(&ctb, &cta, &n, &m, &k, &one, b, &ldb, a, &lda, &zero, c, &ldc, 1, 1);
}
void gemm_rm(bool ta, bool tb, int m, int n, int k, const float* a, const float* b, float* c) {
    const float one = 1.0f, zero = 0.0f;
    const int lda = ta ? m : k, ldb = tb ? k : n, ldc = n;
    const char cta = ta ? 'T' : 'N', ctb = tb ? 'T' : 'N';
    scipy_sgemm_(&ctb, &cta, &n, &m, &k, &one, b, &ldb, a, &lda, &zero, c, &ldc, 1, 1);
}

template <typename T>
void lapack_check(int info, const char* what) {
    if (info != 0) throw data_error(std::string("oracle linalg: LAPACK failure in ") + what);
}

template <typename T>
void validate_svd_args(const Matrix<T>& m, std::size_t rank) {
    if (m.rows == 0 || m.cols == 0) throw shape_error("truncated_svd: matrix must be non-empty");
    if (rank < 1 || rank > std::min(m.rows, m.cols))
        throw parameter_error("truncated_svd: rank must be in [1, min(rows, cols)]");
    if (!m.all_finite()) throw data_error("truncated_svd: matrix contains non-finite values");
}

template <typename T>
bool is_zero(const Matrix<T>& m) {
    return std::all_of(m.data.begin(), m.data.end(), [](T v) { return v == T(0); });
}

template <typename T>
FactorPair<T> zero_factors(std::size_t rows, std::size_t cols, std::size_t rank) {
    FactorPair<T> f;
    f.left = Matrix<T>(rows, rank);
    f.right = Matrix<T>(rank, cols);
    for (std::size_t r = 0; r < rank; ++r) f.right(r, r) = T(1);
    return f;
}

// Thin SVD of a (rows x cols) row-major buffer; returns U (rows x k),
// s (k), Vt (k x cols), k = min(rows, cols).
template <typename T>
void thin_svd(std::size_t rows, std::size_t cols, std::vector<T> a, std::vector<T>& u,
              std::vector<T>& s, std::vector<T>& vt) {
    const std::size_t k = std::min(rows, cols);
    u.assign(rows * k, T(0));
    s.assign(k, T(0));
    vt.assign(k * cols, T(0));
    lapack_check<T>(gesdd(int(rows), int(cols), a.data(), s.data(), u.data(), vt.data()), "gesdd");
}

// sigma-scaled left columns, orthonormal right rows, truncated to `rank`.
template <typename T>
FactorPair<T> fold_sigma(std::size_t rows, std::size_t cols, const std::vector<T>& u,
                         const std::vector<T>& s, const std::vector<T>& vt, std::size_t k,
                         std::size_t rank) {
    FactorPair<T> f;
    f.left = Matrix<T>(rows, rank);
    f.right = Matrix<T>(rank, cols);
    for (std::size_t i = 0; i < rows; ++i)
        for (std::size_t r = 0; r < rank; ++r) f.left(i, r) = u[i * k + r] * s[r];
    for (std::size_t r = 0; r < rank; ++r)
        for (std::size_t j = 0; j < cols; ++j) f.right(r, j) = vt[r * cols + j];
    return f;
}

template <typename T>
FactorPair<T> exact_factor(const Matrix<T>& m, std::size_t rank) {
    if (is_zero(m)) return zero_factors<T>(m.rows, m.cols, rank);
    std::vector<T> u, s, vt;
    thin_svd<T>(m.rows, m.cols, m.data, u, s, vt);
    return fold_sigma<T>(m.rows, m.cols, u, s, vt, std::min(m.rows, m.cols), rank);
}

// Orthonormal basis of the column space of y (rows x cols), Householder QR,
// returned as rows x min(rows, cols).
template <typename T>
std::vector<T> householder_basis(std::size_t rows, std::size_t cols, const std::vector<T>& y,
                                 std::size_t& out_cols) {
    const std::size_t k = std::min(rows, cols);
    std::vector<T> a = y;
    std::vector<T> tau(k);
    lapack_check<T>(geqrf(int(rows), int(cols), a.data(), tau.data()), "geqrf");
    // orgqr wants the leading k columns; compact them into a rows x k buffer.
    std::vector<T> q(rows * k);
    for (std::size_t i = 0; i < rows; ++i)
        for (std::size_t j = 0; j < k; ++j) q[i * k + j] = a[i * cols + j];
    lapack_check<T>(orgqr(int(rows), int(k), int(k), q.data(), int(k), tau.data()), "orgqr");
    out_cols = k;
    return q;
}

template <typename T>
FactorPair<T> sketch_factor(const Matrix<T>& m, std::size_t rank, const SvdOptions& opts) {
    if (is_zero(m)) return exact_factor(m, rank);
    const std::size_t rows = m.rows, cols = m.cols;
    const std::size_t k = std::min(rank + opts.oversampling, std::min(rows, cols));
    const Matrix<T> omega = gaussian_matrix<T>(cols, k, opts.seed, 0x72737664ull);

    // Y = A * Omega  (rows x k)
    std::vector<T> y(rows * k);
    gemm_rm(false, false, int(rows), int(k), int(cols), m.data.data(), omega.data.data(), y.data());
    std::size_t qc = 0;
    std::vector<T> q = householder_basis<T>(rows, k, y, qc);
    for (std::size_t it = 0; it < opts.power_iterations; ++it) {
        std::vector<T> z(cols * qc); // A^T Q : cols x qc
        gemm_rm(true, false, int(cols), int(qc), int(rows), m.data.data(), q.data(), z.data());
        std::size_t zc = 0;
        std::vector<T> zq = householder_basis<T>(cols, qc, z, zc);
        std::vector<T> w(rows * zc); // A Z : rows x zc
        gemm_rm(false, false, int(rows), int(zc), int(cols), m.data.data(), zq.data(), w.data());
        q = householder_basis<T>(rows, zc, w, qc);
    }
    // B = Q^T A : qc x cols, then its exact SVD.
    std::vector<T> b(qc * cols);
    gemm_rm(true, false, int(qc), int(cols), int(rows), q.data(), m.data.data(), b.data());
    std::vector<T> ub, s, vt;
    thin_svd<T>(qc, cols, b, ub, s, vt);
    const std::size_t kb = std::min(qc, cols);
    // left = (Q * Ub)[:, :rank] * sigma
    std::vector<T> qu(rows * kb);
    gemm_rm(false, false, int(rows), int(kb), int(qc), q.data(), ub.data(), qu.data());
    return fold_sigma<T>(rows, cols, qu, s, vt, kb, rank);
}

} // namespace

template <typename T>
FactorPair<T> truncated_svd(const Matrix<T>& m, std::size_t rank, const SvdOptions& opts) {
    validate_svd_args(m, rank);
    return opts.method == SvdMethod::randomized ? sketch_factor(m, rank, opts)
                                                : exact_factor(m, rank);
}

template <typename T>
std::vector<double> singular_values(const Matrix<T>& m) {
    if (m.rows == 0 || m.cols == 0) throw shape_error("singular_values: matrix must be non-empty");
    std::vector<double> a(m.data.begin(), m.data.end());
    std::vector<double> s(std::min(m.rows, m.cols));
    lapack_check<double>(gesdd_values(int(m.rows), int(m.cols), a.data(), s.data()), "gesdd");
    return s;
}

template <typename T>
double explained_variance_ratio(const Matrix<T>& m, std::size_t rank) {
    if (rank > std::min(m.rows, m.cols))
        throw parameter_error("explained_variance_ratio: rank exceeds min(rows, cols)");
    const std::vector<double> s = singular_values(m);
    double all = 0.0, lead = 0.0;
    for (std::size_t i = 0; i < s.size(); ++i) {
        all += s[i] * s[i];
        if (i < rank) lead += s[i] * s[i];
    }
    return all == 0.0 ? 1.0 : lead / all;
}

template <typename T>
VarianceRank rank_for_variance(const Matrix<T>& m, double target, std::size_t max_rank) {
    if (!(target > 0.0) || target > 1.0)
        throw parameter_error("rank_for_variance: target must be in (0, 1]");
    if (max_rank < 1) throw parameter_error("rank_for_variance: max_rank must be >= 1");
    const std::size_t cap = std::min(max_rank, std::min(m.rows, m.cols));
    const std::vector<double> s = singular_values(m);
    double all = 0.0;
    for (double v : s) all += v * v;
    if (all == 0.0) return {1, 1.0};
    VarianceRank out;
    double lead = 0.0;
    for (std::size_t r = 1; r <= cap; ++r) {
        lead += s[r - 1] * s[r - 1];
        out.rank = r;
        out.achieved = lead / all;
        if (out.achieved >= target) break;
    }
    return out;
}

template <typename T>
Matrix<T> matmul(const Matrix<T>& a, const Matrix<T>& b) {
    if (a.cols != b.rows) throw shape_error("matmul: inner dimensions disagree");
    Matrix<T> c(a.rows, b.cols);
    if (a.rows && b.cols && a.cols)
        gemm_rm(false, false, int(a.rows), int(b.cols), int(a.cols), a.data.data(), b.data.data(),
                c.data.data());
    return c;
}

template <typename T>
Matrix<T> gaussian_matrix(std::size_t rows, std::size_t cols, std::uint64_t seed,
                          std::uint64_t stream) {
    Philox4x32 gen(seed, stream);
    Matrix<T> g(rows, cols);
    for (T& v : g.data) v = static_cast<T>(gen.next_gaussian());
    return g;
}

#define ORACLE_LINALG(T)                                                                      \
    template FactorPair<T> truncated_svd<T>(const Matrix<T>&, std::size_t, const SvdOptions&); \
    template std::vector<double> singular_values<T>(const Matrix<T>&);                         \
    template double explained_variance_ratio<T>(const Matrix<T>&, std::size_t);                \
    template VarianceRank rank_for_variance<T>(const Matrix<T>&, double, std::size_t);         \
    template Matrix<T> matmul<T>(const Matrix<T>&, const Matrix<T>&);                          \
    template Matrix<T> gaussian_matrix<T>(std::size_t, std::size_t, std::uint64_t, std::uint64_t);
ORACLE_LINALG(float)
ORACLE_LINALG(double)
#undef ORACLE_LINALG

} // namespace kvpack
