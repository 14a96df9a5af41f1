// Port of the reference's hot-path C++ tests (proj/tests/test_decompose.cpp,
// proj/tests/test_workspace.cpp identity cases, the diagonal-weight cases of
// test_decompose.cpp:88-126,208-229 and the container cases of
// test_io.cpp:273-345) onto the B200 C++ mirror
// (include/rbd/*.hpp). Same fixtures (helpers.hpp:14-26 draws), same
// assertions and tolerances. Exit code = number of failed checks.
#include <cmath>
#include <cstdint>
#include <filesystem>
#include <fstream>
#include <string>
#include <cstdio>
#include <limits>
#include <random>

#include "rbd/decompose.hpp"
#include "rbd/io.hpp"
#include "rbd/workspace.hpp"

using namespace rbd;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                          \
  do {                                                                    \
    ++g_checks;                                                           \
    if (!(c)) {                                                           \
      ++g_fail;                                                           \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);            \
    }                                                                     \
  } while (0)
#define CHECK_THROWS_AS(expr, T)                                          \
  do {                                                                    \
    ++g_checks;                                                           \
    bool ok_ = false;                                                     \
    try {                                                                 \
      (void)(expr);                                                       \
    } catch (const T&) {                                                  \
      ok_ = true;                                                         \
    } catch (...) {                                                       \
    }                                                                     \
    if (!ok_) {                                                           \
      ++g_fail;                                                           \
      std::printf("FAIL %s:%d: %s does not throw %s\n", __FILE__, __LINE__, #expr, #T); \
    }                                                                     \
  } while (0)

// ---- helpers.hpp:14-26 ----
static Matrix random_matrix(Index m, Index n, std::uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> gauss;
  Matrix x(m, n);
  for (Index j = 0; j < n; ++j)
    for (Index i = 0; i < m; ++i) x(i, j) = gauss(rng);
  return x;
}
static Matrix matmul(const Matrix& a, const Matrix& b) {
  Matrix c(a.rows(), b.cols());
  for (Index j = 0; j < b.cols(); ++j)
    for (Index k = 0; k < a.cols(); ++k)
      for (Index i = 0; i < a.rows(); ++i) c(i, j) += a(i, k) * b(k, j);
  return c;
}
static Matrix transpose(const Matrix& a) {
  Matrix t(a.cols(), a.rows());
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) t(j, i) = a(i, j);
  return t;
}
static double max_abs_diff(const Matrix& a, const Matrix& b) {
  double m = 0.0;
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) m = std::max(m, std::abs(a(i, j) - b(i, j)));
  return m;
}
static double orthonormality_defect(const Matrix& y) {
  return max_abs_diff(matmul(transpose(y), y), Matrix::Identity(y.cols(), y.cols()));
}
// helpers.hpp:28-34
static Vector random_positive(Index n, std::uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u(0.5, 3.0);
  Vector v(n);
  for (Index i = 0; i < n; ++i) v[i] = u(rng);
  return v;
}
static double a_norm_sq(const Matrix& x, Index j, const RbdModel& model, const Vector& a) {
  double s = 0.0;
  for (Index i = 0; i < x.rows(); ++i) {
    double r = x(i, j);
    for (Index k = 0; k < model.d; ++k) r -= model.Y(i, k) * model.T(k, j);
    s += a[i] * r * r;
  }
  return std::max(s, 0.0);
}
static RbdConfig basic(Index d_max, double eps = 0.0) {
  RbdConfig c;
  c.d_max = d_max;
  c.eps_R = eps;
  return c;
}

int main() {
  // decompose_many (the pipelined host entry) == decompose per matrix, bit for bit
  {
    std::vector<Matrix> xs;
    for (std::uint64_t seed : {700u, 701u, 702u}) xs.push_back(random_matrix(300, 40, seed));
    const std::vector<RbdModel> many = decompose_many(xs, basic(15));
    CHECK(many.size() == xs.size());
    for (size_t i = 0; i < xs.size() && i < many.size(); ++i) {
      const RbdModel one = decompose(xs[i], basic(15));
      CHECK(many[i].d == one.d);
      CHECK(many[i].selected == one.selected);
      CHECK(max_abs_diff(many[i].Y, one.Y) == 0.0);
      CHECK(max_abs_diff(many[i].T, one.T) == 0.0);
    }
    CHECK_THROWS_AS(decompose_many({xs[0], random_matrix(30, 4, 9)}, basic(3)), InvalidArgument);
  }
  // test_decompose.cpp:29-40 rank-1 outer product
  {
    const Vector u = random_matrix(30, 1, 100).col(0);
    const Vector v = random_matrix(20, 1, 101).col(0);
    Matrix x(30, 20);
    for (Index j = 0; j < 20; ++j)
      for (Index i = 0; i < 30; ++i) x(i, j) = u[i] * v[j];
    const RbdModel model = decompose(x, basic(10, 1e-10));
    CHECK(model.d == 1);
    CHECK(max_abs_diff(x, compress_matrix(model)) < 1e-10);
    CHECK(std::abs(std::abs(model.Y.col(0).dot(u) / u.norm()) - 1.0) < 1e-12);
  }
  // :42-49 orthonormal basis
  for (std::uint64_t seed : {200u, 201u, 202u}) {
    const RbdModel model = decompose(random_matrix(25, 18, seed), basic(12));
    CHECK(model.d == 12);
    CHECK(orthonormality_defect(model.Y) < 1e-10);
  }
  // :51-57 rank-deficient input via the noise floor
  {
    const Matrix x = matmul(random_matrix(40, 5, 210), random_matrix(5, 30, 211));
    const RbdModel model = decompose(x, basic(30));
    CHECK(model.d == 5);
    CHECK(orthonormality_defect(model.Y) < 1e-10);
    CHECK(max_abs_diff(x, compress_matrix(model)) < 1e-9);
  }
  // :59-65 monotone history
  {
    const RbdModel model = decompose(random_matrix(30, 22, 220), basic(15));
    CHECK(model.residual_history.size() == static_cast<size_t>(model.d));
    for (size_t k = 1; k < model.residual_history.size(); ++k)
      CHECK(model.residual_history[k] <= model.residual_history[k - 1] + 1e-12);
  }
  // :67-74 rows of T are exact inner products
  {
    const Matrix x = random_matrix(17, 12, 230);
    const RbdModel model = decompose(x, basic(6));
    const Matrix expect = matmul(transpose(model.Y), x);
    CHECK(max_abs_diff(expect, model.T) < 1e-13);
  }
  // :76-86 selected distinct and in range
  {
    const RbdModel model = decompose(random_matrix(26, 14, 240), basic(10));
    CHECK(model.selected.size() == static_cast<size_t>(model.d));
    for (size_t a = 0; a < model.selected.size(); ++a) {
      CHECK(model.selected[a] >= 0 && model.selected[a] < 14);
      for (size_t b = a + 1; b < model.selected.size(); ++b)
        CHECK(model.selected[a] != model.selected[b]);
    }
  }
  // :128-137 deterministic bit for bit
  {
    const Matrix x = random_matrix(24, 16, 270);
    const RbdModel a = decompose(x, basic(9, 1e-8)), b = decompose(x, basic(9, 1e-8));
    CHECK(a.Y == b.Y);
    CHECK(a.T == b.T);
    CHECK(a.selected == b.selected);
    CHECK(a.residual_history == b.residual_history);
  }
  // :153-169 start column control
  {
    const Matrix x = random_matrix(15, 10, 290);
    RbdConfig cfg = basic(3);
    cfg.start = StartSpec::column(7);
    CHECK(decompose(x, cfg).selected.front() == 7);
    cfg.start = StartSpec::column(10);
    CHECK_THROWS_AS(decompose(x, cfg), IndexOutOfRange);
    cfg.start = StartSpec::seeded(42);
    const RbdModel a = decompose(x, cfg), b = decompose(x, cfg);
    CHECK(a.selected.front() == b.selected.front());
    std::mt19937_64 rng(42);   // decompose.cpp:43-46
    CHECK(a.selected.front() == std::uniform_int_distribution<Index>(0, 9)(rng));
  }
  // :182-206 input and configuration gating
  {
    const Matrix x = random_matrix(10, 6, 310);
    CHECK_THROWS_AS(decompose(Matrix::Zero(4, 3), basic(2)), DegenerateInput);
    CHECK_THROWS_AS(decompose(x, basic(0)), InvalidArgument);
    CHECK_THROWS_AS(decompose(x, basic(7)), InvalidArgument);
    RbdConfig bad_eps = basic(2);
    bad_eps.eps_R = -1.0;
    CHECK_THROWS_AS(decompose(x, bad_eps), InvalidArgument);
    Matrix with_nan = x;
    with_nan(3, 2) = std::numeric_limits<double>::quiet_NaN();
    CHECK_THROWS_AS(decompose(with_nan, basic(2)), InvalidArgument);
    RbdConfig wrong_dim = basic(2);
    wrong_dim.weight = WeightSpec::diagonal(Vector::Ones(9));
    CHECK_THROWS_AS(decompose(x, wrong_dim), IncompatibleWeight);
    Matrix zero_col = x;
    for (Index i = 0; i < 10; ++i) zero_col(i, 0) = 0.0;
    RbdConfig from_zero = basic(2);
    from_zero.breakdown_tol = 1e-12;
    CHECK_THROWS_AS(decompose(zero_col, from_zero), DegenerateInput);
  }
  // :231-244 reorthogonalisation on Krylov-like input
  {
    Matrix x(60, 8);
    for (Index j = 0; j < 8; ++j)
      for (Index i = 0; i < 60; ++i) x(i, j) = std::pow((i + 1) / 60.0, (double)j);
    RbdConfig cfg = basic(8);
    cfg.reorthogonalize = true;
    cfg.breakdown_tol = 1e-12;
    CHECK(orthonormality_defect(decompose(x, cfg).Y) < 1e-12);
  }
  // :246-256 project and reconstruct
  {
    const RbdModel model = decompose(random_matrix(18, 12, 320), basic(5));
    const Vector c = random_matrix(5, 1, 321).col(0);
    const Vector v = reconstruct(model, c);
    const Vector back = project(model, v);
    double err = 0.0;
    for (Index k = 0; k < 5; ++k) err = std::max(err, std::abs(back[k] - c[k]));
    CHECK(err < 1e-12);
    CHECK_THROWS_AS(project(model, Vector::Ones(17)), DimensionMismatch);
    CHECK_THROWS_AS(reconstruct(model, Vector::Ones(4)), DimensionMismatch);
  }
  // :274-289 mgs_project
  {
    const Matrix x = random_matrix(10, 3, 340);
    Matrix y(10, 1);
    const Vector x0 = x.col(0);
    for (Index i = 0; i < 10; ++i) y(i, 0) = x0[i] / x0.norm();
    const auto r = mgs_project(x.col(1), y, 1e-12);
    CHECK(r.has_value());
    if (r) {
      CHECK(std::abs(r->xi.norm() - 1.0) < 1e-14);
      CHECK(std::abs(r->xi.dot(y.col(0))) < 1e-13);
    }
    Vector in_span(10);
    for (Index i = 0; i < 10; ++i) in_span[i] = 3.7 * y(i, 0);
    CHECK(!mgs_project(in_span, y, 1e-10).has_value());
  }
  // test_workspace.cpp:28-37, 124-153 (identity), 200-212
  {
    Matrix x(3, 2);
    x(0, 0) = 1.0;
    x(1, 1) = 2.0;
    const ErrorWorkspace ws = workspace_init(x, WeightSpec::identity());
    const Vector cs = ws.col_sq();
    CHECK(cs[0] == 1.0 && cs[1] == 4.0);
    CHECK_THROWS_AS(workspace_init(random_matrix(5, 3, 14), WeightSpec::diagonal(Vector::Ones(4))),
                    IncompatibleWeight);
  }
  {
    const Matrix x = random_matrix(15, 9, 40);
    const RbdModel model = decompose(x, basic(3));
    ErrorWorkspace ws = workspace_init(x, WeightSpec::identity());
    for (Index k = 0; k < 3; ++k) workspace_extend(ws, model.Y.col(k), x, WeightSpec::identity());
    const Matrix t = matmul(transpose(model.Y), x);
    double best = -1.0;
    Index best_j = 0;
    for (Index j = 0; j < 9; ++j) {
      double e = 0.0;
      for (Index i = 0; i < 15; ++i) {
        double r = x(i, j);
        for (Index k = 0; k < 3; ++k) r -= model.Y(i, k) * t(k, j);
        e += r * r;
      }
      CHECK(std::abs(error_sq(ws, j, t.col(j)) - e) <= 1e-9 * std::max(1.0, ws.col_sq()[j]));
      if (e > best) {
        best = e;
        best_j = j;
      }
    }
    const ScanResult scan = residual_scan(ws, t);
    CHECK(scan.argmax == best_j);
    CHECK(std::abs(scan.e_cur - std::sqrt(best)) <= 1e-7 * std::sqrt(best));
    CHECK_THROWS_AS(error_sq(ws, -1, Vector::Zero(3)), IndexOutOfRange);
    CHECK_THROWS_AS(error_sq(ws, 0, Vector::Zero(2)), DimensionMismatch);
  }
  // test_decompose.cpp:113-126: the history equals the directly computed A-norm errors
  {
    const Matrix x = random_matrix(20, 15, 260);
    RbdConfig cfg = basic(8);
    const Vector a = random_positive(20, 261);
    cfg.weight = WeightSpec::diagonal(a);
    const RbdModel model = decompose(x, cfg);
    double worst = 0.0;
    for (Index j = 0; j < 15; ++j) worst = std::max(worst, std::sqrt(a_norm_sq(x, j, model, a)));
    CHECK(std::abs(model.residual_history.back() - worst) <= 1e-7 * worst);
    RbdConfig wrong = basic(2);                     // test_decompose.cpp:196-198
    Vector ones9(9);
    for (Index i = 0; i < 9; ++i) ones9[i] = 1.0;
    wrong.weight = WeightSpec::diagonal(ones9);
    CHECK_THROWS_AS(decompose(random_matrix(10, 6, 310), wrong), IncompatibleWeight);
  }
  // test_decompose.cpp:208-229: a diagonal weight steers the greedy selection
  {
    Matrix x(4, 3);
    x(0, 0) = 1.0;
    x(1, 1) = 2.0;
    x(2, 2) = 0.5;
    RbdConfig plain = basic(2);
    plain.start = StartSpec::column(2);
    CHECK(decompose(x, plain).selected[1] == 1);
    RbdConfig weighted = plain;
    weighted.weight = WeightSpec::diagonal(Vector{100.0, 1.0, 1.0, 1.0});
    CHECK(decompose(x, weighted).selected[1] == 0);
  }
  // test_workspace.cpp:39-60 (identity and diagonal kinds) and a weighted scan
  {
    const Index m = 11, n = 6;
    const Matrix x = random_matrix(m, n, 11);
    const Vector a = random_positive(m, 12);
    const WeightSpec kinds[] = {WeightSpec::identity(), WeightSpec::diagonal(a)};
    for (const WeightSpec& w : kinds) {
      const ErrorWorkspace ws = workspace_init(x, w);
      const Vector cs = ws.col_sq();
      for (Index j = 0; j < n; ++j) {
        double q = 0.0;
        for (Index i = 0; i < m; ++i)
          q += (w.kind() == WeightKind::diagonal ? a[i] : 1.0) * x(i, j) * x(i, j);
        CHECK(std::abs(cs[j] - q) <= 1e-12 * q);
      }
    }
    Vector ones4(4);
    for (Index i = 0; i < 4; ++i) ones4[i] = 1.0;
    CHECK_THROWS_AS(workspace_init(random_matrix(5, 3, 14), WeightSpec::diagonal(ones4)),
                    IncompatibleWeight);
    CHECK_THROWS_AS(WeightSpec::diagonal(Vector(4)), InvalidArgument);   // test_weight.cpp:21-32
    RbdConfig cfg = basic(4);
    cfg.weight = WeightSpec::diagonal(a);
    const RbdModel model = decompose(x, cfg);
    ErrorWorkspace ws = workspace_init(x, cfg.weight);
    for (Index k = 0; k < model.d; ++k) workspace_extend(ws, model.Y.col(k), x, cfg.weight);
    const ScanResult scan = residual_scan(ws, model.T);
    CHECK(std::abs(scan.e_cur - model.residual_history.back()) <=
          1e-9 * std::max(1.0, model.residual_history.back()));
  }
  // test_io.cpp:273-332: container round trip, size, corruption, missing file
  {
    namespace fs = std::filesystem;
    const fs::path dir = fs::temp_directory_path() / "rbd_b200_cpp_io";
    fs::create_directories(dir);
    const fs::path p = dir / "model.rbd";
    const Matrix x = random_matrix(12, 9, 1040);
    const WeightSpec kinds[] = {WeightSpec::identity(),
                                WeightSpec::diagonal(random_positive(12, 1041))};
    for (const WeightSpec& w : kinds) {
      RbdConfig cfg = basic(5, 1e-9);
      cfg.weight = w;
      const RbdModel model = decompose(x, cfg);
      write_model(model, cfg.eps_R, p);
      const LoadedModel back = read_model(p);
      CHECK(max_abs_diff(back.model.Y, model.Y) == 0.0);
      CHECK(max_abs_diff(back.model.T, model.T) == 0.0);
      CHECK(back.model.d == model.d);
      CHECK(back.model.residual_history == model.residual_history);
      CHECK(back.eps_r == cfg.eps_R);
      CHECK(back.model.weight.kind() == w.kind());
      size_t expect = 29 + 8 * static_cast<size_t>(12 * model.d + model.d * 9 + 1 + model.d);
      if (w.kind() == WeightKind::diagonal) {
        expect += 8 * 12;
        bool same = true;
        for (Index i = 0; i < 12; ++i)
          same = same && back.model.weight.diagonal_values()[i] == w.diagonal_values()[i];
        CHECK(same);
      }
      CHECK(fs::file_size(p) == expect);
    }
    std::string raw;
    {
      std::ifstream in(p, std::ios::binary);
      raw.assign(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
    }
    auto put = [&](const std::string& bytes) {
      std::ofstream out(p, std::ios::binary | std::ios::trunc);
      out.write(bytes.data(), static_cast<std::streamsize>(bytes.size()));
    };
    put("XXXX" + raw.substr(4));
    CHECK_THROWS_AS(read_model(p), ParseError);
    put(raw.substr(0, raw.size() - 8));
    CHECK_THROWS_AS(read_model(p), ParseError);
    std::string bad_tag = raw;
    bad_tag[28] = 9;
    put(bad_tag);
    CHECK_THROWS_AS(read_model(p), ParseError);
    CHECK_THROWS_AS(read_model(dir / "nope.rbd"), IoError);
    fs::remove_all(dir);
  }
  {  // per-vector project / reconstruct through the model's device-resident Y
     // (classify.cpp:22-23 calls project once per query): same values as the
     // first call, Y uploaded once, a copied model builds its own cache
    Matrix x = random_matrix(300, 40, 700);
    RbdModel model = decompose(x, basic(20));
    Matrix q = random_matrix(300, 64, 701);
    double worst = 0.0;
    for (Index j = 0; j < q.cols(); ++j) {
      Vector v = q.col(j);
      Vector c = project(model, v);
      for (Index k = 0; k < model.d; ++k) {
        double s = 0.0;
        for (Index i = 0; i < 300; ++i) s += model.Y(i, k) * v[i];
        worst = std::max(worst, std::abs(s - c[k]));
      }
      Vector back = reconstruct(model, c);
      Vector again = project(model, back);
      for (Index k = 0; k < model.d; ++k) worst = std::max(worst, std::abs(again[k] - c[k]));
    }
    CHECK(worst < 1e-12);
    RbdModel copy = model;
    Vector c1 = project(copy, q.col(3)), c2 = project(model, q.col(3));
    bool same = true;
    for (Index k = 0; k < model.d; ++k) same = same && c1[k] == c2[k];
    CHECK(same);
  }
  std::printf("%d checks, %d failed\n", g_checks, g_fail);
  return g_fail;
}
