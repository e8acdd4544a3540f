// JSON problem / solution files (include/tsylv/io.hpp) checked the way the
// reference's tests/test_random_io.cpp checks its own: round trips of both
// families, solution files with and without timings, byte-stable re-saves,
// io_error on every malformed envelope, a hand-written file.  No GPU work:
// built and run by tests/test_io_cli.py on the CPU.
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <iterator>
#include <string>
#include <vector>

#include "tsylv/io.hpp"
#include "tsylv/random.hpp"

static int failures = 0;
#define CHECK(c)                                                                 \
  do {                                                                           \
    if (!(c)) {                                                                  \
      ++failures;                                                                \
      std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #c); \
    }                                                                            \
  } while (0)

template <typename Fn>
bool throws_io(Fn&& fn) {
  try {
    fn();
  } catch (const tsylv::io_error&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

using namespace tsylv;
namespace fs = std::filesystem;

static bool same(const Matrix<double>& a, const Matrix<double>& b) {
  if (a.rows() != b.rows() || a.cols() != b.cols()) return false;
  for (int j = 0; j < a.cols(); ++j)
    for (int i = 0; i < a.rows(); ++i)
      if (a(i, j) != b(i, j)) return false;
  return true;
}
static std::string slurp(const fs::path& p) {
  std::ifstream in(p, std::ios::binary);
  return std::string(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
}

int main(int argc, char** argv) {
  const fs::path dir = argc > 1 ? fs::path(argv[1]) : fs::temp_directory_path() / "tsylv_io_tests";
  fs::create_directories(dir);
  RandomStream rng(2026);

  // round trips, bit-exact (%.17g-faithful JSON numbers)
  {
    LaplaceProblem<double> lp;
    for (int n : {4, 3, 5}) lp.coeffs.push_back(randn_matrix(rng, n, n));
    lp.rhs = randn_tensor(rng, {4, 3, 5});
    const std::string lpath = (dir / "lap.json").string();
    save_problem(lpath, lp);
    const AnyProblem any = load_problem(lpath);
    CHECK(std::holds_alternative<LaplaceProblem<double>>(any));
    const auto& q = std::get<LaplaceProblem<double>>(any);
    CHECK(q.dims() == lp.dims());
    for (int m = 0; m < 3; ++m) CHECK(same(q.coeffs[m], lp.coeffs[m]));
    CHECK(q.rhs.values() == lp.rhs.values());

    GSylvProblem<double> gp;
    for (int n : {3, 2, 2}) gp.coeffs.push_back(randn_matrix(rng, n, n));
    gp.c = randn_matrix(rng, 3, 3);
    gp.rhs = randn_tensor(rng, {3, 2, 2});
    const std::string gpath = (dir / "gsylv.json").string();
    save_problem(gpath, gp);
    const AnyProblem ganya = load_problem(gpath);
    CHECK(std::holds_alternative<GSylvProblem<double>>(ganya));
    const auto& g = std::get<GSylvProblem<double>>(ganya);
    CHECK(same(g.c, gp.c));
    for (int m = 0; m < 3; ++m) CHECK(same(g.coeffs[m], gp.coeffs[m]));
    CHECK(g.rhs.values() == gp.rhs.values());
    // storage order: rhs(i, j, k) is flat element i + 4 j + 12 k, mode 0 fastest
    CHECK(lp.rhs.values()[1 + 4 * 2 + 12 * 3] == lp.rhs(1, 2, 3));
  }

  // solution files: solution + report, optional timings, byte-stable without
  {
    LaplaceProblem<double> p;
    p.coeffs = {randn_matrix(rng, 2, 2), randn_matrix(rng, 3, 3)};
    p.rhs = randn_tensor(rng, {2, 3});
    SolveReport<double> rep;
    rep.solution = randn_tensor(rng, {2, 3});
    rep.residual = 1.25e-15;
    rep.n_min = 8;
    rep.strategy = Strategy::recursion_only;
    rep.timings.reduction_s = 0.5;
    const std::string path = (dir / "sol.json").string();
    save_solution(path, p, rep);
    const Tensor<double> x = load_solution<double>(path);
    CHECK(x.dims() == rep.solution.dims());
    CHECK(x.values() == rep.solution.values());
    const std::string with = slurp(path);
    CHECK(with.find("\"timings\"") != std::string::npos);
    CHECK(with.find("\"recursion\"") != std::string::npos);
    CHECK(with.find("\"n_min\": 8") != std::string::npos);
    save_solution(path, p, rep, /*include_timings=*/false);
    CHECK(slurp(path).find("timings") == std::string::npos);
    // the solution file is also a problem file
    CHECK(std::holds_alternative<LaplaceProblem<double>>(load_problem(path)));

    const fs::path p1 = dir / "stable1.json", p2 = dir / "stable2.json";
    SolveReport<double> rep2 = rep;
    rep2.timings.reduction_s = 99;  // differs only in timings
    save_solution(p1.string(), p, rep, false);
    save_solution(p2.string(), p, rep2, false);
    CHECK(slurp(p1) == slurp(p2));
    CHECK(throws_io([&] { load_solution<double>((dir / "lap.json").string()); }));  // no "solution"
  }

  // malformed envelopes all raise io_error
  {
    const std::string path = (dir / "bad.json").string();
    auto bad = [&](const std::string& text) {
      {
        std::ofstream out(path, std::ios::binary);
        out << text;
      }
      return throws_io([&] { load_problem(path); });
    };
    CHECK(bad("this is not json"));
    CHECK(bad("[1, 2, 3]"));
    CHECK(bad("{\"family\": \"heat\"}"));
    CHECK(bad("{\"family\": \"laplace\", \"dims\": [2, 2]}"));  // missing coeffs
    CHECK(bad("{\"family\": \"laplace\", \"dims\": [2], \"coeffs\": [[[1, 0], [0, 1]]], \"rhs\": [1, 2, 3]}"));
    CHECK(bad("{\"family\": \"laplace\", \"dims\": [2, 2], \"coeffs\": [[[1]], [[1]]], \"rhs\": [1, 2, 3, 4]}"));
    CHECK(bad("{\"family\": \"gsylv\", \"dims\": [2, 2], \"coeffs\": [[[1, 0], [0, 1]], [[1, 0], [0, 1]]], "
              "\"rhs\": [1, 2, 3, 4]}"));  // gsylv without C
    CHECK(bad("{\"family\": \"laplace\", \"dims\": [2, 0], \"coeffs\": [[[1, 0], [0, 1]], [[1]]], \"rhs\": []}"));
    CHECK(bad("{\"family\": \"laplace\", \"dims\": [1, 1], \"coeffs\": [[[1]], [[\"x\"]]], \"rhs\": [1]}"));
    CHECK(bad("{\"family\": \"laplace\", \"dims\": [2, 1], \"coeffs\": [[[1, 0], [0]], [[1]]], \"rhs\": [1, 2]}"));
    // complex files need [re, im] pairs (a bare number is not a complex scalar)
    CHECK(bad("{\"family\": \"laplace\", \"complex\": true, \"dims\": [1, 1], \"coeffs\": [[[1]], [[[1, "
              "0]]]], \"rhs\": [[1, 0]]}"));
    CHECK(throws_io([&] { load_problem((dir / "missing.json").string()); }));
  }

  // a hand-written file
  {
    const std::string path = (dir / "hand.json").string();
    {
      std::ofstream out(path, std::ios::binary);
      out << R"({
        "family": "gsylv",
        "dims": [2, 1],
        "coeffs": [[[1.0, 0.5], [0.0, 2.0]], [[3.0]]],
        "c_coeff": [[1.0, 0.0], [0.25, 1.0]],
        "rhs": [1.0, -2.0]
      })";
    }
    const AnyProblem any = load_problem(path);
    CHECK(std::holds_alternative<GSylvProblem<double>>(any));
    const auto& p = std::get<GSylvProblem<double>>(any);
    CHECK(p.order() == 2);
    CHECK(p.coeffs[0](0, 1) == 0.5);  // row-major rows
    CHECK(p.coeffs[0](1, 1) == 2.0);
    CHECK(p.coeffs[1](0, 0) == 3.0);
    CHECK(p.c(1, 0) == 0.25);
    CHECK(p.rhs(1, 0) == -2.0);
  }

  std::printf("%s (%d failures)\n", failures ? "FAIL" : "PASS", failures);
  return failures ? 1 : 0;
}
