// tsylv drop-in (B200 build) — JSON problem and solution files (the
// reference's proj/include/tsylv/io.hpp), with the
// same envelope:
//
//   {"family": "laplace"|"gsylv", "complex": bool, "dims": [n_0, ...],
//    "coeffs": [row-major 2-D arrays], "c_coeff": 2-D array (gsylv only),
//    "rhs": flat array in storage order (mode 0 fastest)}
//
// solution files add "solution" (flat) and "report" (residual,
// discarded_imag, n_min, strategy, optional timings).  Malformed files raise
// io_error with the reference's messages.  Complex-scalar problems
// ("complex": true) are SURVEY row f1, not built: they raise io_error.
// Needs nlohmann/json on the include path (the CLI build finds the copy in
// the image, paper_1905_09539_b200/build.py).
#pragma once
#include <fstream>
#include <string>
#include <type_traits>
#include <variant>
#include <vector>

#include <nlohmann/json.hpp>

#include "tsylv/config.hpp"
#include "tsylv/errors.hpp"
#include "tsylv/matrix.hpp"
#include "tsylv/problems.hpp"
#include "tsylv/tensor.hpp"

namespace tsylv {

using AnyProblem = std::variant<LaplaceProblem<double>, GSylvProblem<double>>;

namespace detail {

inline nlohmann::json matrix_json(const Matrix<double>& m) {
  nlohmann::json rows = nlohmann::json::array();
  for (int i = 0; i < m.rows(); ++i) {
    nlohmann::json row = nlohmann::json::array();
    for (int j = 0; j < m.cols(); ++j) row.push_back(m(i, j));
    rows.push_back(std::move(row));
  }
  return rows;
}

inline Matrix<double> json_matrix(const nlohmann::json& j, const char* what) {
  if (!j.is_array() || j.empty()) throw io_error(std::string(what) + ": expected a non-empty 2-D array");
  if (!j[0].is_array()) throw io_error(std::string(what) + ": expected nested rows");
  const int rows = static_cast<int>(j.size()), cols = static_cast<int>(j[0].size());
  Matrix<double> m(rows, cols);
  for (int i = 0; i < rows; ++i) {
    if (!j[i].is_array() || static_cast<int>(j[i].size()) != cols) throw io_error(std::string(what) + ": ragged rows");
    for (int c = 0; c < cols; ++c) {
      if (!j[i][c].is_number()) throw io_error("expected a real number");
      m(i, c) = j[i][c].get<double>();
    }
  }
  return m;
}

inline std::vector<double> json_flat(const nlohmann::json& j, std::size_t want, const char* what) {
  if (!j.is_array() || j.size() != want)
    throw io_error(std::string(what) + ": expected a flat array of length " + std::to_string(want));
  std::vector<double> v(want);
  for (std::size_t i = 0; i < want; ++i) {
    if (!j[i].is_number()) throw io_error("expected a real number");
    v[i] = j[i].get<double>();
  }
  return v;
}

inline nlohmann::json envelope(const char* family, const std::vector<int>& dims, const std::vector<Matrix<double>>& co,
                               const Tensor<double>& rhs) {
  nlohmann::json j;
  j["family"] = family;
  j["complex"] = false;
  j["dims"] = dims;
  nlohmann::json cj = nlohmann::json::array();
  for (const auto& a : co) cj.push_back(matrix_json(a));
  j["coeffs"] = std::move(cj);
  j["rhs"] = rhs.values();
  return j;
}

inline nlohmann::json problem_json(const LaplaceProblem<double>& p) {
  return envelope("laplace", p.dims(), p.coeffs, p.rhs);
}
inline nlohmann::json problem_json(const GSylvProblem<double>& p) {
  nlohmann::json j = envelope("gsylv", p.dims(), p.coeffs, p.rhs);
  j["c_coeff"] = matrix_json(p.c);
  return j;
}

inline void write_json(const std::string& path, const nlohmann::json& j) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw io_error("cannot open for writing: " + path);
  out << j.dump(2) << '\n';
  if (!out) throw io_error("write failed: " + path);
}

inline nlohmann::json read_json(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw io_error("cannot open: " + path);
  try {
    nlohmann::json j;
    in >> j;
    return j;
  } catch (const nlohmann::json::exception& e) {
    throw io_error("cannot parse " + path + ": " + e.what());
  }
}

}  // namespace detail

inline AnyProblem problem_from_json(const nlohmann::json& j) {
  if (!j.is_object()) throw io_error("problem file: expected a JSON object");
  if (!j.contains("family") || !j["family"].is_string()) throw io_error("problem file: missing \"family\"");
  const std::string family = j["family"].get<std::string>();
  if (family != "laplace" && family != "gsylv") throw io_error("problem file: unknown family \"" + family + "\"");
  if (j.value("complex", false))
    throw io_error("problem file: complex-scalar problems are not supported by the B200 build");
  if (!j.contains("dims") || !j["dims"].is_array()) throw io_error("problem file: missing \"dims\"");
  std::vector<int> dims;
  for (const auto& e : j["dims"]) {
    if (!e.is_number_integer() || e.get<int>() <= 0) throw io_error("problem file: dims must be positive integers");
    dims.push_back(e.get<int>());
  }
  if (!j.contains("coeffs") || !j["coeffs"].is_array() || j["coeffs"].size() != dims.size())
    throw io_error("problem file: need one coefficient per mode");
  std::vector<Matrix<double>> co;
  for (std::size_t m = 0; m < dims.size(); ++m) co.push_back(detail::json_matrix(j["coeffs"][m], "coeffs"));
  std::size_t total = 1;
  for (int n : dims) total *= static_cast<std::size_t>(n);
  if (!j.contains("rhs")) throw io_error("problem file: missing \"rhs\"");
  Tensor<double> rhs(dims, detail::json_flat(j["rhs"], total, "rhs"));
  try {
    if (family == "gsylv") {
      if (!j.contains("c_coeff")) throw io_error("problem file: gsylv needs \"c_coeff\"");
      GSylvProblem<double> p;
      p.coeffs = std::move(co);
      p.c = detail::json_matrix(j["c_coeff"], "c_coeff");
      p.rhs = std::move(rhs);
      validate(p);
      return p;
    }
    LaplaceProblem<double> p;
    p.coeffs = std::move(co);
    p.rhs = std::move(rhs);
    validate(p);
    return p;
  } catch (const dimension_error& e) {
    throw io_error(std::string("problem file: ") + e.what());
  }
}

inline AnyProblem load_problem(const std::string& path) { return problem_from_json(detail::read_json(path)); }

template <typename P>
void save_problem(const std::string& path, const P& p) {
  detail::write_json(path, detail::problem_json(p));
}

// problem envelope + flat "solution" + "report"; timings optional so files
// of repeated runs compare byte for byte
template <typename P>
void save_solution(const std::string& path, const P& p, const SolveReport<double>& rep, bool include_timings = true) {
  nlohmann::json j = detail::problem_json(p);
  j["solution"] = rep.solution.values();
  nlohmann::json r;
  r["residual"] = rep.residual;
  r["discarded_imag"] = rep.discarded_imag;
  r["n_min"] = rep.n_min;
  r["strategy"] = to_string(rep.strategy);
  if (include_timings)
    r["timings"] = {{"reduction_s", rep.timings.reduction_s},
                    {"recursion_s", rep.timings.recursion_s},
                    {"back_transform_s", rep.timings.back_transform_s}};
  j["report"] = std::move(r);
  detail::write_json(path, j);
}

template <typename T = double>
Tensor<T> load_solution(const std::string& path) {
  static_assert(std::is_same_v<T, double>, "the B200 build reads real solution files only");
  const nlohmann::json j = detail::read_json(path);
  if (!j.contains("solution")) throw io_error(path + ": not a solution file");
  std::vector<int> dims;
  for (const auto& e : j["dims"]) dims.push_back(e.get<int>());
  std::size_t total = 1;
  for (int n : dims) total *= static_cast<std::size_t>(n);
  return Tensor<double>(dims, detail::json_flat(j["solution"], total, "solution"));
}

}  // namespace tsylv
