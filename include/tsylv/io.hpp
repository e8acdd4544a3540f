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
// ("complex": true, scalars as [re, im] pairs) load as LaplaceProblem<Complex>
// / GSylvProblem<Complex>.
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
#include "tsylv/scalar.hpp"
#include "tsylv/tensor.hpp"

namespace tsylv {

using AnyProblem = std::variant<LaplaceProblem<double>, LaplaceProblem<Complex>,
                                GSylvProblem<double>, GSylvProblem<Complex>>;

namespace detail {

// scalars: numbers, or [re, im] pairs in complex files
inline nlohmann::json scalar_json(double v) { return v; }
inline nlohmann::json scalar_json(const Complex& v) { return nlohmann::json::array({v.real(), v.imag()}); }
inline void json_scalar(const nlohmann::json& j, double& out) {
  if (!j.is_number()) throw io_error("expected a real number");
  out = j.get<double>();
}
inline void json_scalar(const nlohmann::json& j, Complex& out) {
  if (!j.is_array() || j.size() != 2 || !j[0].is_number() || !j[1].is_number())
    throw io_error("expected a [re, im] pair");
  out = Complex(j[0].get<double>(), j[1].get<double>());
}

template <typename T>
nlohmann::json matrix_json(const Matrix<T>& m) {
  nlohmann::json rows = nlohmann::json::array();
  for (int i = 0; i < m.rows(); ++i) {
    nlohmann::json row = nlohmann::json::array();
    for (int j = 0; j < m.cols(); ++j) row.push_back(scalar_json(m(i, j)));
    rows.push_back(std::move(row));
  }
  return rows;
}

template <typename T>
Matrix<T> json_matrix(const nlohmann::json& j, const char* what) {
  if (!j.is_array() || j.empty()) throw io_error(std::string(what) + ": expected a non-empty 2-D array");
  if (!j[0].is_array()) throw io_error(std::string(what) + ": expected nested rows");
  const int rows = static_cast<int>(j.size()), cols = static_cast<int>(j[0].size());
  Matrix<T> m(rows, cols);
  for (int i = 0; i < rows; ++i) {
    if (!j[i].is_array() || static_cast<int>(j[i].size()) != cols) throw io_error(std::string(what) + ": ragged rows");
    for (int c = 0; c < cols; ++c) json_scalar(j[i][c], m(i, c));
  }
  return m;
}

template <typename T>
nlohmann::json flat_json(const std::vector<T>& v) {
  nlohmann::json out = nlohmann::json::array();
  for (const T& x : v) out.push_back(scalar_json(x));
  return out;
}

template <typename T>
std::vector<T> json_flat(const nlohmann::json& j, std::size_t want, const char* what) {
  if (!j.is_array() || j.size() != want)
    throw io_error(std::string(what) + ": expected a flat array of length " + std::to_string(want));
  std::vector<T> v(want);
  for (std::size_t i = 0; i < want; ++i) json_scalar(j[i], v[i]);
  return v;
}

template <typename T>
nlohmann::json envelope(const char* family, const std::vector<int>& dims, const std::vector<Matrix<T>>& co,
                        const Tensor<T>& rhs) {
  nlohmann::json j;
  j["family"] = family;
  j["complex"] = is_complex_v<T>;
  j["dims"] = dims;
  nlohmann::json cj = nlohmann::json::array();
  for (const auto& a : co) cj.push_back(matrix_json(a));
  j["coeffs"] = std::move(cj);
  j["rhs"] = flat_json(rhs.values());
  return j;
}

template <typename T>
nlohmann::json problem_json(const LaplaceProblem<T>& p) {
  return envelope("laplace", p.dims(), p.coeffs, p.rhs);
}
template <typename T>
nlohmann::json problem_json(const GSylvProblem<T>& p) {
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

inline std::vector<int> json_dims(const nlohmann::json& j) {
  if (!j.contains("dims") || !j["dims"].is_array()) throw io_error("problem file: missing \"dims\"");
  std::vector<int> dims;
  for (const auto& e : j["dims"]) {
    if (!e.is_number_integer() || e.get<int>() <= 0) throw io_error("problem file: dims must be positive integers");
    dims.push_back(e.get<int>());
  }
  return dims;
}

template <typename T>
AnyProblem typed_problem(const nlohmann::json& j, bool gsylv) {
  const std::vector<int> dims = json_dims(j);
  if (!j.contains("coeffs") || !j["coeffs"].is_array() || j["coeffs"].size() != dims.size())
    throw io_error("problem file: need one coefficient per mode");
  std::vector<Matrix<T>> co;
  for (std::size_t m = 0; m < dims.size(); ++m) co.push_back(json_matrix<T>(j["coeffs"][m], "coeffs"));
  std::size_t total = 1;
  for (int n : dims) total *= static_cast<std::size_t>(n);
  if (!j.contains("rhs")) throw io_error("problem file: missing \"rhs\"");
  Tensor<T> rhs(dims, json_flat<T>(j["rhs"], total, "rhs"));
  try {
    if (gsylv) {
      if (!j.contains("c_coeff")) throw io_error("problem file: gsylv needs \"c_coeff\"");
      GSylvProblem<T> p;
      p.coeffs = std::move(co);
      p.c = json_matrix<T>(j["c_coeff"], "c_coeff");
      p.rhs = std::move(rhs);
      validate(p);
      return p;
    }
    LaplaceProblem<T> p;
    p.coeffs = std::move(co);
    p.rhs = std::move(rhs);
    validate(p);
    return p;
  } catch (const dimension_error& e) {
    throw io_error(std::string("problem file: ") + e.what());
  }
}

}  // namespace detail

inline AnyProblem problem_from_json(const nlohmann::json& j) {
  if (!j.is_object()) throw io_error("problem file: expected a JSON object");
  if (!j.contains("family") || !j["family"].is_string()) throw io_error("problem file: missing \"family\"");
  const std::string family = j["family"].get<std::string>();
  if (family != "laplace" && family != "gsylv") throw io_error("problem file: unknown family \"" + family + "\"");
  const bool gsylv = family == "gsylv";
  if (j.value("complex", false)) return detail::typed_problem<Complex>(j, gsylv);
  return detail::typed_problem<double>(j, gsylv);
}

inline AnyProblem load_problem(const std::string& path) { return problem_from_json(detail::read_json(path)); }

template <typename P>
void save_problem(const std::string& path, const P& p) {
  detail::write_json(path, detail::problem_json(p));
}

// problem envelope + flat "solution" + "report"; timings optional so files
// of repeated runs compare byte for byte
template <typename P, typename T>
void save_solution(const std::string& path, const P& p, const SolveReport<T>& rep, bool include_timings = true) {
  nlohmann::json j = detail::problem_json(p);
  j["solution"] = detail::flat_json(rep.solution.values());
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
  const nlohmann::json j = detail::read_json(path);
  if (!j.contains("solution")) throw io_error(path + ": not a solution file");
  if (j.value("complex", false) != is_complex_v<T>)
    throw io_error(path + ": scalar type does not match the solution file");
  const std::vector<int> dims = detail::json_dims(j);
  std::size_t total = 1;
  for (int n : dims) total *= static_cast<std::size_t>(n);
  return Tensor<T>(dims, detail::json_flat<T>(j["solution"], total, "solution"));
}

}  // namespace tsylv
