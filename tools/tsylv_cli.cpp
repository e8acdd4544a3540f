// tsylv — command-line front end of the B200 build (the
// reference's proj/tools/tsylv.cpp): solve JSON problem files on the GPU,
// time n_min sweeps and scaling grids (CSV), run the seeded verification
// suite.  Same subcommands, flags, output lines and exit codes:
//
//   0 success, 1 I/O or bad input (parse errors included), 2 numerically
//   singular operator, 3 factorization non-convergence, 4 verify failure.
//
// The reference parses argv with CLI11, which this image lacks; the small
// table-driven parser below accepts the same spellings ("--flag value",
// "--flag=value", comma lists, --help on every level).  Built by
// paper_1905_09539_b200/build.py:build_cli() into paper_1905_09539_b200/bin/.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <functional>
#include <stdexcept>
#include <string>
#include <variant>
#include <vector>

#include "tsylv/bench.hpp"
#include "tsylv/io.hpp"
#include "tsylv/tsylv.hpp"

namespace {

using namespace tsylv;

struct usage_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ---- argv parsing ---------------------------------------------------------

struct Option {
  std::string name, help;
  bool flag = false;  // no value
  bool required = false;
  std::vector<std::string> choices;
  std::function<void(const std::string&)> set;
  bool seen = false;
};

struct Command {
  std::string name, help;
  std::vector<Option> opts;

  Option& add(std::string name, std::string help, std::function<void(const std::string&)> set) {
    opts.push_back(Option{std::move(name), std::move(help), false, false, {}, std::move(set)});
    return opts.back();
  }
  void usage(FILE* f) const {
    std::fprintf(f, "tsylv %s — %s\n\noptions:\n", name.c_str(), help.c_str());
    for (const Option& o : opts) {
      std::string spell = o.name + (o.flag ? "" : " VALUE");
      std::string extra = o.required ? " (required)" : "";
      if (!o.choices.empty()) {
        extra += " {";
        for (std::size_t i = 0; i < o.choices.size(); ++i) extra += (i ? "," : "") + o.choices[i];
        extra += "}";
      }
      std::fprintf(f, "  %-22s %s%s\n", spell.c_str(), o.help.c_str(), extra.c_str());
    }
  }
  // returns false when --help was asked for
  bool parse(const std::vector<std::string>& args) {
    for (std::size_t i = 0; i < args.size(); ++i) {
      std::string key = args[i], value;
      bool inline_value = false;
      if (key == "--help" || key == "-h") return false;
      if (const auto eq = key.find('='); key.rfind("--", 0) == 0 && eq != std::string::npos) {
        value = key.substr(eq + 1);
        key = key.substr(0, eq);
        inline_value = true;
      }
      Option* o = nullptr;
      for (Option& c : opts)
        if (c.name == key) o = &c;
      if (!o) throw usage_error(name + ": unknown option " + args[i]);
      if (o->flag) {
        if (inline_value) throw usage_error(name + ": " + key + " takes no value");
        value = "1";
      } else if (!inline_value) {
        if (i + 1 >= args.size()) throw usage_error(name + ": " + key + " needs a value");
        value = args[++i];
      }
      if (!o->choices.empty() && std::find(o->choices.begin(), o->choices.end(), value) == o->choices.end())
        throw usage_error(name + ": " + key + " must be one of its listed values, got '" + value + "'");
      try {
        o->set(value);
      } catch (const std::logic_error&) {  // stoi / stod failures
        throw usage_error(name + ": bad value '" + value + "' for " + key);
      }
      o->seen = true;
    }
    for (const Option& o : opts)
      if (o.required && !o.seen) throw usage_error(name + ": " + o.name + " is required");
    return true;
  }
};

auto to_int(int& dst) {
  return [&dst](const std::string& v) {
    std::size_t k = 0;
    dst = std::stoi(v, &k);
    if (k != v.size()) throw std::invalid_argument(v);
  };
}
auto to_u64(std::uint64_t& dst) {
  return [&dst](const std::string& v) {
    std::size_t k = 0;
    dst = std::stoull(v, &k);
    if (k != v.size()) throw std::invalid_argument(v);
  };
}
auto to_double(double& dst) {
  return [&dst](const std::string& v) {
    std::size_t k = 0;
    dst = std::stod(v, &k);
    if (k != v.size()) throw std::invalid_argument(v);
  };
}
auto to_str(std::string& dst) {
  return [&dst](const std::string& v) { dst = v; };
}
auto to_flag(bool& dst) {
  return [&dst](const std::string&) { dst = true; };
}
auto to_ints(std::vector<int>& dst) {  // comma list, repeatable
  return [&dst](const std::string& v) {
    std::size_t pos = 0;
    while (pos <= v.size()) {
      const std::size_t comma = std::min(v.find(',', pos), v.size());
      const std::string item = v.substr(pos, comma - pos);
      std::size_t k = 0;
      dst.push_back(std::stoi(item, &k));
      if (k != item.size()) throw std::invalid_argument(item);
      pos = comma + 1;
    }
  };
}

// ---- subcommands ----------------------------------------------------------

struct SolveFlags {
  std::string in, out, strategy = "merge", arithmetic = "complex";
  int n_min = 0;
  double tol = 0;
};

struct BenchFlags {
  std::string family = "laplace", strategy = "both", out;
  int d = 0, reps = 5;
  std::vector<int> n, dims, n_min;
  std::uint64_t seed = 1, mem_cap_bytes = std::uint64_t(2) << 30;
  bool baseline = false;
  double tol = 0;
};

struct VerifyFlags {
  std::uint64_t seed = 1;
  int count = 50;
  std::string out;
  double tol = 1e-9;
};

template <typename T>
void print_report(const char* family, const std::vector<int>& dims, const SolveReport<T>& rep) {
  std::string shape;
  for (std::size_t i = 0; i < dims.size(); ++i) shape += (i ? "x" : "") + std::to_string(dims[i]);
  std::printf("family: %s\ndims: %s\nstrategy: %s\nn_min: %d\n", family, shape.c_str(),
              to_string(rep.strategy).c_str(), rep.n_min);
  std::printf("residual: %.6e\ndiscarded_imag: %.6e\n", rep.residual, rep.discarded_imag);
  std::printf("reduction_s: %.6e\nrecursion_s: %.6e\nback_transform_s: %.6e\n", rep.timings.reduction_s,
              rep.timings.recursion_s, rep.timings.back_transform_s);
}

int run_solve(const SolveFlags& f) {
  SolverConfig cfg;
  cfg.n_min = f.n_min;
  cfg.strategy = f.strategy == "recursion" ? Strategy::recursion_only : Strategy::merge;
  cfg.arithmetic = f.arithmetic == "real" ? Arithmetic::real_quasitriangular : Arithmetic::complex_triangular;
  cfg.singularity_tol = f.tol;
  const AnyProblem any = load_problem(f.in);
  std::visit(
      [&](const auto& p) {
        using P = std::decay_t<decltype(p)>;
        constexpr bool lap =
            std::is_same_v<P, LaplaceProblem<double>> || std::is_same_v<P, LaplaceProblem<Complex>>;
        const auto rep = [&] {
          if constexpr (lap)
            return solve_laplace(p, cfg);
          else
            return solve_gsylv(p, cfg);
        }();
        print_report(lap ? "laplace" : "gsylv", p.dims(), rep);
        if (!f.out.empty()) save_solution(f.out, p, rep);
      },
      any);
  return 0;
}

BenchSpec spec_from(const BenchFlags& f) {
  BenchSpec s;
  s.family = f.family == "gsylv" ? Family::gsylv : Family::laplace;
  s.seed = f.seed;
  s.repetitions = f.reps;
  s.mem_cap_bytes = static_cast<std::size_t>(f.mem_cap_bytes);
  s.include_baseline = f.baseline;
  s.singularity_tol = f.tol;
  s.n_min_values = f.n_min;
  if (f.strategy == "recursion")
    s.strategies = {Strategy::recursion_only};
  else if (f.strategy == "merge")
    s.strategies = {Strategy::merge};
  else
    s.strategies = {Strategy::recursion_only, Strategy::merge};
  return s;
}

// CSV to stdout and, when asked, byte-identically to a file (LF endings)
void emit_rows(const std::vector<ResultRow>& rows, const std::string& out) {
  std::string text = csv_header() + "\n";
  for (const ResultRow& r : rows) text += to_csv(r) + "\n";
  std::fwrite(text.data(), 1, text.size(), stdout);
  if (out.empty()) return;
  std::ofstream file(out, std::ios::binary);
  if (!file) throw io_error("cannot open for writing: " + out);
  file << text;
  if (!file) throw io_error("write failed: " + out);
}

int run_bench_nmin(const BenchFlags& f) {
  BenchSpec s = spec_from(f);
  if (!f.dims.empty())
    s.dims = f.dims;
  else if (f.d >= 2 && !f.n.empty())
    s.dims.assign(static_cast<std::size_t>(f.d), f.n.front());
  else
    throw io_error("bench-nmin: pass --dims, or --d with --n");
  emit_rows(bench_nmin(s), f.out);
  return 0;
}

int run_bench_scaling(const BenchFlags& f) {
  if (f.d < 2 || f.n.empty()) throw io_error("bench-scaling: pass --d and an --n grid");
  emit_rows(bench_scaling(spec_from(f), f.d, f.n), f.out);
  return 0;
}

int run_verify_cmd(const VerifyFlags& f) {
  if (!f.out.empty()) std::filesystem::create_directories(f.out);
  const VerifyReport vr = run_verify(f.seed, f.count, f.out, f.tol);
  std::printf("instances: %d\n", vr.instances);
  std::printf("worst_rel_error: %.6e (%s)\n", vr.worst_rel, vr.worst_case.c_str());
  std::printf("worst_residual_vs_bound: %.6e\n", vr.worst_residual);
  std::printf("verify: %s\n", vr.pass ? "PASS" : "FAIL");
  return vr.pass ? 0 : 4;
}

void top_usage(FILE* f, const std::vector<Command*>& cmds) {
  std::fprintf(f,
               "tsylv — Sylvester-type tensor equations on the GPU (B200 build)\n\n"
               "usage: tsylv SUBCOMMAND [options]   (tsylv SUBCOMMAND --help for its options)\n\nsubcommands:\n");
  for (const Command* c : cmds) std::fprintf(f, "  %-15s %s\n", c->name.c_str(), c->help.c_str());
}

}  // namespace

int main(int argc, char** argv) {
  SolveFlags sf;
  Command solve{"solve", "Solve a problem file and report residual and timings", {}};
  solve.add("--in", "JSON problem file", to_str(sf.in)).required = true;
  solve.add("--out", "write the solution file here", to_str(sf.out));
  solve.add("--nmin", "recursion cutoff (0 = tuned default)", to_int(sf.n_min));
  solve.add("--strategy", "reduced-solve strategy", to_str(sf.strategy)).choices = {"recursion", "merge"};
  solve.add("--arithmetic", "complex (triangular) or real (quasi-triangular)", to_str(sf.arithmetic)).choices = {
      "complex", "real"};
  solve.add("--tol", "singularity tolerance (0 = roundoff-scaled)", to_double(sf.tol));

  BenchFlags nf, scf;
  Command bn{"bench-nmin", "Time one instance across a grid of recursion cutoffs", {}};
  bn.add("--family", "equation family", to_str(nf.family)).choices = {"laplace", "gsylv"};
  bn.add("--d", "tensor order (with --n)", to_int(nf.d));
  bn.add("--n", "extent for cubic instances", to_ints(nf.n));
  bn.add("--dims", "explicit extents, e.g. 40,30,20", to_ints(nf.dims));
  bn.add("--nmin", "cutoff grid, e.g. 2,4,8,16", to_ints(nf.n_min));
  bn.add("--strategy", "strategies timed", to_str(nf.strategy)).choices = {"recursion", "merge", "both"};
  bn.add("--seed", "instance seed", to_u64(nf.seed));
  bn.add("--reps", "runs averaged per row", to_int(nf.reps));
  bn.add("--out", "also write the CSV here", to_str(nf.out));
  bn.add("--tol", "singularity tolerance", to_double(nf.tol));

  Command bs{"bench-scaling", "Compare strategies (and the flattened baseline) over an extent grid", {}};
  bs.add("--family", "equation family", to_str(scf.family)).choices = {"laplace", "gsylv"};
  bs.add("--d", "tensor order", to_int(scf.d)).required = true;
  bs.add("--n", "extent grid, e.g. 8,16,24,32", to_ints(scf.n)).required = true;
  bs.add("--strategy", "strategies timed", to_str(scf.strategy)).choices = {"recursion", "merge", "both"};
  bs.add("--baseline", "also time the flattened one-equation baseline", to_flag(scf.baseline)).flag = true;
  bs.add("--seed", "instance seed", to_u64(scf.seed));
  bs.add("--reps", "runs averaged per row", to_int(scf.reps));
  bs.add("--out", "also write the CSV here", to_str(scf.out));
  bs.add("--mem-cap-bytes", "skip the baseline (status=oom) beyond this footprint", to_u64(scf.mem_cap_bytes));
  bs.add("--tol", "singularity tolerance", to_double(scf.tol));

  VerifyFlags vf;
  Command ver{"verify", "Run the seeded solver-vs-reference suite", {}};
  ver.add("--seed", "suite seed", to_u64(vf.seed));
  ver.add("--count", "instances per family", to_int(vf.count));
  ver.add("--out", "directory for solution files", to_str(vf.out));
  ver.add("--tol", "relative-error tolerance", to_double(vf.tol));

  const std::vector<Command*> cmds{&solve, &bn, &bs, &ver};
  if (argc < 2) {
    top_usage(stderr, cmds);
    std::fprintf(stderr, "error: a subcommand is required\n");
    return 1;
  }
  const std::string sub = argv[1];
  if (sub == "--help" || sub == "-h") {
    top_usage(stdout, cmds);
    return 0;
  }
  Command* cmd = nullptr;
  for (Command* c : cmds)
    if (c->name == sub) cmd = c;
  if (!cmd) {
    top_usage(stderr, cmds);
    std::fprintf(stderr, "error: unknown subcommand '%s'\n", sub.c_str());
    return 1;
  }
  try {
    if (!cmd->parse(std::vector<std::string>(argv + 2, argv + argc))) {
      cmd->usage(stdout);
      return 0;
    }
  } catch (const usage_error& e) {
    cmd->usage(stderr);
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }

  try {
    if (cmd == &solve) return run_solve(sf);
    if (cmd == &bn) return run_bench_nmin(nf);
    if (cmd == &bs) return run_bench_scaling(scf);
    return run_verify_cmd(vf);
  } catch (const singular_error& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  } catch (const factorization_error& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 3;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
