// mprof — command line front end over the GPU engines (drop-in for the reference's
// tools/mprof_main.cpp: same subcommands, flags, output bytes and exit codes: 0 ok, 1 I/O error,
// 2 usage or any other error). The reference uses CLI11, which is not available here; this is a
// small hand-written parser accepting `--flag value` and `--flag=value`.
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <memory>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "mprof/aamp.hpp"
#include "mprof/acamp.hpp"
#include "mprof/bench.hpp"
#include "mprof/csv_io.hpp"
#include "mprof/multi_gpu.hpp"
#include "mprof/oracle.hpp"

namespace {

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Option {
  std::string help;
  bool flag = false;                 // takes no value
  std::set<std::string> choices;     // empty: any value
  bool required = false;
  bool seen = false;
  std::string value;
};

class Command {
 public:
  explicit Command(std::string about) : about_(std::move(about)) {}
  Option& add(const std::string& name, const std::string& help, bool flag = false) {
    order_.push_back(name);
    Option& o = opts_[name];
    o.help = help;
    o.flag = flag;
    return o;
  }
  // returns false when --help was requested (help already printed)
  bool parse(int argc, char** argv, int first) {
    for (int a = first; a < argc; ++a) {
      std::string arg = argv[a];
      if (arg == "--help" || arg == "-h") {
        print_help(std::cout);
        return false;
      }
      if (arg.rfind("--", 0) != 0) throw UsageError("unexpected argument '" + arg + "'");
      std::string name = arg.substr(2), value;
      bool has_value = false;
      if (const auto eq = name.find('='); eq != std::string::npos) {
        value = name.substr(eq + 1);
        name = name.substr(0, eq);
        has_value = true;
      }
      auto it = opts_.find(name);
      if (it == opts_.end()) throw UsageError("unknown option --" + name);
      Option& o = it->second;
      if (o.flag) {
        if (has_value) throw UsageError("--" + name + " takes no value");
      } else if (!has_value) {
        if (a + 1 >= argc) throw UsageError("--" + name + " needs a value");
        value = argv[++a];
      }
      if (!o.choices.empty() && !o.choices.count(value))
        throw UsageError("--" + name + ": '" + value + "' is not one of the accepted values");
      o.seen = true;
      o.value = value;
    }
    for (const auto& n : order_)
      if (opts_[n].required && !opts_[n].seen) throw UsageError("--" + n + " is required");
    return true;
  }
  bool seen(const std::string& n) const { return opts_.at(n).seen; }
  const std::string& str(const std::string& n) const { return opts_.at(n).value; }
  void print_help(std::ostream& out) const {
    out << about_ << "\n\noptions:\n";
    for (const auto& n : order_) {
      const Option& o = opts_.at(n);
      out << "  --" << n << (o.flag ? "" : " <value>") << "   " << o.help
          << (o.required ? " (required)" : "") << "\n";
    }
  }

 private:
  std::string about_;
  std::vector<std::string> order_;
  std::map<std::string, Option> opts_;
};

std::size_t to_size(const std::string& name, const std::string& v) {
  if (v.empty() || v[0] == '-') throw UsageError("--" + name + ": expected a non-negative integer");
  char* end = nullptr;
  const unsigned long long x = std::strtoull(v.c_str(), &end, 10);
  if (*end) throw UsageError("--" + name + ": expected a non-negative integer");
  return static_cast<std::size_t>(x);
}

double to_real(const std::string& name, const std::string& v) {
  char* end = nullptr;
  const double x = std::strtod(v.c_str(), &end);
  if (v.empty() || *end) throw UsageError("--" + name + ": expected a number");
  return x;
}

std::vector<std::string> split(const std::string& v) {
  std::vector<std::string> out;
  std::stringstream ss(v);
  std::string item;
  while (std::getline(ss, item, ',')) out.push_back(item);
  return out;
}

// ---- compute ---------------------------------------------------------------------------------

// What `compute` was asked to do, after flag validation.
struct ComputeRequest {
  std::string input, output;
  mprof::ProfileConfig cfg{1, mprof::DistanceKind::euclidean()};
  bool brute = false;      // --engine oracle
  bool sq_space = false;   // --acamp-variant sq
  bool progress = false;
  std::vector<int> devices;
};

// Reads the series from a path or, for "-", standard input.
mprof::TimeSeries load_series(const std::string& path) {
  if (path == "-") return mprof::read_series_csv(std::cin);
  std::ifstream file(path, std::ios::binary);
  if (!file.is_open()) throw mprof::Error(mprof::ErrorCode::Io, "input '" + path + "' cannot be opened");
  return mprof::read_series_csv(file);
}

// Runs `emit` on standard output ("" or "-") or on a freshly created file.
template <class Emit>
void with_output(const std::string& path, Emit&& emit) {
  if (path.empty() || path == "-") {
    emit(std::cout);
    return;
  }
  std::ofstream file(path, std::ios::binary);
  if (!file.is_open()) throw mprof::Error(mprof::ErrorCode::Io, "output '" + path + "' cannot be created");
  emit(file);
  if (!file) throw mprof::Error(mprof::ErrorCode::Io, "writing '" + path + "' failed");
}

// Percent lines on standard error, one per change of the integer percentage.
class PercentReporter {
 public:
  bool operator()(std::size_t done, std::size_t total) {
    const int pct = total == 0 ? 100 : static_cast<int>(100.0 * double(done) / double(total));
    if (pct != *shown_) {
      *shown_ = pct;
      std::fprintf(stderr, "%d%%\n", pct);
    }
    return true;  // never cancels
  }

 private:
  std::shared_ptr<int> shown_ = std::make_shared<int>(-1);  // shared by the ProgressFn copies
};

mprof::MatrixProfile execute(const ComputeRequest& rq) {
  const mprof::TimeSeries ts = load_series(rq.input);
  const mprof::DistanceFamily fam = rq.cfg.kind.family;
  if (rq.brute) return mprof::brute_profile(ts, rq.cfg);
  if (!rq.devices.empty()) {
    using E = mprof::Engine;
    const E engine = fam == mprof::DistanceFamily::PNorm ? E::AampPnorm
                     : fam == mprof::DistanceFamily::ZNormalized ? E::Acamp : E::Aamp;
    return mprof::profile_on_devices(ts, rq.cfg, rq.devices, engine);
  }
  const mprof::ProgressFn observer = rq.progress ? mprof::ProgressFn(PercentReporter{}) : mprof::ProgressFn{};
  switch (fam) {
    case mprof::DistanceFamily::PNorm:
      return mprof::aamp_pnorm(ts, rq.cfg, observer);
    case mprof::DistanceFamily::ZNormalized:
      return mprof::acamp(ts, rq.cfg,
                          rq.sq_space ? mprof::AcampVariant::SquaredDistance : mprof::AcampVariant::FScore,
                          observer);
    default:
      return mprof::aamp(ts, rq.cfg, observer);
  }
}

int compute(int argc, char** argv) {
  Command c("mprof compute: compute a matrix profile from a CSV series");
  c.add("input", "input CSV path, '-' for standard input").required = true;
  c.add("m", "subsequence length").required = true;
  Option& dist = c.add("distance", "distance kind: euclidean | pnorm | znorm");
  dist.required = true;
  dist.choices = {"euclidean", "pnorm", "znorm"};
  c.add("p", "p-norm exponent >= 1 (required with --distance pnorm)");
  c.add("output", "output CSV path (default: standard output)");
  c.add("exclusion", "minimum |i - j| between paired subsequences (default 1)");
  c.add("order", "diagonal schedule: asc | random (result is schedule-independent)").choices = {"asc", "random"};
  c.add("seed", "schedule seed for --order random");
  c.add("engine", "auto = the diagonal sweep on the GPU; oracle = brute force (GPU)").choices = {"auto", "oracle"};
  c.add("acamp-variant", "znorm comparison space: f | sq").choices = {"f", "sq"};
  c.add("threads", "accepted for compatibility (the GPU sweep ignores it)");
  c.add("devices", "comma-separated CUDA devices to split the diagonals across (default: one)");
  c.add("progress", "emit percent lines to standard error", true);
  if (!c.parse(argc, argv, 2)) return 0;

  // --p belongs to the p-norm and only to it (usage error otherwise)
  const std::string distance = c.str("distance");
  if ((distance == "pnorm") != c.seen("p"))
    throw UsageError(c.seen("p") ? "--p applies to --distance pnorm only"
                                 : "--distance pnorm needs an exponent (--p)");
  ComputeRequest rq;
  const mprof::DistanceKind kind = distance == "pnorm"   ? mprof::DistanceKind::pnorm(to_real("p", c.str("p")))
                                   : distance == "znorm" ? mprof::DistanceKind::znormalized()
                                                         : mprof::DistanceKind::euclidean();
  rq.cfg = mprof::ProfileConfig(to_size("m", c.str("m")), kind);
  if (c.seen("exclusion")) rq.cfg.exclusion = to_size("exclusion", c.str("exclusion"));
  if (c.seen("order") && c.str("order") == "random") rq.cfg.order = mprof::DiagonalOrder::RandomPermutation;
  if (c.seen("seed")) rq.cfg.order_seed = to_size("seed", c.str("seed"));
  if (c.seen("threads")) (void)to_size("threads", c.str("threads"));
  rq.input = c.str("input");
  rq.output = c.seen("output") ? c.str("output") : std::string();
  rq.brute = c.seen("engine") && c.str("engine") == "oracle";
  rq.sq_space = c.seen("acamp-variant") && c.str("acamp-variant") == "sq";
  rq.progress = c.seen("progress");
  if (c.seen("devices")) {
    for (const auto& d : split(c.str("devices"))) rq.devices.push_back(static_cast<int>(to_size("devices", d)));
    if (rq.devices.empty()) throw UsageError("--devices: expected a device list");
  }
  const mprof::MatrixProfile profile = execute(rq);
  with_output(rq.output, [&](std::ostream& out) { mprof::write_profile_csv(profile, out); });
  return 0;
}

// ---- bench -----------------------------------------------------------------------------------

std::vector<std::size_t> size_list(const Command& c, const char* name) {
  std::vector<std::size_t> v;
  if (c.seen(name))
    for (const auto& x : split(c.str(name))) v.push_back(to_size(name, x));
  return v;
}

int bench(int argc, char** argv) {
  Command c("mprof bench: time the engines on seeded random series");
  c.add("sweep", "vary n (m fixed) or m (n fixed); default n").choices = {"n", "m"};
  c.add("n-list", "comma-separated series lengths");
  c.add("m-list", "comma-separated subsequence lengths");
  c.add("engines", "comma-separated: aamp, aamp_pnorm, acamp_sq, acamp_f, oracle (default aamp,acamp_f)");
  c.add("repeats", "runs averaged per row (default 2)");
  c.add("seed", "series generator seed");
  c.add("output", "report CSV path (default: standard output)");
  if (!c.parse(argc, argv, 2)) return 0;
  mprof::BenchPlan plan;
  plan.sweep = c.seen("sweep") && c.str("sweep") == "m" ? mprof::BenchPlan::Sweep::M : mprof::BenchPlan::Sweep::N;
  plan.n_list = size_list(c, "n-list");
  plan.m_list = size_list(c, "m-list");
  if (c.seen("engines")) plan.engines = split(c.str("engines"));
  for (const auto& e : plan.engines)
    if (!mprof::is_bench_engine(e)) throw UsageError("--engines: '" + e + "' is not a bench engine");
  if (c.seen("repeats")) {
    const std::size_t r = to_size("repeats", c.str("repeats"));
    if (r == 0) throw UsageError("--repeats must be at least 1");
    plan.repeats = static_cast<int>(r);
  }
  if (c.seen("seed")) plan.seed = to_size("seed", c.str("seed"));
  with_output(c.seen("output") ? c.str("output") : std::string(),
              [&](std::ostream& out) { mprof::run_bench(plan, &out); });
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  const std::string usage =
      "mprof: matrix profile engines over CSV time series (GPU)\n\n"
      "subcommands:\n  compute   compute a matrix profile from a CSV series\n"
      "  bench     time the engines on seeded random series\n\nrun 'mprof <subcommand> --help'\n";
  try {
    if (argc < 2) throw UsageError("a subcommand is required");
    const std::string sub = argv[1];
    if (sub == "--help" || sub == "-h") {
      std::cout << usage;
      return 0;
    }
    if (sub == "compute") return compute(argc, argv);
    if (sub == "bench") return bench(argc, argv);
    throw UsageError("unknown subcommand '" + sub + "'");
  } catch (const UsageError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  } catch (const mprof::Error& e) {
    std::cerr << "error: " << e.what() << "\n";
    return e.code() == mprof::ErrorCode::Io ? 1 : 2;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  }
}
