// CSV front-end checks re-hosted from the reference's tests/test_csv.cpp (known bytes and error
// codes). Prints one line per failed check; exit 0 iff all pass. CPU only (no CUDA call).
#include <cmath>
#include <cstdio>
#include <limits>
#include <random>
#include <sstream>
#include <string>

#include "mprof/csv_io.hpp"

using namespace mprof;

static int failures = 0;
#define CHECK(cond)                                               \
  do {                                                            \
    if (!(cond)) {                                                \
      std::printf("FAIL line %d: %s\n", __LINE__, #cond);         \
      ++failures;                                                 \
    }                                                             \
  } while (0)

static TimeSeries parse(const std::string& s) {
  std::istringstream in(s);
  return read_series_csv(in);
}
static int code_of(const std::string& s, std::size_t* line = nullptr) {
  try {
    parse(s);
  } catch (const Error& e) {
    if (line) *line = e.line();
    return static_cast<int>(e.code());
  }
  return -1;
}
static std::string render(const MatrixProfile& p) {
  std::ostringstream out;
  write_profile_csv(p, out);
  return out.str();
}

int main() {
  {  // test_csv.cpp:30-38
    const TimeSeries ts = parse("1.5\n2\n-3.25\n4e2\n");
    CHECK(ts.size() == 4 && ts[0] == 1.5 && ts[1] == 2.0 && ts[2] == -3.25 && ts[3] == 400.0);
  }
  CHECK(parse("value\n1\n2\n").size() == 2);                      // header
  {
    const TimeSeries ts = parse("t,extra\n1.5,99\n2.5,98\n");     // first column only
    CHECK(ts.size() == 2 && ts[0] == 1.5 && ts[1] == 2.5);
  }
  {
    const TimeSeries ts = parse("  1.5 \r\n\n\t2.5\r\n+3.5\n");  // whitespace quirks
    CHECK(ts.size() == 3 && ts[0] == 1.5 && ts[1] == 2.5 && ts[2] == 3.5);
  }
  std::size_t line = 0;
  CHECK(code_of("1\nbogus\n3\n", &line) == static_cast<int>(ErrorCode::ParseError) && line == 2);
  CHECK(code_of("1\n2.5abc\n") == static_cast<int>(ErrorCode::ParseError));
  CHECK(code_of("1\n2 3\n") == static_cast<int>(ErrorCode::ParseError));
  CHECK(code_of("1\ninf\n2\n") == static_cast<int>(ErrorCode::NonFinite));
  CHECK(code_of("1\nnan\n2\n") == static_cast<int>(ErrorCode::NonFinite));
  CHECK(code_of("1\n-inf\n2\n") == static_cast<int>(ErrorCode::NonFinite));
  CHECK(code_of("") == static_cast<int>(ErrorCode::EmptyInput));
  CHECK(code_of("value\n") == static_cast<int>(ErrorCode::EmptyInput));
  CHECK(code_of("\n\n") == static_cast<int>(ErrorCode::EmptyInput));
  CHECK(code_of("7.5\n") == static_cast<int>(ErrorCode::TooShort));
  {  // known bytes (test_csv.cpp:99-109)
    MatrixProfile p;
    p.m = 3;
    const double r3 = std::sqrt(3.0);
    p.distances = {0.0, r3, r3, r3, 0.0};
    p.nn_index = {4, 0, 1, 0, 0};
    CHECK(render(p) ==
          "index,distance,nn_index\n0,0.00000000,4\n1,1.73205081,0\n2,1.73205081,1\n"
          "3,1.73205081,0\n4,0.00000000,0\n");
  }
  {  // unresolved entries (test_csv.cpp:111-121)
    MatrixProfile p;
    p.m = 2;
    p.distances = {1.25, std::numeric_limits<double>::infinity()};
    p.nn_index = {1, kNoNeighbor};
    CHECK(render(p) == "index,distance,nn_index\n0,1.25000000,1\n1,inf,\n");
  }
  {  // lossless series round trip (test_csv.cpp:123-135)
    std::mt19937_64 rng(801);
    std::normal_distribution<double> g(0.0, 1.0);
    std::vector<double> s(300);
    for (double& x : s) x = g(rng);
    s[0] = 0.1 + 0.2;
    s[1] = 1e-300;
    s[2] = 12345678901234.5678;
    std::ostringstream out;
    write_series_csv(s, out);
    const TimeSeries back = parse(out.str());
    bool same = back.size() == s.size();
    for (std::size_t i = 0; same && i < s.size(); ++i) same = back[i] == s[i];
    CHECK(same);
  }
  std::printf("%s (%d failures)\n", failures ? "FAIL" : "PASS", failures);
  return failures ? 1 : 0;
}
