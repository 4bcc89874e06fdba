// hshard-b200 planner: dtypes, error names, exact rationals.
// The names, widths and rational semantics are the reference's API
// (common.hpp:28-113, common.cpp:22-146; planner notice in NOTICE): one table
// per enum, gcd-normalised rationals, floor_mul exact for negative products.
// BF16 is an appended dtype (width 2), the executor error codes are appended
// to Errc.
#include <array>
#include <numeric>
#include <sstream>

#include "hshard/common.hpp"

namespace hshard {

namespace {

struct DTypeInfo {
  DType type;
  const char* name;
  int width;
};

constexpr std::array<DTypeInfo, 5> kDTypes{{
    {DType::F32, "f32", 4},
    {DType::F64, "f64", 8},
    {DType::I32, "i32", 4},
    {DType::I64, "i64", 8},
    {DType::BF16, "bf16", 2},
}};

const DTypeInfo& info(DType t) {
  for (const auto& d : kDTypes)
    if (d.type == t) return d;
  return kDTypes[0];
}

constexpr const char* kErrcNames[] = {
    "OverlappingSubgroups", "CardinalityMismatch", "BadSplitDim",
    "IndivisibleSplit",     "BadRatios",           "DeviceNotInAnnotation",
    "NotRefinable",         "InexactDivision",     "MissingSymbol",
    "NonPositive",          "CycleDetected",       "DgUnionMismatch",
    "UnderivableSharding",  "PartialUnderBsr",     "UnsupportedHdimTransition",
    "NoOwner",              "UnknownDevice",       "ConflictingStageOrder",
    "SymbolBindingError",   "ShapeMismatch",       "DeadlockDetected",
    "ReplicaDivergence",    "MissingShard",        "UnsupportedOp",
    "UndeducedStrategy",    "ParseError",          "UnexecutableStep",
    "CudaError",            "CommError",
};

int64_t abs64(int64_t v) { return v < 0 ? -v : v; }

}  // namespace

int dtype_width(DType dtype) { return info(dtype).width; }
const char* dtype_name(DType dtype) { return info(dtype).name; }

DType dtype_from_name(const std::string& name) {
  for (const auto& d : kDTypes)
    if (name == d.name) return d.type;
  fail(Errc::ParseError, "'" + name + "' is not a dtype (f32, f64, i32, i64, bf16)");
}

const char* errc_name(Errc code) {
  auto i = static_cast<size_t>(code);
  if (i < sizeof(kErrcNames) / sizeof(kErrcNames[0])) return kErrcNames[i];
  return "UnknownError";
}

Rational::Rational(int64_t n, int64_t d) {
  if (d == 0) fail(Errc::ParseError, "a rational needs a non-zero denominator");
  if (d < 0) {
    n = -n;
    d = -d;
  }
  const int64_t g = std::gcd(abs64(n), d);
  num = g > 1 ? n / g : n;
  den = g > 1 ? d / g : d;
}

Rational Rational::operator+(const Rational& o) const {
  return {num * o.den + o.num * den, den * o.den};
}
Rational Rational::operator-(const Rational& o) const {
  return {num * o.den - o.num * den, den * o.den};
}
Rational Rational::operator*(const Rational& o) const { return {num * o.num, den * o.den}; }
Rational Rational::operator/(const Rational& o) const {
  if (o.num == 0) fail(Errc::ParseError, "division of a rational by zero");
  return {num * o.den, den * o.num};
}
bool Rational::operator<(const Rational& o) const { return num * o.den < o.num * den; }

int64_t Rational::floor_mul(int64_t x) const {
  // den > 0 by construction, so only a negative product needs rounding down.
  const int64_t p = num * x;
  const int64_t q = p / den;
  return (p % den != 0 && p < 0) ? q - 1 : q;
}

std::string Rational::str() const {
  return den == 1 ? std::to_string(num) : std::to_string(num) + "/" + std::to_string(den);
}

Rational Rational::parse(const std::string& text) {
  const size_t slash = text.find('/');
  try {
    if (slash == std::string::npos) return Rational(std::stoll(text));
    return Rational(std::stoll(text.substr(0, slash)), std::stoll(text.substr(slash + 1)));
  } catch (const Error&) {
    throw;
  } catch (const std::exception&) {
    fail(Errc::ParseError, "'" + text + "' is not a rational (N or N/D)");
  }
}

std::string join_ints(const std::vector<int64_t>& v, const std::string& sep) {
  std::string out;
  for (size_t i = 0; i < v.size(); ++i) {
    if (i) out += sep;
    out += std::to_string(v[i]);
  }
  return out;
}

}  // namespace hshard
