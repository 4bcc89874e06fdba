// hshard-b200: host Tensor (the reference tensor.hpp API; semantics of its
// tensor.cpp:22-156, planner notice in NOTICE: row-major doubles whatever the
// dtype tag, ShapeMismatch on a box outside the tensor or an empty one, cell
// order row-major over the box).  Box copies here move contiguous innermost
// runs located by precomputed row strides, not one cell per callback.
#include <algorithm>
#include <cmath>
#include <functional>
#include <numeric>
#include <sstream>

#include "hshard/tensor.hpp"

namespace hshard {

int64_t shape_numel(const Shape& s) {
  return std::accumulate(s.begin(), s.end(), int64_t{1}, std::multiplies<int64_t>());
}

Tensor::Tensor(Shape s, DType t) : shape(std::move(s)), dtype(t), data(shape_numel(shape), 0.0) {}

Tensor Tensor::zeros(Shape s, DType t) { return filled(std::move(s), 0.0, t); }

Tensor Tensor::filled(Shape s, double v, DType t) {
  Tensor out;
  out.data.assign(static_cast<size_t>(shape_numel(s)), v);
  out.shape = std::move(s);
  out.dtype = t;
  return out;
}

int64_t Tensor::numel() const { return shape_numel(shape); }

int64_t Tensor::offset_of(const std::vector<int64_t>& idx) const {  // row-major (Horner)
  int64_t off = 0;
  auto e = shape.begin();
  for (auto i = idx.begin(); e != shape.end(); ++e, ++i) off = off * *e + *i;
  return off;
}

// Row-major over the box: the k-th cell's index is k's mixed-radix digits over
// the box extents, offset by the box origin.
void for_each_cell(const SliceRegion& region, const std::function<void(const std::vector<int64_t>&)>& fn) {
  const size_t rank = region.bounds.size();
  const int64_t cells = region.cells();
  std::vector<int64_t> idx(rank);
  for (int64_t k = 0; k < (rank ? cells : 1); ++k) {
    int64_t rest = k;
    for (size_t d = rank; d-- > 0;) {
      const int64_t ext = region.bounds[d][1] - region.bounds[d][0];
      idx[d] = region.bounds[d][0] + rest % ext;
      rest /= ext;
    }
    fn(idx);
  }
}

namespace {

void check_box(const Tensor& t, const SliceRegion& r) {
  if (static_cast<int>(r.bounds.size()) != t.ndim())
    fail(Errc::ShapeMismatch, "a rank-" + std::to_string(r.bounds.size()) + " box on a rank-" +
                                  std::to_string(t.ndim()) + " tensor");
  for (size_t d = 0; d < r.bounds.size(); ++d) {
    const auto [lo, hi] = r.bounds[d];
    if (lo < 0 || hi > t.shape[d] || lo >= hi)
      fail(Errc::ShapeMismatch, "box " + r.str() + " is empty or leaves the tensor [" + join_ints(t.shape) + "]");
  }
}

void check_payload(const SliceRegion& r, const Tensor& v) {
  if (v.shape != r.extents())
    fail(Errc::ShapeMismatch, "a [" + join_ints(v.shape) + "] payload for box " + r.str());
}

// fn(tensor_offset, box_offset, run_length) for every innermost run of the
// box, in row-major order; rows are located through the tensor's strides.
template <class Fn>
void for_each_run(const Tensor& t, const SliceRegion& r, Fn&& fn) {
  const size_t rank = r.bounds.size();
  if (rank == 0) {
    fn(int64_t{0}, int64_t{0}, int64_t{1});
    return;
  }
  std::vector<int64_t> stride(rank, 1);
  for (size_t d = rank - 1; d > 0; --d) stride[d - 1] = stride[d] * t.shape[d];
  const int64_t run = r.bounds[rank - 1][1] - r.bounds[rank - 1][0];
  int64_t rows = 1;
  for (size_t d = 0; d + 1 < rank; ++d) rows *= r.bounds[d][1] - r.bounds[d][0];
  for (int64_t row = 0; row < rows; ++row) {
    int64_t at = r.bounds[rank - 1][0], rest = row;
    for (size_t d = rank - 1; d-- > 0;) {
      const int64_t ext = r.bounds[d][1] - r.bounds[d][0];
      at += (r.bounds[d][0] + rest % ext) * stride[d];
      rest /= ext;
    }
    fn(at, row * run, run);
  }
}

}  // namespace

Tensor Tensor::slice(const SliceRegion& region) const {
  check_box(*this, region);
  Tensor out(region.extents(), dtype);
  for_each_run(*this, region, [&](int64_t at, int64_t box, int64_t n) {
    std::copy_n(data.begin() + at, n, out.data.begin() + box);
  });
  return out;
}

void Tensor::write_slice(const SliceRegion& region, const Tensor& value) {
  check_box(*this, region);
  check_payload(region, value);
  for_each_run(*this, region, [&](int64_t at, int64_t box, int64_t n) {
    std::copy_n(value.data.begin() + box, n, data.begin() + at);
  });
}

void Tensor::add_slice(const SliceRegion& region, const Tensor& value) {
  check_box(*this, region);
  check_payload(region, value);
  for_each_run(*this, region, [&](int64_t at, int64_t box, int64_t n) {
    for (int64_t i = 0; i < n; ++i) data[at + i] += value.data[box + i];
  });
}

bool Tensor::bit_equal(const Tensor& o) const { return shape == o.shape && data == o.data; }

namespace {

// Largest per-element |a - b| / scale(a, b) of two equally shaped tensors.
template <class Scale>
double max_diff(const Tensor& a, const Tensor& b, const char* what, Scale scale) {
  if (a.shape != b.shape)
    fail(Errc::ShapeMismatch, std::string(what) + " of [" + join_ints(a.shape) + "] and [" + join_ints(b.shape) + "]");
  return std::transform_reduce(a.data.begin(), a.data.end(), b.data.begin(), 0.0,
                               [](double x, double y) { return std::max(x, y); },
                               [&](double x, double y) { return std::fabs(x - y) / scale(x, y); });
}

}  // namespace

double Tensor::max_abs_diff(const Tensor& o) const {
  return max_diff(*this, o, "max_abs_diff", [](double, double) { return 1.0; });
}

double Tensor::max_rel_diff(const Tensor& o) const {
  return max_diff(*this, o, "max_rel_diff",
                  [](double x, double y) { return std::max({std::fabs(x), std::fabs(y), 1.0}); });
}

Tensor& Tensor::operator+=(const Tensor& o) {
  if (shape != o.shape)
    fail(Errc::ShapeMismatch, "cannot add [" + join_ints(o.shape) + "] into [" + join_ints(shape) + "]");
  for (size_t i = 0; i < data.size(); ++i) data[i] += o.data[i];
  return *this;
}

std::string Tensor::str() const {  // dtype[shape]{first 16 values,...}
  std::ostringstream vals;
  const size_t shown = std::min<size_t>(data.size(), 16);
  for (size_t i = 0; i < shown; ++i) vals << (i ? "," : "") << data[i];
  return std::string(dtype_name(dtype)) + "[" + join_ints(shape) + "]{" + vals.str() +
         (data.size() > shown ? ",...}" : "}");
}

}  // namespace hshard
