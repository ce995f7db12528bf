// Processor grid, shard placement and activation index maps (pure host code).
//
// Generalises the reference's p x p x p cube to px x py x pz:
//   rank linearisation      cube3d/topology.hpp:68-77
//   axis groups / lines     cube3d/topology.hpp:79-107
//   shard_bounds            cube3d/layout.hpp:93-123
//   diagonal placement      cube3d/layout.hpp:134-142
//   activation map          cube3d/activation.hpp:103-138
// On a cube (px == py == pz) every formula reduces to the reference's, including
// its divisibility errors (both dimensions divisible by p^2).
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <string>
#include <vector>

#include "common.hpp"

namespace c3d {

enum Axis : int { kX = 0, kY = 1, kZ = 2 };
enum Layout : int { kInput = 0, kWeight = 1, kOutput = 2, kWeightOfTranspose = 3 };

inline const char* axis_name(int a) { return a == 0 ? "x" : a == 1 ? "y" : a == 2 ? "z" : "?"; }
inline const char* layout_name(int l) {
  switch (l) {
    case kInput: return "Input";
    case kWeight: return "Weight";
    case kOutput: return "Output";
    case kWeightOfTranspose: return "WeightOfTranspose";
  }
  return "?";
}

// DirectionTriple (cube3d/layout.hpp:44-61).
struct Dirs {
  int in = kY, w = kX, out = kZ;
  void validate() const {
    if (in < 0 || in > 2 || w < 0 || w > 2 || out < 0 || out > 2 || in == w || in == out ||
        w == out)
      fail(C3D_ERR_DIRECTION_CLASH, std::string("axes must be pairwise distinct, got (") +
                                         axis_name(in) + "," + axis_name(w) + "," +
                                         axis_name(out) + ")");
  }
  Dirs swapped() const { return Dirs{out, w, in}; }
  bool operator==(const Dirs& o) const { return in == o.in && w == o.w && out == o.out; }
  bool operator!=(const Dirs& o) const { return !(*this == o); }
};

// triple_for_group (cube3d/activation.hpp:28-35): group 0 -> (y,x,z), 1 -> (z,x,y).
inline int axis_of_group(int g) {
  if (g != 0 && g != 1) fail(C3D_ERR_GROUP_MISMATCH, "group index must be 0 or 1");
  return g == 0 ? kY : kZ;
}
inline Dirs triple_for_group(int g) { return Dirs{axis_of_group(g), kX, axis_of_group(1 - g)}; }

struct Range {
  int64_t begin = 0, end = 0;
  int64_t size() const { return end - begin; }
};
struct Bounds {
  Range rows, cols;
};

struct Grid {
  std::array<int, 3> dims{1, 1, 1};

  Grid() = default;
  explicit Grid(const int d[3]) {
    for (int a = 0; a < 3; ++a) {
      if (d[a] < 1)
        fail(C3D_ERR_NOT_A_CUBE, "grid extent along " + std::string(axis_name(a)) +
                                     " must be >= 1, got " + std::to_string(d[a]));
      dims[a] = d[a];
    }
  }
  int size() const { return dims[0] * dims[1] * dims[2]; }
  bool cubic() const { return dims[0] == dims[1] && dims[1] == dims[2]; }
  int extent(int axis) const { return dims[axis]; }

  void check(const std::array<int, 3>& c) const {
    for (int a = 0; a < 3; ++a)
      if (c[a] < 0 || c[a] >= dims[a])
        fail(C3D_ERR_OUT_OF_RANGE, "coords (" + std::to_string(c[0]) + "," +
                                       std::to_string(c[1]) + "," + std::to_string(c[2]) +
                                       ") outside grid " + std::to_string(dims[0]) + "x" +
                                       std::to_string(dims[1]) + "x" + std::to_string(dims[2]));
  }
  int rank_of(const std::array<int, 3>& c) const {
    check(c);
    return (c[0] * dims[1] + c[1]) * dims[2] + c[2];
  }
  std::array<int, 3> coords_of(int rank) const {
    if (rank < 0 || rank >= size())
      fail(C3D_ERR_OUT_OF_RANGE,
           "rank " + std::to_string(rank) + " not in [0, " + std::to_string(size()) + ")");
    return {rank / (dims[1] * dims[2]), (rank / dims[2]) % dims[1], rank % dims[2]};
  }
  std::vector<int> axis_group(const std::array<int, 3>& c, int axis) const {
    check(c);
    std::vector<int> m;
    for (int q = 0; q < dims[axis]; ++q) {
      auto cc = c;
      cc[axis] = q;
      m.push_back(rank_of(cc));
    }
    return m;
  }
  int line_index(const std::array<int, 3>& c, int axis) const {
    check(c);
    switch (axis) {
      case kX: return c[1] * dims[2] + c[2];
      case kY: return c[0] * dims[2] + c[2];
      default: return c[0] * dims[1] + c[1];
    }
  }
};

inline void require_divisible(int64_t value, int64_t divisor, const std::string& dim) {
  if (divisor <= 0 || value % divisor != 0)
    fail(C3D_ERR_INDIVISIBLE_SHAPE,
         dim + "=" + std::to_string(value) + " must be divisible by " + std::to_string(divisor));
}

// shard_bounds (cube3d/layout.hpp:93-123) with per-axis extents.
inline Bounds shard_bounds(int layout, const Grid& g, const std::array<int, 3>& c, int64_t rows,
                           int64_t cols, const Dirs& d) {
  d.validate();
  g.check(c);
  const int64_t Pi = g.dims[d.in], Pw = g.dims[d.w], Po = g.dims[d.out];
  if (g.cubic()) {
    const int64_t p = g.dims[0];
    require_divisible(rows, p * p, "rows");
    require_divisible(cols, p * p, "cols");
  }
  const int64_t a = c[d.in], w = c[d.w], o = c[d.out];
  Bounds b;
  switch (layout) {
    case kInput:
    case kOutput: {
      require_divisible(rows, Pw * Pi, "rows");
      require_divisible(cols, Po, "cols");
      const int64_t r2 = rows / (Pw * Pi), cl = cols / Po;
      b.rows = {(w * Pi + a) * r2, (w * Pi + a) * r2 + r2};
      b.cols = {o * cl, o * cl + cl};
      return b;
    }
    case kWeight: {
      require_divisible(rows, Po, "rows");
      require_divisible(cols, Pi * Pw, "cols");
      const int64_t rl = rows / Po, c2 = cols / (Pi * Pw);
      b.rows = {o * rl, o * rl + rl};
      b.cols = {(a * Pw + w) * c2, (a * Pw + w) * c2 + c2};
      return b;
    }
    case kWeightOfTranspose: {
      require_divisible(rows, Pi * Pw, "rows");
      require_divisible(cols, Po, "cols");
      const int64_t r2 = rows / (Pi * Pw), cl = cols / Po;
      b.rows = {(a * Pw + w) * r2, (a * Pw + w) * r2 + r2};
      b.cols = {o * cl, o * cl + cl};
      return b;
    }
  }
  fail(C3D_ERR_INTERNAL, "unknown layout " + std::to_string(layout));
}

// Diagonal placement (cube3d/layout.hpp:134-142), generalised to py != pz.
// The reference (py == pz == q): rank (i, j, l) holds b[j*N/q + i*N/(q*px), +N/(q*px))
// iff j == l. Sub-grids with one of py, pz equal to 1 (the north star's 2x2x1): every
// rank holds b[u*N/Q + i*N/(Q*px), +N/(Q*px)) with Q = max(py, pz) and u its coordinate
// on the longer of the two axes -- each (i, u) owns one slice, and expand_diagonal /
// reduce_to_diagonal gather / reduce along that axis instead of broadcasting from the
// diagonal. Other py != pz grids have no consistent rule (the slice index would depend on
// the direction triple) and are rejected.
inline void require_diagonal_grid(const Grid& g) {
  const int py = g.dims[1], pz = g.dims[2];
  if (py != pz && py != 1 && pz != 1)
    fail(C3D_ERR_CONFIG_INVALID, "diagonal vectors need py == pz or one of them 1, got " +
                                     std::to_string(py) + " and " + std::to_string(pz));
}
inline bool diagonal_holder(const Grid& g, const std::array<int, 3>& c) {
  require_diagonal_grid(g);
  return g.dims[1] == g.dims[2] ? c[1] == c[2] : true;
}
inline Range diagonal_slice(const Grid& g, const std::array<int, 3>& c, int64_t len) {
  require_diagonal_grid(g);
  const int64_t Q = std::max(g.dims[1], g.dims[2]), r = g.dims[0];
  if (g.cubic()) require_divisible(len, Q * Q, "vector length");
  require_divisible(len, Q * r, "vector length");
  const int64_t n2 = len / (Q * r);
  const int64_t u = g.dims[1] >= g.dims[2] ? c[1] : c[2];
  const int64_t b0 = u * (len / Q) + static_cast<int64_t>(c[0]) * n2;
  return {b0, b0 + n2};
}

// Activation geometry for group g on this grid.
struct ActGeom {
  int64_t bl, sl, hl;  // local batch, seq, hidden
  int in_axis, out_axis;
};
inline ActGeom act_geom(const Grid& g, int64_t batch, int64_t seq, int64_t hidden, int group) {
  const int ia = axis_of_group(group), oa = axis_of_group(1 - group);
  require_divisible(batch, g.dims[kX], "batch");
  require_divisible(seq, g.dims[ia], "seq");
  if (g.cubic()) require_divisible(hidden, static_cast<int64_t>(g.dims[0]) * g.dims[0], "hidden");
  require_divisible(hidden, g.dims[oa], "hidden");
  return {batch / g.dims[kX], seq / g.dims[ia], hidden / g.dims[oa], ia, oa};
}

}  // namespace c3d
