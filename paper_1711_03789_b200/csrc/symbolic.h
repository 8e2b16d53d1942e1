// Nested-dissection symbolic analysis of one sparse matrix (host C++).
#pragma once
#include <stdint.h>

#include <vector>

namespace mdd {

struct SymIn {
  int32_t n = 0;
  const int32_t* rowptr = nullptr;  // local pattern (sorted, structurally symmetric)
  const int32_t* cols = nullptr;
  const int32_t* xyz = nullptr;     // (n,3) DOF coordinates in 1/grid cell units
  int32_t grid = 2;                 // coordinate units per mesh cell (vertex planes at multiples)
};

struct SymNode {
  int32_t piv_begin = 0, np = 0;  // pivots = ND indices [piv_begin, piv_begin+np)
  int32_t parent = -1;
  int32_t level = 0;              // height: leaves 0
  std::vector<int32_t> children;
  std::vector<int32_t> upd;       // sorted ND indices >= piv_begin+np coupled to the node
};

struct SymOut {
  std::vector<int32_t> perm;   // ND index -> local index
  std::vector<int32_t> iperm;  // local index -> ND index
  std::vector<SymNode> nodes;  // post-order (children before parents)
  int32_t nlevels = 0;
};

// Recursive geometric bisection on grid planes (exact separators for the
// Kuhn mesh; any left-right coupling found is moved into the separator, so
// the result is valid for an arbitrary pattern), then multifrontal update
// sets.
void nd_analyze(const SymIn& in, int32_t leaf, SymOut& out);

}  // namespace mdd
