// Geometric nested dissection + multifrontal symbolic factorisation.
//
// Replaces nothing in the reference directly: the reference factors each
// subdomain block densely (linalg.DenseLU, linalg.py:73-101, via
// precond.py:166-183).  The DOFs of an edge space carry integer midpoint
// coordinates in half-cell units (order 2: sixth-cell units for edge
// midpoints and face centroids, SymIn::grid); a vertex plane x_axis = c (c a
// multiple of the grid unit) contains exactly the edges (faces) lying in it, and because every
// tetrahedron lies inside one cell, no matrix entry couples an edge with
// coordinate < c to one with coordinate > c.  Recursive bisection along the
// longest axis therefore yields an exact nested-dissection tree whose
// separators are planar edge sets ("Separators are grid
// planes").
#include "symbolic.h"

#include <algorithm>
#include <stdexcept>

namespace mdd {

namespace {

struct Builder {
  const SymIn& in;
  int32_t leaf;
  SymOut& out;
  int32_t next = 0;          // next ND index to assign
  std::vector<int8_t> side;  // scratch: 0 left, 1 sep, 2 right, -1 outside

  Builder(const SymIn& i, int32_t l, SymOut& o) : in(i), leaf(l), out(o) {
    side.assign(in.n, -1);
  }

  int32_t make_node(const std::vector<int32_t>& piv, std::vector<int32_t>&& kids) {
    SymNode nd;
    nd.piv_begin = next;
    nd.np = (int32_t)piv.size();
    for (int32_t v : piv) {
      out.perm[next] = v;
      out.iperm[v] = next;
      ++next;
    }
    nd.children = std::move(kids);
    const int32_t id = (int32_t)out.nodes.size();
    for (int32_t c : nd.children) out.nodes[c].parent = id;
    int32_t lv = 0;
    for (int32_t c : nd.children) lv = std::max(lv, out.nodes[c].level + 1);
    nd.level = lv;
    out.nodes.push_back(std::move(nd));
    return id;
  }

  // returns node id of the subtree root over `set` (local indices)
  int32_t build(std::vector<int32_t>& set) {
    if ((int32_t)set.size() <= leaf) {
      std::sort(set.begin(), set.end());
      return make_node(set, {});
    }
    int32_t lo[3], hi[3];
    for (int a = 0; a < 3; ++a) { lo[a] = INT32_MAX; hi[a] = INT32_MIN; }
    for (int32_t v : set)
      for (int a = 0; a < 3; ++a) {
        lo[a] = std::min(lo[a], in.xyz[3 * v + a]);
        hi[a] = std::max(hi[a], in.xyz[3 * v + a]);
      }
    int axes[3] = {0, 1, 2};
    std::stable_sort(axes, axes + 3, [&](int x, int y) { return hi[x] - lo[x] > hi[y] - lo[y]; });
    int best_axis = -1;
    int32_t best_c = 0;
    std::vector<int32_t> vals;
    for (int ai = 0; ai < 3 && best_axis < 0; ++ai) {
      const int a = axes[ai];
      if (hi[a] - lo[a] < 2) continue;
      vals.clear();
      for (int32_t v : set) vals.push_back(in.xyz[3 * v + a]);
      std::nth_element(vals.begin(), vals.begin() + vals.size() / 2, vals.end());
      const int32_t med = vals[vals.size() / 2];
      // vertex planes lie at multiples of the grid unit
      const int32_t g = in.grid > 0 ? in.grid : 2;
      const int32_t fl = (med >= 0 ? med / g : -((-med + g - 1) / g)) * g;
      int32_t cands[2];
      if (fl == med) { cands[0] = med; cands[1] = med; }
      else { cands[0] = fl; cands[1] = fl + g; }
      int64_t best_imb = INT64_MAX;
      for (int32_t c : cands) {
        if (c <= lo[a] || c >= hi[a]) continue;
        int64_t nl = 0, nr = 0;
        for (int32_t v : set) {
          const int32_t x = in.xyz[3 * v + a];
          nl += x < c;
          nr += x > c;
        }
        if (nl == 0 || nr == 0) continue;
        const int64_t imb = nl > nr ? nl - nr : nr - nl;
        if (imb < best_imb) { best_imb = imb; best_axis = a; best_c = c; }
      }
    }
    if (best_axis < 0) {  // cannot split: dense leaf
      std::sort(set.begin(), set.end());
      return make_node(set, {});
    }
    for (int32_t v : set) {
      const int32_t x = in.xyz[3 * v + best_axis];
      side[v] = x < best_c ? 0 : (x == best_c ? 1 : 2);
    }
    // safety: any left vertex coupled to a right vertex joins the separator
    for (int32_t v : set) {
      if (side[v] != 0) continue;
      for (int32_t k = in.rowptr[v]; k < in.rowptr[v + 1]; ++k)
        if (side[in.cols[k]] == 2) { side[v] = 1; break; }
    }
    std::vector<int32_t> L, S, R;
    for (int32_t v : set) {
      if (side[v] == 0) L.push_back(v);
      else if (side[v] == 1) S.push_back(v);
      else R.push_back(v);
    }
    for (int32_t v : set) side[v] = -1;
    std::vector<int32_t>().swap(set);
    std::vector<int32_t> kids;
    if (!L.empty()) kids.push_back(build(L));
    if (!R.empty()) kids.push_back(build(R));
    std::sort(S.begin(), S.end());
    if (S.empty() && kids.size() == 1) return kids[0];
    return make_node(S, std::move(kids));
  }
};

}  // namespace

void nd_analyze(const SymIn& in, int32_t leaf, SymOut& out) {
  if (leaf < 1) leaf = 1;
  out.perm.assign(in.n, -1);
  out.iperm.assign(in.n, -1);
  out.nodes.clear();
  if (in.n == 0) { out.nlevels = 0; return; }
  Builder b(in, leaf, out);
  std::vector<int32_t> all(in.n);
  for (int32_t i = 0; i < in.n; ++i) all[i] = i;
  b.build(all);
  if (b.next != in.n) throw std::runtime_error("nd_analyze: incomplete ordering");
  // update sets in post-order
  std::vector<int32_t> buf;
  int32_t maxlv = 0;
  for (size_t k = 0; k < out.nodes.size(); ++k) {
    SymNode& nd = out.nodes[k];
    const int32_t pend = nd.piv_begin + nd.np;
    buf.clear();
    for (int32_t q = nd.piv_begin; q < pend; ++q) {
      const int32_t v = out.perm[q];
      for (int32_t e = in.rowptr[v]; e < in.rowptr[v + 1]; ++e) {
        const int32_t j = out.iperm[in.cols[e]];
        if (j >= pend) buf.push_back(j);
      }
    }
    for (int32_t c : nd.children)
      for (int32_t j : out.nodes[c].upd)
        if (j >= pend) buf.push_back(j);
    std::sort(buf.begin(), buf.end());
    buf.erase(std::unique(buf.begin(), buf.end()), buf.end());
    nd.upd = buf;
    maxlv = std::max(maxlv, nd.level);
  }
  out.nlevels = maxlv + 1;
}

}  // namespace mdd
