// ref_shim.cpp -- extern "C" shim over the reference's own headers.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile (target `ref`) with
// -I/root/reference/proj/include into oracle/_ref/libvpref.so, so the
// reference's implemented foundations can pin the oracle: Koornwinder
// values (koornwinder.hpp:123-132), Gauss-Legendre rules (gauss.hpp:17-46)
// and quadtree rectangle queries (quadtree.hpp:24-62).  rules.hpp/ggq.hpp
// need Eigen (absent), so they are not built; their tables are pinned via
// tests/golden/ fixtures instead.
#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <vector>

#include "volpot/gauss.hpp"
#include "volpot/geom.hpp"
#include "volpot/koornwinder.hpp"
#include "volpot/quadtree.hpp"

extern "C" {

int vpref_koornwinder(int order, double x, double y, double* out) {
  try {
    volpot::koornwinder_eval(order, x, y, std::span<double>(out, volpot::koorn_size(order)));
  } catch (const std::domain_error&) {
    return 2;
  }
  return 0;
}

int vpref_gauss_legendre(int n, double* x, double* w) {
  try {
    volpot::Rule1d r = volpot::gauss_legendre(n);
    for (int i = 0; i < n; ++i) { x[i] = r.x[i]; w[i] = r.w[i]; }
  } catch (const std::invalid_argument&) {
    return 1;
  }
  return 0;
}

int vpref_quadtree_query(int64_t n_pts, const double* pts, int leaf_cap, double lox, double loy,
                         double hix, double hiy, int32_t* out, int64_t cap, int64_t* n_out,
                         int64_t* visited) {
  try {
    std::vector<volpot::Vec2> p(n_pts);
    for (int64_t i = 0; i < n_pts; ++i) p[i] = {pts[2 * i], pts[2 * i + 1]};
    volpot::Quadtree t = volpot::Quadtree::build(p, leaf_cap);
    volpot::Quadtree::QueryStats st;
    std::vector<int> r = t.query_rect(volpot::Rect{{lox, loy}, {hix, hiy}}, &st);
    std::sort(r.begin(), r.end());
    if (n_out) *n_out = (int64_t)r.size();
    if (visited) *visited = (int64_t)st.nodes_visited;
    if (out) {
      if ((int64_t)r.size() > cap) return 1;
      for (size_t i = 0; i < r.size(); ++i) out[i] = r[i];
    }
  } catch (const std::invalid_argument&) {
    return 1;
  }
  return 0;
}

}  // extern "C"
