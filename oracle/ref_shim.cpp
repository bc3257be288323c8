// ref_shim.cpp -- extern "C" shim over the reference's own headers.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile (target `ref`) with
// -I/root/reference/proj/include into oracle/_ref/libvpref.so, so the
// reference's implemented foundations can pin the oracle: Koornwinder
// values (koornwinder.hpp:123-132), Gauss-Legendre rules (gauss.hpp:17-46)
// quadtree rectangle queries (quadtree.hpp:24-62) and the arc-length
// reparametrisation of the boundary curves (curve.hpp:16-332).  rules.hpp/ggq.hpp
// need Eigen (absent), so they are not built; their tables are pinned via
// tests/golden/ fixtures instead.
#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <vector>

#include "volpot/curve.hpp"  // needs <algorithm>, included above
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

// ArcLengthCurve::reparametrize of a reference curve (kind 0 circle (cx, cy,
// r), 1 ellipse (a, b), 2 wobbly (a, b, k), 3 Hermite rows t x y dx dy);
// positions, unit tangents and d2/ds2 at n arc lengths
int vpref_arclength(int kind, const double* prm, int n_prm, int64_t n, const double* s, double* xy,
                    double* tangent, double* dd, double* length, int* ccw) {
  try {
    std::shared_ptr<const volpot::ParamCurve> base;
    if (kind == 0) {
      base = std::make_shared<volpot::CircleCurve>(volpot::Vec2{prm[0], prm[1]}, prm[2]);
    } else if (kind == 1) {
      base = std::make_shared<volpot::EllipseCurve>(prm[0], prm[1]);
    } else if (kind == 2) {
      base = std::make_shared<volpot::WobblyEllipseCurve>(prm[0], prm[1], (int)prm[2]);
    } else if (kind == 3) {
      std::vector<double> t;
      std::vector<volpot::Vec2> p, d;
      for (int i = 0; i + 4 < n_prm; i += 5) {
        t.push_back(prm[i]);
        p.push_back({prm[i + 1], prm[i + 2]});
        d.push_back({prm[i + 3], prm[i + 4]});
      }
      base = std::make_shared<volpot::HermiteCurve>(t, p, d);
    } else {
      return 1;
    }
    const volpot::ArcLengthCurve c = volpot::ArcLengthCurve::reparametrize(base);
    if (length) *length = c.length();
    if (ccw) *ccw = c.counterclockwise() ? 1 : 0;
    for (int64_t i = 0; i < n; ++i) {
      const volpot::Vec2 q = c.position(s[i]);
      xy[2 * i] = q.x;
      xy[2 * i + 1] = q.y;
      if (tangent) {
        const volpot::Vec2 tg = c.tangent(s[i]);
        tangent[2 * i] = tg.x;
        tangent[2 * i + 1] = tg.y;
      }
      if (dd) {
        const volpot::Vec2 a = c.second_derivative(s[i]);
        dd[2 * i] = a.x;
        dd[2 * i + 1] = a.y;
      }
    }
  } catch (const std::exception&) {
    return 1;
  }
  return 0;
}

}  // extern "C"
