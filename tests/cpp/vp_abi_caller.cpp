// vp_abi_caller.cpp -- a plain C++ caller of libvp_b200.so through the C-ABI
// (include/vp.h, include/vp_setup.h) with no Python and no torch: the
// binding a reference maintainer would write.
//
//   vp_abi_caller OUT.bin [config]
//
// builds BASELINE config `config` (default 1) with the library's seeded
// generators, sets mesh / rules / density, evaluates every target, then
// evaluates the two shards of vp_shard_plan separately and checks they
// reproduce the one-shot u bit for bit; writes u (float64, target order) to
// OUT.bin.  Exit status: 0 ok, 3 no usable device (the library has no CPU
// fallback), 1 any other failure.  Built and run by tests/test_abi.py and
// tests/test_gpu_r02.py.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "vp.h"
#include "vp_setup.h"

static int fail(vp_ctx* c, int rc, const char* what) {
  std::fprintf(stderr, "%s failed (%d): %s\n", what, rc, c ? vp_last_error(c) : vps_last_error());
  return rc == 3 ? 3 : 1;
}

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s OUT.bin [config]\n", argv[0]);
    return 1;
  }
  const int cfg = argc > 2 ? std::atoi(argv[2]) : 1;
  vps_config_info info;
  if (int rc = vps_config_info_get(cfg, 0, 0, &info)) return fail(nullptr, rc, "vps_config_info_get");
  const int M = vps_koorn_size(info.p);
  std::vector<double> vxy(2 * info.n_vert), txy(2 * info.n_tgt), coeffs((size_t)info.n_tri * M);
  std::vector<int32_t> tri(3 * info.n_tri);
  if (int rc = vps_config_fill(cfg, 0, 0, vxy.data(), tri.data(), txy.data(), coeffs.data()))
    return fail(nullptr, rc, "vps_config_fill");
  // rules: far order q, near order 12, Gauss-Legendre 16, GGQ order 8
  int lq = 0, ln = 0;
  vps_quad_rule(info.q, &lq, nullptr, nullptr, nullptr);
  vps_quad_rule(12, &ln, nullptr, nullptr, nullptr);
  std::vector<double> fx(lq), fy(lq), fw(lq), nx(ln), ny(ln), nw(ln), gx(16), gw(16), gr(9), gg(9);
  double res = 0.0;
  if (vps_quad_rule(info.q, &lq, fx.data(), fy.data(), fw.data()) ||
      vps_quad_rule(12, &ln, nx.data(), ny.data(), nw.data()) || vps_gauss_legendre(16, gx.data(), gw.data()) ||
      vps_ggq(8, gr.data(), gg.data(), &res))
    return fail(nullptr, 1, "rules");
  vp_rules rules{info.q, lq, fx.data(), fy.data(), fw.data(), 12, ln, nx.data(), ny.data(), nw.data(),
                 16, gx.data(), gw.data(), 8, gr.data(), gg.data(), info.eps};
  vp_ctx* c = nullptr;
  if (int rc = vp_create(0, &c)) {
    std::fprintf(stderr, "vp_create: status %d (no usable sm_100 device; there is no CPU fallback)\n", rc);
    return rc == 3 ? 3 : 1;
  }
  int rc = vp_set_mesh(c, info.n_vert, vxy.data(), info.n_tri, tri.data());
  if (!rc) rc = vp_set_rules(c, &rules);
  if (!rc) rc = vp_set_density(c, info.p, coeffs.data());
  if (rc) return fail(c, rc, "setup");
  std::vector<double> u(info.n_tgt);
  vp_stats st;
  if ((rc = vp_evaluate(c, info.n_tgt, txy.data(), u.data(), &st))) return fail(c, rc, "vp_evaluate");
  // two shards of the cost-balanced Morton plan, evaluated separately
  const int world = 2;
  std::vector<int32_t> order(info.n_tgt);
  int64_t bounds[world + 1], cost[world];
  if ((rc = vp_shard_plan(c, info.n_tgt, txy.data(), world, order.data(), bounds, cost)))
    return fail(c, rc, "vp_shard_plan");
  for (int r = 0; r < world; ++r) {
    const int64_t n = bounds[r + 1] - bounds[r];
    std::vector<double> t(2 * n), us(n);
    for (int64_t i = 0; i < n; ++i) {
      t[2 * i] = txy[2 * order[bounds[r] + i]];
      t[2 * i + 1] = txy[2 * order[bounds[r] + i] + 1];
    }
    if ((rc = vp_evaluate(c, n, t.data(), us.data(), nullptr))) return fail(c, rc, "vp_evaluate shard");
    for (int64_t i = 0; i < n; ++i)
      if (std::memcmp(&us[i], &u[order[bounds[r] + i]], sizeof(double)) != 0) {
        std::fprintf(stderr, "shard %d target %lld differs from the one-shot u\n", r, (long long)i);
        return 1;
      }
  }
  FILE* f = std::fopen(argv[1], "wb");
  if (!f || std::fwrite(u.data(), sizeof(double), u.size(), f) != u.size()) return fail(c, 1, "write");
  std::fclose(f);
  std::printf("config %d: %lld targets, %lld near pairs, %lld leaves, %lld panels, %.3f ms device; "
              "shards (%lld, %lld) bitwise equal\n",
              cfg, (long long)st.n_targets, (long long)st.n_near_pairs, (long long)st.n_leaves,
              (long long)st.n_panels, st.t_total_ms, (long long)(bounds[1] - bounds[0]),
              (long long)(bounds[2] - bounds[1]));
  vp_destroy(c);
  return 0;
}
