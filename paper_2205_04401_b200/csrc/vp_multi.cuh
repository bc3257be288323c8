// vp_multi.cuh -- multi-GPU entry points of the C-ABI:
// targets are sharded over ranks (one process or context per GPU), mesh and
// density are replicated, and the only collective is the gather of u
// (BASELINE.json north_star).  Included at the end of vp_b200.cu.
//
//   vp_shard_plan   Morton order of a target set + a cost-balanced split
//                   into contiguous shards (cost from the near-field lists)
//   vp_shard_bounds the same split from caller-supplied costs (host only)
//   vp_nccl_unique_id / vp_comm_init / vp_gather / vp_allreduce_stats
//                   the library's own NCCL communicator over NVLink/NVSwitch
//
// NCCL is resolved with dlopen("libnccl.so.2") on first use, so a single-GPU
// caller never needs it; in a process that already loaded NCCL (e.g. torch's
// bundled copy) the loaded library is reused.
#include <dlfcn.h>
#include <nccl.h>

namespace {

// ---- NCCL, resolved at run time ---------------------------------------------
struct NcclApi {
  bool tried = false, ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi A;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (A.tried) return A;
  A.tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    A.why = std::string("dlopen libnccl.so.2 failed: ") + (dlerror() ? dlerror() : "?");
    return A;
  }
  auto sym = [&](const char* n) { return dlsym(h, n); };
  A.GetUniqueId = (decltype(A.GetUniqueId))sym("ncclGetUniqueId");
  A.CommInitRank = (decltype(A.CommInitRank))sym("ncclCommInitRank");
  A.CommDestroy = (decltype(A.CommDestroy))sym("ncclCommDestroy");
  A.Broadcast = (decltype(A.Broadcast))sym("ncclBroadcast");
  A.AllReduce = (decltype(A.AllReduce))sym("ncclAllReduce");
  A.GroupStart = (decltype(A.GroupStart))sym("ncclGroupStart");
  A.GroupEnd = (decltype(A.GroupEnd))sym("ncclGroupEnd");
  A.GetErrorString = (decltype(A.GetErrorString))sym("ncclGetErrorString");
  A.ok = A.GetUniqueId && A.CommInitRank && A.CommDestroy && A.Broadcast && A.AllReduce && A.GroupStart &&
         A.GroupEnd && A.GetErrorString;
  if (!A.ok) A.why = "libnccl.so.2 lacks an expected symbol";
  return A;
}

#define NCCL_TRY(ctx, x)                                                                              \
  do {                                                                                                \
    ncclResult_t r_ = (x);                                                                            \
    if (r_ != ncclSuccess)                                                                            \
      return set_err(ctx, 3, std::string("nccl: ") + nccl().GetErrorString(r_) + " at " #x);        \
  } while (0)

// ---- shard plan ----------------------------------------------------------------
// Morton code of a target, the same arithmetic as dist.morton_order (numpy):
// q = min(trunc((t - lo) / span * 65535), 65535) per axis, bits interleaved
// x even / y odd.  Explicitly rounded, so the order equals numpy's.
__device__ __forceinline__ unsigned spread16(unsigned v) {
  v = (v | (v << 8)) & 0x00FF00FFu;
  v = (v | (v << 4)) & 0x0F0F0F0Fu;
  v = (v | (v << 2)) & 0x33333333u;
  v = (v | (v << 1)) & 0x55555555u;
  return v;
}

__global__ void k_morton(int64_t n, const double2* __restrict__ t, double lox, double loy, double spx, double spy,
                         unsigned* __restrict__ code, int32_t* __restrict__ idx) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double2 p = t[i];
  const double fx = __dmul_rn(__ddiv_rn(__dsub_rn(p.x, lox), spx), 65535.0);
  const double fy = __dmul_rn(__ddiv_rn(__dsub_rn(p.y, loy), spy), 65535.0);
  const unsigned qx = fx >= 65535.0 ? 65535u : (unsigned)fx;  // inputs >= 0: truncation = astype(uint64)
  const unsigned qy = fy >= 65535.0 ? 65535u : (unsigned)fy;
  code[i] = spread16(qx) | (spread16(qy) << 1);
  idx[i] = (int32_t)i;
}

__global__ void k_gather_targets_i32(int64_t n, const int32_t* __restrict__ ord, const double2* __restrict__ src,
                                     double2* __restrict__ dst) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[ord[i]];
}

// per-target cost in Morton order: far + near pairs + self (units: FP64 flops)
__global__ void k_shard_cost(int64_t n, const int64_t* __restrict__ nn, const int32_t* __restrict__ self,
                             int64_t c_far, int64_t c_near, int64_t c_self, int64_t* __restrict__ cost) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) cost[i] = c_far + c_near * nn[i] + (self[i] >= 0 ? c_self : 0);
}

// bounds[r] = smallest i with P[i] * world >= r * P[n] (P: exclusive prefix, n+1 entries)
__global__ void k_shard_search(int64_t n, const int64_t* __restrict__ P, int world, int64_t* __restrict__ bounds) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r > world) return;
  const __int128 tot = (__int128)P[n];
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if ((__int128)P[mid] * world >= (__int128)r * tot) hi = mid;
    else lo = mid + 1;
  }
  bounds[r] = r == 0 ? 0 : r == world ? n : lo;
}

// Cost model of one target (FP64 flops): the far field (direct:
// 17 per source; FMM: the P2P of ~9 leaves of `leaf` sources plus L2P), a near
// pair (about 6 leaves x len_n nodes x 13 flops plus a point sum) and the self
// pair (about 16 panels x 16 nodes x 2(p+1) flops plus a point sum).
void shard_cost_model(const vp_ctx* c, int64_t& c_far, int64_t& c_near, int64_t& c_self) {
  const int64_t S = c->n_tri * c->rules.len_q;
  const int64_t lq = c->rules.len_q;
  c_far = c->far_method == 1 ? 17ll * 9 * c->fmm_leaf + 8ll * (c->fmm_p + 1) : c->far_method == 2 ? 0 : 17ll * S;
  c_near = 6ll * c->rules.len_n * 13 + 11ll * lq;
  c_self = 16ll * c->rules.n_l * (2 * (c->p + 1) + 13) + 11ll * lq;
}

}  // namespace

namespace {
void vp_comm_release(vp_ctx* c) {
  if (c && c->comm && nccl().ok) nccl().CommDestroy((ncclComm_t)c->comm);
  if (c) c->comm = nullptr;
}
}  // namespace

extern "C" {

int vp_shard_bounds(int64_t n, const int64_t* cost, int world, int64_t* bounds) {
  if (n < 0 || world <= 0 || !bounds || (n > 0 && !cost)) return 1;
  std::vector<int64_t> P(n + 1, 0);
  for (int64_t i = 0; i < n; ++i) {
    if (cost[i] < 0) return 1;
    P[i + 1] = P[i] + cost[i];
  }
  const __int128 tot = P[n];
  for (int r = 0; r <= world; ++r) {
    if (r == 0 || r == world) {
      bounds[r] = r == 0 ? 0 : n;
      continue;
    }
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = lo + (hi - lo) / 2;
      if ((__int128)P[mid] * world >= (__int128)r * tot) hi = mid;
      else lo = mid + 1;
    }
    bounds[r] = lo;
  }
  return 0;
}

int vp_shard_plan(vp_ctx* c, int64_t n_tgt, const double* txy, int world, int32_t* order_out, int64_t* bounds_out,
                  int64_t* shard_cost_out) {
  if (int rc = ensure_ready(c, true)) return rc;
  if (n_tgt < 0 || n_tgt > (int64_t)INT32_MAX || world <= 0 || (n_tgt > 0 && !txy) || !order_out || !bounds_out)
    return set_err(c, 1, "shard_plan: need 0 <= n_tgt < 2^31 (with targets), world >= 1, order and bounds arrays");
  if (n_tgt == 0) {
    for (int r = 0; r <= world; ++r) bounds_out[r] = 0;
    if (shard_cost_out)
      for (int r = 0; r < world; ++r) shard_cost_out[r] = 0;
    return 0;
  }
  CUDA_TRY(c, cudaSetDevice(c->device));
  double lox = txy[0], loy = txy[1], hix = txy[0], hiy = txy[1];
  for (int64_t i = 0; i < n_tgt; ++i) {
    const double x = txy[2 * i], y = txy[2 * i + 1];
    if (!std::isfinite(x) || !std::isfinite(y)) return set_err(c, 2, "shard_plan: non-finite target coordinate");
    lox = std::min(lox, x); hix = std::max(hix, x);
    loy = std::min(loy, y); hiy = std::max(hiy, y);
  }
  const double spx = hix > lox ? hix - lox : 1.0, spy = hiy > loy ? hiy - loy : 1.0;
  DevBuf dt, dts, code, code2, idx;
  CUDA_TRY(c, dt.ensure(sizeof(double2) * n_tgt));
  CUDA_TRY(c, dts.ensure(sizeof(double2) * n_tgt));
  CUDA_TRY(c, code.ensure(sizeof(unsigned) * n_tgt));
  CUDA_TRY(c, code2.ensure(sizeof(unsigned) * n_tgt));
  CUDA_TRY(c, idx.ensure(sizeof(int32_t) * n_tgt));
  DevBuf ord;
  CUDA_TRY(c, ord.ensure(sizeof(int32_t) * n_tgt));
  CUDA_TRY(c, cudaMemcpyAsync(dt.p, txy, sizeof(double2) * n_tgt, cudaMemcpyHostToDevice, c->stream));
  k_morton<<<nblk(n_tgt, 256), 256, 0, c->stream>>>(n_tgt, dt.as<double2>(), lox, loy, spx, spy,
                                                     code.as<unsigned>(), idx.as<int32_t>());
  size_t tmpb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmpb, code.as<unsigned>(), code2.as<unsigned>(), idx.as<int32_t>(),
                                  ord.as<int32_t>(), (int)n_tgt, 0, 32, c->stream);
  CUDA_TRY(c, c->d_tmp.ensure(tmpb));
  cub::DeviceRadixSort::SortPairs(c->d_tmp.p, tmpb, code.as<unsigned>(), code2.as<unsigned>(), idx.as<int32_t>(),
                                  ord.as<int32_t>(), (int)n_tgt, 0, 32, c->stream);
  k_gather_targets_i32<<<nblk(n_tgt, 256), 256, 0, c->stream>>>(n_tgt, ord.as<int32_t>(), dt.as<double2>(),
                                                                 dts.as<double2>());
  // near-field lists of the Morton-ordered targets give |N(t)| and S(t)
  CUDA_TRY(c, c->d_err.ensure(2 * sizeof(int)));
  CUDA_TRY(c, cudaMemsetAsync(c->d_err.p, 0, 2 * sizeof(int), c->stream));
  int64_t n_ids = 0;
  if (int rc = build_lists(c, n_tgt, dts.as<double2>(), &n_ids)) return rc;
  int64_t cf, cn, cs;
  shard_cost_model(c, cf, cn, cs);
  DevBuf cost, P;
  CUDA_TRY(c, cost.ensure(sizeof(int64_t) * (n_tgt + 1)));
  CUDA_TRY(c, P.ensure(sizeof(int64_t) * (n_tgt + 1)));
  k_shard_cost<<<nblk(n_tgt, 256), 256, 0, c->stream>>>(n_tgt, c->d_cnt.as<int64_t>(), c->d_self.as<int32_t>(), cf,
                                                         cn, cs, cost.as<int64_t>());
  CUDA_TRY(c, cudaMemsetAsync(cost.as<int64_t>() + n_tgt, 0, sizeof(int64_t), c->stream));
  tmpb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmpb, cost.as<int64_t>(), P.as<int64_t>(), n_tgt + 1, c->stream);
  CUDA_TRY(c, c->d_tmp.ensure(tmpb));
  cub::DeviceScan::ExclusiveSum(c->d_tmp.p, tmpb, cost.as<int64_t>(), P.as<int64_t>(), n_tgt + 1, c->stream);
  DevBuf db;
  CUDA_TRY(c, db.ensure(sizeof(int64_t) * (world + 1)));
  k_shard_search<<<nblk(world + 1, 128), 128, 0, c->stream>>>(n_tgt, P.as<int64_t>(), world, db.as<int64_t>());
  CUDA_TRY(c, cudaGetLastError());
  CUDA_TRY(c, cudaMemcpyAsync(bounds_out, db.p, sizeof(int64_t) * (world + 1), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(order_out, ord.p, sizeof(int32_t) * n_tgt, cudaMemcpyDeviceToHost, c->stream));
  int herr[2] = {0, 0};
  CUDA_TRY(c, cudaMemcpyAsync(herr, c->d_err.p, sizeof(herr), cudaMemcpyDeviceToHost, c->stream));
  std::vector<int64_t> Ph;
  if (shard_cost_out) {
    Ph.resize(world + 1);
    // P at the bounds: one small gather per bound (world + 1 entries)
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    for (int r = 0; r <= world; ++r)
      CUDA_TRY(c, cudaMemcpyAsync(&Ph[r], P.as<int64_t>() + bounds_out[r], sizeof(int64_t), cudaMemcpyDeviceToHost,
                                  c->stream));
  }
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (herr[1]) return set_err(c, 2, "shard_plan: non-finite target coordinate");
  if (shard_cost_out)
    for (int r = 0; r < world; ++r) shard_cost_out[r] = Ph[r + 1] - Ph[r];
  return 0;
}

int vp_nccl_unique_id(unsigned char* id_out) {
  if (!id_out) return 1;
  NcclApi& A = nccl();
  if (!A.ok) return 3;
  ncclUniqueId id;
  if (A.GetUniqueId(&id) != ncclSuccess) return 3;
  static_assert(sizeof(ncclUniqueId) == VP_NCCL_ID_BYTES, "ncclUniqueId size");
  std::memcpy(id_out, &id, sizeof(id));
  return 0;
}

int vp_comm_init(vp_ctx* c, int world, int rank, const unsigned char* id) {
  if (!c) return 1;
  if (world <= 0 || rank < 0 || rank >= world || !id)
    return set_err(c, 1, "comm_init: need 0 <= rank < world and the rank-0 unique id");
  NcclApi& A = nccl();
  if (!A.ok) return set_err(c, 3, "comm_init: " + A.why);
  CUDA_TRY(c, cudaSetDevice(c->device));
  vp_comm_release(c);
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclComm_t comm = nullptr;
  NCCL_TRY(c, A.CommInitRank(&comm, world, uid, rank));
  c->comm = comm;
  c->comm_world = world;
  c->comm_rank = rank;
  return 0;
}

int vp_gather(vp_ctx* c, const int64_t* bounds, const double* d_u_local, double* d_u_all, void* stream) {
  if (!c) return 1;
  if (!c->comm) return set_err(c, 1, "gather: vp_comm_init must precede vp_gather");
  if (!bounds || !d_u_all) return set_err(c, 1, "gather: need the shard bounds and the output");
  const int W = c->comm_world;
  for (int r = 0; r < W; ++r)
    if (bounds[r] > bounds[r + 1] || bounds[0] != 0) return set_err(c, 1, "gather: bounds must be non-decreasing from 0");
  NcclApi& A = nccl();
  CUDA_TRY(c, cudaSetDevice(c->device));
  cudaStream_t s = stream ? (cudaStream_t)stream : c->stream;
  // one broadcast per shard, rooted at its owner, straight into place: shards
  // may differ in length (cost-balanced plan), so there is no padding copy
  NCCL_TRY(c, A.GroupStart());
  for (int r = 0; r < W; ++r) {
    const size_t cnt = (size_t)(bounds[r + 1] - bounds[r]);
    if (!cnt) continue;
    const void* src = r == c->comm_rank ? (const void*)d_u_local : (const void*)(d_u_all + bounds[r]);
    ncclResult_t e = A.Broadcast(src, d_u_all + bounds[r], cnt, ncclFloat64, r, (ncclComm_t)c->comm, s);
    if (e != ncclSuccess) {
      A.GroupEnd();
      return set_err(c, 3, std::string("nccl: ") + A.GetErrorString(e) + " in gather broadcast");
    }
  }
  NCCL_TRY(c, A.GroupEnd());
  return 0;
}

int vp_allreduce_stats(vp_ctx* c, vp_stats* st) {
  if (!c || !st) return 1;
  if (!c->comm) return set_err(c, 1, "allreduce_stats: vp_comm_init must precede it");
  NcclApi& A = nccl();
  CUDA_TRY(c, cudaSetDevice(c->device));
  // counters summed, max_depth and device times maxed over ranks
  int64_t cnt[10] = {st->n_targets, st->n_outside, st->n_near_pairs, st->n_self, st->n_leaves,
                     st->n_panels, st->n_rho_le1, st->n_degenerate, st->fmm_outside, (int64_t)st->gpu_launches};
  double mx[10] = {st->t_list_ms, st->t_far_ms, st->t_near_ms, st->t_self_ms, st->t_total_ms,
                   st->t_sources_ms, st->t_far_kernel_ms, st->t_pair_ms, (double)st->max_depth, 0.0};
  DevBuf b;
  CUDA_TRY(c, b.ensure(sizeof(int64_t) * 10 + sizeof(double) * 10));
  CUDA_TRY(c, cudaMemcpyAsync(b.p, cnt, sizeof(cnt), cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync((char*)b.p + sizeof(cnt), mx, sizeof(mx), cudaMemcpyHostToDevice, c->stream));
  NCCL_TRY(c, A.GroupStart());
  NCCL_TRY(c, A.AllReduce(b.p, b.p, 10, ncclInt64, ncclSum, (ncclComm_t)c->comm, c->stream));
  NCCL_TRY(c, A.AllReduce((char*)b.p + sizeof(cnt), (char*)b.p + sizeof(cnt), 10, ncclFloat64, ncclMax,
                          (ncclComm_t)c->comm, c->stream));
  NCCL_TRY(c, A.GroupEnd());
  CUDA_TRY(c, cudaMemcpyAsync(cnt, b.p, sizeof(cnt), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(mx, (char*)b.p + sizeof(cnt), sizeof(mx), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  st->n_targets = cnt[0]; st->n_outside = cnt[1]; st->n_near_pairs = cnt[2]; st->n_self = cnt[3];
  st->n_leaves = cnt[4]; st->n_panels = cnt[5]; st->n_rho_le1 = cnt[6]; st->n_degenerate = cnt[7];
  st->fmm_outside = cnt[8]; st->gpu_launches = (int32_t)cnt[9];
  st->t_list_ms = mx[0]; st->t_far_ms = mx[1]; st->t_near_ms = mx[2]; st->t_self_ms = mx[3];
  st->t_total_ms = mx[4]; st->t_sources_ms = mx[5]; st->t_far_kernel_ms = mx[6]; st->t_pair_ms = mx[7];
  st->max_depth = (int32_t)mx[8];
  return 0;
}

}  // extern "C"
