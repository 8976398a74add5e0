// z-slab partitioned STMG solve -- see slab_mg.hpp for the scheme.
#include "slab_mg.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <stdexcept>

namespace stmgb {

// ------------------------------------------------------------------ NCCL
namespace {
struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
    a.send = reinterpret_cast<decltype(a.send)>(dlsym(h, "ncclSend"));
    a.recv = reinterpret_cast<decltype(a.recv)>(dlsym(h, "ncclRecv"));
    a.group_start = reinterpret_cast<decltype(a.group_start)>(dlsym(h, "ncclGroupStart"));
    a.group_end = reinterpret_cast<decltype(a.group_end)>(dlsym(h, "ncclGroupEnd"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
    return a;
  }();
  if (!api.get_unique_id || !api.comm_init_rank || !api.send || !api.recv || !api.all_reduce)
    throw std::runtime_error("NCCL: libnccl.so.2 not found or incomplete");
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw std::runtime_error(std::string("NCCL ") + what + ": " +
                             (nccl().error_string ? nccl().error_string(r) : "error"));
}
}  // namespace

std::string NcclComm::unique_id() {
  ncclUniqueId id;
  nccl_check(nccl().get_unique_id(&id), "get_unique_id");
  return std::string(id.internal, sizeof(id.internal));
}

NcclComm::NcclComm(int world, int rank, const std::string& id) : Comm(world, rank) {
  if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("NcclComm: bad world/rank");
  if (id.size() != sizeof(ncclUniqueId::internal)) throw std::invalid_argument("NcclComm: unique id must be 128 bytes");
  ncclUniqueId uid;
  std::memcpy(uid.internal, id.data(), sizeof(uid.internal));
  ncclComm_t c = nullptr;
  nccl_check(nccl().comm_init_rank(&c, world, uid, rank), "comm_init_rank");
  comm_ = c;
}

NcclComm::~NcclComm() {
  if (comm_ && nccl().comm_destroy) nccl().comm_destroy(static_cast<ncclComm_t>(comm_));
}

void NcclComm::allreduce_sum(double* d, size_t n, cudaStream_t s) const {
  if (world_ == 1 || n == 0) return;
  nccl_check(nccl().all_reduce(d, d, n, ncclDouble, ncclSum, static_cast<ncclComm_t>(comm_), s), "all_reduce");
}

void NcclComm::exchange(const double* lo_send, double* lo_recv, const double* hi_send, double* hi_recv, size_t n,
                        bool lo, bool hi, cudaStream_t s) const {
  if (world_ == 1 || (!lo && !hi)) return;
  const auto c = static_cast<ncclComm_t>(comm_);
  nccl_check(nccl().group_start(), "group_start");
  if (lo) {
    nccl_check(nccl().send(lo_send, n, ncclDouble, rank_ - 1, c, s), "send");
    nccl_check(nccl().recv(lo_recv, n, ncclDouble, rank_ - 1, c, s), "recv");
  }
  if (hi) {
    nccl_check(nccl().send(hi_send, n, ncclDouble, rank_ + 1, c, s), "send");
    nccl_check(nccl().recv(hi_recv, n, ncclDouble, rank_ + 1, c, s), "recv");
  }
  nccl_check(nccl().group_end(), "group_end");
}

// ------------------------------------------------------------ host staged
HostComm::HostComm(int world, int rank, const HostTransport& t) : Comm(world, rank), t_(t) {
  if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("HostComm: bad world/rank");
  if (!t.allreduce_sum || !t.sendrecv) throw std::invalid_argument("HostComm: transport callbacks missing");
}
HostComm::~HostComm() {
  if (buf_) cudaFreeHost(buf_);
}
double* HostComm::host(size_t n) const {
  if (n > cap_) {
    if (buf_) cudaFreeHost(buf_);
    buf_ = nullptr;
    cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&buf_), sizeof(double) * n, cudaHostAllocDefault),
               "HostComm staging");
    cap_ = n;
  }
  return buf_;
}
void HostComm::allreduce_sum(double* d, size_t n, cudaStream_t s) const {
  if (world_ == 1 || n == 0) return;
  double* h = host(n);
  cuda_check(cudaMemcpyAsync(h, d, sizeof(double) * n, cudaMemcpyDeviceToHost, s), "HostComm D2H");
  cuda_check(cudaStreamSynchronize(s), "HostComm sync");
  if (t_.allreduce_sum(t_.ctx, h, static_cast<long long>(n)) != 0)
    throw std::runtime_error("HostComm: allreduce callback failed");
  cuda_check(cudaMemcpyAsync(d, h, sizeof(double) * n, cudaMemcpyHostToDevice, s), "HostComm H2D");
  cuda_check(cudaStreamSynchronize(s), "HostComm sync");
}
void HostComm::exchange(const double* lo_send, double* lo_recv, const double* hi_send, double* hi_recv, size_t n,
                        bool lo, bool hi, cudaStream_t s) const {
  if (world_ == 1 || (!lo && !hi)) return;
  double* h = host(4 * n);
  double *hls = h, *hlr = h + n, *hhs = h + 2 * n, *hhr = h + 3 * n;
  if (lo) cuda_check(cudaMemcpyAsync(hls, lo_send, sizeof(double) * n, cudaMemcpyDeviceToHost, s), "HostComm D2H");
  if (hi) cuda_check(cudaMemcpyAsync(hhs, hi_send, sizeof(double) * n, cudaMemcpyDeviceToHost, s), "HostComm D2H");
  cuda_check(cudaStreamSynchronize(s), "HostComm sync");
  // the lower neighbour first: rank r pairs its lo exchange with rank r-1's hi
  // exchange, so the chain resolves from rank 0 upwards
  if (lo && t_.sendrecv(t_.ctx, rank_ - 1, hls, hlr, static_cast<long long>(n)) != 0)
    throw std::runtime_error("HostComm: sendrecv callback failed");
  if (hi && t_.sendrecv(t_.ctx, rank_ + 1, hhs, hhr, static_cast<long long>(n)) != 0)
    throw std::runtime_error("HostComm: sendrecv callback failed");
  if (lo) cuda_check(cudaMemcpyAsync(lo_recv, hlr, sizeof(double) * n, cudaMemcpyHostToDevice, s), "HostComm H2D");
  if (hi) cuda_check(cudaMemcpyAsync(hi_recv, hhr, sizeof(double) * n, cudaMemcpyHostToDevice, s), "HostComm H2D");
  cuda_check(cudaStreamSynchronize(s), "HostComm sync");
}

// ------------------------------------------------------------------ plan
SlabPlan make_slab_plan(const std::vector<LevelSpec>& plan, Index cells_z, int finest_mesh_level, int n_parts) {
  if (n_parts < 1) throw std::invalid_argument("slab plan: n_parts must be >= 1");
  if (plan.size() < 2) throw std::invalid_argument("slab plan: the level plan needs at least two levels");
  if (cells_z % n_parts != 0)
    throw std::invalid_argument("slab plan: the finest cell layers must divide evenly among the parts");
  SlabPlan sp;
  sp.n_parts = n_parts;
  const Index nz = cells_z / n_parts;
  for (int i = 0; i < n_parts; ++i) {
    sp.cz0.push_back(i * nz);
    sp.nz.push_back(nz);
  }
  int D = 0;
  for (size_t l = 0; l + 1 < plan.size(); ++l) {
    const int shift = finest_mesh_level - plan[l].mesh_level;
    if (shift < 0 || shift >= 62 || nz % (Index{1} << shift) != 0) break;
    const Index nzl = nz >> shift;
    if (nzl < 1) break;
    if (plan[l + 1].from_finer == Coarsening::SpaceH && nzl % 2 != 0) break;
    D = static_cast<int>(l) + 1;
  }
  if (D == 0) throw std::invalid_argument("slab plan: too few cell layers per part to partition the finest level");
  sp.dist_levels = D;
  return sp;
}

// ------------------------------------------------------------------ slabs
namespace {
MeshLevel slab_level(const MeshLevel& g, Index cz0, Index nz) {
  if (g.dim != 3) throw std::invalid_argument("SlabMultigrid: the z-slab partition needs dim == 3");
  if (cz0 < 0 || nz < 1 || cz0 + nz > g.cells[2]) throw std::invalid_argument("SlabMultigrid: slab out of range");
  MeshLevel s = g;
  const double hz = (g.hi[2] - g.lo[2]) / static_cast<double>(g.cells[2]);
  s.cells[2] = nz;
  s.lo[2] = g.lo[2] + static_cast<double>(cz0) * hz;
  s.hi[2] = g.lo[2] + static_cast<double>(cz0 + nz) * hz;
  s.cz0 = cz0;
  s.zbc = (cz0 == 0 ? 1 : 0) | (cz0 + nz == g.cells[2] ? 2 : 0);
  if (!g.vertices.empty()) {
    const auto nv = g.n_verts_axis();
    const size_t plane = static_cast<size_t>(3 * nv[0] * nv[1]);
    s.vertices.assign(g.vertices.begin() + static_cast<std::ptrdiff_t>(plane * cz0),
                      g.vertices.begin() + static_cast<std::ptrdiff_t>(plane * (cz0 + nz + 1)));
  }
  return s;
}

// the slab [cz0, cz0 + nz) (finest level L) on every mesh level where it is a
// whole number of layers; other levels are copies of the global ones (unused)
MeshHierarchy slab_hierarchy(const MeshHierarchy& g, int L, Index cz0, Index nz, bool halo) {
  MeshHierarchy h;
  h.global_cells0 = g.levels.front().cells;
  for (int m = 0; m < g.n_levels(); ++m) {
    const MeshLevel& gm = g.levels[static_cast<size_t>(m)];
    const int shift = L - m;
    if (m > L || shift >= 62 || cz0 % (Index{1} << shift) != 0 || nz % (Index{1} << shift) != 0 ||
        (nz >> shift) < 1) {
      h.levels.push_back(gm);
      continue;
    }
    Index c0 = cz0 >> shift, n = nz >> shift;
    if (halo) {
      const bool lo = c0 > 0, hi = c0 + n < gm.cells[2];
      c0 -= lo ? 1 : 0;
      n += (lo ? 1 : 0) + (hi ? 1 : 0);
    }
    h.levels.push_back(slab_level(gm, c0, n));
  }
  return h;
}
}  // namespace

SlabMultigrid::SlabMultigrid(Equation equation, TimeScheme scheme, const MeshHierarchy& global, const Coefficient& rho,
                             const std::vector<LevelSpec>& plan, const MultigridOptions& options, int n_parts,
                             int first_part, int local_parts, const Comm* comm)
    : options_(options), comm_(comm), global_(&global) {
  if (plan.empty()) throw std::invalid_argument("SlabMultigrid: empty plan");
  const int L = plan[0].mesh_level;
  if (L < 0 || L >= global.n_levels()) throw std::invalid_argument("SlabMultigrid: bad finest mesh level");
  const MeshLevel& gf = global.levels[static_cast<size_t>(L)];
  if (gf.dim != 3) throw std::invalid_argument("SlabMultigrid: the z-slab partition needs dim == 3");
  {
    const int nt = scheme == TimeScheme::DG ? plan[0].k + 1 : plan[0].k;
    if (plan[0].n_steps * nt > kMaxF)
      throw std::invalid_argument("SlabMultigrid: the partitioned solve needs n_steps * n_t <= 8");
  }
  plan_ = make_slab_plan(plan, gf.cells[2], L, n_parts);
  if (first_part < 0 || local_parts < 1 || first_part + local_parts > n_parts)
    throw std::invalid_argument("SlabMultigrid: bad local part range");
  if (comm_ && comm_->world() > 1 && local_parts * comm_->world() != n_parts)
    throw std::invalid_argument("SlabMultigrid: every rank must hold the same number of parts");
  const int D = plan_.dist_levels;
  n_levels_ = static_cast<int>(plan.size());
  levels_.resize(static_cast<size_t>(D));
  for (int l = 0; l < D; ++l) {
    Level& lv = levels_[static_cast<size_t>(l)];
    lv.spec = plan[static_cast<size_t>(l)];
    lv.weights = scheme == TimeScheme::DG ? dg_weights(lv.spec.k) : cgp_weights(lv.spec.k);
    lv.F = lv.spec.n_steps * lv.weights.n_t;
  }
  // per part: slab operators, smoothers (probed on a one-layer halo across
  // each interface), transfers; the last partitioned level transfers into a
  // slab view of the replicated next level
  for (int i = 0; i < local_parts; ++i) {
    Part part;
    part.index = first_part + i;
    const Index cz0 = plan_.cz0[static_cast<size_t>(part.index)], nz = plan_.nz[static_cast<size_t>(part.index)];
    part.mesh = slab_hierarchy(global, L, cz0, nz, false);
    parts_.push_back(std::move(part));
  }
  for (Part& part : parts_) {
    const Index cz0 = plan_.cz0[static_cast<size_t>(part.index)], nz = plan_.nz[static_cast<size_t>(part.index)];
    const bool interfaces = n_parts > 1;
    MeshHierarchy halo;
    if (interfaces) halo = slab_hierarchy(global, L, cz0, nz, true);
    part.lv.resize(static_cast<size_t>(D));
    for (int l = 0; l < D; ++l) {
      const Level& lv = levels_[static_cast<size_t>(l)];
      PartLevel& pl = part.lv[static_cast<size_t>(l)];
      pl.op = std::make_unique<SpaceTimeOperator>(equation, lv.weights, lv.spec.tau, lv.spec.n_steps, part.mesh,
                                                  lv.spec.mesh_level, lv.spec.p, rho);
      if (interfaces) {
        const SpaceTimeOperator hop(equation, lv.weights, lv.spec.tau, lv.spec.n_steps, halo, lv.spec.mesh_level,
                                    lv.spec.p, rho);
        const int below = static_cast<int>(pl.op->desc().cz0 - hop.desc().cz0);
        pl.sm = std::make_unique<ASMSmoother>(*pl.op, &hop, below);
      } else {
        pl.sm = std::make_unique<ASMSmoother>(*pl.op);
      }
    }
    for (int l = 0; l < D; ++l) {
      PartLevel& pl = part.lv[static_cast<size_t>(l)];
      if (l + 1 < D) {
        pl.down = std::make_unique<Transfer>(*pl.op, *part.lv[static_cast<size_t>(l) + 1].op);
      } else {
        const LevelSpec& cs = plan[static_cast<size_t>(D)];
        const TemporalWeights cw = scheme == TimeScheme::DG ? dg_weights(cs.k) : cgp_weights(cs.k);
        pl.cop = std::make_unique<SpaceTimeOperator>(equation, cw, cs.tau, cs.n_steps, part.mesh, cs.mesh_level, cs.p,
                                                     rho);
        pl.down = std::make_unique<Transfer>(*pl.op, *pl.cop);
      }
    }
  }
  // level vectors and owned segments
  for (int l = 0; l < D; ++l) {
    Level& lv = levels_[static_cast<size_t>(l)];
    Index off = 0;
    lv.seg.n = 0;
    for (const Part& part : parts_) {
      const DevLevel& d = part.lv[static_cast<size_t>(l)].op->desc();
      lv.off.push_back(off);
      const Index dxy = d.dofs[0] * d.dofs[1];
      for (int f = 0; f < d.F; ++f) {
        if (lv.seg.n >= kMaxSeg) throw std::invalid_argument("SlabMultigrid: too many local parts x fields");
        lv.seg.begin[lv.seg.n] = off + f * d.n_space + ((d.zbc & 1) ? 0 : dxy);
        lv.seg.end[lv.seg.n] = off + (f + 1) * d.n_space;
        ++lv.seg.n;
      }
      off += d.n_dofs;
    }
    lv.n_local = off;
    lv.r.allocate(sizeof(double) * off);
  }
  for (int l = 0; l + 1 < D; ++l) {
    Level& lv = levels_[static_cast<size_t>(l)];
    lv.rc.allocate(sizeof(double) * levels_[static_cast<size_t>(l) + 1].n_local);
    lv.ec.allocate(sizeof(double) * levels_[static_cast<size_t>(l) + 1].n_local);
  }
  size_t xmax = 1;
  for (int l = 0; l < D; ++l) {
    const DevLevel& d = parts_.front().lv[static_cast<size_t>(l)].op->desc();
    xmax = std::max<size_t>(xmax, static_cast<size_t>(d.F * d.dofs[0] * d.dofs[1]));
  }
  xbuf_.allocate(sizeof(double) * 4 * xmax);
  dot_ptrs_.allocate(sizeof(double*));
  dot_scratch_.allocate(sizeof(double) * kDotBlocks * 2);
  dot_out_.allocate(sizeof(double) * 2);
  // replicated tail (levels D..), seeds as if it were part of the full plan
  MultigridOptions to = options;
  to.seed = options.seed + static_cast<std::uint64_t>(D);
  tail_ = std::make_unique<SpaceTimeMultigrid>(equation, scheme, global, rho,
                                              std::vector<LevelSpec>(plan.begin() + D, plan.end()), to);
  full_coarse_n_ = tail_->fine_operator().n_dofs();
  full_coarse_nspace_ = tail_->fine_operator().n_space();
  full_rc_.allocate(sizeof(double) * full_coarse_n_);
  full_ec_.allocate(sizeof(double) * full_coarse_n_);
  // relaxation factors of the partitioned levels: the reference's Arnoldi
  // estimate (multigrid.cpp:127-172) with the same global start vector
  for (int l = 0; l < D; ++l)
    levels_[static_cast<size_t>(l)].omega = estimate_relaxation(l, options.seed + static_cast<std::uint64_t>(l));
  dots_.seg = levels_[0].seg;
  if (comm_ && comm_->world() > 1) {
    const Comm* c = comm_;
    dots_.allreduce = [c](double* d, int k, cudaStream_t s) { c->allreduce_sum(d, static_cast<size_t>(k), s); };
  }
}

SlabMultigrid::~SlabMultigrid() = default;

Index SlabMultigrid::part_dofs(int i) const { return parts_[static_cast<size_t>(i)].lv[0].op->n_dofs(); }
Index SlabMultigrid::part_plane0(int i) const {
  const DevLevel& d = parts_[static_cast<size_t>(i)].lv[0].op->desc();
  return d.cz0 * d.p;
}
double SlabMultigrid::omega_at(int l) const {
  if (l < 0 || l >= n_levels_) throw std::invalid_argument("SlabMultigrid: bad level");
  if (l < plan_.dist_levels) return levels_[static_cast<size_t>(l)].omega;
  return tail_->omega_at(l - plan_.dist_levels);
}
void SlabMultigrid::set_omega(int l, double w) {
  if (l < 0 || l >= n_levels_) throw std::invalid_argument("SlabMultigrid: bad level");
  if (l < plan_.dist_levels)
    levels_[static_cast<size_t>(l)].omega = w;
  else
    tail_->set_omega(l - plan_.dist_levels, w);
}

void SlabMultigrid::allreduce(double* d, size_t n, cudaStream_t s) const {
  if (comm_) comm_->allreduce_sum(d, n, s);
}

void SlabMultigrid::iface_sum(int l, double* v, cudaStream_t s) const {
  const Level& lv = levels_[static_cast<size_t>(l)];
  for (size_t i = 0; i + 1 < parts_.size(); ++i) {
    const DevLevel& a = parts_[i].lv[static_cast<size_t>(l)].op->desc();
    const DevLevel& b = parts_[i + 1].lv[static_cast<size_t>(l)].op->desc();
    plane_pair_sum(v + lv.off[i], a.dofs[2] - 1, v + lv.off[i + 1], 0, a.F, a.n_space, b.n_space,
                   a.dofs[0] * a.dofs[1], s);
  }
  if (!comm_ || comm_->world() == 1) return;
  const bool lo = parts_.front().index > 0, hi = parts_.back().index < plan_.n_parts - 1;
  const DevLevel& a = parts_.front().lv[static_cast<size_t>(l)].op->desc();
  const DevLevel& b = parts_.back().lv[static_cast<size_t>(l)].op->desc();
  const Index len = a.dofs[0] * a.dofs[1];
  const size_t n = static_cast<size_t>(a.F * len);
  double* lo_send = xbuf_.d();
  double* lo_recv = lo_send + n;
  double* hi_send = lo_recv + n;
  double* hi_recv = hi_send + n;
  double* va = v + lv.off.front();
  double* vb = v + lv.off.back();
  if (lo) plane_pack(va, a.F, a.n_space, 0, len, lo_send, s);
  if (hi) plane_pack(vb, b.F, b.n_space, b.dofs[2] - 1, len, hi_send, s);
  comm_->exchange(lo_send, lo_recv, hi_send, hi_recv, n, lo, hi, s);
  if (lo) plane_unpack_add(va, a.F, a.n_space, 0, len, lo_recv, s);
  if (hi) plane_unpack_add(vb, b.F, b.n_space, b.dofs[2] - 1, len, hi_recv, s);
}

void SlabMultigrid::zero_nonowned(int l, double* v, cudaStream_t s) const {
  const Level& lv = levels_[static_cast<size_t>(l)];
  for (size_t i = 0; i < parts_.size(); ++i) {
    const DevLevel& d = parts_[i].lv[static_cast<size_t>(l)].op->desc();
    if (!(d.zbc & 1)) plane_fill(v + lv.off[i], d.F, d.n_space, 0, d.dofs[0] * d.dofs[1], 0.0, s);
  }
}

void SlabMultigrid::op_apply(int l, const double* u, double* y, cudaStream_t s) const {
  const Level& lv = levels_[static_cast<size_t>(l)];
  for (size_t i = 0; i < parts_.size(); ++i) parts_[i].lv[static_cast<size_t>(l)].op->apply(u + lv.off[i], y + lv.off[i], s);
  iface_sum(l, y, s);
}

void SlabMultigrid::asm_apply(int l, const double* r, double* z, double scale, cudaStream_t s) const {
  const Level& lv = levels_[static_cast<size_t>(l)];
  zero_nonowned(l, z, s);
  for (size_t i = 0; i < parts_.size(); ++i)
    parts_[i].lv[static_cast<size_t>(l)].sm->add_correction(r + lv.off[i], z + lv.off[i], s, scale);
  iface_sum(l, z, s);
}

void SlabMultigrid::residual(int l, const double* f, const double* u, double* r, cudaStream_t s) const {
  // each part starts from f on its owned planes (the residual kernel zeroes a
  // non-owned interface plane), subtracts its cells' S u; the interface sum
  // assembles f - S u
  const Level& lv = levels_[static_cast<size_t>(l)];
  for (size_t i = 0; i < parts_.size(); ++i)
    parts_[i].lv[static_cast<size_t>(l)].op->residual(f + lv.off[i], u + lv.off[i], r + lv.off[i], s);
  iface_sum(l, r, s);
}

void SlabMultigrid::smooth(int l, const double* f, double* u, cudaStream_t s) const {
  const Level& lv = levels_[static_cast<size_t>(l)];
  residual(l, f, u, lv.r.d(), s);
  asm_apply(l, lv.r.d(), u, lv.omega, s);
}

void SlabMultigrid::v_cycle(int l, const double* f, double* u, cudaStream_t s) const {
  // u enters as zero (multigrid.cpp:219,231)
  const Level& lv = levels_[static_cast<size_t>(l)];
  const int D = plan_.dist_levels;
  for (int i = 0; i < options_.n_smooth; ++i) {
    if (i == 0)
      asm_apply(l, f, u, lv.omega, s);  // S 0 = 0
    else
      smooth(l, f, u, s);
  }
  residual(l, f, u, lv.r.d(), s);
  if (l + 1 < D) {
    const Level& nx = levels_[static_cast<size_t>(l) + 1];
    for (size_t i = 0; i < parts_.size(); ++i)
      parts_[i].lv[static_cast<size_t>(l)].down->restrict_(lv.r.d() + lv.off[i], lv.rc.d() + nx.off[i], s);
    iface_sum(l + 1, lv.rc.d(), s);
    vec_fill(lv.ec.d(), 0.0, nx.n_local, s);
    v_cycle(l + 1, lv.rc.d(), lv.ec.d(), s);
    for (size_t i = 0; i < parts_.size(); ++i)
      parts_[i].lv[static_cast<size_t>(l)].down->prolong(lv.ec.d() + nx.off[i], u + lv.off[i], s, true);
  } else {
    // into the replicated hierarchy: each part restricts into its slab view of
    // the full coarse vector, the ranks sum, every rank runs the same tail
    vec_fill(full_rc_.d(), 0.0, full_coarse_n_, s);
    auto view = [&](size_t i) {
      const DevLevel& c = parts_[i].lv[static_cast<size_t>(l)].cop->desc();
      return c.cz0 * c.p * c.dofs[0] * c.dofs[1];
    };
    for (size_t i = 0; i < parts_.size(); ++i)
      parts_[i].lv[static_cast<size_t>(l)].down->restrict_(lv.r.d() + lv.off[i], full_rc_.d() + view(i), s, true,
                                                           full_coarse_nspace_);
    allreduce(full_rc_.d(), static_cast<size_t>(full_coarse_n_), s);
    tail_->apply(full_rc_.d(), full_ec_.d(), s);
    for (size_t i = 0; i < parts_.size(); ++i)
      parts_[i].lv[static_cast<size_t>(l)].down->prolong(full_ec_.d() + view(i), u + lv.off[i], s, true,
                                                         full_coarse_nspace_);
  }
  for (int i = 0; i < options_.n_smooth; ++i) smooth(l, f, u, s);
}

void SlabMultigrid::apply(const double* u, double* y, cudaStream_t s) const { op_apply(0, u, y, s); }

void SlabMultigrid::vcycle(const double* r, double* z, cudaStream_t s) const {
  vec_fill(z, 0.0, levels_[0].n_local, s);
  v_cycle(0, r, z, s);
}

void SlabMultigrid::asm_add_correction(const double* r, double* z, cudaStream_t s) const {
  asm_apply(0, r, z, 1.0, s);
}

double SlabMultigrid::level_dot(int l, const double* a, const double* b, cudaStream_t s) const {
  const double* hp[1] = {a};
  cuda_check(cudaMemcpyAsync(dot_ptrs_.raw(), hp, sizeof(hp), cudaMemcpyHostToDevice, s), "dot ptrs");
  vec_multidot_seg(static_cast<const double* const*>(dot_ptrs_.raw()), 1, b, levels_[static_cast<size_t>(l)].seg,
                   dot_out_.d(), dot_scratch_.d(), s);
  allreduce(dot_out_.d(), 1, s);
  double r = 0.0;
  cuda_check(cudaMemcpyAsync(&r, dot_out_.d(), sizeof(double), cudaMemcpyDeviceToHost, s), "dot");
  cuda_check(cudaStreamSynchronize(s), "dot sync");
  return r;
}

double SlabMultigrid::dot(const double* a, const double* b, cudaStream_t s) const { return level_dot(0, a, b, s); }

double SlabMultigrid::estimate_relaxation(int l, std::uint64_t seed) {
  const Level& lv = levels_[static_cast<size_t>(l)];
  cudaStream_t s = nullptr;
  // the global level-l start vector in ST index order (identical on every
  // rank), normalised, then each part takes its slab
  const MeshLevel& gm = global_->levels[static_cast<size_t>(lv.spec.mesh_level)];
  Index gd[3];
  Index gns = 1;
  for (int a = 0; a < 3; ++a) {
    gd[a] = gm.cells[a] * lv.spec.p + 1;
    gns *= gd[a];
  }
  const Index gn = gns * lv.F;
  const int m = static_cast<int>(std::min<Index>(options_.eig_iters, gn));
  Xoshiro256pp rng(seed);
  std::vector<double> hv(static_cast<size_t>(gn));
  double nrm2 = 0.0;
  for (Index i = 0; i < gn; ++i) {
    hv[static_cast<size_t>(i)] = rng.normal();
    nrm2 += hv[static_cast<size_t>(i)] * hv[static_cast<size_t>(i)];
  }
  if (nrm2 == 0.0) return 1.0;
  const double inv = 1.0 / std::sqrt(nrm2);
  for (double& x : hv) x *= inv;
  const Index n = lv.n_local;
  std::vector<DeviceBuffer> V;
  V.emplace_back(sizeof(double) * n);
  const Index dxy = gd[0] * gd[1];
  for (size_t i = 0; i < parts_.size(); ++i) {
    const DevLevel& d = parts_[i].lv[static_cast<size_t>(l)].op->desc();
    const Index plane0 = d.cz0 * d.p;
    for (int f = 0; f < d.F; ++f)
      cuda_check(cudaMemcpy(V[0].d() + lv.off[i] + f * d.n_space, hv.data() + f * gns + plane0 * dxy,
                            sizeof(double) * d.n_space, cudaMemcpyHostToDevice),
                 "arnoldi v0");
  }
  DeviceBuffer w(sizeof(double) * n), z(sizeof(double) * n);
  std::vector<double> H(static_cast<size_t>((m + 1) * m), 0.0);
  int kdim = 0;
  for (int j = 0; j < m; ++j) {
    op_apply(l, V[static_cast<size_t>(j)].d(), w.d(), s);
    vec_fill(z.d(), 0.0, n, s);
    asm_apply(l, w.d(), z.d(), 1.0, s);
    for (int i = 0; i <= j; ++i) {
      const double h = level_dot(l, V[static_cast<size_t>(i)].d(), z.d(), s);
      H[static_cast<size_t>(i * m + j)] = h;
      vec_axpy(z.d(), -h, V[static_cast<size_t>(i)].d(), n, s);
    }
    const double hn = std::sqrt(level_dot(l, z.d(), z.d(), s));
    H[static_cast<size_t>((j + 1) * m + j)] = hn;
    kdim = j + 1;
    if (hn < 1e-13) break;
    V.emplace_back(sizeof(double) * n);
    vec_scale_into(V.back().d(), 1.0 / hn, z.d(), n, s);
  }
  std::vector<double> Hk(static_cast<size_t>(kdim * kdim));
  for (int i = 0; i < kdim; ++i)
    for (int j = 0; j < kdim; ++j) Hk[static_cast<size_t>(i * kdim + j)] = H[static_cast<size_t>(i * m + j)];
  std::vector<std::pair<double, double>> ev;
  try {
    ev = eigenvalues_small(Hk, kdim);
  } catch (const std::exception&) {
    return 1.0;
  }
  double lmax = -1e300, lmin = 1e300;
  for (const auto& e : ev) {
    lmax = std::max(lmax, e.first);
    lmin = std::min(lmin, e.first);
  }
  lmin = std::max(0.0, lmin);
  const double omega = 2.0 / (lmax + lmin);
  if (!std::isfinite(omega) || omega <= 0.0) return 1.0;
  return std::min(omega, 1.0);
}

GmresResult SlabMultigrid::solve(const double* b, double* x, const GmresOptions& o, cudaStream_t s) const {
  return gmres([this](const double* in, double* out, cudaStream_t st) { apply(in, out, st); }, b, x,
               levels_[0].n_local, o,
               [this](const double* in, double* out, cudaStream_t st) { vcycle(in, out, st); }, ws_, s, &dots_);
}

void SlabMultigrid::scatter(const double* full, double* local, cudaStream_t s) const {
  const Level& lv = levels_[0];
  for (size_t i = 0; i < parts_.size(); ++i) {
    const DevLevel& d = parts_[i].lv[0].op->desc();
    const MeshLevel& gm = global_->levels[static_cast<size_t>(lv.spec.mesh_level)];
    const Index gdx = gm.cells[0] * d.p + 1, gdy = gm.cells[1] * d.p + 1, gdz = gm.cells[2] * d.p + 1;
    const Index gns = gdx * gdy * gdz, off = d.cz0 * d.p * gdx * gdy;
    for (int f = 0; f < d.F; ++f)
      cuda_check(cudaMemcpyAsync(local + lv.off[i] + f * d.n_space, full + f * gns + off, sizeof(double) * d.n_space,
                                 cudaMemcpyDeviceToDevice, s),
                 "scatter");
  }
}

void SlabMultigrid::gather(const double* local, double* full, cudaStream_t s) const {
  const Level& lv = levels_[0];
  for (size_t i = 0; i < parts_.size(); ++i) {
    const DevLevel& d = parts_[i].lv[0].op->desc();
    const MeshLevel& gm = global_->levels[static_cast<size_t>(lv.spec.mesh_level)];
    const Index gdx = gm.cells[0] * d.p + 1, gdy = gm.cells[1] * d.p + 1, gdz = gm.cells[2] * d.p + 1;
    const Index gns = gdx * gdy * gdz, dxy = d.dofs[0] * d.dofs[1];
    const Index skip = (d.zbc & 1) ? 0 : dxy;
    const Index off = d.cz0 * d.p * gdx * gdy + skip;
    for (int f = 0; f < d.F; ++f)
      cuda_check(cudaMemcpyAsync(full + f * gns + off, local + lv.off[i] + f * d.n_space + skip,
                                 sizeof(double) * (d.n_space - skip), cudaMemcpyDeviceToDevice, s),
                 "gather");
  }
}

size_t SlabMultigrid::device_bytes() const {
  size_t b = full_rc_.bytes() + full_ec_.bytes() + tail_->device_bytes();
  for (const Level& lv : levels_) b += lv.r.bytes() + lv.rc.bytes() + lv.ec.bytes();
  for (const Part& p : parts_)
    for (const PartLevel& pl : p.lv) b += pl.sm->bytes();
  return b;
}

}  // namespace stmgb
