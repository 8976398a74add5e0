// z-slab partitioned STMG solve (north_star: "the spatial mesh is
// partitioned across 1, 2, 4 and 8 GPUs ... NCCL only for ghost-layer halo
// exchange and dot-product allreduce").
//
// The finest lattice is cut into n_parts contiguous ranges of cell layers
// along z (the slowest axis, so a slab is one contiguous range of every field
// block). Part i holds its slab's lattice INCLUDING the interface planes it
// shares with parts i-1 / i+1; after every cell loop (operator, smoother,
// restriction) both copies of an interface plane hold partial sums, and one
// interface sum (in-process kernel, or ncclSend/ncclRecv of the packed planes
// between neighbouring ranks) makes them the assembled value. Entries of an
// interface plane are owned by the lower part (dot products, residual RHS,
// restriction input). Levels stay partitioned while every part keeps an even
// number >= 2 of cell layers; below that the rest of the hierarchy is
// replicated on every rank (restriction into a full-length coarse vector +
// allreduce, the same SpaceTimeMultigrid tail everywhere, prolongation from
// the part's slab view of it).
//
// One process may hold several consecutive parts (in-process interface sums):
// with one process and n_parts > 1 this runs the exact partitioned algorithm
// on one GPU, which is how the parity tests check it.
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "stmg.hpp"

namespace stmgb {

// NCCL communicator, loaded at run time (dlopen "libnccl.so.2"), so the
// library carries no link-time NCCL dependency and shares the copy torch has
// already loaded.
// The data-path exchange of the partition: the interface-plane sum with the
// neighbouring ranks and the dot-product / coarse-vector allreduce.
class Comm {
 public:
  Comm(int world, int rank) : world_(world), rank_(rank) {}
  virtual ~Comm() = default;
  Comm(const Comm&) = delete;
  Comm& operator=(const Comm&) = delete;
  int world() const { return world_; }
  int rank() const { return rank_; }
  // in-place sum over ranks (device buffer, stream-ordered)
  virtual void allreduce_sum(double* d, size_t n, cudaStream_t s) const = 0;
  // grouped exchange with the neighbouring ranks: send lo_send to rank-1 and
  // receive its data into lo_recv (if lo), same with rank+1 (if hi)
  virtual void exchange(const double* lo_send, double* lo_recv, const double* hi_send, double* hi_recv, size_t n,
                        bool lo, bool hi, cudaStream_t s) const = 0;

 protected:
  int world_, rank_;
};

// NCCL over NVLink / NVSwitch (libnccl.so.2 loaded at run time)
class NcclComm : public Comm {
 public:
  static std::string unique_id();  // 128 bytes, on the root rank
  NcclComm(int world, int rank, const std::string& id);
  ~NcclComm() override;
  void allreduce_sum(double* d, size_t n, cudaStream_t s) const override;
  void exchange(const double* lo_send, double* lo_recv, const double* hi_send, double* hi_recv, size_t n, bool lo,
                bool hi, cudaStream_t s) const override;

 private:
  void* comm_ = nullptr;
};

// Host-staged transport: device buffers are copied to page-locked host
// memory and handed to caller-supplied callbacks (e.g. torch.distributed over
// gloo), then copied back. For ranks without a device-to-device path, and for
// exercising the per-rank code path with several processes on one GPU.
struct HostTransport {
  void* ctx = nullptr;
  // in-place sum over ranks of n host doubles; 0 on success
  int (*allreduce_sum)(void* ctx, double* h, long long n) = nullptr;
  // send n doubles to rank `peer` and receive n doubles from it; 0 on success
  int (*sendrecv)(void* ctx, int peer, const double* h_send, double* h_recv, long long n) = nullptr;
};
class HostComm : public Comm {
 public:
  HostComm(int world, int rank, const HostTransport& t);
  ~HostComm() override;
  void allreduce_sum(double* d, size_t n, cudaStream_t s) const override;
  void exchange(const double* lo_send, double* lo_recv, const double* hi_send, double* hi_recv, size_t n, bool lo,
                bool hi, cudaStream_t s) const override;

 private:
  double* host(size_t n) const;
  HostTransport t_;
  mutable double* buf_ = nullptr;
  mutable size_t cap_ = 0;
};

struct SlabPlan {
  int n_parts = 1;
  int dist_levels = 0;           // plan levels [0, dist_levels) are partitioned
  std::vector<Index> cz0, nz;    // per part: first cell layer and layer count on the finest mesh level
};
SlabPlan make_slab_plan(const std::vector<LevelSpec>& plan, Index cells_z_finest, int finest_mesh_level,
                        int n_parts);

class SlabMultigrid {
 public:
  // parts [first_part, first_part + local_parts) of n_parts live in this
  // process; comm (may be null for one process) connects the processes, one
  // rank per block of local_parts consecutive parts
  SlabMultigrid(Equation equation, TimeScheme scheme, const MeshHierarchy& global, const Coefficient& rho,
                const std::vector<LevelSpec>& plan, const MultigridOptions& options, int n_parts, int first_part,
                int local_parts, const Comm* comm);
  ~SlabMultigrid();

  int n_parts() const { return plan_.n_parts; }
  int local_parts() const { return static_cast<int>(parts_.size()); }
  int dist_levels() const { return plan_.dist_levels; }
  int n_levels() const { return n_levels_; }
  Index local_dofs(int l = 0) const { return levels_[static_cast<size_t>(l)].n_local; }
  // offset / length / first lattice plane of local part i inside the level-0
  // distributed vector
  Index part_offset(int i) const { return levels_[0].off[static_cast<size_t>(i)]; }
  Index part_dofs(int i) const;
  Index part_plane0(int i) const;
  double omega_at(int l) const;
  void set_omega(int l, double w);

  // y = S u on the distributed finest level (interface-summed)
  void apply(const double* u, double* y, cudaStream_t s) const;
  // z = one V-cycle applied to r (overwrite)
  void vcycle(const double* r, double* z, cudaStream_t s) const;
  // the level-0 smoother: z += W sum R^T B^-1 R r over all parts (interface-summed)
  void asm_add_correction(const double* r, double* z, cudaStream_t s) const;
  // right-preconditioned GMRES on the distributed system
  GmresResult solve(const double* b, double* x, const GmresOptions& o, cudaStream_t s) const;
  // owned-entry inner product (summed over ranks)
  double dot(const double* a, const double* b, cudaStream_t s) const;
  // slices of a full-length finest-level vector <-> the local parts (device)
  void scatter(const double* full, double* local, cudaStream_t s) const;
  void gather(const double* local, double* full, cudaStream_t s) const;  // owned planes of the local parts
  size_t device_bytes() const;

 private:
  struct PartLevel {
    std::unique_ptr<SpaceTimeOperator> op;
    std::unique_ptr<ASMSmoother> sm;
    std::unique_ptr<SpaceTimeOperator> cop;  // next level's slab (transfer partner)
    std::unique_ptr<Transfer> down;
  };
  struct Part {
    int index = 0;
    MeshHierarchy mesh;
    std::vector<PartLevel> lv;
  };
  struct Level {
    LevelSpec spec;
    TemporalWeights weights;
    double omega = 1.0;
    int F = 1;
    std::vector<Index> off;   // per local part: offset in the distributed vector
    Index n_local = 0;
    mutable DeviceBuffer r, rc, ec;  // work vectors (rc/ec: next level, distributed)
    DotSegments seg{};
  };
  void iface_sum(int l, double* v, cudaStream_t s) const;
  void zero_nonowned(int l, double* v, cudaStream_t s) const;
  void residual(int l, const double* f, const double* u, double* r, cudaStream_t s) const;
  void smooth(int l, const double* f, double* u, cudaStream_t s) const;
  void v_cycle(int l, const double* f, double* u, cudaStream_t s) const;
  void op_apply(int l, const double* u, double* y, cudaStream_t s) const;
  void asm_apply(int l, const double* r, double* z, double scale, cudaStream_t s) const;
  double level_dot(int l, const double* a, const double* b, cudaStream_t s) const;
  double estimate_relaxation(int l, std::uint64_t seed);
  void allreduce(double* d, size_t n, cudaStream_t s) const;

  SlabPlan plan_;
  MultigridOptions options_;
  std::vector<Part> parts_;
  std::vector<Level> levels_;  // the partitioned levels
  int n_levels_ = 0;
  const Comm* comm_ = nullptr;
  std::unique_ptr<SpaceTimeMultigrid> tail_;
  const MeshHierarchy* global_ = nullptr;
  Index full_coarse_n_ = 0, full_coarse_nspace_ = 0;
  mutable DeviceBuffer full_rc_, full_ec_;
  mutable DeviceBuffer xbuf_;  // exchange buffers: lo send, lo recv, hi send, hi recv
  mutable DeviceBuffer dot_ptrs_, dot_scratch_, dot_out_;
  mutable GmresWorkspace ws_;
  DotPolicy dots_;
};

}  // namespace stmgb
