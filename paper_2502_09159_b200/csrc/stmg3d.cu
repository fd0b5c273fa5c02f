// C ABI (include/stmg_b200.h, "3D") and host orchestration of the 3D
// hp-STMG path (BASELINE C3 / C5): levels with the fused space-time vmult,
// cell-Vanka colour sweeps, the hp space-time hierarchy with h-coarsening in
// space AND time (PAPER.md Eq. DeftPrRe) and p-coarsening in k and r, the
// all-at-once V-cycle with an exact coarse solve by forward substitution in
// time, and FGMRES over a time slab (time-slab partition through
// stmg_comm_ops, as in 2D).
#include "../../include/stmg_b200.h"
#include "krylov.hpp"
#include <chrono>
#include <cstdlib>
#include "runtime.hpp"
#include "st3d.hpp"

#include <cmath>
#include <cstring>
#include <memory>

using namespace stmg_b200;
using namespace stmg_rt;

namespace
{
__global__ void
coarse3_step_kernel(const double *__restrict__ G, const double *__restrict__ H, int n, int mv,
                    const double *__restrict__ b, const double *__restrict__ v, double *__restrict__ x)
{
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= n)
    return;
  const double *g = G + static_cast<long long>(row) * n;
  double s = 0.0;
  for (int j = lane; j < n; j += 32)
    s = fma(g[j], b[j], s);
  if (v)
    {
      const double *h = H + static_cast<long long>(row) * mv;
      for (int j = lane; j < mv; j += 32)
        s = fma(h[j], v[j], s);
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
    s += __shfl_down_sync(0xffffffffu, s, o);
  if (lane == 0)
    x[row] = s;
}
} // namespace

/// dir 0: global[n][map[part][i]] = parts[part][n][i] (the parts of a z-split
/// coarse level into the whole-mesh vector; shared interface entries hold
/// equal values); dir 1: local[n][i] = global[n][map[i]].
__global__ void
coarse_map_kernel(const double *__restrict__ src, const int *__restrict__ map, int n_loc, int n_glob, int nI,
                  double *__restrict__ dst, int dir)
{
  const int i = blockIdx.x * blockDim.x + threadIdx.x, n = blockIdx.y, part = blockIdx.z;
  if (i >= n_loc)
    return;
  const int g = map[static_cast<long long>(part) * n_loc + i];
  if (dir == 0)
    dst[static_cast<long long>(n) * n_glob + g] = src[(static_cast<long long>(part) * nI + n) * n_loc + i];
  else
    dst[static_cast<long long>(n) * n_loc + i] = src[static_cast<long long>(n) * n_glob + g];
}

// ================================================================ level
struct stmg3_level
{
  stmg_ctx *ctx = nullptr;
  Level3Spec spec;
  Level3Consts consts{};
  DevGeom3 geom{};
  bool deformed = false;
  std::vector<double> verts_h;
  DevArray<double> verts, pmean, one_w, gemmE;
  double inv_vol = 1.0;
  int smoother_kind = STMG_SMOOTHER_NONE;
  // Vanka: classes, colour batches (8 parity colours), anchors
  std::vector<DevArray<long long>> cls_rel;
  std::vector<DevArray<double>> cls_weight, cls_inverse;
  // exact per-cell patches built on the GPU (deformed levels, patch3_gpu.cu):
  // concatenated dof offsets, weights and inverses
  DevArray<long long> rel_all;
  DevArray<double> weight_all, inv_all, fac_all;
  // time-diagonalised per-cell blocks (DG(2) deformed levels, vanka_big_fac_kernel)
  bool fac3 = false;
  Fac3Params fac3p{};
  bool gpu_patches = false;
  double patch_setup_s = 0.0;
  DevArray<DevPatchClass> classes;
  DevArray<VankaBatch> batches;
  DevArray<long long> vel_anchor, pre_anchor;
  std::vector<int> colour_first, colour_count;
  int max_nt = 0, n_classes = 0;
  bool affine_patches = false;
  std::uint64_t total_matrix_elements = 0;
  // time-diagonalised blocks: doubles the apply kernel streams per sweep (the
  // real block and the u-columns [P; Q] of the pair block) and its
  // multiply-adds per (patch, interval) column
  std::uint64_t fac_streamed_elements = 0, fac_macs = 0;
  DevArray<double> work, zeros;
  // z-split level (stmg3_solver_create_split): normalisations of the
  // projections over the whole mesh (the sums are reduced over the parts)
  double vol_global = 0.0, ncells_global = 0.0;

  void
  vmult(const double *x, const double *b, double *y, int n, const double *xprev, int coupled, int mode)
  {
    check(launch_vmult3(spec.r, spec.S(), consts, x, b, y, n, xprev, coupled, mode, ctx->stream), "vmult3");
    ctx->count(vmult3_launch_count(consts, spec.S(), n));
  }
  void
  project(double *x, int n)
  {
    check(launch_project3(geom, pmean.p, inv_vol, x, n, ctx->stream), "project3");
    ctx->count();
  }
  /// Residual (dual) vectors: remove the component along the left null
  /// vector of the pressure rows (the constant-mode coefficients). Equal to
  /// project() on Cartesian meshes; on deformed meshes the |K|-weighted mean
  /// would leave restricted residuals inconsistent.
  void
  project_residual(double *x, int n)
  {
    check(launch_project3(geom, one_w.p, 1.0 / static_cast<double>(spec.ncells()), x, n, ctx->stream),
          "project3");
    ctx->count();
  }
  void
  zero_constrained(double *x, int n)
  {
    check(launch_zero_constrained3(geom, x, n, ctx->stream), "zero3");
    ctx->count();
  }
  void
  vanka(const double *r, double *u, int n, double omega)
  {
    if (smoother_kind == STMG_SMOOTHER_NONE)
      throw std::invalid_argument("level has no smoother");
    for (size_t c = 0; c < colour_first.size(); ++c)
      if (colour_count[c] > 0)
        {
          if (fac3)
            check(launch_vanka_big_fac(classes.p, batches.p + colour_first[c], colour_count[c], max_nt, vel_anchor.p,
                                       pre_anchor.p, fac3p, r, u, spec.isz(), n, omega, ctx->stream),
                  "vanka3_fac");
          else
            check(launch_vanka_colour(classes.p, batches.p + colour_first[c], nullptr, colour_count[c], max_nt,
                                      vel_anchor.p, pre_anchor.p, r, u, spec.isz(), n, omega, ctx->stream),
                  "vanka3");
          ctx->count();
        }
  }
  double *
  scratch(int n)
  {
    work.resize(static_cast<size_t>(spec.isz()) * n);
    return work.p;
  }
  const double *
  zero_vector(int n)
  {
    const size_t need = static_cast<size_t>(spec.isz()) * n;
    if (zeros.n < need)
      {
        zeros.resize(need);
        check(cudaMemsetAsync(zeros.p, 0, sizeof(double) * zeros.n, ctx->stream), "memset");
      }
    return zeros.p;
  }
  void
  smooth_step(const double *b, double *u, double omega, int n, const double *xprev, int coupled, double *wbuf,
              bool u_is_zero = false)
  {
    if (!(omega > 0.0 && omega <= 1.0))
      throw std::invalid_argument("smooth_step: omega must be in (0, 1]");
    double *r = wbuf ? wbuf : scratch(n);
    if (u_is_zero && !coupled)
      check(cudaMemcpyAsync(r, b, sizeof(double) * spec.isz() * n, cudaMemcpyDeviceToDevice, ctx->stream), "copy");
    else
      vmult(u, b, r, n, xprev, coupled, 1);
    vanka(r, u, n, omega);
  }
};

namespace
{
void
build_level3(stmg3_level &L, const std::vector<double> *verts_host, bool affine_patches = false,
             const std::vector<double> *verts_ext = nullptr)
{
  const Level3Spec &s = L.spec;
  if (s.split() && (!verts_host || !verts_ext || affine_patches))
    throw std::invalid_argument("3D split level: needs deformed-geometry vertices (with the ghost layer) and exact "
                                "patches");
  if (s.nx < 1 || s.ny < 1 || s.nz < 1)
    throw std::invalid_argument("3D level: need at least one cell per direction");
  if (!vmult3_supported(s.r, s.S()))
    throw std::invalid_argument("3D level: instantiated for r in {1, 2}, k in {0, 1, 2}");
  if (!(s.tau > 0.0))
    throw std::invalid_argument("3D level: tau must be positive");
  if (verts_host)
    {
      if (static_cast<long long>(verts_host->size()) != 3 * s.nverts())
        throw std::invalid_argument("3D level: vertex array has the wrong size");
      L.deformed = true;
      L.verts_h = *verts_host;
      L.verts.upload(L.verts_h);
    }
  L.consts = make_level3_consts(s, L.deformed ? L.verts.p : nullptr);
  if (!L.deformed && s.r == 1) // one element operator for every cell: DMMA GEMM kernel
    {
      L.gemmE.upload(gemm_element_operator(s));
      L.consts.gemmE = L.gemmE.p;
    }
  L.geom = geom3(s);
  double vol = 1.0;
  L.pmean.upload(pressure_mean3(s, L.deformed ? &L.verts_h : nullptr, &vol));
  L.inv_vol = 1.0 / vol;
  {
    std::vector<double> one(static_cast<size_t>(s.mp()), 0.0);
    for (long long c = 0; c < s.ncells(); ++c)
      one[c * s.np()] = 1.0;
    L.one_w.upload(one);
  }
  if (L.smoother_kind == STMG_SMOOTHER_NONE)
    return;
  if (L.smoother_kind != STMG_SMOOTHER_CELL)
    throw std::invalid_argument("3D level: only cell Vanka is available in 3D");
  // affine_patches: the patch inverses of the undeformed (Cartesian) mesh
  // stand in for the per-cell ones on a deformed mesh (same dof patterns;
  // an approximate local solve)
  L.affine_patches = L.deformed && affine_patches;
  std::vector<int> cell_class;
  std::vector<DevPatchClass> dc;
  // Deformed levels with exact patches: one class per cell, set up on the
  // GPU (element matrices, R_T S R_T^T, batched Gauss-Jordan inverses); the
  // host path (LU with partial pivoting, setup3d.cpp cell_patch) remains for
  // 1-cell directions (singular whole-domain patches), a vanishing pivot,
  // and as the A/B switch STMG_PATCH3_HOST.
  const bool exact = L.deformed && !affine_patches;
  bool gpu_done = false;
  const bool gpu_ok = exact && s.nx >= 2 && s.ny >= 2 && s.nz >= 2 && (s.r == 1 || s.r == 2);
  if (s.split() && L.smoother_kind != STMG_SMOOTHER_NONE && !gpu_ok)
    throw std::invalid_argument("3D split level: the smoothed levels need >= 2 local cells per direction, r <= 2");
  if (gpu_ok && (s.split() || !std::getenv("STMG_PATCH3_HOST")))
    {
      const auto t0 = std::chrono::steady_clock::now();
      const Patch3Layout lo = cell_patch_layouts3(s);
      const long long nc = s.ncells();
      L.rel_all.upload(lo.rel);
      L.weight_all.upload(lo.weight);
      DevArray<int> ntv, st, cnt;
      st.upload(std::vector<int>{0});
      // element matrices: the level itself, or for a split level the owned
      // cells plus one ghost cell layer across each interface (the patches of
      // the interface cells sum the neighbour part's cells too: R_T S R_T^T
      // of the whole mesh)
      Level3Spec ex = s;
      const int gl = s.zlo_bc ? 0 : 1, gh = s.zhi_bc ? 0 : 1;
      ex.nz = s.nz + gl + gh;
      DevArray<double> vext, E;
      Level3Consts Pe = L.consts;
      if (s.split())
        {
          if (static_cast<long long>(verts_ext->size()) != 3 * ex.nverts())
            throw std::invalid_argument("3D split level: ghost-layer vertex array has the wrong size");
          vext.upload(*verts_ext);
          Pe = make_level3_consts(ex, vext.p);
        }
      const long long ncells_elem = ex.ncells(), cell0 = static_cast<long long>(gl) * s.nx * s.ny;
      E.resize(static_cast<size_t>(ncells_elem) * elem3_stride(s.r));
      // DG(2) (S = 3): time-diagonalised blocks, one real and one pair block
      // (0.56x the inverse bytes of the dense patch inverse);
      // A/B switch STMG_VANKA3_DENSE=1
      Fac3Params F{};
      bool fac = s.S() == 3 && !std::getenv("STMG_VANKA3_DENSE");
      if (fac)
        {
          const TemporalEigen eg = temporal_eigen(time_tables(s.k, s.tau));
          fac = eg.ok && !eg.blk_c0.empty() && eg.blk_c0.size() <= 2;
          if (fac)
            {
              F.S = s.S();
              F.nb = static_cast<int>(eg.blk_c0.size());
              for (int b = 0; b < F.nb; ++b)
                {
                  F.c0[b] = eg.blk_c0[b];
                  F.sz[b] = eg.blk_sz[b];
                  F.alpha[b] = eg.alpha[b];
                  F.beta[b] = eg.beta[b];
                  fac = fac && F.alpha[b] > 0.0 && (b == 0 ? F.c0[b] == 0 : F.c0[b] == F.c0[b - 1] + F.sz[b - 1]);
                }
              for (int i = 0; i < F.S * F.S; ++i)
                {
                  F.V[i] = eg.V[i];
                  F.W[i] = eg.W[i];
                }
            }
        }
      std::vector<long long> foff;
      std::uint64_t fac_streamed = 0, fac_macs = 0;
      if (fac)
        {
          // matrices 2c, 2c + 1: the blocks of cell c (sizes sz_b * n_s)
          std::vector<int> msz(2 * nc, 0);
          fac_streamed = fac_macs = 0;
          foff.assign(2 * nc + 1, 0);
          int max_m = 0;
          for (long long c = 0; c < nc; ++c)
            for (int b = 0; b < 2; ++b)
              {
                const int m = b < F.nb ? F.sz[b] * (lo.nt[c] / F.S) : 0;
                msz[2 * c + b] = m;
                // n_s columns of m rows each: all of a real block, the u-columns of a pair block
                fac_streamed += static_cast<std::uint64_t>(m) * (lo.nt[c] / F.S);
                fac_macs += static_cast<std::uint64_t>(m) * m;
                // even (16-byte aligned) starts: the apply kernel bulk-copies chunks
                foff[2 * c + b + 1] = foff[2 * c + b] + (static_cast<long long>(m) * m + 8 + 1) / 2 * 2;
                max_m = std::max(max_m, m);
              }
          L.fac_all.resize(static_cast<size_t>(foff.back()));
          DevArray<long long> aoff;
          aoff.upload(std::vector<long long>(foff.begin(), foff.end() - 1));
          ntv.upload(msz);
          cnt.upload(lo.nt);
          check(launch_patch3_fac_setup(Pe, s.r, s.S(), F, E.p, L.fac_all.p, aoff.p, ntv.p, cnt.p, max_m, nc, st.p,
                                        L.ctx->stream, ncells_elem, cell0),
                "patch3_fac_setup");
        }
      else
        {
          L.inv_all.resize(static_cast<size_t>(lo.inv_off.back()));
          DevArray<long long> aoff;
          aoff.upload(std::vector<long long>(lo.inv_off.begin(), lo.inv_off.end() - 1));
          ntv.upload(lo.nt);
          check(launch_patch3_setup(Pe, s.r, s.S(), E.p, L.inv_all.p, aoff.p, ntv.p, lo.max_nt, nc, st.p,
                                    L.ctx->stream, ncells_elem, cell0),
                "patch3_setup");
        }
      L.ctx->count(3);
      check(cudaStreamSynchronize(L.ctx->stream), "patch3_setup");
      E.release();
      int status = 0;
      check(cudaMemcpy(&status, st.p, sizeof(int), cudaMemcpyDeviceToHost), "status");
      if (status == 2)
        throw std::runtime_error("3D level: inverted cell");
      if (status != 0 && s.split())
        throw std::runtime_error("3D split level: GPU patch setup failed (vanishing pivot or layout mismatch)");
      if (status == 0)
        {
          cell_class.resize(nc);
          dc.resize(nc);
          for (long long c = 0; c < nc; ++c)
            {
              cell_class[c] = static_cast<int>(c);
              dc[c] = fac ? DevPatchClass{lo.nt[c], lo.nvel[c], L.rel_all.p + lo.rel_off[c],
                                          L.weight_all.p + lo.rel_off[c], nullptr, lo.nt[c] / F.S,
                                          lo.nvel[c] / F.S, L.fac_all.p + foff[2 * c]}
                          : DevPatchClass{lo.nt[c], lo.nvel[c], L.rel_all.p + lo.rel_off[c],
                                          L.weight_all.p + lo.rel_off[c], L.inv_all.p + lo.inv_off[c], 0, 0, nullptr};
            }
          L.n_classes = static_cast<int>(nc);
          L.max_nt = lo.max_nt;
          L.total_matrix_elements = fac ? static_cast<std::uint64_t>(foff.back()) : lo.total_matrix_elements;
          L.gpu_patches = gpu_done = true;
          L.fac3 = fac;
          L.fac3p = F;
          L.fac_streamed_elements = fac ? fac_streamed : 0;
          L.fac_macs = fac ? fac_macs : 0;
        }
      else
        {
          L.inv_all.release();
          L.fac_all.release();
          L.rel_all.release();
          L.weight_all.release();
        }
      L.patch_setup_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
  if (!gpu_done)
    {
      const auto t0 = std::chrono::steady_clock::now();
      const Patch3Set ps = build_patches3(s, exact ? &L.verts_h : nullptr);
      L.n_classes = static_cast<int>(ps.classes.size());
      L.max_nt = ps.max_nt;
      L.total_matrix_elements = ps.total_matrix_elements;
      cell_class = ps.cell_class;
      dc.resize(ps.classes.size());
      L.cls_rel.resize(ps.classes.size());
      L.cls_weight.resize(ps.classes.size());
      L.cls_inverse.resize(ps.classes.size());
      for (size_t i = 0; i < ps.classes.size(); ++i)
        {
          const PatchClass &pc = ps.classes[i];
          L.cls_rel[i].upload(pc.rel);
          L.cls_weight[i].upload(pc.weight);
          L.cls_inverse[i].upload(pc.inverse);
          dc[i] = DevPatchClass{pc.n_t, pc.n_vel, L.cls_rel[i].p, L.cls_weight[i].p, L.cls_inverse[i].p, 0, 0, nullptr};
        }
      L.patch_setup_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
  L.classes.upload(dc);
  // 8 parity colours: cells of one colour share no node, so a launch writes
  // every dof at most once (read-modify-write, deterministic)
  std::vector<VankaBatch> batches;
  std::vector<long long> va, pa;
  const int cols = vanka_cols_per_batch();
  const int p = s.p();
  for (int col = 0; col < 8; ++col)
    {
      L.colour_first.push_back(static_cast<int>(batches.size()));
      std::vector<std::vector<long long>> by_class(dc.size());
      for (int cz = col >> 2; cz < s.nz; cz += 2)
        for (int cy = (col >> 1) & 1; cy < s.ny; cy += 2)
          for (int cx = col & 1; cx < s.nx; cx += 2)
            by_class[cell_class[(static_cast<size_t>(cz) * s.ny + cy) * s.nx + cx]].push_back(
              (static_cast<long long>(cz) * s.ny + cy) * s.nx + cx);
      for (size_t c = 0; c < by_class.size(); ++c)
        for (size_t i = 0; i < by_class[c].size(); i += cols)
          {
            VankaBatch b{static_cast<int>(c), static_cast<int>(va.size()),
                         static_cast<int>(std::min<size_t>(cols, by_class[c].size() - i))};
            for (int j = 0; j < b.count; ++j)
              {
                const long long cell = by_class[c][i + j];
                const int cx = static_cast<int>(cell % s.nx), cy = static_cast<int>((cell / s.nx) % s.ny),
                          cz = static_cast<int>(cell / (static_cast<long long>(s.nx) * s.ny));
                va.push_back((static_cast<long long>(cz * p) * s.gy() + cy * p) * s.gx() + cx * p);
                pa.push_back(s.S() * s.mv() + cell * s.np());
              }
            batches.push_back(b);
          }
      L.colour_count.push_back(static_cast<int>(batches.size()) - L.colour_first.back());
    }
  L.batches.upload(batches);
  L.vel_anchor.upload(va);
  L.pre_anchor.upload(pa);
}

struct Solver3Level
{
  std::unique_ptr<stmg3_level> level;
  int tshift = 0;
  // transfer to the next coarser level (absent on level 0)
  DevArray<int> csr_i[6];
  DevArray<double> csr_v[6], child;
  DevTransfer3 dt{};
  DevArray<double> x, b, r, t, halo, tw;
};

void
upload_csr(const Csr1D &c, DevArray<int> &ip, DevArray<double> &v, DevCsr &d, std::vector<int> &colbuf)
{
  // ptr and col packed in one int array: [ptr (rows+1) | col]
  colbuf.assign(c.ptr.begin(), c.ptr.end());
  colbuf.insert(colbuf.end(), c.col.begin(), c.col.end());
  ip.upload(colbuf);
  v.upload(c.val);
  d.ptr = ip.p;
  d.col = ip.p + c.ptr.size();
  d.val = v.p;
}
} // namespace

// ================================================================ solver
struct stmg3_solver
{
  stmg_ctx *ctx = nullptr;
  int nu1 = 2, nu2 = 2;
  double omega = 0.8;
  bool project_pressure = true;
  double rtol = 1e-8, atol = 1e-14;
  int max_iterations = 200;
  int ortho = stmg_krylov::kMGS; // Arnoldi orthogonalization (stmg_solver_set_krylov)
  std::vector<std::unique_ptr<Solver3Level>> levels;
  DevArray<double> cG, cH, cB, cX;
  int coarse_n = 0;
  std::vector<std::unique_ptr<DevArray<double>>> V, Z;
  DevArray<double> w, scal, part, rhs;
  std::vector<double> hist;
  stmg_comm_ops comm{};
  bool has_comm = false;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_x = nullptr, ev_h = nullptr;

  // ---- C5 hybrid split: z parts (stmg3_solver_create_split)
  int zpart = 0, zparts = 1;
  stmg_comm_space_ops sops{};
  bool has_space = false;
  int coarse_n_loc = 0;     // coarse level: local interval size (coarse_n is the global one)
  long long coarse_mv = 0;  // velocity block of the (global) coarse level
  DevArray<int> cmap;       // [parts][coarse_n_loc]: local coarse dof -> global coarse dof
  DevArray<double> pl_a[2], pl_b[2], pl_s[2], psum, pdpart, cBs, cBg;

  stmg3_level &fine() { return *levels.back()->level; }
  int rank() const { return has_comm ? comm.rank : 0; }
  int world() const { return has_comm ? comm.world : 1; }
  int n_at(int l, int nI_fine) const { return nI_fine >> levels[l]->tshift; }
  bool split() const { return zparts > 1; }
  void
  need_space() const
  {
    if (split() && !has_space)
      throw std::runtime_error("z-split solver: install the parts' communicator (stmg3_solver_set_space_comm)");
  }
  static bool
  iface(const stmg3_level &L, int side)
  {
    return side == 0 ? !L.spec.zlo_bc : !L.spec.zhi_bc;
  }
  /// Exchange the interface planes (pl_a[side] -> partner, partner -> pl_b[side]).
  void
  exchange_planes(const stmg3_level &L, long long n)
  {
    need_space();
    if (sops.exchange_planes(sops.user, iface(L, 0) ? pl_a[0].p : nullptr, iface(L, 0) ? pl_b[0].p : nullptr,
                             iface(L, 1) ? pl_a[1].p : nullptr, iface(L, 1) ? pl_b[1].p : nullptr, n, ctx->stream) != 0)
      throw std::runtime_error("comm: exchange_planes failed");
  }
  void
  plane_op(const stmg3_level &L, int side, int op, int nI, double *x, double *buf, const double *other,
           const double *b = nullptr, const double *saved = nullptr)
  {
    check(launch_plane_op3(L.geom, side, op, nI, x, buf, other, b, saved, ctx->stream), "plane_op3");
    ctx->count();
  }
  /// Owner-accumulate of the interface rows after a local application:
  /// y += partner's partial sums (mode 0), r = r_own + r_partner - b (mode 1).
  void
  iface_sum(int l, double *y, const double *b, int nI, int mode)
  {
    if (!split())
      return;
    STMG_NVTX("iface_sum L%d", l);
    const stmg3_level &L = *levels[l]->level;
    const long long n = plane3_doubles(L.geom, nI);
    for (int side = 0; side < 2; ++side)
      if (iface(L, side))
        {
          pl_a[side].resize(n);
          pl_b[side].resize(n);
          plane_op(L, side, 0, nI, y, pl_a[side].p, nullptr);
        }
    exchange_planes(L, n);
    for (int side = 0; side < 2; ++side)
      if (iface(L, side))
        plane_op(L, side, mode == 1 ? 2 : 1, nI, y, nullptr, pl_b[side].p, b);
  }
  /// Additive Vanka update of a split level: both parts' interface
  /// increments are added to the pre-sweep interface values.
  void
  vanka(int l, const double *r, double *u, int nI)
  {
    stmg3_level &L = *levels[l]->level;
    if (!split())
      {
        L.vanka(r, u, nI, omega);
        return;
      }
    const long long n = plane3_doubles(L.geom, nI);
    for (int side = 0; side < 2; ++side)
      if (iface(L, side))
        {
          pl_s[side].resize(n);
          pl_a[side].resize(n);
          pl_b[side].resize(n);
          plane_op(L, side, 0, nI, u, pl_s[side].p, nullptr);
        }
    L.vanka(r, u, nI, omega);
    for (int side = 0; side < 2; ++side)
      if (iface(L, side))
        plane_op(L, side, 4, nI, u, pl_a[side].p, nullptr, nullptr, pl_s[side].p);
    exchange_planes(L, n);
    for (int side = 0; side < 2; ++side)
      if (iface(L, side))
        plane_op(L, side, 5, nI, u, pl_a[side].p, pl_b[side].p, nullptr, pl_s[side].p);
  }
  /// Mean-zero projection (residual: along the constant-mode coefficients).
  void
  project(int l, double *x, int nI, bool residual)
  {
    stmg3_level &L = *levels[l]->level;
    if (!split())
      {
        if (residual)
          L.project_residual(x, nI);
        else
          L.project(x, nI);
        return;
      }
    need_space();
    const int cnt = nI * L.spec.S();
    psum.resize(cnt);
    check(launch_project3_sums(L.geom, residual ? L.one_w.p : L.pmean.p, x, nI, psum.p, ctx->stream), "project3");
    if (sops.allreduce_sum(sops.user, psum.p, cnt, ctx->stream) != 0)
      throw std::runtime_error("comm: allreduce_sum (parts) failed");
    check(launch_project3_apply(L.geom, psum.p, residual ? 1.0 / L.ncells_global : 1.0 / L.vol_global, x, nI,
                                ctx->stream),
          "project3");
    ctx->count(2);
  }

  ~stmg3_solver()
  {
    if (comm_stream)
      cudaStreamDestroy(comm_stream);
    if (ev_x)
      cudaEventDestroy(ev_x);
    if (ev_h)
      cudaEventDestroy(ev_h);
  }

  // y = A x (mode 0) or b - A x (mode 1) with the jump coupling; the halo of
  // the previous rank travels on a side stream while intervals 1..nI-1 run.
  void
  coupled_vmult(int l, const double *x, const double *b, double *y, int nI, int mode)
  {
    stmg3_level &L = *levels[l]->level;
    if (world() == 1)
      {
        L.vmult(x, b, y, nI, nullptr, 1, mode);
        iface_sum(l, y, b, nI, mode);
        return;
      }
    if (!comm_stream)
      {
        check(cudaStreamCreateWithFlags(&comm_stream, cudaStreamNonBlocking), "stream");
        check(cudaEventCreateWithFlags(&ev_x, cudaEventDisableTiming), "event");
        check(cudaEventCreateWithFlags(&ev_h, cudaEventDisableTiming), "event");
      }
    const long long isz = L.spec.isz(), mv = L.spec.mv();
    DevArray<double> &h = levels[l]->halo;
    h.resize(mv);
    check(cudaEventRecord(ev_x, ctx->stream), "event");
    check(cudaStreamWaitEvent(comm_stream, ev_x, 0), "wait");
    const double *send = x + (nI - 1) * isz + (L.spec.S() - 1) * mv;
    if (comm.exchange_halo(comm.user, send, h.p, mv, comm_stream) != 0)
      throw std::runtime_error("comm: exchange_halo failed");
    check(cudaEventRecord(ev_h, comm_stream), "event");
    if (nI > 1)
      L.vmult(x + isz, b ? b + isz : nullptr, y + isz, nI - 1, x + (L.spec.S() - 1) * mv, 1, mode);
    check(cudaStreamWaitEvent(ctx->stream, ev_h, 0), "wait");
    // interval 0 alone: its init kernel must not touch intervals 1..nI-1
    L.vmult(x, b, y, 1, rank() == 0 ? nullptr : h.p, 1, mode);
    iface_sum(l, y, b, nI, mode);
  }

  /// Krylov sums over every rank: the time slabs, then the z parts.
  void
  allreduce(double *buf, int n)
  {
    if (world() > 1 && comm.allreduce_sum(comm.user, buf, n, ctx->stream) != 0)
      throw std::runtime_error("comm: allreduce_sum failed");
    if (split())
      {
        need_space();
        if (sops.allreduce_sum(sops.user, buf, n, ctx->stream) != 0)
          throw std::runtime_error("comm: allreduce_sum (parts) failed");
      }
  }
  /// Inner products of the finest level count the plane shared with the
  /// lower part once (the lower part owns it).
  void
  plane_fix(const double *const *V, int m, bool with_norm, const double *w, double *out, int nI)
  {
    const stmg3_level &L = fine();
    if (!split() || !iface(L, 0))
      return;
    pdpart.resize(plane_multidot_part_doubles());
    check(launch_plane_multidot_sub(L.geom, 0, nI, V, m, with_norm, w, pdpart.p, out, ctx->stream), "plane_dot");
    ctx->count(2);
  }

  /// restrict_residual: R fine, zero constrained, project (transfer.cpp:117-132)
  void
  restrict_residual(int l, const double *fine_v, double *coarse_v, int nc, bool project)
  {
    Solver3Level &F = *levels[l];
    stmg3_level &C = *levels[l - 1]->level;
    F.tw.resize(std::max<long long>(1, transfer3_work_doubles(F.dt, nc)));
    const int nf = F.dt.h_time ? 2 * nc : nc;
    double *fv = const_cast<double *>(fine_v); // split: interface planes halved, restored below
    if (split())
      for (int side = 0; side < 2; ++side)
        if (iface(*F.level, side))
          {
            pl_s[side].resize(plane3_doubles(F.level->geom, nf));
            plane_op(*F.level, side, 0, nf, fv, pl_s[side].p, nullptr);
            plane_op(*F.level, side, 3, nf, fv, nullptr, nullptr);
          }
    check(launch_restrict3(F.dt, fine_v, coarse_v, nc, ctx->stream, F.dt.spatial ? F.tw.p : nullptr), "restrict3");
    ctx->count(F.dt.spatial ? 4 : 2);
    if (split())
      {
        for (int side = 0; side < 2; ++side)
          if (iface(*F.level, side))
            plane_op(*F.level, side, 6, nf, fv, pl_s[side].p, nullptr);
        iface_sum(l - 1, coarse_v, nullptr, nc, 0);
      }
    C.zero_constrained(coarse_v, nc);
    if (project)
      this->project(l - 1, coarse_v, nc, true);
  }

  /// prolongate_correction (transfer.cpp:102-115), then fine (+)= result
  void
  prolongate_correction(int l, const double *coarse_v, double *fine_v, int nc, bool project, bool accumulate)
  {
    Solver3Level &F = *levels[l];
    stmg3_level &L = *F.level;
    const int nf = F.dt.h_time ? 2 * nc : nc;
    const long long n = L.spec.isz() * nf;
    F.t.resize(n);
    F.tw.resize(std::max<long long>(1, transfer3_work_doubles(F.dt, nc)));
    check(launch_prolongate3(F.dt, coarse_v, F.t.p, nc, ctx->stream, F.dt.spatial ? F.tw.p : nullptr),
          "prolongate3");
    ctx->count(F.dt.spatial ? 4 : 2);
    L.zero_constrained(F.t.p, nf);
    if (project)
      this->project(l, F.t.p, nf, false);
    if (accumulate)
      {
        check(launch_axpy(n, 1.0, nullptr, 1.0, F.t.p, fine_v, ctx->stream), "axpy");
        ctx->count();
      }
    else
      check(cudaMemcpyAsync(fine_v, F.t.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream), "copy");
  }

  /// Exact coarse solve of the all-at-once system on level 0 by forward
  /// substitution x_t = G b_t + H v_{t-1}; every rank gathers the coarse
  /// right-hand sides, walks the whole time axis and keeps its slab.
  void
  coarse_forward(const double *b_v, double *x_v, int nI)
  {
    if (split())
      {
        // parts -> the global coarse vector of every local interval
        need_space();
        const long long per_loc = static_cast<long long>(coarse_n_loc) * nI;
        cBs.resize(per_loc * zparts);
        if (sops.allgather(sops.user, b_v, cBs.p, per_loc, ctx->stream) != 0)
          throw std::runtime_error("comm: allgather (parts) failed");
        cBg.resize(static_cast<long long>(coarse_n) * nI);
        coarse_map_kernel<<<dim3((coarse_n_loc + 127) / 128, nI, zparts), 128, 0, ctx->stream>>>(
          cBs.p, cmap.p, coarse_n_loc, coarse_n, nI, cBg.p, 0);
        check(cudaGetLastError(), "coarse_map");
        ctx->count();
      }
    const Level3Spec &sp = levels[0]->level->spec;
    const long long per = static_cast<long long>(coarse_n) * nI;
    const double *B = split() ? cBg.p : b_v;
    if (world() > 1)
      {
        cB.resize(per * world());
        if (comm.allgather(comm.user, B, cB.p, per, ctx->stream) != 0)
          throw std::runtime_error("comm: allgather failed");
        B = cB.p;
      }
    const int n_all = nI * world();
    cX.resize(static_cast<size_t>(coarse_n) * n_all);
    const int mv = static_cast<int>(coarse_mv);
    const long long v_off = (sp.S() - 1) * coarse_mv;
    const int rows_per_block = 8;
    for (int t = 0; t < n_all; ++t)
      {
        coarse3_step_kernel<<<(coarse_n + rows_per_block - 1) / rows_per_block, 32 * rows_per_block, 0,
                              ctx->stream>>>(cG.p, cH.p, coarse_n, mv, B + static_cast<long long>(t) * coarse_n,
                                             t > 0 ? cX.p + static_cast<long long>(t - 1) * coarse_n + v_off : nullptr,
                                             cX.p + static_cast<long long>(t) * coarse_n);
        check(cudaGetLastError(), "coarse3_step");
        ctx->count();
      }
    if (split())
      {
        // this part's dofs of this slab's intervals
        coarse_map_kernel<<<dim3((coarse_n_loc + 127) / 128, nI, 1), 128, 0, ctx->stream>>>(
          cX.p + static_cast<long long>(rank()) * per, cmap.p + static_cast<long long>(zpart) * coarse_n_loc,
          coarse_n_loc, coarse_n, nI, x_v, 1);
        check(cudaGetLastError(), "coarse_map");
        ctx->count();
        return;
      }
    check(cudaMemcpyAsync(x_v, cX.p + static_cast<long long>(rank()) * per, sizeof(double) * per,
                          cudaMemcpyDeviceToDevice, ctx->stream),
          "copy");
  }

  /// All-at-once VCycle::cycle (solver.cpp:69-93); nI = intervals of level l.
  void
  cycle(int l, const double *b_v, double *x_v, int nI)
  {
    STMG_NVTX("vcycle3 L%d (%d intervals)", l, nI);
    if (l == 0)
      {
        coarse_forward(b_v, x_v, nI);
        return;
      }
    Solver3Level &S = *levels[l];
    stmg3_level &L = *S.level;
    const long long isz = L.spec.isz() * nI;
    S.r.resize(isz);
    check(cudaMemsetAsync(x_v, 0, sizeof(double) * isz, ctx->stream), "memset");
    for (int s = 0; s < nu1; ++s)
      {
        STMG_NVTX("L%d pre-smooth", l);
        if (s == 0) // x = 0 on every rank: b - A 0 = b
          {
            check(cudaMemcpyAsync(S.r.p, b_v, sizeof(double) * isz, cudaMemcpyDeviceToDevice, ctx->stream), "copy");
            vanka(l, S.r.p, x_v, nI);
          }
        else
          {
            coupled_vmult(l, x_v, b_v, S.r.p, nI, 1);
            vanka(l, S.r.p, x_v, nI);
          }
      }
    coupled_vmult(l, x_v, b_v, S.r.p, nI, 1);
    Solver3Level &C = *levels[l - 1];
    const int nc = S.dt.h_time ? nI / 2 : nI;
    const long long csz = C.level->spec.isz() * nc;
    C.b.resize(csz);
    C.x.resize(csz);
    {
      STMG_NVTX("L%d restrict", l);
      restrict_residual(l, S.r.p, C.b.p, nc, project_pressure);
    }
    cycle(l - 1, C.b.p, C.x.p, nc);
    {
      STMG_NVTX("L%d prolongate", l);
      prolongate_correction(l, C.x.p, x_v, nc, project_pressure, true);
    }
    for (int s = 0; s < nu2; ++s)
      {
        STMG_NVTX("L%d post-smooth", l);
        coupled_vmult(l, x_v, b_v, S.r.p, nI, 1);
        vanka(l, S.r.p, x_v, nI);
      }
  }

  void
  check_slab(int nI) const
  {
    const int tmax = levels.front()->tshift;
    if (nI < 1 || (nI % (1 << tmax)) != 0)
      throw std::invalid_argument("3D all-at-once: the slab's interval count must be divisible by 2^(time coarsenings)");
  }

  double
  dot(const double *a, const double *b, long long n, int slot, int nI)
  {
    check(launch_dot(a, b, n, part.p, scal.p + slot, ctx->stream), "dot");
    ctx->count(2);
    plane_fix(&b, 1, false, a, scal.p + slot, nI);
    allreduce(scal.p + slot, 1);
    double h = 0.0;
    check(cudaMemcpyAsync(&h, scal.p + slot, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream), "d2h");
    check(cudaStreamSynchronize(ctx->stream), "sync");
    return h;
  }

  DevArray<double> &
  basis(std::vector<std::unique_ptr<DevArray<double>>> &B, int j, long long n)
  {
    while (static_cast<int>(B.size()) <= j)
      B.push_back(std::make_unique<DevArray<double>>());
    B[j]->resize(n);
    return *B[j];
  }

  /// gmres (solver.cpp:95-202): right preconditioning with the all-at-once
  /// V-cycle, modified Gram-Schmidt with device-resident coefficients,
  /// Givens rotations on the host, Z stored (flexible form).
  int
  gmres(const double *b_v, double *x_v, int *iterations, double *history, int history_cap, int nI)
  {
    stmg3_level &L = fine();
    const int top = static_cast<int>(levels.size()) - 1;
    const long long n = L.spec.isz() * nI;
    w.resize(n);
    part.resize(stmg_krylov::part_doubles());
    scal.resize(2 * (max_iterations + 2));
    hist.clear();
    const double norm_b = std::sqrt(dot(b_v, b_v, n, 0, nI));
    const double tol = std::max(rtol * norm_b, atol);
    hist.push_back(norm_b);
    check(cudaMemsetAsync(x_v, 0, sizeof(double) * n, ctx->stream), "memset");
    int iters = 0;
    bool converged = norm_b <= tol;
    if (!converged)
      {
        const int m = max_iterations;
        std::vector<double> H(static_cast<size_t>(m + 1) * m, 0.0), g(m + 1, 0.0), cs(m), sn(m);
        g[0] = norm_b;
        DevArray<double> &v0 = basis(V, 0, n);
        check(cudaMemcpyAsync(v0.p, b_v, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream), "copy");
        check(launch_scale(n, 1.0 / norm_b, v0.p, ctx->stream), "scale");
        ctx->count();
        int j = 0;
        std::vector<double> hcol(m + 2);
        for (; j < m; ++j)
          {
            STMG_NVTX("fgmres3 it %d", j);
            DevArray<double> &zj = basis(Z, j, n);
            cycle(top, V[j]->p, zj.p, nI);
            coupled_vmult(top, zj.p, nullptr, w.p, nI, 0);
            // Arnoldi: MGS (the reference's, solver.cpp:146-152) or CGS2
            // (two batched all-reduces per iteration), krylov.hpp
            const double h_next = stmg_krylov::orthogonalize(
              ortho, V, j, w.p, n, part.p, scal.p, hcol, [&](double *buf, int cnt) { allreduce(buf, cnt); }, ctx,
              [&](const double *const *Vp, int m, bool wn, const double *wp, double *out) {
                plane_fix(Vp, m, wn, wp, out, nI);
              });
            const bool breakdown = !(h_next > 1e-300);
            auto Hc = [&](int i) -> double & { return H[static_cast<size_t>(j) * (m + 1) + i]; };
            for (int i = 0; i <= j; ++i)
              Hc(i) = hcol[i];
            for (int i = 0; i < j; ++i)
              {
                const double tt = cs[i] * Hc(i) + sn[i] * Hc(i + 1);
                Hc(i + 1) = -sn[i] * Hc(i) + cs[i] * Hc(i + 1);
                Hc(i) = tt;
              }
            const double denom = std::hypot(Hc(j), h_next);
            cs[j] = Hc(j) / denom;
            sn[j] = h_next / denom;
            Hc(j) = denom;
            g[j + 1] = -sn[j] * g[j];
            g[j] = cs[j] * g[j];
            const double res = std::abs(g[j + 1]);
            hist.push_back(res);
            if (res <= tol || breakdown)
              {
                ++j;
                converged = true;
                break;
              }
            DevArray<double> &vn = basis(V, j + 1, n);
            check(cudaMemcpyAsync(vn.p, w.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream), "copy");
            check(launch_scale(n, 1.0 / h_next, vn.p, ctx->stream), "scale");
            ctx->count();
          }
        iters = std::min(j, m);
        std::vector<double> y(iters);
        for (int i = iters - 1; i >= 0; --i)
          {
            double s = g[i];
            for (int c = i + 1; c < iters; ++c)
              s -= H[static_cast<size_t>(c) * (m + 1) + i] * y[c];
            y[i] = s / H[static_cast<size_t>(i) * (m + 1) + i];
          }
        stmg_krylov::update_solution(Z, y, x_v, n, ctx);
      }
    if (iterations)
      *iterations = iters;
    for (int i = 0; history && i < history_cap && i < static_cast<int>(hist.size()); ++i)
      history[i] = hist[i];
    if (!converged)
      throw std::runtime_error("gmres: not converged within max_iterations");
    return iters;
  }

  int
  solve(const double *F, double *X, int nI, const double *v_init, int *iterations, double *history, int cap)
  {
    check_slab(nI);
    stmg3_level &L = fine();
    const long long n = L.spec.isz() * nI;
    rhs.resize(n);
    check(cudaMemcpyAsync(rhs.p, F, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream), "copy");
    if (v_init && rank() == 0)
      {
        // F_0 += C v_init (coupling_rhs, constrained rows zero); a z part
        // sums the coupling's interface rows with its neighbours
        L.vmult(L.zero_vector(1), F, rhs.p, 1, v_init, 1, 1);
        iface_sum(static_cast<int>(levels.size()) - 1, rhs.p, F, 1, 1);
        L.zero_constrained(rhs.p, 1);
      }
    const int it = gmres(rhs.p, X, iterations, history, cap, nI);
    project(static_cast<int>(levels.size()) - 1, X, nI, false);
    return it;
  }
};

namespace
{
stmg3_level *
make_level3(stmg_ctx *ctx, const Level3Spec &s, int smoother, const std::vector<double> *verts,
            bool affine_patches = false, const std::vector<double> *verts_ext = nullptr)
{
  auto L = std::make_unique<stmg3_level>();
  L->ctx = ctx;
  L->spec = s;
  L->smoother_kind = smoother;
  build_level3(*L, verts, affine_patches, verts_ext);
  return L.release();
}

/// Vertex planes [z_lo, z_hi] of a level's vertex array.
std::vector<double>
vertex_planes(const Level3Spec &g, const std::vector<double> &v, int z_lo, int z_hi)
{
  const size_t plane = static_cast<size_t>(g.nx + 1) * (g.ny + 1) * 3;
  return std::vector<double>(v.begin() + plane * z_lo, v.begin() + plane * (z_hi + 1));
}

/// Local coarse dof -> whole-mesh coarse dof of every z part (one interval).
std::vector<int>
coarse_part_map(const Level3Spec &g, int parts)
{
  const int nzl = g.nz / parts, p = g.p();
  std::vector<int> map;
  for (int part = 0; part < parts; ++part)
    {
      Level3Spec l = g;
      l.nz = nzl;
      const long long lgz = l.gz(), gxy = static_cast<long long>(g.gx()) * g.gy();
      for (int a = 0; a < g.S(); ++a)
        for (int c = 0; c < 3; ++c)
          for (long long Z = 0; Z < lgz; ++Z)
            for (long long xy = 0; xy < gxy; ++xy)
              map.push_back(static_cast<int>(a * g.mv() + c * g.nsc() + (Z + part * nzl * p) * gxy + xy));
      for (int a = 0; a < g.S(); ++a)
        for (long long cell = 0; cell < l.ncells(); ++cell)
          for (int m = 0; m < g.np(); ++m)
            map.push_back(static_cast<int>(g.S() * g.mv() + a * g.mp() +
                                           (cell + static_cast<long long>(part) * nzl * g.nx * g.ny) * g.np() + m));
    }
  return map;
}
} // namespace

namespace
{
struct PlanLevel3
{
  Level3Spec s;
  int tsh;
};

// combine_hierarchies (hierarchy.cpp:9-97) in 3D, fine first: spatial list
// (r -> r/2 ... -> 1, then n_hcoarse h-steps, each also halving the time
// grid when time_coarsen) and temporal list (k, k/2, ..., k_min) aligned at
// the COARSE end, so the temporal p-steps sit on the coarsest levels (the
// reference's C2 plan has L1 = h_space + p_time). Measured: putting them on
// the fine levels instead costs 35 / 77 iterations at 8^3 / 16^3 (r = 2,
// k = 2) against 7.
std::vector<PlanLevel3>
plan3(const Level3Spec &f, int n_hcoarse, int time_coarsen, int k_min)
{
  if (k_min < 0 || k_min > f.k)
    throw std::invalid_argument("3D solver: need 0 <= k_min <= k");
  if (n_hcoarse < 0)
    throw std::invalid_argument("3D solver: n_hcoarse must be >= 0");
  using D = PlanLevel3;
  std::vector<D> sp{{f, 0}};
  while (sp.back().s.r > 1)
    {
      D e = sp.back();
      e.s.r /= 2;
      sp.push_back(e);
    }
  for (int i = 0; i < n_hcoarse; ++i)
    {
      D e = sp.back();
      if (e.s.nx % 2 || e.s.ny % 2 || e.s.nz % 2)
        throw std::invalid_argument("3D solver: mesh not divisible for h-coarsening");
      e.s.nx /= 2;
      e.s.ny /= 2;
      e.s.nz /= 2;
      if (time_coarsen)
        {
          e.tsh += 1;
          e.s.tau *= 2.0;
        }
      sp.push_back(e);
    }
  std::vector<int> tk{f.k};
  while (tk.back() > k_min)
    tk.push_back(tk.back() / 2);
  const size_t nlev = std::max(sp.size(), tk.size());
  std::vector<D> d(nlev);
  for (size_t i = 0; i < nlev; ++i)
    {
      const size_t c = nlev - 1 - i; // distance from the coarse end
      d[i] = sp[std::min(sp.size() - 1, i)];
      d[i].s.k = tk[tk.size() - 1 - std::min(c, tk.size() - 1)];
    }
  return d;
}
} // namespace

extern "C" {

int
stmg3_level_create(stmg_ctx *ctx, int nx, int ny, int nz, int r, int k, double tau, double nu, double gamma,
                   int smoother_kind, const double *vertices, stmg3_level **out)
{
  return guarded([&] {
    STMG_NVTX("stmg3_level_create");
    if (!ctx || !out)
      throw std::invalid_argument("null argument");
    check(cudaSetDevice(ctx->device), "cudaSetDevice");
    Level3Spec s;
    s.nx = nx;
    s.ny = ny;
    s.nz = nz;
    s.r = r;
    s.k = k;
    s.tau = tau;
    s.nu = nu;
    s.gamma = gamma;
    std::vector<double> v;
    if (vertices)
      v.assign(vertices, vertices + 3 * s.nverts());
    *out = make_level3(ctx, s, smoother_kind, vertices ? &v : nullptr);
  });
}

int
stmg3_level_destroy(stmg3_level *level)
{
  delete level;
  return STMG_OK;
}

int
stmg3_level_sizes(const stmg3_level *L, int64_t *out)
{
  return guarded([&] {
    STMG_NVTX("stmg3_level_sizes");
    if (!L || !out)
      throw std::invalid_argument("null argument");
    const Level3Spec &s = L->spec;
    const int64_t v[12] = {s.S(), s.mv(), s.mp(), s.isz(), s.nsc(), s.gx(), s.gy(), s.gz(), s.np(), L->max_nt,
                           L->n_classes, static_cast<int64_t>(L->total_matrix_elements)};
    std::memcpy(out, v, sizeof(v));
  });
}

int
stmg3_level_patch_info(const stmg3_level *L, double *out)
{
  return guarded([&] {
    if (!L || !out)
      throw std::invalid_argument("stmg3_level_patch_info: null argument");
    out[0] = L->patch_setup_s;
    out[1] = L->gpu_patches ? (L->fac3 ? 2.0 : 1.0) : 0.0;
    out[2] = L->affine_patches ? 1.0 : 0.0;
    out[3] = static_cast<double>(L->n_classes);
    out[4] = static_cast<double>(L->fac_streamed_elements);
    out[5] = static_cast<double>(L->fac_macs);
  });
}

int
stmg3_apply_block(stmg3_level *L, const double *x, double *y, int n, int raw)
{
  return guarded([&] { L->vmult(x, nullptr, y, n, nullptr, 0, raw ? 2 : 0); });
}

int
stmg3_vmult(stmg3_level *L, const double *x, double *y, int n, const double *x_prev_slot)
{
  return guarded([&] { L->vmult(x, nullptr, y, n, x_prev_slot, 1, 0); });
}

int
stmg3_residual(stmg3_level *L, const double *b, const double *x, double *r, int n, const double *x_prev_slot,
               int coupled)
{
  return guarded([&] { L->vmult(x, b, r, n, x_prev_slot, coupled ? 1 : 0, 1); });
}

int
stmg3_apply_additive(stmg3_level *L, const double *r, double *out, int n)
{
  return guarded([&] {
    STMG_NVTX("stmg3_apply_additive");
    check(cudaMemsetAsync(out, 0, sizeof(double) * L->spec.isz() * n, L->ctx->stream), "memset");
    L->vanka(r, out, n, 1.0);
  });
}

int
stmg3_smooth_step(stmg3_level *L, const double *b, double *u, double omega, int n, const double *x_prev_slot,
                  int coupled, double *work)
{
  return guarded([&] { L->smooth_step(b, u, omega, n, x_prev_slot, coupled ? 1 : 0, work); });
}

int
stmg3_vanka_update(stmg3_level *L, const double *r, double *u, double omega, int n)
{
  return guarded([&] {
    STMG_NVTX("stmg3_vanka_update");
    if (!(omega > 0.0 && omega <= 1.0))
      throw std::invalid_argument("vanka_update: omega must be in (0, 1]");
    L->vanka(r, u, n, omega);
  });
}

int
stmg3_project_mean_zero(stmg3_level *L, double *x, int n)
{
  return guarded([&] { L->project(x, n); });
}

namespace
{
stmg3_solver *
create_solver3(stmg_ctx *ctx, int nx, int ny, int nz, int r, int k, double tau, double nu, double gamma, int n_hcoarse,
               int time_coarsen, int k_min, int affine_patches, const double *vertices, int nu1, int nu2,
               double omega, double rtol, double atol, int max_iterations, int z_parts, int z_part)
{
  if (!ctx)
    throw std::invalid_argument("null argument");
  if (!(omega > 0.0 && omega <= 1.0))
    throw std::invalid_argument("omega must be in (0, 1]");
  if (z_parts < 1 || z_part < 0 || z_part >= z_parts)
    throw std::invalid_argument("3D split: need 0 <= z_part < z_parts");
  if (z_parts > 1 && (!vertices || affine_patches))
    throw std::invalid_argument("3D split: needs the (global) vertex array and exact patches");
  check(cudaSetDevice(ctx->device), "cudaSetDevice");
  auto S = std::make_unique<stmg3_solver>();
  S->ctx = ctx;
  S->nu1 = nu1;
  S->nu2 = nu2;
  S->omega = omega;
  S->rtol = rtol;
  S->atol = atol;
  S->max_iterations = max_iterations;
  S->zparts = z_parts;
  S->zpart = z_part;
  Level3Spec f;
  f.nx = nx;
  f.ny = ny;
  f.nz = nz;
  f.r = r;
  f.k = k;
  f.tau = tau;
  f.nu = nu;
  f.gamma = gamma;
  const std::vector<PlanLevel3> d = plan3(f, n_hcoarse, time_coarsen, k_min);
  // geometry of every level: the finest vertices restricted to the coarse
  // vertex set (nested index sets; non-nested geometry on deformed meshes)
  std::vector<std::vector<double>> vv(d.size());
  if (vertices)
    {
      vv[0].assign(vertices, vertices + 3 * f.nverts());
      for (size_t i = 1; i < d.size(); ++i)
        {
          const Level3Spec &c = d[i].s;
          const Level3Spec &fs = d[0].s;
          const int ratio = fs.nx / c.nx;
          vv[i].resize(3 * c.nverts());
          for (int vz = 0; vz <= c.nz; ++vz)
            for (int vy = 0; vy <= c.ny; ++vy)
              for (int vx = 0; vx <= c.nx; ++vx)
                for (int q = 0; q < 3; ++q)
                  vv[i][((static_cast<size_t>(vz) * (c.ny + 1) + vy) * (c.nx + 1) + vx) * 3 + q] =
                    vv[0][((static_cast<size_t>(vz * ratio) * (fs.ny + 1) + vy * ratio) * (fs.nx + 1) + vx * ratio) *
                            3 + q];
        }
    }
  // z-split: every level holds the cells [z0, z0 + nz / z_parts) of its mesh
  auto local_spec = [&](const Level3Spec &g) {
    Level3Spec l = g;
    if (z_parts > 1)
      {
        if (g.nz % z_parts)
          throw std::invalid_argument("3D split: nz of every level must be divisible by z_parts");
        l.nz = g.nz / z_parts;
        l.nz_glob = g.nz;
        l.zlo_bc = z_part == 0;
        l.zhi_bc = z_part == z_parts - 1;
      }
    return l;
  };
  for (size_t i = d.size(); i-- > 0;)
    {
      auto SL = std::make_unique<Solver3Level>();
      SL->tshift = d[i].tsh;
      const Level3Spec ls = local_spec(d[i].s);
      const int smoother = i + 1 == d.size() ? STMG_SMOOTHER_NONE : STMG_SMOOTHER_CELL;
      if (z_parts > 1)
        {
          const int z0 = z_part * ls.nz, gl = ls.zlo_bc ? 0 : 1, gh = ls.zhi_bc ? 0 : 1;
          const std::vector<double> own = vertex_planes(d[i].s, vv[i], z0, z0 + ls.nz);
          const std::vector<double> ext = vertex_planes(d[i].s, vv[i], z0 - gl, z0 + ls.nz + gh);
          SL->level.reset(make_level3(ctx, ls, smoother, &own, false, &ext));
          double vol = 0.0;
          pressure_mean3(d[i].s, &vv[i], &vol);
          SL->level->vol_global = vol;
          SL->level->ncells_global = static_cast<double>(d[i].s.ncells());
        }
      else
        SL->level.reset(make_level3(ctx, ls, smoother, vertices ? &vv[i] : nullptr, affine_patches != 0));
      S->levels.push_back(std::move(SL));
    }
  for (size_t l = 1; l < S->levels.size(); ++l)
    {
      Solver3Level &F = *S->levels[l];
      const Level3Spec &cs = S->levels[l - 1]->level->spec, &fs = F.level->spec;
      const bool ht = S->levels[l - 1]->tshift > F.tshift;
      const Transfer3Tables t = build_transfer3(cs, fs, ht);
      DevTransfer3 &dt = F.dt;
      dt = DevTransfer3{};
      dt.spatial = t.spatial;
      dt.pmode = t.pmode;
      dt.h_time = t.h_time;
      std::vector<int> buf;
      if (t.spatial)
        {
          const Csr1D *cc[6] = {&t.px, &t.py, &t.pz, &t.rx, &t.ry, &t.rz};
          DevCsr *dd[6] = {&dt.px, &dt.py, &dt.pz, &dt.rx, &dt.ry, &dt.rz};
          for (int q = 0; q < 6; ++q)
            upload_csr(*cc[q], F.csr_i[q], F.csr_v[q], *dd[q], buf);
          F.child.upload(t.child);
          dt.child = F.child.p;
        }
      const int Sf = fs.S(), Sc = cs.S();
      for (int h = 0; h < 2; ++h)
        for (int a = 0; a < Sf; ++a)
          for (int b = 0; b < Sc; ++b)
            dt.E[h * kMaxS * kMaxS + a * kMaxS + b] = t.E[(static_cast<size_t>(h) * Sf + a) * Sc + b];
      dt.f = F.level->geom;
      dt.c = S->levels[l - 1]->level->geom;
    }
  // coarse level: G, H of the forward substitution (whole mesh)
  {
    const Level3Spec &g0 = d.back().s;
    const stmg3_level &L0 = *S->levels[0]->level;
    std::vector<double> G, H, pm;
    coarse3_tables(g0, vertices ? &vv.back() : nullptr, G, H, pm);
    S->cG.upload(G);
    S->cH.upload(H);
    S->coarse_n = static_cast<int>(g0.isz());
    S->coarse_mv = g0.mv();
    S->coarse_n_loc = static_cast<int>(L0.spec.isz());
    if (z_parts > 1)
      S->cmap.upload(coarse_part_map(g0, z_parts));
  }
  return S.release();
}
} // namespace

int
stmg3_solver_create(stmg_ctx *ctx, int nx, int ny, int nz, int r, int k, double tau, double nu, double gamma,
                    int n_hcoarse, int time_coarsen, int k_min, int affine_patches, const double *vertices, int nu1,
                    int nu2, double omega, double rtol, double atol, int max_iterations, stmg3_solver **out)
{
  return guarded([&] {
    STMG_NVTX("stmg3_solver_create");
    if (!out)
      throw std::invalid_argument("null argument");
    *out = create_solver3(ctx, nx, ny, nz, r, k, tau, nu, gamma, n_hcoarse, time_coarsen, k_min, affine_patches,
                          vertices, nu1, nu2, omega, rtol, atol, max_iterations, 1, 0);
  });
}

int
stmg3_solver_create_split(stmg_ctx *ctx, int nx, int ny, int nz, int r, int k, double tau, double nu, double gamma,
                          int n_hcoarse, int time_coarsen, int k_min, const double *vertices, int z_parts, int z_part,
                          int nu1, int nu2, double omega, double rtol, double atol, int max_iterations,
                          stmg3_solver **out)
{
  return guarded([&] {
    STMG_NVTX("stmg3_solver_create_split");
    if (!out)
      throw std::invalid_argument("null argument");
    *out = create_solver3(ctx, nx, ny, nz, r, k, tau, nu, gamma, n_hcoarse, time_coarsen, k_min, 0, vertices, nu1,
                          nu2, omega, rtol, atol, max_iterations, z_parts, z_part);
  });
}

int
stmg3_solver_set_space_comm(stmg3_solver *s, const stmg_comm_space_ops *ops)
{
  return guarded([&] {
    STMG_NVTX("stmg3_solver_set_space_comm");
    if (!s)
      throw std::invalid_argument("null solver");
    if (ops)
      {
        if (ops->parts != s->zparts || ops->part != s->zpart || !ops->exchange_planes || !ops->allreduce_sum ||
            !ops->allgather)
          throw std::invalid_argument("space communicator does not match the solver's z partition");
        s->sops = *ops;
        s->has_space = true;
      }
    else
      s->has_space = false;
  });
}

int
stmg3_plan_levels(int nx, int ny, int nz, int r, int k, int n_hcoarse, int time_coarsen, int k_min, int64_t *out)
{
  return guarded([&] {
    STMG_NVTX("stmg3_plan_levels");
    if (!out)
      throw std::invalid_argument("null argument");
    Level3Spec f;
    f.nx = nx;
    f.ny = ny;
    f.nz = nz;
    f.r = r;
    f.k = k;
    const std::vector<PlanLevel3> d = plan3(f, n_hcoarse, time_coarsen, k_min);
    out[0] = static_cast<int64_t>(d.size());
    for (size_t i = 0; i < d.size(); ++i) // coarse first, as stmg3_solver_info
      {
        const PlanLevel3 &e = d[d.size() - 1 - i];
        int64_t *o = out + 1 + 7 * i;
        o[0] = e.s.nx;
        o[1] = e.s.ny;
        o[2] = e.s.nz;
        o[3] = e.s.r;
        o[4] = e.s.k;
        o[5] = e.tsh;
        o[6] = e.s.isz();
      }
  });
}

int
stmg3_solver_destroy(stmg3_solver *s)
{
  delete s;
  return STMG_OK;
}

int
stmg3_solver_info(const stmg3_solver *s, int64_t *out)
{
  return guarded([&] {
    STMG_NVTX("stmg3_solver_info");
    out[0] = static_cast<int64_t>(s->levels.size());
    for (size_t l = 0; l < s->levels.size(); ++l)
      {
        const Level3Spec &sp = s->levels[l]->level->spec;
        int64_t *o = out + 1 + 7 * l;
        o[0] = sp.nx;
        o[1] = sp.ny;
        o[2] = sp.nz;
        o[3] = sp.r;
        o[4] = sp.k;
        o[5] = s->levels[l]->tshift;
        o[6] = sp.isz();
      }
  });
}

stmg3_level *
stmg3_solver_level(stmg3_solver *s, int l)
{
  if (!s || l < 0 || l >= static_cast<int>(s->levels.size()))
    return nullptr;
  return s->levels[l]->level.get();
}

int
stmg3_solver_set_krylov(stmg3_solver *s, int orthogonalization)
{
  return guarded([&] {
    if (!s)
      throw std::invalid_argument("stmg3_solver_set_krylov: null solver");
    if (orthogonalization != STMG_ORTHO_MGS && orthogonalization != STMG_ORTHO_CGS2)
      throw std::invalid_argument("stmg3_solver_set_krylov: unknown orthogonalization");
    s->ortho = orthogonalization;
  });
}

int
stmg3_solver_set_comm(stmg3_solver *s, const stmg_comm_ops *ops)
{
  return guarded([&] {
    STMG_NVTX("stmg3_solver_set_comm");
    if (ops)
      {
        if (ops->world < 1 || ops->rank < 0 || ops->rank >= ops->world || !ops->exchange_halo ||
            !ops->allreduce_sum || !ops->allgather)
          throw std::invalid_argument("invalid communicator");
        s->comm = *ops;
        s->has_comm = true;
      }
    else
      s->has_comm = false;
  });
}

int
stmg3_restrict_residual(stmg3_solver *s, int l, const double *fine, double *coarse, int nc, int project)
{
  return guarded([&] {
    STMG_NVTX("stmg3_restrict_residual");
    if (l < 1 || l >= static_cast<int>(s->levels.size()))
      throw std::invalid_argument("level out of range");
    s->restrict_residual(l, fine, coarse, nc, project != 0);
  });
}

int
stmg3_prolongate_correction(stmg3_solver *s, int l, const double *coarse, double *fine, int nc, int project,
                            int accumulate)
{
  return guarded([&] {
    STMG_NVTX("stmg3_prolongate_correction");
    if (l < 1 || l >= static_cast<int>(s->levels.size()))
      throw std::invalid_argument("level out of range");
    s->prolongate_correction(l, coarse, fine, nc, project != 0, accumulate != 0);
  });
}

int
stmg3_coarse_forward(stmg3_solver *s, const double *b, double *x, int n)
{
  return guarded([&] { s->coarse_forward(b, x, n); });
}

int
stmg3_vcycle_all_at_once(stmg3_solver *s, const double *b, double *x, int n)
{
  return guarded([&] {
    STMG_NVTX("stmg3_vcycle_all_at_once");
    s->check_slab(n);
    s->cycle(static_cast<int>(s->levels.size()) - 1, b, x, n);
  });
}

int
stmg3_solve_all_at_once(stmg3_solver *s, const double *F, double *X, int n, const double *v_init, int *iterations,
                        double *history, int history_cap)
{
  return guarded([&] { s->solve(F, X, n, v_init, iterations, history, history_cap); });
}

} // extern "C"
