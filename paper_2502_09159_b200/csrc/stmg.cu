// C ABI (include/stmg_b200.h) and host orchestration of the B200 hp-STMG
// path: levels, smoother colour sweeps, V-cycle, FGMRES and time marching.
// Mirrors the reference's operator/smoother/transfer/solver interfaces
// (st_operator.hpp, vanka.hpp, transfer.hpp, solver.hpp) on device vectors.
#include "../../include/stmg_b200.h"
#include "kernels.hpp"
#include "setup.hpp"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

using namespace stmg_b200;

#include "krylov.hpp"
#include "runtime.hpp"

using namespace stmg_rt;

// ================================================================ level
struct stmg_level
{
  stmg_ctx *ctx = nullptr;
  LevelSpec spec;
  LevelConsts consts{};
  DevGeom geom{};
  int smoother_kind = STMG_SMOOTHER_NONE;
  // Vanka
  std::vector<DevArray<long long>> cls_rel;
  std::vector<DevArray<double>> cls_weight, cls_inverse;
  DevArray<DevPatchClass> classes;
  DevArray<VankaBatch> batches;
  DevArray<long long> vel_anchor, pre_anchor;
  std::vector<int> colour_first, colour_count;
  // super-cell sweeps (DMMA path): 4 passes, block b of pass s runs items
  // [pass_ptr[s][b], pass_ptr[s][b+1])
  struct SuperSet
  {
    std::vector<DevArray<int>> pass_ptr;
    std::vector<int> pass_blocks;
    DevArray<VankaBatch> items;
    DevArray<long long> va, pa;
    // pipelined tensor-core tiles (vanka_tc.cu): per pass, block b runs
    // tiles [tile_ptr[b], tile_ptr[b+1]); each tile <= 32 (patch, interval)
    // columns of one class and one colour sub-phase
    int ng_full = 1;
    std::vector<DevArray<int>> tile_ptr;
    std::vector<int> tile_blocks;
    DevArray<VankaTile> tiles;
  };
  bool super = false;
  SuperSet sup[3]; // intervals per block: [0] 16, [2] 8 (slabs), [1] 1 (time marching)
  int max_nt = 0;
  // time-diagonalised patch inverses (vanka_fac_kernel), DG(k >= 2) levels
  bool factored = false;
  FacParams fac{};
  std::vector<DevArray<double>> cls_fac;
  std::uint64_t factored_matrix_elements = 0;
  int n_classes = 0;
  std::uint64_t total_matrix_elements = 0;
  // scratch
  DevArray<double> work, zeros, host_in, host_out, host_prev, proj, err_part, err_out;
  // host-buffer entry points: staging of stmg_vmult_host (host_in / host_out /
  // host_prev_v) and stmg_smooth_step_host (host_b / host_u / host_prev), and
  // per set the events that free its input (kernels done) and output (D2H
  // done) staging for the next call, so *_async calls can queue back to back
  DevArray<double> host_b, host_u, host_prev_v;
  cudaEvent_t ev_in_free[2] = {nullptr, nullptr}, ev_out_free[2] = {nullptr, nullptr};
  ~stmg_level()
  {
    for (cudaEvent_t e : {ev_in_free[0], ev_in_free[1], ev_out_free[0], ev_out_free[1]})
      if (e)
        cudaEventDestroy(e);
  }
  /// Before a host-buffer call of set k: wait until the previous call of the
  /// same set released its staging.
  void
  host_begin(int k)
  {
    if (!ev_in_free[k])
      {
        check(cudaEventCreateWithFlags(&ev_in_free[k], cudaEventDisableTiming), "event");
        check(cudaEventCreateWithFlags(&ev_out_free[k], cudaEventDisableTiming), "event");
        check(cudaEventRecord(ev_in_free[k], ctx->stream), "event");
        check(cudaEventRecord(ev_out_free[k], ctx->d2h), "event");
      }
    check(cudaStreamWaitEvent(ctx->h2d, ev_in_free[k], 0), "wait");
    check(cudaStreamWaitEvent(ctx->stream, ev_out_free[k], 0), "wait");
  }
  void
  host_end(int k, bool sync)
  {
    check(cudaEventRecord(ev_in_free[k], ctx->stream), "event");
    check(cudaEventRecord(ev_out_free[k], ctx->d2h), "event");
    if (sync)
      check(cudaStreamSynchronize(ctx->d2h), "sync");
  }
  // built-in problem tables (problems.cu), built on first use
  ProblemTables ptab{};
  bool ptab_ready = false;
  const ProblemTables &
  problem_tab()
  {
    if (!ptab_ready)
      {
        ptab = problem_tables(spec);
        ptab_ready = true;
      }
    return ptab;
  }

  /// u_p <- u_p - mean per slot (PressureSpace::project_mean_zero)
  void
  project(double *x, int n)
  {
    proj.resize(project_scratch_doubles(geom, n));
    check(launch_project_mean_zero(geom, x, n, proj.p, ctx->stream), "project");
    ctx->count(2);
  }

  void
  vmult(const double *x, const double *b, double *y, int n, const double *xprev0, int coupled, int mode)
  {
    check(launch_vmult(spec.r, spec.S(), consts, x, b, y, n, xprev0, coupled, mode, ctx->stream), "vmult");
    ctx->count();
  }

  /// u += omega * sum over colours of the patch corrections of residual r.
  void
  vanka(const double *r, double *u, int n, double omega)
  {
    if (smoother_kind == STMG_SMOOTHER_NONE)
      throw std::invalid_argument("level has no smoother");
    if (super)
      {
        // widest interval group that the launch fills: 16, 8 or 1 per block
        const SuperSet &ss = sup[n >= 16 ? 0 : (n >= 8 ? 2 : 1)];
        if (!ss.tile_ptr.empty() && factored)
          {
            for (size_t sc = 0; sc < ss.tile_ptr.size(); ++sc)
              if (ss.tile_blocks[sc] > 0)
                {
                  check(launch_vanka_fac(classes.p, ss.tiles.p, ss.va.p, ss.pa.p, ss.tile_ptr[sc].p,
                                         ss.tile_blocks[sc], ss.ng_full, fac, r, u, spec.isz(), n, omega,
                                         ctx->stream),
                        "vanka_fac");
                  ctx->count();
                }
            return;
          }
        if (!ss.tile_ptr.empty())
          {
            for (size_t sc = 0; sc < ss.tile_ptr.size(); ++sc)
              if (ss.tile_blocks[sc] > 0)
                {
                  check(launch_vanka_tc(classes.p, ss.tiles.p, ss.va.p, ss.pa.p, ss.tile_ptr[sc].p,
                                        ss.tile_blocks[sc], ss.ng_full, max_nt, r, u, spec.isz(), n, omega,
                                        ctx->stream),
                        "vanka_tc");
                  ctx->count();
                }
            return;
          }
        for (size_t sc = 0; sc < ss.pass_ptr.size(); ++sc)
          if (ss.pass_blocks[sc] > 0)
            {
              check(launch_vanka_colour(classes.p, ss.items.p, ss.pass_ptr[sc].p, ss.pass_blocks[sc], max_nt, ss.va.p,
                                        ss.pa.p, r, u, spec.isz(), n, omega, ctx->stream),
                    "vanka");
              ctx->count();
            }
        return;
      }
    for (size_t c = 0; c < colour_first.size(); ++c)
      if (colour_count[c] > 0)
        {
          check(launch_vanka_colour(classes.p, batches.p + colour_first[c], nullptr, colour_count[c], max_nt,
                                    vel_anchor.p, pre_anchor.p, r, u, spec.isz(), n, omega, ctx->stream),
                "vanka");
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
  smooth_step(const double *b, double *u, double omega, int n, const double *xprev, int coupled, double *work_buf,
              bool u_is_zero = false)
  {
    if (!(omega > 0.0 && omega <= 1.0))
      throw std::invalid_argument("smooth_step: omega must be in (0, 1]");
    double *r = work_buf ? work_buf : scratch(n);
    if (u_is_zero && !coupled)
      check(cudaMemcpyAsync(r, b, sizeof(double) * spec.isz() * n, cudaMemcpyDeviceToDevice, ctx->stream),
            "copy"); // b - D*0 == b exactly
    else
      vmult(u, b, r, n, xprev, coupled, 1);
    vanka(r, u, n, omega);
  }
};

namespace
{
void
build_level(stmg_level &L)
{
  const LevelSpec &s = L.spec;
  if (s.r < 1 || s.r > 4)
    throw std::invalid_argument("stmg_level: r must be in 1..4");
  if (s.k < 0 || s.k > 4)
    throw std::invalid_argument("stmg_level: k must be in 0..4");
  if (s.nx < 1 || s.ny < 1)
    throw std::invalid_argument("stmg_level: need at least one cell per direction");
  if (s.isz() >= (1ll << 31))
    throw std::invalid_argument("stmg_level: one interval must hold fewer than 2^31 dofs (int32 patch offsets)");
  if (!(s.tau > 0.0))
    throw std::invalid_argument("stmg_level: tau must be positive");
  L.consts = make_level_consts(s);
  L.geom = DevGeom{s.nx, s.ny, s.gx(), s.gy(), s.S(), s.np(), s.nsc(), s.mv(), s.mp(), s.isz(), s.hx, s.hy};
  if (L.smoother_kind == STMG_SMOOTHER_NONE)
    return;
  const PatchSet ps = build_patches(s, L.smoother_kind == STMG_SMOOTHER_CELL ? PatchKind::cell : PatchKind::vertex_star);
  L.n_classes = static_cast<int>(ps.classes.size());
  L.total_matrix_elements = ps.total_matrix_elements;
  std::vector<DevPatchClass> dc(ps.classes.size());
  L.cls_rel.resize(ps.classes.size());
  L.cls_weight.resize(ps.classes.size());
  L.cls_inverse.resize(ps.classes.size());
  L.cls_fac.resize(ps.classes.size());
  for (size_t i = 0; i < ps.classes.size(); ++i)
    {
      const PatchClass &pc = ps.classes[i];
      L.cls_rel[i].upload(pc.rel);
      if (ps.factored)
        L.cls_fac[i].upload(pc.fac_inv);
      L.cls_weight[i].upload(pc.weight);
      L.cls_inverse[i].upload(pc.inverse);
      dc[i] = DevPatchClass{pc.n_t, pc.n_vel, L.cls_rel[i].p, L.cls_weight[i].p, L.cls_inverse[i].p,
                            pc.n_s, pc.n_vs, ps.factored ? L.cls_fac[i].p : nullptr};
      L.max_nt = std::max(L.max_nt, pc.n_t);
    }
  L.classes.upload(dc);
  // Time-diagonalised inverses are opt-in (STMG_VANKA_FACTORED=1): for DG(2)
  // they cut the DMMA work to 0.61x but the slot-mixing stages add 38% more
  // instructions, so the C2 update measured 5.85 ms against 5.69 ms dense
  // (DESIGN.md 3.2). The dense kernel is the default.
  const char *fac_env = std::getenv("STMG_VANKA_FACTORED");
  if (ps.factored && vanka_fac_supported(s.S(), ps.n_sp) && fac_env && fac_env[0] == '1')
    {
      L.factored = true;
      L.factored_matrix_elements = ps.factored_matrix_elements;
      FacParams &F = L.fac;
      F.S = s.S();
      F.nsp = ps.n_sp;
      for (int a = 0; a < F.S; ++a)
        for (int b = 0; b < F.S; ++b)
          {
            F.V[a * kMaxS + b] = ps.eig.V[a * F.S + b];
            F.W[a * kMaxS + b] = ps.eig.W[a * F.S + b];
          }
      for (int w = 0; w < 16; ++w)
        {
          const int row0 = 8 * w;
          F.kbase[w] = 0;
          F.ksteps[w] = 0;
          if (row0 >= F.S * F.nsp)
            continue;
          const int coord = row0 / F.nsp;
          for (size_t b = 0; b < ps.eig.blk_c0.size(); ++b)
            if (coord >= ps.eig.blk_c0[b] && coord < ps.eig.blk_c0[b] + ps.eig.blk_sz[b])
              {
                F.kbase[w] = ps.eig.blk_c0[b] * F.nsp;
                F.ksteps[w] = ps.eig.blk_sz[b] * F.nsp / 4;
              }
        }
    }
  std::vector<VankaBatch> batches;
  std::vector<long long> va, pa;
  const int cols = vanka_cols_per_batch();
  for (const auto &col : ps.colours)
    {
      L.colour_first.push_back(static_cast<int>(batches.size()));
      size_t i = 0;
      while (i < col.size())
        {
          VankaBatch b{col[i].cls, static_cast<int>(va.size()), 0};
          while (i < col.size() && col[i].cls == b.cls && b.count < cols)
            {
              va.push_back(patch_vel_anchor(s, ps.kind, col[i].ax, col[i].ay));
              pa.push_back(patch_pre_anchor(s, ps.kind, col[i].ax, col[i].ay));
              ++b.count;
              ++i;
            }
          batches.push_back(b);
        }
      L.colour_count.push_back(static_cast<int>(batches.size()) - L.colour_first.back());
    }
  L.batches.upload(batches);
  L.vel_anchor.upload(va);
  L.pre_anchor.upload(pa);

  // Super-cell sweeps for the DMMA path: a super-cell holds P x P patch
  // anchors (one of each colour, P = colour period); a block processes the
  // P^2 colours of a row of super-cells one after the other, separated by
  // block barriers, so its data stays cache-resident across colours.
  // Super-cells are 2x2-coloured over 4 launches: same-launch super-cells
  // are a full super-cell apart and never share a dof.
  if (L.max_nt <= 128)
    {
      const int P = ps.kind == PatchKind::cell ? 2 : 3;
      const int nax = ps.kind == PatchKind::cell ? s.nx : s.nx + 1;
      const int nay = ps.kind == PatchKind::cell ? s.ny : s.ny + 1;
      std::vector<int> cls_of(static_cast<size_t>(nax) * nay, -1);
      for (const auto &col : ps.colours)
        for (const auto &e : col)
          cls_of[static_cast<size_t>(e.ay) * nax + e.ax] = e.cls;
      const int nsx = (nax + P - 1) / P, nsy = (nay + P - 1) / P;
      // B super-cells (one contiguous strip) per block: few for many
      // intervals (columns = B x 16 intervals), twice as many for 8-interval
      // slabs, up to 32 for time marching (one interval per block).
      for (int set = 0; set < 3; ++set)
        {
#ifndef STMG_STRIP_CELL
#define STMG_STRIP_CELL 8 // measured: C2 Vanka 5.60 (4) -> 5.33 ms (8); 16 overflows the staged tile table
#endif
#ifndef STMG_STRIP_VSP
#define STMG_STRIP_VSP 8 // with the 48-tile staging: C4 vertex stars 12.03 -> 11.79 ms
#endif
          // super-cells per strip with 16 intervals per block; 8-interval
          // slabs use twice as many (same columns per colour sub-phase)
          // narrower strips on mid-size levels so a pass still has ~2 blocks
          // per SM (strips per pass ~ nwx/2 * nsy/2; 16-interval blocks are
          // counted with 4 interval groups)
          int B0 = P == 2 ? STMG_STRIP_CELL : STMG_STRIP_VSP;
          {
            const int ngroups = set == 0 ? 4 : 1, mult = set == 2 ? 2 : 1;
            while (B0 > 1)
              {
                const long long wx = (nax + P * B0 * mult - 1) / (P * B0 * mult);
                if ((wx + 1) / 2 * ((nsy + 1) / 2) * ngroups >= 2 * stmg_b200::device_sm_count())
                  break;
                B0 /= 2;
              }
          }
          // time-marching set: 32 super-cells per block, fewer on small levels
          // so that a pass still spreads over ~2 blocks per SM (latency)
          const long long per_pass = std::max(1LL, static_cast<long long>(nsx) * nsy / 4);
          const int B1 = static_cast<int>(std::min(32LL, std::max(1LL, per_pass / (2LL * stmg_b200::device_sm_count()))));
          const int B = set == 0 ? B0 : (set == 2 ? 2 * B0 : B1);
          stmg_level::SuperSet &ss = L.sup[set];
          std::vector<VankaBatch> items;
          std::vector<int> item_phase; // colour sub-phase (qy, qx) of each item
          std::vector<long long> sva, spa;
          ss.pass_ptr.resize(4);
          ss.pass_blocks.assign(4, 0);
          std::vector<std::vector<int>> host_ptr(4);
          for (int sc = 0; sc < 4; ++sc)
            {
              std::vector<int> ptr{static_cast<int>(items.size())};
              // A block owns one contiguous strip of B super-cells (P*B anchors
              // wide, P high); strips are 2x2-coloured over the 4 passes, so
              // same-pass strips are a full strip apart (no shared dof) and
              // each block reads contiguous node runs (DRAM bursts fully used).
              const int nwx = (nax + P * B - 1) / (P * B);
              for (int SY = sc / 2; SY < nsy; SY += 2)
                {
                  for (int WX = sc % 2; WX < nwx; WX += 2)
                    {
                      for (int qy = 0; qy < P; ++qy)
                        for (int qx = 0; qx < P; ++qx)
                          {
                            std::vector<std::pair<int, std::pair<int, int>>> anchors; // (cls, (ax, ay))
                            for (int w = 0; w < B; ++w)
                              {
                                const int ax = P * B * WX + P * w + qx, ay = P * SY + qy;
                                if (ax < nax && ay < nay)
                                  anchors.push_back({cls_of[static_cast<size_t>(ay) * nax + ax], {ax, ay}});
                              }
                            std::stable_sort(anchors.begin(), anchors.end(),
                                             [](const auto &x, const auto &y) { return x.first < y.first; });
                            size_t i = 0;
                            while (i < anchors.size())
                              {
                                VankaBatch it{anchors[i].first, static_cast<int>(sva.size()), 0};
                                while (i < anchors.size() && anchors[i].first == it.cls)
                                  {
                                    sva.push_back(patch_vel_anchor(s, ps.kind, anchors[i].second.first,
                                                                   anchors[i].second.second));
                                    spa.push_back(patch_pre_anchor(s, ps.kind, anchors[i].second.first,
                                                                   anchors[i].second.second));
                                    ++it.count;
                                    ++i;
                                  }
                                items.push_back(it);
                                item_phase.push_back(qy * P + qx);
                              }
                          }
                      ptr.push_back(static_cast<int>(items.size()));
                    }
                }
              ss.pass_blocks[sc] = static_cast<int>(ptr.size()) - 1;
              ss.pass_ptr[sc].upload(ptr);
              host_ptr[sc] = std::move(ptr);
            }
          ss.items.upload(items);
          ss.va.upload(sva);
          ss.pa.upload(spa);

          // expand the items into tensor-core tiles of <= 32 columns
          // (patch-major, interval-minor; ng_full intervals per block)
          ss.ng_full = set == 0 ? 16 : (set == 2 ? 8 : 1);
          const int tc = vanka_tc_cols();
          bool tc_ok = true;
          std::vector<VankaTile> tiles;
          ss.tile_ptr.resize(4);
          ss.tile_blocks.assign(4, 0);
          for (int sc = 0; sc < 4; ++sc)
            {
              const std::vector<int> &hptr = host_ptr[sc];
              std::vector<int> tptr{static_cast<int>(tiles.size())};
              for (int blk = 0; blk < ss.pass_blocks[sc]; ++blk)
                {
                  for (int it = hptr[blk]; it < hptr[blk + 1]; ++it)
                    {
                      const VankaBatch &item = items[it];
                      const int ncols = item.count * ss.ng_full;
                      for (int c0 = 0; c0 < ncols; c0 += tc)
                        tiles.push_back(VankaTile{item.cls, std::min(tc, ncols - c0), item.first, c0, item_phase[it]});
                    }
                  tptr.push_back(static_cast<int>(tiles.size()));
                  if (tptr.back() - tptr[tptr.size() - 2] > vanka_tc_max_tiles())
                    tc_ok = false; // block too long for the staged tile data
                }
              ss.tile_blocks[sc] = ss.pass_blocks[sc];
              ss.tile_ptr[sc].upload(tptr);
            }
          ss.tiles.upload(tiles);
          if (!tc_ok)
            ss.tile_ptr.clear(); // use the item-based DMMA kernel instead
        }
      L.super = true;
    }
}
} // namespace

// ================================================================ solver
namespace
{
struct SolverLevel
{
  std::unique_ptr<stmg_level> level;
  TransferKind kind = TransferKind::identity;
  // transfer to the next coarser level (absent on level 0)
  DevArray<int> px_ptr, px_col, py_ptr, py_col, rx_ptr, rx_col, ry_ptr, ry_col, embed;
  DevArray<double> px_val, py_val, rx_val, ry_val, child;
  DevTransfer dt{};
  // V-cycle buffers (one interval, or a slab in all-at-once mode)
  DevArray<double> x, b, r, t, halo;
};
} // namespace

struct stmg_solver
{
  stmg_ctx *ctx = nullptr;
  HierarchyConfig cfg;
  int n_steps = 0;
  int nu1 = 1, nu2 = 1;
  double omega = 0.8;
  bool project_pressure = true;
  double rtol = 1e-8, atol = 1e-14;
  int max_iterations = 200;
  int ortho = stmg_krylov::kMGS; // Arnoldi orthogonalization (stmg_solver_set_krylov)
  std::vector<std::unique_ptr<SolverLevel>> levels;
  DevArray<double> coarse_inv;
  DevArray<long long> coarse_pinned;
  int n_pinned = 0, coarse_n = 0;
  // Krylov workspace
  std::vector<std::unique_ptr<DevArray<double>>> V, Z;
  DevArray<double> w, scal, part, rhs, vprev;
  std::vector<double> hist;

  stmg_level &fine() { return *levels.back()->level; }

  // ---- time-slab communicator (all-at-once mode only; see stmg_comm_ops)
  stmg_comm_ops comm{};
  bool has_comm = false;
  int
  rank() const
  {
    return has_comm ? comm.rank : 0;
  }
  int
  world() const
  {
    return has_comm ? comm.world : 1;
  }

  // Coupled application on the slab at level l: y = A x (mode 0) or
  // y = b - A x (mode 1), A with the jump coupling (Eq. GloSys). With a
  // communicator the halo (slot-k velocity of the previous rank's last
  // interval) travels on a side stream while intervals 1..nI-1, whose
  // predecessor is local, are computed; interval 0 waits for the halo.
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_x = nullptr, ev_h = nullptr;
  void
  coupled_vmult(int l, const double *x, const double *b, double *y, int nI, int mode)
  {
    stmg_level &L = *levels[l]->level;
    if (world() == 1)
      {
        L.vmult(x, b, y, nI, nullptr, 1, mode);
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
    check(cudaEventRecord(ev_x, ctx->stream), "event"); // x final, previous use of h done
    check(cudaStreamWaitEvent(comm_stream, ev_x, 0), "wait");
    const double *send = x + (nI - 1) * isz + (L.spec.S() - 1) * mv;
    if (comm.exchange_halo(comm.user, send, h.p, mv, comm_stream) != 0)
      throw std::runtime_error("comm: exchange_halo failed");
    check(cudaEventRecord(ev_h, comm_stream), "event");
    if (nI > 1) // interior intervals: predecessor is interval 0 of this slab
      L.vmult(x + isz, b ? b + isz : nullptr, y + isz, nI - 1, x + (L.spec.S() - 1) * mv, 1, mode);
    check(cudaStreamWaitEvent(ctx->stream, ev_h, 0), "wait");
    L.vmult(x, b, y, 1, rank() == 0 ? nullptr : h.p, 1, mode);
  }

  void
  allreduce(double *buf, int n)
  {
    if (world() > 1 && comm.allreduce_sum(comm.user, buf, n, ctx->stream) != 0)
      throw std::runtime_error("comm: allreduce_sum failed");
  }

  void
  restrict_residual(int l, const double *fine_v, double *coarse_v, bool project, int nI = 1)
  {
    SolverLevel &F = *levels[l];
    check(launch_restrict(F.dt, fine_v, coarse_v, nI, ctx->stream), "restrict");
    ctx->count(2);
    if (F.kind != TransferKind::identity && project)
      {
        levels[l - 1]->level->project(coarse_v, nI);
      }
  }

  void
  prolongate_correction(int l, const double *coarse_v, double *fine_v, bool project, bool accumulate, int nI = 1)
  {
    SolverLevel &F = *levels[l];
    const long long n = F.level->spec.isz() * nI;
    if (F.kind != TransferKind::identity && project)
      {
        // out = P c, zero constrained, project mean-zero, then (x +=) out
        F.t.resize(n);
        check(launch_prolongate(F.dt, coarse_v, F.t.p, nI, 0, ctx->stream), "prolongate");
        ctx->count(2);
        F.level->project(F.t.p, nI);
        if (accumulate)
          {
            check(launch_axpy(n, 1.0, nullptr, 1.0, F.t.p, fine_v, ctx->stream), "axpy");
            ctx->count();
          }
        else
          check(cudaMemcpyAsync(fine_v, F.t.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream), "copy");
      }
    else
      {
        check(launch_prolongate(F.dt, coarse_v, fine_v, nI, accumulate ? 1 : 0, ctx->stream), "prolongate");
        ctx->count(2);
      }
  }

  void
  coarse_solve(const double *b_v, double *x_v)
  {
    check(launch_coarse_solve(coarse_inv.p, coarse_pinned.p, n_pinned, coarse_n, b_v, x_v, ctx->stream), "coarse");
    ctx->count();
    levels[0]->level->project(x_v, 1);
  }

  // ---- all-at-once coarse solve: x_t = G b_t + H v_{t-1} with
  // G = P A^+ (pinned solve then mean-zero projection, solver.cpp:43-54) and
  // H = G C_c (the jump coupling of level 0, st_operator.cpp:409-421).
  DevArray<double> cf_G, cf_H, cf_B;
  int cf_mv = 0;
  bool cf_ready = false;

  void
  prepare_coarse_forward()
  {
    if (cf_ready)
      return;
    stmg_level &L0 = *levels[0]->level;
    const LevelSpec &sp = L0.spec;
    const int n = coarse_n, mv = static_cast<int>(sp.mv());
    std::vector<double> inv(static_cast<size_t>(n) * n);
    std::vector<long long> pin(n_pinned);
    check(cudaMemcpy(inv.data(), coarse_inv.p, sizeof(double) * inv.size(), cudaMemcpyDeviceToHost), "d2h");
    check(cudaMemcpy(pin.data(), coarse_pinned.p, sizeof(long long) * pin.size(), cudaMemcpyDeviceToHost), "d2h");
    for (long long q : pin) // pinned right-hand-side entries are ignored
      for (int i = 0; i < n; ++i)
        inv[static_cast<size_t>(i) * n + q] = 0.0;
    // mean-zero projection per slot: mode-0 pressure entries minus their
    // cell-area-weighted mean (dof_space.cpp:110-119; uniform cells)
    const int ncell = sp.nx * sp.ny;
    std::vector<double> G(inv);
    for (int a = 0; a < sp.S(); ++a)
      {
        const long long base = sp.S() * sp.mv() + a * sp.mp();
        for (int j = 0; j < n; ++j)
          {
            double mean = 0.0;
            for (int c = 0; c < ncell; ++c)
              mean += inv[static_cast<size_t>(base + static_cast<long long>(c) * sp.np()) * n + j];
            mean /= ncell;
            for (int c = 0; c < ncell; ++c)
              G[static_cast<size_t>(base + static_cast<long long>(c) * sp.np()) * n + j] -= mean;
          }
      }
    // C_c column by column: residual of x = 0 with unit previous velocity
    DevArray<double> e, out;
    e.resize(mv);
    out.resize(n);
    const double *zero = L0.zero_vector(1);
    std::vector<double> Cc(static_cast<size_t>(n) * mv);
    std::vector<double> col(n);
    const double one = 1.0;
    for (int j = 0; j < mv; ++j)
      {
        check(cudaMemsetAsync(e.p, 0, sizeof(double) * mv, ctx->stream), "memset");
        check(cudaMemcpyAsync(e.p + j, &one, sizeof(double), cudaMemcpyHostToDevice, ctx->stream), "h2d");
        L0.vmult(zero, zero, out.p, 1, e.p, 1, 1);
        check(launch_zero_constrained(L0.geom, out.p, 1, ctx->stream), "zero");
        check(cudaMemcpyAsync(col.data(), out.p, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream), "d2h");
        check(cudaStreamSynchronize(ctx->stream), "sync");
        for (int i = 0; i < n; ++i)
          Cc[static_cast<size_t>(i) * mv + j] = col[i];
      }
    std::vector<double> H(static_cast<size_t>(n) * mv, 0.0);
    for (int i = 0; i < n; ++i)
      for (int q = 0; q < n; ++q)
        {
          const double g = G[static_cast<size_t>(i) * n + q];
          if (g != 0.0)
            for (int j = 0; j < mv; ++j)
              H[static_cast<size_t>(i) * mv + j] += g * Cc[static_cast<size_t>(q) * mv + j];
        }
    cf_G.upload(G);
    cf_H.upload(H);
    cf_mv = mv;
    cf_ready = true;
  }

  void
  coarse_forward(const double *b_v, double *x_v, int nI)
  {
    prepare_coarse_forward();
    const LevelSpec &sp = levels[0]->level->spec;
    const long long per = static_cast<long long>(coarse_n) * nI;
    const double *B = b_v;
    if (world() > 1)
      {
        cf_B.resize(per * world());
        if (comm.allgather(comm.user, b_v, cf_B.p, per, ctx->stream) != 0)
          throw std::runtime_error("comm: allgather failed");
        B = cf_B.p;
      }
    check(launch_coarse_forward(cf_G.p, cf_H.p, coarse_n, cf_mv, (sp.S() - 1) * sp.mv(), B, nI * world(),
                                nI * rank(), nI, x_v, ctx->stream),
          "coarse_forward");
    ctx->count();
  }

  // VCycle::cycle (solver.cpp:69-93); writes the result into x_v. With aao,
  // the cycle acts on nI intervals of the all-at-once system: residuals carry
  // the jump coupling (halo from the previous rank), the coarse solve is the
  // block forward substitution.
  void
  cycle(int l, const double *b_v, double *x_v, int nI = 1, bool aao = false)
  {
    STMG_NVTX("vcycle L%d (%d intervals)", l, nI);
    if (l == 0)
      {
        if (aao)
          coarse_forward(b_v, x_v, nI);
        else
          coarse_solve(b_v, x_v);
        return;
      }
    SolverLevel &S = *levels[l];
    stmg_level &L = *S.level;
    const long long isz = L.spec.isz() * nI;
    S.r.resize(isz);
    check(cudaMemsetAsync(x_v, 0, sizeof(double) * isz, ctx->stream), "memset");
    // smoothing step: residual (coupled in all-at-once mode), then Vanka
    const auto smooth = [&](bool first) {
      STMG_NVTX("L%d smooth", l);
      if (first) // x = 0 on every rank before the first sweep: b - A 0 = b exactly
        L.smooth_step(b_v, x_v, omega, nI, nullptr, 0, S.r.p, true);
      else if (aao)
        {
          coupled_vmult(l, x_v, b_v, S.r.p, nI, 1);
          L.vanka(S.r.p, x_v, nI, omega);
        }
      else
        L.smooth_step(b_v, x_v, omega, nI, nullptr, 0, S.r.p);
    };
    for (int s = 0; s < nu1; ++s)
      smooth(s == 0);
    if (aao)
      coupled_vmult(l, x_v, b_v, S.r.p, nI, 1);
    else
      L.vmult(x_v, b_v, S.r.p, nI, nullptr, 0, 1);
    SolverLevel &C = *levels[l - 1];
    const long long csz = C.level->spec.isz() * nI;
    C.b.resize(csz);
    C.x.resize(csz);
    {
      STMG_NVTX("L%d restrict", l);
      restrict_residual(l, S.r.p, C.b.p, project_pressure, nI);
    }
    cycle(l - 1, C.b.p, C.x.p, nI, aao);
    {
      STMG_NVTX("L%d prolongate", l);
      prolongate_correction(l, C.x.p, x_v, project_pressure, true, nI);
    }
    for (int s = 0; s < nu2; ++s)
      smooth(false);
  }

  void
  vcycle(const double *b_v, double *x_v)
  {
    cycle(static_cast<int>(levels.size()) - 1, b_v, x_v);
  }

  // ---- CUDA graph of the whole V-cycle for launch-bound (small) problems:
  // replayed on fixed in/out buffers; captured on the second call with a
  // given shape, after an uncaptured call has allocated every workspace.
  cudaGraphExec_t vc_exec = nullptr;
  int vc_nI = -1, vc_calls = 0;
  bool vc_aao = false;
  int64_t vc_launches = 0;
  uint64_t vc_gen = 0;
  cudaStream_t vc_stream = nullptr;
  DevArray<double> vc_in, vc_out;
  static constexpr long long kGraphMaxDofs = 2'000'000;

  void
  drop_graph()
  {
    if (vc_exec)
      cudaGraphExecDestroy(vc_exec);
    vc_exec = nullptr;
    vc_calls = 0;
  }

  void
  precondition(const double *b_v, double *x_v, int nI, bool aao)
  {
    const int top = static_cast<int>(levels.size()) - 1;
    const long long n = fine().spec.isz() * nI;
    if (n > kGraphMaxDofs || world() > 1)
      {
        cycle(top, b_v, x_v, nI, aao);
        return;
      }
    vc_in.resize(n);
    vc_out.resize(n);
    if (nI != vc_nI || aao != vc_aao || (vc_exec && vc_gen != g_reallocs.load()))
      {
        drop_graph();
        vc_nI = nI;
        vc_aao = aao;
      }
    if (!vc_exec && vc_calls++ == 0)
      {
        cycle(top, b_v, x_v, nI, aao); // first call: allocates the workspaces
        return;
      }
    if (!vc_exec)
      {
        const int64_t before = ctx->launches;
        cudaGraph_t g = nullptr;
        // the context stream may be the legacy default stream, which cannot
        // be captured: record on a private stream (the replay goes to ctx->stream)
        if (!vc_stream)
          check(cudaStreamCreateWithFlags(&vc_stream, cudaStreamNonBlocking), "stream");
        cudaStream_t user = ctx->stream;
        check(cudaStreamSynchronize(user), "sync");
        ctx->stream = vc_stream;
        check(cudaStreamBeginCapture(vc_stream, cudaStreamCaptureModeRelaxed), "capture");
        try
          {
            cycle(top, vc_in.p, vc_out.p, nI, aao);
          }
        catch (...)
          {
            cudaStreamEndCapture(vc_stream, &g);
            ctx->stream = user;
            if (g)
              cudaGraphDestroy(g);
            throw;
          }
        ctx->stream = user;
        check(cudaStreamEndCapture(vc_stream, &g), "capture");
        const cudaError_t e = cudaGraphInstantiate(&vc_exec, g, 0);
        cudaGraphDestroy(g);
        check(e, "graph instantiate");
        vc_launches = ctx->launches - before;
        ctx->launches = before;
        vc_gen = g_reallocs.load();
      }
    check(cudaMemcpyAsync(vc_in.p, b_v, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream), "copy");
    check(cudaGraphLaunch(vc_exec, ctx->stream), "graph launch");
    ctx->count(static_cast<int>(vc_launches));
    check(cudaMemcpyAsync(x_v, vc_out.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream), "copy");
  }

  ~stmg_solver()
  {
    drop_graph();
    if (vc_stream)
      cudaStreamDestroy(vc_stream);
    if (comm_stream)
      cudaStreamDestroy(comm_stream);
    if (ev_x)
      cudaEventDestroy(ev_x);
    if (ev_h)
      cudaEventDestroy(ev_h);
  }

  double
  dot(const double *a, const double *b, long long n, int slot)
  {
    check(launch_dot(a, b, n, part.p, scal.p + slot, ctx->stream), "dot");
    ctx->count(2);
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

  // gmres (solver.cpp:95-202), x0 = 0, preconditioner = V-cycle. With aao,
  // the operator and V-cycle are the all-at-once ones over nI intervals and
  // every inner product is summed over the ranks of the time-slab partition.
  int
  gmres(const double *b_v, double *x_v, int *iterations, double *history, int history_cap, int nI = 1,
        bool aao = false)
  {
    stmg_level &L = fine();
    const int top = static_cast<int>(levels.size()) - 1;
    const long long n = L.spec.isz() * nI;
    w.resize(n);
    part.resize(stmg_krylov::part_doubles());
    scal.resize(2 * (max_iterations + 2));
    hist.clear();
    const double norm_b = std::sqrt(dot(b_v, b_v, n, 0));
    const double tol = std::max(rtol * norm_b, atol);
    // r = b - A*0 = b
    const double beta = norm_b;
    hist.push_back(beta);
    check(cudaMemsetAsync(x_v, 0, sizeof(double) * n, ctx->stream), "memset");
    int iters = 0;
    bool converged = false;
    if (beta <= tol)
      converged = true;
    else
      {
        const int m = max_iterations;
        std::vector<double> H(static_cast<size_t>(m + 1) * m, 0.0), g(m + 1, 0.0), cs(m), sn(m);
        g[0] = beta;
        DevArray<double> &v0 = basis(V, 0, n);
        check(cudaMemcpyAsync(v0.p, b_v, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream), "copy");
        check(launch_scale(n, 1.0 / beta, v0.p, ctx->stream), "scale");
        ctx->count();
        int j = 0;
        std::vector<double> hcol(m + 2);
        for (; j < m; ++j)
          {
            STMG_NVTX("fgmres it %d", j);
            DevArray<double> &zj = basis(Z, j, n);
            precondition(V[j]->p, zj.p, nI, aao);
            if (aao)
              coupled_vmult(top, zj.p, nullptr, w.p, nI, 0);
            else
              L.vmult(zj.p, nullptr, w.p, nI, nullptr, 0, 0);
            // Arnoldi: MGS (the reference's, solver.cpp:146-152) or CGS2
            // (two batched all-reduces per iteration), krylov.hpp
            const double h_next = stmg_krylov::orthogonalize(
              ortho, V, j, w.p, n, part.p, scal.p, hcol, [&](double *buf, int cnt) { allreduce(buf, cnt); }, ctx);
            const bool breakdown = !(h_next > 1e-300);
            for (int i = 0; i <= j; ++i)
              H[static_cast<size_t>(j) * (m + 1) + i] = hcol[i];
            auto Hc = [&](int i) -> double & { return H[static_cast<size_t>(j) * (m + 1) + i]; };
            for (int i = 0; i < j; ++i)
              {
                const double t = cs[i] * Hc(i) + sn[i] * Hc(i + 1);
                Hc(i + 1) = -sn[i] * Hc(i) + cs[i] * Hc(i + 1);
                Hc(i) = t;
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
        if (iters > 0)
          {
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
      }
    if (iterations)
      *iterations = iters;
    for (int i = 0; history && i < history_cap && i < static_cast<int>(hist.size()); ++i)
      history[i] = hist[i];
    if (!converged)
      throw std::runtime_error("gmres: not converged within max_iterations");
    return iters;
  }

  // All-at-once solve of A X = F on a slab (Eq. GloSys).
  // v_init enters the slab's first interval like time_march's v_prev
  // (solver.cpp:251-268): F_0 += C v_init, constrained rows zeroed.
  int
  solve_all_at_once(const double *F, double *X, int nI, const double *v_init, int *iterations, double *history,
                    int history_cap)
  {
    if (nI < 1)
      throw std::invalid_argument("solve_all_at_once: need at least one interval");
    stmg_level &L = fine();
    const long long n = L.spec.isz() * nI;
    rhs.resize(n);
    check(cudaMemcpyAsync(rhs.p, F, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream), "copy");
    if (v_init && rank() == 0)
      {
        L.vmult(L.zero_vector(1), F, rhs.p, 1, v_init, 1, 1);
        check(launch_zero_constrained(L.geom, rhs.p, 1, ctx->stream), "zero");
        ctx->count();
      }
    const int it = gmres(rhs.p, X, iterations, history, history_cap, nI, true);
    L.project(X, nI);
    return it;
  }

  // time_march (solver.cpp:204-325) with per-step load vectors F, or a
  // built-in problem (force assembled per step; boundary data by lifting).
  DevArray<double> fstep, lift, lifted;
  void
  time_march(const double *F, double *X, int *iterations, int problem = -1, const double *Lifts = nullptr,
             const double *v_init = nullptr)
  {
    stmg_level &L = fine();
    const long long n = L.spec.isz();
    rhs.resize(n);
    vprev.resize(L.spec.mv());
    if (v_init) // initial velocity at the nodes (solver.cpp:229-236)
      check(cudaMemcpyAsync(vprev.p, v_init, sizeof(double) * L.spec.mv(), cudaMemcpyDeviceToDevice, ctx->stream),
            "copy");
    else
      check(cudaMemsetAsync(vprev.p, 0, sizeof(double) * L.spec.mv(), ctx->stream), "memset");
    const double *zero = L.zero_vector(1);
    const double tau = L.spec.tau;
    const bool inhomogeneous = problem == STMG_PROBLEM_CAVITY || Lifts != nullptr;
    if (problem >= 0)
      fstep.resize(n);
    if (inhomogeneous)
      {
        lift.resize(n);
        lifted.resize(n);
      }
    for (int step = 0; step < n_steps; ++step)
      {
        STMG_NVTX("time_march step %d", step);
        const double t_start = step * tau;
        const double *Fn = F ? F + step * n : zero;
        if (problem == STMG_PROBLEM_MANUFACTURED)
          {
            check(launch_assemble_manufactured(L.geom, L.spec.r, L.problem_tab(), L.spec.nu, t_start, tau, fstep.p, 1,
                                               ctx->stream),
                  "assemble_rhs");
            ctx->count(5);
            Fn = fstep.p;
          }
        // rhs = F_n + C v_prev (coupling_rhs)
        L.vmult(zero, Fn, rhs.p, 1, vprev.p, 1, 1);
        if (inhomogeneous)
          {
            // rhs -= A_raw lift (solver.cpp:251-262)
            if (Lifts)
              check(cudaMemcpyAsync(lift.p, Lifts + step * n, sizeof(double) * n, cudaMemcpyDeviceToDevice,
                                    ctx->stream),
                    "copy");
            else
              {
                check(launch_lift_cavity(L.geom, L.spec.r, L.problem_tab(), t_start, tau, lift.p, 1, ctx->stream),
                      "lift");
                ctx->count();
              }
            L.vmult(lift.p, nullptr, lifted.p, 1, nullptr, 0, 2);
            check(launch_axpy(n, -1.0, nullptr, 1.0, lifted.p, rhs.p, ctx->stream), "axpy");
            ctx->count();
          }
        check(launch_zero_constrained(L.geom, rhs.p, 1, ctx->stream), "zero");
        ctx->count();
        double *x = X + step * n;
        int it = 0;
        gmres(rhs.p, x, &it, nullptr, 0);
        if (inhomogeneous)
          {
            check(launch_axpy(n, 1.0, nullptr, 1.0, lift.p, x, ctx->stream), "axpy"); // x += lift
            ctx->count();
          }
        L.project(x, 1);
        if (iterations)
          iterations[step] = it;
        check(cudaMemcpyAsync(vprev.p, x + (L.spec.S() - 1) * L.spec.mv(), sizeof(double) * L.spec.mv(),
                              cudaMemcpyDeviceToDevice, ctx->stream),
              "copy");
      }
  }
};

namespace
{
void
upload_transfer(SolverLevel &F, const LevelSpec &coarse, const LevelSpec &fine, TransferKind kind)
{
  const TransferTables t = build_transfer(coarse, fine, kind);
  DevTransfer &d = F.dt;
  d = DevTransfer{};
  d.spatial = t.spatial;
  d.temporal = t.temporal;
  d.pmode = t.pmode;
  d.zero_constrained = kind != TransferKind::identity;
  if (t.spatial)
    {
      F.px_ptr.upload(t.px.ptr);
      F.px_col.upload(t.px.col);
      F.px_val.upload(t.px.val);
      F.py_ptr.upload(t.py.ptr);
      F.py_col.upload(t.py.col);
      F.py_val.upload(t.py.val);
      F.rx_ptr.upload(t.rx.ptr);
      F.rx_col.upload(t.rx.col);
      F.rx_val.upload(t.rx.val);
      F.ry_ptr.upload(t.ry.ptr);
      F.ry_col.upload(t.ry.col);
      F.ry_val.upload(t.ry.val);
      d.px = DevCsr{F.px_ptr.p, F.px_col.p, F.px_val.p};
      d.py = DevCsr{F.py_ptr.p, F.py_col.p, F.py_val.p};
      d.rx = DevCsr{F.rx_ptr.p, F.rx_col.p, F.rx_val.p};
      d.ry = DevCsr{F.ry_ptr.p, F.ry_col.p, F.ry_val.p};
    }
  if (t.pmode == 1)
    {
      F.child.upload(t.child);
      d.child = F.child.p;
    }
  if (t.pmode == 2)
    {
      F.embed.upload(t.embed);
      d.embed = F.embed.p;
    }
  if (t.temporal)
    for (int a = 0; a <= fine.k; ++a)
      for (int b = 0; b <= coarse.k; ++b)
        d.E[a * kMaxS + b] = t.e_time[a * (coarse.k + 1) + b];
  const auto geom = [](const LevelSpec &s) {
    return DevGeom{s.nx, s.ny, s.gx(), s.gy(), s.S(), s.np(), s.nsc(), s.mv(), s.mp(), s.isz(), s.hx, s.hy};
  };
  d.f = geom(fine);
  d.c = geom(coarse);
}
} // namespace

// ================================================================ C ABI
extern "C" {

const char *
stmg_last_error(void)
{
  return g_error.c_str();
}

const char *
stmg_version(void)
{
  return "stmg_b200 0.2 sm_100a fp64";
}

int
stmg_set_tuning(const char *key, int64_t value)
{
  return guarded([&] {
    STMG_NVTX("stmg_set_tuning");
    if (!key)
      throw std::invalid_argument("stmg_set_tuning: null key");
    static int64_t groups[2] = {0, 0};
    const std::string k(key);
    if (value < 0 || value > 1024)
      throw std::invalid_argument("stmg_set_tuning: value out of range");
    if (k == "vanka_group")
      groups[0] = value;
    else if (k == "vanka_big_group")
      groups[1] = value;
    else
      throw std::invalid_argument("stmg_set_tuning: unknown key " + k);
    set_vanka_group_override(static_cast<int>(groups[0]), static_cast<int>(groups[1]));
  });
}

int
stmg_ctx_create(int device, stmg_ctx **out)
{
  return guarded([&] {
    STMG_NVTX("stmg_ctx_create");
    if (!out)
      throw std::invalid_argument("stmg_ctx_create: null out");
    check(cudaSetDevice(device), "cudaSetDevice");
    auto c = std::make_unique<stmg_ctx>();
    c->device = device;
    *out = c.release();
  });
}

int
stmg_ctx_destroy(stmg_ctx *ctx)
{
  delete ctx;
  return STMG_OK;
}

int
stmg_ctx_set_stream(stmg_ctx *ctx, void *stream)
{
  return guarded([&] {
    STMG_NVTX("stmg_ctx_set_stream");
    if (!ctx)
      throw std::invalid_argument("null ctx");
    ctx->stream = static_cast<cudaStream_t>(stream);
  });
}

int
stmg_ctx_synchronize(stmg_ctx *ctx)
{
  return guarded([&] {
    check(cudaStreamSynchronize(ctx->stream), "sync");
    if (ctx->h2d) // the host-buffer entry points' copy streams
      check(cudaStreamSynchronize(ctx->h2d), "sync");
    if (ctx->d2h)
      check(cudaStreamSynchronize(ctx->d2h), "sync");
  });
}

int64_t
stmg_ctx_launch_count(const stmg_ctx *ctx)
{
  return ctx ? ctx->launches : 0;
}

int
stmg_level_create(stmg_ctx *ctx, int nx, int ny, int r, int k, double tau, double nu, double gamma, int smoother_kind,
                  stmg_level **out)
{
  return guarded([&] {
    STMG_NVTX("stmg_level_create");
    if (!ctx || !out)
      throw std::invalid_argument("stmg_level_create: null argument");
    if (smoother_kind < -1 || smoother_kind > 1)
      throw std::invalid_argument("stmg_level_create: unknown smoother kind");
    auto L = std::make_unique<stmg_level>();
    L->ctx = ctx;
    L->spec.nx = nx;
    L->spec.ny = ny;
    L->spec.r = r;
    L->spec.k = k;
    L->spec.hx = 1.0 / nx;
    L->spec.hy = 1.0 / ny;
    L->spec.tau = tau;
    L->spec.nu = nu;
    L->spec.gamma = gamma;
    L->smoother_kind = smoother_kind;
    build_level(*L);
    *out = L.release();
  });
}

int
stmg_level_destroy(stmg_level *level)
{
  delete level;
  return STMG_OK;
}

int
stmg_level_sizes(const stmg_level *L, int64_t *out)
{
  return guarded([&] {
    STMG_NVTX("stmg_level_sizes");
    out[0] = L->spec.S();
    out[1] = L->spec.mv();
    out[2] = L->spec.mp();
    out[3] = L->spec.isz();
    out[4] = L->spec.nsc();
    out[5] = L->spec.gx();
    out[6] = L->n_classes;
    out[7] = static_cast<int64_t>(L->total_matrix_elements);
    out[8] = L->factored ? 1 : 0;
    out[9] = static_cast<int64_t>(L->factored_matrix_elements);
  });
}

int
stmg_apply_block(stmg_level *L, const double *x, double *y, int n, int raw)
{
  return guarded([&] { L->vmult(x, nullptr, y, n, nullptr, 0, raw ? 2 : 0); });
}

int
stmg_vmult(stmg_level *L, const double *x, double *y, int n, const double *x_prev_slot)
{
  return guarded([&] { L->vmult(x, nullptr, y, n, x_prev_slot, 1, 0); });
}

int
stmg_residual(stmg_level *L, const double *b, const double *x, double *r, int n, const double *x_prev_slot,
              int coupled)
{
  return guarded([&] { L->vmult(x, b, r, n, x_prev_slot, coupled ? 1 : 0, 1); });
}

int
stmg_coupling_rhs(stmg_level *L, const double *v_prev, double *out)
{
  return guarded([&] {
    STMG_NVTX("stmg_coupling_rhs");
    // raw apply of D*0 - C v_prev on every row, negated: out = C v_prev
    L->vmult(L->zero_vector(1), nullptr, out, 1, v_prev, 1, 2);
    check(launch_scale(L->spec.isz(), -1.0, out, L->ctx->stream), "scale");
    L->ctx->count();
  });
}

int
stmg_step_health(stmg_level *L, const double *X, int n, double *out)
{
  return guarded([&] {
    STMG_NVTX("stmg_step_health");
    if (n < 1 || !X || !out)
      throw std::invalid_argument("step_health: bad arguments");
    const LevelSpec &s = L->spec;
    // y = [M v^a ; B v^a] per slot: the fused operator with K_t = M_t = I,
    // no coupling, nu = gamma = 0 and the pressure input zeroed
    LevelSpec hs = s;
    hs.nu = 0.0;
    hs.gamma = 0.0;
    LevelConsts hc = make_level_consts(hs);
    const double J = s.hx * s.hy / 4.0;
    const int S = s.S();
    for (int a = 0; a < S; ++a)
      {
        hc.lv[a] = hc.lvJ[a] = 0.0;
        for (int b = 0; b < S; ++b)
          {
            hc.Kt[a * S + b] = hc.Mt[a * S + b] = (a == b) ? 1.0 : 0.0;
            hc.KtJ[a * S + b] = hc.MtJ[a * S + b] = (a == b) ? J : 0.0;
          }
      }
    const long long isz = s.isz(), tot = isz * n;
    DevArray<double> xv, y, sums;
    xv.resize(tot);
    y.resize(tot);
    sums.resize(4 * static_cast<size_t>(S) * n);
    check(cudaMemcpyAsync(xv.p, X, sizeof(double) * tot, cudaMemcpyDeviceToDevice, L->ctx->stream), "copy");
    for (int t = 0; t < n; ++t)
      check(cudaMemsetAsync(xv.p + t * isz + S * s.mv(), 0, sizeof(double) * S * s.mp(), L->ctx->stream), "memset");
    check(launch_vmult(s.r, S, hc, xv.p, nullptr, y.p, n, nullptr, 0, 2, L->ctx->stream), "vmult");
    check(launch_health(L->geom, s.hx * s.hy, X, y.p, sums.p, n, L->ctx->stream), "health");
    L->ctx->count(2);
    std::vector<double> h(4 * static_cast<size_t>(S) * n);
    check(cudaMemcpyAsync(h.data(), sums.p, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, L->ctx->stream),
          "d2h");
    check(cudaStreamSynchronize(L->ctx->stream), "sync");
    for (int t = 0; t < n; ++t)
      {
        double max_div = 0.0, max_mean = 0.0;
        for (int a = 0; a < S; ++a)
          {
            const double *q = &h[4 * (static_cast<size_t>(t) * S + a)];
            const double vnorm = std::sqrt(std::abs(q[1]));
            if (vnorm > 0.0)
              max_div = std::max(max_div, std::sqrt(q[0]) / vnorm);
            if (q[3] > 0.0)
              max_mean = std::max(max_mean, std::abs(q[2]) / std::sqrt(q[3]));
          }
        out[2 * t] = max_div;
        out[2 * t + 1] = max_mean;
      }
  });
}

int
stmg_apply_additive(stmg_level *L, const double *r, double *out, int n)
{
  return guarded([&] {
    STMG_NVTX("stmg_apply_additive");
    check(cudaMemsetAsync(out, 0, sizeof(double) * L->spec.isz() * n, L->ctx->stream), "memset");
    L->vanka(r, out, n, 1.0);
  });
}

int
stmg_smooth_step(stmg_level *L, const double *b, double *u, double omega, int n, const double *x_prev_slot,
                 int coupled, double *work)
{
  return guarded([&] { L->smooth_step(b, u, omega, n, x_prev_slot, coupled ? 1 : 0, work); });
}

int
stmg_vanka_update(stmg_level *L, const double *r, double *u, double omega, int n)
{
  return guarded([&] {
    STMG_NVTX("stmg_vanka_update");
    if (!(omega > 0.0 && omega <= 1.0))
      throw std::invalid_argument("vanka_update: omega must be in (0, 1]");
    L->vanka(r, u, n, omega);
  });
}

// Host-buffer entry points, pipelined over chunks of kHostChunk intervals:
// the H2D copy of chunk c+1, the kernels of chunk c and the D2H copy of
// chunk c-1 run concurrently (two copy engines + SMs), so one call costs
// about max(H2D, D2H) bytes over PCIe instead of their sum.
namespace
{
#ifndef STMG_HOST_CHUNK
#define STMG_HOST_CHUNK 4 // intervals per pipelined chunk (measured: 4 beats 8 by 3.7% on the C2 e2e step)
#endif
constexpr int kHostChunk = STMG_HOST_CHUNK;
}

namespace
{
void
vmult_host_impl(stmg_level *L, const double *x, double *y, int n, const double *x_prev_slot, bool sync)
{
  stmg_ctx &C = *L->ctx;
  C.copy_streams();
  const long long isz = L->spec.isz(), mv = L->spec.mv();
  const size_t sz = static_cast<size_t>(isz) * n;
  L->host_in.resize(sz);
  L->host_out.resize(sz);
  L->host_begin(0);
  const double *prev = nullptr;
  if (x_prev_slot)
    {
      L->host_prev_v.resize(mv);
      check(cudaMemcpyAsync(L->host_prev_v.p, x_prev_slot, sizeof(double) * mv, cudaMemcpyHostToDevice, C.h2d),
            "h2d");
      prev = L->host_prev_v.p;
    }
  const int nch = (n + kHostChunk - 1) / kHostChunk;
  for (int c = 0; c < nch; ++c)
    {
      const int i0 = c * kHostChunk, m = std::min(kHostChunk, n - i0);
      const size_t off = static_cast<size_t>(i0) * isz, len = static_cast<size_t>(m) * isz;
      check(cudaMemcpyAsync(L->host_in.p + off, x + off, sizeof(double) * len, cudaMemcpyHostToDevice, C.h2d), "h2d");
      check(cudaEventRecord(C.event(2 * c), C.h2d), "event");
      check(cudaStreamWaitEvent(C.stream, C.event(2 * c), 0), "wait");
      const double *pc = c == 0 ? prev : L->host_in.p + off - isz + (L->spec.S() - 1) * mv;
      L->vmult(L->host_in.p + off, nullptr, L->host_out.p + off, m, pc, 1, 0);
      check(cudaEventRecord(C.event(2 * c + 1), C.stream), "event");
      check(cudaStreamWaitEvent(C.d2h, C.event(2 * c + 1), 0), "wait");
      check(cudaMemcpyAsync(y + off, L->host_out.p + off, sizeof(double) * len, cudaMemcpyDeviceToHost, C.d2h), "d2h");
    }
  L->host_end(0, sync);
}

void
smooth_step_host_impl(stmg_level *L, const double *b, double *u, double omega, int n, const double *x_prev_slot,
                      int coupled, bool sync)
{
  if (!(omega > 0.0 && omega <= 1.0))
    throw std::invalid_argument("smooth_step: omega must be in (0, 1]");
  stmg_ctx &C = *L->ctx;
  C.copy_streams();
  const long long isz = L->spec.isz(), mv = L->spec.mv();
  const size_t sz = static_cast<size_t>(isz) * n;
  L->host_b.resize(sz);
  L->host_u.resize(sz);
  L->host_prev.resize(3 * mv); // [0]: x_prev_slot, [1], [2]: ring of pre-update chunk halos
  L->host_begin(1);
  const double *prev = nullptr;
  if (x_prev_slot && coupled)
    {
      check(cudaMemcpyAsync(L->host_prev.p, x_prev_slot, sizeof(double) * mv, cudaMemcpyHostToDevice, C.h2d), "h2d");
      prev = L->host_prev.p;
    }
  double *r = L->scratch(std::min(n, kHostChunk));
  const int nch = (n + kHostChunk - 1) / kHostChunk;
  for (int c = 0; c < nch; ++c)
    {
      const int i0 = c * kHostChunk, m = std::min(kHostChunk, n - i0);
      const size_t off = static_cast<size_t>(i0) * isz, len = static_cast<size_t>(m) * isz;
      check(cudaMemcpyAsync(L->host_b.p + off, b + off, sizeof(double) * len, cudaMemcpyHostToDevice, C.h2d), "h2d");
      check(cudaMemcpyAsync(L->host_u.p + off, u + off, sizeof(double) * len, cudaMemcpyHostToDevice, C.h2d), "h2d");
      check(cudaEventRecord(C.event(2 * c), C.h2d), "event");
      check(cudaStreamWaitEvent(C.stream, C.event(2 * c), 0), "wait");
      // residual with the pre-update halo of the previous chunk (Jacobi: the
      // whole step sees the old u, as in VankaSmoother::smooth_step)
      const double *halo = c == 0 ? prev : L->host_prev.p + (1 + ((c - 1) & 1)) * mv;
      double *uc = L->host_u.p + off;
      L->vmult(uc, L->host_b.p + off, r, m, coupled ? halo : nullptr, coupled ? 1 : 0, 1);
      if (coupled && c + 1 < nch)
        check(cudaMemcpyAsync(L->host_prev.p + (1 + (c & 1)) * mv, uc + (m - 1) * isz + (L->spec.S() - 1) * mv,
                              sizeof(double) * mv, cudaMemcpyDeviceToDevice, C.stream),
              "halo");
      L->vanka(r, uc, m, omega);
      check(cudaEventRecord(C.event(2 * c + 1), C.stream), "event");
      check(cudaStreamWaitEvent(C.d2h, C.event(2 * c + 1), 0), "wait");
      check(cudaMemcpyAsync(u + off, uc, sizeof(double) * len, cudaMemcpyDeviceToHost, C.d2h), "d2h");
    }
  L->host_end(1, sync);
}
} // namespace

int
stmg_vmult_host(stmg_level *L, const double *x, double *y, int n, const double *x_prev_slot)
{
  return guarded([&] {
    STMG_NVTX("stmg_vmult_host");
    vmult_host_impl(L, x, y, n, x_prev_slot, true);
  });
}

int
stmg_smooth_step_host(stmg_level *L, const double *b, double *u, double omega, int n, const double *x_prev_slot,
                      int coupled)
{
  return guarded([&] {
    STMG_NVTX("stmg_smooth_step_host");
    smooth_step_host_impl(L, b, u, omega, n, x_prev_slot, coupled, true);
  });
}

int
stmg_vmult_host_async(stmg_level *L, const double *x, double *y, int n, const double *x_prev_slot)
{
  return guarded([&] {
    STMG_NVTX("stmg_vmult_host_async");
    vmult_host_impl(L, x, y, n, x_prev_slot, false);
  });
}

int
stmg_smooth_step_host_async(stmg_level *L, const double *b, double *u, double omega, int n,
                            const double *x_prev_slot, int coupled)
{
  return guarded([&] {
    STMG_NVTX("stmg_smooth_step_host_async");
    smooth_step_host_impl(L, b, u, omega, n, x_prev_slot, coupled, false);
  });
}

int
stmg_solver_create(stmg_ctx *ctx, int refinements, int r, int k, int n_steps, double t_end, double nu, double gamma,
                   int smoother_kind, int nu1, int nu2, double omega, int h_only, double rtol, double atol,
                   int max_iterations, stmg_solver **out)
{
  return guarded([&] {
    STMG_NVTX("stmg_solver_create");
    if (!ctx || !out)
      throw std::invalid_argument("stmg_solver_create: null argument");
    if (smoother_kind != STMG_SMOOTHER_CELL && smoother_kind != STMG_SMOOTHER_VERTEX_STAR)
      throw std::invalid_argument("stmg_solver_create: smoother must be cell or vertex_star");
    if (!(omega > 0.0 && omega <= 1.0))
      throw std::invalid_argument("stmg_solver_create: omega must be in (0, 1]");
    if (refinements < 0 || max_iterations < 1 || nu1 < 0 || nu2 < 0)
      throw std::invalid_argument("stmg_solver_create: invalid configuration");
    auto S = std::make_unique<stmg_solver>();
    S->ctx = ctx;
    S->cfg.refinements = refinements;
    S->cfg.r = r;
    S->cfg.k = k;
    S->cfg.n_steps = n_steps;
    S->cfg.t_end = t_end;
    S->cfg.nu = nu;
    S->cfg.gamma = gamma;
    S->cfg.h_only = h_only;
    S->cfg.smoother = smoother_kind == STMG_SMOOTHER_CELL ? PatchKind::cell : PatchKind::vertex_star;
    S->nu1 = nu1;
    S->nu2 = nu2;
    S->omega = omega;
    S->rtol = rtol;
    S->atol = atol;
    S->max_iterations = max_iterations;
    const std::vector<LevelPlan> plan = plan_levels(S->cfg, &S->n_steps);
    for (size_t l = 0; l < plan.size(); ++l)
      {
        auto SL = std::make_unique<SolverLevel>();
        SL->kind = plan[l].kind_to_coarser;
        SL->level = std::make_unique<stmg_level>();
        SL->level->ctx = ctx;
        SL->level->spec = plan[l].spec;
        SL->level->smoother_kind = l == 0 ? STMG_SMOOTHER_NONE : smoother_kind;
        build_level(*SL->level);
        if (l > 0)
          upload_transfer(*SL, plan[l - 1].spec, plan[l].spec, SL->kind);
        S->levels.push_back(std::move(SL));
      }
    std::vector<long long> pinned;
    const std::vector<double> inv = coarse_inverse(plan[0].spec, pinned);
    S->coarse_inv.upload(inv);
    S->coarse_pinned.upload(pinned);
    S->n_pinned = static_cast<int>(pinned.size());
    S->coarse_n = static_cast<int>(plan[0].spec.isz());
    *out = S.release();
  });
}

int
stmg_solver_destroy(stmg_solver *s)
{
  delete s;
  return STMG_OK;
}

int
stmg_solver_info(const stmg_solver *s, int64_t *out)
{
  return guarded([&] {
    STMG_NVTX("stmg_solver_info");
    out[0] = static_cast<int64_t>(s->levels.size());
    out[1] = s->n_steps;
    for (size_t l = 0; l < s->levels.size(); ++l)
      {
        const LevelSpec &sp = s->levels[l]->level->spec;
        out[2 + 5 * l + 0] = sp.nx;
        out[2 + 5 * l + 1] = sp.r;
        out[2 + 5 * l + 2] = sp.k;
        out[2 + 5 * l + 3] = static_cast<int64_t>(s->levels[l]->kind);
        out[2 + 5 * l + 4] = sp.isz();
      }
  });
}

stmg_level *
stmg_solver_level(stmg_solver *s, int l)
{
  if (!s || l < 0 || l >= static_cast<int>(s->levels.size()))
    return nullptr;
  return s->levels[l]->level.get();
}

int
stmg_restrict_residual(stmg_solver *s, int l, const double *fine, double *coarse, int project_pressure)
{
  return guarded([&] {
    STMG_NVTX("stmg_restrict_residual");
    if (l < 1 || l >= static_cast<int>(s->levels.size()))
      throw std::invalid_argument("stmg_restrict_residual: level out of range");
    s->restrict_residual(l, fine, coarse, project_pressure != 0);
  });
}

int
stmg_prolongate_correction(stmg_solver *s, int l, const double *coarse, double *fine, int project_pressure,
                           int accumulate)
{
  return guarded([&] {
    STMG_NVTX("stmg_prolongate_correction");
    if (l < 1 || l >= static_cast<int>(s->levels.size()))
      throw std::invalid_argument("stmg_prolongate_correction: level out of range");
    s->prolongate_correction(l, coarse, fine, project_pressure != 0, accumulate != 0);
  });
}

int
stmg_coarse_solve(stmg_solver *s, const double *b, double *x)
{
  return guarded([&] { s->coarse_solve(b, x); });
}

int
stmg_vcycle(stmg_solver *s, const double *b, double *x)
{
  return guarded([&] { s->vcycle(b, x); });
}

int
stmg_gmres(stmg_solver *s, const double *b, double *x, int *iterations, double *history, int history_cap)
{
  return guarded([&] { s->gmres(b, x, iterations, history, history_cap); });
}

int
stmg_assemble_rhs(stmg_level *L, int problem, double t_start, double *F, int n)
{
  return guarded([&] {
    STMG_NVTX("stmg_assemble_rhs");
    if (problem != STMG_PROBLEM_MANUFACTURED)
      throw std::invalid_argument("stmg_assemble_rhs: unknown problem");
    if (n < 0 || !F)
      throw std::invalid_argument("stmg_assemble_rhs: invalid arguments");
    check(launch_assemble_manufactured(L->geom, L->spec.r, L->problem_tab(), L->spec.nu, t_start, L->spec.tau, F, n,
                                       L->ctx->stream),
          "assemble_rhs");
    L->ctx->count(5);
  });
}

int
stmg_interpolate_exact(stmg_level *L, int problem, double t_start, double *X, int n)
{
  return guarded([&] {
    STMG_NVTX("stmg_interpolate_exact");
    if (problem != STMG_PROBLEM_MANUFACTURED)
      throw std::invalid_argument("stmg_interpolate_exact: unknown problem");
    if (n < 0 || !X)
      throw std::invalid_argument("stmg_interpolate_exact: invalid arguments");
    check(launch_interpolate_manufactured(L->geom, L->spec.r, L->problem_tab(), t_start, L->spec.tau, X, n,
                                          L->ctx->stream),
          "interpolate_exact");
    L->ctx->count(2);
  });
}

int
stmg_compute_errors(stmg_level *L, int problem, double t_start, const double *X, int n, double *out)
{
  return guarded([&] {
    STMG_NVTX("stmg_compute_errors");
    if (problem != STMG_PROBLEM_MANUFACTURED)
      throw std::invalid_argument("stmg_compute_errors: unknown problem");
    if (n < 1 || !X || !out)
      throw std::invalid_argument("stmg_compute_errors: invalid arguments");
    L->err_part.resize(errors_partials(L->geom, n));
    L->err_out.resize(5);
    check(launch_errors_manufactured(L->geom, L->spec.r, L->problem_tab(), t_start, L->spec.tau, X, n,
                                     L->err_part.p, L->err_out.p, L->ctx->stream),
          "compute_errors");
    L->ctx->count(2);
    check(cudaMemcpyAsync(out, L->err_out.p, sizeof(double) * 5, cudaMemcpyDeviceToHost, L->ctx->stream), "d2h");
    check(cudaStreamSynchronize(L->ctx->stream), "sync");
  });
}

int
stmg_solver_set_krylov(stmg_solver *s, int orthogonalization)
{
  return guarded([&] {
    if (!s)
      throw std::invalid_argument("stmg_solver_set_krylov: null solver");
    if (orthogonalization != STMG_ORTHO_MGS && orthogonalization != STMG_ORTHO_CGS2)
      throw std::invalid_argument("stmg_solver_set_krylov: unknown orthogonalization");
    s->ortho = orthogonalization;
  });
}

int
stmg_solver_set_comm(stmg_solver *s, const stmg_comm_ops *ops)
{
  return guarded([&] {
    STMG_NVTX("stmg_solver_set_comm");
    if (!ops)
      {
        s->has_comm = false;
        s->comm = stmg_comm_ops{};
        return;
      }
    if (ops->world < 1 || ops->rank < 0 || ops->rank >= ops->world)
      throw std::invalid_argument("stmg_solver_set_comm: invalid rank/world");
    if (ops->world > 1 && (!ops->exchange_halo || !ops->allreduce_sum || !ops->allgather))
      throw std::invalid_argument("stmg_solver_set_comm: missing callback");
    s->comm = *ops;
    s->has_comm = true;
  });
}

int
stmg_vcycle_all_at_once(stmg_solver *s, const double *b, double *x, int n_intervals)
{
  return guarded([&] {
    STMG_NVTX("stmg_vcycle_all_at_once");
    if (n_intervals < 1)
      throw std::invalid_argument("stmg_vcycle_all_at_once: need at least one interval");
    s->cycle(static_cast<int>(s->levels.size()) - 1, b, x, n_intervals, true);
  });
}

int
stmg_solve_all_at_once(stmg_solver *s, const double *F, double *X, int n_intervals, const double *v_init,
                       int *iterations, double *history, int history_cap)
{
  return guarded([&] { s->solve_all_at_once(F, X, n_intervals, v_init, iterations, history, history_cap); });
}

int
stmg_time_march(stmg_solver *s, const double *F, double *X, int *iterations)
{
  return guarded([&] { s->time_march(F, X, iterations); });
}

int
stmg_time_march_problem(stmg_solver *s, int problem, double *X, int *iterations)
{
  return guarded([&] {
    STMG_NVTX("stmg_time_march_problem");
    if (problem != STMG_PROBLEM_MANUFACTURED && problem != STMG_PROBLEM_CAVITY)
      throw std::invalid_argument("stmg_time_march_problem: unknown problem");
    s->time_march(nullptr, X, iterations, problem);
  });
}

int
stmg_time_march_ex(stmg_solver *s, const double *F, const double *lifts, const double *v_init, double *X,
                   int *iterations)
{
  return guarded([&] { s->time_march(F, X, iterations, -1, lifts, v_init); });
}

int
stmg_time_march_host(stmg_solver *s, const double *F, double *X, int *iterations)
{
  return guarded([&] {
    STMG_NVTX("stmg_time_march_host");
    stmg_level &L = s->fine();
    const size_t sz = static_cast<size_t>(L.spec.isz()) * s->n_steps;
    L.host_in.resize(sz);
    L.host_out.resize(sz);
    cudaStream_t st = s->ctx->stream;
    check(cudaMemcpyAsync(L.host_in.p, F, sizeof(double) * sz, cudaMemcpyHostToDevice, st), "h2d");
    s->time_march(L.host_in.p, L.host_out.p, iterations);
    check(cudaMemcpyAsync(X, L.host_out.p, sizeof(double) * sz, cudaMemcpyDeviceToHost, st), "d2h");
    check(cudaStreamSynchronize(st), "sync");
  });
}

int
stmg_plan_levels(int refinements, int r, int k, int n_steps, double t_end, int h_only, int64_t *out)
{
  return guarded([&] {
    STMG_NVTX("stmg_plan_levels");
    HierarchyConfig cfg;
    cfg.refinements = refinements;
    cfg.r = r;
    cfg.k = k;
    cfg.n_steps = n_steps;
    cfg.t_end = t_end;
    cfg.h_only = h_only;
    int ns = 0;
    const std::vector<LevelPlan> plan = plan_levels(cfg, &ns);
    out[0] = static_cast<int64_t>(plan.size());
    out[1] = ns;
    for (size_t l = 0; l < plan.size(); ++l)
      {
        out[2 + 5 * l + 0] = plan[l].spec.nx;
        out[2 + 5 * l + 1] = plan[l].spec.r;
        out[2 + 5 * l + 2] = plan[l].spec.k;
        out[2 + 5 * l + 3] = static_cast<int64_t>(plan[l].kind_to_coarser);
        out[2 + 5 * l + 4] = plan[l].spec.isz();
      }
  });
}

int
stmg_patch_info(int nx, int ny, int r, int k, double tau, double nu, double gamma, int smoother_kind, int64_t *out,
                double *inverse_out, int class_index)
{
  return guarded([&] {
    STMG_NVTX("stmg_patch_info");
    LevelSpec s;
    s.nx = nx;
    s.ny = ny;
    s.r = r;
    s.k = k;
    s.hx = 1.0 / nx;
    s.hy = 1.0 / ny;
    s.tau = tau;
    s.nu = nu;
    s.gamma = gamma;
    const PatchSet ps = build_patches(s, smoother_kind == STMG_SMOOTHER_VERTEX_STAR ? PatchKind::vertex_star
                                                                                   : PatchKind::cell);
    long long n = 0;
    for (const auto &c : ps.colours)
      n += static_cast<long long>(c.size());
    out[0] = n;
    out[1] = static_cast<int64_t>(ps.classes.size());
    out[2] = static_cast<int64_t>(ps.total_matrix_elements);
    out[3] = static_cast<int64_t>(ps.colours.size());
    for (size_t c = 0; c < ps.classes.size() && c < 56; ++c)
      out[4 + c] = ps.classes[c].n_t;
    out[60] = ps.factored ? 1 : 0;
    out[61] = ps.n_sp;
    out[62] = static_cast<int64_t>(ps.factored_matrix_elements);
    if (inverse_out)
      {
        if (class_index < 0 || class_index >= static_cast<int>(ps.classes.size()))
          throw std::invalid_argument("stmg_patch_info: class index out of range");
        const auto &inv = ps.classes[class_index].inverse;
        std::memcpy(inverse_out, inv.data(), sizeof(double) * inv.size());
      }
  });
}

} // extern "C"
