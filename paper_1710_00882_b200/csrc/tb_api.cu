// tb_api.cu -- C ABI (include/tersoff_b200.h) over the sm_100a kernels.
//
// Unity build: the kernels live in tb_kernels.cuh / tb_math.cuh.  Host logic
// here mirrors the reference's orchestration of the hot path:
//   build_neighbor_list  neighbor.py:194-217   -> tb_build_neighbors
//   needs_rebuild        neighbor.py:220-229   -> tb_needs_rebuild
//   compute()            kernels.py:517-527    -> tb_compute / tb_compute_device
//   velocity_verlet_step system.py:355-380     -> tb_md_step
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/tersoff_b200.h"
#include "tb_kernels.cuh"
#include "tb_scan.cuh"
#include "tb_warp.cuh"
#include "tb_dnl.cuh"
#include "tb_dd.cuh"
#include "tb_stream.cuh"
#include "tb_row.cuh"

#ifndef TB_VERSION_TAG
#define TB_VERSION_TAG "dev"
#endif

using namespace tb;

namespace {

struct DevBuf {
  void *p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    size_t want = std::max<size_t>(bytes, 256);
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) cap = want;
    return e;
  }
  template <class X>
  X *as() const { return static_cast<X *>(p); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

}  // namespace

struct tb_context {
  int device = 0;
  cudaStream_t own = nullptr, stream = nullptr;
  std::string err;
  // parameters
  int S = 0;
  int param_version = 0;  // bumped by tb_set_params (captured MD graphs hold the tables)
  bool lam3 = false;
  double r_cut = 0.0;
  std::vector<double> pair_mat, trip_mat;
  // scratch
  DevBuf pos, species, forces, per_atom, result, stats, partials, errf, drift, bounds,
      scan_tmp, facc, stats_acc, ke_part, snap;
  DevBuf dyn_pair64, dyn_trip64, dyn_pair32, dyn_trip32;  // S > SMAX: tables of the S = 0 kernel
  cudaStream_t cap[2] = {nullptr, nullptr};  // tb_md_run graph capture
  int64_t facc_n = -1;
  ErrFlags *h_err = nullptr;      // pinned
  double *h_small = nullptr;      // pinned scratch (64 doubles)
  // kernel timing (tb_profile)
  bool profile = false;
  bool force_tile = false;
  int live_pack = 2;  // TB_OPT_LIVE_PACK: 0 off, 1 on, 2 auto
#ifndef TB_MD_LOOSE_DEFAULT
#define TB_MD_LOOSE_DEFAULT 0.3
#endif
  double md_loose = TB_MD_LOOSE_DEFAULT;  // TB_OPT_MD_LOOSE_SKIN: extra list skin (A) of tb_md_run, 0 = off
  double list_margin = 0.25;  // TB_OPT_LIST_MARGIN
#ifndef TB_REPACK_MARGIN_DEFAULT
#define TB_REPACK_MARGIN_DEFAULT 0.001  // c3 step (A): 0 -> 333 us, 1e-3 -> 261, 5e-3 -> 268, 0.01 -> 276, 0.05 -> 331
#endif
  double repack_margin = TB_REPACK_MARGIN_DEFAULT;  // TB_OPT_REPACK_MARGIN (A)
  bool md_live = getenv("TB_NO_MD_REPACK") == nullptr;  // live repack inside tb_md_run (S > 1)
  bool nl_atoms = getenv("TB_NL_CELLS") == nullptr;  // atom-centric list scan (all-periodic grids)
  bool warp_per_chunk = getenv("TB_WARP_PER_CHUNK") != nullptr;
  bool no_filter = getenv("TB_NO_FILTER") != nullptr;  // disable the species-pair compute filter
  bool err_unchecked = false;     // kernels may have raised error flags nobody read yet
  // tb_compute with host buffers: finalize also copies the error flags here
  // (device alias of pinned host memory) and an event marks the end of the
  // Tersoff kernel so the per-atom energies go back on the side stream
  unsigned long long *fin_err_dst = nullptr;
  cudaEvent_t ev_kernel_done = nullptr;
  cudaStream_t side = nullptr;
  const int *dplan = nullptr;  // tb_md_run capture: device {nchunks, n_empty}
  bool md_fuse = false;  // tb_md_run capture (atomic): finalize folded into the kick kernels
  // streamed tb_compute (tb_stream.cuh): pinned host buffers, ranges of atoms
  // copied in / evaluated / copied out concurrently
  int stream_range = 131072;  // TB_OPT_STREAM_RANGE: atoms per range at least; 0 = off
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  std::vector<cudaEvent_t> ev_h2d, ev_stage;
  cudaEvent_t ev_fork = nullptr;
  struct StreamCtl *sctl = nullptr;  // set by tb_compute around enqueue_compute
  int part_off = 0;     // first block-partial slot of the next warp launch
  bool row_kernel = getenv("TB_NO_ROW_KERNEL") == nullptr;  // TB_OPT_ROW_KERNEL: atom-per-lane kernel for rows <= 4
  // ... for lists with at least this many such rows (tools/row_crossover.py,
  // fp64 row vs warp-chunk kernel: 64k atoms 34 vs 21 us, 512k 94 vs 87 us,
  // 1M 152 vs 159 us, 2.1M 285 vs 318 us)
  int64_t row_min = getenv("TB_ROW_MIN") ? atoll(getenv("TB_ROW_MIN")) : 1000000;
  int last_blocks = 0;  // grid of the last Tersoff launch (partials to reduce)  // tb_set_option(TB_OPT_TILE_KERNEL): general tile kernel only
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_used, ev_free;
};

struct tb_nlist {
  tb_context *ctx = nullptr;
  int64_t n = 0;
  double L[3] = {0, 0, 0};
  int per[3] = {0, 0, 0};
  double r_cut = 0.0, skin = 0.0, bc = 0.0;
  int64_t entries = 0, max_row = 0;
  bool built = false;
  DevBuf offsets, nbr, rev, ref_pos, atom_cell, cell_count, cell_start, cell_atoms, row_count,
      maxrow, nl_row, sorted_atoms, sort_keys, iota, lanes, hist, cpos, crow, coff, centry,
      fnbr, scratch,  // TMPW-wide per-atom rows of the single-pass scan
      crel;           // fp32 cell-relative candidate records (k_cell_rel)
  bool filtered = false;                 // chunks built from the species-pair filter
  DevBuf fbuf;                           // gather mode: per-entry force pieces
  bool fbuf_zero = false;                // entries without lanes hold zeros
  const int *filter_species = nullptr;   // species array the filter was built for
  int filter_param_version = -1;         // tb_set_params version the filter was built for
  DevBuf fspecies;                       // copy of the species the filter was built for
  std::vector<int> host_species;         // host species last staged for this list
  bool rev_valid = false;
  int nchunks = 0;  // > 0: warp-chunk fast path available (max_row <= 32)
  int n_empty = 0;  // atoms with empty rows: sorted_atoms[0, n_empty)
  int64_t lanes_used = 0;  // warp-chunk lanes holding an entry (of 32 * nchunks)
  // capacities for the device-resident rebuild (tb_md_run): entry-sized
  // buffers hold ecap entries, the lane table ccap warp chunks
  double margin = -1.0;  // < 0: the context's list margin at the next build
  int64_t ecap = 0, ccap = 0;
  Grid grid;
  int64_t ncell = 0;
  DevBuf plan;      // DevPlan
  // live repack (TB_OPT_LIVE_PACK): rows cut to their entries with r < r_cut at
  // the evaluation's positions (pack_adjacency, neighbor.py:330-360), re-chunked
  // on the device every evaluation
  DevBuf lplan, llen, lrow, lrowj, lsorted, llanes;
  DevBuf ref_log;  // tb_md_run loose list: positions of the reference's last rebuild
  // margin repack (TB_OPT_REPACK_MARGIN): positions of the last repack, the
  // gate's drift word and flag; valid until the list or its filter changes
  DevBuf lref, lgate, lforce;  // lforce: device flag, set by the in-graph rebuild
  bool lvalid = false, lfilt = false;
  double lmargin = -1.0;
  bool fnbr_ok = false;  // fnbr matches centry (written by every filter pass since)
  int64_t lcap = 0;  // chunk capacity of llanes
  // rows of 1..ROW_LM entries (tb_row.cuh): sorted_atoms[r4_first, r4_first + r4_count),
  // their warp chunks are lanes[0, r4_chunks)
  int r4_first = 0, r4_count = 0, r4_chunks = 0;
  // streamed tb_compute: chunks sorted by stage (tb_stream.cuh)
  int64_t lanes_version = 0;  // bumped whenever `lanes` is rewritten
  int64_t sp_version = -1;
  int sp_K = 0, sp_R = 0;
  std::vector<int> sp_cstart, sp_fin;  // [K+1] first chunk of a stage; [K] last stage touching a range
  DevBuf sp_lanes, sp_tmp;
  bool imported = false;  // rows from tb_nlist_import (no cell grid: no device rebuild)
  struct MdGraph *md = nullptr;
};

// streamed tb_compute: host endpoints of one call (tb_stream.cuh)
struct StreamCtl {
  const double *h_pos;   // pinned host positions (n,3)
  double *h_forces;      // pinned host forces (n,3)
  double *h_per_atom;    // pinned host per-atom energies (n) or nullptr
  double *d_pos;         // device staging of the positions
};

// captured device-resident NVE loop (tb_md_run), reused while its key holds
struct MdKey {
  const void *ptr[48];
  int64_t n, ecap, ccap, ncell;
  double dt, accel, skin, r_cut;
  double L[3], width[3], origin[3];  // the graph bakes the box and cell grid in by value
  int per[3], nc[3], stencil_image;
  int rebuild_every, precision, scatter, record_every, param_version, filtered, S, tile;
  double loose, margin;
  int64_t lcap;
};

struct MdGraph {
  MdKey key;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
};

static void md_graph_release(tb_nlist *nl) {
  if (!nl->md) return;
  if (nl->md->exec) cudaGraphExecDestroy(nl->md->exec);
  if (nl->md->graph) cudaGraphDestroy(nl->md->graph);
  delete nl->md;
  nl->md = nullptr;
}

// ---------------------------------------------------------------------------
// error helpers
// ---------------------------------------------------------------------------

static int fail(tb_context *ctx, int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (ctx) ctx->err = buf;
  return code;
}

#define CK(call)                                                                    \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess)                                                          \
      return fail(ctx, TB_ERR_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

static bool is_device_ptr(const void *p) {
  if (!p) return false;
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged;
}

// wait for a stream by polling (a synchronous call of ~0.1 ms: polling avoids
// the scheduler wake-up latency of a blocking wait)
static cudaError_t spin_sync(cudaStream_t s) {
  cudaError_t e;
  while ((e = cudaStreamQuery(s)) == cudaErrorNotReady) {
  }
  return e;
}

// device-accessible alias of a host pointer (pinned / registered host memory,
// mapped under unified addressing), or nullptr for pageable memory
static void *host_alias(const void *p) {
  if (!p) return nullptr;
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return attr.type == cudaMemoryTypeHost ? attr.devicePointer : nullptr;
}

// python-style %g of a double for messages
static std::string fmt_g(double v) {
  char b[64];
  snprintf(b, sizeof(b), "%g", v);
  return b;
}

static Box make_box(const double *L, const int *per) {
  Box b;
  for (int ax = 0; ax < 3; ++ax) {
    b.L[ax] = L[ax];
    b.invL[ax] = 1.0 / L[ax];
    b.per[ax] = per[ax] ? 1 : 0;
  }
  return b;
}

static inline int nblk(int64_t n, int t) { return (int)((n + t - 1) / t); }

constexpr int SCAN_G = 4;  // lanes per atom in the CSR compaction (rows of ~4-8 entries)

// ---------------------------------------------------------------------------
// parameter tables (potential.py:127-155 column order)
// ---------------------------------------------------------------------------

// per-entry constants of the flattened tables (any species count)
template <class T>
static void fill_entries(const tb_context *ctx, int S, PairP<T> *pair, TripP<T> *trip) {
  const double kNegQuarterPi = -0.25 * 3.141592653589793;
  for (int q = 0; q < S * S * S; ++q) {
    const double *r = &ctx->trip_mat[8 * q];
    TripP<T> &t = trip[q];
    memset(&t, 0, sizeof(t));
    T R = (T)r[0], D = (T)r[1];
    t.Rm = R - D;
    t.Rp = R + D;
    t.R = R;
    t.halfInvD = (T)(0.5 / r[1]);
    t.nqpInvD = (T)kNegQuarterPi / D;
    t.gamma = (T)r[2];
    double c2 = r[3] * r[3], d2 = r[4] * r[4];
    t.gc2d2 = (T)(r[2] * c2 / d2);
    t.m2gc2 = (T)(-2.0 * r[2] * c2);
    t.d2 = (T)d2;
    t.h = (T)r[5];
    t.lam3 = (T)r[6];
    t.lam3x3 = (T)(3.0 * r[6]);
    t.m = (int)r[7];
  }
  for (int q = 0; q < S * S; ++q) {
    const double *r = &ctx->pair_mat[8 * q];
    PairP<T> &p = pair[q];
    memset(&p, 0, sizeof(p));
    T R = (T)r[0], D = (T)r[1];
    p.Rm = R - D;
    p.Rp = R + D;
    p.R = R;
    p.halfInvD = (T)(0.5 / r[1]);
    p.nqpInvD = (T)kNegQuarterPi / D;
    p.A = (T)r[2];
    p.lam1 = (T)r[3];
    p.B = (T)r[4];
    p.lam2 = (T)r[5];
    p.beta = (T)r[6];
    p.eta = (T)r[7];
    p.neg_half_inv_eta = (T)(-0.5 / r[7]);
    p.neg_half_beta = (T)(-0.5 * r[6]);
  }
}

template <class T, int S>
static Tables<T, S> make_tables(const tb_context *ctx) {
  Tables<T, S> tab;
  memset(&tab, 0, sizeof(tab));
  if (S == 0) return tab;  // runtime species count: tables in ctx->dyn (global memory)
  fill_entries<T>(ctx, S, tab.pair, tab.trip);
  tab.gsym = 1;
  for (int i = 0; i < S; ++i)
    for (int j = 0; j < S; ++j)
      for (int k = 0; k < S; ++k) {
        const TripP<T> &x = tab.trip[(i * S + j) * S + k], &y = tab.trip[(i * S + k) * S + j];
        if (!(x.gamma == y.gamma && x.gc2d2 == y.gc2d2 && x.m2gc2 == y.m2gc2 && x.d2 == y.d2 &&
              x.h == y.h && x.lam3 == y.lam3 && x.lam3x3 == y.lam3x3 && x.m == y.m))
          tab.gsym = 0;
      }
  tab.ang_i = 1;
  for (int i = 0; i < S; ++i)
    for (int q = 0; q < S * S; ++q) {
      const TripP<T> &x = tab.trip[i * S * S + q], &y = tab.trip[i * S * S];
      if (!(x.gamma == y.gamma && x.gc2d2 == y.gc2d2 && x.m2gc2 == y.m2gc2 && x.d2 == y.d2 &&
            x.h == y.h))
        tab.ang_i = 0;
    }
  tab.fc_same = S == 1 && ctx->pair_mat[0] == ctx->trip_mat[0] && ctx->pair_mat[1] == ctx->trip_mat[1];
  return tab;
}

// ---------------------------------------------------------------------------
// context
// ---------------------------------------------------------------------------

extern "C" int tb_create(int device, tb_context **out) {
  if (!out) return TB_ERR_ARG;
  tb_context *ctx = new tb_context();
  ctx->device = device;
  *out = nullptr;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    delete ctx;
    return TB_ERR_CUDA;
  }
  if (cudaStreamCreateWithFlags(&ctx->own, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMallocHost(&ctx->h_err, sizeof(ErrFlags)) != cudaSuccess ||
      cudaMallocHost(&ctx->h_small, 64 * sizeof(double)) != cudaSuccess) {
    delete ctx;
    return TB_ERR_CUDA;
  }
  ctx->stream = ctx->own;
  *out = ctx;
  return TB_OK;
}

extern "C" void tb_destroy(tb_context *ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  DevBuf *bufs[] = {&ctx->pos, &ctx->species, &ctx->forces, &ctx->per_atom, &ctx->result,
                    &ctx->stats, &ctx->partials, &ctx->facc, &ctx->stats_acc, &ctx->ke_part, &ctx->errf,
                    &ctx->drift, &ctx->bounds, &ctx->scan_tmp, &ctx->snap,
                    &ctx->dyn_pair64, &ctx->dyn_trip64, &ctx->dyn_pair32, &ctx->dyn_trip32};
  for (DevBuf *b : bufs) b->release();
  for (auto *v : {&ctx->ev_used, &ctx->ev_free})
    for (auto &ev : *v) {
      cudaEventDestroy(ev.first);
      cudaEventDestroy(ev.second);
    }
  if (ctx->side) cudaStreamDestroy(ctx->side);
  if (ctx->s_h2d) cudaStreamDestroy(ctx->s_h2d);
  if (ctx->s_d2h) cudaStreamDestroy(ctx->s_d2h);
  for (auto *v : {&ctx->ev_h2d, &ctx->ev_stage})
    for (cudaEvent_t ev : *v) cudaEventDestroy(ev);
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_kernel_done) cudaEventDestroy(ctx->ev_kernel_done);
  if (ctx->h_err) cudaFreeHost(ctx->h_err);
  if (ctx->h_small) cudaFreeHost(ctx->h_small);
  if (ctx->own) cudaStreamDestroy(ctx->own);
  for (cudaStream_t c : ctx->cap)
    if (c) cudaStreamDestroy(c);
  delete ctx;
}

extern "C" const char *tb_last_error(const tb_context *ctx) {
  return ctx ? ctx->err.c_str() : "null context";
}

extern "C" int tb_set_stream(tb_context *ctx, void *stream) {
  if (!ctx) return TB_ERR_ARG;
  ctx->stream = (cudaStream_t)stream;
  return TB_OK;
}

extern "C" int tb_set_option(tb_context *ctx, int option, int value) {
  if (!ctx) return TB_ERR_ARG;
  if (option == TB_OPT_TILE_KERNEL) {
    ctx->force_tile = value != 0;
    return TB_OK;
  }
  if (option == TB_OPT_LIVE_PACK) {
    if (value < 0 || value > 2) return fail(ctx, TB_ERR_ARG, "live-pack mode %d out of range", value);
    ctx->live_pack = value;
    return TB_OK;
  }
  if (option == TB_OPT_MD_LOOSE_SKIN) {
    if (value < 0 || value > 300) return fail(ctx, TB_ERR_ARG, "loose skin %d out of range", value);
    ctx->md_loose = value / 100.0;
    return TB_OK;
  }
  if (option == TB_OPT_REPACK_MARGIN) {
    if (value < 0 || value > 1000)
      return fail(ctx, TB_ERR_ARG, "repack margin %d mA out of range", value);
    ctx->repack_margin = value / 1000.0;
    return TB_OK;
  }
  if (option == TB_OPT_LIST_MARGIN) {
    if (value < 0 || value > 1000) return fail(ctx, TB_ERR_ARG, "list margin %d%% out of range", value);
    ctx->list_margin = value / 100.0;
    return TB_OK;
  }
  if (option == TB_OPT_ROW_KERNEL) {
    if (value < 0) return fail(ctx, TB_ERR_ARG, "row-kernel threshold %d out of range", value);
    ctx->row_kernel = value != 0;
    if (value > 0) ctx->row_min = value == 1 ? 1000000 : value;
    return TB_OK;
  }
  if (option == TB_OPT_STREAM_RANGE) {
    if (value < 0) return fail(ctx, TB_ERR_ARG, "stream range %d out of range", value);
    ctx->stream_range = value;
    return TB_OK;
  }
  return fail(ctx, TB_ERR_ARG, "unknown option %d", option);
}

extern "C" int tb_synchronize(tb_context *ctx) {
  if (!ctx) return TB_ERR_ARG;
  CK(cudaStreamSynchronize(ctx->stream));
  return TB_OK;
}

extern "C" int tb_set_params(tb_context *ctx, int nspecies, const double *pair_mat,
                             const double *trip_mat, double *r_cut_out) {
  if (!ctx || !pair_mat || !trip_mat) return fail(ctx, TB_ERR_ARG, "null argument");
  if (nspecies < 1 || nspecies > SDYN_MAX)
    return fail(ctx, TB_ERR_CONFIG, "the B200 kernels support 1..%d species, got %d", SDYN_MAX,
                nspecies);
  const int S = nspecies;
  // validate everything before touching the context (a refused table leaves
  // the previous one in place)
  double rc = 0.0;
  bool lam3 = false;
  for (int q = 0; q < S * S * S; ++q) {
    const double *r = trip_mat + 8 * q;
    rc = std::max(rc, r[0] + r[1]);
    lam3 |= r[6] != 0.0;
    if (!(r[7] == 1.0 || r[7] == 3.0))
      return fail(ctx, TB_ERR_CONFIG, "m must be 1 or 3, got %g", r[7]);
  }
  // the fp64 kernel's fast exp / log domains (tb_fastmath.h): exp(-lambda r)
  // for r < R + D and log(beta zeta) for zeta >= 1e-30 -- no physical table
  // comes near these bounds; others are refused instead of silently rounded
  for (int q = 0; q < S * S; ++q) {
    const double *r = pair_mat + 8 * q;
    const double reach = r[0] + r[1];
    if (!(std::fabs(r[3]) * reach <= 700.0 && std::fabs(r[5]) * reach <= 700.0))
      return fail(ctx, TB_ERR_CONFIG,
                  "lambda1 %g / lambda2 %g times the cutoff %g exceeds the kernel's exp range", r[3],
                  r[5], reach);
    if (!(r[6] == 0.0 || r[6] >= 1e-250))
      return fail(ctx, TB_ERR_CONFIG, "beta must be 0 or in [1e-250, inf), got %g", r[6]);
  }
  ctx->S = S;
  ctx->pair_mat.assign(pair_mat, pair_mat + 8 * S * S);
  ctx->trip_mat.assign(trip_mat, trip_mat + 8 * S * S * S);
  ctx->lam3 = lam3;
  ctx->r_cut = rc;
  ctx->param_version += 1;
  if (S > SMAX) {
    // runtime-S tile kernel: the derived tables in device memory, per precision
    CK(cudaSetDevice(ctx->device));
    std::vector<PairP<double>> p64(S * S);
    std::vector<TripP<double>> t64((size_t)S * S * S);
    std::vector<PairP<float>> p32(S * S);
    std::vector<TripP<float>> t32((size_t)S * S * S);
    fill_entries<double>(ctx, S, p64.data(), t64.data());
    fill_entries<float>(ctx, S, p32.data(), t32.data());
    CK(ctx->dyn_pair64.ensure(sizeof(PairP<double>) * p64.size()));
    CK(ctx->dyn_trip64.ensure(sizeof(TripP<double>) * t64.size()));
    CK(ctx->dyn_pair32.ensure(sizeof(PairP<float>) * p32.size()));
    CK(ctx->dyn_trip32.ensure(sizeof(TripP<float>) * t32.size()));
    CK(cudaMemcpy(ctx->dyn_pair64.p, p64.data(), sizeof(PairP<double>) * p64.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->dyn_trip64.p, t64.data(), sizeof(TripP<double>) * t64.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->dyn_pair32.p, p32.data(), sizeof(PairP<float>) * p32.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->dyn_trip32.p, t32.data(), sizeof(TripP<float>) * t32.size(), cudaMemcpyHostToDevice));
  }
  if (r_cut_out) *r_cut_out = rc;
  return TB_OK;
}

template <class T>
static int peak_t(tb_context *ctx, double *tflops) {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
  const int blocks = sms * 8, threads = 256, iters = 1 << 14;
  DevBuf out;
  CK(out.ensure(sizeof(T) * blocks));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float best = 1e30f;
  for (int rep = 0; rep < 6; ++rep) {
    CK(cudaEventRecord(e0, ctx->stream));
    k_fma_peak<T><<<blocks, threads, 0, ctx->stream>>>(out.as<T>(), iters, T(0.999999), T(1e-7));
    CK(cudaEventRecord(e1, ctx->stream));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (rep > 0) best = std::min(best, ms);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  out.release();
  double flops = 2.0 * 8.0 * (double)iters * blocks * threads;
  *tflops = flops / (best * 1e-3) / 1e12;
  return TB_OK;
}

extern "C" int tb_measure_peak(tb_context *ctx, int precision, double *tflops) {
  if (!ctx || !tflops) return fail(ctx, TB_ERR_ARG, "null argument");
  CK(cudaSetDevice(ctx->device));
  return precision == TB_PREC_DOUBLE ? peak_t<double>(ctx, tflops) : peak_t<float>(ctx, tflops);
}

extern "C" const char *tb_version(void) { return "tersoff_b200 sm_100a " TB_VERSION_TAG; }

// copy a host or device array into a context buffer; returns the device pointer
template <class X>
static const X *stage_in(tb_context *ctx, const X *src, size_t count, DevBuf &buf, int &rc) {
  rc = TB_OK;
  if (is_device_ptr(src)) return src;
  if (buf.ensure(sizeof(X) * count) != cudaSuccess) {
    rc = fail(ctx, TB_ERR_CUDA, "device allocation of %zu bytes failed", sizeof(X) * count);
    return nullptr;
  }
  if (count &&
      cudaMemcpyAsync(buf.p, src, sizeof(X) * count, cudaMemcpyHostToDevice, ctx->stream) !=
          cudaSuccess) {
    rc = fail(ctx, TB_ERR_CUDA, "host-to-device copy failed");
    return nullptr;
  }
  return buf.as<X>();
}

// ---------------------------------------------------------------------------
// neighbour list (neighbor.py:194-217)
// ---------------------------------------------------------------------------

extern "C" int tb_nlist_create(tb_context *ctx, tb_nlist **out) {
  if (!ctx || !out) return TB_ERR_ARG;
  tb_nlist *nl = new tb_nlist();
  nl->ctx = ctx;
  *out = nl;
  return TB_OK;
}

extern "C" void tb_nlist_destroy(tb_nlist *nl) {
  if (!nl) return;
  cudaSetDevice(nl->ctx->device);
  cudaStreamSynchronize(nl->ctx->stream);
  DevBuf *bufs[] = {&nl->offsets, &nl->nbr, &nl->rev, &nl->ref_pos, &nl->atom_cell,
                    &nl->cell_count, &nl->cell_start, &nl->cell_atoms, &nl->row_count,
                    &nl->maxrow, &nl->nl_row, &nl->sorted_atoms, &nl->sort_keys,
                    &nl->iota, &nl->lanes, &nl->hist, &nl->cpos, &nl->crow, &nl->coff,
                    &nl->centry, &nl->fnbr, &nl->fbuf, &nl->plan, &nl->scratch, &nl->lplan,
                    &nl->llen, &nl->lrow, &nl->lrowj, &nl->lsorted, &nl->llanes, &nl->ref_log,
                    &nl->fspecies, &nl->lref, &nl->lgate, &nl->lforce, &nl->sp_lanes,
                    &nl->sp_tmp, &nl->crel};
  for (DevBuf *b : bufs) b->release();
  md_graph_release(nl);
  delete nl;
}

// exclusive prefix sum (tb_scan.cuh); the tile-sum scratch is context-owned
// and pre-sized by md_prepare before a graph capture
static int exclusive_scan(tb_context *ctx, const int *in, int *out, int64_t count) {
  CK(ctx->scan_tmp.ensure(sizeof(int) * (scan_tiles(count) + 4)));
  CK(scan_exclusive(in, out, count, ctx->scan_tmp.as<int>(), ctx->stream));
  return TB_OK;
}

// atoms sorted stably by row length into sorted_atoms (tb_scan.cuh)
static int sort_rows_by_length(tb_context *ctx, tb_nlist *nl, const int *row_len) {
  CK(ctx->scan_tmp.ensure(sizeof(int) * lsort_scratch((int)nl->n)));
  CK(sort_by_length(row_len, (int)nl->n, nl->sorted_atoms.as<int>(), ctx->scan_tmp.as<int>(),
                    ctx->stream));
  return TB_OK;
}

static int build_rev(tb_context *ctx, tb_nlist *nl) {
  CK(nl->rev.ensure(sizeof(int) * std::max<int64_t>(nl->ecap, 1)));
  if (nl->n)
    k_nl_reverse<<<nblk(nl->n, 256), 256, 0, ctx->stream>>>(
        (int)nl->n, nl->offsets.as<int>(), nl->nbr.as<int>(), nl->rev.as<int>());
  CK(cudaGetLastError());
  nl->rev_valid = true;
  return TB_OK;
}

constexpr int ROW_LM = 4;  // rows the atom-per-lane kernel takes (tb_row.cuh)

// where the rows of 1..ROW_LM entries and their chunks sit (hist = row-length histogram)
static void set_row_info(tb_nlist *nl, const int *hist) {
  nl->r4_first = hist[0];
  nl->r4_count = 0;
  nl->r4_chunks = 0;
  for (int L = 1; L <= ROW_LM; ++L) {
    nl->r4_count += hist[L];
    nl->r4_chunks += (hist[L] + 32 / L - 1) / (32 / L);
  }
}

// Warp chunks: rows sorted by length (stable radix sort -> deterministic),
// floor(32/L) rows of length L per warp.  row_len[i] = lanes of atom i; lane
// k of row i maps to entry coff[i] + k of centry (or offsets[i] + k when
// centry == nullptr).  hist = row-length histogram (hist[0] = empty rows).
static int build_chunks(tb_context *ctx, tb_nlist *nl, const int *row_len, const int *coff,
                        const int *centry, const int *hist) {
  const int N = (int)nl->n;
  CK(nl->sorted_atoms.ensure(sizeof(int) * N));
  int rcs = sort_rows_by_length(ctx, nl, row_len);  // stable -> deterministic chunks
  if (rcs) return rcs;
  ChunkPlan plan;
  memset(&plan, 0, sizeof(plan));
  int start = hist[0], chunks = 0;
  for (int L = 1; L <= 32; ++L) {
    plan.count[L] = hist[L];
    plan.bucket_start[L] = start;
    plan.chunk_base[L] = chunks;
    start += hist[L];
    chunks += (hist[L] + 32 / L - 1) / (32 / L);
  }
  plan.chunk_base[33] = chunks;
  set_row_info(nl, hist);
  nl->n_empty = hist[0];
  nl->lanes_used = 0;
  for (int L = 1; L <= 32; ++L) nl->lanes_used += (int64_t)L * hist[L];
  nl->ccap = chunks + (int64_t)(nl->margin * (double)chunks) + (nl->margin > 0 ? 64 : 0);
  if (chunks > 0) {
    CK(nl->lanes.ensure(sizeof(int4) * 32 * (size_t)nl->ccap));
    k_fill_lanes<<<nblk(chunks, 8), 256, 0, ctx->stream>>>(plan, nl->sorted_atoms.as<int>(),
                                                  coff ? coff : nl->offsets.as<int>(), centry,
                                                  nl->nbr.as<int>(), nl->lanes.as<int4>(), chunks);
    CK(cudaGetLastError());
  }
  nl->nchunks = chunks;
  nl->lanes_version++;
  return TB_OK;
}

// Stage plan of the streamed tb_compute (tb_stream.cuh): K ranges of R atoms,
// chunks sorted stably by stage into sp_lanes; cached per list version.
static int stream_plan(tb_context *ctx, tb_nlist *nl, int K, int R) {
  if (nl->sp_version == nl->lanes_version && nl->sp_K == K && nl->sp_R == R) return TB_OK;
  const int nc = nl->nchunks;
  // [stage nc | order nc | hist 34 | touch 32]
  CK(nl->sp_tmp.ensure(sizeof(int) * (2 * (size_t)nc + 34 + STREAM_KMAX)));
  int *stage = nl->sp_tmp.as<int>(), *order = stage + nc, *hist = order + nc;
  unsigned *touch = reinterpret_cast<unsigned *>(hist + 34);
  CK(nl->sp_lanes.ensure(sizeof(int4) * 32 * (size_t)nc));
  CK(ctx->scan_tmp.ensure(sizeof(int) * lsort_scratch(nc)));
  CK(cudaMemsetAsync(hist, 0, sizeof(int) * (34 + STREAM_KMAX), ctx->stream));
  k_chunk_stage<<<nblk(nc, 8), 256, 0, ctx->stream>>>(nl->lanes.as<int4>(), nc, R, stage, touch);
  k_len_hist<<<std::min(nblk(nc, 256), 592), 256, 0, ctx->stream>>>(nc, stage, hist);
  CK(sort_by_length(stage, nc, order, ctx->scan_tmp.as<int>(), ctx->stream));
  k_permute_chunks<<<nblk(nc, 8), 256, 0, ctx->stream>>>(nl->lanes.as<int4>(), order,
                                                         nl->sp_lanes.as<int4>(), nc);
  CK(cudaGetLastError());
  int h[34 + STREAM_KMAX];
  CK(cudaMemcpyAsync(h, hist, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  nl->sp_cstart.assign(K + 1, 0);
  for (int q = 0; q < K; ++q) nl->sp_cstart[q + 1] = nl->sp_cstart[q] + h[q];
  if (nl->sp_cstart[K] != nc) return fail(ctx, TB_ERR_CUDA, "internal error: stage plan");
  // a range's forces / per-atom energies are final after the last stage that
  // touches it; atoms with empty rows are written by the last launch
  nl->sp_fin.assign(K, nl->n_empty > 0 ? K - 1 : 0);
  for (int q = 0; q < K; ++q) {
    const unsigned m = (unsigned)h[34 + q];
    for (int r = 0; r < K; ++r)
      if (m >> r & 1u) nl->sp_fin[r] = std::max(nl->sp_fin[r], q);
  }
  nl->sp_version = nl->lanes_version;
  nl->sp_K = K;
  nl->sp_R = R;
  return TB_OK;
}

// Species-pair compute filter (S > 1): an entry (i,j) whose build-time
// distance exceeds need(si,sj) + skin can never become live before the next
// rebuild, need(si,sj) = max(R+D of pair (si,sj,sj), R+D of every (si,q,sj))
// -- it is exactly zero as a pair and as a k.  Such entries stay in the
// exported list (bit-exact pair set, zeta_visits) but get no warp lanes.
// Computed at the first evaluation after a build (species are known then).
static NeedTable need_table(const tb_context *ctx, const tb_nlist *nl) {
  const int S = ctx->S;
  NeedTable nt;
  float *need2 = nt.need2;
  for (int a = 0; a < S; ++a)
    for (int b = 0; b < S; ++b) {
      double nd = ctx->pair_mat[8 * (a * S + b)] + ctx->pair_mat[8 * (a * S + b) + 1];
      for (int q = 0; q < S; ++q) {
        const double *t = &ctx->trip_mat[8 * ((a * S + q) * S + b)];
        nd = std::max(nd, t[0] + t[1]);
      }
      const double c = nd + nl->skin;
      need2[a * 4 + b] = (float)(c * c * (1.0 + 1e-6));  // conservative (float table)
    }
  return nt;
}

static int build_filter(tb_context *ctx, tb_nlist *nl, const int *d_species) {
  const int N = (int)nl->n, S = ctx->S;
  CK(nl->crow.ensure(sizeof(int) * (N + 1)));
  CK(nl->coff.ensure(sizeof(int) * (N + 1)));
  CK(nl->centry.ensure(sizeof(int) * std::max<int64_t>(nl->ecap, 1)));
  CK(cudaMemsetAsync(nl->crow.p, 0, sizeof(int) * (N + 1), ctx->stream));
  Box b = make_box(nl->L, nl->per);
  const NeedTable nt = need_table(ctx, nl);
  k_filter_rows<false><<<nblk(N, 128), 128, 0, ctx->stream>>>(
      N, nl->ref_pos.as<double>(), d_species, S, nt, b, nl->offsets.as<int>(), nl->nbr.as<int>(),
      nl->crow.as<int>(), nullptr, nullptr);
  CK(cudaGetLastError());
  int rc = exclusive_scan(ctx, nl->crow.as<int>(), nl->coff.as<int>(), N + 1);
  if (rc) return rc;
  CK(nl->fnbr.ensure(sizeof(int) * std::max<int64_t>(nl->ecap, 1)));
  k_filter_rows<true><<<nblk(N, 128), 128, 0, ctx->stream>>>(
      N, nl->ref_pos.as<double>(), d_species, S, nt, b, nl->offsets.as<int>(), nl->nbr.as<int>(),
      nullptr, nl->coff.as<int>(), nl->centry.as<int>(), nl->fnbr.as<int>());
  nl->fnbr_ok = true;
  CK(cudaGetLastError());
  CK(cudaMemsetAsync(nl->hist.p, 0, sizeof(int) * 34, ctx->stream));
  k_len_hist<<<std::min(nblk(N, 256), 296), 256, 0, ctx->stream>>>(N, nl->crow.as<int>(),
                                                                    nl->hist.as<int>());
  CK(cudaGetLastError());
  int *hm = reinterpret_cast<int *>(ctx->h_small);
  CK(cudaMemcpyAsync(hm, nl->hist.p, sizeof(int) * 34, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  int hist[34];
  memcpy(hist, hm, sizeof(hist));
  rc = build_chunks(ctx, nl, nl->crow.as<int>(), nl->coff.as<int>(), nl->centry.as<int>(), hist);
  if (rc) return rc;
  CK(nl->fspecies.ensure(sizeof(int) * std::max(N, 1)));
  CK(cudaMemcpyAsync(nl->fspecies.p, d_species, sizeof(int) * N, cudaMemcpyDeviceToDevice,
                     ctx->stream));
  nl->filtered = true;
  nl->lvalid = false;
  nl->filter_species = d_species;
  nl->filter_param_version = ctx->param_version;
  nl->fbuf_zero = false;
  return TB_OK;
}

extern "C" int tb_build_neighbors(tb_context *ctx, tb_nlist *nl, int64_t n,
                                  const double *positions, const double *box,
                                  const int32_t *periodic, double r_cut, double skin) {
  return tb_build_neighbors_owned(ctx, nl, n, n, positions, box, periodic, r_cut, skin);
}

static int build_owned(tb_context *ctx, tb_nlist *nl, int64_t n, int64_t n_owned,
                       const double *positions, const double *box, const int32_t *periodic,
                       double r_cut, double skin, int cx_lo, int cx_hi);

extern "C" int tb_build_neighbors_owned(tb_context *ctx, tb_nlist *nl, int64_t n,
                                        int64_t n_owned, const double *positions,
                                        const double *box, const int32_t *periodic,
                                        double r_cut, double skin) {
  return build_owned(ctx, nl, n, n_owned, positions, box, periodic, r_cut, skin, 0, INT_MAX);
}

// cx_lo..cx_hi: x columns holding every owned atom (slab decomposition); the
// cell scan skips the others
static int build_owned(tb_context *ctx, tb_nlist *nl, int64_t n, int64_t n_owned,
                       const double *positions, const double *box, const int32_t *periodic,
                       double r_cut, double skin, int cx_lo, int cx_hi) {
  if (n_owned < 0 || n_owned > n) return fail(ctx, TB_ERR_ARG, "n_owned outside [0, n]");
  if (!ctx || !nl || !box || !periodic || (n && !positions))
    return fail(ctx, TB_ERR_ARG, "null argument");
  if (n > INT_MAX / 2) return fail(ctx, TB_ERR_ARG, "too many atoms (%lld)", (long long)n);
  CK(cudaSetDevice(ctx->device));
  // argument checks in the reference's order and wording (neighbor.py:195-207)
  if (skin < 0) return fail(ctx, TB_ERR_CONFIG, "negative skin %s", fmt_g(skin).c_str());
  const double bc = r_cut + skin;
  for (int ax = 0; ax < 3; ++ax) {
    if (!(box[ax] > 0))
      return fail(ctx, TB_ERR_CONFIG, "box edge lengths must be positive, got %g", box[ax]);
    if (periodic[ax] && box[ax] < 2.0 * bc)
      return fail(ctx, TB_ERR_CONFIG,
                  "periodic edge %s A along axis %d is shorter than twice the build cutoff "
                  "%s A; replicate the cell",
                  fmt_g(box[ax]).c_str(), ax, fmt_g(bc).c_str());
  }
  int rc;
  const double *d_pos = stage_in(ctx, positions, 3 * (size_t)n, ctx->pos, rc);
  if (rc) return rc;

  nl->n = n;
  for (int ax = 0; ax < 3; ++ax) {
    nl->L[ax] = box[ax];
    nl->per[ax] = periodic[ax] ? 1 : 0;
  }
  nl->r_cut = r_cut;
  nl->skin = skin;
  nl->bc = bc;
  nl->rev_valid = false;
  nl->imported = false;
  nl->lvalid = false;

  // ---- grid geometry (CellList.__init__, neighbor.py:54-81) ----
  Grid g;
  g.box = make_box(nl->L, nl->per);
  bool any_free = !(nl->per[0] && nl->per[1] && nl->per[2]);
  double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
  if (any_free && n) {
    CK(ctx->bounds.ensure(6 * sizeof(unsigned long long)));
    unsigned long long init[6] = {~0ull, ~0ull, ~0ull, 0, 0, 0};
    CK(cudaMemcpyAsync(ctx->bounds.p, init, sizeof(init), cudaMemcpyHostToDevice, ctx->stream));
    k_bounds<<<std::min(nblk(n, 256), 1184), 256, 0, ctx->stream>>>(
        n, d_pos, ctx->bounds.as<unsigned long long>());
    CK(cudaGetLastError());
    unsigned long long res[6];
    CK(cudaMemcpyAsync(res, ctx->bounds.p, sizeof(res), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    auto unkey = [](unsigned long long k) {
      unsigned long long u = (k & 0x8000000000000000ull) ? (k & ~0x8000000000000000ull) : ~k;
      double v;
      memcpy(&v, &u, 8);
      return v;
    };
    for (int ax = 0; ax < 3; ++ax) {
      lo[ax] = unkey(res[ax]);
      hi[ax] = unkey(res[3 + ax]);
    }
  }
  int64_t ncell = 1;
  for (int ax = 0; ax < 3; ++ax) {
    int64_t nc;
    if (nl->per[ax]) {
      if (nl->L[ax] < bc)
        return fail(ctx, TB_ERR_CONFIG,
                    "periodic edge %s A on axis %d is smaller than the cell size %s A",
                    fmt_g(nl->L[ax]).c_str(), ax, fmt_g(bc).c_str());
      nc = std::max<int64_t>((int64_t)(nl->L[ax] / bc), 1);
      g.origin[ax] = 0.0;
      g.width[ax] = nl->L[ax] / (double)nc;
    } else {
      g.origin[ax] = lo[ax];
      double span = (hi[ax] - lo[ax]) / bc;
      if (!(span < 1e7))
        return fail(ctx, TB_ERR_CONFIG, "free-axis extent %g A too large for the cell grid",
                    hi[ax] - lo[ax]);
      nc = std::max<int64_t>((int64_t)span + 1, 1);
      g.width[ax] = bc;
    }
    g.nc[ax] = (int)nc;
    ncell *= nc;
  }
  // stencil-implied minimum images (k_nl_cells): every periodic axis
  // needs >= 4 cells (merged z-runs never mix images) strictly wider than bc
  // (a pair within bc then lies in adjacent unwrapped cells)
  g.stencil_image = nl->per[0] && nl->per[1] && nl->per[2] ? 2 : 1;
  for (int ax = 0; ax < 3; ++ax)
    if (nl->per[ax] && !(g.nc[ax] >= 4 && g.width[ax] > bc * (1.0 + 1e-9))) g.stencil_image = 0;
  if (ncell > (int64_t)1 << 28)
    return fail(ctx, TB_ERR_CONFIG, "cell grid of %lld cells is too large", (long long)ncell);

  const int N = (int)n;
  // cells [c0, c1) are scanned (the slab's own x columns, or all)
  const int64_t nyz = ncell / g.nc[0];
  const int64_t c0 = (int64_t)std::min(std::max(cx_lo, 0), g.nc[0]) * nyz;
  const int64_t c1 = std::max<int64_t>(std::min<int64_t>((int64_t)std::min(cx_hi, g.nc[0] - 1) + 1,
                                                         g.nc[0]) * nyz, c0);
  CK(nl->atom_cell.ensure(sizeof(int) * std::max(N, 1)));
  CK(nl->cell_count.ensure(sizeof(int) * (ncell + 1)));
  CK(nl->cell_start.ensure(sizeof(int) * (ncell + 1)));
  CK(nl->cell_atoms.ensure(sizeof(int) * std::max(N, 1)));
  CK(nl->row_count.ensure(sizeof(int) * (N + 1)));
  CK(nl->offsets.ensure(sizeof(int) * (N + 1)));
  CK(nl->maxrow.ensure(2 * sizeof(int)));  // [max row, unwrapped-coordinate flag]
  CK(nl->ref_pos.ensure(sizeof(double) * 3 * std::max(N, 1)));

  CK(nl->hist.ensure(sizeof(int) * 34));
  CK(nl->scratch.ensure(sizeof(int) * TMPW * (size_t)std::max(N, 1)));
  CK(cudaMemsetAsync(nl->cell_count.p, 0, sizeof(int) * (ncell + 1), ctx->stream));
  CK(cudaMemsetAsync(nl->maxrow.p, 0, 2 * sizeof(int), ctx->stream));
  CK(cudaMemsetAsync(nl->hist.p, 0, sizeof(int) * 34, ctx->stream));
  CK(cudaMemsetAsync(nl->row_count.p, 0, sizeof(int) * (N + 1), ctx->stream));
  if (N) {
    k_cell_index<<<nblk(N, 256), 256, 0, ctx->stream>>>(N, d_pos, g, nl->atom_cell.as<int>(),
                                                         nl->cell_count.as<int>(),
                                                         nl->maxrow.as<int>() + 1);
    CK(cudaGetLastError());
  }
  rc = exclusive_scan(ctx, nl->cell_count.as<int>(), nl->cell_start.as<int>(), ncell + 1);
  if (rc) return rc;
  // cursor copy for the counting-sort scatter (cell_count reused as cursor)
  CK(cudaMemcpyAsync(nl->cell_count.p, nl->cell_start.p, sizeof(int) * (ncell + 1),
                     cudaMemcpyDeviceToDevice, ctx->stream));
  if (N) {
    k_cell_fill<<<nblk(N, 256), 256, 0, ctx->stream>>>(N, nl->atom_cell.as<int>(),
                                                        nl->cell_count.as<int>(),
                                                        nl->cell_atoms.as<int>());
    CK(cudaGetLastError());
    CK(nl->cpos.ensure(sizeof(double4) * N));
    k_cell_gather<<<nblk(N, 256), 256, 0, ctx->stream>>>(N, d_pos, nl->cell_atoms.as<int>(),
                                                          nl->cpos.as<double4>());
    CK(cudaGetLastError());
    // single pass: rows of <= TMPW entries land in the scratch rows, counts,
    // max row and the row-length histogram (for the warp chunks) come along
    if (c1 > c0 && g.stencil_image == 2 && ctx->nl_atoms) {
      CK(nl->crel.ensure(sizeof(float4) * N));
      k_cell_rel<<<nblk(N, 256), 256, 0, ctx->stream>>>(N, nl->cpos.as<double4>(),
                                                         nl->atom_cell.as<int>(), g,
                                                         nl->crel.as<float4>());
      k_nl_atoms<<<nblk(N, 256), 256, 0, ctx->stream>>>(
          (int)c0, (int)c1, (int)n_owned, nl->cpos.as<double4>(), g, bc * bc,
          nl->cell_start.as<int>(), nl->row_count.as<int>(), nl->scratch.as<int>(),
          nl->maxrow.as<int>(), nl->hist.as<int>(), nl->maxrow.as<int>() + 1,
          nl->crel.as<float4>());
    }
    else if (c1 > c0)
      k_nl_cells<<<nblk(c1 - c0, 8), 256, 0, ctx->stream>>>(
          (int)c1, (int)n_owned, nl->cpos.as<double4>(), g, bc * bc, nl->cell_start.as<int>(),
          nl->row_count.as<int>(), nl->scratch.as<int>(), nl->maxrow.as<int>(),
          nl->hist.as<int>(), nl->maxrow.as<int>() + 1, (int)c0);
    CK(cudaGetLastError());
  }
  rc = exclusive_scan(ctx, nl->row_count.as<int>(), nl->offsets.as<int>(), N + 1);
  if (rc) return rc;
  int *hm = reinterpret_cast<int *>(ctx->h_small);  // pinned: [entries, max_row, hist[34]]
  CK(cudaMemcpyAsync(&hm[0], nl->offsets.as<int>() + N, sizeof(int), cudaMemcpyDeviceToHost,
                     ctx->stream));
  CK(cudaMemcpyAsync(&hm[1], nl->maxrow.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(&hm[2], nl->hist.p, sizeof(int) * 34, cudaMemcpyDeviceToHost, ctx->stream));
  const bool partial = c0 > 0 || c1 < ncell;
  if (partial) {  // atoms of the unscanned cells (ghosts) have empty rows too
    CK(cudaMemcpyAsync(&hm[36], nl->cell_start.as<int>() + c0, sizeof(int), cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaMemcpyAsync(&hm[37], nl->cell_start.as<int>() + c1, sizeof(int), cudaMemcpyDeviceToHost,
                       ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  nl->entries = hm[0];
  nl->max_row = hm[1];
  int hist[34];
  memcpy(hist, hm + 2, sizeof(hist));
  if (partial) hist[0] += N - (hm[37] - hm[36]);
  // entry-sized buffers carry a margin so that the device-resident rebuild
  // (tb_md_run) can regrow the list in place
  if (nl->margin < 0) nl->margin = ctx->list_margin;
  nl->ecap = nl->entries + (int64_t)(nl->margin * (double)nl->entries) + (nl->margin > 0 ? 256 : 0);
  nl->grid = g;
  nl->ncell = ncell;
  CK(nl->nbr.ensure(sizeof(int) * nl->ecap));
  if (N && nl->max_row <= TMPW) {
    k_nl_compact<SCAN_G><<<nblk((int64_t)N * SCAN_G, 256), 256, 0, ctx->stream>>>(
        N, nl->scratch.as<int>(), nl->row_count.as<int>(), nl->offsets.as<int>(),
        nl->nbr.as<int>(), nullptr, nullptr);
    CK(cudaGetLastError());
  } else if (N) {
    // rows longer than the scratch rows: second full scan straight into CSR
    k_nl_scan<true><<<nblk(N, 128), 128, 0, ctx->stream>>>(
        N, (int)n_owned, nl->cpos.as<double4>(), g, bc * bc, nl->atom_cell.as<int>(), nl->cell_start.as<int>(),
        nl->cell_atoms.as<int>(), nullptr, nl->offsets.as<int>(), nl->nbr.as<int>(), nullptr,
        nullptr);
    CK(cudaGetLastError());
  }
  if (N) {
    CK(cudaMemcpyAsync(nl->ref_pos.p, d_pos, sizeof(double) * 3 * N, cudaMemcpyDeviceToDevice,
                       ctx->stream));
  }
  // warp chunks for the fast kernel (tb_warp.cuh) over the full rows; a
  // species-pair compute filter may replace them at the first evaluation
  nl->filter_species = nullptr;
  nl->filtered = false;
  nl->fbuf_zero = false;
  if (nl->max_row <= 32 && N > 0) {
    int rc2 = build_chunks(ctx, nl, nl->row_count.as<int>(), nullptr, nullptr, hist);
    if (rc2) return rc2;
  } else {
    nl->nchunks = 0;
    nl->r4_count = 0;
    nl->lanes_version++;
    nl->n_empty = 0;
  }
  nl->built = true;
  return TB_OK;
}

// Import a CSR list built elsewhere (the reference's NeighborList:
// offsets/neighbors int64, neighbor.py:170-191) so the reference's own callers
// can run the B200 kernels on their list.  The rows are taken as given (the
// evaluation re-tests r < r_cut, like pack_adjacency); warp chunks are built
// from the row lengths.  Imported lists have no cell grid: the device rebuild
// paths (tb_nlist_rebuild_device, tb_md_run) refuse them.
extern "C" int tb_nlist_import(tb_context *ctx, tb_nlist *nl, int64_t n, const int64_t *offsets,
                               const int64_t *neighbors, const double *ref_positions,
                               const double *box, const int32_t *periodic, double r_cut,
                               double skin) {
  if (!ctx || !nl || !offsets || !box || !periodic || (n && !ref_positions))
    return fail(ctx, TB_ERR_ARG, "null argument");
  if (n < 0 || n > INT_MAX / 2) return fail(ctx, TB_ERR_ARG, "bad atom count %lld", (long long)n);
  if (skin < 0) return fail(ctx, TB_ERR_CONFIG, "negative skin %s", fmt_g(skin).c_str());
  CK(cudaSetDevice(ctx->device));
  const int N = (int)n;
  std::vector<int64_t> off(N + 1);
  if (is_device_ptr(offsets))
    CK(cudaMemcpy(off.data(), offsets, sizeof(int64_t) * (N + 1), cudaMemcpyDeviceToHost));
  else
    memcpy(off.data(), offsets, sizeof(int64_t) * (N + 1));
  const int64_t m = off[N];
  if (off[0] != 0 || m < 0 || m > INT_MAX)
    return fail(ctx, TB_ERR_ARG, "offsets must start at 0 and end at the entry count");
  std::vector<int> row(N + 1, 0), off32(N + 1, 0);
  int hist[34] = {0};
  int64_t max_row = 0;
  for (int i = 0; i < N; ++i) {
    const int64_t len = off[i + 1] - off[i];
    if (len < 0) return fail(ctx, TB_ERR_ARG, "offsets decrease at row %d", i);
    row[i] = (int)len;
    off32[i] = (int)off[i];
    max_row = std::max(max_row, len);
    if (len <= 32) hist[len] += 1;
  }
  off32[N] = (int)m;
  std::vector<int64_t> nb64(std::max<int64_t>(m, 1));
  if (m) {
    if (!neighbors) return fail(ctx, TB_ERR_ARG, "null neighbors");
    if (is_device_ptr(neighbors))
      CK(cudaMemcpy(nb64.data(), neighbors, sizeof(int64_t) * m, cudaMemcpyDeviceToHost));
    else
      memcpy(nb64.data(), neighbors, sizeof(int64_t) * m);
  }
  std::vector<int> nb(std::max<int64_t>(m, 1), 0);
  for (int64_t e = 0; e < m; ++e) {
    if (nb64[e] < 0 || nb64[e] >= n)
      return fail(ctx, TB_ERR_ARG, "neighbour index %lld out of range", (long long)nb64[e]);
    nb[e] = (int)nb64[e];
  }
  md_graph_release(nl);
  nl->n = n;
  for (int ax = 0; ax < 3; ++ax) {
    if (!(box[ax] > 0))
      return fail(ctx, TB_ERR_CONFIG, "box edge lengths must be positive, got %g", box[ax]);
    nl->L[ax] = box[ax];
    nl->per[ax] = periodic[ax] ? 1 : 0;
  }
  nl->r_cut = r_cut;
  nl->skin = skin;
  nl->bc = r_cut + skin;
  nl->entries = m;
  nl->max_row = max_row;
  nl->margin = 0.0;
  nl->ecap = std::max<int64_t>(m, 1);
  nl->ncell = 0;
  nl->imported = true;
  nl->lvalid = false;
  nl->rev_valid = false;
  nl->filtered = false;
  nl->filter_species = nullptr;
  nl->fbuf_zero = false;
  CK(nl->offsets.ensure(sizeof(int) * (N + 1)));
  CK(nl->row_count.ensure(sizeof(int) * (N + 1)));
  CK(nl->nbr.ensure(sizeof(int) * nl->ecap));
  CK(nl->ref_pos.ensure(sizeof(double) * 3 * std::max(N, 1)));
  CK(nl->hist.ensure(sizeof(int) * 34));
  CK(cudaMemcpyAsync(nl->offsets.p, off32.data(), sizeof(int) * (N + 1), cudaMemcpyHostToDevice,
                     ctx->stream));
  CK(cudaMemcpyAsync(nl->row_count.p, row.data(), sizeof(int) * (N + 1), cudaMemcpyHostToDevice,
                     ctx->stream));
  CK(cudaMemcpyAsync(nl->nbr.p, nb.data(), sizeof(int) * std::max<int64_t>(m, 1),
                     cudaMemcpyHostToDevice, ctx->stream));
  if (N)
    CK(cudaMemcpyAsync(nl->ref_pos.p, ref_positions, sizeof(double) * 3 * N,
                       is_device_ptr(ref_positions) ? cudaMemcpyDeviceToDevice
                                                    : cudaMemcpyHostToDevice,
                       ctx->stream));
  if (max_row <= 32 && N > 0) {
    int rc = build_chunks(ctx, nl, nl->row_count.as<int>(), nullptr, nullptr, hist);
    if (rc) return rc;
  } else {
    nl->nchunks = 0;
    nl->r4_count = 0;
    nl->lanes_version++;
    nl->n_empty = 0;
  }
  CK(cudaStreamSynchronize(ctx->stream));  // host staging vectors go out of scope
  nl->built = true;
  return TB_OK;
}

extern "C" int tb_nlist_refilter(tb_context *ctx, tb_nlist *nl) {
  if (!ctx || !nl) return fail(ctx, TB_ERR_ARG, "null argument");
  nl->filtered = false;  // rebuilt for the current species at the next evaluation
  return TB_OK;
}

extern "C" int tb_nlist_info(const tb_nlist *nl, int64_t *n_atoms, int64_t *n_entries,
                             int64_t *max_row) {
  if (!nl) return TB_ERR_ARG;
  if (n_atoms) *n_atoms = nl->n;
  if (n_entries) *n_entries = nl->entries;
  if (max_row) *max_row = nl->max_row;
  return TB_OK;
}

extern "C" int tb_nlist_lanes(const tb_nlist *nl, int64_t *nchunks, int64_t *lanes_used) {
  if (!nl || !nchunks || !lanes_used) return TB_ERR_ARG;
  *nchunks = nl->nchunks;
  *lanes_used = nl->nchunks > 0 ? nl->lanes_used : 0;
  return TB_OK;
}

extern "C" int tb_nlist_export(tb_context *ctx, const tb_nlist *nl, int64_t *offsets,
                               int64_t *neighbors) {
  if (!ctx || !nl || !nl->built) return fail(ctx, TB_ERR_ARG, "neighbour list not built");
  CK(cudaSetDevice(ctx->device));
  struct Part {
    const int *src;
    int64_t count;
    int64_t *dst;
  } parts[2] = {{nl->offsets.as<int>(), nl->n + 1, offsets},
                {nl->nbr.as<int>(), nl->entries, neighbors}};
  for (auto &pt : parts) {
    if (!pt.dst || pt.count == 0) continue;
    int64_t *d = pt.dst;
    DevBuf tmp;
    bool dev = is_device_ptr(pt.dst);
    if (!dev) {
      CK(tmp.ensure(sizeof(int64_t) * pt.count));
      d = tmp.as<int64_t>();
    }
    k_export_i64<<<nblk(pt.count, 256), 256, 0, ctx->stream>>>((int)pt.count, pt.src, d);
    CK(cudaGetLastError());
    if (!dev) {
      CK(cudaMemcpyAsync(pt.dst, d, sizeof(int64_t) * pt.count, cudaMemcpyDeviceToHost,
                         ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
      tmp.release();
    }
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return TB_OK;
}

static int drift_check(tb_context *ctx, const tb_nlist *nl, const double *d_pos, int32_t *out) {
  CK(ctx->drift.ensure(sizeof(unsigned long long)));
  CK(cudaMemsetAsync(ctx->drift.p, 0, sizeof(unsigned long long), ctx->stream));
  if (nl->n) {
    k_max_drift<<<std::min(nblk(nl->n, 256), 1184), 256, 0, ctx->stream>>>(
        (int)nl->n, d_pos, nl->ref_pos.as<double>(), make_box(nl->L, nl->per),
        ctx->drift.as<unsigned long long>());
    CK(cudaGetLastError());
  }
  unsigned long long *h = reinterpret_cast<unsigned long long *>(ctx->h_small);
  CK(cudaMemcpyAsync(h, ctx->drift.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                     ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  double mx;
  memcpy(&mx, h, 8);
  double half = 0.5 * nl->skin;
  *out = mx > half * half ? 1 : 0;
  return TB_OK;
}

extern "C" int tb_needs_rebuild(tb_context *ctx, const tb_nlist *nl, const double *positions,
                                int32_t *out) {
  if (!ctx || !nl || !out || (nl->n && !positions)) return fail(ctx, TB_ERR_ARG, "null argument");
  if (!nl->built) return fail(ctx, TB_ERR_ARG, "neighbour list not built");
  CK(cudaSetDevice(ctx->device));
  int rc;
  const double *d_pos = stage_in(ctx, positions, 3 * (size_t)nl->n, ctx->pos, rc);
  if (rc) return rc;
  return drift_check(ctx, nl, d_pos, out);
}

// ---------------------------------------------------------------------------
// the Tersoff evaluation
// ---------------------------------------------------------------------------

template <class T, int S, bool LAM3, int MODE>
static int launch_tersoff_t(tb_context *ctx, const tb_nlist *nl, KArgs &a, int C) {
  size_t smem = SmemLayout<T, S>::bytes(C, S > 0 ? S : ctx->S);
  DynTab dyn;
  dyn.nspecies = ctx->S;
  dyn.pair = sizeof(T) == 8 ? ctx->dyn_pair64.p : ctx->dyn_pair32.p;
  dyn.trip = sizeof(T) == 8 ? ctx->dyn_trip64.p : ctx->dyn_trip32.p;
  if (smem > 220 * 1024)
    return fail(ctx, TB_ERR_CONFIG, "neighbour rows of %lld entries exceed the kernel's staging",
                (long long)nl->max_row);
  auto kern = k_tersoff<T, S, LAM3, MODE>;
  // opt in to the dynamic shared memory this launch needs (per instantiation)
  static size_t opted = 48 * 1024;
  if (smem > opted) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    opted = smem;
  }
  int nb = nblk(a.n, a.atoms_per_block);
  Tables<T, S> tab = make_tables<T, S>(ctx);
  std::pair<cudaEvent_t, cudaEvent_t> ev{nullptr, nullptr};
  if (ctx->profile) {
    if (ctx->ev_free.empty()) {
      CK(cudaEventCreate(&ev.first));
      CK(cudaEventCreate(&ev.second));
    } else {
      ev = ctx->ev_free.back();
      ctx->ev_free.pop_back();
    }
    CK(cudaEventRecord(ev.first, ctx->stream));
  }
  kern<<<nb, NT, smem, ctx->stream>>>(a, tab, C, dyn);
  CK(cudaGetLastError());
  if (ctx->profile) {
    CK(cudaEventRecord(ev.second, ctx->stream));
    ctx->ev_used.push_back(ev);
  }
  return TB_OK;
}

template <class T, int S, bool LAM3, int MODE, bool ST>
static int launch_warp_t(tb_context *ctx, const tb_nlist *nl, KArgs &a, WArgs &w) {
  auto kern = k_tersoff_warp<T, S, LAM3, MODE, ST>;
  static int per_sm = 0;
  if (!per_sm) {
    // all of the unified L1/shared array as shared memory: occupancy is set
    // by registers and the per-warp staging, not by a small default carveout
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                            cudaSharedmemCarveoutMaxShared));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, WarpCfg<T>::nt, 0));
    per_sm = std::max(per_sm, 1);
  }
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
  int need = nblk(w.nchunks, WarpCfg<T>::wpb);
  // persistent grid: one resident wave, warps stride over the chunks
  int nb = std::max(1, ctx->warp_per_chunk ? need : std::min(need, sms * per_sm));
  if (ctx->part_off == 0) CK(ctx->partials.ensure(sizeof(double) * 8 * nb));
  // (streamed stages: pre-sized by the caller, one slot range per launch)
  a.partials = ctx->partials.as<double>() + 8 * (int64_t)ctx->part_off;
  Tables<T, S> tab = make_tables<T, S>(ctx);
  std::pair<cudaEvent_t, cudaEvent_t> ev{nullptr, nullptr};
  if (ctx->profile) {
    if (ctx->ev_free.empty()) {
      CK(cudaEventCreate(&ev.first));
      CK(cudaEventCreate(&ev.second));
    } else {
      ev = ctx->ev_free.back();
      ctx->ev_free.pop_back();
    }
    CK(cudaEventRecord(ev.first, ctx->stream));
  }
  kern<<<nb, WarpCfg<T>::nt, 0, ctx->stream>>>(a, w, tab);
  ctx->last_blocks = nb;
  CK(cudaGetLastError());
  if (ctx->profile) {
    CK(cudaEventRecord(ev.second, ctx->stream));
    ctx->ev_used.push_back(ev);
  }
  return TB_OK;
}

// atom-per-lane kernel for the rows of 1..ROW_LM entries (tb_row.cuh)
template <class T, int MODE, bool ST>
static int launch_row_t(tb_context *ctx, KArgs &a, const RArgs &r, int cap) {
  auto kern = k_tersoff_row<T, ROW_LM, MODE, ST>;
  static int per_sm = 0;
  if (!per_sm) {
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, RowCfg<T>::nt, 0));
    per_sm = std::max(per_sm, 1);
  }
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
  const int nb = std::max(1, std::min(nblk(cap, RowCfg<T>::nt), sms * per_sm));
  if (ctx->part_off == 0) CK(ctx->partials.ensure(sizeof(double) * 8 * nb));
  a.partials = ctx->partials.as<double>() + 8 * (int64_t)ctx->part_off;
  Tables<T, 1> tab = make_tables<T, 1>(ctx);
  std::pair<cudaEvent_t, cudaEvent_t> ev{nullptr, nullptr};
  if (ctx->profile) {
    if (ctx->ev_free.empty()) {
      CK(cudaEventCreate(&ev.first));
      CK(cudaEventCreate(&ev.second));
    } else {
      ev = ctx->ev_free.back();
      ctx->ev_free.pop_back();
    }
    CK(cudaEventRecord(ev.first, ctx->stream));
  }
  constexpr int bs = (int)(offsetof(DevPlan, bucket_start) / sizeof(int));
  kern<<<nb, RowCfg<T>::nt, 0, ctx->stream>>>(a, r, tab, bs + 1, bs + ROW_LM + 1);
  ctx->last_blocks = nb;
  CK(cudaGetLastError());
  if (ctx->profile) {
    CK(cudaEventRecord(ev.second, ctx->stream));
    ctx->ev_used.push_back(ev);
  }
  return TB_OK;
}

static int launch_row(tb_context *ctx, KArgs &a, const RArgs &r, int cap, int precision, int mode,
                      bool stats) {
  if (precision == TB_PREC_DOUBLE) {
    if (mode) return stats ? launch_row_t<double, 1, true>(ctx, a, r, cap)
                           : launch_row_t<double, 1, false>(ctx, a, r, cap);
    return stats ? launch_row_t<double, 0, true>(ctx, a, r, cap)
                 : launch_row_t<double, 0, false>(ctx, a, r, cap);
  }
  if (mode) return stats ? launch_row_t<float, 1, true>(ctx, a, r, cap)
                         : launch_row_t<float, 1, false>(ctx, a, r, cap);
  return stats ? launch_row_t<float, 0, true>(ctx, a, r, cap)
               : launch_row_t<float, 0, false>(ctx, a, r, cap);
}

template <class T, int S, int MODE>
static int launch_warp_m(tb_context *ctx, const tb_nlist *nl, KArgs &a, WArgs &w, bool stats) {
  if (ctx->lam3)
    return stats ? launch_warp_t<T, S, true, MODE, true>(ctx, nl, a, w)
                 : launch_warp_t<T, S, true, MODE, false>(ctx, nl, a, w);
  return stats ? launch_warp_t<T, S, false, MODE, true>(ctx, nl, a, w)
               : launch_warp_t<T, S, false, MODE, false>(ctx, nl, a, w);
}

template <class T>
static int launch_warp_prec(tb_context *ctx, const tb_nlist *nl, KArgs &a, WArgs &w, int mode,
                            bool stats) {
  switch (ctx->S) {
    case 1:
      return mode ? launch_warp_m<T, 1, 1>(ctx, nl, a, w, stats)
                  : launch_warp_m<T, 1, 0>(ctx, nl, a, w, stats);
    case 2:
      return mode ? launch_warp_m<T, 2, 1>(ctx, nl, a, w, stats)
                  : launch_warp_m<T, 2, 0>(ctx, nl, a, w, stats);
  }
  return fail(ctx, TB_ERR_CONFIG, "warp kernel: unsupported species count %d", ctx->S);
}

template <class T, int S>
static int launch_s(tb_context *ctx, const tb_nlist *nl, KArgs &a, int C, int mode) {
  if (ctx->lam3)
    return mode ? launch_tersoff_t<T, S, true, 1>(ctx, nl, a, C)
                : launch_tersoff_t<T, S, true, 0>(ctx, nl, a, C);
  return mode ? launch_tersoff_t<T, S, false, 1>(ctx, nl, a, C)
              : launch_tersoff_t<T, S, false, 0>(ctx, nl, a, C);
}

template <class T>
static int launch_prec(tb_context *ctx, const tb_nlist *nl, KArgs &a, int C, int mode) {
  switch (ctx->S) {
    case 1: return launch_s<T, 1>(ctx, nl, a, C, mode);
    case 2: return launch_s<T, 2>(ctx, nl, a, C, mode);
    case 3: return launch_s<T, 3>(ctx, nl, a, C, mode);
    case 4: return launch_s<T, 4>(ctx, nl, a, C, mode);
  }
  if (ctx->S <= SDYN_MAX) return launch_s<T, 0>(ctx, nl, a, C, mode);  // runtime species count
  return fail(ctx, TB_ERR_CONFIG, "unsupported species count %d", ctx->S);
}

static ErrFlags err_init() {
  ErrFlags e;
  e.nonfinite_atom = INT_MAX;
  e.bad_species_atom = INT_MAX;
  e.coinc_key = ~0ull;
  e.overflow = 0;
  e.stale_filter = 0;
  return e;
}

static int reset_errors(tb_context *ctx) {
  static_assert(sizeof(ErrFlags) <= 64, "result block layout");
  CK(ctx->errf.ensure(256));  // [ErrFlags | tb_compute result @64 | stats @128]
  ctx->err_unchecked = false;
  *ctx->h_err = err_init();
  CK(cudaMemcpyAsync(ctx->errf.p, ctx->h_err, sizeof(ErrFlags), cudaMemcpyHostToDevice,
                     ctx->stream));
  return TB_OK;
}

// Live repack of the warp chunks (pack_adjacency at the evaluation's
// positions, neighbor.py:330-360): every row is cut to its entries with
// r^2 < r_cut^2 -- the same exact arithmetic as the kernel's own test -- and
// the rows are re-bucketed by live length into warp chunks, all on the device
// (k_live_rows, then the tb_md_run plan kernels).  Rows of the skin list that
// are mostly dead (SiC: 12 Si-Si second neighbours at 3.08 A just outside the
// 3.0 A cutoff) then no longer occupy idle lanes.
// buffers of the live repack (sized before a graph capture by md_prepare)
static int live_reserve(tb_context *ctx, tb_nlist *nl, bool filtered) {
  const int N = (int)nl->n;
  const int64_t ent = filtered ? nl->ecap : std::max<int64_t>(nl->ecap, nl->entries);
  // chunk bound: a bucket of length L holds floor(32/L) rows of L lanes, and
  // floor(32/L) * L >= 17 for every L <= 32, so chunks <= entries / 17 + 34
  const int64_t cap = ent / 17 + 34;
  CK(nl->lplan.ensure(sizeof(DevPlan)));
  CK(nl->llen.ensure(sizeof(int) * std::max(N, 1)));
  CK(nl->lrow.ensure(sizeof(int) * std::max<int64_t>(ent, 1)));
  CK(nl->lrowj.ensure(sizeof(int) * std::max<int64_t>(ent, 1)));
  CK(nl->lsorted.ensure(sizeof(int) * std::max(N, 1)));
  if (nl->lcap < cap) {
    CK(nl->llanes.ensure(sizeof(int4) * 32 * cap));
    nl->lcap = cap;
    nl->lvalid = false;
  }
  if (ctx->repack_margin > 0) {
    CK(nl->lref.ensure(sizeof(double) * 3 * std::max(N, 1)));
    CK(nl->lgate.ensure(16));
  }
  return TB_OK;
}

static int live_repack(tb_context *ctx, tb_nlist *nl, const double *d_pos, double r_cut,
                       bool filtered, const Box &box, ErrFlags *err) {
  const int N = (int)nl->n;
  int rr = live_reserve(ctx, nl, filtered);
  if (rr) return rr;
  DevPlan *plan = nl->lplan.as<DevPlan>();
  const int *start = filtered ? nl->coff.as<int>() : nl->offsets.as<int>();
#ifndef TB_LIVE_G
#define TB_LIVE_G 2  // measured at c3: G = 1/2/4/8/16 -> step 364/347/353/370/416 us
#endif
  constexpr int G = TB_LIVE_G;  // lanes per row
  // Margin repack (TB_OPT_REPACK_MARGIN = delta): rows cut to r < r_cut + delta,
  // redone only when some atom moved more than delta/2 since the last repack
  // (a two-level Verlet list: every pair with r < r_cut now was within
  // r_cut + delta then).  The kernel's own exact r < r_cut test picks the live
  // set, so the terms are those of an exact repack (dead lanes add exact
  // zeros).  The decision is made on the device (no host round trip).
  const double margin = ctx->repack_margin;
  const int *go = nullptr;
  double *lref = nullptr;
  if (margin > 0) {
    unsigned long long *dbits = nl->lgate.as<unsigned long long>();
    int *gop = reinterpret_cast<int *>(dbits + 1);
    // inside tb_md_run's graph the list may be rebuilt on the device: the
    // rebuild raises lforce and the gate repacks unconditionally then
    const bool in_graph = ctx->dplan != nullptr;
    const bool force = !in_graph && (!nl->lvalid || nl->lmargin != margin || nl->lfilt != filtered);
    CK(cudaMemsetAsync(dbits, 0, sizeof(unsigned long long), ctx->stream));
    if (!force && N)
      k_max_drift<<<std::min(nblk(N, 256), 4 * 148), 256, 0, ctx->stream>>>(
          N, d_pos, nl->lref.as<double>(), box, dbits);
    k_repack_gate<<<1, 128, 0, ctx->stream>>>(dbits, 0.25 * margin * margin, force ? 1 : 0,
                                               in_graph ? nl->lforce.as<int>() : nullptr, gop,
                                               plan);
    CK(cudaGetLastError());
    go = gop;
    lref = nl->lref.as<double>();
  } else {
    CK(cudaMemsetAsync(plan, 0, sizeof(DevPlan), ctx->stream));
  }
  const double cut = r_cut + std::max(margin, 0.0);
  if (filtered)
    k_live_rows<true, G><<<nblk((int64_t)N * G, 256), 256, 0, ctx->stream>>>(
        N, d_pos, box, cut * cut, start, nl->crow.as<int>(), nl->centry.as<int>(),
        nl->fnbr.as<int>(), nl->llen.as<int>(), nl->lrow.as<int>(), nl->lrowj.as<int>(), err, go,
        lref);
  else
    k_live_rows<false, G><<<nblk((int64_t)N * G, 256), 256, 0, ctx->stream>>>(
        N, d_pos, box, cut * cut, start, nullptr, nullptr, nl->nbr.as<int>(), nl->llen.as<int>(),
        nl->lrow.as<int>(), nl->lrowj.as<int>(), err, go, lref);
  CK(cudaGetLastError());
  k_len_hist_plan<<<std::min(nblk(N, 256), 296), 256, 0, ctx->stream>>>(N, nl->llen.as<int>(), plan,
                                                                          go);
  k_plan<<<1, 32, 0, ctx->stream>>>(plan, nullptr, N, 0, (int)nl->lcap, go);
  k_bucket_fill<<<nblk(N, 256), 256, 0, ctx->stream>>>(N, nl->llen.as<int>(), start,
                                                       nl->lrow.as<int>(), nl->lrowj.as<int>(),
                                                       plan, nl->lsorted.as<int>(),
                                                       nl->llanes.as<int4>(), go);
  CK(cudaGetLastError());
  nl->lvalid = true;
  nl->lmargin = margin;
  nl->lfilt = filtered;
  return TB_OK;
}

// enqueue the evaluation; every pointer is a device pointer
static int enqueue_compute(tb_context *ctx, const tb_nlist *nl, const double *d_pos,
                           const int *d_species, double r_cut, int precision, int scatter,
                           double *d_forces, double *d_per_atom, double *d_result,
                           unsigned long long *d_stats, bool direct_ok = true) {
  if (ctx->S == 0) return fail(ctx, TB_ERR_CONFIG, "parameters not set");
  if (!nl->built) return fail(ctx, TB_ERR_ARG, "neighbour list not built");
  if (r_cut > nl->r_cut)
    return fail(ctx, TB_ERR_CONFIG,
                "cutoff %s A exceeds the %s A the neighbor list was built for",
                fmt_g(r_cut).c_str(), fmt_g(nl->r_cut).c_str());
  if (precision != TB_PREC_DOUBLE && precision != TB_PREC_MIXED)
    return fail(ctx, TB_ERR_ARG, "unknown precision %d", precision);
  if (scatter != TB_SCATTER_ATOMIC && scatter != TB_SCATTER_GATHER)
    return fail(ctx, TB_ERR_ARG, "unknown scatter mode %d", scatter);
  if (!ctx->errf.p) {
    int rc = reset_errors(ctx);
    if (rc) return rc;
  }
  ctx->err_unchecked = true;  // kernels below may raise flags (tb_compute reads them back)
  const int n = (int)nl->n;
  // tile sizing: atoms per block so that the tile's skin-list rows fit
  int C = SLOT_CAP;
  int maxrow = (int)std::max<int64_t>(nl->max_row, 1);
  if (maxrow > C) C = (maxrow + 31) & ~31;
  int A = std::max(1, std::min(NT, C / maxrow));
  int nb = n ? nblk(n, A) : 0;
  CK(ctx->partials.ensure(sizeof(double) * 8 * std::max(nb, 1)));
  if (scatter == TB_SCATTER_GATHER) {
    if (!nl->rev_valid) {
      int rc = build_rev(ctx, const_cast<tb_nlist *>(nl));
      if (rc) return rc;
    }
    tb_nlist *nlm = const_cast<tb_nlist *>(nl);
    CK(nlm->fbuf.ensure(sizeof(double) * 3 * std::max<int64_t>(nl->ecap, 1)));
  }
  // warp-chunk kernel for rows <= 32 entries and <= 2 species; else the tile kernel
  const bool warp_path = nl->nchunks > 0 && !ctx->force_tile && ctx->S <= 2;
  if (warp_path && ctx->S > 1 && !ctx->no_filter &&
      (!nl->filtered || nl->filter_species != d_species ||
       nl->filter_param_version != ctx->param_version)) {
    int rc = build_filter(ctx, const_cast<tb_nlist *>(nl), d_species);
    if (rc) return rc;
  }
  const bool filtered = warp_path && nl->filtered;
  if (filtered && !ctx->dplan && n > 0) {
    // same pointer, changed contents: latch stale_filter (tb_compute rebuilds
    // the filter and re-evaluates; tb_check_errors reports it)
    k_species_guard<<<std::min(nblk(n, 256), 2 * 148), 256, 0, ctx->stream>>>(
        n, d_species, nl->fspecies.as<int>(), ctx->errf.as<ErrFlags>());
    CK(cudaGetLastError());
  }
  if (scatter == TB_SCATTER_GATHER && filtered && !nl->fbuf_zero) {
    // entries the filter gave no lane are never written: zero them once per build
    CK(cudaMemsetAsync(nl->fbuf.p, 0, sizeof(double) * 3 * std::max<int64_t>(nl->entries, 1),
                       ctx->stream));
    const_cast<tb_nlist *>(nl)->fbuf_zero = true;
  }
  // force accumulator and stats counters: zero once, left zeroed by k_finalize
  if (ctx->facc_n < n) {
    CK(ctx->facc.ensure(sizeof(double) * 3 * std::max(n, 1)));
    CK(cudaMemsetAsync(ctx->facc.p, 0, sizeof(double) * 3 * std::max(n, 1), ctx->stream));
    ctx->facc_n = n;
  }
  if (!ctx->stats_acc.p) {
    CK(ctx->stats_acc.ensure(sizeof(unsigned long long) * TB_NSTATS));
    CK(cudaMemsetAsync(ctx->stats_acc.p, 0, sizeof(unsigned long long) * TB_NSTATS, ctx->stream));
  }
  if (n == 0) {
    CK(cudaMemsetAsync(d_result, 0, sizeof(double) * 7, ctx->stream));
    if (d_stats) CK(cudaMemsetAsync(d_stats, 0, sizeof(unsigned long long) * TB_NSTATS, ctx->stream));
    return TB_OK;
  }
  KArgs a;
  a.n = n;
  a.atoms_per_block = A;
  a.rc2 = r_cut * r_cut;
  a.box = make_box(nl->L, nl->per);
  a.pos = d_pos;
  a.species = d_species;
  a.off = nl->offsets.as<int>();
  a.nbr = nl->nbr.as<int>();
  // Atomic scatter into a device force array: the kernels accumulate straight
  // into the caller's array after one memset (24 B/atom written), instead of
  // into the context accumulator that the finalize copies out and re-zeroes
  // (24 B read + 48 B written per atom; config 5: ~200 -> ~60 us).  Starting
  // from +0.0, a sum of forces cannot come out as -0.0, so the reference's
  // +0.0 flush holds without the copy.  Host-mapped outputs (tb_compute with
  // pinned buffers) and the fused MD graph keep the accumulator.
  // (below ~256k atoms the extra memset node costs more than the copy it
  // saves: config 2 step 24.9 -> 26.7 us; config 5 2.86 -> 2.60 ms)
  const bool direct = direct_ok && scatter == TB_SCATTER_ATOMIC && !ctx->md_fuse &&
                      (n >= (1 << 18) || ctx->sctl);
  if (direct) CK(cudaMemsetAsync(d_forces, 0, sizeof(double) * 3 * (size_t)n, ctx->stream));
  a.forces = direct ? d_forces : ctx->facc.as<double>();
  a.fbuf = nl->fbuf.as<double>();
  a.per_atom = d_per_atom;
  a.partials = ctx->partials.as<double>();
  a.stats = ctx->stats_acc.as<unsigned long long>();
  a.err = ctx->errf.as<ErrFlags>();
  int rc;
  int nparts = nb;
  if (warp_path) {
    WArgs w;
    w.lanes = nl->lanes.as<int4>();
    w.empty_atoms = nl->sorted_atoms.as<int>();
    w.nchunks = nl->nchunks;
    w.n_empty = nl->n_empty;
    w.dinfo = nullptr;
    w.dskip = 0;
    w.count_packed = filtered ? 0 : 1;
    // live repack: atomic scatter only (the gather finalize reads every entry's
    // slot, which must then be rewritten each evaluation); auto = species-
    // filtered rows (SiC: 12 mostly dead Si-Si entries per Si row; c3 step
    // 501 -> 395 us).  Long single-species rows (disordered Si, c4) gain
    // 575 -> 371 us in the kernel but pay it back in the repack pass.
    // Auto also takes long single-species rows (skin rows of >= 6 entries on
    // average, e.g. disordered Si at 6.9): with the margin gate (§3.5) the
    // repack pass runs only after atoms moved, so repeated evaluations keep
    // the short rows for free.
    const bool long_rows = nl->n > 0 && nl->entries >= 6 * nl->n;
    // Inside tb_md_run's graph (dplan set): species-filtered rows only, with
    // the margin gate and its device-side force flag (md_prepare sized the
    // buffers; the in-graph rebuild raises lforce).
    const bool live_ok = ctx->dplan ? (filtered && ctx->md_live && ctx->repack_margin > 0 &&
                                       nl->lforce.p != nullptr)
                                    : true;
    const bool live = live_ok && scatter == TB_SCATTER_ATOMIC && (!filtered || nl->fnbr_ok) &&
                      (ctx->live_pack == 1 ||
                       (ctx->live_pack == 2 && (filtered || (long_rows && ctx->repack_margin > 0))));
    if (ctx->dplan && !live) {  // tb_md_run capture: chunk counts live in the device plan
      w.dinfo = ctx->dplan;
      w.nchunks = (int)nl->ccap;  // grid sizing only
    } else if (live) {
      int lrc = live_repack(ctx, const_cast<tb_nlist *>(nl), d_pos, r_cut, filtered, a.box, a.err);
      if (lrc) return lrc;
      w.lanes = nl->llanes.as<int4>();
      w.empty_atoms = nl->lsorted.as<int>();
      w.dinfo = nl->lplan.as<int>();  // DevPlan starts with {nchunks, n_empty}
      w.nchunks = (int)nl->lcap;      // grid sizing only
      // unfiltered: the chunked rows are exactly the packed rows (zeta_visits
      // counted in the kernel); filtered rows miss entries the reference
      // counts, so k_pack_stats still counts over the full rows
      w.count_packed = filtered ? 0 : 1;
    }
    w.facc = a.forces;
    const bool want_stats = d_stats != nullptr;
    if (ctx->sctl) {
      // streamed: one launch per stage, behind the stage's last range of
      // positions; finished ranges of forces / per-atom energies go back on
      // the D2H stream while later stages run (tb_stream.cuh)
      if (live || !direct) return fail(ctx, TB_ERR_CUDA, "internal error: streamed evaluation");
      const StreamCtl &sc = *ctx->sctl;
      const int K = nl->sp_K;
      const int64_t R = nl->sp_R;
      int total = 0;
      rc = TB_OK;
      for (int s = 0; s < K && !rc; ++s) {
        CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_h2d[s], 0));
        const int c0 = nl->sp_cstart[s], c1 = nl->sp_cstart[s + 1];
        const bool last = s == K - 1;
        if (c1 > c0 || (last && nl->n_empty > 0) || (last && total == 0)) {
          w.lanes = nl->sp_lanes.as<int4>() + 32 * (int64_t)c0;
          w.nchunks = c1 - c0;
          w.n_empty = last ? nl->n_empty : 0;
          ctx->part_off = total;
          rc = precision == TB_PREC_DOUBLE
                   ? launch_warp_prec<double>(ctx, nl, a, w, scatter, want_stats)
                   : launch_warp_prec<float>(ctx, nl, a, w, scatter, want_stats);
          ctx->part_off = 0;
          if (rc) break;
          total += ctx->last_blocks;
        }
        CK(cudaEventRecord(ctx->ev_stage[s], ctx->stream));
        bool waited = false;
        for (int r = 0; r < K; ++r) {
          if (nl->sp_fin[r] != s) continue;
          int r1 = r;  // merge the run of ranges finishing with this stage
          while (r1 + 1 < K && nl->sp_fin[r1 + 1] == s) ++r1;
          const int64_t a0 = r * R, a1 = std::min<int64_t>(n, (r1 + 1) * R);
          if (!waited) CK(cudaStreamWaitEvent(ctx->s_d2h, ctx->ev_stage[s], 0));
          waited = true;
          CK(cudaMemcpyAsync(sc.h_forces + 3 * a0, d_forces + 3 * a0,
                             sizeof(double) * 3 * (a1 - a0), cudaMemcpyDeviceToHost, ctx->s_d2h));
          if (sc.h_per_atom)
            CK(cudaMemcpyAsync(sc.h_per_atom + a0, d_per_atom + a0, sizeof(double) * (a1 - a0),
                               cudaMemcpyDeviceToHost, ctx->s_d2h));
          r = r1;
        }
      }
      ctx->last_blocks = total;
      a.partials = ctx->partials.as<double>();  // the finalize reduces every stage's slots
    } else if (ctx->row_kernel && ctx->S == 1 && !ctx->lam3 && !live &&
               nl->r4_count >= ctx->row_min && make_tables<double, 1>(ctx).fc_same) {
      // rows of <= ROW_LM entries: one lane per atom (tb_row.cuh); the warp
      // chunks of the longer rows follow, with their own partial slots
      int sms = 0;
      CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
      CK(ctx->partials.ensure(sizeof(double) * 8 * (size_t)2 * sms * 16));
      RArgs r;
      r.atoms = nl->sorted_atoms.as<int>();
      r.first = nl->r4_first;
      r.count = nl->r4_count;
      r.dplan = ctx->dplan;  // tb_md_run capture: the bounds live in the device plan
      r.n_empty = nl->n_empty;
      r.count_packed = w.count_packed;
      rc = launch_row(ctx, a, r, ctx->dplan ? n : nl->r4_count, precision, scatter, want_stats);
      int total = ctx->last_blocks;
      if (!rc && (ctx->dplan || nl->nchunks > nl->r4_chunks)) {
        if (ctx->dplan) {
          // the longer rows' chunks start at chunk_base[ROW_LM + 1] of the plan
          w.dskip = (int)(offsetof(DevPlan, chunk_base) / sizeof(int)) + ROW_LM + 1;
          w.nchunks = (int)std::max<int64_t>(nl->ccap / 8, 1024);  // grid sizing only
        } else {
          w.lanes += 32 * (int64_t)nl->r4_chunks;
          w.nchunks -= nl->r4_chunks;
        }
        w.n_empty = 0;
        ctx->part_off = total;
        rc = precision == TB_PREC_DOUBLE
                 ? launch_warp_prec<double>(ctx, nl, a, w, scatter, want_stats)
                 : launch_warp_prec<float>(ctx, nl, a, w, scatter, want_stats);
        ctx->part_off = 0;
        total += ctx->last_blocks;
      }
      ctx->last_blocks = total;
      a.partials = ctx->partials.as<double>();
    } else {
      rc = precision == TB_PREC_DOUBLE ? launch_warp_prec<double>(ctx, nl, a, w, scatter, want_stats)
                                       : launch_warp_prec<float>(ctx, nl, a, w, scatter, want_stats);
    }
    nparts = ctx->last_blocks;
    if (!rc && filtered && want_stats && !w.count_packed) {
      k_pack_stats<<<nblk(n, 256), 256, 0, ctx->stream>>>(n, d_pos, a.box, a.rc2, a.off, a.nbr,
                                                           a.stats);
      CK(cudaGetLastError());
    }
  } else {
    rc = precision == TB_PREC_DOUBLE ? launch_prec<double>(ctx, nl, a, C, scatter)
                                     : launch_prec<float>(ctx, nl, a, C, scatter);
  }
  if (rc) return rc;
  if (ctx->md_fuse && scatter == TB_SCATTER_ATOMIC) {
    ctx->last_blocks = nparts;  // k_md_kick_ke<true> + k_md_tail do the finalize's work
    return TB_OK;
  }
  // finalize grid: block 0 reduces E/W; the rest move the forces (atomic: 16-byte
  // vectors, ~4 per thread; gather: one atom row per thread)
  int fb = direct ? 1
                  : 1 + std::min(scatter == TB_SCATTER_GATHER ? nblk(n, 256)
                                                              : nblk(3 * (int64_t)n, 256 * 2 * 4),
                                 4 * 148);
  // (a programmatic-dependent finalize launch, a cooperative grid-barrier
  //  finalize and a last-block reduction were all measured slower)
#ifdef TB_DBG_NO_FINALIZE
  if (getenv("TB_DBG_NO_FINALIZE")) return TB_OK;  // timing experiments only
#endif
  if (ctx->ev_kernel_done) CK(cudaEventRecord(ctx->ev_kernel_done, ctx->stream));
  const unsigned long long *err_src = reinterpret_cast<const unsigned long long *>(a.err);
  if (scatter == TB_SCATTER_GATHER)
    k_finalize<1><<<fb, 256, 0, ctx->stream>>>(n, nullptr, a.off, nl->rev.as<int>(), a.fbuf,
                                                d_forces, nparts, a.partials, d_result, a.stats,
                                                d_stats, err_src, ctx->fin_err_dst);
  else
    k_finalize<0><<<fb, 256, 0, ctx->stream>>>(n, direct ? nullptr : a.forces, nullptr, nullptr,
                                                nullptr, d_forces, nparts, a.partials, d_result,
                                                a.stats, d_stats, err_src, ctx->fin_err_dst);
  CK(cudaGetLastError());
  return TB_OK;
}

// Map latched device error flags to the reference's exceptions and wording.
// decode the flags the caller read back into h_err; resets them on error
static int report_errors(tb_context *ctx, const tb_nlist *nl, const double *d_pos,
                         const int *d_species) {
  ErrFlags e = *ctx->h_err;
  int rc = TB_OK;
  if (e.overflow) {
    rc = fail(ctx, TB_ERR_CUDA, "internal error: tile staging overflow");
  } else if (e.stale_filter) {
    rc = fail(ctx, TB_ERR_INPUT,
              "species changed since the neighbour list's species filter was built; "
              "rebuild the list (tb_build_neighbors) or call tb_nlist_refilter");
  } else if (e.nonfinite_atom != INT_MAX) {
    // kernels.py:111-116
    rc = fail(ctx, TB_ERR_INPUT, "non-finite position for atom %d", e.nonfinite_atom);
  } else if (e.bad_species_atom != INT_MAX) {
    // kernels.py:95-108
    int v = 0;
    CK(cudaMemcpy(&v, d_species + e.bad_species_atom, sizeof(int), cudaMemcpyDeviceToHost));
    rc = fail(ctx, TB_ERR_CONFIG, "species index %d outside the %d-species parameter table", v,
              ctx->S);
  } else if (e.coinc_key != ~0ull) {
    // neighbor.py:346-352
    int ent = (int)(e.coinc_key & 0xffffffffu);
    std::vector<int> off(nl->n + 1);
    CK(cudaMemcpy(off.data(), nl->offsets.p, sizeof(int) * (nl->n + 1), cudaMemcpyDeviceToHost));
    int i = (int)(std::upper_bound(off.begin(), off.end(), ent) - off.begin()) - 1;
    int j = 0;
    CK(cudaMemcpy(&j, nl->nbr.as<int>() + ent, sizeof(int), cudaMemcpyDeviceToHost));
    double xi[3], xj[3];
    CK(cudaMemcpy(xi, d_pos + 3 * (int64_t)i, 3 * sizeof(double), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(xj, d_pos + 3 * (int64_t)j, 3 * sizeof(double), cudaMemcpyDeviceToHost));
    double r2 = 0;
    for (int ax = 0; ax < 3; ++ax) {
      double d = xj[ax] - xi[ax];
      if (nl->per[ax]) d -= nl->L[ax] * std::nearbyint(d / nl->L[ax]);
      r2 += d * d;
    }
    rc = fail(ctx, TB_ERR_INPUT, "atoms %d and %d are coincident (r = %.3e A)", i, j,
              std::sqrt(r2));
  }
  if (rc) {
    int r2 = reset_errors(ctx);
    (void)r2;
  }
  return rc;
}

extern "C" int tb_compute(tb_context *ctx, const tb_nlist *nl, const double *positions,
                          const int32_t *species, double r_cut, int precision, int scatter,
                          double *forces, double *per_atom, double *energy, double *virial,
                          int64_t *stats) {
  if (!ctx || !nl || !forces || !energy) return fail(ctx, TB_ERR_ARG, "null argument");
  CK(cudaSetDevice(ctx->device));
  const int64_t n = nl->n;
  if (n && (!positions || !species)) return fail(ctx, TB_ERR_ARG, "null positions/species");
  int rc = TB_OK;
  if (ctx->err_unchecked || !ctx->errf.p) rc = reset_errors(ctx);
  if (rc) return rc;
  // Streamed path (tb_stream.cuh): pinned host positions in, pinned host
  // forces / per-atom energies out, one species, atomic scatter, warp chunks
  // without the live repack, at least 8 ranges of stream_range atoms.
  bool streamed = false;
  int sK = 0, sR = 0;
  StreamCtl sctl{nullptr, nullptr, nullptr, nullptr};
  {
    const int64_t rmin = ctx->stream_range;
    const bool long_rows = n > 0 && nl->entries >= 6 * n;
    const bool live = ctx->live_pack == 1 ||
                      (ctx->live_pack == 2 && long_rows && ctx->repack_margin > 0);
    if (rmin > 0 && n >= 8 * rmin && scatter == TB_SCATTER_ATOMIC && ctx->S == 1 && nl->built &&
        nl->nchunks > 0 && !ctx->force_tile && !live && r_cut <= nl->r_cut &&
        (precision == TB_PREC_DOUBLE || precision == TB_PREC_MIXED) &&
        !is_device_ptr(positions) && host_alias(positions) && !is_device_ptr(forces) &&
        host_alias(forces) && (!per_atom || (!is_device_ptr(per_atom) && host_alias(per_atom)))) {
      sR = (int)std::max<int64_t>(rmin, (n + STREAM_KMAX - 1) / STREAM_KMAX);
      sK = (int)((n + sR - 1) / sR);
      streamed = sK >= 2;
    }
  }
  const double *d_pos = nullptr;
  if (streamed) {
    rc = stream_plan(ctx, const_cast<tb_nlist *>(nl), sK, sR);
    if (rc) return rc;
    if (!ctx->s_h2d) {
      CK(cudaStreamCreateWithFlags(&ctx->s_h2d, cudaStreamNonBlocking));
      CK(cudaStreamCreateWithFlags(&ctx->s_d2h, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
    }
    while ((int)ctx->ev_h2d.size() < sK) {
      cudaEvent_t e1, e2;
      CK(cudaEventCreateWithFlags(&e1, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&e2, cudaEventDisableTiming));
      ctx->ev_h2d.push_back(e1);
      ctx->ev_stage.push_back(e2);
    }
    CK(ctx->pos.ensure(sizeof(double) * 3 * (size_t)n));
    CK(ctx->forces.ensure(sizeof(double) * 3 * (size_t)n));
    if (per_atom) CK(ctx->per_atom.ensure(sizeof(double) * (size_t)n));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
    CK(ctx->partials.ensure(sizeof(double) * 8 * (size_t)sK * sms * 16));
    // the staging buffers may still be read by earlier work on the stream
    CK(cudaEventRecord(ctx->ev_fork, ctx->stream));
    CK(cudaStreamWaitEvent(ctx->s_h2d, ctx->ev_fork, 0));
    CK(cudaStreamWaitEvent(ctx->s_d2h, ctx->ev_fork, 0));
    for (int r = 0; r < sK; ++r) {
      const int64_t a0 = (int64_t)r * sR, a1 = std::min<int64_t>(n, a0 + sR);
      CK(cudaMemcpyAsync(ctx->pos.as<double>() + 3 * a0, positions + 3 * a0,
                         sizeof(double) * 3 * (a1 - a0), cudaMemcpyHostToDevice, ctx->s_h2d));
      CK(cudaEventRecord(ctx->ev_h2d[r], ctx->s_h2d));
    }
    d_pos = ctx->pos.as<double>();
    sctl.h_pos = positions;
    sctl.h_forces = forces;
    sctl.h_per_atom = per_atom;
    sctl.d_pos = ctx->pos.as<double>();
  } else {
    d_pos = stage_in(ctx, positions, 3 * (size_t)n, ctx->pos, rc);
    if (rc) return rc;
  }
  // a failing call drains the side streams before it returns
  auto drain = [&](int code) {
    if (streamed) {
      cudaStreamSynchronize(ctx->s_h2d);
      cudaStreamSynchronize(ctx->stream);
      cudaStreamSynchronize(ctx->s_d2h);
    }
    return code;
  };
  const bool sp_host = !is_device_ptr(species);
  const int *d_sp = stage_in(ctx, species, (size_t)n, ctx->species, rc);
  if (rc) return drain(rc);
  if (sp_host && ctx->S > 1) {
    // host species go through one staging buffer: a content change (checked
    // per list) invalidates the species-pair compute filter built for the old
    // values (the device guard below catches in-place device changes)
    tb_nlist *nlm = const_cast<tb_nlist *>(nl);
    if (nlm->host_species.size() != (size_t)n ||
        memcmp(nlm->host_species.data(), species, sizeof(int) * n) != 0) {
      nlm->host_species.assign(species, species + n);
      nlm->filtered = false;
    }
  }
  if (n == 0) {  // validation only (parameters, list, cutoff); empty results
    CK(ctx->result.ensure(sizeof(double) * 8));
    CK(ctx->stats.ensure(sizeof(unsigned long long) * TB_NSTATS));
    rc = enqueue_compute(ctx, nl, d_pos, d_sp, r_cut, precision, scatter, forces, per_atom,
                         ctx->result.as<double>(), ctx->stats.as<unsigned long long>());
    if (rc) return rc;
    CK(cudaStreamSynchronize(ctx->stream));
    *energy = 0.0;
    if (virial)
      for (int q = 0; q < 6; ++q) virial[q] = 0.0;
    if (stats)
      for (int q = 0; q < TB_NSTATS; ++q) stats[q] = 0;
    return TB_OK;
  }
  // results: device buffers are written in place; pinned host buffers are
  // written by the finalize kernel through their device alias (no copy-back);
  // pageable host buffers go through staging and a copy
  const bool f_dev = is_device_ptr(forces);
  double *f_alias = f_dev || streamed ? nullptr : static_cast<double *>(host_alias(forces));
  double *d_f = f_dev ? forces : f_alias;
  if (!d_f) {
    CK(ctx->forces.ensure(sizeof(double) * 3 * std::max<int64_t>(n, 1)));
    d_f = ctx->forces.as<double>();
  }
  const bool e_dev = per_atom && is_device_ptr(per_atom);
  double *d_e = per_atom;
  if (per_atom && !e_dev) {
    CK(ctx->per_atom.ensure(sizeof(double) * std::max<int64_t>(n, 1)));
    d_e = ctx->per_atom.as<double>();
  }
  // [ErrFlags | result @64 | stats @128] of this call land in pinned h_small,
  // written by the finalize kernel
  char *h = reinterpret_cast<char *>(ctx->h_small);
  char *hd = static_cast<char *>(host_alias(h));
  if (!hd) return drain(fail(ctx, TB_ERR_CUDA, "pinned result block is not device-mapped"));
  const bool pa_async = !streamed && per_atom && !e_dev && host_alias(per_atom);
  if (pa_async && !ctx->side) {
    CK(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ctx->ev_kernel_done, cudaEventDisableTiming));
  }
  bool retried_stale = false;
evaluate:
  ctx->fin_err_dst = reinterpret_cast<unsigned long long *>(hd);
  cudaEvent_t keep_ev = ctx->ev_kernel_done;
  if (!pa_async) ctx->ev_kernel_done = nullptr;
  ctx->sctl = streamed ? &sctl : nullptr;
  rc = enqueue_compute(ctx, nl, d_pos, d_sp, r_cut, precision, scatter, d_f, d_e,
                       reinterpret_cast<double *>(hd + 64),
                       reinterpret_cast<unsigned long long *>(hd + 128), f_dev || streamed);
  ctx->sctl = nullptr;
  ctx->part_off = 0;
  ctx->fin_err_dst = nullptr;
  ctx->ev_kernel_done = keep_ev;
  if (rc) return drain(rc);
  if (streamed) {
    // every range was queued on the D2H stream behind its last stage
    CK(spin_sync(ctx->stream));
    CK(spin_sync(ctx->s_d2h));
  } else if (pa_async) {
    // per-atom energies are final when the Tersoff kernel ends: copy them back
    // on the side stream while the finalize kernel runs
    CK(cudaStreamWaitEvent(ctx->side, ctx->ev_kernel_done, 0));
    CK(cudaMemcpyAsync(per_atom, d_e, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->side));
  } else if (per_atom && !e_dev) {
    CK(cudaMemcpyAsync(per_atom, d_e, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
  }
  if (!streamed && !f_dev && !f_alias)
    CK(cudaMemcpyAsync(forces, d_f, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, ctx->stream));
  CK(spin_sync(ctx->stream));
  if (pa_async) CK(spin_sync(ctx->side));
  ctx->err_unchecked = false;
  memcpy(ctx->h_err, h, sizeof(ErrFlags));
  if (ctx->h_err->stale_filter && !retried_stale) {
    // device species changed in place since the filter was built: rebuild it
    // for the current species and evaluate again
    const_cast<tb_nlist *>(nl)->filtered = false;
    rc = reset_errors(ctx);
    if (rc) return rc;
    retried_stale = true;
    goto evaluate;
  }
  rc = report_errors(ctx, nl, d_pos, d_sp);
  if (rc) return rc;
  const double *hr = reinterpret_cast<const double *>(h + 64);
  const unsigned long long *hs = reinterpret_cast<const unsigned long long *>(h + 128);
  *energy = hr[0];
  if (virial)
    for (int q = 0; q < 6; ++q) virial[q] = hr[1 + q];
  if (stats)
    for (int q = 0; q < TB_NSTATS; ++q) stats[q] = (int64_t)hs[q];
  return TB_OK;
}

extern "C" int tb_compute_device(tb_context *ctx, const tb_nlist *nl, const double *d_positions,
                                 const int32_t *d_species, double r_cut, int precision,
                                 int scatter, double *d_forces, double *d_per_atom,
                                 double *d_result, uint64_t *d_stats) {
  if (!ctx || !nl || !d_forces || !d_result) return fail(ctx, TB_ERR_ARG, "null argument");
  if (nl->n && (!d_positions || !d_species)) return fail(ctx, TB_ERR_ARG, "null positions/species");
  return enqueue_compute(ctx, nl, d_positions, d_species, r_cut, precision, scatter, d_forces,
                         d_per_atom, d_result, reinterpret_cast<unsigned long long *>(d_stats));
}

#ifdef TB_TRACE
extern "C" int tb_debug_trace(void *host, size_t bytes) {
  return cudaMemcpyFromSymbol(host, tb::g_trace, std::min(bytes, sizeof(tb::g_trace))) == cudaSuccess
             ? TB_OK : TB_ERR_CUDA;
}
#endif

extern "C" int tb_check_errors(tb_context *ctx) {
  if (!ctx) return TB_ERR_ARG;
  if (!ctx->errf.p) return TB_OK;
  CK(cudaMemcpyAsync(ctx->h_err, ctx->errf.p, sizeof(ErrFlags), cudaMemcpyDeviceToHost,
                     ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  ErrFlags e = *ctx->h_err;
  int rc = TB_OK;
  if (e.overflow) rc = fail(ctx, TB_ERR_CUDA, "internal error: tile staging overflow");
  else if (e.stale_filter)
    rc = fail(ctx, TB_ERR_INPUT,
              "species changed since the neighbour list's species filter was built; "
              "rebuild the list (tb_build_neighbors) or call tb_nlist_refilter");
  else if (e.nonfinite_atom != INT_MAX)
    rc = fail(ctx, TB_ERR_INPUT, "non-finite position for atom %d", e.nonfinite_atom);
  else if (e.bad_species_atom != INT_MAX)
    rc = fail(ctx, TB_ERR_CONFIG, "species index outside the %d-species parameter table (atom %d)",
              ctx->S, e.bad_species_atom);
  else if (e.coinc_key != ~0ull)
    rc = fail(ctx, TB_ERR_INPUT, "atoms are coincident (list entry %u)",
              (unsigned)(e.coinc_key & 0xffffffffu));
  if (rc) reset_errors(ctx);
  ctx->err_unchecked = false;
  return rc;
}

extern "C" int tb_profile(tb_context *ctx, int enable) {
  if (!ctx) return TB_ERR_ARG;
  ctx->profile = enable != 0;
  return TB_OK;
}

extern "C" int tb_profile_read(tb_context *ctx, double *total_ms, int64_t *launches) {
  if (!ctx || !total_ms || !launches) return fail(ctx, TB_ERR_ARG, "null argument");
  CK(cudaStreamSynchronize(ctx->stream));
  double tot = 0.0;
  for (auto &ev : ctx->ev_used) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, ev.first, ev.second));
    tot += ms;
    ctx->ev_free.push_back(ev);
  }
  *launches = (int64_t)ctx->ev_used.size();
  ctx->ev_used.clear();
  *total_ms = tot;
  return TB_OK;
}

// ---------------------------------------------------------------------------
// device-resident velocity Verlet (system.py:355-380)
// ---------------------------------------------------------------------------

extern "C" int tb_md_step(tb_context *ctx, tb_nlist *nl, int64_t n, double *d_positions,
                          double *d_velocities, double *d_forces, const double *d_mass,
                          const int32_t *d_species, const double *box, const int32_t *periodic,
                          double dt, double accel, double r_cut, double skin, int precision,
                          int scatter, int force_rebuild, double *d_per_atom, double *d_result,
                          int32_t *rebuilt) {
  if (!ctx || !nl || !box || !periodic || !d_result) return fail(ctx, TB_ERR_ARG, "null argument");
  if (!(dt > 0)) return fail(ctx, TB_ERR_CONFIG, "dt must be positive, got %s", fmt_g(dt).c_str());
  CK(cudaSetDevice(ctx->device));
  int per[3] = {periodic[0] ? 1 : 0, periodic[1] ? 1 : 0, periodic[2] ? 1 : 0};
  Box b = make_box(box, per);
  const double half = 0.5 * dt * accel;
  if (n) {
    k_kick_drift<<<nblk(n, 256), 256, 0, ctx->stream>>>((int)n, d_positions, d_velocities,
                                                         d_forces, d_mass, half, dt, b);
    CK(cudaGetLastError());
  }
  int32_t need = 1;
  if (!force_rebuild && nl->built && nl->n == n) {
    int rc = drift_check(ctx, nl, d_positions, &need);
    if (rc) return rc;
  }
  if (need) {
    int rc = tb_build_neighbors(ctx, nl, n, d_positions, box, periodic, r_cut, skin);
    if (rc) return rc;
  }
  if (rebuilt) *rebuilt = need;
  int rc = enqueue_compute(ctx, nl, d_positions, d_species, r_cut, precision, scatter, d_forces,
                           d_per_atom, d_result, nullptr);
  if (rc) return rc;
  if (n) {
    k_kick<<<nblk(n, 256), 256, 0, ctx->stream>>>((int)n, d_velocities, d_forces, d_mass, half);
    CK(cudaGetLastError());
  }
  // kinetic energy 0.5 sum m v^2 / accel (system.py:129-134) -> d_result[7]
  const int kb = std::max(1, std::min(nblk(n, 256), 4 * 148));
  CK(ctx->ke_part.ensure(sizeof(double) * kb));
  k_kinetic<<<kb, 256, 0, ctx->stream>>>((int)n, d_velocities, d_mass, ctx->ke_part.as<double>());
  k_kinetic_sum<<<1, 256, 0, ctx->stream>>>(kb, ctx->ke_part.as<double>(), 0.5 / accel,
                                            d_result + 7);
  CK(cudaGetLastError());
  return TB_OK;
}

// ---------------------------------------------------------------------------
// device-resident NVE loop: one graph launch for a whole run (tb_dnl.cuh)
// ---------------------------------------------------------------------------

// The complete neighbour-list rebuild with every size taken from the device
// plan: cell binning, count pass, offsets, fill pass, snapshot, species-pair
// filter, warp chunks, reverse index.  No host synchronisation; capacities
// were fixed by the last host build (tb_build_neighbors_owned).
static int enqueue_rebuild_device(tb_context *ctx, tb_nlist *nl, const double *d_pos,
                                  const int *d_species, int scatter, bool filter, DevPlan *plan) {
  const int N = (int)nl->n;
  const Grid &g = nl->grid;
  cudaStream_t st = ctx->stream;
  const int ecap = (int)nl->ecap, ccap = (int)nl->ccap;
  k_plan_reset<<<1, 64, 0, st>>>(plan, 1);
  CK(cudaMemsetAsync(nl->cell_count.p, 0, sizeof(int) * (nl->ncell + 1), st));
  k_cell_index<<<nblk(N, 256), 256, 0, st>>>(N, d_pos, g, nl->atom_cell.as<int>(),
                                               nl->cell_count.as<int>(), &plan->unwrapped);
  int rc = exclusive_scan(ctx, nl->cell_count.as<int>(), nl->cell_start.as<int>(), nl->ncell + 1);
  if (rc) return rc;
  k_cell_fill_gather<<<nblk(N, 256), 256, 0, st>>>(
      N, d_pos, nl->atom_cell.as<int>(), nl->cell_start.as<int>(), nl->cell_count.as<int>(),
      nl->cell_atoms.as<int>(), nl->cpos.as<double4>(), nl->ref_pos.as<double>());
  const double bc2 = nl->bc * nl->bc;
  if (g.stencil_image == 2 && ctx->nl_atoms) {
    // (crel is sized by the host build that precedes every device rebuild)
    const float4 *crel = nl->crel.cap >= sizeof(float4) * (size_t)N ? nl->crel.as<float4>() : nullptr;
    if (crel)
      k_cell_rel<<<nblk(N, 256), 256, 0, st>>>(N, nl->cpos.as<double4>(), nl->atom_cell.as<int>(), g,
                                                nl->crel.as<float4>());
    k_nl_atoms<<<nblk(N, 256), 256, 0, st>>>(0, (int)nl->ncell, N, nl->cpos.as<double4>(), g, bc2,
                                              nl->cell_start.as<int>(), nl->row_count.as<int>(),
                                              nl->scratch.as<int>(), &plan->max_row, plan->hist,
                                              &plan->unwrapped, crel);
  }
  else
    k_nl_cells<<<nblk(nl->ncell, 8), 256, 0, st>>>(
        (int)nl->ncell, N, nl->cpos.as<double4>(), g, bc2, nl->cell_start.as<int>(),
        nl->row_count.as<int>(), nl->scratch.as<int>(), &plan->max_row, plan->hist,
        &plan->unwrapped);
  CK(cudaGetLastError());
  rc = exclusive_scan(ctx, nl->row_count.as<int>(), nl->offsets.as<int>(), N + 1);
  if (rc) return rc;
  const int hb = std::min(nblk(N, 256), 296);
  // with the species-pair filter the chunks come from the filtered rows (below)
  k_plan<<<1, 32, 0, st>>>(plan, nl->offsets.as<int>(), N, ecap, filter ? INT_MAX : ccap);
  k_guard_offsets<<<nblk(N + 1, 256), 256, 0, st>>>(N, plan, nl->offsets.as<int>());
  k_nl_compact<SCAN_G><<<nblk((int64_t)N * SCAN_G, 256), 256, 0, st>>>(
      N, nl->scratch.as<int>(), nl->row_count.as<int>(), nl->offsets.as<int>(), nl->nbr.as<int>(),
      nullptr, &plan->list_overflow);
  CK(cudaGetLastError());
  const int *row_len = nl->row_count.as<int>(), *loff = nl->offsets.as<int>();
  const int *cent = nullptr;
  if (filter) {
    const NeedTable nt = need_table(ctx, nl);
    const Box b = make_box(nl->L, nl->per);
    CK(cudaMemsetAsync(nl->crow.p, 0, sizeof(int) * (N + 1), st));
    k_filter_rows<false><<<nblk(N, 128), 128, 0, st>>>(
        N, nl->ref_pos.as<double>(), d_species, ctx->S, nt, b, nl->offsets.as<int>(),
        nl->nbr.as<int>(), nl->crow.as<int>(), nullptr, nullptr);
    rc = exclusive_scan(ctx, nl->crow.as<int>(), nl->coff.as<int>(), N + 1);
    if (rc) return rc;
    k_filter_rows<true><<<nblk(N, 128), 128, 0, st>>>(
        N, nl->ref_pos.as<double>(), d_species, ctx->S, nt, b, nl->offsets.as<int>(),
        nl->nbr.as<int>(), nullptr, nl->coff.as<int>(), nl->centry.as<int>(),
        nl->fnbr.p ? nl->fnbr.as<int>() : nullptr);
    nl->fnbr_ok = nl->fnbr.p != nullptr && nl->fnbr.cap >= sizeof(int) * (size_t)nl->ecap;
    k_plan_reset<<<1, 64, 0, st>>>(plan, 0);
    k_len_hist_plan<<<hb, 256, 0, st>>>(N, nl->crow.as<int>(), plan);
    k_plan<<<1, 32, 0, st>>>(plan, nullptr, N, ecap, ccap);
    CK(cudaGetLastError());
    row_len = nl->crow.as<int>();
    loff = nl->coff.as<int>();
    cent = nl->centry.as<int>();
    if (scatter == TB_SCATTER_GATHER)
      CK(cudaMemsetAsync(nl->fbuf.p, 0, sizeof(double) * 3 * (size_t)ecap, st));
  }
  if (scatter == TB_SCATTER_GATHER) {
    rc = sort_rows_by_length(ctx, nl, row_len);  // stable: reproducible chunk layout
    if (rc) return rc;
  } else if (!filter) {
    // rows bucketed by length and written straight into their chunks (one pass)
    k_bucket_fill<<<nblk(N, 256), 256, 0, st>>>(N, row_len, loff, nullptr, nl->nbr.as<int>(),
                                                plan, nl->sorted_atoms.as<int>(),
                                                nl->lanes.as<int4>());
  } else {
    k_bucket_rows<<<nblk(N, 256), 256, 0, st>>>(N, row_len, plan, nl->sorted_atoms.as<int>());
  }
  if (scatter == TB_SCATTER_GATHER || filter)
    k_fill_lanes_dev<<<(int)std::min<int64_t>(nblk(ccap, 8), 148 * 8), 256, 0, st>>>(
        plan, nl->sorted_atoms.as<int>(), loff, cent, nl->nbr.as<int>(), nl->lanes.as<int4>());
  if (scatter == TB_SCATTER_GATHER)
    k_nl_reverse<<<nblk(N, 256), 256, 0, st>>>(N, nl->offsets.as<int>(), nl->nbr.as<int>(),
                                                 nl->rev.as<int>());
  if (nl->lforce.p) k_set_flag<<<1, 1, 0, st>>>(nl->lforce.as<int>());  // live repack: redo
  CK(cudaGetLastError());
  return TB_OK;
}

namespace {
struct MdArgs {
  int64_t n;
  double *pos, *vel, *forces;
  const double *mass;
  const int *species;
  double dt, accel, r_cut, skin;
  int rebuild_every, precision, scatter, record_every;
  double *series, *result;
  double loose = 0.0;         // > 0: the list carries skin + loose (see k_md_decide)
  double *ref_log = nullptr;  // loose: positions of the reference's last rebuild
};
}  // namespace

static MdKey md_key(const tb_context *ctx, const tb_nlist *nl, const MdArgs &m) {
  MdKey k;
  memset(&k, 0, sizeof(k));
  const void *p[] = {m.pos, m.vel, m.forces, m.mass, m.species, m.series, m.result,
                     nl->plan.p, nl->offsets.p, nl->nbr.p, nl->rev.p, nl->ref_pos.p,
                     nl->atom_cell.p, nl->cell_count.p, nl->cell_start.p, nl->cell_atoms.p,
                     nl->row_count.p, nl->nl_row.p, nl->sorted_atoms.p, nl->sort_keys.p,
                     nl->iota.p, nl->lanes.p, nl->cpos.p, nl->crow.p, nl->coff.p, nl->centry.p,
                     nl->fbuf.p, ctx->facc.p, ctx->partials.p, ctx->ke_part.p, ctx->errf.p,
                     ctx->scan_tmp.p, nl->scratch.p, m.ref_log, nl->lplan.p, nl->llen.p,
                     nl->lrow.p, nl->lrowj.p, nl->lsorted.p, nl->llanes.p, nl->lref.p,
                     nl->lgate.p, nl->lforce.p, nl->fnbr.p, nl->fspecies.p};
  static_assert(sizeof(p) / sizeof(p[0]) <= 48, "MdKey::ptr too small");
  memcpy(k.ptr, p, sizeof(p));
  k.n = m.n;
  k.ecap = nl->ecap;
  k.ccap = nl->ccap;
  k.ncell = nl->ncell;
  for (int ax = 0; ax < 3; ++ax) {
    k.L[ax] = nl->L[ax];
    k.per[ax] = nl->per[ax];
    k.width[ax] = nl->grid.width[ax];
    k.origin[ax] = nl->grid.origin[ax];
    k.nc[ax] = nl->grid.nc[ax];
  }
  k.stencil_image = nl->grid.stencil_image;
  k.dt = m.dt;
  k.accel = m.accel;
  k.skin = m.skin;
  k.r_cut = m.r_cut;
  k.loose = m.loose;
  k.margin = ctx->repack_margin;
  k.lcap = nl->lcap;
  k.rebuild_every = m.rebuild_every;
  k.precision = m.precision;
  k.scatter = m.scatter;
  k.record_every = m.record_every;
  k.param_version = ctx->param_version;
  k.filtered = nl->filtered ? 1 : 0;
  k.S = ctx->S;
  k.tile = ctx->force_tile ? 1 : 0;
  return k;
}

// capture: WHILE(steps) { kick+drift ; decide ; IF(rebuild) { rebuild } ;
//                         Tersoff ; finalize ; kick+KE ; tail }
static int md_capture(tb_context *ctx, tb_nlist *nl, const MdArgs &m, MdGraph *G) {
  for (cudaStream_t &c : ctx->cap)
    if (!c) CK(cudaStreamCreateWithFlags(&c, cudaStreamNonBlocking));
  DevPlan *plan = nl->plan.as<DevPlan>();
  const int n = (int)m.n;
  const Box box = make_box(nl->L, nl->per);
  const double half = 0.5 * m.dt * m.accel;
  const double hs = 0.5 * m.skin;
  const int kb = std::max(1, std::min(nblk(n, 256), 4 * 148));
  const bool filter = ctx->S > 1 && nl->filtered;

  CK(cudaGraphCreate(&G->graph, 0));
  cudaGraphConditionalHandle h_loop, h_reb;
  CK(cudaGraphConditionalHandleCreate(&h_loop, G->graph, 1, cudaGraphCondAssignDefault));
  CK(cudaGraphConditionalHandleCreate(&h_reb, G->graph, 0, 0));
  cudaGraphNodeParams wp = {cudaGraphNodeTypeConditional};
  wp.conditional.handle = h_loop;
  wp.conditional.type = cudaGraphCondTypeWhile;
  wp.conditional.size = 1;
  cudaGraphNode_t wnode;
  CK(cudaGraphAddNode(&wnode, G->graph, nullptr, 0, &wp));
  cudaGraph_t body = wp.conditional.phGraph_out[0];

  cudaStream_t saved = ctx->stream;
  const bool saved_prof = ctx->profile;
  ctx->profile = false;  // event nodes are not allowed in conditional bodies
  auto restore = [&]() {
    ctx->stream = saved;
    ctx->profile = saved_prof;
    ctx->dplan = nullptr;
  };
  cudaStream_t s0 = ctx->cap[0], s1 = ctx->cap[1];
  CK(cudaStreamBeginCaptureToGraph(s0, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  ctx->stream = s0;
  int rc = TB_OK;
  do {
    const double hl = 0.5 * (m.skin + m.loose);
    // (step 1's kick + drift is launched by tb_md_run ahead of the graph; each
    // step's second kick carries the next step's first kick + drift)
    k_md_decide<<<1, 1, 0, s0>>>(plan, hs * hs, m.rebuild_every, h_reb, m.loose > 0 ? 1 : 0,
                                 hl * hl);
    if (cudaGetLastError() != cudaSuccess) {
      rc = fail(ctx, TB_ERR_CUDA, "md capture: launch failed");
      break;
    }
    cudaStreamCaptureStatus cs;
    cudaGraph_t cg;
    const cudaGraphNode_t *deps = nullptr;
    size_t ndeps = 0;
    if (cudaStreamGetCaptureInfo(s0, &cs, nullptr, &cg, &deps, &ndeps) != cudaSuccess) {
      rc = fail(ctx, TB_ERR_CUDA, "md capture: capture info failed");
      break;
    }
    cudaGraphNodeParams ip = {cudaGraphNodeTypeConditional};
    ip.conditional.handle = h_reb;
    ip.conditional.type = cudaGraphCondTypeIf;
    ip.conditional.size = 1;
    cudaGraphNode_t inode;
    cudaError_t e = cudaGraphAddNode(&inode, cg, deps, ndeps, &ip);
    if (e == cudaSuccess) e = cudaStreamUpdateCaptureDependencies(s0, &inode, 1,
                                                                  cudaStreamSetCaptureDependencies);
    if (e == cudaSuccess)
      e = cudaStreamBeginCaptureToGraph(s1, ip.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                        cudaStreamCaptureModeRelaxed);
    if (e != cudaSuccess) {
      rc = fail(ctx, TB_ERR_CUDA, "md capture: conditional node: %s", cudaGetErrorString(e));
      break;
    }
    ctx->stream = s1;
    rc = enqueue_rebuild_device(ctx, nl, m.pos, m.species, m.scatter, filter, plan);
    cudaGraph_t tmp;
    e = cudaStreamEndCapture(s1, &tmp);
    ctx->stream = s0;
    if (!rc && e != cudaSuccess)
      rc = fail(ctx, TB_ERR_CUDA, "md capture: rebuild body: %s", cudaGetErrorString(e));
    if (rc) break;
    ctx->dplan = &plan->nchunks;
    const bool fuse = m.scatter == TB_SCATTER_ATOMIC;
    ctx->md_fuse = fuse;
    rc = enqueue_compute(ctx, nl, m.pos, m.species, m.r_cut, m.precision, m.scatter, m.forces,
                         nullptr, m.result, nullptr);
    ctx->md_fuse = false;
    ctx->dplan = nullptr;
    if (rc) break;
    const int nparts = fuse ? ctx->last_blocks : 0;
    if (fuse)
      k_md_kick2_drift<true><<<kb, 256, 0, s0>>>(n, m.pos, m.vel, m.forces, m.mass, half, m.dt,
                                                 box, ctx->ke_part.as<double>(),
                                                 ctx->facc.as<double>(), plan,
                                                 nl->ref_pos.as<double>(),
                                                 m.loose > 0 ? m.ref_log : nullptr);
    else
      k_md_kick2_drift<false><<<kb, 256, 0, s0>>>(n, m.pos, m.vel, m.forces, m.mass, half, m.dt,
                                                  box, ctx->ke_part.as<double>(), nullptr, plan,
                                                  nl->ref_pos.as<double>(),
                                                  m.loose > 0 ? m.ref_log : nullptr);
    k_md_tail<<<1, 256, 0, s0>>>(kb, ctx->ke_part.as<double>(), 0.5 / m.accel, m.result, plan,
                                 m.series, m.record_every, h_loop, nparts,
                                 ctx->partials.as<double>());
    if (cudaGetLastError() != cudaSuccess) rc = fail(ctx, TB_ERR_CUDA, "md capture: launch failed");
  } while (false);
  cudaGraph_t tmp;
  cudaError_t e = cudaStreamEndCapture(s0, &tmp);
  restore();
  if (rc) return rc;
  if (e != cudaSuccess)
    return fail(ctx, TB_ERR_CUDA, "md capture: step body: %s", cudaGetErrorString(e));
  CK(cudaGraphInstantiate(&G->exec, G->graph, 0));
  return TB_OK;
}

// capacities and every lazily sized buffer of the device rebuild and the
// Tersoff launch, fixed before a capture (nothing may allocate inside one)
static int md_prepare(tb_context *ctx, tb_nlist *nl, const int *d_species, int scatter) {
  const int N = (int)nl->n;
  const bool filter_wanted = ctx->S > 1 && !ctx->no_filter;
  if (filter_wanted && (!nl->filtered || nl->filter_species != d_species ||
                        nl->filter_param_version != ctx->param_version)) {
    int rc = build_filter(ctx, nl, d_species);
    if (rc) return rc;
  }
  CK(nl->plan.ensure(sizeof(DevPlan)));
  if (filter_wanted && scatter == TB_SCATTER_ATOMIC && ctx->md_live && ctx->repack_margin > 0 &&
      ctx->live_pack != 0) {
    int rc = live_reserve(ctx, nl, true);
    if (rc) return rc;
    CK(nl->lforce.ensure(sizeof(int)));
    const int one = 1;
    CK(cudaMemcpyAsync(nl->lforce.p, &one, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  }
  CK(nl->centry.ensure(sizeof(int) * nl->ecap));
  CK(nl->crow.ensure(sizeof(int) * (N + 1)));
  CK(nl->coff.ensure(sizeof(int) * (N + 1)));
  CK(nl->lanes.ensure(sizeof(int4) * 32 * (size_t)nl->ccap));
  if (scatter == TB_SCATTER_GATHER) {
    CK(nl->fbuf.ensure(sizeof(double) * 3 * (size_t)nl->ecap));
    CK(cudaMemsetAsync(nl->fbuf.p, 0, sizeof(double) * 3 * (size_t)nl->ecap, ctx->stream));
    nl->fbuf_zero = true;
    int rc = build_rev(ctx, nl);
    if (rc) return rc;
  }
  // scan / length-sort scratch for every size the device rebuild uses
  CK(ctx->scan_tmp.ensure(sizeof(int) * std::max<int64_t>(
                              std::max(scan_tiles(nl->ncell + 1), scan_tiles((int64_t)N + 1)) + 4,
                              lsort_scratch(N))));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
  CK(ctx->partials.ensure(sizeof(double) * 8 * (size_t)sms * 64));
  CK(ctx->ke_part.ensure(sizeof(double) * 4 * 148));
  if (!ctx->errf.p) {
    int rc = reset_errors(ctx);
    if (rc) return rc;
  }
  if (ctx->facc_n < N) {
    CK(ctx->facc.ensure(sizeof(double) * 3 * N));
    CK(cudaMemsetAsync(ctx->facc.p, 0, sizeof(double) * 3 * N, ctx->stream));
    ctx->facc_n = N;
  }
  if (!ctx->stats_acc.p) {
    CK(ctx->stats_acc.ensure(sizeof(unsigned long long) * TB_NSTATS));
    CK(cudaMemsetAsync(ctx->stats_acc.p, 0, sizeof(unsigned long long) * TB_NSTATS, ctx->stream));
  }
  return TB_OK;
}

extern "C" int tb_md_run(tb_context *ctx, tb_nlist *nl, int64_t n, double *d_positions,
                         double *d_velocities, double *d_forces, const double *d_mass,
                         const int32_t *d_species, double dt, double accel, double r_cut,
                         double skin, int rebuild_every, int precision, int scatter,
                         int64_t steps, int record_every, double *d_series, double *d_result,
                         int64_t *rebuilds) {
  if (!ctx || !nl || !d_result || (n && (!d_positions || !d_velocities || !d_forces || !d_mass ||
                                         !d_species)))
    return fail(ctx, TB_ERR_ARG, "null argument");
  if (!(dt > 0)) return fail(ctx, TB_ERR_CONFIG, "dt must be positive, got %s", fmt_g(dt).c_str());
  if (steps < 0 || steps > INT_MAX - 1) return fail(ctx, TB_ERR_ARG, "bad step count");
  if (record_every < 0) return fail(ctx, TB_ERR_ARG, "bad record interval");
  if (rebuilds) *rebuilds = 0;
  if (steps == 0) return TB_OK;
  CK(cudaSetDevice(ctx->device));
  // the loop keeps the list geometry and the warp-chunk kernel: anything else
  // goes through the per-step path (tb_md_step)
  if (!nl->built || nl->imported || nl->n != n || n == 0 ||
      !(nl->per[0] && nl->per[1] && nl->per[2]) || nl->nchunks <= 0 || ctx->force_tile || ctx->S > 2 || r_cut != nl->r_cut || skin != nl->skin)
    return fail(ctx, TB_ERR_UNSUPPORTED,
                "device-resident loop needs a built periodic list with rows <= 32 entries");
  MdArgs m{n, d_positions, d_velocities, d_forces, d_mass, d_species, dt, accel, r_cut, skin,
           rebuild_every, precision, scatter, record_every, d_series, d_result};
  const int N = (int)n;
  int64_t extra = 0;
  // Loose list (one species, atomic scatter; TB_OPT_MD_LOOSE_SKIN): the run's
  // list carries skin + loose and is rebuilt only when some atom moved more
  // than (skin + loose)/2 since its build; the reference's rebuilds (skin/2
  // trigger, fixed cadence) are still decided, counted and their positions
  // kept (ref_log) -- and the exact list at the last of them is rebuilt when
  // the run ends.  Pair terms are the same either way: every evaluation
  // re-tests r < r_cut on a list that holds all such pairs.
  const bool loose = ctx->md_loose > 0 && scatter == TB_SCATTER_ATOMIC;
  double skin_list = loose ? skin + ctx->md_loose : skin;
  // snapshot: x, v, F, E of the entry state and the entry list's reference
  // positions (every failing exit rebuilds that exact list: the in-graph
  // rebuilds may have left the list at a later trajectory point)
  CK(ctx->snap.ensure(sizeof(double) * 12 * (size_t)N + sizeof(double)));
  double *snap = ctx->snap.as<double>();
  double *snap_ref = snap + 9 * N + 1;
  CK(cudaMemcpyAsync(snap_ref, nl->ref_pos.p, sizeof(double) * 3 * N, cudaMemcpyDeviceToDevice,
                     ctx->stream));
  if (loose) {
    CK(nl->ref_log.ensure(sizeof(double) * 3 * (size_t)N));
    CK(cudaMemcpyAsync(nl->ref_log.p, nl->ref_pos.p, sizeof(double) * 3 * N,
                       cudaMemcpyDeviceToDevice, ctx->stream));
    // The wider list must not push rows out of the row kernel (tb_row.cuh, rows
    // of <= 4 entries): in Si the second-neighbour shell (3.84 A) starts to
    // enter at skin + 0.3 -- 42% of the rows of config 5 get a fifth entry and
    // fall to the warp-chunk kernel, which costs what the saved rebuilds gain
    // (4.83 ms/step; 4.94 with the exact list; 4.35 at 0.2).  When the exact
    // list's rows are nearly all short, the extra skin is reduced (x 2/3, then
    // x 1/2) until 90% of the wider list's rows are.  (Config 5 over a run: the
    // short-row fraction is 0.62-0.89 at skin + 0.3, 0.92-0.99 at skin + 0.2;
    // tools/row_fraction_vs_time.py.)
    const bool row_ok = ctx->row_kernel && ctx->S == 1 && !ctx->lam3 && n >= ctx->row_min;
    const double f_exact = n ? (double)nl->r4_count / (double)n : 0.0;
    double lw = ctx->md_loose;
    int rc = TB_OK;
    for (int t = 0;; ++t) {
      skin_list = skin + lw;
      rc = tb_build_neighbors(ctx, nl, n, d_positions, nl->L, nl->per, r_cut, skin_list);
      if (rc || !row_ok || f_exact < 0.98 || t == 2 || nl->nchunks <= 0) break;
      if ((double)nl->r4_count >= 0.90 * (double)n) break;
      lw *= t == 0 ? 2.0 / 3.0 : 0.5;
    }
    if (rc) return rc;
    if (nl->nchunks <= 0) {  // rows beyond the warp kernel: back to the exact list, per-step path
      rc = tb_build_neighbors(ctx, nl, n, nl->ref_log.as<double>(), nl->L, nl->per, r_cut, skin);
      return rc ? rc : fail(ctx, TB_ERR_UNSUPPORTED, "device-resident loop: rows exceed 32 entries");
    }
    m.loose = lw;
    m.ref_log = nl->ref_log.as<double>();
  }
  // the exact list at the reference's last rebuild (loose runs, any exit)
  auto finish = [&](int rc) -> int {
    if (!loose) return rc;
    int rc2 = tb_build_neighbors(ctx, nl, n, nl->ref_log.as<double>(), nl->L, nl->per, r_cut, skin);
    return rc ? rc : rc2;
  };
  // failing exit after a graph launch (non-loose): the list back at its entry
  // state, so a per-step fallback (tb_md_step) sees consistent lanes and drift
  auto fail_restore = [&](int rc) -> int {
    if (loose) return finish(rc);
    const double *ref = snap_ref;
    int rc2 = tb_build_neighbors(ctx, nl, n, ref, nl->L, nl->per, r_cut, skin);
    if (rc2) nl->built = false;
    return rc;
  };
  CK(cudaMemcpyAsync(snap, d_positions, sizeof(double) * 3 * N, cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaMemcpyAsync(snap + 3 * N, d_velocities, sizeof(double) * 3 * N, cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaMemcpyAsync(snap + 6 * N, d_forces, sizeof(double) * 3 * N, cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaMemcpyAsync(snap + 9 * N, d_result, sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  for (int attempt = 0;; ++attempt) {
    int rc0 = md_prepare(ctx, nl, d_species, scatter);
    if (rc0) return finish(rc0);
    const bool filter_wanted = ctx->S > 1 && !ctx->no_filter;
    // ---- graph (re)capture when anything it holds changed ----
    const MdKey key = md_key(ctx, nl, m);
    if (!nl->md || memcmp(&nl->md->key, &key, sizeof(key)) != 0) {
      md_graph_release(nl);
      nl->md = new MdGraph();
      nl->md->key = key;
      int rc = md_capture(ctx, nl, m, nl->md);
      if (rc) {
        md_graph_release(nl);
        return finish(rc);
      }
    }
    // ---- run ----
    DevPlan hp;
    memset(&hp, 0, sizeof(hp));
    hp.nchunks = nl->nchunks;
    hp.n_empty = nl->n_empty;
    hp.entries = (int)nl->entries;
    hp.max_row = (int)nl->max_row;
    hp.target = (int)steps;
    CK(cudaMemcpyAsync(nl->plan.p, &hp, sizeof(hp), cudaMemcpyHostToDevice, ctx->stream));
    {  // step 1's half-kick + drift (later steps' are fused into the graph's kick pass)
      const Box box = make_box(nl->L, nl->per);
      k_md_kick_drift<<<nblk(n, 256), 256, 0, ctx->stream>>>(
          (int)n, d_positions, d_velocities, d_forces, d_mass, nl->ref_pos.as<double>(),
          0.5 * dt * accel, dt, box, nl->plan.as<DevPlan>(), loose ? m.ref_log : nullptr);
      CK(cudaGetLastError());
    }
    CK(cudaGraphLaunch(nl->md->exec, ctx->stream));
    CK(cudaMemcpyAsync(&hp, nl->plan.p, sizeof(hp), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (hp.overflow == 0) {
      nl->entries = hp.entries;
      nl->max_row = hp.max_row;
      nl->nchunks = hp.nchunks;
      nl->lanes_version++;
      set_row_info(nl, hp.hist);
      nl->n_empty = hp.n_empty;
      nl->lanes_used = hp.lanes_used;
      if (hp.rebuilds > 0 && scatter != TB_SCATTER_GATHER) nl->rev_valid = false;
      nl->lvalid = false;  // the margin repack refers to the entry list
      if (hp.rebuilds > 0 && filter_wanted) nl->fbuf_zero = scatter == TB_SCATTER_GATHER;
      if (rebuilds) *rebuilds = hp.rebuilds + extra;
      return finish(tb_check_errors(ctx));
    }
    // ---- capacity overflow: back to the entry state, regrow, replay ----
    CK(cudaMemcpyAsync(d_positions, snap, sizeof(double) * 3 * N, cudaMemcpyDeviceToDevice, ctx->stream));
    CK(cudaMemcpyAsync(d_velocities, snap + 3 * N, sizeof(double) * 3 * N, cudaMemcpyDeviceToDevice, ctx->stream));
    CK(cudaMemcpyAsync(d_forces, snap + 6 * N, sizeof(double) * 3 * N, cudaMemcpyDeviceToDevice, ctx->stream));
    CK(cudaMemcpyAsync(d_result, snap + 9 * N, sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    if (loose)
      CK(cudaMemcpyAsync(nl->ref_log.p, snap_ref, sizeof(double) * 3 * N,
                         cudaMemcpyDeviceToDevice, ctx->stream));
    if ((hp.overflow & OVF_ROW) || attempt >= 3)
      return fail_restore(fail(ctx, TB_ERR_UNSUPPORTED,
                               "device-resident loop: neighbour rows outgrew the warp kernel "
                               "(overflow %d)", hp.overflow));
    nl->margin = std::max(2.0 * nl->margin, 0.25);
    int rc = tb_build_neighbors(ctx, nl, n, d_positions, nl->L, nl->per, r_cut, skin_list);
    if (rc) return finish(rc);
    nl->filtered = false;
    extra += 1;
    if (nl->nchunks <= 0)
      return fail_restore(fail(ctx, TB_ERR_UNSUPPORTED, "device-resident loop: rows exceed 32 entries"));
  }
}

extern "C" int tb_nlist_rebuild_device(tb_context *ctx, tb_nlist *nl, const double *d_positions,
                                       const int32_t *d_species, int scatter) {
  if (!ctx || !nl || !d_positions || !d_species) return fail(ctx, TB_ERR_ARG, "null argument");
  CK(cudaSetDevice(ctx->device));
  if (!nl->built || nl->imported || nl->n == 0 || !(nl->per[0] && nl->per[1] && nl->per[2]) ||
      nl->nchunks <= 0 || ctx->force_tile || ctx->S > 2)
    return fail(ctx, TB_ERR_UNSUPPORTED,
                "device rebuild needs a built periodic list with rows <= 32 entries");
  int rc = md_prepare(ctx, nl, d_species, scatter);
  if (rc) return rc;
  DevPlan hp;
  memset(&hp, 0, sizeof(hp));
  CK(cudaMemcpyAsync(nl->plan.p, &hp, sizeof(hp), cudaMemcpyHostToDevice, ctx->stream));
  const bool filter = ctx->S > 1 && nl->filtered;
  rc = enqueue_rebuild_device(ctx, nl, d_positions, d_species, scatter, filter,
                              nl->plan.as<DevPlan>());
  if (rc) return rc;
  CK(cudaMemcpyAsync(&hp, nl->plan.p, sizeof(hp), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (hp.overflow) {
    // regrow through the host-synchronised build (same list, new capacities)
    nl->margin = std::max(2.0 * nl->margin, 0.25);
    return tb_build_neighbors(ctx, nl, nl->n, d_positions, nl->L, nl->per, nl->r_cut, nl->skin);
  }
  nl->entries = hp.entries;
  nl->max_row = hp.max_row;
  nl->nchunks = hp.nchunks;
  nl->lanes_version++;
  set_row_info(nl, hp.hist);
  nl->n_empty = hp.n_empty;
  nl->lanes_used = hp.lanes_used;
  nl->lvalid = false;
  nl->rev_valid = scatter == TB_SCATTER_GATHER;
  nl->fbuf_zero = filter && scatter == TB_SCATTER_GATHER;
  if (filter) nl->filter_species = d_species;
  return TB_OK;
}

// ---------------------------------------------------------------------------
// slab domain decomposition (north_star (4))
// ---------------------------------------------------------------------------
#include "tb_dd_api.inc"
