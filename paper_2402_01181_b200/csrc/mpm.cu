// mpm.cu -- C ABI (include/softmpm_b200.h) over the sm_100a kernels.
//
// One mpm_ctx = one SimState on one device: it owns every device buffer and a
// private stream; host pointers are borrowed per call.  The fast path keeps
// particles binned (8^3-cell bins, counting sort) and runs each stretch of
// substeps as  rebin -> P2G -> [grid op -> fused G2P/P2G] x (L-1) -> grid op
// -> G2P, with only active bricks visited on the grid.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <emmintrin.h>
#include <cmath>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <pthread.h>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/softmpm_b200.h"
#include "kernels.cuh"

using namespace mpm;

// Persistent host worker threads (the fp64 <-> fp32 conversions of the
// particle transfers): run(f) calls f(thread, nthreads) on every worker and
// the caller, and returns when all are done.
struct HostPool {
  explicit HostPool(int n) : nt(std::max(1, n)) {
    for (int i = 1; i < nt; ++i) th.emplace_back([this, i] { loop(i); });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> l(m);
      stop = true;
    }
    cv.notify_all();
    for (auto& t : th) t.join();
  }
  void run(const std::function<void(int, int)>& f) {
    {
      std::lock_guard<std::mutex> l(m);
      job = &f;
      pending = nt - 1;
      ++gen;
    }
    cv.notify_all();
    f(0, nt);
    std::unique_lock<std::mutex> l(m);
    done_cv.wait(l, [&] { return pending == 0; });
  }
  int nt;

 private:
  void loop(int id) {
    long long seen = 0;
    for (;;) {
      const std::function<void(int, int)>* j;
      {
        std::unique_lock<std::mutex> l(m);
        cv.wait(l, [&] { return stop || gen != seen; });
        if (stop) return;
        seen = gen;
        j = job;
      }
      (*j)(id, nt);
      std::lock_guard<std::mutex> l(m);
      if (--pending == 0) done_cv.notify_one();
    }
  }
  std::vector<std::thread> th;
  std::mutex m;
  std::condition_variable cv, done_cv;
  const std::function<void(int, int)>* job = nullptr;
  long long gen = 0;
  int pending = 0;
  bool stop = false;
};

struct mpm_ctx {
  mpm_config cfg{};
  int dev = 0;
  int sms = 148;
  cudaStream_t stream = nullptr;
  cudaStream_t xstream = nullptr;  // host<->device field copies, pipelined with the conversions
  cudaEvent_t field_ev[4] = {nullptr, nullptr, nullptr, nullptr};
  // host-converted particle transfers of pageable buffers (option
  // "host_xfer", on by default; the workers are process-wide: XferShared)
  bool host_xfer = true;
  bool g2p_tiled = true;     // stretch-end G2P from staged velocity tiles (SOFTMPM_G2P_TILED=0: thread per particle)
  int g2p_tile_blocks = 0;
  bool xfer_direct = true;  // with pinned buffers x / v cross as fp64 beside it (SOFTMPM_XFER_DIRECT=0: off)
  std::string err;
  long long launches = 0;

  // grid
  long long nbricks = 0;
  float4* gm = nullptr;
  float4* gv = nullptr;
  int* brick_flag = nullptr;
  int* active_list = nullptr;
  int* counters = nullptr;  // [0] active_count, [1] nwork, [2] halo, [3] work_next, [4..] work classes
  int grid_phase = 0;       // 0 momentum view, 1 velocity view, 2 uploaded velocities
  int grid_dirty = 2;       // 0 clean, 1 active-list bricks dirty, 2 fully dirty

  // particles (double-buffered SoA)
  long long n = 0, cap = 0;
  bool uploaded = false;  // a particle set (possibly empty) was uploaded
  float* P[2] = {nullptr, nullptr};
  int* mat[2] = {nullptr, nullptr};
  int* orig[2] = {nullptr, nullptr};
  int cur = 0;
  int* key = nullptr;
  int* rank = nullptr;
  int* lcell = nullptr;  // local cell in bin
  int* sidx = nullptr;   // slots grouped by bin
  int* slc = nullptr;    // their local cells
  int* bperm = nullptr;  // final (bin, cell) order -> source slot
  int* item_box = nullptr;

  // bins
  int nbin[3] = {0, 0, 0};
  int nbins = 0;
  int* bin_count = nullptr;
  int* bin_start = nullptr;
  int* bin_maxcnt = nullptr;
  int4* work = nullptr;
  float4* item_bounds = nullptr;
  float4* item_bounds2 = nullptr;  // fused kernel: bounds of substep n (in) / n+1 (out)
  float* pay = nullptr;  // stage A -> stage B payload, NPAY x cap
  long long work_cap = 0;
  std::vector<int*> scan_tmp;  // per level block sums (two per level)
  std::vector<long long> scan_len;

  // materials
  float* mu = nullptr;
  float* lam = nullptr;
  int nmat = 0;
  unsigned long long* inverted = nullptr;
  unsigned long long* stats = nullptr;  // [0] fixed-point guard fallbacks (cumulative)
  // slab windows: slots [0, hole_n) flagged in mflag have migrated away;
  // hole_count of them; compacted by the next rebin (compact_if_needed)
  long long hole_n = 0, hole_count = 0;
  // cross-frame re-binning: frames since the last frame-start re-binning of
  // an untouched state (-1: positions changed outside the fast path, re-bin)
  int bins_age = -1;
  int rebin_frames = 1;  // option "rebin_frames" / SOFTMPM_REBIN_FRAMES: re-bin every k-th frame (1 = every frame)
  int fx_shift = 0;                     // test hook: tile scale x 2^fx_shift, cell limit / 2^fx_shift

  // colliders
  int ncol = 0;
  ColliderGeo* geo = nullptr;
  ColliderPose* pose = nullptr;
  int pose_rows = 0, pose_cap = 0, pose_width = 0;
  double* sdf = nullptr;
  std::vector<ColliderGeo> geo_h;

  // deterministic mode
  long long ncells = 0;
  int* cell_count = nullptr;
  int* cell_start = nullptr;
  int* perm = nullptr;
  float* payload = nullptr;

  // staging for fp64 transfers
  double* stage = nullptr;
  size_t stage_bytes = 0;
  int* flag = nullptr;
  double* x0 = nullptr;  // compute_metrics reference positions (caller order)
  // isosurface: the last device density field and the last extracted mesh
  double* field = nullptr;
  long long field_n = 0;
  int field_res[3] = {0, 0, 0};
  double field_dx = 0.0;
  int* mc_flag = nullptr;  // 3 nn crossing flags, then vertex ids
  int* mc_vid = nullptr;
  int* mc_cnt = nullptr;  // cells: triangle counts, then offsets
  int* mc_off = nullptr;
  long long mc_cap = 0;
  double* mesh_v = nullptr;  // vertices, then normals
  unsigned char* enc = nullptr;  // encoded frame body
  long long enc_cap = 0;
  int* mesh_t = nullptr;
  long long mesh_nv = 0, mesh_nt = 0, mesh_vcap = 0, mesh_tcap = 0;
  long long x0_n = -1;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  int fused_blocks = 0;

  // slab decomposition window (config 5): global offset / resolution
  int goff[3] = {0, 0, 0};
  int gres[3] = {0, 0, 0};
  int ghost_bricks = 1;
  // halo buffers (device): per side {ids, data} for send and receive
  int* h_send_ids[2] = {nullptr, nullptr};
  float4* h_send_data[2] = {nullptr, nullptr};
  int* h_recv_ids[2] = {nullptr, nullptr};
  float4* h_recv_data[2] = {nullptr, nullptr};
  int* h_local_ids[2] = {nullptr, nullptr};
  int h_recv_n[2] = {0, 0};
  long long h_cap = 0;  // records per buffer
  // peer-memory exchange (mpm_ipc_*): per side our velocity receive buffer,
  // counters {recv count, received last, sent}, events, and the neighbour's
  // mapped buffers / events
  float4* ipc_vrecv[2] = {nullptr, nullptr};
  int* ipc_cnt[2] = {nullptr, nullptr};
  cudaEvent_t ipc_free[2] = {nullptr, nullptr}, ipc_ready[2] = {nullptr, nullptr};
  int* peer_ids[2] = {nullptr, nullptr};
  float4* peer_data[2] = {nullptr, nullptr};
  int* peer_cnt[2] = {nullptr, nullptr};
  float4* peer_vdata[2] = {nullptr, nullptr};
  bool peer_local[2] = {false, false};  // peer pointers from mpm_peer_connect (same process: not IPC-mapped)
  cudaEvent_t peer_free[2] = {nullptr, nullptr}, peer_ready[2] = {nullptr, nullptr};
  // stream-memory-op protocol (no host barriers): per side, writes into the
  // neighbour's buffers done / the neighbour's writes consumed
  unsigned ipc_writes[2] = {0, 0}, ipc_reads[2] = {0, 0};
  int stage_nsub = 0, stage_col = 0;
  // migration scratch
  int* mflag = nullptr;
  float* mig_rows[2] = {nullptr, nullptr};
  long long mig_cap = 0;
  int gridop_blocks = 0;  // persistent grid sizes (SMs x resident CTAs)
  int gridop_simple_blocks = 0;
  bool gridop_simple = true;  // option "gridop_simple": warp-per-brick grid op (0 spills); 0 = the prefetching persistent kernel
  int gsA_blocks = 0, gsA0_blocks = 0, clear_blocks = 0, fused_only_blocks = 0;

  // optional per-kernel timing: event pairs per launch, resolved lazily
  bool timing = false;
  struct Mark { int kind; cudaEvent_t a, b; bool graph_owned; int weight; };
  std::vector<Mark> marks;

  // CUDA graphs of whole fast-path frames, keyed by the host-side start state
  struct GraphEntry {
    int nsub, col, cur, border, dirty, timing;
    int prows;  // pose-table rows baked into the collider tables (make_colliders clamps row to prows - 1)
    int skip;   // frame without its frame-start re-binning
    bool cclean, bclean;  // counters / bounds_out known zero at the start
    long long n;
    long long kernels;  // kernel nodes in the graph (evidence counter)
    cudaGraphExec_t exec;
    int end_cur, end_border, end_dirty;
    bool end_cclean, end_bclean;
    std::vector<Mark> marks;  // event nodes captured inside the graph
  };
  std::vector<GraphEntry> graphs;
  bool graphs_on = true;
  float4* bounds_a = nullptr;  // the two item-bound arrays as allocated (swap parity)
  std::vector<cudaEvent_t> event_pool;
  double acc[16] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  bool split_mode = false;  // SOFTMPM_SPLIT=1: stage A+B every substep (A/B comparison)
  int items_per_sm = 4;     // work-item granularity target (SOFTMPM_ITEMS_PER_SM)
  bool mega_on = false;   // substeps 2..L as one cooperative substeps_kernel (option "mega" / SOFTMPM_MEGA=1)
  bool pdl_on = true;     // fused kernel / grid op with programmatic dependent launch (option "pdl" / SOFTMPM_PDL=0 to disable;
                          // on by default: +1% at C3 with the plain grid op, within noise at C4 / C5)
  int mega_blocks = 0;
  bool mega_coop = false;  // device supports cooperative launches
  bool counters_clean = true;     // counters[0] (active bricks) and [3] (work_next) known zero
  bool bounds_out_clean = false;  // item_bounds2 known zero
};

namespace {

#define CK(call)                                                              \
  do {                                                                        \
    cudaError_t e_ = (call);                                                  \
    if (e_ != cudaSuccess) {                                                  \
      ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);          \
      return MPM_ECUDA;                                                       \
    }                                                                         \
  } while (0)

#define LAUNCHED()                                                            \
  do {                                                                        \
    ++ctx->launches;                                                          \
    cudaError_t e_ = cudaGetLastError();                                      \
    if (e_ != cudaSuccess) {                                                  \
      ctx->err = std::string("kernel launch: ") + cudaGetErrorString(e_);     \
      return MPM_ECUDA;                                                       \
    }                                                                         \
  } while (0)

int fail(mpm_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return code;
}

template <typename T>
int dalloc(mpm_ctx* ctx, T** ptr, size_t count) {
  if (*ptr) cudaFree(*ptr);
  *ptr = nullptr;
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc((void**)ptr, count * sizeof(T));
  if (e != cudaSuccess) {
    ctx->err = std::string("cudaMalloc(") + std::to_string(count * sizeof(T)) + "): " + cudaGetErrorString(e);
    cudaGetLastError();
    return MPM_ENOMEM;
  }
  return 0;
}

#define TRY(x)              \
  do {                      \
    int r_ = (x);           \
    if (r_) return r_;      \
  } while (0)

cudaEvent_t pool_event(mpm_ctx* ctx) {
  if (!ctx->event_pool.empty()) {
    cudaEvent_t e = ctx->event_pool.back();
    ctx->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

// kind: 0 stage A (g2p_stress), 1 grid op, 2 rebin, 3 g2p, 4 stage B (p2g_tile), 5 fused
struct TimedRegion {
  mpm_ctx* ctx;
  int kind;
  int weight;  // launches this region stands for (substeps_kernel: its substeps)
  cudaEvent_t a = nullptr;
  TimedRegion(mpm_ctx* c, int k, int w = 1) : ctx(c), kind(k), weight(w) {
    if (ctx->timing) {
      a = pool_event(ctx);
      record(a);
    }
  }
  ~TimedRegion() {
    if (a) {
      cudaEvent_t b = pool_event(ctx);
      record(b);
      ctx->marks.push_back({kind, a, b, false, weight});
    }
  }
  // inside stream capture a plain record is only a dependency marker: timing
  // needs an event record node (cudaEventRecordExternal)
  void record(cudaEvent_t e) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(ctx->stream, &st);
    if (st == cudaStreamCaptureStatusActive)
      cudaEventRecordWithFlags(e, ctx->stream, cudaEventRecordExternal);
    else
      cudaEventRecord(e, ctx->stream);
  }
};

void resolve_marks(mpm_ctx* ctx) {
  if (ctx->marks.empty()) return;
  cudaStreamSynchronize(ctx->stream);
  for (auto& mk : ctx->marks) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, mk.a, mk.b);
    ctx->acc[2 * mk.kind] += ms;
    ctx->acc[2 * mk.kind + 1] += mk.weight;
    if (!mk.graph_owned) {
      ctx->event_pool.push_back(mk.a);
      ctx->event_pool.push_back(mk.b);
    }
  }
  ctx->marks.clear();
}

void invalidate_graphs(mpm_ctx* ctx) {
  if (ctx->graphs.empty()) return;
  cudaStreamSynchronize(ctx->stream);
  resolve_marks(ctx);
  for (auto& g : ctx->graphs) {
    cudaGraphExecDestroy(g.exec);
    for (auto& mk : g.marks) {
      cudaEventDestroy(mk.a);
      cudaEventDestroy(mk.b);
    }
  }
  ctx->graphs.clear();
}

inline unsigned blocks_for(long long n, int t) { return (unsigned)std::max<long long>(1, (n + t - 1) / t); }

Params make_params(mpm_ctx* ctx) {
  Params p{};
  const mpm_config& c = ctx->cfg;
  for (int a = 0; a < 3; ++a) {
    p.res[a] = c.res[a];
    p.nb[a] = (c.res[a] + 3) / 4;
    if (a == 1) p.fd_nb1 = make_fastdiv(p.nb[1]);
    if (a == 2) p.fd_nb2 = make_fastdiv(p.nb[2]);
    p.nbin[a] = ctx->nbin[a];
    if (a == 1) p.fd_nbin1 = make_fastdiv(std::max(ctx->nbin[1], 1));
    if (a == 2) p.fd_nbin2 = make_fastdiv(std::max(ctx->nbin[2], 1));
    p.gravity[a] = (float)c.gravity[a];
    const int et = c.env_tiles[a] > 1 ? c.env_tiles[a] : 1;
    p.goff[a] = ctx->goff[a];
    p.gres[a] = ctx->gres[a] > 0 ? ctx->gres[a] : c.res[a];
    p.goffx[a] = (float)(ctx->goff[a] * c.dx);
    p.env_res[a] = p.gres[a] / et;
    p.env_ext[a] = (float)(p.env_res[a] * c.dx);
    p.fd_env[a] = make_fastdiv(std::max(p.env_res[a], 1));
    p.inv_env_ext[a] = p.env_ext[a] > 0.0f ? 1.0f / p.env_ext[a] : 0.0f;
    double hd = (p.env_res[a] - 1.5 - 1.0e-7) * c.dx;
    float hf = (float)hd;
    if ((double)hf > hd) hf = std::nextafter(hf, 0.0f);
    p.hi[a] = hf;
  }
  p.dx = (float)c.dx;
  p.inv_dx = 1.0f / p.dx;
  p.dt = (float)c.dt;
  p.lo = (float)(1.5 * c.dx);
  p.stress_coef = -4.0f * p.dt * p.inv_dx * p.inv_dx;
  p.apic_coef = 4.0f * p.inv_dx * p.inv_dx;
  p.dx64 = c.dx;
  p.dt64 = c.dt;
  p.bwidth = c.boundary_width;
  p.stick = c.stick;
  p.stress_form = c.stress_form;
  p.gm = ctx->gm;
  p.gv = ctx->gv;
  p.brick_flag = ctx->brick_flag;
  p.active_list = ctx->active_list;
  p.active_count = ctx->counters;
  p.P = ctx->P[ctx->cur];
  for (int f = 0; f < NF; ++f) p.Pf[f] = p.P ? p.P + (long long)f * ctx->cap : nullptr;
  p.mat = ctx->mat[ctx->cur];
  p.orig = ctx->orig[ctx->cur];
  p.cap = ctx->cap;
  p.n = ctx->n;
  p.mu = ctx->mu;
  p.lam = ctx->lam;
  p.inverted = ctx->inverted;
  p.stats = ctx->stats;
  p.fx_shift = ctx->fx_shift;
  p.hole_flag = ctx->mflag;
  p.hole_n = ctx->hole_n;
  p.work = ctx->work;
  p.nwork = ctx->counters + 1;
  p.work_next = ctx->counters + 3;
  return p;
}

Colliders make_colliders(mpm_ctx* ctx, int row, bool use) {
  Colliders cs{};
  const int per_env = ctx->cfg.colliders_per_env > 0 ? ctx->cfg.colliders_per_env : 0;
  cs.count = use ? (per_env ? per_env : ctx->ncol) : 0;
  cs.per_env = per_env;
  for (int a = 0; a < 3; ++a) cs.env_tiles[a] = ctx->cfg.env_tiles[a] > 1 ? ctx->cfg.env_tiles[a] : 1;
  cs.theta = use && ctx->ncol > 0 ? ctx->cfg.theta : -1.0;
  cs.geo = ctx->geo;
  int r = ctx->pose_rows > 0 ? std::min(row, ctx->pose_rows - 1) : 0;
  cs.pose = ctx->pose ? ctx->pose + (size_t)r * std::max(ctx->ncol, 1) : nullptr;
  cs.sdf = ctx->sdf;
  // prefilter margin: far above fp32 rounding of O(1) coordinates, far below dx
  cs.theta_f = (float)(cs.theta + 1e-4 * ctx->cfg.dx + 1e-6);
  return cs;
}

int validate(const mpm_config* c, std::string& why) {
  for (int a = 0; a < 3; ++a)
    if (c->res[a] < 8) {
      why = "grid resolution too small";
      return 1;
    }
  if (!(c->dx > 0.0)) { why = "dx must be positive"; return 1; }
  if (!(c->dt > 0.0)) { why = "dt must be positive"; return 1; }
  if (c->boundary_width < 0) { why = "boundary_width must be >= 0"; return 1; }
  if (c->stress_form != 0 && c->stress_form != 1) { why = "unknown stress form"; return 1; }
  for (int a = 0; a < 3; ++a) {
    const int et = c->env_tiles[a] > 1 ? c->env_tiles[a] : 1;
    if (c->res[a] % et != 0 || c->res[a] / et < 8) { why = "env_tiles must divide res into tiles of >= 8 nodes"; return 1; }
  }
  if (c->colliders_per_env < 0) { why = "colliders_per_env must be >= 0"; return 1; }
  double nodes = (double)((c->res[0] + 3) / 4) * ((c->res[1] + 3) / 4) * ((c->res[2] + 3) / 4) * 64.0;
  if (nodes >= 2147483647.0) { why = "grid too large for 32-bit node indexing on one device"; return 1; }
  return 0;
}

int alloc_grid(mpm_ctx* ctx) {
  const mpm_config& c = ctx->cfg;
  long long nb = (long long)((c.res[0] + 3) / 4) * ((c.res[1] + 3) / 4) * ((c.res[2] + 3) / 4);
  ctx->nbricks = nb;
  TRY(dalloc(ctx, &ctx->gm, (size_t)nb * 64));
  TRY(dalloc(ctx, &ctx->gv, (size_t)nb * 64));
  TRY(dalloc(ctx, &ctx->brick_flag, (size_t)nb));
  TRY(dalloc(ctx, &ctx->active_list, (size_t)nb));
  CK(cudaMemsetAsync(ctx->gm, 0, sizeof(float4) * nb * 64, ctx->stream));
  CK(cudaMemsetAsync(ctx->gv, 0, sizeof(float4) * nb * 64, ctx->stream));
  CK(cudaMemsetAsync(ctx->brick_flag, 0, sizeof(int) * nb, ctx->stream));
  for (int a = 0; a < 3; ++a) ctx->nbin[a] = (c.res[a] + BIN - 1) / BIN;
  ctx->nbins = ctx->nbin[0] * ctx->nbin[1] * ctx->nbin[2];
  TRY(dalloc(ctx, &ctx->bin_count, (size_t)ctx->nbins));
  TRY(dalloc(ctx, &ctx->bin_start, (size_t)ctx->nbins));
  TRY(dalloc(ctx, &ctx->bin_maxcnt, (size_t)ctx->nbins));
  ctx->grid_dirty = 0;
  ctx->grid_phase = 0;
  return 0;
}

// temp storage for the exclusive scan of up to `n` ints
int ensure_scan(mpm_ctx* ctx, long long n) {
  long long need = n;
  size_t level = 0;
  while (true) {
    long long nb = (need + SCAN_TILE - 1) / SCAN_TILE;
    if (level >= ctx->scan_len.size() || ctx->scan_len[level] < nb) {
      if (level < ctx->scan_len.size()) {
        cudaFree(ctx->scan_tmp[2 * level]);
        cudaFree(ctx->scan_tmp[2 * level + 1]);
      } else {
        ctx->scan_len.push_back(0);
        ctx->scan_tmp.push_back(nullptr);
        ctx->scan_tmp.push_back(nullptr);
      }
      int* a = nullptr;
      int* b = nullptr;
      TRY(dalloc(ctx, &a, (size_t)nb));
      TRY(dalloc(ctx, &b, (size_t)nb));
      ctx->scan_tmp[2 * level] = a;
      ctx->scan_tmp[2 * level + 1] = b;
      ctx->scan_len[level] = nb;
    }
    if (nb <= 1) break;
    need = nb;
    ++level;
  }
  return 0;
}

int scan_exclusive(mpm_ctx* ctx, const int* in, int* out, long long n, size_t level = 0) {
  long long nb = (n + SCAN_TILE - 1) / SCAN_TILE;
  int* sums = ctx->scan_tmp[2 * level];
  int* sums_scanned = ctx->scan_tmp[2 * level + 1];
  scan_tile_kernel<<<(unsigned)nb, SCAN_THREADS, 0, ctx->stream>>>(in, out, sums, n);
  LAUNCHED();
  if (nb > 1) {
    TRY(scan_exclusive(ctx, sums, sums_scanned, nb, level + 1));
    scan_add_kernel<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(out, sums_scanned, n);
    LAUNCHED();
  }
  return 0;
}

int ensure_stage(mpm_ctx* ctx, size_t bytes) {
  if (ctx->stage_bytes >= bytes) return 0;
  TRY(dalloc(ctx, &ctx->stage, bytes / sizeof(double) + 1));
  ctx->stage_bytes = bytes;
  return 0;
}

int ensure_gm_clean(mpm_ctx* ctx) {
  if (ctx->grid_dirty == 2) {
    CK(cudaMemsetAsync(ctx->gm, 0, sizeof(float4) * ctx->nbricks * 64, ctx->stream));
    CK(cudaMemsetAsync(ctx->brick_flag, 0, sizeof(int) * ctx->nbricks, ctx->stream));
  } else if (ctx->grid_dirty == 1) {
    Params p = make_params(ctx);
    clear_active_kernel<<<ctx->clear_blocks, 256, 0, ctx->stream>>>(p);
    LAUNCHED();
  }
  ctx->grid_dirty = 0;
  return 0;
}

// Counting sort of particles by 8^3-cell bin + work list (bin, start, end).
int rebin(mpm_ctx* ctx) {
  TimedRegion tr(ctx, 2);
  Params p = make_params(ctx);
  CK(cudaMemsetAsync(ctx->bin_count, 0, sizeof(int) * ctx->nbins, ctx->stream));
  CK(cudaMemsetAsync(ctx->counters + 1, 0, sizeof(int), ctx->stream));
  bin_key_kernel<<<blocks_for(ctx->n, 256), 256, 0, ctx->stream>>>(p, ctx->key, ctx->lcell, ctx->rank,
                                                                     ctx->bin_count);
  LAUNCHED();
  TRY(scan_exclusive(ctx, ctx->bin_count, ctx->bin_start, ctx->nbins));
  bin_fill_kernel<<<blocks_for(ctx->n, 256), 256, 0, ctx->stream>>>(ctx->key, ctx->lcell, ctx->rank, ctx->bin_start,
                                                                     ctx->sidx, ctx->slc, ctx->n);
  LAUNCHED();
  bin_local_sort_kernel<<<ctx->sms * 4, 256, 0, ctx->stream>>>(ctx->bin_count, ctx->bin_start, ctx->nbins,
                                                                ctx->sidx, ctx->slc, ctx->rank, ctx->bperm,
                                                                ctx->bin_maxcnt);
  LAUNCHED();
  int nxt = ctx->cur ^ 1;
  const long long nvalid = ctx->n - ctx->hole_count;  // migrants' slots are dropped here
  gather_permute_kernel<<<blocks_for(nvalid, 256), 256, 0, ctx->stream>>>(
      ctx->P[ctx->cur], ctx->mat[ctx->cur], ctx->orig[ctx->cur], ctx->P[nxt], ctx->mat[nxt], ctx->orig[nxt],
      ctx->bperm, nvalid, ctx->cap);
  LAUNCHED();
  ctx->cur = nxt;
  ctx->n = nvalid;
  ctx->hole_n = 0;
  ctx->hole_count = 0;
  // ~4 items per SM at least: small scenes split bins, large ones keep whole bins
  const int chunk = (int)std::max<long long>(MIN_CHUNK, std::min<long long>(CHUNK, ctx->n / ((long long)ctx->items_per_sm * ctx->sms)));
  static_assert(4 + 2 * WORK_CLASSES <= 64, "counters too small");
  int* classes = ctx->counters + 4;
  CK(cudaMemsetAsync(classes, 0, sizeof(int) * WORK_CLASSES, ctx->stream));
  make_work_count_kernel<<<blocks_for(ctx->nbins, 256), 256, 0, ctx->stream>>>(ctx->bin_count, ctx->nbins, chunk,
                                                                               classes);
  LAUNCHED();
  make_work_offsets_kernel<<<1, 32, 0, ctx->stream>>>(classes, classes + WORK_CLASSES, ctx->counters + 1);
  LAUNCHED();
  make_work_kernel<<<blocks_for(ctx->nbins, 256), 256, 0, ctx->stream>>>(
      ctx->bin_count, ctx->bin_start, ctx->bin_maxcnt, ctx->nbins, ctx->work, classes + WORK_CLASSES, chunk);
  LAUNCHED();
  return 0;
}

// Slab windows: drop the slots of extracted migrants before anything reads
// the particles in slot order (a re-binning compacts them).
int compact_if_needed(mpm_ctx* ctx) {
  if (ctx->hole_count > 0 || ctx->hole_n > 0) TRY(rebin(ctx));
  return 0;
}

// Launch with programmatic stream serialization when enabled: the kernel may
// be scheduled while its predecessor drains (griddep_wait / griddep_trigger in
// kernels.cuh order the dependent part).
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(mpm_ctx* ctx, void (*kernel)(KArgs...), unsigned grid, unsigned block, size_t smem,
                       Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = ctx->pdl_on ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// One substep's particle work.  g2p=false: first substep after a re-binning
// (v, C from memory): stage A<false> (exact bounds + payload) then stage B.
// g2p=true: the fused steady-state kernel (bounds of the previous substep).
int launch_fused(mpm_ctx* ctx, bool g2p) {
  Params p = make_params(ctx);
  // brick-list / work counters: zeroed by the last clearing grid op, else here
  if (!ctx->counters_clean) {
    CK(cudaMemsetAsync(ctx->counters, 0, sizeof(int), ctx->stream));
    CK(cudaMemsetAsync(ctx->counters + 3, 0, sizeof(int), ctx->stream));
  }
  ctx->counters_clean = false;
  if (!g2p || ctx->split_mode) {
    ctx->bounds_out_clean = false;
    CK(cudaMemsetAsync(ctx->item_bounds, 0, sizeof(float4) * ctx->work_cap, ctx->stream));
    {
      TimedRegion tr(ctx, 0);
      if (g2p)
        g2p_stress_kernel<true><<<ctx->gsA_blocks, FUSED_THREADS, sizeof(float) * 6 * TILE_NODES, ctx->stream>>>(
            p, ctx->pay, ctx->item_bounds, ctx->item_box);
      else
        g2p_stress_kernel<false><<<ctx->gsA0_blocks, FUSED_THREADS, 0, ctx->stream>>>(p, ctx->pay, ctx->item_bounds,
                                                                                 ctx->item_box);
      LAUNCHED();
    }
    {
      TimedRegion tr(ctx, 4);
      p2g_tile_kernel<<<ctx->fused_blocks, P2G_THREADS, P2G_SMEM, ctx->stream>>>(
          p, ctx->pay, ctx->item_bounds, ctx->item_box);
      LAUNCHED();
    }
    return 0;
  }
  // fused: bounds_in = item_bounds (last substep), bounds_out = item_bounds2, then swap
  // (the kernel zeroes each bounds_in entry it consumes, so after one steady
  // launch both buffers stay clean)
  if (!ctx->bounds_out_clean)
    CK(cudaMemsetAsync(ctx->item_bounds2, 0, sizeof(float4) * ctx->work_cap, ctx->stream));
  ctx->bounds_out_clean = true;
  {
    TimedRegion tr(ctx, 5);
    const bool single = p.env_res[0] == p.gres[0] && p.env_res[1] == p.gres[1] && p.env_res[2] == p.gres[2] &&
                        !p.goff[0] && !p.goff[1] && !p.goff[2];
    CK(launch_pdl(ctx, single ? fused_kernel<true> : fused_kernel<false>, ctx->fused_only_blocks, FUSED_K_THREADS, FUSED_SMEM, p,
                  ctx->item_bounds, ctx->item_bounds2, ctx->item_box));
    LAUNCHED();
  }
  std::swap(ctx->item_bounds, ctx->item_bounds2);
  return 0;
}

int launch_grid_op(mpm_ctx* ctx, bool dense, bool use_col, int row, bool clear) {
  Params p = make_params(ctx);
  Colliders cs = make_colliders(ctx, row, use_col);
  TimedRegion tr(ctx, 1);
  int* done = clear && !dense ? ctx->counters + 63 : nullptr;  // counters reset by the last CTA
  if (dense)
    CK(launch_pdl(ctx, grid_op_kernel<true>, ctx->gridop_blocks, 256, 0, p, cs, clear ? 1 : 0, done));
  else if (ctx->gridop_simple)
    CK(launch_pdl(ctx, grid_op_simple_kernel, ctx->gridop_simple_blocks, 256, 0, p, cs, clear ? 1 : 0, done));
  else
    CK(launch_pdl(ctx, grid_op_kernel<false>, ctx->gridop_blocks, 256, 0, p, cs, clear ? 1 : 0, done));
  LAUNCHED();
  if (done) ctx->counters_clean = true;
  return 0;
}

// Substeps row0 .. row0 + nsub - 1 (after the first of a stretch) as one
// cooperative substeps_kernel launch.
int launch_substeps(mpm_ctx* ctx, bool use_col, int row0, int nsub, bool last_clear) {
  Params p = make_params(ctx);
  Colliders cs = make_colliders(ctx, row0, use_col);
  int* ctr = ctx->counters + 50;  // [50..51] active bricks, [52..53] work cursor (by substep parity)
  CK(cudaMemsetAsync(ctr, 0, 4 * sizeof(int), ctx->stream));
  if (!ctx->bounds_out_clean)
    CK(cudaMemsetAsync(ctx->item_bounds2, 0, sizeof(float4) * ctx->work_cap, ctx->stream));
  const ColliderPose* pose_base = ctx->pose;
  int pose_rows = std::max(ctx->pose_rows, 1);
  int pose_stride = std::max(ctx->ncol, 1);
  int lc = last_clear ? 1 : 0;
  float4* bin = ctx->item_bounds;
  float4* bout = ctx->item_bounds2;
  int* final_active = ctx->counters;
  void* args[] = {&p, &cs, &pose_base, &pose_rows, &pose_stride, &row0, &nsub, &lc, &bin, &bout,
                  &ctx->item_box, &ctr, &final_active};
  cudaLaunchConfig_t lc_cfg = {};
  lc_cfg.gridDim = dim3(ctx->mega_blocks);
  lc_cfg.blockDim = dim3(FUSED_K_THREADS);
  lc_cfg.dynamicSmemBytes = FUSED_SMEM;
  lc_cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  lc_cfg.attrs = attr;
  lc_cfg.numAttrs = 1;
  {
    TimedRegion tr(ctx, 6, nsub);
    CK(cudaLaunchKernelExC(&lc_cfg, (const void*)substeps_kernel, args));
    LAUNCHED();
  }
  if (nsub & 1) std::swap(ctx->item_bounds, ctx->item_bounds2);
  ctx->bounds_out_clean = true;
  ctx->counters_clean = false;
  return 0;
}

int launch_g2p(mpm_ctx* ctx);

// The stretch-end G2P of the fast path, per work item from a staged
// velocity tile (work list and item boxes of the stretch's last substep).
int launch_g2p_tiled(mpm_ctx* ctx) {
  if (!ctx->g2p_tiled) return launch_g2p(ctx);
  TimedRegion tr(ctx, 3);
  Params p = make_params(ctx);
  const bool single = p.env_res[0] == p.gres[0] && p.env_res[1] == p.gres[1] && p.env_res[2] == p.gres[2] &&
                      !p.goff[0] && !p.goff[1] && !p.goff[2];
  if (single)
    g2p_tile_kernel<true><<<ctx->g2p_tile_blocks, 256, sizeof(float) * 3 * TILE_NODES, ctx->stream>>>(p, ctx->item_box);
  else
    g2p_tile_kernel<false><<<ctx->g2p_tile_blocks, 256, sizeof(float) * 3 * TILE_NODES, ctx->stream>>>(p, ctx->item_box);
  LAUNCHED();
  return 0;
}

int launch_g2p(mpm_ctx* ctx) {
  TimedRegion tr(ctx, 3);
  Params p = make_params(ctx);
  g2p_kernel<<<blocks_for(ctx->n, 256), 256, 0, ctx->stream>>>(p);
  LAUNCHED();
  return 0;
}

// Deterministic P2G: cell-sorted permutation (ascending cell key, then
// original index), payload, node-owner gather over every node.
int det_p2g(mpm_ctx* ctx) {
  long long ncells = (long long)ctx->cfg.res[0] * ctx->cfg.res[1] * ctx->cfg.res[2];
  if (ctx->ncells != ncells) {
    TRY(dalloc(ctx, &ctx->cell_count, (size_t)ncells));
    TRY(dalloc(ctx, &ctx->cell_start, (size_t)ncells));
    TRY(ensure_scan(ctx, ncells));
    ctx->ncells = ncells;
  }
  if (!ctx->perm) {
    TRY(dalloc(ctx, &ctx->perm, (size_t)ctx->cap));
    TRY(dalloc(ctx, &ctx->payload, (size_t)ctx->cap * 12));
  }
  Params p = make_params(ctx);
  CK(cudaMemsetAsync(ctx->cell_count, 0, sizeof(int) * ncells, ctx->stream));
  cell_key_kernel<<<blocks_for(ctx->n, 256), 256, 0, ctx->stream>>>(p, ctx->key, ctx->rank, ctx->cell_count);
  LAUNCHED();
  TRY(scan_exclusive(ctx, ctx->cell_count, ctx->cell_start, ncells));
  cell_fill_kernel<<<blocks_for(ctx->n, 256), 256, 0, ctx->stream>>>(ctx->key, ctx->rank, ctx->cell_start,
                                                                      ctx->perm, ctx->n);
  LAUNCHED();
  cell_sort_kernel<<<blocks_for(ncells, 256), 256, 0, ctx->stream>>>(ctx->cell_count, ctx->cell_start, ctx->perm,
                                                                      p.orig, ncells);
  LAUNCHED();
  det_payload_kernel<<<blocks_for(ctx->n, 256), 256, 0, ctx->stream>>>(p, ctx->payload);
  LAUNCHED();
  det_gather_kernel<<<blocks_for(ncells, 256), 256, 0, ctx->stream>>>(p, ctx->payload, ctx->cell_count,
                                                                       ctx->cell_start, ctx->perm);
  LAUNCHED();
  ctx->grid_dirty = 2;
  return 0;
}

// An uploaded empty particle set (not a slab window, whose set migrates).
bool empty_state(const mpm_ctx* ctx) { return ctx->n == 0 && ctx->uploaded && ctx->h_cap == 0; }

int zero_grid(mpm_ctx* ctx) {
  CK(cudaMemsetAsync(ctx->gm, 0, sizeof(float4) * ctx->nbricks * 64, ctx->stream));
  CK(cudaMemsetAsync(ctx->brick_flag, 0, sizeof(int) * ctx->nbricks, ctx->stream));
  ctx->grid_dirty = 0;
  return 0;
}

int need_particles(mpm_ctx* ctx, bool materials = true) {
  // a slab window may run empty after migration (it still takes part in the
  // halo protocol and can receive migrants): only its capacity must exist
  if (ctx->n <= 0 && !ctx->uploaded && !(ctx->h_cap > 0 && ctx->cap > 0))
    return fail(ctx, MPM_ESTATE, "no particles uploaded");
  if (materials && ctx->nmat <= 0) return fail(ctx, MPM_ESTATE, "no materials set");
  return 0;
}

int read_inverted(mpm_ctx* ctx, int64_t* out) {
  unsigned long long h = 0;
  CK(cudaMemcpyAsync(&h, ctx->inverted, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (out) *out = (int64_t)h;
  return 0;
}

// The fast-path frame: re-binning + L-substep stretches (captured as a graph).
// skip_rebin: the particles are still in the order of a re-binning at most
// rebin_frames - 1 frames old and nothing outside the fast path moved them;
// the frame keeps that order and work list (the first substep recomputes the
// exact item bounds; particles that drifted off their tiles take the exact
// float path).
int run_fast_sequence(mpm_ctx* ctx, int nsub, bool col, bool skip_rebin = false) {
  TRY(ensure_gm_clean(ctx));
  int s = 0;
  while (s < nsub) {
    const int L = std::min(ctx->cfg.rebin_interval, nsub - s);
    if (!(skip_rebin && s == 0)) TRY(rebin(ctx));
    if (ctx->mega_on && L > 1) {
      TRY(launch_fused(ctx, false));
      TRY(launch_grid_op(ctx, false, col, s, s != nsub - 1));
      TRY(launch_substeps(ctx, col, s + 1, L - 1, s + L - 1 != nsub - 1));
    } else {
      for (int t = 0; t < L; ++t) {
        TRY(launch_fused(ctx, t > 0));
        TRY(launch_grid_op(ctx, false, col, s + t, s + t != nsub - 1));
      }
    }
    TRY(launch_g2p_tiled(ctx));
    s += L;
  }
  ctx->grid_dirty = 1;
  return 0;
}

// ---- host-converted particle transfers -----------------------------------
// The caller's fp64 AoS fields (pageable or pinned) are narrowed to fp32 on
// host worker threads into pinned slots and only fp32 crosses PCIe (half the
// bytes); downloads cross as fp32 and are widened on the host.  Each worker
// owns a contiguous range of the masked fields' concatenated values and
// pipelines its own slots (convert slot k while slot k^1 is in flight) on its
// own copy stream.  Narrowing is (float)d, round to nearest even like the
// device's cvt.rn.f32.f64; widening is exact: results are bit-identical to
// the device-converted path.
constexpr long long XFER_SLOT = 1 << 19;  // floats per pinned slot (2 MB)
constexpr long long XFER_MIN = 1 << 20;   // values below which the calling thread converts alone

// Process-wide transfer workers (contexts come and go: the reference's tests
// build one per SimState): the thread pool, the pinned slots (portable), and
// per device a copy stream and three events per worker.  Transfers of all
// contexts are serialised on its mutex.  Never freed (idle threads at exit).
struct XferShared {
  std::mutex m;
  HostPool* pool = nullptr;
  float* slots = nullptr;
  int nt = 0;
  struct Dev {
    int dev;
    std::vector<cudaStream_t> st;
    std::vector<cudaEvent_t> ev;  // 3 per worker: slot 0, slot 1, done
  };
  std::vector<Dev> devs;
};
XferShared* g_xfer = nullptr;
XferShared& xfer_shared() {
  static std::once_flag once;
  std::call_once(once, [] {
    g_xfer = new XferShared;
    // a forked child has none of the parent's worker threads (nor a usable
    // CUDA context): it starts from an empty state instead of waiting on them
    pthread_atfork(nullptr, nullptr, [] { g_xfer = new XferShared; });
  });
  return *g_xfer;
}

// (called with the XferShared mutex held)
int ensure_xfer(mpm_ctx* ctx, XferShared::Dev** out) {
  XferShared& g = xfer_shared();
  if (!g.pool) {
    // (1 M particles, 192 MB of fp64 each way, on the B200 box's 16 host
    // threads: 8 workers 4.0 / 4.3 ms down / up, 12: 3.1 / 3.0, 16: 2.9 / 2.8;
    // fp64 over PCIe with device conversion: 3.4 / 3.5)
    int nt = (int)std::min<unsigned>(16u, std::max(1u, std::thread::hardware_concurrency()));
    const char* e = getenv("SOFTMPM_HOST_THREADS");
    if (e && atoi(e) > 0) nt = atoi(e);
    void* h = nullptr;
    CK(cudaHostAlloc(&h, sizeof(float) * XFER_SLOT * 2 * nt, cudaHostAllocPortable));
    g.slots = static_cast<float*>(h);
    g.nt = nt;
    g.pool = new HostPool(nt);
  }
  for (auto& d : g.devs)
    if (d.dev == ctx->dev) {
      *out = &d;
      return 0;
    }
  XferShared::Dev d;
  d.dev = ctx->dev;
  d.st.resize(g.nt);
  d.ev.resize(3 * g.nt);
  for (int t = 0; t < g.nt; ++t) {
    CK(cudaStreamCreateWithFlags(&d.st[t], cudaStreamNonBlocking));
    for (int k = 0; k < 3; ++k) CK(cudaEventCreateWithFlags(&d.ev[3 * t + k], cudaEventDisableTiming));
  }
  g.devs.push_back(std::move(d));
  *out = &g.devs.back();
  return 0;
}

struct XferSeg {
  double* host;
  long long count, voff;
};

// Pageable (not pinned / registered) host memory: DMA from it is staged by
// the driver at a fraction of PCIe bandwidth.
bool host_pageable(const void* ptr) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

// fp64 -> fp32 into a pinned slot with streaming (non-temporal) stores: the
// slot is read by the DMA engine right after, and a slot left dirty in the
// CPU caches is read over PCIe at ~11 GB/s instead of ~55 (measured on the
// B200 box's host); cvtpd2ps rounds to nearest even like (float)d.
static void narrow_stream(const double* src, float* dst, long long m) {
  long long i = 0;
  for (; i < m && (reinterpret_cast<uintptr_t>(dst + i) & 15); ++i) dst[i] = (float)src[i];
  for (; i + 4 <= m; i += 4) {
    const __m128 lo = _mm_cvtpd_ps(_mm_loadu_pd(src + i));
    const __m128 hi = _mm_cvtpd_ps(_mm_loadu_pd(src + i + 2));
    _mm_stream_ps(dst + i, _mm_movelh_ps(lo, hi));
  }
  for (; i < m; ++i) dst[i] = (float)src[i];
  _mm_sfence();
}

// fp32 slot -> the caller's fp64 array with streaming stores (no read for
// ownership of the destination lines).  keep_equal: a destination value
// whose fp32 rounding equals the slot value is kept (MPM_DOWNLOAD_KEEP_EQUAL).
static void widen_stream(const float* src, double* dst, long long m, bool keep_equal) {
  long long i = 0;
  auto one = [&](long long k) {
    if (!keep_equal || (float)dst[k] != src[k]) dst[k] = (double)src[k];
  };
  for (; i < m && (reinterpret_cast<uintptr_t>(dst + i) & 15); ++i) one(i);
  for (; i + 2 <= m; i += 2) {
    const __m128d w = _mm_cvtps_pd(_mm_castsi128_ps(_mm_loadl_epi64(reinterpret_cast<const __m128i*>(src + i))));
    if (keep_equal) {
      const __m128d old = _mm_load_pd(dst + i);
      // keep old where its fp32 rounding equals the new value (== on the
      // fp32 values, so NaN never compares equal and -0 == +0 as in C)
      const __m128 eq = _mm_cmpeq_ps(_mm_cvtpd_ps(old), _mm_cvtpd_ps(w));
      const __m128d m2 = _mm_castps_pd(_mm_unpacklo_ps(eq, eq));
      _mm_stream_pd(dst + i, _mm_or_pd(_mm_and_pd(m2, old), _mm_andnot_pd(m2, w)));
    } else {
      _mm_stream_pd(dst + i, w);
    }
  }
  for (; i < m; ++i) one(i);
  _mm_sfence();
}

// Values [a, b) of the virtual (concatenated) field array: dir 0 narrows host
// fp64 into dst, dir 1 widens src into host fp64.
static void xfer_convert(const std::vector<XferSeg>& segs, long long a, long long b, float* slot, int dir,
                         bool keep_equal) {
  for (const XferSeg& g : segs) {
    const long long lo = std::max(a, g.voff), hi = std::min(b, g.voff + g.count);
    if (lo >= hi) continue;
    double* hp = g.host + (lo - g.voff);
    float* sp = slot + (lo - a);
    const long long m = hi - lo;
    if (dir == 0)
      narrow_stream(hp, sp, m);
    else
      widen_stream(sp, hp, m, keep_equal);
  }
}

// dir 0: host -> device stage; dir 1: device stage -> host.  `ready` is
// recorded on ctx->stream before (the stage may be written / has been
// written); the workers' completion is joined into ctx->stream (upload).
int xfer_run(mpm_ctx* ctx, const std::vector<XferSeg>& segs, long long total, float* dstage, int dir,
             cudaEvent_t ready, bool keep_equal = false) {
  XferShared& g = xfer_shared();
  std::lock_guard<std::mutex> guard(g.m);
  XferShared::Dev* dv = nullptr;
  TRY(ensure_xfer(ctx, &dv));
  const int nrun = total < XFER_MIN ? 1 : g.nt;
  std::atomic<int> err{0};
  std::string msg;
  std::mutex msg_m;
  auto fn = [&](int t, int nt) {
    auto ck = [&](cudaError_t e) {
      if (e != cudaSuccess && !err.exchange(1)) {
        std::lock_guard<std::mutex> l(msg_m);
        msg = cudaGetErrorString(e);
      }
      return e == cudaSuccess;
    };
    if (!ck(cudaSetDevice(ctx->dev))) return;
    const long long lo = total * t / nt, hi = total * (t + 1) / nt;
    cudaStream_t st = dv->st[t];
    float* slot[2] = {g.slots + XFER_SLOT * 2 * t, g.slots + XFER_SLOT * (2 * t + 1)};
    cudaEvent_t ev[2] = {dv->ev[3 * t], dv->ev[3 * t + 1]};
    if (!ck(cudaStreamWaitEvent(st, ready, 0))) return;
    if (dir == 0) {
      bool used[2] = {false, false};
      int k = 0;
      for (long long a = lo; a < hi; a += XFER_SLOT, k ^= 1) {
        const long long b = std::min(a + XFER_SLOT, hi);
        if (used[k] && !ck(cudaEventSynchronize(ev[k]))) return;  // the slot's last copy is done
        xfer_convert(segs, a, b, slot[k], 0, false);
        if (!ck(cudaMemcpyAsync(dstage + a, slot[k], sizeof(float) * (b - a), cudaMemcpyHostToDevice, st))) return;
        if (!ck(cudaEventRecord(ev[k], st))) return;
        used[k] = true;
      }
      ck(cudaEventRecord(dv->ev[3 * t + 2], st));
    } else {
      // copy of chunk j + 1 in flight while chunk j is widened
      auto issue = [&](long long a, int k) {
        const long long b = std::min(a + XFER_SLOT, hi);
        return ck(cudaMemcpyAsync(slot[k], dstage + a, sizeof(float) * (b - a), cudaMemcpyDeviceToHost, st)) &&
               ck(cudaEventRecord(ev[k], st));
      };
      if (lo < hi && !issue(lo, 0)) return;
      int k = 0;
      for (long long a = lo; a < hi; a += XFER_SLOT, k ^= 1) {
        if (a + XFER_SLOT < hi && !issue(a + XFER_SLOT, k ^ 1)) return;
        if (!ck(cudaEventSynchronize(ev[k]))) return;
        xfer_convert(segs, a, std::min(a + XFER_SLOT, hi), slot[k], 1, keep_equal);
      }
    }
  };
  if (nrun == 1)
    fn(0, 1);
  else
    g.pool->run(fn);
  if (err.load()) return fail(ctx, MPM_ECUDA, "host transfer: " + msg);
  if (dir == 0)
    for (int t = 0; t < nrun; ++t) CK(cudaStreamWaitEvent(ctx->stream, dv->ev[3 * t + 2], 0));
  if (dir == 0 && cudaStreamSynchronize(ctx->stream) != cudaSuccess)  // slots reusable once the copies are done
    return fail(ctx, MPM_ECUDA, "host transfer: sync");
  return 0;
}

}  // namespace

extern "C" {

const char* mpm_version(void) { return "softmpm_b200 0.1 (sm_100a)"; }

const char* mpm_last_error(mpm_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int64_t mpm_launch_count(mpm_ctx* ctx) { return ctx ? ctx->launches : 0; }

int mpm_create(mpm_ctx** out, const mpm_config* cfg) {
  if (!out || !cfg) return MPM_EINVAL;
  *out = nullptr;
  std::string why;
  if (validate(cfg, why)) {
    static thread_local std::string last;
    last = why;
    return MPM_EINVAL;
  }
  mpm_ctx* ctx = new mpm_ctx();
  ctx->cfg = *cfg;
  if (ctx->cfg.rebin_interval < 1) ctx->cfg.rebin_interval = 25;
  ctx->dev = cfg->device;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= 0) {
    cudaGetLastError();
    delete ctx;
    return MPM_ECUDA;
  }
  if (cudaSetDevice(ctx->dev) != cudaSuccess) {
    delete ctx;
    return MPM_ECUDA;
  }
  cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, ctx->dev);
  int rc = 0;
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) rc = MPM_ECUDA;
  if (!rc && cudaStreamCreateWithFlags(&ctx->xstream, cudaStreamNonBlocking) != cudaSuccess) rc = MPM_ECUDA;
  for (int k = 0; k < 4 && !rc; ++k)
    if (cudaEventCreateWithFlags(&ctx->field_ev[k], cudaEventDisableTiming) != cudaSuccess) rc = MPM_ECUDA;
  if (!rc) rc = alloc_grid(ctx);
  if (!rc) rc = dalloc(ctx, &ctx->counters, 64);
  if (!rc) rc = dalloc(ctx, &ctx->inverted, 1);
  if (!rc) rc = dalloc(ctx, &ctx->stats, 8);
  if (!rc) rc = cudaMemset(ctx->stats, 0, 8 * sizeof(unsigned long long)) == cudaSuccess ? 0 : MPM_ECUDA;
  if (!rc) rc = dalloc(ctx, &ctx->flag, 1);
  if (!rc) rc = ensure_scan(ctx, ctx->nbins);
  if (!rc && cudaMemsetAsync(ctx->counters, 0, 64 * sizeof(int), ctx->stream) != cudaSuccess) rc = MPM_ECUDA;
  if (!rc) {
    cudaEventCreate(&ctx->ev0);
    cudaEventCreate(&ctx->ev1);
    size_t smem = P2G_SMEM;
    cudaFuncSetAttribute(fused_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(FUSED_SMEM));
    cudaFuncSetAttribute(fused_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(FUSED_SMEM));
    {
      const char* e = getenv("SOFTMPM_SPLIT");
      ctx->split_mode = e && e[0] == '1';
      const char* g = getenv("SOFTMPM_GRAPHS");
      ctx->graphs_on = !(g && g[0] == '0');
      const char* ips = getenv("SOFTMPM_ITEMS_PER_SM");
      if (ips && atoi(ips) > 0) ctx->items_per_sm = atoi(ips);
    }
    cudaFuncSetAttribute(g2p_stress_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(sizeof(float) * 6 * TILE_NODES));
    cudaFuncSetAttribute(p2g_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, p2g_tile_kernel, P2G_THREADS, smem);
    ctx->fused_blocks = ctx->sms * std::max(1, occ);
    auto persistent = [&](const void* fn, int threads, size_t dyn) {
      int o = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, threads, dyn);
      return ctx->sms * std::max(1, o);
    };
    {
      const char* gb = getenv("SOFTMPM_GRIDOP_BLOCKS");  // CTAs per SM (A/B runs)
      ctx->gridop_blocks = ctx->sms * (gb && atoi(gb) > 0 ? atoi(gb) : GRIDOP_MIN_BLOCKS);
      ctx->gridop_simple_blocks = persistent((const void*)grid_op_simple_kernel, 256, 0);
      const char* gs = getenv("SOFTMPM_GRIDOP_SIMPLE");
      if (gs) ctx->gridop_simple = gs[0] == '1';
      const char* hx = getenv("SOFTMPM_HOST_XFER");
      if (hx) ctx->host_xfer = hx[0] == '1';
      const char* xd = getenv("SOFTMPM_XFER_DIRECT");
      if (xd) ctx->xfer_direct = xd[0] == '1';
      const char* rf = getenv("SOFTMPM_REBIN_FRAMES");
      if (rf && atoi(rf) >= 1) ctx->rebin_frames = atoi(rf);
    }
    ctx->gsA_blocks = persistent((const void*)g2p_stress_kernel<true>, FUSED_THREADS, sizeof(float) * 6 * TILE_NODES);
    ctx->gsA0_blocks = persistent((const void*)g2p_stress_kernel<false>, FUSED_THREADS, 0);
    ctx->clear_blocks = persistent((const void*)clear_active_kernel, 256, 0);
    ctx->g2p_tile_blocks = persistent((const void*)g2p_tile_kernel<true>, 256, sizeof(float) * 3 * TILE_NODES);
    {
      const char* gt = getenv("SOFTMPM_G2P_TILED");
      if (gt) ctx->g2p_tiled = gt[0] == '1';
    }
    ctx->fused_only_blocks = persistent((const void*)fused_kernel<true>, FUSED_K_THREADS, FUSED_SMEM);
    cudaFuncSetAttribute(substeps_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(FUSED_SMEM));
    ctx->mega_blocks = persistent((const void*)substeps_kernel, FUSED_K_THREADS, FUSED_SMEM);
    {
      int coop = 0;
      cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, ctx->dev);
      const char* mg = getenv("SOFTMPM_MEGA");
      ctx->mega_coop = coop != 0;
      ctx->mega_on = coop && mg && mg[0] == '1';
      const char* pd = getenv("SOFTMPM_PDL");
      if (pd) ctx->pdl_on = pd[0] == '1';
    }
    if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) rc = MPM_ECUDA;
  }
  if (rc) {
    mpm_destroy(ctx);
    return rc;
  }
  *out = ctx;
  return 0;
}

int mpm_destroy(mpm_ctx* ctx) {
  if (!ctx) return 0;
  cudaSetDevice(ctx->dev);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
#ifdef FUSED_PROFILE
  {
    unsigned long long h[6];
    cudaMemcpyFromSymbol(h, g_fprof, sizeof(h));
    const double tot = (double)(h[0] + h[1] + h[2] + h[3] + h[4]);
    fprintf(stderr, "[fused profile] warp-cycles: particles %.3f  wait[B] %.3f  flush %.3f  next-tile %.3f  wait[A] %.3f  (total %.3e, ctas %llu)\n",
            h[0] / tot, h[1] / tot, h[2] / tot, h[3] / tot, h[4] / tot, tot, h[5]);
    unsigned long long g[8];
    cudaMemcpyFromSymbol(g, g_gprof, sizeof(g));
    if (g[3])
      fprintf(stderr, "[grid profile] launches %llu  mean CTA %.2f us  mean per-launch max CTA %.2f us (clearing launches %llu, bricks/launch %.0f)  CTAs/launch %llu\n",
              g[3], g[0] / (double)(g[2] ? g[2] : 1) / 1e3, g[4] / (double)(g[5] ? g[5] : 1) / 1e3, g[5],
              g[6] / (double)(g[5] ? g[5] : 1), g[2] / g[3]);
    unsigned long long gw[4];
    cudaMemcpyFromSymbol(gw, g_gwin, sizeof(gw));
    if (g[5])
      fprintf(stderr, "[grid window] first CTA start -> last CTA end %.2f us, start spread %.2f us (per clearing launch)\n",
              (gw[2] >> 20) / (double)g[5] / 1e3, (gw[2] & ((1ull << 20) - 1)) / (double)g[5] / 1e3);
    unsigned long long bb[8];
    cudaMemcpyFromSymbol(bb, g_bub, sizeof(bb));
    fprintf(stderr, "[bubbles] fused last CTA end -> grid op first CTA start %.2f us (n %llu); grid op end -> fused first start %.2f us (n %llu)\n",
            bb[4] / (double)(bb[5] ? bb[5] : 1) / 1e3, bb[5], bb[6] / (double)(bb[7] ? bb[7] : 1) / 1e3, bb[7]);
    unsigned long long fw[4];
    cudaMemcpyFromSymbol(fw, g_fwin, sizeof(fw));
    fprintf(stderr, "[fused window] first CTA start -> last CTA end %.2f us (n %llu), mean CTA duration %.2f us\n",
            fw[0] / (double)(fw[1] ? fw[1] : 1) / 1e3, fw[1], fw[2] / (double)(fw[3] ? fw[3] : 1) / 1e3);
    unsigned long long cc[4];
    cudaMemcpyFromSymbol(cc, g_cprof, sizeof(cc));
    if (g[3])
      fprintf(stderr, "[contact profile] warp calls/launch %.1f  lanes/call %.1f  cycles/call %.0f  max %llu\n",
              cc[0] / (double)g[3], cc[1] / (double)(cc[0] ? cc[0] : 1), cc[2] / (double)(cc[0] ? cc[0] : 1), cc[3]);
    unsigned long long ph[4];
    cudaMemcpyFromSymbol(ph, g_cph, sizeof(ph));
    fprintf(stderr, "[contact phases] thread-cycles: nearest %.3e  pre-normal %.3e  normal %.3e  nearest->end %.3e\n",
            (double)ph[0], (double)ph[1], (double)ph[2], (double)ph[3]);
    unsigned long long c[4];
    cudaMemcpyFromSymbol(c, g_fcnt, sizeof(c));
    fprintf(stderr, "[fused profile] particles %llu  g2p off-tile %llu (%.4f)  p2g fallback %llu (%.4f, bound %llu)\n",
            c[0], c[1], c[1] / (double)(c[0] ? c[0] : 1), c[2], c[2] / (double)(c[0] ? c[0] : 1), c[3]);
  }
#endif
  invalidate_graphs(ctx);
  for (int sd = 0; sd < 2; ++sd) {
    if (!ctx->peer_local[sd])
      for (void* q : {(void*)ctx->peer_ids[sd], (void*)ctx->peer_data[sd], (void*)ctx->peer_cnt[sd], (void*)ctx->peer_vdata[sd]})
        if (q) cudaIpcCloseMemHandle(q);
    for (cudaEvent_t e : {ctx->ipc_free[sd], ctx->ipc_ready[sd]})
      if (e) cudaEventDestroy(e);
    if (!ctx->peer_local[sd])  // same-process peers: the neighbour owns these events
      for (cudaEvent_t e : {ctx->peer_free[sd], ctx->peer_ready[sd]})
        if (e) cudaEventDestroy(e);
    if (ctx->ipc_vrecv[sd]) cudaFree(ctx->ipc_vrecv[sd]);
    if (ctx->ipc_cnt[sd]) cudaFree(ctx->ipc_cnt[sd]);
  }
  void* bufs[] = {ctx->gm, ctx->gv, ctx->brick_flag, ctx->active_list, ctx->counters, ctx->P[0], ctx->P[1], ctx->item_bounds, ctx->item_bounds2, ctx->pay, ctx->lcell, ctx->sidx, ctx->slc, ctx->bperm, ctx->item_box, ctx->mflag, ctx->mig_rows[0], ctx->mig_rows[1], ctx->h_send_ids[0], ctx->h_send_ids[1],
                  ctx->h_send_data[0], ctx->h_send_data[1], ctx->h_recv_ids[0], ctx->h_recv_ids[1], ctx->h_recv_data[0],
                  ctx->h_recv_data[1], ctx->h_local_ids[0], ctx->h_local_ids[1],
                  ctx->mat[0], ctx->mat[1], ctx->orig[0], ctx->orig[1], ctx->key, ctx->rank, ctx->bin_count,
                  ctx->bin_start, ctx->bin_maxcnt, ctx->work, ctx->mu, ctx->lam, ctx->inverted, ctx->stats, ctx->geo, ctx->pose, ctx->sdf,
                  ctx->cell_count, ctx->cell_start, ctx->perm, ctx->payload, ctx->stage, ctx->flag, ctx->x0, ctx->field, ctx->mc_flag, ctx->mc_vid, ctx->mc_cnt, ctx->mc_off, ctx->mesh_v, ctx->mesh_t, ctx->enc};
  for (void* b : bufs)
    if (b) cudaFree(b);
  for (int* b : ctx->scan_tmp)
    if (b) cudaFree(b);
  for (auto& mk : ctx->marks) {
    cudaEventDestroy(mk.a);
    cudaEventDestroy(mk.b);
  }
  for (cudaEvent_t e : ctx->event_pool) cudaEventDestroy(e);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  if (ctx->xstream) cudaStreamDestroy(ctx->xstream);
  for (cudaEvent_t e : ctx->field_ev)
    if (e) cudaEventDestroy(e);
  delete ctx;
  return 0;
}

int mpm_set_config(mpm_ctx* ctx, const mpm_config* cfg) {
  if (ctx) ctx->bins_age = -1;  // particle order / positions may change: the next frame re-bins
  if (!ctx || !cfg) return MPM_EINVAL;
  invalidate_graphs(ctx);
  std::string why;
  if (validate(cfg, why)) return fail(ctx, MPM_EINVAL, why);
  for (int a = 0; a < 3; ++a)
    if (cfg->res[a] != ctx->cfg.res[a] || cfg->dx != ctx->cfg.dx)
      return fail(ctx, MPM_EINVAL, "grid geometry cannot change on a live context");
  int keep_dev = ctx->cfg.device;
  ctx->cfg = *cfg;
  ctx->cfg.device = keep_dev;
  if (ctx->cfg.rebin_interval < 1) ctx->cfg.rebin_interval = 25;
  return 0;
}

int mpm_set_materials(mpm_ctx* ctx, const double* mu, const double* lam, int count) {
  if (!ctx || !mu || !lam || count <= 0) return fail(ctx, MPM_EINVAL, "materials: bad arguments");
  CK(cudaSetDevice(ctx->dev));
  if (count != ctx->nmat) invalidate_graphs(ctx);
  std::vector<float> m(count), l(count);
  for (int i = 0; i < count; ++i) {
    m[i] = (float)mu[i];
    l[i] = (float)lam[i];
  }
  if (count != ctx->nmat) {
    TRY(dalloc(ctx, &ctx->mu, (size_t)count));
    TRY(dalloc(ctx, &ctx->lam, (size_t)count));
    ctx->nmat = count;
  }
  CK(cudaMemcpyAsync(ctx->mu, m.data(), sizeof(float) * count, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->lam, l.data(), sizeof(float) * count, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return 0;
}

int mpm_upload_particles(mpm_ctx* ctx, int64_t n, const double* x, const double* v, const double* F,
                         const double* C, const double* mass, const double* vol0, const int32_t* material_id) {
  if (ctx) ctx->bins_age = -1;  // particle order / positions may change: the next frame re-bins
  if (!ctx || n < 0 || (n > 0 && (!x || !v || !F || !C || !mass || !vol0 || !material_id)))
    return fail(ctx, MPM_EINVAL, "upload_particles: bad arguments");
  if (n == 0) {
    // an empty state (the reference steps it: grid ops on an empty grid, the
    // clock advances): nothing to allocate, every particle stage a no-op
    invalidate_graphs(ctx);
    ctx->n = 0;
    ctx->cur = 0;
    ctx->uploaded = true;
    return 0;
  }
  if (n >= (1LL << 31) - CHUNK) return fail(ctx, MPM_EINVAL, "too many particles for one context");
  for (int64_t i = 0; i < n; ++i)
    if (material_id[i] < 0 || (ctx->nmat > 0 && material_id[i] >= ctx->nmat))
      return fail(ctx, MPM_EINVAL, "material id out of range");
  CK(cudaSetDevice(ctx->dev));
  invalidate_graphs(ctx);
  if (n > ctx->cap) {
    long long cap = n;
    for (int b = 0; b < 2; ++b) {
      TRY(dalloc(ctx, &ctx->P[b], (size_t)cap * NF));
      TRY(dalloc(ctx, &ctx->mat[b], (size_t)cap));
      TRY(dalloc(ctx, &ctx->orig[b], (size_t)cap));
    }
    TRY(dalloc(ctx, &ctx->key, (size_t)cap));
    TRY(dalloc(ctx, &ctx->rank, (size_t)cap));
    TRY(dalloc(ctx, &ctx->lcell, (size_t)cap));
    TRY(dalloc(ctx, &ctx->sidx, (size_t)cap));
    TRY(dalloc(ctx, &ctx->slc, (size_t)cap));
    TRY(dalloc(ctx, &ctx->bperm, (size_t)cap));
    ctx->work_cap = ctx->nbins + cap / MIN_CHUNK + 1;
    TRY(dalloc(ctx, &ctx->work, (size_t)ctx->work_cap));
    TRY(dalloc(ctx, &ctx->item_bounds, (size_t)ctx->work_cap));
    TRY(dalloc(ctx, &ctx->item_bounds2, (size_t)ctx->work_cap));
    ctx->bounds_a = ctx->item_bounds;
    ctx->bounds_out_clean = false;
    TRY(dalloc(ctx, &ctx->pay, (size_t)cap * NPAY));
    TRY(dalloc(ctx, &ctx->item_box, (size_t)ctx->work_cap));
    if (ctx->perm) {
      cudaFree(ctx->perm);
      cudaFree(ctx->payload);
      ctx->perm = nullptr;
      ctx->payload = nullptr;
    }
    ctx->cap = cap;
  }
  ctx->n = n;
  ctx->cur = 0;
  ctx->uploaded = true;
  TRY(ensure_stage(ctx, sizeof(double) * (size_t)n * 24));
  double* s = ctx->stage;
  CK(cudaMemcpyAsync(s, mass, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(s + n, vol0, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(s + 2 * n, material_id, sizeof(int32_t) * n, cudaMemcpyHostToDevice, ctx->stream));
  Params p = make_params(ctx);
  upload_static_kernel<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(p, s, s + n, (const int*)(s + 2 * n));
  LAUNCHED();
  return mpm_upload_fields(ctx, MPM_FIELD_ALL, x, v, F, C);
}

int mpm_upload_fields(mpm_ctx* ctx, uint32_t mask, const double* x, const double* v, const double* F,
                      const double* C) {
  if (ctx) ctx->bins_age = -1;  // particle order / positions may change: the next frame re-bins
  if (!ctx) return MPM_EINVAL;
  if (ctx->n <= 0) return ctx->uploaded ? 0 : fail(ctx, MPM_ESTATE, "upload_fields: no particles");
  if (!mask) return 0;
  CK(cudaSetDevice(ctx->dev));
  long long n = ctx->n;
  TRY(ensure_stage(ctx, sizeof(double) * (size_t)n * 24));
  const double* src[4] = {x, v, F, C};
  const int width[4] = {3, 3, 9, 9};
  Params p = make_params(ctx);
  // host-converted fp32 wire: pageable buffers (driver-staged DMA from them
  // runs at ~11 GB/s) and every large transfer (host conversion on all
  // threads beats the fp64 DMA); small pinned ones go as fp64
  bool pageable = false;
  long long nval = 0;
  for (int k = 0; k < 4; ++k)
    if (((mask >> k) & 1u) && src[k]) {
      pageable |= host_pageable(src[k]);
      nval += width[k] * n;
    }
  if (ctx->host_xfer && (pageable || nval >= XFER_MIN)) {
    // pinned buffers: x and v cross as fp64 straight from the caller's memory
    // (device conversion) while the host threads narrow F and C, so PCIe and
    // host memory bandwidth are both busy
    const uint32_t direct = (!pageable && ctx->xfer_direct) ? (mask & 3u) : 0u;
    double* st64 = ctx->stage;                                  // direct: x at 0, v at 3n
    float* dst = reinterpret_cast<float*>(ctx->stage + 6 * n);  // fp32 wire after it
    CK(cudaEventRecord(ctx->field_ev[0], ctx->stream));  // stage buffer free
    if (direct) {
      CK(cudaStreamWaitEvent(ctx->xstream, ctx->field_ev[0], 0));
      for (int k = 0; k < 2; ++k)
        if (((direct >> k) & 1u) && src[k])
          CK(cudaMemcpyAsync(st64 + 3 * n * k, src[k], sizeof(double) * 3 * n, cudaMemcpyHostToDevice, ctx->xstream));
      CK(cudaEventRecord(ctx->field_ev[1], ctx->xstream));
    }
    std::vector<XferSeg> segs;
    float* f32[4] = {nullptr, nullptr, nullptr, nullptr};
    long long total = 0;
    for (int k = 0; k < 4; ++k) {
      if (!((mask >> k) & 1u) || !src[k] || ((direct >> k) & 1u)) continue;
      segs.push_back({const_cast<double*>(src[k]), width[k] * n, total});
      f32[k] = dst + total;
      total += width[k] * n;
    }
    if (total) TRY(xfer_run(ctx, segs, total, dst, 0, ctx->field_ev[0]));
    if (direct) {
      CK(cudaStreamWaitEvent(ctx->stream, ctx->field_ev[1], 0));
      upload_fields_kernel<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(p, st64, st64 + 3 * n, nullptr, nullptr,
                                                                          direct);
      LAUNCHED();
    }
    if (total) {
      upload_fields32_kernel<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(p, f32[0], f32[1], f32[2], f32[3]);
      LAUNCHED();
    }
    CK(cudaStreamSynchronize(ctx->stream));
    return 0;
  }
  double* st[4] = {ctx->stage, ctx->stage + 3 * n, ctx->stage + 6 * n, ctx->stage + 15 * n};
  // field k's H2D copy (copy stream) overlaps field k-1's conversion
  CK(cudaEventRecord(ctx->field_ev[0], ctx->stream));
  CK(cudaStreamWaitEvent(ctx->xstream, ctx->field_ev[0], 0));  // stage buffer free
  for (int k = 0; k < 4; ++k) {
    if (!((mask >> k) & 1u) || !src[k]) continue;
    CK(cudaMemcpyAsync(st[k], src[k], sizeof(double) * width[k] * n, cudaMemcpyHostToDevice, ctx->xstream));
    CK(cudaEventRecord(ctx->field_ev[k], ctx->xstream));
    CK(cudaStreamWaitEvent(ctx->stream, ctx->field_ev[k], 0));
    upload_fields_kernel<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(p, st[0], st[1], st[2], st[3], 1u << k);
    LAUNCHED();
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return 0;
}

int mpm_download_particles(mpm_ctx* ctx, uint32_t mask, double* x, double* v, double* F, double* C) {
  if (!ctx) return MPM_EINVAL;
  if (ctx->n <= 0 && ctx->h_cap == 0) return ctx->uploaded ? 0 : fail(ctx, MPM_ESTATE, "download: no particles");
  CK(cudaSetDevice(ctx->dev));
  TRY(compact_if_needed(ctx));
  long long n = ctx->n;
  if (n <= 0) return 0;  // (a slab window that currently owns no particles)
  TRY(ensure_stage(ctx, sizeof(double) * (size_t)n * 24));
  double* dst[4] = {x, v, F, C};
  const int width[4] = {3, 3, 9, 9};
  Params p = make_params(ctx);
  const bool keep_equal = (mask & MPM_DOWNLOAD_KEEP_EQUAL) != 0;
  bool pageable = false;  // (as in mpm_upload_fields)
  long long nval = 0;
  for (int k = 0; k < 4; ++k)
    if (((mask >> k) & 1u) && dst[k]) {
      pageable |= host_pageable(dst[k]);
      nval += width[k] * n;
    }
  if (keep_equal || (ctx->host_xfer && (pageable || nval >= XFER_MIN))) {
    const uint32_t direct = (!pageable && !keep_equal && ctx->xfer_direct) ? (mask & 3u) : 0u;
    double* st64 = ctx->stage;
    float* sb = reinterpret_cast<float*>(ctx->stage + 6 * n);
    if (direct) {
      download_fields_kernel<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(p, st64, st64 + 3 * n, nullptr, nullptr,
                                                                            direct);
      LAUNCHED();
      CK(cudaEventRecord(ctx->field_ev[1], ctx->stream));
      CK(cudaStreamWaitEvent(ctx->xstream, ctx->field_ev[1], 0));
      for (int k = 0; k < 2; ++k)
        if (((direct >> k) & 1u) && dst[k])
          CK(cudaMemcpyAsync(dst[k], st64 + 3 * n * k, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, ctx->xstream));
    }
    std::vector<XferSeg> segs;
    float* f32[4] = {nullptr, nullptr, nullptr, nullptr};
    long long total = 0;
    for (int k = 0; k < 4; ++k) {
      if (!((mask >> k) & 1u) || !dst[k] || ((direct >> k) & 1u)) continue;
      segs.push_back({dst[k], width[k] * n, total});
      f32[k] = sb + total;
      total += width[k] * n;
    }
    if (total) {
      download_fields32_kernel<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(p, f32[0], f32[1], f32[2], f32[3]);
      LAUNCHED();
      CK(cudaEventRecord(ctx->field_ev[0], ctx->stream));
      TRY(xfer_run(ctx, segs, total, sb, 1, ctx->field_ev[0], keep_equal));
    }
    if (direct) CK(cudaStreamSynchronize(ctx->xstream));
    return 0;
  }
  double* st[4] = {ctx->stage, ctx->stage + 3 * n, ctx->stage + 6 * n, ctx->stage + 15 * n};
  // field k's D2H copy (copy stream) overlaps field k+1's conversion
  for (int k = 0; k < 4; ++k) {
    if (!((mask >> k) & 1u) || !dst[k]) continue;
    download_fields_kernel<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(p, st[0], st[1], st[2], st[3], 1u << k);
    LAUNCHED();
    CK(cudaEventRecord(ctx->field_ev[k], ctx->stream));
    CK(cudaStreamWaitEvent(ctx->xstream, ctx->field_ev[k], 0));
    CK(cudaMemcpyAsync(dst[k], st[k], sizeof(double) * width[k] * n, cudaMemcpyDeviceToHost, ctx->xstream));
  }
  CK(cudaStreamSynchronize(ctx->xstream));
  CK(cudaStreamSynchronize(ctx->stream));
  return 0;
}

int64_t mpm_particle_count(mpm_ctx* ctx) { return ctx ? ctx->n - ctx->hole_count : 0; }

int mpm_upload_grid(mpm_ctx* ctx, int target, const double* grid_mv, const double* grid_m) {
  if (ctx) ctx->bins_age = -1;  // particle order / positions may change: the next frame re-bins
  if (!ctx || !grid_mv || (target != 0 && target != 1)) return fail(ctx, MPM_EINVAL, "upload_grid: bad arguments");
  CK(cudaSetDevice(ctx->dev));
  long long nn = (long long)ctx->cfg.res[0] * ctx->cfg.res[1] * ctx->cfg.res[2];
  TRY(ensure_stage(ctx, sizeof(double) * (size_t)nn * 4));
  CK(cudaMemcpyAsync(ctx->stage, grid_mv, sizeof(double) * 3 * nn, cudaMemcpyHostToDevice, ctx->stream));
  const double* dm_ = nullptr;
  if (target == 0) {
    if (!grid_m) return fail(ctx, MPM_EINVAL, "upload_grid: momentum target needs grid_m");
    CK(cudaMemcpyAsync(ctx->stage + 3 * nn, grid_m, sizeof(double) * nn, cudaMemcpyHostToDevice, ctx->stream));
    dm_ = ctx->stage + 3 * nn;
  }
  Params p = make_params(ctx);
  if (target == 0) {
    upload_grid_kernel<<<blocks_for(nn, 256), 256, 0, ctx->stream>>>(p, ctx->gm, ctx->stage, dm_);
    LAUNCHED();
    ctx->grid_phase = 0;
  } else {
    // velocities for g2p: keep masses, overwrite gv
    upload_grid_kernel<<<blocks_for(nn, 256), 256, 0, ctx->stream>>>(p, ctx->gv, ctx->stage, nullptr);
    LAUNCHED();
    ctx->grid_phase = 2;
  }
  ctx->grid_dirty = 2;
  CK(cudaStreamSynchronize(ctx->stream));
  return 0;
}

int mpm_download_grid(mpm_ctx* ctx, double* grid_mv, double* grid_m) {
  if (!ctx || !grid_mv) return fail(ctx, MPM_EINVAL, "download_grid: bad arguments");
  CK(cudaSetDevice(ctx->dev));
  long long nn = (long long)ctx->cfg.res[0] * ctx->cfg.res[1] * ctx->cfg.res[2];
  TRY(ensure_stage(ctx, sizeof(double) * (size_t)nn * 4));
  Params p = make_params(ctx);
  download_grid_kernel<<<blocks_for(nn, 256), 256, 0, ctx->stream>>>(p, ctx->grid_phase, ctx->stage,
                                                                      grid_m ? ctx->stage + 3 * nn : nullptr);
  LAUNCHED();
  CK(cudaMemcpyAsync(grid_mv, ctx->stage, sizeof(double) * 3 * nn, cudaMemcpyDeviceToHost, ctx->stream));
  if (grid_m) CK(cudaMemcpyAsync(grid_m, ctx->stage + 3 * nn, sizeof(double) * nn, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return 0;
}

int mpm_set_colliders(mpm_ctx* ctx, int count, const int32_t* kind, const double* half, const double* rotation,
                      const double* translation, const double* linear_velocity, const double* angular_velocity,
                      const double* friction, const int32_t* mode, const double* sdf_values, int64_t sdf_len,
                      const int64_t* sdf_offset, const int32_t* sdf_resolution, const double* sdf_bounds_min,
                      const double* sdf_extent) {
  if (!ctx || count < 0) return fail(ctx, MPM_EINVAL, "set_colliders: bad count");
  {
    const int per = ctx->cfg.colliders_per_env > 0 ? ctx->cfg.colliders_per_env : count;
    if (per > MAX_COLLIDERS) return fail(ctx, MPM_EINVAL, "set_colliders: too many colliders per environment");
    if (ctx->cfg.colliders_per_env > 0) {
      int tiles = 1;
      for (int a = 0; a < 3; ++a) tiles *= ctx->cfg.env_tiles[a] > 1 ? ctx->cfg.env_tiles[a] : 1;
      if (count != per * tiles) return fail(ctx, MPM_EINVAL, "set_colliders: count != colliders_per_env x env tiles");
    }
  }
  CK(cudaSetDevice(ctx->dev));
  invalidate_graphs(ctx);
  ctx->ncol = count;
  ctx->geo_h.assign(std::max(count, 1), ColliderGeo{});
  std::vector<ColliderPose> pose(std::max(count, 1));
  for (int i = 0; i < count; ++i) {
    ColliderGeo& g = ctx->geo_h[i];
    g.kind = kind[i];
    if (g.kind != 0 && g.kind != 1) return fail(ctx, MPM_EINVAL, "unknown collider kind");
    for (int a = 0; a < 3; ++a) {
      g.half[a] = half[3 * i + a];
      g.sdf_res[a] = sdf_resolution ? sdf_resolution[3 * i + a] : 0;
      g.sdf_bmin[a] = sdf_bounds_min ? sdf_bounds_min[3 * i + a] : 0.0;
    }
    g.fric = friction[i];
    g.mode = mode[i];
    g.sdf_off = sdf_offset ? sdf_offset[i] : -1;
    g.sdf_ext = sdf_extent ? sdf_extent[i] : 1.0;
    g.far_r = (float)(std::sqrt(g.half[0] * g.half[0] + g.half[1] * g.half[1] + g.half[2] * g.half[2]) * (1.0 + 1e-6));
    g.far_min = -1.0f;
    if (g.kind == 1) {
      if (!sdf_values || g.sdf_off < 0 || g.sdf_res[0] < 2 || g.sdf_res[1] < 2 || g.sdf_res[2] < 2 ||
          g.sdf_off + (long long)g.sdf_res[0] * g.sdf_res[1] * g.sdf_res[2] > sdf_len)
        return fail(ctx, MPM_EINVAL, "baked collider: SDF lattice out of range");
      // smallest value on the outer layer (x-fastest lattice), in metres, shaded down for fp32
      const int rx = g.sdf_res[0], ry = g.sdf_res[1], rz = g.sdf_res[2];
      double mn = 1e300;
      for (int z = 0; z < rz; ++z)
        for (int y = 0; y < ry; ++y)
          for (int x = 0; x < rx; ++x) {
            if (x != 0 && x != rx - 1 && y != 0 && y != ry - 1 && z != 0 && z != rz - 1) continue;
            mn = std::min(mn, sdf_values[g.sdf_off + x + (long long)rx * (y + (long long)ry * z)]);
          }
      g.far_min = (float)(mn * g.sdf_ext * (mn > 0 ? 0.999999 : 1.000001));
    }
    ColliderPose& q = pose[i];
    for (int a = 0; a < 9; ++a) q.R[a] = rotation[9 * i + a];
    for (int a = 0; a < 3; ++a) {
      q.T[a] = translation[3 * i + a];
      q.lv[a] = linear_velocity[3 * i + a];
      q.av[a] = angular_velocity[3 * i + a];
    }
    q.mode = mode[i];
  }
  TRY(dalloc(ctx, &ctx->geo, (size_t)std::max(count, 1)));
  CK(cudaMemcpyAsync(ctx->geo, ctx->geo_h.data(), sizeof(ColliderGeo) * std::max(count, 1), cudaMemcpyHostToDevice,
                     ctx->stream));
  if (ctx->pose_cap < 1 || ctx->pose_width < std::max(count, 1)) {
    TRY(dalloc(ctx, &ctx->pose, (size_t)std::max(count, MAX_COLLIDERS)));
    ctx->pose_cap = 1;
    ctx->pose_width = std::max(count, MAX_COLLIDERS);
  }
  CK(cudaMemcpyAsync(ctx->pose, pose.data(), sizeof(ColliderPose) * std::max(count, 1), cudaMemcpyHostToDevice,
                     ctx->stream));
  ctx->pose_rows = 1;
  if (sdf_values && sdf_len > 0) {
    TRY(dalloc(ctx, &ctx->sdf, (size_t)sdf_len));
    CK(cudaMemcpyAsync(ctx->sdf, sdf_values, sizeof(double) * sdf_len, cudaMemcpyHostToDevice, ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return 0;
}

int mpm_set_pose_table(mpm_ctx* ctx, int nsub, const double* rotation, const double* translation,
                       const double* linear_velocity, const double* angular_velocity, const int32_t* mode) {
  if (!ctx || nsub <= 0 || !rotation || !translation || !linear_velocity || !angular_velocity)
    return fail(ctx, MPM_EINVAL, "set_pose_table: bad arguments");
  if (ctx->ncol <= 0) return 0;
  CK(cudaSetDevice(ctx->dev));
  int k = ctx->ncol;
  std::vector<ColliderPose> rows((size_t)nsub * k);
  for (int s = 0; s < nsub; ++s)
    for (int i = 0; i < k; ++i) {
      size_t r = (size_t)s * k + i;
      ColliderPose& q = rows[r];
      for (int a = 0; a < 9; ++a) q.R[a] = rotation[9 * r + a];
      for (int a = 0; a < 3; ++a) {
        q.T[a] = translation[3 * r + a];
        q.lv[a] = linear_velocity[3 * r + a];
        q.av[a] = angular_velocity[3 * r + a];
      }
      q.mode = mode ? mode[r] : ctx->geo_h[i].mode;
    }
  if (ctx->pose_cap < nsub || ctx->pose_width < k) {
    invalidate_graphs(ctx);
    const int width = std::max(k, MAX_COLLIDERS);
    TRY(dalloc(ctx, &ctx->pose, (size_t)nsub * width));
    ctx->pose_cap = nsub;
    ctx->pose_width = width;
  }
  CK(cudaMemcpyAsync(ctx->pose, rows.data(), sizeof(ColliderPose) * rows.size(), cudaMemcpyHostToDevice, ctx->stream));
  ctx->pose_rows = nsub;
  CK(cudaStreamSynchronize(ctx->stream));
  return 0;
}

int mpm_p2g(mpm_ctx* ctx, int64_t* inverted) {
  if (ctx) ctx->bins_age = -1;  // particle order / positions may change: the next frame re-bins
  if (!ctx) return MPM_EINVAL;
  TRY(need_particles(ctx));
  CK(cudaSetDevice(ctx->dev));
  CK(cudaMemsetAsync(ctx->inverted, 0, sizeof(unsigned long long), ctx->stream));
  if (empty_state(ctx)) {
    TRY(zero_grid(ctx));
    ctx->grid_phase = 0;
    return read_inverted(ctx, inverted);
  }
  if (ctx->cfg.deterministic) {
    TRY(det_p2g(ctx));
  } else {
    ctx->grid_dirty = 2;  // stage p2g overwrites the whole grid (p2g_reduce writes every node)
    TRY(ensure_gm_clean(ctx));
    TRY(rebin(ctx));
    TRY(launch_fused(ctx, false));
    ctx->grid_dirty = 2;
  }
  ctx->grid_phase = 0;
  return read_inverted(ctx, inverted);
}

int mpm_grid_update(mpm_ctx* ctx, int use_colliders) {
  if (ctx) ctx->bins_age = -1;  // particle order / positions may change: the next frame re-bins
  if (!ctx) return MPM_EINVAL;
  CK(cudaSetDevice(ctx->dev));
  if (ctx->grid_phase == 2) return fail(ctx, MPM_ESTATE, "grid holds velocities; run p2g first");
  TRY(launch_grid_op(ctx, true, use_colliders != 0, 0, false));
  ctx->grid_phase = 1;
  ctx->grid_dirty = 2;
  CK(cudaStreamSynchronize(ctx->stream));
  return 0;
}

int mpm_g2p(mpm_ctx* ctx) {
  if (ctx) ctx->bins_age = -1;  // particle order / positions may change: the next frame re-bins
  if (!ctx) return MPM_EINVAL;
  TRY(need_particles(ctx, false));  // g2p_advect (core.py:254-258) takes no materials
  if (empty_state(ctx)) return 0;
  CK(cudaSetDevice(ctx->dev));
  TRY(launch_g2p(ctx));
  CK(cudaStreamSynchronize(ctx->stream));
  return 0;
}

int mpm_substeps(mpm_ctx* ctx, int nsub, int use_colliders, int64_t* inverted, double* device_ms) {
  if (!ctx || nsub <= 0) return fail(ctx, MPM_EINVAL, "substeps: nsub must be >= 1");
  TRY(need_particles(ctx));
  CK(cudaSetDevice(ctx->dev));
  if (empty_state(ctx)) {
    // no particles: every substep's P2G leaves the grid empty and the grid op
    // keeps massless nodes as they are (kernels.py:364-365)
    TRY(zero_grid(ctx));
    ctx->grid_phase = 1;
    ctx->bins_age = -1;
    if (inverted) *inverted = 0;
    if (device_ms) *device_ms = 0.0;
    CK(cudaStreamSynchronize(ctx->stream));
    return 0;
  }
  bool col = use_colliders && ctx->ncol > 0 && ctx->cfg.theta >= 0.0;
  // cross-frame re-binning (one stretch per frame only)
  const bool skip = !ctx->cfg.deterministic && ctx->rebin_frames > 1 && ctx->cfg.rebin_interval >= nsub &&
                    ctx->bins_age >= 0 && ctx->bins_age < ctx->rebin_frames;
  CK(cudaEventRecord(ctx->ev0, ctx->stream));
  CK(cudaMemsetAsync(ctx->inverted, 0, sizeof(unsigned long long), ctx->stream));
  if (ctx->cfg.deterministic) {
    for (int s = 0; s < nsub; ++s) {
      TRY(det_p2g(ctx));
      TRY(launch_grid_op(ctx, true, col, s, false));
      TRY(launch_g2p(ctx));
    }
    ctx->grid_dirty = 2;
  } else if (!ctx->graphs_on) {
    TRY(run_fast_sequence(ctx, nsub, col, skip));
  } else {
    const int border = ctx->item_bounds == ctx->bounds_a ? 0 : 1;
    const int timing = ctx->timing ? 1 : 0;
    // the substeps' pose pointers are baked into the graph: a table with a
    // different row count (step() with / without pose_fn) needs its own graph
    const int prows = col ? std::max(ctx->pose_rows, 1) : 0;
    mpm_ctx::GraphEntry* hit = nullptr;
    for (auto& g : ctx->graphs)
      if (g.nsub == nsub && g.col == (int)col && g.prows == prows && g.skip == (int)skip && g.cur == ctx->cur &&
          g.border == border &&
          g.dirty == ctx->grid_dirty && g.timing == timing && g.n == ctx->n && g.cclean == ctx->counters_clean &&
          g.bclean == ctx->bounds_out_clean)
        hit = &g;
    if (!hit) {
      mpm_ctx::GraphEntry e{};
      e.nsub = nsub;
      e.col = (int)col;
      e.prows = prows;
      e.skip = (int)skip;
      e.cur = ctx->cur;
      e.border = border;
      e.dirty = ctx->grid_dirty;
      e.timing = timing;
      e.n = ctx->n;
      e.cclean = ctx->counters_clean;
      e.bclean = ctx->bounds_out_clean;
      const size_t marks0 = ctx->marks.size();
      const long long launches0 = ctx->launches;
      CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
      const int rc = run_fast_sequence(ctx, nsub, col, skip);
      cudaGraph_t graph = nullptr;
      const cudaError_t ce = cudaStreamEndCapture(ctx->stream, &graph);
      if (rc || ce != cudaSuccess) {
        if (graph) cudaGraphDestroy(graph);
        cudaGetLastError();
        if (!rc) ctx->err = std::string("graph capture: ") + cudaGetErrorString(ce);
        return rc ? rc : MPM_ECUDA;
      }
      const cudaError_t ie = cudaGraphInstantiate(&e.exec, graph, 0);
      cudaGraphDestroy(graph);
      if (ie != cudaSuccess) {
        ctx->err = std::string("graph instantiate: ") + cudaGetErrorString(ie);
        return MPM_ECUDA;
      }
      for (size_t i = marks0; i < ctx->marks.size(); ++i) {
        e.marks.push_back(ctx->marks[i]);
        e.marks.back().graph_owned = true;
      }
      ctx->marks.resize(marks0);
      e.kernels = ctx->launches - launches0;
      ctx->launches = launches0;
      e.end_cur = ctx->cur;
      e.end_border = ctx->item_bounds == ctx->bounds_a ? 0 : 1;
      e.end_dirty = ctx->grid_dirty;
      e.end_cclean = ctx->counters_clean;
      e.end_bclean = ctx->bounds_out_clean;
      // the capture advanced the host state as a real run would; restore the
      // start state so the replay below applies the same transition
      ctx->cur = e.cur;
      if ((ctx->item_bounds == ctx->bounds_a ? 0 : 1) != e.border) std::swap(ctx->item_bounds, ctx->item_bounds2);
      ctx->grid_dirty = e.dirty;
      ctx->counters_clean = e.cclean;
      ctx->bounds_out_clean = e.bclean;
      ctx->graphs.push_back(std::move(e));
      hit = &ctx->graphs.back();
    }
    CK(cudaGraphLaunch(hit->exec, ctx->stream));
    ctx->launches += hit->kernels;
    ctx->cur = hit->end_cur;
    if ((ctx->item_bounds == ctx->bounds_a ? 0 : 1) != hit->end_border) std::swap(ctx->item_bounds, ctx->item_bounds2);
    ctx->grid_dirty = hit->end_dirty;
    ctx->counters_clean = hit->end_cclean;
    ctx->bounds_out_clean = hit->end_bclean;
    if (timing)
      for (auto& mk : hit->marks) ctx->marks.push_back(mk);
  }
  ctx->grid_phase = 1;
  if (ctx->cfg.deterministic || ctx->cfg.rebin_interval < nsub)
    ctx->bins_age = -1;
  else
    ctx->bins_age = skip ? ctx->bins_age + 1 : 1;
  CK(cudaEventRecord(ctx->ev1, ctx->stream));
  TRY(read_inverted(ctx, inverted));
  if (device_ms) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
    *device_ms = ms;
  }
  return 0;
}

int mpm_set_option(mpm_ctx* ctx, const char* key, int value) {
  if (!ctx || !key) return MPM_EINVAL;
  CK(cudaSetDevice(ctx->dev));
  if (!strcmp(key, "graphs")) {
    invalidate_graphs(ctx);
    ctx->graphs_on = value != 0;
  } else if (!strcmp(key, "split")) {
    invalidate_graphs(ctx);
    ctx->split_mode = value != 0;
  } else if (!strcmp(key, "mega")) {
    if (value && !ctx->mega_coop) return fail(ctx, MPM_EINVAL, "mega: device has no cooperative launch");
    invalidate_graphs(ctx);
    ctx->mega_on = value != 0;
  } else if (!strcmp(key, "pdl")) {
    invalidate_graphs(ctx);
    ctx->pdl_on = value != 0;
  } else if (!strcmp(key, "rebin_frames")) {
    if (value < 1) return fail(ctx, MPM_EINVAL, "rebin_frames: >= 1");
    ctx->rebin_frames = value;
    ctx->bins_age = -1;
  } else if (!strcmp(key, "host_xfer")) {
    ctx->host_xfer = value != 0;
  } else if (!strcmp(key, "gridop_simple")) {
    invalidate_graphs(ctx);
    ctx->gridop_simple = value != 0;
  } else if (!strcmp(key, "fx_shift")) {
    if (value < 0 || value > 8) return fail(ctx, MPM_EINVAL, "fx_shift: 0..8");
    invalidate_graphs(ctx);
    ctx->fx_shift = value;
  } else {
    return fail(ctx, MPM_EINVAL, std::string("unknown option ") + key);
  }
  return 0;
}

// Cumulative device statistics: 0 = particles the fixed-point overflow guard
// routed to the float scatter path.
int mpm_get_stat(mpm_ctx* ctx, int index, int64_t* out) {
  if (!ctx || index < 0 || index >= 8 || !out) return MPM_EINVAL;
  CK(cudaSetDevice(ctx->dev));
  unsigned long long h = 0;
  CK(cudaMemcpyAsync(&h, ctx->stats + index, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  *out = (int64_t)h;
  return 0;
}

int mpm_collision_field(mpm_ctx* ctx, double theta, double* dist, int32_t* obj) {
  if (!ctx || !dist || !obj) return fail(ctx, MPM_EINVAL, "collision_field: bad arguments");
  CK(cudaSetDevice(ctx->dev));
  long long nn = (long long)ctx->cfg.res[0] * ctx->cfg.res[1] * ctx->cfg.res[2];
  TRY(ensure_stage(ctx, sizeof(double) * (size_t)nn * 2));
  Params p = make_params(ctx);
  Colliders cs = make_colliders(ctx, 0, true);
  cs.theta = theta;
  collision_field_kernel<<<blocks_for(nn, 256), 256, 0, ctx->stream>>>(p, cs, 2.0 * theta, ctx->stage,
                                                                        (int*)(ctx->stage + nn));
  LAUNCHED();
  CK(cudaMemcpyAsync(dist, ctx->stage, sizeof(double) * nn, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(obj, ctx->stage + nn, sizeof(int32_t) * nn, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return 0;
}

int mpm_has_nan(mpm_ctx* ctx, int* flag) {
  if (!ctx || !flag) return MPM_EINVAL;
  CK(cudaSetDevice(ctx->dev));
  TRY(compact_if_needed(ctx));
  *flag = 0;
  if (ctx->n <= 0) return 0;
  CK(cudaMemsetAsync(ctx->flag, 0, sizeof(int), ctx->stream));
  Params p = make_params(ctx);
  has_nan_kernel<<<blocks_for(ctx->n, 256), 256, 0, ctx->stream>>>(p, ctx->flag);
  LAUNCHED();
  CK(cudaMemcpyAsync(flag, ctx->flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return 0;
}

int mpm_metrics(mpm_ctx* ctx, const double* x0, double dx, double* out) {
  if (!ctx || !out) return MPM_EINVAL;
  CK(cudaSetDevice(ctx->dev));
  TRY(compact_if_needed(ctx));
  for (int k = 0; k < 5; ++k) out[k] = 0.0;
  out[4] = (double)ctx->n;
  if (ctx->n <= 0) return 0;
  if (x0) {
    if (ctx->x0_n != ctx->n) {
      TRY(dalloc(ctx, &ctx->x0, (size_t)ctx->n * 3));
      ctx->x0_n = ctx->n;
    }
    CK(cudaMemcpyAsync(ctx->x0, x0, sizeof(double) * 3 * ctx->n, cudaMemcpyHostToDevice, ctx->stream));
  } else if (ctx->x0_n != ctx->n) {
    return fail(ctx, MPM_ESTATE, "metrics: no initial positions uploaded for this particle count");
  }
  const int blocks = ctx->sms * 4;
  std::vector<double> part((size_t)blocks * 4);
  TRY(ensure_stage(ctx, sizeof(double) * part.size()));
  Params p = make_params(ctx);
  metrics_kernel<<<blocks, METRICS_THREADS, 0, ctx->stream>>>(p, ctx->x0, dx, ctx->stage);
  LAUNCHED();
  CK(cudaMemcpyAsync(part.data(), ctx->stage, sizeof(double) * part.size(), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  double r[4] = {0.0, 0.0, 0.0, 0.0};
  for (int b = 0; b < blocks; ++b) {
    r[0] += part[4 * b];
    r[1] += part[4 * b + 1];
    r[2] += part[4 * b + 2];
    r[3] = std::max(r[3], part[4 * b + 3]);
  }
  const double n = (double)ctx->n;
  out[0] = r[0] / n;
  out[1] = r[1] / n;
  out[2] = r[2] / n;
  out[3] = r[3];
  return 0;
}

namespace {
int splat_run(mpm_ctx* ctx, int dev, cudaStream_t st, const double* positions, const double* masses, long long n,
              const int32_t* res, double field_dx, double* out, double* keep = nullptr) {
  const long long nn = (long long)res[0] * res[1] * res[2];
  double* d_out = keep;
  double* d_pos = nullptr;
  if (!d_out && cudaMallocAsync((void**)&d_out, sizeof(double) * std::max(nn, 1LL), st) != cudaSuccess) return MPM_ENOMEM;
  int rc = 0;
  if (cudaMemsetAsync(d_out, 0, sizeof(double) * nn, st) != cudaSuccess) rc = MPM_ECUDA;
  if (!rc && n > 0) {
    Params p{};
    if (ctx) p = make_params(ctx);
    const double* dp = nullptr;
    const double* dm = nullptr;
    if (positions) {
      if (cudaMallocAsync((void**)&d_pos, sizeof(double) * 4 * n, st) != cudaSuccess) rc = MPM_ENOMEM;
      if (!rc && (cudaMemcpyAsync(d_pos, positions, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, st) != cudaSuccess ||
                  cudaMemcpyAsync(d_pos + 3 * n, masses, sizeof(double) * n, cudaMemcpyHostToDevice, st) != cudaSuccess))
        rc = MPM_ECUDA;
      dp = d_pos;
      dm = d_pos + 3 * n;
    }
    if (!rc) {
      splat_kernel<<<blocks_for(n, 256), 256, 0, st>>>(p, dp, dm, n, res[0], res[1], res[2], 1.0 / field_dx, d_out);
      if (cudaGetLastError() != cudaSuccess) rc = MPM_ECUDA;
      if (ctx) ctx->launches++;
    }
  }
  if (!rc && nn > 0) {
    scale_kernel<<<blocks_for(nn, 256), 256, 0, st>>>(d_out, nn, 1.0 / (field_dx * field_dx * field_dx));
    if (cudaGetLastError() != cudaSuccess) rc = MPM_ECUDA;
    if (ctx) ctx->launches++;
  }
  if (!rc && out && cudaMemcpyAsync(out, d_out, sizeof(double) * nn, cudaMemcpyDeviceToHost, st) != cudaSuccess)
    rc = MPM_ECUDA;
  if (d_pos) cudaFreeAsync(d_pos, st);
  if (!keep) cudaFreeAsync(d_out, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) rc = MPM_ECUDA;
  (void)dev;
  return rc;
}
}  // namespace

int mpm_splat_density(mpm_ctx* ctx, const double* positions, const double* masses, int64_t n, const int32_t* res,
                      double field_dx, double* out) {
  if (!ctx || !res || !(field_dx > 0.0) || res[0] < 1 || res[1] < 1 || res[2] < 1) return MPM_EINVAL;
  if (positions && (!masses || n < 0)) return MPM_EINVAL;
  CK(cudaSetDevice(ctx->dev));
  const long long cnt = positions ? n : ctx->n;
  const long long nn = (long long)res[0] * res[1] * res[2];
  if (ctx->field_n < nn) {
    TRY(dalloc(ctx, &ctx->field, (size_t)nn));
    ctx->field_n = nn;
  }
  const int rc = splat_run(ctx, ctx->dev, ctx->stream, positions, masses, cnt, res, field_dx, out, ctx->field);
  if (rc) return fail(ctx, rc, "splat_density failed");
  for (int a = 0; a < 3; ++a) ctx->field_res[a] = res[a];
  ctx->field_dx = field_dx;
  return 0;
}

int mpm_marching_cubes(mpm_ctx* ctx, const double* values, const int32_t* res, double dx, double iso, int64_t* nverts,
                       int64_t* ntris) {
  if (!ctx || !nverts || !ntris) return MPM_EINVAL;
  CK(cudaSetDevice(ctx->dev));
  int r[3];
  double h = dx;
  if (values) {
    if (!res || res[0] < 1 || res[1] < 1 || res[2] < 1 || !(dx > 0.0)) return fail(ctx, MPM_EINVAL, "marching_cubes: bad field");
    const long long nn = (long long)res[0] * res[1] * res[2];
    if (ctx->field_n < nn) {
      TRY(dalloc(ctx, &ctx->field, (size_t)nn));
      ctx->field_n = nn;
    }
    CK(cudaMemcpyAsync(ctx->field, values, sizeof(double) * nn, cudaMemcpyHostToDevice, ctx->stream));
    for (int a = 0; a < 3; ++a) r[a] = res[a];
  } else {
    if (ctx->field_res[0] < 1) return fail(ctx, MPM_ESTATE, "marching_cubes: no device field (splat first)");
    for (int a = 0; a < 3; ++a) r[a] = ctx->field_res[a];
    h = ctx->field_dx;
  }
  *nverts = 0;
  *ntris = 0;
  ctx->mesh_nv = ctx->mesh_nt = 0;
  if (r[0] < 2 || r[1] < 2 || r[2] < 2) return 0;
  const long long nn = (long long)r[0] * r[1] * r[2];
  const long long ne = 3 * nn, nc = (long long)(r[0] - 1) * (r[1] - 1) * (r[2] - 1);
  if (ne + 1 > INT32_MAX) return fail(ctx, MPM_EINVAL, "marching_cubes: field too large");
  if (ctx->mc_cap < ne) {
    TRY(dalloc(ctx, &ctx->mc_flag, (size_t)ne));
    TRY(dalloc(ctx, &ctx->mc_vid, (size_t)ne));
    TRY(dalloc(ctx, &ctx->mc_cnt, (size_t)ne));
    TRY(dalloc(ctx, &ctx->mc_off, (size_t)ne));
    ctx->mc_cap = ne;
  }
  TRY(ensure_scan(ctx, ne));
  mc_edge_flag_kernel<<<blocks_for(ne, 256), 256, 0, ctx->stream>>>(ctx->field, r[0], r[1], r[2], iso, ctx->mc_flag);
  LAUNCHED();
  TRY(scan_exclusive(ctx, ctx->mc_flag, ctx->mc_vid, ne));
  mc_cell_count_kernel<<<blocks_for(nc, 256), 256, 0, ctx->stream>>>(ctx->field, r[0], r[1], r[2], iso, ctx->mc_cnt);
  LAUNCHED();
  TRY(scan_exclusive(ctx, ctx->mc_cnt, ctx->mc_off, nc));
  int tail[4];
  CK(cudaMemcpyAsync(tail, ctx->mc_vid + ne - 1, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(tail + 1, ctx->mc_flag + ne - 1, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(tail + 2, ctx->mc_off + nc - 1, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(tail + 3, ctx->mc_cnt + nc - 1, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  const long long nv = (long long)tail[0] + tail[1], nt = (long long)tail[2] + tail[3];
  if (ctx->mesh_vcap < nv) {
    TRY(dalloc(ctx, &ctx->mesh_v, (size_t)std::max(nv, 1LL) * 6));
    ctx->mesh_vcap = nv;
  }
  if (ctx->mesh_tcap < nt) {
    TRY(dalloc(ctx, &ctx->mesh_t, (size_t)std::max(nt, 1LL) * 3));
    ctx->mesh_tcap = nt;
  }
  if (nv > 0) {
    mc_edge_vertex_kernel<<<blocks_for(ne, 256), 256, 0, ctx->stream>>>(ctx->field, r[0], r[1], r[2], iso, h, ctx->mc_flag,
                                                                       ctx->mc_vid, ctx->mesh_v, ctx->mesh_v + 3 * nv);
    LAUNCHED();
  }
  if (nt > 0) {
    mc_cell_emit_kernel<<<blocks_for(nc, 256), 256, 0, ctx->stream>>>(ctx->field, r[0], r[1], r[2], iso, ctx->mc_cnt,
                                                                     ctx->mc_off, ctx->mc_vid, ctx->mesh_t);
    LAUNCHED();
  }
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->mesh_nv = nv;
  ctx->mesh_nt = nt;
  *nverts = nv;
  *ntris = nt;
  return 0;
}

int mpm_mesh_fetch(mpm_ctx* ctx, double* verts, int32_t* tris, double* normals) {
  if (!ctx) return MPM_EINVAL;
  CK(cudaSetDevice(ctx->dev));
  const long long nv = ctx->mesh_nv, nt = ctx->mesh_nt;
  if (verts && nv) CK(cudaMemcpyAsync(verts, ctx->mesh_v, sizeof(double) * 3 * nv, cudaMemcpyDeviceToHost, ctx->stream));
  if (normals && nv)
    CK(cudaMemcpyAsync(normals, ctx->mesh_v + 3 * nv, sizeof(double) * 3 * nv, cudaMemcpyDeviceToHost, ctx->stream));
  if (tris && nt) CK(cudaMemcpyAsync(tris, ctx->mesh_t, sizeof(int) * 3 * nt, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return 0;
}

int mpm_mesh_encode(mpm_ctx* ctx, const double* extent, uint8_t* out, int64_t cap, int64_t* len) {
  if (!ctx || !extent || !len) return MPM_EINVAL;
  CK(cudaSetDevice(ctx->dev));
  const long long nv = ctx->mesh_nv, nt = ctx->mesh_nt;
  const long long bytes = 32 * nv + 12 * nt;
  *len = bytes;
  if (!out) return 0;  // size query
  if (cap < bytes) return fail(ctx, MPM_EINVAL, "mesh_encode: output buffer too small");
  if (!bytes) return 0;
  if (ctx->enc_cap < bytes) {
    TRY(dalloc(ctx, &ctx->enc, (size_t)bytes));
    ctx->enc_cap = bytes;
  }
  float* ov = reinterpret_cast<float*>(ctx->enc);
  float* on = ov + 3 * nv;
  float* ouv = on + 3 * nv;
  unsigned* ot = reinterpret_cast<unsigned*>(ouv + 2 * nv);
  const long long work = std::max(3 * nv, 3 * nt);
  mesh_encode_kernel<<<blocks_for(work, 256), 256, 0, ctx->stream>>>(ctx->mesh_v, ctx->mesh_v + 3 * nv, nv, ctx->mesh_t,
                                                                     nt, extent[0], extent[2], ov, on, ouv, ot);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, ctx->enc, (size_t)bytes, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return 0;
}

int mpm_splat_density_host(int device, const double* positions, const double* masses, int64_t n, const int32_t* res,
                           double field_dx, double* out) {
  if (!res || !out || !(field_dx > 0.0) || res[0] < 1 || res[1] < 1 || res[2] < 1 || n < 0) return MPM_EINVAL;
  if (n > 0 && (!positions || !masses)) return MPM_EINVAL;
  if (cudaSetDevice(device) != cudaSuccess) return MPM_ECUDA;
  cudaStream_t st;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return MPM_ECUDA;
  const int rc = splat_run(nullptr, device, st, positions, masses, n, res, field_dx, out);
  cudaStreamDestroy(st);
  return rc;
}

int mpm_set_timing(mpm_ctx* ctx, int enable) {
  if (!ctx) return MPM_EINVAL;
  CK(cudaSetDevice(ctx->dev));
  resolve_marks(ctx);
  ctx->timing = enable != 0;
  for (double& a : ctx->acc) a = 0.0;
  return 0;
}

int mpm_get_timing(mpm_ctx* ctx, double* out) {
  if (!ctx || !out) return MPM_EINVAL;
  CK(cudaSetDevice(ctx->dev));
  resolve_marks(ctx);
  for (int i = 0; i < 8; ++i) out[i] = ctx->acc[i];
  int h[2] = {0, 0};
  CK(cudaMemcpyAsync(h, ctx->counters, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  out[8] = h[0];
  out[9] = h[1];
  out[10] = ctx->acc[8];
  out[11] = ctx->acc[9];
  out[12] = ctx->acc[10];
  out[13] = ctx->acc[11];
  out[14] = ctx->acc[12];
  out[15] = ctx->acc[13];
  for (double& a : ctx->acc) a = 0.0;
  return 0;
}

// ---- slab decomposition (BASELINE config 5) ----------------------------

int mpm_set_slab(mpm_ctx* ctx, const int* global_res, const int* offset, int ghost_bricks) {
  if (ctx) ctx->bins_age = -1;  // particle order / positions may change: the next frame re-bins
  if (!ctx || !global_res || !offset || ghost_bricks < 1) return fail(ctx, MPM_EINVAL, "set_slab: bad arguments");
  CK(cudaSetDevice(ctx->dev));
  for (int a = 0; a < 3; ++a) {
    if (offset[a] % 4 != 0) return fail(ctx, MPM_EINVAL, "set_slab: window offset must be a multiple of 4 nodes");
    if (offset[a] < 0 || offset[a] + ctx->cfg.res[a] > global_res[a] + 4 * ghost_bricks)
      return fail(ctx, MPM_EINVAL, "set_slab: window outside the global grid");
  }
  if (ctx->cfg.res[1] != global_res[1] || ctx->cfg.res[2] != global_res[2] || offset[1] || offset[2])
    return fail(ctx, MPM_EINVAL, "set_slab: slabs split x only");
  invalidate_graphs(ctx);
  for (int a = 0; a < 3; ++a) {
    ctx->goff[a] = offset[a];
    ctx->gres[a] = global_res[a];
  }
  ctx->ghost_bricks = ghost_bricks;
  const long long cap = (long long)ghost_bricks * ((ctx->cfg.res[1] + 3) / 4) * ((ctx->cfg.res[2] + 3) / 4);
  if (cap > ctx->h_cap) {
    for (int s = 0; s < 2; ++s) {
      TRY(dalloc(ctx, &ctx->h_send_ids[s], (size_t)cap + 1));
      TRY(dalloc(ctx, &ctx->h_send_data[s], (size_t)cap * 64));
      TRY(dalloc(ctx, &ctx->h_recv_ids[s], (size_t)cap + 1));
      TRY(dalloc(ctx, &ctx->h_recv_data[s], (size_t)cap * 64));
      TRY(dalloc(ctx, &ctx->h_local_ids[s], (size_t)cap));
    }
    ctx->h_cap = cap;
  }
  return 0;
}

// ---- peer-memory halo exchange --------------------------------------------
constexpr size_t IPC_BLOB = 4 * sizeof(cudaIpcMemHandle_t) + 2 * sizeof(cudaIpcEventHandle_t);

int mpm_ipc_export(mpm_ctx* ctx, int side, void* out) {
  if (!ctx || side < 0 || side > 1 || !out) return MPM_EINVAL;
  if (!ctx->h_cap) return fail(ctx, MPM_ESTATE, "ipc_export: call mpm_set_slab first");
  CK(cudaSetDevice(ctx->dev));
  if (!ctx->ipc_vrecv[side]) {
    TRY(dalloc(ctx, &ctx->ipc_vrecv[side], (size_t)(ctx->h_cap + 1) * 64));
    TRY(dalloc(ctx, &ctx->ipc_cnt[side], 8));
    CK(cudaMemset(ctx->ipc_cnt[side], 0, 8 * sizeof(int)));
    CK(cudaEventCreateWithFlags(&ctx->ipc_free[side], cudaEventInterprocess | cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ctx->ipc_ready[side], cudaEventInterprocess | cudaEventDisableTiming));
  }
  char* o = static_cast<char*>(out);
  cudaIpcMemHandle_t mh;
  void* mems[4] = {ctx->h_recv_ids[side], ctx->h_recv_data[side], ctx->ipc_cnt[side], ctx->ipc_vrecv[side]};
  for (int k = 0; k < 4; ++k) {
    CK(cudaIpcGetMemHandle(&mh, mems[k]));
    memcpy(o + k * sizeof(mh), &mh, sizeof(mh));
  }
  cudaIpcEventHandle_t eh;
  CK(cudaIpcGetEventHandle(&eh, ctx->ipc_free[side]));
  memcpy(o + 4 * sizeof(mh), &eh, sizeof(eh));
  CK(cudaIpcGetEventHandle(&eh, ctx->ipc_ready[side]));
  memcpy(o + 4 * sizeof(mh) + sizeof(eh), &eh, sizeof(eh));
  return 0;
}

int mpm_ipc_import(mpm_ctx* ctx, int side, const void* peer) {
  if (!ctx || side < 0 || side > 1 || !peer) return MPM_EINVAL;
  CK(cudaSetDevice(ctx->dev));
  const char* o = static_cast<const char*>(peer);
  cudaIpcMemHandle_t mh[4];
  for (int k = 0; k < 4; ++k) memcpy(&mh[k], o + k * sizeof(cudaIpcMemHandle_t), sizeof(cudaIpcMemHandle_t));
  void* q[4];
  for (int k = 0; k < 4; ++k) CK(cudaIpcOpenMemHandle(&q[k], mh[k], cudaIpcMemLazyEnablePeerAccess));
  ctx->peer_ids[side] = static_cast<int*>(q[0]);
  ctx->peer_data[side] = static_cast<float4*>(q[1]);
  ctx->peer_cnt[side] = static_cast<int*>(q[2]);
  ctx->peer_vdata[side] = static_cast<float4*>(q[3]);
  cudaIpcEventHandle_t eh[2];
  memcpy(&eh[0], o + 4 * sizeof(cudaIpcMemHandle_t), sizeof(cudaIpcEventHandle_t));
  memcpy(&eh[1], o + 4 * sizeof(cudaIpcMemHandle_t) + sizeof(cudaIpcEventHandle_t), sizeof(cudaIpcEventHandle_t));
  CK(cudaIpcOpenEventHandle(&ctx->peer_free[side], eh[0]));
  CK(cudaIpcOpenEventHandle(&ctx->peer_ready[side], eh[1]));
  return 0;
}

int64_t mpm_ipc_blob_size(void) { return (int64_t)IPC_BLOB; }

// Same-process neighbours (several windows driven by one process: one GPU,
// or one GPU each with peer access): window a's `side` neighbour is b and
// b's opposite side is a.  The peer pointers are the neighbour's own device
// buffers, so the IPC halo kernels and the device-ordered counter protocol
// (mpm_ipc_halo) run unchanged, without IPC handles.
int mpm_peer_connect(mpm_ctx* a, int side, mpm_ctx* b) {
  if (!a || !b || side < 0 || side > 1 || a == b) return MPM_EINVAL;
  if (!a->h_cap || !b->h_cap) return fail(a, MPM_ESTATE, "peer_connect: call mpm_set_slab on both windows first");
  mpm_ctx* w[2] = {a, b};
  const int sd[2] = {side, 1 - side};
  for (int k = 0; k < 2; ++k) {
    mpm_ctx* ctx = w[k];
    CK(cudaSetDevice(ctx->dev));
    if (!ctx->ipc_vrecv[sd[k]]) {
      TRY(dalloc(ctx, &ctx->ipc_vrecv[sd[k]], (size_t)(ctx->h_cap + 1) * 64));
      TRY(dalloc(ctx, &ctx->ipc_cnt[sd[k]], 8));
      CK(cudaMemset(ctx->ipc_cnt[sd[k]], 0, 8 * sizeof(int)));
    }
    if (!ctx->ipc_free[sd[k]]) {
      CK(cudaEventCreateWithFlags(&ctx->ipc_free[sd[k]], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ctx->ipc_ready[sd[k]], cudaEventDisableTiming));
    }
  }
  if (a->dev != b->dev) {
    for (int k = 0; k < 2; ++k) {
      mpm_ctx* ctx = w[k];
      CK(cudaSetDevice(ctx->dev));
      const cudaError_t e = cudaDeviceEnablePeerAccess(w[1 - k]->dev, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return fail(a, MPM_ECUDA, "peer_connect: no peer access");
      cudaGetLastError();
    }
  }
  for (int k = 0; k < 2; ++k) {
    mpm_ctx* c = w[k];
    mpm_ctx* o = w[1 - k];
    const int s = sd[k];
    c->peer_ids[s] = o->h_recv_ids[1 - s];
    c->peer_data[s] = o->h_recv_data[1 - s];
    c->peer_cnt[s] = o->ipc_cnt[1 - s];
    c->peer_vdata[s] = o->ipc_vrecv[1 - s];
    c->peer_free[s] = o->ipc_free[1 - s];
    c->peer_ready[s] = o->ipc_ready[1 - s];
    c->peer_local[s] = true;
  }
  return cudaSetDevice(a->dev) == cudaSuccess ? 0 : MPM_ECUDA;
}

// Stream memory operations (driver entry points through the runtime): the
// halo protocol orders the neighbours' streams with counters in device memory
// -- a wait on our own counter, a write into the neighbour's (IPC-mapped,
// NVLink between GPUs) -- so no host barrier is needed per substep.
typedef CUresult (*StreamWaitValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*StreamWriteValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static StreamWaitValue32Fn stream_wait_value32() {
  static StreamWaitValue32Fn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<StreamWaitValue32Fn>(f);
  }();
  return fn;
}
static StreamWriteValue32Fn stream_write_value32() {
  static StreamWriteValue32Fn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<StreamWriteValue32Fn>(f);
  }();
  return fn;
}

int mpm_ipc_mode(mpm_ctx* ctx, int* device_ordered) {
  if (!ctx || !device_ordered) return MPM_EINVAL;
  *device_ordered = stream_wait_value32() && stream_write_value32() && !getenv("SOFTMPM_IPC_EVENTS") ? 1 : 0;
  return 0;
}

// Wait until our counter cnt[k] reaches v / set the neighbour's counter to v.
static int ipc_wait(mpm_ctx* ctx, int* cnt, int k, unsigned v) {
  if (stream_wait_value32()(reinterpret_cast<CUstream>(ctx->stream), reinterpret_cast<CUdeviceptr>(cnt + k), v,
                            CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
    return fail(ctx, MPM_ECUDA, "ipc_halo: stream wait failed");
  return 0;
}
static int ipc_signal(mpm_ctx* ctx, int* peer_cnt, int k, unsigned v) {
  if (stream_write_value32()(reinterpret_cast<CUstream>(ctx->stream), reinterpret_cast<CUdeviceptr>(peer_cnt + k), v,
                             CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
    return fail(ctx, MPM_ECUDA, "ipc_halo: stream write failed");
  return 0;
}

int mpm_ipc_halo(mpm_ctx* ctx, int phase, int sides) {
  if (!ctx || phase < 0 || phase > 3) return MPM_EINVAL;
  CK(cudaSetDevice(ctx->dev));
  int ordered = 0;
  TRY(mpm_ipc_mode(ctx, &ordered));
  Params p = make_params(ctx);
  for (int sd = 0; sd < 2; ++sd) {
    if (!((sides >> sd) & 1)) continue;
    if (!ctx->peer_ids[sd] || !ctx->ipc_cnt[sd]) return fail(ctx, MPM_ESTATE, "ipc_halo: side not connected");
    // same-process neighbours order their streams with plain events: a
    // stream wait on a value that a LATER-issued operation of another stream
    // of this process writes can deadlock when both streams alias one
    // hardware work queue; an event wait always follows its record in host
    // order (the caller issues each phase for every window before the next)
    const bool ordered_sd = ordered && !ctx->peer_local[sd];
    // [0] records received, [1] received last, [2] records sent,
    // [4] neighbour's writes ready (set by it), [5] our writes consumed (set by it)
    int* cnt = ctx->ipc_cnt[sd];
    int* pcnt = ctx->peer_cnt[sd];
    // before writing into the neighbour: it consumed our previous write
    auto before_write = [&]() -> int {
      if (ordered_sd) return ipc_wait(ctx, cnt, 5, ctx->ipc_writes[sd]);
      CK(cudaStreamWaitEvent(ctx->stream, ctx->peer_free[sd], 0));
      return 0;
    };
    auto after_write = [&]() -> int {
      if (ordered_sd) return ipc_signal(ctx, pcnt, 4, ++ctx->ipc_writes[sd]);
      CK(cudaEventRecord(ctx->ipc_ready[sd], ctx->stream));
      return 0;
    };
    auto before_read = [&]() -> int {
      if (ordered_sd) return ipc_wait(ctx, cnt, 4, ++ctx->ipc_reads[sd]);
      CK(cudaStreamWaitEvent(ctx->stream, ctx->peer_ready[sd], 0));
      return 0;
    };
    auto after_read = [&]() -> int {
      if (ordered_sd) return ipc_signal(ctx, pcnt, 5, ctx->ipc_reads[sd]);
      CK(cudaEventRecord(ctx->ipc_free[sd], ctx->stream));
      return 0;
    };
    switch (phase) {
      case 0:  // ghost momentum -> neighbour (after it consumed our last writes)
        TRY(before_write());
        ipc_pack_kernel<<<ctx->sms * 4, 256, 0, ctx->stream>>>(p, sd, ctx->ghost_bricks, ctx->peer_ids[sd],
                                                               ctx->peer_data[sd], pcnt, ctx->h_send_ids[sd], cnt + 2);
        LAUNCHED();
        TRY(after_write());
        break;
      case 1:  // add the neighbour's ghost momentum into our owned bricks
        TRY(before_read());
        ipc_unpack_add_kernel<<<ctx->sms * 4, 256, 0, ctx->stream>>>(p, ctx->h_recv_ids[sd], ctx->h_recv_data[sd], cnt,
                                                                     ctx->h_local_ids[sd]);
        LAUNCHED();
        CK(cudaMemcpyAsync(cnt + 1, cnt, sizeof(int), cudaMemcpyDeviceToDevice, ctx->stream));
        CK(cudaMemsetAsync(cnt, 0, sizeof(int), ctx->stream));
        TRY(after_read());
        break;
      case 2:  // velocities of the received bricks -> neighbour
        TRY(before_write());
        ipc_pack_vel_kernel<<<ctx->sms * 4, 256, 0, ctx->stream>>>(p, ctx->h_local_ids[sd], cnt + 1,
                                                                   ctx->peer_vdata[sd]);
        LAUNCHED();
        TRY(after_write());
        break;
      case 3:  // the owner's velocities into our ghost bricks
        TRY(before_read());
        ipc_unpack_vel_kernel<<<ctx->sms * 4, 256, 0, ctx->stream>>>(p, ctx->h_send_ids[sd], cnt + 2,
                                                                     ctx->ipc_vrecv[sd]);
        LAUNCHED();
        CK(cudaMemsetAsync(cnt + 2, 0, sizeof(int), ctx->stream));
        TRY(after_read());
        break;
    }
  }
  return 0;
}

int mpm_halo_buffers(mpm_ctx* ctx, int side, void** send_ids, void** send_data, void** recv_ids, void** recv_data,
                     int64_t* capacity) {
  if (!ctx || side < 0 || side > 1 || !ctx->h_cap) return fail(ctx, MPM_ESTATE, "halo_buffers: call mpm_set_slab first");
  if (send_ids) *send_ids = ctx->h_send_ids[side];
  if (send_data) *send_data = ctx->h_send_data[side];
  if (recv_ids) *recv_ids = ctx->h_recv_ids[side];
  if (recv_data) *recv_data = ctx->h_recv_data[side];
  if (capacity) *capacity = ctx->h_cap;
  return 0;
}

int mpm_stage_begin(mpm_ctx* ctx, int nsub, int use_colliders) {
  if (ctx) ctx->bins_age = -1;  // particle order / positions may change: the next frame re-bins
  if (!ctx || nsub <= 0) return fail(ctx, MPM_EINVAL, "stage_begin: bad arguments");
  TRY(need_particles(ctx));
  CK(cudaSetDevice(ctx->dev));
  if (ctx->cfg.deterministic) return fail(ctx, MPM_EINVAL, "stage driver: fast mode only");
  ctx->stage_nsub = nsub;
  ctx->stage_col = use_colliders && ctx->ncol > 0 && ctx->cfg.theta >= 0.0;
  CK(cudaMemsetAsync(ctx->inverted, 0, sizeof(unsigned long long), ctx->stream));
  TRY(ensure_gm_clean(ctx));
  TRY(rebin(ctx));
  return 0;
}

int mpm_stage_particles(mpm_ctx* ctx, int first) {
  if (!ctx) return MPM_EINVAL;
  CK(cudaSetDevice(ctx->dev));
  TRY(launch_fused(ctx, first == 0));
  return 0;
}

int mpm_stage_grid(mpm_ctx* ctx, int sub, int clear) {
  if (!ctx) return MPM_EINVAL;
  CK(cudaSetDevice(ctx->dev));
  TRY(launch_grid_op(ctx, false, ctx->stage_col != 0, sub, clear != 0));
  if (!clear) ctx->grid_dirty = 1;
  return 0;
}

int mpm_stage_end(mpm_ctx* ctx, int64_t* inverted) {
  if (!ctx) return MPM_EINVAL;
  CK(cudaSetDevice(ctx->dev));
  TRY(launch_g2p(ctx));
  ctx->grid_dirty = 1;
  ctx->grid_phase = 1;
  return read_inverted(ctx, inverted);
}

int mpm_halo_pack(mpm_ctx* ctx, int side, int64_t* count) {
  if (!ctx || side < 0 || side > 1 || !ctx->h_cap) return fail(ctx, MPM_ESTATE, "halo_pack: no slab");
  CK(cudaSetDevice(ctx->dev));
  int* cnt = ctx->counters + 2;
  CK(cudaMemsetAsync(cnt, 0, sizeof(int), ctx->stream));
  Params p = make_params(ctx);
  halo_pack_kernel<<<ctx->sms * 4, 256, 0, ctx->stream>>>(p, side, ctx->ghost_bricks, ctx->h_send_ids[side],
                                                           ctx->h_send_data[side], cnt);
  LAUNCHED();
  int h = 0;
  CK(cudaMemcpyAsync(&h, cnt, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (h > ctx->h_cap) return fail(ctx, MPM_ESTATE, "halo_pack: overflow");
  if (count) *count = h;
  return 0;
}

int mpm_halo_unpack_add(mpm_ctx* ctx, int side, int64_t n) {
  if (!ctx || side < 0 || side > 1 || n < 0 || n > ctx->h_cap) return fail(ctx, MPM_EINVAL, "halo_unpack_add: bad arguments");
  CK(cudaSetDevice(ctx->dev));
  ctx->h_recv_n[side] = (int)n;
  if (n == 0) return 0;
  Params p = make_params(ctx);
  halo_unpack_add_kernel<<<ctx->sms * 4, 256, 0, ctx->stream>>>(p, ctx->h_recv_ids[side], ctx->h_recv_data[side],
                                                                 (int)n, ctx->h_local_ids[side]);
  LAUNCHED();
  CK(cudaStreamSynchronize(ctx->stream));
  return 0;
}

int mpm_halo_pack_vel(mpm_ctx* ctx, int side, int64_t* count) {
  if (!ctx || side < 0 || side > 1) return MPM_EINVAL;
  CK(cudaSetDevice(ctx->dev));
  const int n = ctx->h_recv_n[side];
  if (count) *count = n;
  if (n == 0) return 0;
  Params p = make_params(ctx);
  halo_pack_vel_kernel<<<ctx->sms * 4, 256, 0, ctx->stream>>>(p, ctx->h_local_ids[side], n, ctx->h_send_data[side]);
  LAUNCHED();
  CK(cudaStreamSynchronize(ctx->stream));
  return 0;
}

int mpm_halo_unpack_vel(mpm_ctx* ctx, int side, int64_t n) {
  if (!ctx || side < 0 || side > 1 || n < 0 || n > ctx->h_cap) return fail(ctx, MPM_EINVAL, "halo_unpack_vel: bad arguments");
  CK(cudaSetDevice(ctx->dev));
  if (n == 0) return 0;
  Params p = make_params(ctx);
  // our packed ids of this side are still in h_send_ids[side]
  halo_unpack_vel_kernel<<<ctx->sms * 4, 256, 0, ctx->stream>>>(p, ctx->h_send_ids[side], ctx->h_recv_data[side],
                                                                 (int)n);
  LAUNCHED();
  CK(cudaStreamSynchronize(ctx->stream));
  return 0;
}

// Remove particles whose global base cell x left [own_lo, own_hi) into two
// device row buffers (low / high neighbour); returns their counts and buffer
// pointers/capacity (rows: NF floats, material id, particle id; SoA by field).
int mpm_extract_migrants(mpm_ctx* ctx, int own_lo, int own_hi, int64_t* n_lo, int64_t* n_hi, void** rows_lo,
                         void** rows_hi, int64_t* rows_cap) {
  if (ctx) ctx->bins_age = -1;  // particle order / positions may change: the next frame re-bins
  if (!ctx) return MPM_EINVAL;
  TRY(need_particles(ctx));
  CK(cudaSetDevice(ctx->dev));
  invalidate_graphs(ctx);
  TRY(compact_if_needed(ctx));  // one extraction per re-binning
  const long long n = ctx->n;
  if (!ctx->mflag || ctx->mig_cap < ctx->cap) {
    TRY(dalloc(ctx, &ctx->mflag, (size_t)ctx->cap * 4));
    for (int s = 0; s < 2; ++s) TRY(dalloc(ctx, &ctx->mig_rows[s], (size_t)ctx->cap * (NF + 2)));
    ctx->mig_cap = ctx->cap;
    TRY(ensure_scan(ctx, ctx->cap));
  }
  int* flag = ctx->mflag;
  int* cls = flag + ctx->cap;
  Params p = make_params(ctx);
  migrant_flag_kernel<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(p, own_lo, own_hi, flag);
  LAUNCHED();
  // ranks of the low / high migrants (class scans back to back, ONE host sync)
  int* posv[3] = {nullptr, ctx->rank, ctx->lcell};  // class scans reuse the rank / lcell scratch
  int last_pos[3] = {0, 0, 0}, last_cls[3] = {0, 0, 0};
  for (int c = 1; c < 3 && n > 0; ++c) {
    flag_class_kernel<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(flag, c, cls, n);
    LAUNCHED();
    TRY(scan_exclusive(ctx, cls, posv[c], n));
    CK(cudaMemcpyAsync(&last_pos[c], posv[c] + n - 1, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(&last_cls[c], cls + n - 1, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  const long long m_lo = last_pos[1] + last_cls[1], m_hi = last_pos[2] + last_cls[2];
  if (m_lo + m_hi > 0) {
    migrant_rows_kernel<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(p, flag, posv[1], posv[2], ctx->mig_rows[0],
                                                                     ctx->mig_rows[1], m_lo, m_hi);
    LAUNCHED();
    CK(cudaStreamSynchronize(ctx->stream));
    // the migrants' slots stay until the next re-binning drops them
    ctx->hole_n = n;
    ctx->hole_count = m_lo + m_hi;
  }
  if (n_lo) *n_lo = m_lo;
  if (n_hi) *n_hi = m_hi;
  if (rows_lo) *rows_lo = ctx->mig_rows[0];
  if (rows_hi) *rows_hi = ctx->mig_rows[1];
  if (rows_cap) *rows_cap = 0;  // packed: each side's rows are a contiguous ROWS x count block
  return 0;
}

// Append m migrant rows (device buffer in the layout above, capacity rows_cap)
// coming from a window whose global x offset is src_offset nodes.
int mpm_append_particles(mpm_ctx* ctx, const void* rows, int64_t m, int64_t rows_cap, int src_offset) {
  if (ctx) ctx->bins_age = -1;  // particle order / positions may change: the next frame re-bins
  if (!ctx || m < 0) return MPM_EINVAL;
  if (m == 0) return 0;
  CK(cudaSetDevice(ctx->dev));
  if (ctx->n + m > ctx->cap) return fail(ctx, MPM_ENOMEM, "append_particles: capacity exceeded (reserve with mpm_reserve)");
  invalidate_graphs(ctx);
  Params p = make_params(ctx);
  const float dxs = (float)((src_offset - ctx->goff[0]) * ctx->cfg.dx);
  // stream-ordered: the rows are complete (mpm_extract_migrants returns after
  // its own stream synchronisation, peer rows arrive through a synchronised
  // copy), and the caller's buffer must stay valid until this stream reaches
  // the kernel (device buffers of the neighbour window / a torch tensor held
  // until the next synchronisation)
  append_rows_kernel<<<blocks_for(m, 256), 256, 0, ctx->stream>>>(p, (const float*)rows, m, rows_cap, ctx->n, dxs);
  LAUNCHED();
  ctx->n += m;
  return 0;
}

// Grow particle capacity (keeps contents) so migrants can be appended.
int mpm_reserve(mpm_ctx* ctx, int64_t cap) {
  if (ctx) ctx->bins_age = -1;  // particle order / positions may change: the next frame re-bins
  if (!ctx || cap <= ctx->cap) return 0;
  CK(cudaSetDevice(ctx->dev));
  invalidate_graphs(ctx);
  TRY(compact_if_needed(ctx));
  float* P = nullptr;
  int *mat = nullptr, *orig = nullptr;
  TRY(dalloc(ctx, &P, (size_t)cap * NF));
  TRY(dalloc(ctx, &mat, (size_t)cap));
  TRY(dalloc(ctx, &orig, (size_t)cap));
  for (int f = 0; f < NF; ++f)
    CK(cudaMemcpyAsync(P + (size_t)f * cap, ctx->P[ctx->cur] + (size_t)f * ctx->cap, sizeof(float) * ctx->n,
                       cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaMemcpyAsync(mat, ctx->mat[ctx->cur], sizeof(int) * ctx->n, cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaMemcpyAsync(orig, ctx->orig[ctx->cur], sizeof(int) * ctx->n, cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  for (int b = 0; b < 2; ++b) {
    cudaFree(ctx->P[b]);
    cudaFree(ctx->mat[b]);
    cudaFree(ctx->orig[b]);
    ctx->P[b] = nullptr;
    ctx->mat[b] = nullptr;
    ctx->orig[b] = nullptr;
  }
  ctx->P[0] = P;
  ctx->mat[0] = mat;
  ctx->orig[0] = orig;
  TRY(dalloc(ctx, &ctx->P[1], (size_t)cap * NF));
  TRY(dalloc(ctx, &ctx->mat[1], (size_t)cap));
  TRY(dalloc(ctx, &ctx->orig[1], (size_t)cap));
  ctx->cur = 0;
  int* const* scratch[] = {&ctx->key, &ctx->rank, &ctx->lcell, &ctx->sidx, &ctx->slc, &ctx->bperm};
  for (auto s : scratch) TRY(dalloc(ctx, const_cast<int**>(s), (size_t)cap));
  ctx->work_cap = ctx->nbins + cap / MIN_CHUNK + 1;
  TRY(dalloc(ctx, &ctx->work, (size_t)ctx->work_cap));
  TRY(dalloc(ctx, &ctx->item_bounds, (size_t)ctx->work_cap));
  TRY(dalloc(ctx, &ctx->item_bounds2, (size_t)ctx->work_cap));
  ctx->bounds_a = ctx->item_bounds;
  ctx->bounds_out_clean = false;
  TRY(dalloc(ctx, &ctx->pay, (size_t)cap * NPAY));
  TRY(dalloc(ctx, &ctx->item_box, (size_t)ctx->work_cap));
  if (ctx->perm) {
    cudaFree(ctx->perm);
    cudaFree(ctx->payload);
    ctx->perm = nullptr;
    ctx->payload = nullptr;
  }
  ctx->cap = cap;
  TRY(ensure_stage(ctx, sizeof(double) * (size_t)cap * 24));
  return 0;
}

// Replace the original-index slot of every particle by ids[original index]
// (slab windows carry global particle ids; field readback is then by id).
int mpm_set_ids(mpm_ctx* ctx, const int32_t* ids) {
  if (ctx) ctx->bins_age = -1;  // particle order / positions may change: the next frame re-bins
  if (!ctx || !ids) return MPM_EINVAL;
  TRY(need_particles(ctx));
  CK(cudaSetDevice(ctx->dev));
  const long long n = ctx->n;
  TRY(ensure_stage(ctx, sizeof(double) * (size_t)n * 24));
  int* sid = (int*)ctx->stage;
  CK(cudaMemcpyAsync(sid, ids, sizeof(int) * n, cudaMemcpyHostToDevice, ctx->stream));
  Params p = make_params(ctx);
  set_ids_kernel<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(p, sid);
  LAUNCHED();
  CK(cudaStreamSynchronize(ctx->stream));
  return 0;
}

// ids, x (global), v, F, C of every particle in device order.
int mpm_download_rows(mpm_ctx* ctx, int32_t* ids, double* x, double* v, double* F, double* C) {
  if (!ctx || !ids || !x || !v || !F || !C) return MPM_EINVAL;
  CK(cudaSetDevice(ctx->dev));
  TRY(compact_if_needed(ctx));
  const long long n = ctx->n;
  if (n <= 0) return 0;
  TRY(ensure_stage(ctx, sizeof(double) * (size_t)n * 25 + 64));
  Params p = make_params(ctx);
  double* s = ctx->stage;
  download_rows_kernel<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(p, s, s + 3 * n, s + 6 * n, s + 15 * n);
  LAUNCHED();
  download_ids_kernel<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(p, (int*)(s + 24 * n), s);
  LAUNCHED();
  CK(cudaMemcpyAsync(ids, s + 24 * n, sizeof(int) * n, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(x, s, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(v, s + 3 * n, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(F, s + 6 * n, sizeof(double) * 9 * n, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(C, s + 15 * n, sizeof(double) * 9 * n, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return 0;
}

// Device-to-device copy (halo / migrant buffers between contexts or to
// communication buffers).
// The copy is complete (and ordered after all prior work of every stream of
// the device) when the call returns: contexts run on non-blocking streams,
// which a blocking cudaMemcpy does not order against, so the device is
// synchronised on both sides of the copy.
int mpm_device_copy(void* dst, const void* src, int64_t bytes) {
  if (bytes <= 0) return 0;
  if (cudaDeviceSynchronize() != cudaSuccess) return MPM_ECUDA;
  if (cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDefault, cudaStreamPerThread) != cudaSuccess) return MPM_ECUDA;
  return cudaStreamSynchronize(cudaStreamPerThread) == cudaSuccess ? 0 : MPM_ECUDA;
}

// Particle ids (original indices) and global positions in device order.
int mpm_download_ids(mpm_ctx* ctx, int32_t* ids, double* x) {
  if (!ctx || !ids || !x) return MPM_EINVAL;
  CK(cudaSetDevice(ctx->dev));
  TRY(compact_if_needed(ctx));
  const long long n = ctx->n;
  if (n <= 0) return 0;
  TRY(ensure_stage(ctx, sizeof(double) * (size_t)n * 4 + 64));
  Params p = make_params(ctx);
  double* sx = ctx->stage;
  int* sid = (int*)(ctx->stage + 3 * n);
  download_ids_kernel<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(p, sid, sx);
  LAUNCHED();
  CK(cudaMemcpyAsync(ids, sid, sizeof(int) * n, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(x, sx, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return 0;
}

void* mpm_host_alloc(int64_t bytes) {
  void* p = nullptr;
  if (cudaMallocHost(&p, (size_t)bytes) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return p;
}

void mpm_host_free(void* ptr) {
  if (ptr) cudaFreeHost(ptr);
}

}  // extern "C"
