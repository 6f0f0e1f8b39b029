// gmaf_api.cu -- host runtime of libgmaf: the C ABI of include/gmaf.h.
//
// Context = caller-owned device workspace carved into fields, a caller stream, and a
// cache of instantiated CUDA graphs (one per preconditioner / start mode).  A solve is
// ONE graph launch: init kernel -> WHILE node {(phase A, phase B) x UNROLL} -> true
// residual kernel; the convergence decision is taken on the device (Eq. 3.9) and the host
// reads the statistics once, after the graph.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>   // types only: NCCL is resolved at run time (world == 1 needs no NCCL)

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <new>
#include <string>
#include <vector>

#include "../../include/gmaf.h"
#include "gmaf_internal.cuh"

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

namespace gmaf {
int quad_ctas_per_condition(const GridParams& g, int K);
cudaError_t configure_pcg_kernels(const TileCfg& t, int K);
int pcg_ctas_per_sm(const TileCfg& t, int K);
}
static_assert(gmaf::SR_HALO_COLS == 4, "sr.cu halo");

using namespace gmaf;

namespace {

// NCCL, loaded on demand (normally the libnccl.so.2 that torch already mapped).
struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) { a.err = dlerror(); return a; }
    a.getUniqueId = reinterpret_cast<decltype(a.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    a.commInitRank = reinterpret_cast<decltype(a.commInitRank)>(dlsym(h, "ncclCommInitRank"));
    a.allGather = reinterpret_cast<decltype(a.allGather)>(dlsym(h, "ncclAllGather"));
    a.commDestroy = reinterpret_cast<decltype(a.commDestroy)>(dlsym(h, "ncclCommDestroy"));
    a.getErrorString = reinterpret_cast<decltype(a.getErrorString)>(dlsym(h, "ncclGetErrorString"));
    a.ok = a.getUniqueId && a.commInitRank && a.allGather && a.commDestroy && a.getErrorString;
    if (!a.ok) a.err = "libnccl.so.2 lacks a required symbol";
    return a;
  }();
  return api;
}

// Contiguous condition blocks: rank r owns [lo, hi); the first K % world ranks one more.
void shard(int K, int world, int rank, int* lo, int* hi) {
  const int base = K / world, extra = K % world;
  *lo = rank * base + (rank < extra ? rank : extra);
  *hi = *lo + base + (rank < extra ? 1 : 0);
}

bool dist_mode(const gmaf_dist* dist) {
  return dist && (dist->world > 1 || dist->nccl_unique_id != nullptr || dist->shard == GMAF_SHARD_CONDITIONS_P2P ||
                  dist->shard == GMAF_SHARD_ROWS_P2P);
}
bool rows_mode(const gmaf_dist* dist) { return dist_mode(dist) && dist->shard == GMAF_SHARD_ROWS_P2P; }

// Row slab of `rank`: own rows [y0, y1) (contiguous blocks, the first n_y % world ranks one more)
// and stored rows [yb, ye) = own rows + SLAB_HALO halo rows per side inside the domain.
struct Slab { int y0, y1, yb, ye; };
Slab slab_of(int ny, int world, int rank) {
  Slab sl{};
  shard(ny, world, rank, &sl.y0, &sl.y1);
  sl.yb = sl.y0 - SLAB_HALO < 0 ? 0 : sl.y0 - SLAB_HALO;
  sl.ye = sl.y1 + SLAB_HALO > ny ? ny : sl.y1 + SLAB_HALO;
  return sl;
}

constexpr int kUnroll = 4;          // (A, B) pairs per WHILE-body execution (must be even)
static_assert(kUnroll % 2 == 0, "ping-pong parity");
constexpr size_t kAlign = 256;

enum State { ST_CREATED = 0, ST_THICK = 1, ST_ASSEMBLED = 2, ST_SOLVED = 3 };

struct GraphKey {
  int schedule, precond, warm, fixed;
  bool operator<(const GraphKey& o) const {
    if (schedule != o.schedule) return schedule < o.schedule;
    if (precond != o.precond) return precond < o.precond;
    if (warm != o.warm) return warm < o.warm;
    return fixed < o.fixed;
  }
};

struct Layout {
  size_t off_ct, off_st, off_cth, off_sth, off_cp, off_AP, off_AE, off_AN, off_S, off_p, off_r, off_r2,
      off_u, off_u2,
      off_scratch, off_constrows, off_part, off_wpart, off_wrench, off_state, off_cs, off_counters, off_timing,
      off_guard, off_matrep, off_plocal, off_pall, off_wall, total;
};

size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

// One wave: as many (strip, chunk, condition) tiles as the GPU holds resident CTAs
// (slots = SMs x CTAs/SM from the occupancy calculator), each CTA marching a long chunk.
TileCfg make_tiles(int nt, int ny, int K, int slots, int tw) {
  TileCfg t{};
  t.tw = tw;
  t.n_strips = (nt + t.tw - 1) / t.tw;
  int chunks = slots / (t.n_strips * K);
  if (chunks < 1) chunks = 1;
  int th = (ny + chunks - 1) / chunks;
  if (th < 8) th = 8;
  if (th > ny) th = ny;
  t.th = th;
  t.n_chunks = (ny + th - 1) / th;
  t.n_tiles = t.n_strips * t.n_chunks;
  return t;
}


// strip widths: two-phase kernels 256/128 columns; the single-pass kernel keeps the seam
// inside a strip, so its strips may not be wider than the ring (and need >= 12 columns)
int tw_table1(int nt) { return nt >= 1024 ? 256 : 128; }
int tw_single(int nt) {
  // 512-column strips for wide meshes: one CTA per SM (10 warps) instead of two 256-column CTAs,
  // half the halo columns; slightly more cycles per iteration but less power, so under the
  // B200's power cap the clock stays higher (measured at C3: 259.6-260.3 vs 264.7-266.8 us per
  // iteration, 1912-1927 vs 1852-1856 MHz)
  int cap = nt >= 1024 ? 512 : 256;
  if (const char* e = std::getenv("GMAF_SR_TW")) cap = std::atoi(e);   // A/B experiments
  if (cap < 12 || cap > 1000) cap = 256;
  int w = nt < cap ? nt : cap;
  // a multiple of 4: strip s starts at column s*tw - tw/2, which must be even so that every
  // column pair (and every 16-byte TMA row segment) is aligned
  return w & ~3;
}
bool single_ok(int nt) { return nt % 2 == 0 && nt >= 12; }
constexpr int kConstRowLen = 1024;   // >= the widest TMA row segment (tw + 2*halo)

int check_grid(const gmaf_grid* g) {
  if (!g) return GMAF_E_INVALID_ARG;
  if (g->n_theta < 4 || g->n_y < 4) return GMAF_E_INVALID_MESH;
  // the iteration kernels index a row of one condition's field in 32-bit arithmetic
  // ((n_y + 8) n_theta < 2^31: 2^31 doubles = 16 GiB per condition and field)
  if (((long long)g->n_y + 16) * (long long)g->n_theta >= (1ll << 31)) return GMAF_E_INVALID_MESH;
  if (!(g->R_k > 0.0) || !(g->R_c > g->R_k) || !(g->mu > 0.0)) return GMAF_E_INVALID_ARG;
  if (g->tex_n_theta > 0 || g->tex_n_y > 0) {
    if (g->tex_n_theta <= 0 || g->tex_n_y <= 0 || g->tex_band_rows <= 0 || g->tex_band_rows > g->n_y ||
        g->tex_fill_den <= 0 || g->tex_fill_num < 0 || g->tex_fill_num > g->tex_fill_den ||
        g->tex_depth < 0.0)
      return GMAF_E_INVALID_ARG;
    if (g->n_theta < 2 * g->tex_n_theta || g->tex_band_rows < 2 * g->tex_n_y) return GMAF_E_MESH_TOO_COARSE;
    // the device evaluates the mask in 32-bit unsigned arithmetic (geometry.cu texture_mask)
    if ((unsigned long long)g->n_theta * (unsigned long long)g->tex_n_theta >= (1ull << 32) ||
        (unsigned long long)g->tex_band_rows * (unsigned long long)g->tex_n_y >= (1ull << 32))
      return GMAF_E_INVALID_ARG;
  }
  return GMAF_OK;
}

// Mcap = distinct coefficient sets the bands hold (<= K; conditions with equal (e, L_F) share
// one, Eq. 2.3 has no e-dot: the 9 FD conditions of one state need 5).  The bands come LAST so
// that gmaf_create can read Mcap back from the workspace size.
Layout make_layout(const gmaf_grid* g, int K, int world = 0, int kmax = 0, int rows_stored = 0, int Mcap = 0) {
  Layout L{};
  if (Mcap <= 0 || Mcap > K) Mcap = K;
  const size_t nt = (size_t)g->n_theta, ny = (size_t)g->n_y;
  const size_t n = nt * (size_t)(rows_stored > 0 ? rows_stored : g->n_y);   // per-condition field
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t at = o; o = align_up(o + bytes); return at; };
  L.off_ct = take(nt * 8); L.off_st = take(nt * 8); L.off_cth = take(nt * 8); L.off_sth = take(nt * 8);
  L.off_cp = take((size_t)K * sizeof(CondParams));
  L.off_S = take((size_t)K * n * 8); L.off_p = take((size_t)K * n * 8);
  L.off_r = take((size_t)K * n * 8); L.off_r2 = take((size_t)K * n * 8);
  L.off_u = take((size_t)K * n * 8); L.off_u2 = take((size_t)K * n * 8);
  L.off_scratch = take((ny + 2) * nt * 8);
  L.off_constrows = take((size_t)2 * kConstRowLen * 8);   // a zero row and a one row (TMA sources)
  L.off_part = take((size_t)4 * K * kMaxTilesPerCondition * 8);
  L.off_wpart = take((size_t)(148 * 8 + K) * 12 * 8);
  L.off_wrench = take((size_t)(K > kmax ? K : kmax) * 12 * 8);
  L.off_plocal = take((size_t)4 * (kmax > 0 ? kmax : 1) * 8);
  L.off_pall = take((size_t)4 * (world > 0 ? world : 1) * (kmax > 0 ? kmax : 1) * 8);
  L.off_wall = take((size_t)12 * (world > 0 ? world : 1) * (kmax > 0 ? kmax : 1) * 8);
  L.off_state = take(sizeof(SolverState));
  L.off_cs = take((size_t)9 * K * 8);   // 7 double arrays + 2 int arrays
  L.off_counters = take(16 * sizeof(unsigned int));
  L.off_timing = take(sizeof(Timing));
  L.off_guard = take(4 * sizeof(unsigned long long));
  L.off_matrep = take((size_t)K * sizeof(int32_t));
  L.off_AP = take((size_t)Mcap * n * 8); L.off_AE = take((size_t)Mcap * n * 8); L.off_AN = take((size_t)Mcap * n * 8);
  L.total = o;
  return L;
}

}  // namespace

struct gmaf_ctx {
  gmaf_grid grid{};
  GridParams gp{};
  int K = 0;
  gmaf_dist dist{0, 1, nullptr, 0};
  cudaStream_t stream = nullptr;
  cudaStream_t cap_stream = nullptr;
  char* ws = nullptr;
  size_t ws_bytes = 0;
  Layout L{};
  TileCfg tiles{};      // two-phase (Table-1 schedule) kernels
  TileCfg tiles_sr{};   // single-pass kernel
  int schedule = GMAF_SCHEDULE_SINGLE;
  DevPtrs d{};
  int M = 0;
  int Mcap = 0;          // distinct coefficient sets the band storage holds (<= K)
  std::vector<int32_t> mat_of, mat_rep;
  int state = ST_CREATED;
  std::string err;
  std::map<GraphKey, std::pair<cudaGraph_t, cudaGraphExec_t>> graphs;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // pinned staging
  SolverState* h_state = nullptr;
  double* h_cs = nullptr;        // 7*K
  double* h_wrench = nullptr;    // K*12
  unsigned long long* h_guard = nullptr;
  CondParams* h_cp = nullptr;
  Timing* h_timing = nullptr;
  int quad_ctas = 0;
  int r_parity = 0;   // which ping-pong buffer holds the latest residual
  int last_coupling = 0;
  bool stream_mode = false;  // GMAF_LAUNCH_MODE=stream: no CUDA graph (for ncu)
  bool sr_k_ok = true;       // K fits the single-pass kernel's reduction scratch
  bool persist_ok = false;   // the single-pass solve runs as one persistent launch (sr.cu k_srp)
  // multi-rank (condition sharding): this rank owns global conditions [kofs, kofs + K)
  bool distm = false;
  int world = 1, rank = 0, kofs = 0, Kglob = 0, kmax = 0;
  ncclComm_t comm = nullptr;
  // peer-to-peer mode (condition sharding without NCCL)
  bool p2p = false, p2p_ready = false;
  bool rows = false;                       // row-slab sharding (GMAF_SHARD_ROWS_P2P)
  size_t inbox_off = 0;                    // byte offset of the halo inboxes in p2p_buf
  char* p2p_buf = nullptr;                 // library-owned exchange buffer (cudaMalloc, IPC-exported)
  void* peer_bufs[kMaxP2P] = {};           // IPC-opened buffers of the other ranks
  double* h_packed = nullptr;   // [world][4][kmax]
  double* h_wall = nullptr;     // [world][kmax][12]
  cudaEvent_t evb[2] = {nullptr, nullptr};
  int* h_done = nullptr;        // [2]
};

namespace {

thread_local std::string g_create_err;   // reason of the last failed gmaf_create on this thread

gmaf_status fail(gmaf_ctx* c, gmaf_status code, const char* fmt, ...) {
  if (c) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    c->err = buf;
  }
  return code;
}

#define CU(call)                                                                              \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      return fail(ctx, GMAF_E_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call,                \
                  cudaGetErrorString(e_));                                                    \
  } while (0)

template <typename T>
T* at(gmaf_ctx* c, size_t off) { return reinterpret_cast<T*>(c->ws + off); }

// Host evaluation of the per-condition scalars, in the same IEEE operation order as the
// definition (oracle O3/O5): one rounding per operation, no contraction.
CondParams cond_params(const gmaf_grid& g, const gmaf_condition& c, int mat) {
  CondParams p{};
  for (int q = 0; q < 4; ++q) { p.e[q] = c.e[q]; p.edot[q] = c.edot[q]; }
  p.LF = c.L_F; p.Ut = c.U_theta; p.Uy = c.U_y; p.pin = c.p_in; p.pout = c.p_out;
  volatile double dtheta = (2.0 * M_PI) / (double)g.n_theta;
  volatile double dy = c.L_F / (double)(g.n_y + 1);
  volatile double dx = g.R_k * dtheta;
  p.dy = dy;
  p.dx = dx;
  p.rx = p.dy / p.dx;
  p.ry = p.dx / p.dy;
  p.sl = (c.e[2] - c.e[0]) / c.L_F;
  p.tl = (c.e[3] - c.e[1]) / c.L_F;
  p.sld = (c.edot[2] - c.edot[0]) / c.L_F;
  p.tld = (c.edot[3] - c.edot[1]) / c.L_F;
  p.mat = mat;
  return p;
}

bool same_matrix(const gmaf_condition& a, const gmaf_condition& b) {
  // A depends on h only, and h on (e, L_F) only (Eq. 2.3 has no e-dot).
  return std::memcmp(a.e, b.e, sizeof(a.e)) == 0 && std::memcmp(&a.L_F, &b.L_F, sizeof(double)) == 0;
}

// The three pieces of a solve, enqueued on stream `s` (captured into a graph or launched
// directly).  h = graph conditional handle (0 outside a graph).
cudaError_t enqueue_init(gmaf_ctx* ctx, const GraphKey& key, unsigned long long h, cudaStream_t s) {
  if (key.schedule == GMAF_SCHEDULE_TABLE1)
    return launch_init(ctx->gp, ctx->d, ctx->tiles, ctx->K, key.precond, key.warm != 0, h, s);
  if (key.warm) {   // r0 = S - A p0 into r[1], then the single-pass init reads it
    cudaError_t e = cudaSuccess;
    if (ctx->rows) e = launch_slab_exchange(ctx->gp, ctx->d, ctx->d.p, ctx->K, s);   // p0's halo rows
    if (e == cudaSuccess) e = launch_residual_init(ctx->gp, ctx->d, ctx->tiles, ctx->K, 1, s);
    if (e == cudaSuccess && ctx->rows) e = launch_slab_exchange(ctx->gp, ctx->d, ctx->d.r[1], ctx->K, s);
    if (e != cudaSuccess) return e;
  }
  cudaError_t e = launch_sr_init(ctx->gp, ctx->d, ctx->tiles_sr, ctx->K, key.precond, key.warm != 0, h, s);
  if (e != cudaSuccess || !ctx->p2p) return e;
  if (ctx->rows) {   // halos + sums + scalars (+ unpack into the fields when rows == 2)
    cudaError_t e2 = launch_p2p_rows(ctx->gp, ctx->d, true, 1, ctx->K, h, s);
    if (e2 == cudaSuccess && ctx->d.dist.rows == 2) e2 = launch_slab_unpack2(ctx->gp, ctx->d, true, 1, ctx->K, s);
    return e2;
  }
  return launch_p2p_scalar(ctx->d, true, ctx->K, h, s);   // peer-to-peer: gather + scalars
}

cudaError_t enqueue_iterations(gmaf_ctx* ctx, const GraphKey& key, unsigned long long h, cudaStream_t s) {
  cudaError_t e = cudaSuccess;
  for (int u = 0; u < kUnroll && e == cudaSuccess; ++u) {
    // iteration j = kUnroll*m + u: ping-pong parity u % 2 (kUnroll is even)
    if (key.schedule == GMAF_SCHEDULE_TABLE1) {
      e = launch_phase_a(ctx->gp, ctx->d, ctx->tiles, ctx->K, key.precond, u & 1, h, s);
      if (e == cudaSuccess) e = launch_phase_b(ctx->gp, ctx->d, ctx->tiles, ctx->K, key.precond, u & 1, h, s);
    } else {
      e = launch_sr_iter(ctx->gp, ctx->d, ctx->tiles_sr, ctx->K, key.precond, u & 1, h, s);
      if (e == cudaSuccess && ctx->rows) {
        e = launch_p2p_rows(ctx->gp, ctx->d, false, u & 1, ctx->K, h, s);
        if (e == cudaSuccess && ctx->d.dist.rows == 2) e = launch_slab_unpack2(ctx->gp, ctx->d, false, u & 1, ctx->K, s);
      }
      else if (e == cudaSuccess && ctx->p2p) e = launch_p2p_scalar(ctx->d, false, ctx->K, h, s);
    }
  }
  return e;
}

cudaError_t enqueue_final(gmaf_ctx* ctx, const GraphKey& key, cudaStream_t s) {
  if (key.schedule == GMAF_SCHEDULE_SINGLE) {
    cudaError_t e = launch_sr_fixup(ctx->gp, ctx->d, ctx->K, s);
    if (e != cudaSuccess) return e;
  }
  if (ctx->rows) {   // p's halo rows: the true residual below and the quadrature read them
    cudaError_t e = launch_slab_exchange(ctx->gp, ctx->d, ctx->d.p, ctx->K, s);
    if (e != cudaSuccess) return e;
  }
  cudaError_t e = launch_true_residual(ctx->gp, ctx->d, ctx->tiles, ctx->K, s);   // ||S - A p|| at exit
  if (e != cudaSuccess || !ctx->p2p) return e;
  // peer-to-peer mode: gather every rank's ||S_k - A_k p_k||^2, then the global value
  e = launch_p2p_gather(ctx->d, ctx->d.dist.packed_local, ctx->kmax, ctx->d.dist.packed_all, s);
  if (e != cudaSuccess) return e;
  return launch_true_scalar(ctx->d, ctx->world, s);
}

bool use_persistent(const gmaf_ctx* ctx, const GraphKey& key) {
  return ctx->persist_ok && key.schedule == GMAF_SCHEDULE_SINGLE && (!ctx->distm || ctx->p2p);
}

// Persistent solve: init -> ONE launch that runs every iteration (grid barrier per iteration,
// no WHILE node) -> fix-up -> true residual.
cudaError_t enqueue_persistent(gmaf_ctx* ctx, const GraphKey& key, cudaStream_t s) {
  cudaError_t e = enqueue_init(ctx, key, 0ull, s);
  if (e == cudaSuccess) e = launch_sr_persistent(ctx->gp, ctx->d, ctx->tiles_sr, ctx->K, key.precond, s);
  if (e == cudaSuccess) e = enqueue_final(ctx, key, s);
  return e;
}

gmaf_status build_graph(gmaf_ctx* ctx, const GraphKey& key, cudaGraphExec_t* out) {
  auto it = ctx->graphs.find(key);
  if (it != ctx->graphs.end()) { *out = it->second.second; return GMAF_OK; }
  cudaGraph_t graph = nullptr;
  CU(cudaGraphCreate(&graph, 0));
  if (use_persistent(ctx, key)) {
    cudaStream_t cs = ctx->cap_stream;
    CU(cudaStreamBeginCaptureToGraph(cs, graph, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    cudaError_t le = enqueue_persistent(ctx, key, cs);
    cudaGraph_t g2 = nullptr;
    cudaError_t ee = cudaStreamEndCapture(cs, &g2);
    CU(le);
    CU(ee);
    cudaGraphExec_t exec = nullptr;
    CU(cudaGraphInstantiate(&exec, graph, 0));
    ctx->graphs[key] = {graph, exec};
    *out = exec;
    return GMAF_OK;
  }
  cudaGraphConditionalHandle handle;
  CU(cudaGraphConditionalHandleCreate(&handle, graph, 1, cudaGraphCondAssignDefault));
  cudaStream_t cs = ctx->cap_stream;
  CU(cudaStreamBeginCaptureToGraph(cs, graph, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  cudaError_t le = enqueue_init(ctx, key, (unsigned long long)handle, cs);
  cudaGraph_t g2 = nullptr;
  cudaError_t ee = cudaStreamEndCapture(cs, &g2);
  CU(le);
  CU(ee);
  // the init chain's leaf node
  size_t nn = 0;
  CU(cudaGraphGetNodes(graph, nullptr, &nn));
  std::vector<cudaGraphNode_t> nodes(nn);
  CU(cudaGraphGetNodes(graph, nodes.data(), &nn));
  cudaGraphNode_t leaf = nullptr;
  for (size_t q = 0; q < nn; ++q) {
    size_t nd = 0;
    CU(cudaGraphNodeGetDependentNodes(nodes[q], nullptr, &nd));
    if (nd == 0) leaf = nodes[q];
  }
  if (!leaf) return fail(ctx, GMAF_E_CUDA, "graph build: no init leaf");
  cudaGraphNodeParams cp{};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = handle;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t cond_node;
  CU(cudaGraphAddNode(&cond_node, graph, &leaf, 1, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  CU(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  cudaError_t lb = enqueue_iterations(ctx, key, (unsigned long long)handle, cs);
  ee = cudaStreamEndCapture(cs, &g2);
  CU(lb);
  CU(ee);
  CU(cudaStreamBeginCaptureToGraph(cs, graph, &cond_node, nullptr, 1, cudaStreamCaptureModeRelaxed));
  le = enqueue_final(ctx, key, cs);
  ee = cudaStreamEndCapture(cs, &g2);
  CU(le);
  CU(ee);
  cudaGraphExec_t exec = nullptr;
  CU(cudaGraphInstantiate(&exec, graph, 0));
  ctx->graphs[key] = {graph, exec};
  *out = exec;
  return GMAF_OK;
}

#define NC(call)                                                                              \
  do {                                                                                        \
    ncclResult_t r_ = (call);                                                                 \
    if (r_ != ncclSuccess)                                                                    \
      return fail(ctx, GMAF_E_NCCL, "%s:%d %s: %s", __FILE__, __LINE__, #call,                \
                  nccl_api().getErrorString(r_));                                             \
  } while (0)

// Multi-rank solve (condition sharding): every iteration = the single-pass
// kernel on the local conditions, ONE allgather of the packed per-condition sums
// (gamma_k, delta_k, r.r_k, S.S_k; 4 x kmax doubles per rank), and a one-CTA scalar kernel
// that evaluates Eq. 3.9 and alpha/beta in global condition order -- bitwise the same on
// every rank.  Iterations are enqueued in batches with one batch in flight; the host reads
// the device done flag of the previous batch (kernels after convergence are no-ops).
gmaf_status run_solve_dist(gmaf_ctx* ctx, int precond, int warm, gmaf_solve_stats* out, double* cond_rel) {
  NcclApi& N = nccl_api();
  const int K = ctx->K, km = ctx->kmax, W = ctx->world;
  const DevPtrs& d = ctx->d;
  cudaStream_t s = ctx->stream;
  SolverState* hs = ctx->h_state;
  CU(cudaMemcpyAsync(d.st_, hs, sizeof(SolverState), cudaMemcpyHostToDevice, s));
  CU(cudaEventRecord(ctx->ev0, s));
  if (warm) CU(launch_residual_init(ctx->gp, d, ctx->tiles, K, 1, s));
  CU(launch_sr_init(ctx->gp, d, ctx->tiles_sr, K, precond, warm != 0, 0ull, s));
  NC(N.allGather(d.dist.packed_local, d.dist.packed_all, (size_t)4 * km, ncclDouble, ctx->comm, s));
  CU(launch_sr_scalar(d, true, ctx->Kglob, K, ctx->kofs, W, s));
  double* h_init = ctx->h_packed + (size_t)4 * km * W;   // S.S_k of every condition (init sums)
  CU(cudaMemcpyAsync(h_init, d.dist.packed_all, (size_t)4 * km * W * 8, cudaMemcpyDeviceToHost, s));
  constexpr int kBatch = 8;   // even: iteration parity = position in the batch
  for (int b = 0;; ++b) {
    for (int u = 0; u < kBatch; ++u) {
      CU(launch_sr_iter(ctx->gp, d, ctx->tiles_sr, K, precond, u & 1, 0ull, s));
      NC(N.allGather(d.dist.packed_local, d.dist.packed_all, (size_t)4 * km, ncclDouble, ctx->comm, s));
      CU(launch_sr_scalar(d, false, ctx->Kglob, K, ctx->kofs, W, s));
    }
    CU(cudaMemcpyAsync(&ctx->h_done[b & 1], &d.st_->done, sizeof(int), cudaMemcpyDeviceToHost, s));
    CU(cudaEventRecord(ctx->evb[b & 1], s));
    if (b >= 1) {
      CU(cudaEventSynchronize(ctx->evb[(b - 1) & 1]));
      if (ctx->h_done[(b - 1) & 1]) break;
    }
  }
  CU(cudaMemcpyAsync(ctx->h_packed, d.dist.packed_all, (size_t)4 * km * W * 8, cudaMemcpyDeviceToHost, s));
  CU(launch_sr_fixup(ctx->gp, d, K, s));
  CU(launch_true_residual(ctx->gp, d, ctx->tiles, K, s));
  NC(N.allGather(d.dist.packed_local, d.dist.packed_all, (size_t)km, ncclDouble, ctx->comm, s));
  CU(launch_true_scalar(d, W, s));
  CU(cudaEventRecord(ctx->ev1, s));
  CU(cudaMemcpyAsync(hs, d.st_, sizeof(SolverState), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  float ms = 0.f;
  CU(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  if (hs->zero_p) {
    CU(cudaMemsetAsync(d.p, 0, (size_t)K * ctx->grid.n_theta * ctx->grid.n_y * 8, s));
    CU(cudaStreamSynchronize(s));
  }
  if (cond_rel) {
    for (int r = 0; r < W; ++r) {
      int lo, hi;
      shard(ctx->Kglob, W, r, &lo, &hi);
      for (int kl = 0; kl < hi - lo; ++kl) {
        const double rr = ctx->h_packed[(size_t)r * 4 * km + kl], ss = h_init[(size_t)r * 4 * km + 3 * km + kl];
        cond_rel[lo + kl] = ss > 0.0 ? std::sqrt(rr) / std::sqrt(ss) : 0.0;
      }
    }
  }
  if (out) {
    out->iterations = hs->iter; out->converged = hs->converged; out->status = hs->status;
    out->precond = precond; out->schedule = GMAF_SCHEDULE_SINGLE; out->rel_residual = hs->rel;
    out->true_rel_residual = hs->true_rel; out->solve_ms = ms;
  }
  ctx->r_parity = hs->iter & 1;
  ctx->state = ST_SOLVED;
  if (hs->status == GMAF_E_BREAKDOWN)
    return fail(ctx, GMAF_E_BREAKDOWN, "solve: breakdown at iteration %d", hs->iter);
  if (hs->status == GMAF_E_NO_CONVERGENCE)
    return fail(ctx, GMAF_E_NO_CONVERGENCE, "solve: no convergence after %d iterations (rel %.3e)", hs->iter,
                hs->rel);
  return GMAF_OK;
}

gmaf_status run_solve(gmaf_ctx* ctx, double tol, double omega, int precond, int coupling, int max_iter,
                      int warm, int fixed_iters, gmaf_solve_stats* out, double* cond_rel) {
  SolverState* hs = ctx->h_state;
  std::memset(hs, 0, sizeof(SolverState));
  hs->tol = tol;
  hs->omega = omega;
  hs->coupling = coupling;
  hs->max_iter = max_iter;
  hs->fixed_iters = fixed_iters;
  ctx->last_coupling = coupling;
  if (ctx->distm && !ctx->p2p) return run_solve_dist(ctx, precond, warm, out, cond_rel);
  if (ctx->p2p && !ctx->p2p_ready) return fail(ctx, GMAF_E_STATE, "solve: peer-to-peer context not connected");
  const GraphKey key{ctx->schedule, precond, warm ? 1 : 0, fixed_iters > 0 ? 1 : 0};
  CU(cudaMemcpyAsync(ctx->d.st_, hs, sizeof(SolverState), cudaMemcpyHostToDevice, ctx->stream));
  if (ctx->stream_mode) {
    // Plain stream launches (profilers cannot replay kernel nodes of conditional graphs):
    // the host polls the device done-flag every kUnroll iterations.
    CU(cudaEventRecord(ctx->ev0, ctx->stream));
    if (use_persistent(ctx, key)) {
      CU(enqueue_persistent(ctx, key, ctx->stream));
      CU(cudaEventRecord(ctx->ev1, ctx->stream));
    } else {
    CU(enqueue_init(ctx, key, 0ull, ctx->stream));
    for (;;) {
      CU(cudaMemcpyAsync(hs, ctx->d.st_, sizeof(SolverState), cudaMemcpyDeviceToHost, ctx->stream));
      CU(cudaStreamSynchronize(ctx->stream));
      if (hs->done) break;
      CU(enqueue_iterations(ctx, key, 0ull, ctx->stream));
    }
    CU(enqueue_final(ctx, key, ctx->stream));
    CU(cudaEventRecord(ctx->ev1, ctx->stream));
    }
  } else {
    cudaGraphExec_t exec = nullptr;
    gmaf_status gs = build_graph(ctx, key, &exec);
    if (gs != GMAF_OK) return gs;
    CU(cudaEventRecord(ctx->ev0, ctx->stream));
    CU(cudaGraphLaunch(exec, ctx->stream));
    CU(cudaEventRecord(ctx->ev1, ctx->stream));
  }
  CU(cudaMemcpyAsync(hs, ctx->d.st_, sizeof(SolverState), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaMemcpyAsync(ctx->h_cs, ctx->d.cs.alpha, (size_t)7 * ctx->K * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  float ms = 0.f;
  CU(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  if (hs->zero_p) {
    CU(cudaMemsetAsync(ctx->d.p, 0, (size_t)ctx->K * ctx->gp.ns * 8, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
  }
  const int K = ctx->K;
  const double* Sk = ctx->h_cs + 3 * K;
  const double* rrk = ctx->h_cs + 4 * K;
  if (cond_rel && ctx->p2p) {   // every condition of every rank (gathered on the device)
    std::vector<double> rs((size_t)2 * ctx->Kglob);
    CU(cudaMemcpy(rs.data(), ctx->d.dist.rr_all, rs.size() * 8, cudaMemcpyDeviceToHost));
    for (int k = 0; k < ctx->Kglob; ++k) {
      const double rr = rs[k], ss = rs[ctx->Kglob + k];
      cond_rel[k] = ss > 0.0 ? std::sqrt(rr) / std::sqrt(ss) : 0.0;
    }
  } else if (cond_rel) {
    for (int k = 0; k < K; ++k) cond_rel[k] = (Sk[k] > 0.0) ? std::sqrt(rrk[k]) / std::sqrt(Sk[k]) : 0.0;
  }
  if (out) {
    out->iterations = hs->iter;
    out->converged = hs->converged;
    out->status = hs->status;
    out->precond = precond;
    out->schedule = ctx->schedule;
    out->rel_residual = hs->rel;
    out->true_rel_residual = hs->true_rel;
    out->solve_ms = ms;
  }
  ctx->r_parity = hs->iter & 1;
  ctx->state = ST_SOLVED;
  if (hs->status == GMAF_E_CUDA)
    return fail(ctx, GMAF_E_CUDA, "solve: a peer rank did not arrive within the timeout (iteration %d)", hs->iter);
  if (hs->status == GMAF_E_BREAKDOWN)
    return fail(ctx, GMAF_E_BREAKDOWN, "solve: breakdown at iteration %d (u.v<=0 or r.z<=0)", hs->iter);
  if (hs->status == GMAF_E_NO_CONVERGENCE)
    return fail(ctx, GMAF_E_NO_CONVERGENCE, "solve: no convergence after %d iterations (rel %.3e)",
                hs->iter, hs->rel);
  return GMAF_OK;
}

}  // namespace

// Context accessors for the host-side Picard driver (picard.cu), which otherwise uses only
// the public ABI.
namespace gmaf {
int ctx_conditions(const gmaf_ctx* c) { return c ? c->K : 0; }
int ctx_world(const gmaf_ctx* c) { return c ? c->world : 0; }
gmaf_status ctx_fail(gmaf_ctx* c, gmaf_status code, const char* msg) { return fail(c, code, "%s", msg); }
}  // namespace gmaf

extern "C" {

const char* gmaf_version(void) { return "gmaf-b200 0.1 (sm_100a)"; }

size_t gmaf_workspace_bytes_m(const gmaf_grid* grid, int32_t K, int32_t max_matrices, const gmaf_dist* dist) {
  if (check_grid(grid) != GMAF_OK || K < 1) return 0;
  if (dist && (dist->world < 1 || dist->rank < 0 || dist->rank >= dist->world)) return 0;
  if (rows_mode(dist)) {
    if (dist->world > kMaxP2P || grid->n_y < 2 * SLAB_HALO * dist->world) return 0;
    const Slab sl = slab_of(grid->n_y, dist->world, dist->rank);
    return make_layout(grid, K, dist->world, K, sl.ye - sl.yb, max_matrices).total;
  }
  if (dist_mode(dist)) {
    if (dist->world > K) return 0;
    int lo, hi;
    shard(K, dist->world, dist->rank, &lo, &hi);
    return make_layout(grid, hi - lo, dist->world, (K + dist->world - 1) / dist->world, 0, max_matrices).total;
  }
  return make_layout(grid, K, 0, 0, 0, max_matrices).total;
}

size_t gmaf_workspace_bytes(const gmaf_grid* grid, int32_t K, const gmaf_dist* dist) {
  return gmaf_workspace_bytes_m(grid, K, 0, dist);
}

gmaf_status gmaf_create(const gmaf_grid* grid, int32_t K, const gmaf_dist* dist, void* d_workspace,
                        size_t ws_bytes, void* cuda_stream, gmaf_ctx** out) {
  if (!out) return GMAF_E_INVALID_ARG;
  *out = nullptr;
  int rc = check_grid(grid);
  if (rc != GMAF_OK) return (gmaf_status)rc;
  if (K < 1) return GMAF_E_INVALID_ARG;
  if (dist && (dist->world < 1 || dist->rank < 0 || dist->rank >= dist->world)) return GMAF_E_INVALID_ARG;
  const bool dm = dist_mode(dist);
  const bool rm = rows_mode(dist);
  int klo = 0, khi = K, world = 1, kmax = 0;
  Slab sl{0, grid->n_y, 0, grid->n_y};
  if (rm) {
    // row slabs: every rank holds all K conditions on its own rows (peer to peer, <= kMaxP2P
    // ranks, slabs of >= 2*SLAB_HALO rows, the single-pass schedule)
    if (dist->world > kMaxP2P || K > 256 || grid->n_theta % 2 != 0 || grid->n_theta < 12 ||
        grid->n_y < 2 * SLAB_HALO * dist->world)
      return GMAF_E_INVALID_ARG;
    world = dist->world;
    kmax = K;
    sl = slab_of(grid->n_y, world, dist->rank);
  } else if (dm) {
    // condition sharding needs the single-pass schedule and >= 1 condition per rank; without an
    // NCCL id it runs peer to peer (<= kMaxP2P ranks, connected by gmaf_p2p_connect)
    if (dist->world > K || grid->n_theta % 2 != 0 || grid->n_theta < 12) return GMAF_E_INVALID_ARG;
    const bool p2p = !dist->nccl_unique_id || dist->shard == GMAF_SHARD_CONDITIONS_P2P;
    if (p2p && (dist->world > kMaxP2P || K > 256)) return GMAF_E_INVALID_ARG;
    world = dist->world;
    shard(K, world, dist->rank, &klo, &khi);
    kmax = (K + world - 1) / world;
  }
  const int Kglob = K;
  K = khi - klo;   // from here on: the local conditions
  // multi-rank contexts run the single-pass kernel, whose reduction scratch (the dead rings,
  // 48 (tw + 8) doubles) must hold the 4 K per-condition sums
  if (dm && 4 * K > 48 * (tw_single(grid->n_theta) + 2 * SR_HALO_COLS)) return GMAF_E_INVALID_ARG;
  // the band storage the caller's workspace holds: the most distinct coefficient sets that fit
  auto layout_m = [&](int Mc) {
    return rm ? make_layout(grid, K, world, kmax, sl.ye - sl.yb, Mc)
         : dm ? make_layout(grid, K, world, kmax, 0, Mc) : make_layout(grid, K, 0, 0, 0, Mc);
  };
  int Mcap = K;
  while (Mcap > 1 && layout_m(Mcap).total > ws_bytes) --Mcap;
  const Layout L = layout_m(Mcap);
  if (!d_workspace || ws_bytes < L.total || (reinterpret_cast<uintptr_t>(d_workspace) % kAlign) != 0)
    return GMAF_E_WORKSPACE;
  gmaf_ctx* ctx = new (std::nothrow) gmaf_ctx();
  if (!ctx) return GMAF_E_INVALID_ARG;
  ctx->grid = *grid;
  ctx->K = K;
  ctx->Kglob = Kglob;
  ctx->distm = dm;
  ctx->p2p = dm && (!dist->nccl_unique_id || dist->shard == GMAF_SHARD_CONDITIONS_P2P || rm);
  ctx->rows = rm;
  ctx->world = world;
  ctx->rank = dm ? dist->rank : 0;
  ctx->kofs = klo;
  ctx->kmax = kmax;
  ctx->stream = reinterpret_cast<cudaStream_t>(cuda_stream);
  ctx->ws = reinterpret_cast<char*>(d_workspace);
  ctx->ws_bytes = ws_bytes;
  ctx->L = L;
  ctx->Mcap = Mcap;
  GridParams& gp = ctx->gp;
  gp.nt = grid->n_theta; gp.ny = grid->n_y; gp.Rk = grid->R_k; gp.Rc = grid->R_c; gp.mu = grid->mu;
  gp.hmin = grid->h_min;
  gp.twelve_mu = 12.0 * grid->mu;
  gp.dtheta = (2.0 * M_PI) / (double)grid->n_theta;
  const bool tex = grid->tex_n_theta > 0 && grid->tex_n_y > 0;
  gp.tex_nt = tex ? grid->tex_n_theta : 0; gp.tex_ny = tex ? grid->tex_n_y : 0;
  gp.tex_band = tex ? grid->tex_band_rows : 0; gp.tex_num = grid->tex_fill_num;
  gp.tex_den = grid->tex_fill_den > 0 ? grid->tex_fill_den : 1; gp.tex_depth = grid->tex_depth;
  gp.y0 = sl.y0; gp.y1 = sl.y1; gp.yb = sl.yb;
  gp.diag = 0;   // set below once the tiles are known
  gp.ns = (long long)grid->n_theta * (sl.ye - sl.yb);
  DevPtrs& d = ctx->d;
  d.ct = at<double>(ctx, L.off_ct); d.st = at<double>(ctx, L.off_st);
  d.cth = at<double>(ctx, L.off_cth); d.sth = at<double>(ctx, L.off_sth);
  d.cp = at<CondParams>(ctx, L.off_cp);
  d.AP = at<double>(ctx, L.off_AP); d.AE = at<double>(ctx, L.off_AE); d.AN = at<double>(ctx, L.off_AN);
  d.S = at<double>(ctx, L.off_S); d.p = at<double>(ctx, L.off_p);
  d.r[0] = at<double>(ctx, L.off_r); d.r[1] = at<double>(ctx, L.off_r2);
  d.u[0] = at<double>(ctx, L.off_u); d.u[1] = at<double>(ctx, L.off_u2);
  d.scratch = at<double>(ctx, L.off_scratch);
  d.zero_row = at<double>(ctx, L.off_constrows);
  d.one_row = d.zero_row + kConstRowLen;
  d.partials = at<double>(ctx, L.off_part); d.wrench_part = at<double>(ctx, L.off_wpart);
  d.wrench = at<double>(ctx, L.off_wrench); d.st_ = at<SolverState>(ctx, L.off_state);
  double* cs = at<double>(ctx, L.off_cs);
  d.cs.alpha = cs; d.cs.beta = cs + K; d.cs.dk = cs + 2 * K; d.cs.Sk = cs + 3 * K; d.cs.rrk = cs + 4 * K;
  d.cs.uvk = cs + 5 * K; d.cs.ttk = cs + 6 * K;
  d.cs.itk = reinterpret_cast<int32_t*>(cs + 7 * K); d.cs.frz = d.cs.itk + K;
  d.counters = at<unsigned int>(ctx, L.off_counters);
  d.timing = at<Timing>(ctx, L.off_timing);
  d.guard = at<unsigned long long>(ctx, L.off_guard);
  d.mat_rep = at<int32_t>(ctx, L.off_matrep);
  d.dist.world = dm ? world : 0;
  d.dist.rank = ctx->rank;
  d.dist.kofs = klo;
  d.dist.kmax_local = kmax;
  d.dist.packed_local = at<double>(ctx, L.off_plocal);
  d.dist.packed_all = at<double>(ctx, L.off_pall);

  auto cleanup_fail = [&](gmaf_status s) {
    const cudaError_t ce = cudaGetLastError();
    char buf[256];
    std::snprintf(buf, sizeof(buf), "create: status %d (last CUDA error: %s)", (int)s, cudaGetErrorString(ce));
    g_create_err = buf;
    gmaf_destroy(ctx);
    return s;
  };
  if (cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreate(&ctx->ev0) != cudaSuccess || cudaEventCreate(&ctx->ev1) != cudaSuccess ||
      cudaMallocHost((void**)&ctx->h_state, sizeof(SolverState)) != cudaSuccess ||
      cudaMallocHost((void**)&ctx->h_cs, (size_t)7 * K * 8) != cudaSuccess ||
      cudaMallocHost((void**)&ctx->h_wrench, (size_t)K * 12 * 8) != cudaSuccess ||
      cudaMallocHost((void**)&ctx->h_guard, 4 * sizeof(unsigned long long)) != cudaSuccess ||
      cudaMallocHost((void**)&ctx->h_cp, (size_t)K * sizeof(CondParams)) != cudaSuccess ||
      cudaMallocHost((void**)&ctx->h_timing, sizeof(Timing)) != cudaSuccess)
    return cleanup_fail(GMAF_E_CUDA);
  // cos/sin tables with the host libm (shared by nobody: the oracle computes its own)
  const int nt = grid->n_theta;
  std::vector<double> tab((size_t)4 * nt);
  std::vector<double> ones(kConstRowLen, 1.0);
  for (int i = 0; i < nt; ++i) {
    const double th = (double)i * gp.dtheta;
    const double thc = ((double)i + 0.5) * gp.dtheta;
    tab[i] = std::cos(th); tab[nt + i] = std::sin(th);
    tab[2 * nt + i] = std::cos(thc); tab[3 * nt + i] = std::sin(thc);
  }
  if (cudaMemcpyAsync((void*)d.ct, tab.data(), nt * 8, cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess ||
      cudaMemcpyAsync((void*)d.st, tab.data() + nt, nt * 8, cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess ||
      cudaMemcpyAsync((void*)d.cth, tab.data() + 2 * nt, nt * 8, cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess ||
      cudaMemcpyAsync((void*)d.sth, tab.data() + 3 * nt, nt * 8, cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess ||
      cudaMemsetAsync(d.counters, 0, 16 * sizeof(unsigned int), ctx->stream) != cudaSuccess ||
      cudaMemsetAsync(d.st_, 0, sizeof(SolverState), ctx->stream) != cudaSuccess ||
      cudaMemsetAsync((void*)d.cs.alpha, 0, (size_t)9 * K * 8, ctx->stream) != cudaSuccess ||
      cudaMemsetAsync(d.p, 0, (size_t)K * gp.ns * 8, ctx->stream) != cudaSuccess ||
      cudaMemsetAsync((void*)d.zero_row, 0, kConstRowLen * 8, ctx->stream) != cudaSuccess ||
      cudaMemcpyAsync((void*)d.one_row, ones.data(), kConstRowLen * 8, cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess)
    return cleanup_fail(GMAF_E_CUDA);
  std::memset(ctx->h_timing, 0, sizeof(Timing));
  for (int q = 0; q < KK_COUNT; ++q) ctx->h_timing->t_start[q] = ~0ull;
  if (cudaMemcpyAsync(d.timing, ctx->h_timing, sizeof(Timing), cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess)
    return cleanup_fail(GMAF_E_CUDA);
  {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      return cleanup_fail(GMAF_E_CUDA);
    TileCfg probe = make_tiles(grid->n_theta, sl.y1 - sl.y0, K, 1, tw_table1(grid->n_theta));
    if (configure_pcg_kernels(probe, K) != cudaSuccess) return cleanup_fail(GMAF_E_CUDA);
    const int occ = pcg_ctas_per_sm(probe, K);
    ctx->tiles = make_tiles(grid->n_theta, sl.y1 - sl.y0, K, sms * (occ > 0 ? occ : 1), tw_table1(grid->n_theta));
    if (ctx->tiles.n_tiles > kMaxTilesPerCondition) return cleanup_fail(GMAF_E_INVALID_MESH);
    if (configure_pcg_kernels(ctx->tiles, K) != cudaSuccess) return cleanup_fail(GMAF_E_CUDA);
    // single-pass kernel: its own tiles (wider halo, TMA ring) and occupancy
    TileCfg sprobe = make_tiles(grid->n_theta, sl.y1 - sl.y0, K, 1, tw_single(grid->n_theta));
    if (configure_sr_kernels(sprobe, K) != cudaSuccess) return cleanup_fail(GMAF_E_CUDA);
    const int socc = sr_ctas_per_sm(sprobe);
    ctx->tiles_sr = make_tiles(grid->n_theta, sl.y1 - sl.y0, K, sms * (socc > 0 ? socc : 1), tw_single(grid->n_theta));
    if (ctx->tiles_sr.n_tiles > kMaxTilesPerCondition) return cleanup_fail(GMAF_E_INVALID_MESH);
    if (std::getenv("GMAF_DEBUG"))
      std::fprintf(stderr, "gmaf: sms %d | two-phase occ %d tiles %dx%d tw %d th %d | single occ %d tiles %dx%d tw %d th %d\n",
                   sms, occ, ctx->tiles.n_strips, ctx->tiles.n_chunks, ctx->tiles.tw, ctx->tiles.th, socc,
                   ctx->tiles_sr.n_strips, ctx->tiles_sr.n_chunks, ctx->tiles_sr.tw, ctx->tiles_sr.th);
    // the single-pass kernel streams rows with 16-byte TMA copies: needs an even n_theta
    // (and its reduction scratch -- the dead rings, 48 (tw + 8) doubles -- must hold 4 K sums)
    ctx->sr_k_ok = 4 * K <= 48 * (tw_single(grid->n_theta) + 2 * SR_HALO_COLS);
    ctx->schedule = single_ok(grid->n_theta) && ctx->sr_k_ok ? GMAF_SCHEDULE_SINGLE : GMAF_SCHEDULE_TABLE1;
    const char* sch = std::getenv("GMAF_SCHEDULE");
    if (sch && std::strcmp(sch, "table1") == 0) ctx->schedule = GMAF_SCHEDULE_TABLE1;
    // persistent single-pass solve (one rank): needs every CTA of the one-wave grid resident
    // with the persistent kernel's extra shared memory (GMAF_PERSIST=0 selects the per-iteration
    // kernels inside the graph's WHILE loop)
    const char* pe = std::getenv("GMAF_PERSIST");
    const bool want = !(pe && std::strcmp(pe, "0") == 0);
    // (multi-rank: the peer-to-peer contexts, whose exchange runs inside the kernel; the NCCL
    // path keeps its host-driven loop)
    const bool p2p_ctx = dm && (!dist->nccl_unique_id || dist->shard == GMAF_SHARD_CONDITIONS_P2P || rm);
    const int Kall = (dm && !rm) ? Kglob : K;
    ctx->persist_ok = want && (!dm || p2p_ctx) && single_ok(grid->n_theta) && ctx->sr_k_ok &&
                      srp_fits(ctx->tiles_sr, K, Kall) &&
                      (long long)srp_ctas_per_sm(ctx->tiles_sr, K, Kall) * sms >= (long long)ctx->tiles_sr.n_tiles * K;
    // diagnostics (gmaf_cta_arrivals): the arrival stamps live at the end of the partials region,
    // clear of every kernel's partial sums (diag_offset)
    gp.diag = (std::getenv("GMAF_DIAG") && ctx->persist_ok &&
               diag_offset(K, ctx->tiles_sr.n_tiles * K) >=
                   (long long)8 * K * std::max(ctx->tiles_sr.n_tiles, ctx->tiles.n_tiles)) ? 1 : 0;
  }
  if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return cleanup_fail(GMAF_E_CUDA);
  ctx->quad_ctas = quad_ctas_per_condition(gp, K);
  if (dm && ctx->p2p) {
    const size_t xs = (size_t)12 * kmax;
    size_t bytes = (size_t)2 * world * 8 + (size_t)2 * world * xs * 8 + 8 + (size_t)2 * Kglob * 8;
    if (rm) {   // halo inboxes [2 slots][2 sides][2 vectors][K][SLAB_HALO][nt]
      ctx->inbox_off = align_up(bytes);
      bytes = ctx->inbox_off + (size_t)8 * SLAB_HALO * K * grid->n_theta * 8;
    }
    // a whole 2 MiB granule: a small cudaMalloc can be sub-allocated inside a larger driver
    // allocation, and cudaIpcOpenMemHandle maps the ALLOCATION's base, not this pointer
    bytes = (bytes + (2u << 20) - 1) / (2u << 20) * (2u << 20);
    if (cudaMalloc((void**)&ctx->p2p_buf, bytes) != cudaSuccess ||
        cudaMemsetAsync(ctx->p2p_buf, 0, bytes, ctx->stream) != cudaSuccess ||
        cudaMallocHost((void**)&ctx->h_packed, (size_t)2 * 4 * kmax * world * 8) != cudaSuccess ||
        cudaMallocHost((void**)&ctx->h_wall, (size_t)12 * kmax * world * 8) != cudaSuccess ||
        cudaStreamSynchronize(ctx->stream) != cudaSuccess)
      return cleanup_fail(GMAF_E_CUDA);
    DistPtrs& dd = ctx->d.dist;
    dd.p2p = 1;
    dd.xs = (int)xs;
    dd.kglob = Kglob;
    dd.peer[ctx->rank] = ctx->p2p_buf;
    char* tail = ctx->p2p_buf + (size_t)2 * world * 8 + (size_t)2 * world * xs * 8;
    dd.seq = reinterpret_cast<unsigned long long*>(tail);
    dd.rr_all = reinterpret_cast<double*>(tail + 8);
    dd.ss_all = dd.rr_all + Kglob;
    if (rm) {
      const char* up = std::getenv("GMAF_ROWS_UNPACK");
      dd.rows = (up && std::atoi(up) != 0) ? 2 : 1;
      dd.halo_in[ctx->rank] = reinterpret_cast<double*>(ctx->p2p_buf + ctx->inbox_off);
    }
  } else if (dm) {
    NcclApi& N = nccl_api();
    if (!N.ok) { gmaf_status e = fail(ctx, GMAF_E_NCCL, "NCCL unavailable: %s", N.err.c_str()); gmaf_destroy(ctx); return e; }
    if (cudaMallocHost((void**)&ctx->h_packed, (size_t)2 * 4 * kmax * world * 8) != cudaSuccess ||
        cudaMallocHost((void**)&ctx->h_wall, (size_t)12 * kmax * world * 8) != cudaSuccess ||
        cudaMallocHost((void**)&ctx->h_done, 2 * sizeof(int)) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->evb[0], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->evb[1], cudaEventDisableTiming) != cudaSuccess)
      return cleanup_fail(GMAF_E_CUDA);
    ncclUniqueId uid;
    std::memcpy(&uid, dist->nccl_unique_id, sizeof(uid));
    if (N.commInitRank(&ctx->comm, world, uid, ctx->rank) != ncclSuccess) {
      ctx->comm = nullptr;
      return cleanup_fail(GMAF_E_NCCL);
    }
  }
  const char* lm = std::getenv("GMAF_LAUNCH_MODE");
  ctx->stream_mode = lm && std::strcmp(lm, "stream") == 0;
  *out = ctx;
  return GMAF_OK;
}

gmaf_status gmaf_destroy(gmaf_ctx* ctx) {
  if (!ctx) return GMAF_E_INVALID_ARG;
  if (ctx->comm) nccl_api().commDestroy(ctx->comm);
  for (int r = 0; r < kMaxP2P; ++r)
    if (ctx->peer_bufs[r]) cudaIpcCloseMemHandle(ctx->peer_bufs[r]);
  if (ctx->p2p_buf) cudaFree(ctx->p2p_buf);
  if (ctx->h_packed) cudaFreeHost(ctx->h_packed);
  if (ctx->h_wall) cudaFreeHost(ctx->h_wall);
  if (ctx->h_done) cudaFreeHost(ctx->h_done);
  for (int q = 0; q < 2; ++q) if (ctx->evb[q]) cudaEventDestroy(ctx->evb[q]);
  for (auto& kv : ctx->graphs) {
    if (kv.second.second) cudaGraphExecDestroy(kv.second.second);
    if (kv.second.first) cudaGraphDestroy(kv.second.first);
  }
  if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  if (ctx->h_state) cudaFreeHost(ctx->h_state);
  if (ctx->h_cs) cudaFreeHost(ctx->h_cs);
  if (ctx->h_wrench) cudaFreeHost(ctx->h_wrench);
  if (ctx->h_guard) cudaFreeHost(ctx->h_guard);
  if (ctx->h_cp) cudaFreeHost(ctx->h_cp);
  if (ctx->h_timing) cudaFreeHost(ctx->h_timing);
  delete ctx;
  return GMAF_OK;
}

gmaf_status gmaf_thickness(gmaf_ctx* ctx, const gmaf_condition* conds_all) {
  if (!ctx || !conds_all) return GMAF_E_INVALID_ARG;
  const gmaf_condition* conds = conds_all + ctx->kofs;   // this rank's block (all K on every rank)
  const int K = ctx->K;
  ctx->mat_of.assign(K, 0);
  ctx->mat_rep.clear();
  for (int k = 0; k < K; ++k) {
    if (!(conds[k].L_F > 0.0)) return fail(ctx, GMAF_E_INVALID_ARG, "thickness: k=%d L_F <= 0", k);
    int m = -1;
    for (int q = 0; q < (int)ctx->mat_rep.size(); ++q)
      if (same_matrix(conds[ctx->mat_rep[q]], conds[k])) { m = q; break; }
    if (m < 0) { m = (int)ctx->mat_rep.size(); ctx->mat_rep.push_back(k); }
    ctx->mat_of[k] = m;
    ctx->h_cp[k] = cond_params(ctx->grid, conds[k], m);
  }
  ctx->M = (int)ctx->mat_rep.size();
  ctx->state = ST_CREATED;
  if (ctx->M > ctx->Mcap)
    return fail(ctx, GMAF_E_WORKSPACE, "thickness: %d distinct coefficient sets (distinct (e, L_F)), the workspace "
                "holds %d (gmaf_workspace_bytes_m)", ctx->M, ctx->Mcap);
  CU(cudaMemcpyAsync((void*)ctx->d.cp, ctx->h_cp, (size_t)K * sizeof(CondParams), cudaMemcpyHostToDevice,
                     ctx->stream));
  CU(cudaMemcpyAsync(ctx->d.mat_rep, ctx->mat_rep.data(), (size_t)ctx->M * sizeof(int32_t),
                     cudaMemcpyHostToDevice, ctx->stream));
  CU(cudaMemsetAsync(ctx->d.guard, 0, 4 * sizeof(unsigned long long), ctx->stream));
  CU(launch_thickness_guard(ctx->gp, ctx->d, K, ctx->stream));
  CU(cudaMemcpyAsync(ctx->h_guard, ctx->d.guard, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                     ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  if (ctx->h_guard[0]) {
    double h;
    const unsigned long long bits = ctx->h_guard[3];
    std::memcpy(&h, &bits, sizeof(h));
    const int i = (int)(ctx->h_guard[2] >> 32), j = (int)(ctx->h_guard[2] & 0xffffffffu) - 1;
    return fail(ctx, GMAF_E_NONPOSITIVE_THICKNESS, "thickness: k=%d i=%d j=%d h=%.6e < h_min=%.3e",
                (int)ctx->h_guard[1], i, j, h, ctx->grid.h_min);
  }
  ctx->state = ST_THICK;
  return GMAF_OK;
}

gmaf_status gmaf_assemble(gmaf_ctx* ctx) {
  if (!ctx) return GMAF_E_INVALID_ARG;
  if (ctx->state < ST_THICK) return fail(ctx, GMAF_E_STATE, "assemble before thickness");
  CU(launch_assemble(ctx->gp, ctx->d, ctx->K, ctx->stream));
  ctx->state = ST_ASSEMBLED;
  return GMAF_OK;
}

gmaf_status gmaf_solve(gmaf_ctx* ctx, double tol, double omega, int32_t precond, int32_t coupling,
                       int32_t max_iter, int32_t warm_start, gmaf_solve_stats* out, double* cond_rel) {
  if (!ctx) return GMAF_E_INVALID_ARG;
  if (ctx->state < ST_ASSEMBLED) return fail(ctx, GMAF_E_STATE, "solve before assemble");
  if (coupling == GMAF_ASYNC && (ctx->schedule != GMAF_SCHEDULE_SINGLE || ctx->distm))
    return fail(ctx, GMAF_E_INVALID_ARG, "solve: the asynchronous strategy runs on the single-pass schedule, one rank");
  if (precond == GMAF_PRECOND_ASSOR1 && ctx->schedule != GMAF_SCHEDULE_SINGLE)
    return fail(ctx, GMAF_E_INVALID_ARG, "solve: ASSOR-I runs on the single-pass schedule only");
  if (!(tol >= 0.0) || !(omega > 0.0 && omega < 2.0) || precond < 0 || precond > 3 || coupling < 0 ||
      coupling > 2 || max_iter < 0)
    return fail(ctx, GMAF_E_INVALID_ARG, "solve: invalid tol/omega/precond/coupling/max_iter");
  return run_solve(ctx, tol, omega, precond, coupling, max_iter, warm_start, 0, out, cond_rel);
}

gmaf_status gmaf_solve_fixed(gmaf_ctx* ctx, double omega, int32_t precond, int32_t n_iter,
                             gmaf_solve_stats* out) {
  if (!ctx) return GMAF_E_INVALID_ARG;
  if (ctx->state < ST_ASSEMBLED) return fail(ctx, GMAF_E_STATE, "solve before assemble");
  if (precond == GMAF_PRECOND_ASSOR1 && ctx->schedule != GMAF_SCHEDULE_SINGLE)
    return fail(ctx, GMAF_E_INVALID_ARG, "solve_fixed: ASSOR-I runs on the single-pass schedule only");
  if (n_iter < 1 || !(omega > 0.0 && omega < 2.0) || precond < 0 || precond > 3)
    return fail(ctx, GMAF_E_INVALID_ARG, "solve_fixed: invalid arguments");
  return run_solve(ctx, 0.0, omega, precond, 0, n_iter, 0, n_iter, out, nullptr);
}

gmaf_status gmaf_integrate(gmaf_ctx* ctx, double* wrench) {
  if (!ctx || !wrench) return GMAF_E_INVALID_ARG;
  if (ctx->state < ST_SOLVED) return fail(ctx, GMAF_E_STATE, "integrate before solve");
  CU(launch_quadrature(ctx->gp, ctx->d, ctx->K, ctx->stream, nullptr));
  if (ctx->distm) {   // every rank returns all K wrenches (allgather of the padded blocks)
    const int km = ctx->kmax;
    double* wall = reinterpret_cast<double*>(ctx->ws + ctx->L.off_wall);
    if (ctx->p2p) CU(launch_p2p_gather(ctx->d, ctx->d.wrench, 12 * km, wall, ctx->stream));
    else NC(nccl_api().allGather(ctx->d.wrench, wall, (size_t)12 * km, ncclDouble, ctx->comm, ctx->stream));
    CU(cudaMemcpyAsync(ctx->h_wall, wall, (size_t)12 * km * ctx->world * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    if (ctx->rows) {   // row slabs: every rank integrated its own cells of all K; sum in rank order
      for (int q = 0; q < 12 * ctx->K; ++q) {
        double acc = 0.0;
        for (int r = 0; r < ctx->world; ++r) acc += ctx->h_wall[(size_t)r * 12 * km + q];
        wrench[q] = acc;
      }
      return GMAF_OK;
    }
    for (int r = 0; r < ctx->world; ++r) {
      int lo, hi;
      shard(ctx->Kglob, ctx->world, r, &lo, &hi);
      std::memcpy(wrench + (size_t)lo * 12, ctx->h_wall + (size_t)r * 12 * km, (size_t)(hi - lo) * 12 * 8);
    }
    return GMAF_OK;
  }
  CU(cudaMemcpyAsync(ctx->h_wrench, ctx->d.wrench, (size_t)ctx->K * 12 * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  std::memcpy(wrench, ctx->h_wrench, (size_t)ctx->K * 12 * 8);
  return GMAF_OK;
}

gmaf_status gmaf_field_ptr(gmaf_ctx* ctx, int32_t field, int32_t kglob, void** dptr) {
  if (!ctx || !dptr) return GMAF_E_INVALID_ARG;
  const int32_t k = kglob - ctx->kofs;   // fields of this rank's conditions only
  if (k < 0 || k >= ctx->K) return fail(ctx, GMAF_E_INVALID_ARG, "condition %d is not on this rank", kglob);
  const GridParams& g = ctx->gp;
  const int m = ctx->mat_of.empty() ? 0 : ctx->mat_of[k];
  // the own rows [y0, y1) of the field (all rows on one rank), contiguous
  const long long ok = fofs(g, k) + (long long)g.y0 * g.nt, om = fofs(g, m) + (long long)g.y0 * g.nt;
  switch (field) {
    case GMAF_FIELD_P: *dptr = ctx->d.p + ok; break;
    case GMAF_FIELD_S: *dptr = ctx->d.S + ok; break;
    case GMAF_FIELD_R: *dptr = ctx->d.r[ctx->r_parity] + ok; break;   // latest residual
    case GMAF_FIELD_AP: *dptr = ctx->d.AP + om; break;
    case GMAF_FIELD_AE: *dptr = ctx->d.AE + om; break;
    case GMAF_FIELD_AN: *dptr = ctx->d.AN + om; break;
    default: return fail(ctx, GMAF_E_INVALID_ARG, "field_ptr: field %d has no persistent buffer", field);
  }
  return GMAF_OK;
}

gmaf_status gmaf_get(gmaf_ctx* ctx, int32_t field, int32_t kglob, double* host_out) {
  if (!ctx || !host_out) return GMAF_E_INVALID_ARG;
  const int32_t k = kglob - ctx->kofs;
  if (k < 0 || k >= ctx->K) return fail(ctx, GMAF_E_INVALID_ARG, "condition %d is not on this rank", kglob);
  if (field == GMAF_FIELD_H || field == GMAF_FIELD_HDOT) {
    if (ctx->state < ST_THICK) return fail(ctx, GMAF_E_STATE, "get H before thickness");
    CU(launch_field(ctx->gp, ctx->d, field, k, ctx->stream));
    CU(cudaMemcpyAsync(host_out, ctx->d.scratch, (size_t)(ctx->grid.n_y + 2) * ctx->grid.n_theta * 8,
                       cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return GMAF_OK;
  }
  if ((field == GMAF_FIELD_AP || field == GMAF_FIELD_AE || field == GMAF_FIELD_AN || field == GMAF_FIELD_S) &&
      ctx->state < ST_ASSEMBLED)
    return fail(ctx, GMAF_E_STATE, "get bands before assemble");
  void* src = nullptr;
  gmaf_status s = gmaf_field_ptr(ctx, field, kglob, &src);
  if (s != GMAF_OK) return s;
  // row slabs: the own rows land at their global position; the other rows are not written
  const size_t own = (size_t)ctx->grid.n_theta * (ctx->gp.y1 - ctx->gp.y0);
  CU(cudaMemcpyAsync(host_out + (size_t)ctx->gp.y0 * ctx->grid.n_theta, src, own * 8, cudaMemcpyDeviceToHost,
                     ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return GMAF_OK;
}

gmaf_status gmaf_kernel_times(gmaf_ctx* ctx, gmaf_kernel_timing* out, int32_t n, int32_t* count) {
  if (!ctx || !out || !count) return GMAF_E_INVALID_ARG;
  CU(cudaMemcpyAsync(ctx->h_timing, ctx->d.timing, sizeof(Timing), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  static const char* names[KK_COUNT] = {"thickness_guard", "assemble", "pcg_init", "pcg_phase_a",
                                        "pcg_phase_b", "true_residual", "quadrature", "sr_init", "sr_iter",
                                        "tail_of_sr_iter", "gridbar_wait"};
  const double rows = (double)(ctx->gp.y1 - ctx->gp.y0);   // own rows (all n_y on one rank)
  const double n_nodes = (double)ctx->grid.n_theta * rows * ctx->K;
  const double nM = (double)ctx->grid.n_theta * rows * (ctx->M > 0 ? ctx->M : ctx->K);
  // algorithmic DRAM bytes per launch: 8 B per node per field touched;
  // the coefficient bands count once per DISTINCT matrix (M of them).
  const double bytes[KK_COUNT] = {
      0.0,                                  // guard: pure compute
      8.0 * (n_nodes + 3.0 * nM),           // assemble: write S (K) + 3 bands (M)
      8.0 * (3.0 * n_nodes + 3.0 * nM),     // init: read S, write r, p; 3 bands
      8.0 * (3.0 * n_nodes + 3.0 * nM),     // A: read r, u_old, write u; 3 bands
      8.0 * (5.0 * n_nodes + 3.0 * nM),     // B: read p, u, r; write p, r; 3 bands
      8.0 * (2.0 * n_nodes + 3.0 * nM),     // true residual: read S, p; 3 bands
      8.0 * n_nodes,                        // quadrature: read p
      8.0 * (2.0 * n_nodes + 3.0 * nM),     // sr_init: read S, write r (x zeroed: +1)
      8.0 * (5.0 * n_nodes + 3.0 * nM),     // sr_iter: r RW, pd RW, x RW every other; 3 bands
      0.0,                                  // serial tail of sr_iter (inside its time)
      0.0};                                 // persistent: CTA 0's wait at the grid barrier
  int c = 0;
  for (int q = 0; q < KK_COUNT && c < n; ++q, ++c) {
    std::memset(&out[c], 0, sizeof(gmaf_kernel_timing));
    std::snprintf(out[c].name, sizeof(out[c].name), "%s", names[q]);
    out[c].launches = (int64_t)ctx->h_timing->launches[q];
    out[c].total_ms = (double)ctx->h_timing->total_ns[q] * 1e-6;
    out[c].bytes_per_launch = bytes[q];
  }
  *count = c;
  return GMAF_OK;
}

gmaf_status gmaf_reset_kernel_times(gmaf_ctx* ctx) {
  if (!ctx) return GMAF_E_INVALID_ARG;
  std::memset(ctx->h_timing, 0, sizeof(Timing));
  for (int q = 0; q < KK_COUNT; ++q) ctx->h_timing->t_start[q] = ~0ull;
  CU(cudaMemcpyAsync(ctx->d.timing, ctx->h_timing, sizeof(Timing), cudaMemcpyHostToDevice, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return GMAF_OK;
}

gmaf_status gmaf_set_schedule(gmaf_ctx* ctx, int32_t schedule) {
  if (!ctx) return GMAF_E_INVALID_ARG;
  if (ctx->distm && schedule != GMAF_SCHEDULE_SINGLE)
    return fail(ctx, GMAF_E_INVALID_ARG, "set_schedule: multi-rank contexts run the single-pass schedule");
  if (schedule == GMAF_SCHEDULE_TABLE1) { ctx->schedule = schedule; return GMAF_OK; }
  if (schedule == GMAF_SCHEDULE_SINGLE && single_ok(ctx->grid.n_theta) && ctx->sr_k_ok) {
    ctx->schedule = schedule;
    return GMAF_OK;
  }
  return fail(ctx, GMAF_E_INVALID_ARG, "set_schedule: %d not available (n_theta %d)", schedule, ctx->grid.n_theta);
}

gmaf_status gmaf_cond_iterations(gmaf_ctx* ctx, int32_t* out) {
  if (!ctx || !out) return GMAF_E_INVALID_ARG;
  if (ctx->state < ST_SOLVED) return fail(ctx, GMAF_E_STATE, "cond_iterations before solve");
  std::vector<int32_t> tmp((size_t)ctx->K);
  CU(cudaMemcpyAsync(tmp.data(), ctx->d.cs.itk, (size_t)ctx->K * sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  for (int k = 0; k < ctx->K; ++k) out[k] = ctx->last_coupling == GMAF_ASYNC ? tmp[k] : ctx->h_state->iter;
  return GMAF_OK;
}

gmaf_status gmaf_p2p_handle(gmaf_ctx* ctx, void* out) {
  if (!ctx || !out) return GMAF_E_INVALID_ARG;
  if (!ctx->p2p) return fail(ctx, GMAF_E_STATE, "p2p_handle: not a peer-to-peer context");
  cudaIpcMemHandle_t h;
  CU(cudaIpcGetMemHandle(&h, ctx->p2p_buf));
  std::memcpy(out, &h, sizeof(h));
  return GMAF_OK;
}

gmaf_status gmaf_p2p_connect(gmaf_ctx* ctx, const void* handles) {
  if (!ctx || !handles) return GMAF_E_INVALID_ARG;
  if (!ctx->p2p) return fail(ctx, GMAF_E_STATE, "p2p_connect: not a peer-to-peer context");
  if (ctx->p2p_ready) return fail(ctx, GMAF_E_STATE, "p2p_connect: already connected");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  for (int r = 0; r < ctx->world; ++r) {
    if (r == ctx->rank) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, static_cast<const char*>(handles) + 64 * r, 64);
    void* p = nullptr;
    CU(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    ctx->peer_bufs[r] = p;
    // the kernels load and store this buffer directly (NVLink peer memory): refuse loudly if the
    // owning GPU is not peer-accessible from this one (same GPU: always accessible)
    cudaPointerAttributes pa;
    CU(cudaPointerGetAttributes(&pa, p));
    int mydev = 0, can = 1;
    CU(cudaGetDevice(&mydev));
    if (pa.device != mydev) CU(cudaDeviceCanAccessPeer(&can, mydev, pa.device));
    if (!can)
      return fail(ctx, GMAF_E_CUDA, "p2p_connect: GPU %d cannot access rank %d's GPU %d peer to peer (NVLink/P2P "
                  "required by the peer-to-peer exchange)", mydev, r, pa.device);
    ctx->d.dist.peer[r] = static_cast<char*>(p);
    if (ctx->rows) ctx->d.dist.halo_in[r] = reinterpret_cast<double*>(static_cast<char*>(p) + ctx->inbox_off);
  }
  ctx->p2p_ready = true;
  return GMAF_OK;
}

gmaf_status gmaf_nccl_unique_id(void* out) {
  if (!out) return GMAF_E_INVALID_ARG;
  NcclApi& N = nccl_api();
  if (!N.ok) return GMAF_E_NCCL;
  ncclUniqueId uid;
  if (N.getUniqueId(&uid) != ncclSuccess) return GMAF_E_NCCL;
  std::memcpy(out, &uid, sizeof(uid));
  return GMAF_OK;
}

gmaf_status gmaf_slab_rows(int32_t n_y, int32_t world, int32_t rank, int32_t* y0, int32_t* y1,
                           int32_t* yb, int32_t* ye) {
  if (!y0 || !y1 || !yb || !ye || world < 1 || world > kMaxP2P || rank < 0 || rank >= world ||
      n_y < 2 * SLAB_HALO * world)
    return GMAF_E_INVALID_ARG;
  const Slab sl = slab_of(n_y, world, rank);
  *y0 = sl.y0; *y1 = sl.y1; *yb = sl.yb; *ye = sl.ye;
  return GMAF_OK;
}

gmaf_status gmaf_cta_arrivals(gmaf_ctx* ctx, uint64_t* out, int32_t n, int32_t* count) {
  if (!ctx || !out || !count) return GMAF_E_INVALID_ARG;
  *count = 0;
  if (!ctx->gp.diag || !ctx->persist_ok) return GMAF_OK;
  const int nblk = ctx->tiles_sr.n_tiles * ctx->K;
  const int m = kDiagIters * nblk < n ? kDiagIters * nblk : n;
  const double* base = ctx->d.partials + diag_offset(ctx->K, nblk);
  CU(cudaMemcpyAsync(out, base, (size_t)m * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  *count = m;
  return GMAF_OK;
}

gmaf_status gmaf_tile_config(const gmaf_ctx* ctx, gmaf_tiles* out) {
  if (!ctx || !out) return GMAF_E_INVALID_ARG;
  const bool single = ctx->schedule == GMAF_SCHEDULE_SINGLE;
  const TileCfg& t = single ? ctx->tiles_sr : ctx->tiles;
  out->tw = t.tw; out->th = t.th; out->n_strips = t.n_strips; out->n_chunks = t.n_chunks;
  out->n_ctas = t.n_tiles * ctx->K;
  out->schedule = ctx->schedule;
  out->persistent = (single && ctx->persist_ok && (!ctx->distm || ctx->p2p)) ? 1 : 0;
  out->pad = 0;
  return GMAF_OK;
}

gmaf_status gmaf_slab(const gmaf_ctx* ctx, int32_t* y0, int32_t* y1) {
  if (!ctx || !y0 || !y1) return GMAF_E_INVALID_ARG;
  *y0 = ctx->gp.y0;
  *y1 = ctx->gp.y1;
  return GMAF_OK;
}

const char* gmaf_last_error(const gmaf_ctx* ctx) {
  return ctx ? ctx->err.c_str() : (g_create_err.empty() ? "null context" : g_create_err.c_str());
}

}  // extern "C"
