// libhpgmxp.so: context, hierarchy build, and the extern "C" entry points
// declared in include/hpgmxp.h.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <type_traits>
#include <vector>

#include "hpgmxp.h"
#include "hpg_geom.h"
#include "hpg_kernels.cuh"
#include "hpg_coarse.cuh"
#include "hpg_cgs.cuh"
#include "hpg_p2p.cuh"
#include "hpg_wave.cuh"
#include "hpg_lower.cuh"
#include "hpg_tma.cuh"
#include "hpg_brick.cuh"
#include "hpg_jpl.cuh"

using hpg::Geom;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CUDA_TRY(expr)                                                                              \
  do {                                                                                              \
    cudaError_t e_ = (expr);                                                                        \
    if (e_ != cudaSuccess) return fail(HPG_E_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #expr,       \
                                       cudaGetErrorString(e_));                                     \
  } while (0)

#define NCCL_TRY(expr)                                                                              \
  do {                                                                                              \
    ncclResult_t r_ = (expr);                                                                       \
    if (r_ != ncclSuccess) return fail(HPG_E_NCCL, "%s:%d %s: %s", __FILE__, __LINE__, #expr,       \
                                       ncclGetErrorString(r_));                                     \
  } while (0)

#define LAUNCH_CHECK()                                                                              \
  do {                                                                                              \
    cudaError_t e_ = cudaGetLastError();                                                            \
    if (e_ != cudaSuccess) return fail(HPG_E_CUDA, "%s:%d launch: %s", __FILE__, __LINE__,          \
                                       cudaGetErrorString(e_));                                     \
  } while (0)

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Row stride of slot-major planes: a multiple of 32 elements that is an ODD
// multiple of 128 B, so the 27 concurrent plane streams of a warp do not
// alias onto the same L2 slices (2^k strides would).
inline int64_t pad_ld(int64_t n) {
  int64_t ld = cdiv(std::max<int64_t>(n, 1), 32) * 32;
  if ((ld / 32) % 2 == 0) ld += 32;
  return ld;
}

// ------------------------------------------------------------------ geometry (host)

int64_t nnz_axis(int l, int o, int g) {
  int64_t s = 0;
  for (int x = 0; x < l; ++x)
    for (int d = -1; d <= 1; ++d) s += (o + x + d >= 0 && o + x + d < g);
  return s;
}

Geom make_geom(const int l[3], const int c[3], const int p[3]) {
  Geom g;
  memset(&g, 0, sizeof g);
  g.lx = l[0];
  g.ly = l[1];
  g.lz = l[2];
  g.ox = c[0] * l[0];
  g.oy = c[1] * l[1];
  g.oz = c[2] * l[2];
  g.gx = p[0] * l[0];
  g.gy = p[1] * l[1];
  g.gz = p[2] * l[2];
  g.n = (int64_t)l[0] * l[1] * l[2];
  int nact = 0;
  for (int a = 0; a < 3; ++a) g.bit[a] = l[a] >= 2 ? nact++ : -1;
  g.ncolors = g.n ? 1 << nact : 0;
  g.off[0] = 0;
  for (int col = 0; col < g.ncolors; ++col) {
    int64_t size = 1;
    for (int a = 0; a < 3; ++a) {
      const int par = g.bit[a] >= 0 ? (col >> g.bit[a]) & 1 : 0;
      size *= (l[a] - par + 1) / 2;
    }
    g.off[col + 1] = g.off[col] + size;
  }
  for (int col = g.ncolors + 1; col <= hpg::kMaxColors; ++col) g.off[col] = g.n;
  // neighbours sorted by rank id; halo slots in that order (ref: comm.py:219-227)
  struct Nb {
    int rank, idx;
    int64_t cnt;
  };
  std::vector<Nb> nbs;
  for (int i = 0; i < 27; ++i) {
    g.halo_base[i] = -1;
    g.nbr_rank[i] = -1;
  }
  for (int sz = -1; sz <= 1; ++sz)
    for (int sy = -1; sy <= 1; ++sy)
      for (int sx = -1; sx <= 1; ++sx) {
        if (!sx && !sy && !sz) continue;
        const int cx = c[0] + sx, cy = c[1] + sy, cz = c[2] + sz;
        if (cx < 0 || cx >= p[0] || cy < 0 || cy >= p[1] || cz < 0 || cz >= p[2]) continue;
        nbs.push_back({cx + p[0] * (cy + p[1] * cz), hpg::offset_index(sx, sy, sz), hpg::region_size(g, sx, sy, sz)});
      }
  std::sort(nbs.begin(), nbs.end(), [](const Nb& a, const Nb& b) { return a.rank < b.rank; });
  int64_t base = g.n;
  for (auto& nb : nbs) {
    g.halo_base[nb.idx] = base;
    g.nbr_rank[nb.idx] = nb.rank;
    base += nb.cnt;
  }
  g.halo_size = base - g.n;
  return g;
}

int64_t geom_nnz(const Geom& g) {
  return nnz_axis(g.lx, g.ox, g.gx) * nnz_axis(g.ly, g.oy, g.gy) * nnz_axis(g.lz, g.oz, g.gz);
}

size_t esize(int prec) { return prec == HPG_F64 ? 8 : 4; }
ncclDataType_t nccl_type(int prec) { return prec == HPG_F64 ? ncclFloat64 : ncclFloat32; }

struct Nbr {
  int rank;
  int idx;
  int64_t send_off, cnt, recv_base;
};

struct Level {
  Geom g;
  int64_t n = 0, n_ext = 0, ld = 0, nnz = 0;
  int32_t* cols = nullptr;
  double* v64 = nullptr;
  float* v32 = nullptr;
  int32_t* inj = nullptr;  // (coarse levels) dst[j] for fine color-0 row j
  int32_t* f2c = nullptr;  // (coarse levels, general colorings) fine row of coarse row i
  int32_t* perm_d = nullptr;   // general coloring tables (null: greedy closed form)
  int32_t* iperm_d = nullptr;
  hpg::Stencil st{};           // implicit-index rows (st.on when the layout allows, checked at build)
  int64_t st_rows = 0;         // rows that skip their column-index loads
  bool st_lower = false;       // the zero-guess sweep's lower ELL has implicit-index rows too
  hpg::WaveLevel wave;         // dataflow sweep plan (valid when wave_ok)
  bool wave_ok = false;
  int32_t* wave_items = nullptr;
  unsigned int* wave_done = nullptr;
  // strictly-lower part per color for zero-initial-guess sweeps (hpg_lower.cuh)
  bool lower_ok = false;
  hpg::LowerColor lc[hpg::kMaxColors];
  int32_t* lcols = nullptr;
  double* lv64 = nullptr;
  float* lv32 = nullptr;
  double* dg64 = nullptr;
  float* dg32 = nullptr;
  uint8_t* hflag = nullptr;    // rows reading halo slots (multi-rank)
  int32_t* bnd = nullptr;      // all such rows
  int64_t nbnd = 0;
  int32_t* bnd0 = nullptr;     // such rows inside color block 0
  int64_t nbnd0 = 0;
  std::vector<Nbr> nbrs;
  hpg::P2PHalo p2p;            // NVLink peer-memory exchange plan (valid when ctx->p2p)
  int32_t* send_idx = nullptr;
  int64_t send_total = 0;
  void* send_buf = nullptr;
  double* z64 = nullptr;
  float* z32 = nullptr;
  double* r64 = nullptr;
  float* r32 = nullptr;
  size_t bytes = 0;
};

}  // namespace

struct GraphKey {
  int prec;
  const void* r;
  const void* z;
  bool operator==(const GraphKey& o) const { return prec == o.prec && r == o.r && z == o.z; }
};
struct GraphEntry {
  GraphKey key;
  cudaGraphExec_t exec;
  uint64_t stamp;
  int64_t kernels;  // kernel nodes in the graph (added to the launch count per replay)
};

struct hpg_ctx {
  int device = 0, rank = 0, nranks = 1;
  int procs[3] = {1, 1, 1}, coords[3] = {0, 0, 0};
  int nlev = 0, nu1 = 1, nu2 = 1, nu_c = 1;
  std::vector<Level> lev;
  cudaStream_t stream = nullptr;
  bool own_stream = true;
  cudaStream_t halo = nullptr;              // side stream for overlapped halo exchange
  cudaEvent_t ev_ready = nullptr, ev_done = nullptr;
  cudaEvent_t ev_cgs = nullptr;             // (h1, h2, beta) landed in pinned memory
  int cgs_pending_kb = 0, cgs_pending_es = 4;
  bool cgs_pending_norm = false;
  bool overlap = true;  // r02: with the tensor-copy kernels skipping the flagged rows, 4 ranks 706 -> 698 ms/solve
  const uint8_t* pass_skip = nullptr;  // set around an overlapped tensor-copy launch (PassPlan/SpmvPlan::skip)
  // NVLink peer memory (hpg_p2p.cuh): symmetric buffer, peers' mappings, sequence numbers
  bool p2p = false;
  bool p2p_want = true;
  char* sym = nullptr;
  size_t sym_bytes = 0;
  std::vector<char*> peer_sym;
  char** d_peer = nullptr;
  unsigned int* done = nullptr;
  uint64_t halo_seq = 0, ar_seq = 0;
  std::vector<std::pair<int, int>> cgs_cfg;  // (kb max, WR*100 + RPW*10 + U)
  int64_t overlap_rows = 0;  // only levels this large hide an exchange behind interior rows (r02: all, 4 ranks -1 ms)
  ncclComm_t comm = nullptr;
  int nb = 0;                   // reduction grid
  void* partial = nullptr;      // nb * 64 elements (f64-sized)
  double* spmv_partial = nullptr;
  int64_t spmv_partial_len = 0;
  void* scal = nullptr;         // 512 f64-sized device scalars
  void* gather = nullptr;       // nranks * 256
  double* pinned = nullptr;     // 256 host doubles
  int64_t launches = 0;
  bool cgs_fused = true;
  int cgs_force = 0;  // option "cgs_cfg": force one fused-CGS2 configuration (tuning)
  bool overlap_tma = true;  // option "overlap_tma": overlapped levels keep the tensor-copy kernels
  int cgs_solo = 1;    // option "cgs_solo": CgsParams::solo_fold
  int cgs_zigzag = 1;  // option "cgs_zigzag": CgsParams::zigzag of the fused CGS2 (r02: kb 30 -5%)
  bool general = false;  // some level uses an explicit (non-greedy) coloring
  bool graphs = true;    // replay captured V-cycles (single rank)
  // zero sweeps stream only the strictly-lower part (hpg_lower.cuh).  Off by
  // default: it skips the products against z = 0 that the reference forms
  // (smoother.py:95-112) and that the HPG-MxP flop model counts
  bool lower = false;
  bool known_zero = true;  // zero sweeps skip loads of known zeros (same arithmetic)
  // sweeps as one dataflow kernel (hpg_wave.cuh) where the layout allows; bit 0:
  // fp64 sweeps, bit 1: fp32.  Measured at 256^3: fp64 sweep -9%, fp32 +19%
  int wave = 1;
  int64_t wave_min_rows = 0;
  int wave_lag = 8;
  bool wave_coh = false;
  int wave_blocks[2] = {0, 0};
  // bulk-copy pipelined persistent sweeps (hpg_tma.cuh); bit 0: fp64, bit 1: fp32,
  // for levels with at least tma_min_rows rows
  int tma = 3;
  int64_t tma_min_rows = 1 << 18;
  int tma_blocks[2] = {0, 0};
  int tma_contig = 0;  // (persistent sweep) CTAs own contiguous row slabs of every colour block
  int tma_sweep = 0;   // 1: the persistent whole-sweep kernel instead of per-pass launches
  // per-pass kernel (rows * 100 + CTAs per SM) [fp64, fp32]; measured 256^3 level-0 sweeps
  // (r02, tools/sweep_ab.py): fp32 64x16 479 us (256x5 with spills 699, 128x8 490),
  // fp64 64x10 776 us (128x6 897, 64x12 796) vs 581 / 1032 us for k_gs_pass / the wave sweep
  int tma_cfg[2] = {3220, 12808};  // fp64 32x20; fp32 128x8 once face rows compute their columns (r02: sweep 440 -> 374 us, solve 2289 -> 2424 GF/s same box)
  // brick passes (hpg_brick.cuh): bit 0 fp64, bit 1 fp32; (rows * 100 + CTAs per SM).
  // Off: measured slower (r02, fp32 level-0 sweep 638 us at 128x8 vs 480 for the
  // tma pass) -- each CTA's neighbour-z boxes can only be requested after the PDL
  // wait and their latency is exposed per CTA
  int brick = 0;
  int brick_cfg[2] = {12804, 25605};
  size_t brick_smem_max = 64 * 1024;
  // pipelined persistent brick pass: bit 0 fp64, bit 1 fp32; (rows * 10 + stages)
  int bpp = 0;
  int bpp_cfg[2] = {1282, 1283};
  std::map<int, int> bpp_blocks;
  std::map<int, size_t> bpp_smem;
  // SpMV / fp64 residual with staged values: bit 0 fp64, bit 1 fp32; configurations
  int spmv_tma = 3;
  int spmv_cfg[2] = {3220, 6416};  // measured r02: fp32 SpMV 446 -> 417 us, fp64 683 -> 667 us
  int resid_cfg = 6410;
  int restr_cfg[2] = {3220, 6416};  // fused residual + injection (MODE 2) [fp64, fp32]
  int64_t l2_window = 0;   // > 0: persisting L2 set-aside (bytes) for z during the big colour passes
  // face rows off rank interfaces compute their columns (hpg_tma.cuh st_face_cols) in:
  // bit 0 SpMV / residual / restriction, bit 1 fp64 colour passes, bit 2 fp32 colour
  // passes; bit 3: colour passes take x-face rows through a compile-time slot map
  // (st_xface).  Measured r02 (256^3): SpMV fp32 424 -> 350 us, fp64 668 -> 580,
  // residual 825 -> 752, fp64 sweep 761 -> 681; fp32 sweep 489 -> 449 with bits 2+3
  // (bit 2 alone: 513, bit 3 alone: 522)
  int face_cols = 31;  // bit 4: SpMV-type kernels take x-face rows through the slot map too (fp32 SpMV 349 -> 331 us)
  bool l2_limit_set = false;
  size_t l2_setaside = 0, l2_maxwin = 0;  // measured r02: residual 867 -> 800 us (32x20: 913)  // fp64 32x20: 762 us
  unsigned* sweep_done = nullptr;  // pass counters of the persistent sweep
  std::vector<GraphEntry> gcache;
  uint64_t gclock = 0;
  bool pdl = true;
  // SpMV CTA interleave over the color blocks [f64, f32] (HPG_SPMV_ILV, HPG_SPMV_ILV32);
  // measured 1xB200 256^3: f64 SpMV 760 -> 680 us at 4 (x is 134 MB, above L2), f32 454 -> 464 us at 4
  int spmv_ilv[2] = {4, 8};  // r02: fp32 8 (x gathers shared across the colour blocks in L2) -1.6% solve
  int gs_minb = 3;
  bool gs_rev = true;   // odd colors walk their block backwards (L2 reuse of z at the turn)
  bool stencil = true;  // interior rows compute their ELL columns instead of loading them
  int64_t tail_rows = 0;        // levels with n <= tail_rows run in the persistent tail kernel
  int tail_blocks[2] = {0, 0};  // cooperative grid (f64, f32)
  int tail_cluster = 0;         // > 0: run the tail as one cluster of this many CTAs
  // per-motif CUDA-event timers (ref: metrics.py:125-131 Tally.timed)
  bool timing = false;
  std::vector<cudaEvent_t> events;
  size_t ev_used = 0;
  std::vector<std::pair<int, size_t>> marks;  // (motif, index of start event; end = +1)
};

namespace {

enum Motif { M_GS = 0, M_SPMV = 1, M_ORTHO = 2, M_RESTRICT = 3, M_PROLONG = 4, M_VEC = 5, M_GS_L0 = 6, M_GS_L0Z = 7 };

// RAII motif region: records an event pair on the compute stream when timing is on
struct Timed {
  hpg_ctx* c;
  int motif;
  size_t idx = (size_t)-1;
  Timed(hpg_ctx* c_, int m) : c(c_), motif(m) {
    if (!c->timing || m < 0) return;
    while (c->events.size() < c->ev_used + 2) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) return;
      c->events.push_back(e);
    }
    idx = c->ev_used;
    c->ev_used += 2;
    cudaEventRecord(c->events[idx], c->stream);
  }
  ~Timed() {
    if (idx == (size_t)-1) return;
    cudaEventRecord(c->events[idx + 1], c->stream);
    c->marks.push_back({motif, idx});
  }
};

template <typename T>
T* vals_of(const Level& L);
template <>
double* vals_of<double>(const Level& L) { return L.v64; }
template <>
float* vals_of<float>(const Level& L) { return L.v32; }

hpg::Stencil stencil_of(const hpg_ctx* c, const Level& L) { return c->stencil ? L.st : hpg::Stencil{}; }

int grid_for(int64_t n, int threads = 256) { return (int)std::max<int64_t>(1, cdiv(n, threads)); }

// Launch with programmatic dependent launch (PDL) enabled: the kernel may begin
// while its stream predecessor drains (kernels call griddepcontrol.wait before
// touching predecessor-produced data; see hpg_kernels.cuh pdl_wait).
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(hpg_ctx* c, void (*k)(KArgs...), int grid, int block, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = c->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = c->pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, ((KArgs)args)...);
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl_smem(hpg_ctx* c, void (*k)(KArgs...), int grid, int block, size_t smem, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = c->pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, ((KArgs)args)...);
}

// launch_pdl_smem plus an L2 access-policy window (persisting hits on [base, base+bytes))
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl_smem_win(hpg_ctx* c, const void* base, size_t bytes, float hit, void (*k)(KArgs...), int grid,
                                int block, size_t smem, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (c->pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (base && bytes) {
    attr[na].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[na].val.accessPolicyWindow.base_ptr = (void*)base;
    attr[na].val.accessPolicyWindow.num_bytes = bytes;
    attr[na].val.accessPolicyWindow.hitRatio = hit;
    attr[na].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr[na].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, k, ((KArgs)args)...);
}

// one kernel: P2P pack into the neighbours' staging, publish, wait, unpack
int halo_p2p(hpg_ctx* c, int l, int prec, void* v, cudaStream_t st) {
  Level& L = c->lev[l];
  const uint64_t seq = ++c->halo_seq;
  const int grid = (int)std::min<int64_t>(296, std::max<int64_t>(1, cdiv(L.p2p.total, 256 * 8)));
  cudaStream_t keep = c->stream;
  c->stream = st;  // launch_pdl enqueues on c->stream
  cudaError_t e = prec == HPG_F64
                      ? launch_pdl(c, hpg::k_halo_p2p<double>, grid, 256, (double*)v, (const int32_t*)L.send_idx,
                                   L.p2p, seq, c->done)
                      : launch_pdl(c, hpg::k_halo_p2p<float>, grid, 256, (float*)v, (const int32_t*)L.send_idx,
                                   L.p2p, seq, c->done);
  c->stream = keep;
  if (e != cudaSuccess) return fail(HPG_E_CUDA, "halo kernel launch: %s", cudaGetErrorString(e));
  ++c->launches;
  return HPG_OK;
}

int do_exchange(hpg_ctx* c, int l, int prec, void* v) {
  Level& L = c->lev[l];
  if (c->nranks == 1 || L.nbrs.empty()) return HPG_OK;
  if (c->p2p) return halo_p2p(c, l, prec, v, c->stream);
  if (L.send_total) {
    if (prec == HPG_F64)
      hpg::k_pack<double><<<grid_for(L.send_total), 256, 0, c->stream>>>((const double*)v, L.send_idx, L.send_total,
                                                                         (double*)L.send_buf);
    else
      hpg::k_pack<float><<<grid_for(L.send_total), 256, 0, c->stream>>>((const float*)v, L.send_idx, L.send_total,
                                                                        (float*)L.send_buf);
    LAUNCH_CHECK();
    ++c->launches;
  }
  if (!c->comm) return fail(HPG_E_NCCL, "no NCCL communicator (P2P-only context) and peer memory is off");
  const size_t es = esize(prec);
  NCCL_TRY(ncclGroupStart());
  for (auto& nb : L.nbrs) {
    NCCL_TRY(ncclSend((char*)L.send_buf + nb.send_off * es, nb.cnt, nccl_type(prec), nb.rank, c->comm, c->stream));
    NCCL_TRY(ncclRecv((char*)v + nb.recv_base * es, nb.cnt, nccl_type(prec), nb.rank, c->comm, c->stream));
  }
  NCCL_TRY(ncclGroupEnd());
  return HPG_OK;
}

// Overlapped exchange (ref: comm.py:254-272 exchange_overlapped): pack + NCCL on
// the halo stream while the compute stream runs rows that read no halo slot and
// write no send row; exchange_end makes the compute stream wait for the halo.
int exchange_begin(hpg_ctx* c, int l, int prec, void* v) {
  Level& L = c->lev[l];
  CUDA_TRY(cudaEventRecord(c->ev_ready, c->stream));
  CUDA_TRY(cudaStreamWaitEvent(c->halo, c->ev_ready, 0));
  if (c->p2p) {
    int rc = halo_p2p(c, l, prec, v, c->halo);
    if (rc) return rc;
    CUDA_TRY(cudaEventRecord(c->ev_done, c->halo));
    return HPG_OK;
  }
  if (L.send_total) {
    if (prec == HPG_F64)
      hpg::k_pack<double><<<grid_for(L.send_total), 256, 0, c->halo>>>((const double*)v, L.send_idx, L.send_total,
                                                                       (double*)L.send_buf);
    else
      hpg::k_pack<float><<<grid_for(L.send_total), 256, 0, c->halo>>>((const float*)v, L.send_idx, L.send_total,
                                                                      (float*)L.send_buf);
    LAUNCH_CHECK();
    ++c->launches;
  }
  if (!c->comm) return fail(HPG_E_NCCL, "no NCCL communicator (P2P-only context) and peer memory is off");
  const size_t es = esize(prec);
  NCCL_TRY(ncclGroupStart());
  for (auto& nb : L.nbrs) {
    NCCL_TRY(ncclSend((char*)L.send_buf + nb.send_off * es, nb.cnt, nccl_type(prec), nb.rank, c->comm, c->halo));
    NCCL_TRY(ncclRecv((char*)v + nb.recv_base * es, nb.cnt, nccl_type(prec), nb.rank, c->comm, c->halo));
  }
  NCCL_TRY(ncclGroupEnd());
  CUDA_TRY(cudaEventRecord(c->ev_done, c->halo));
  return HPG_OK;
}

int exchange_end(hpg_ctx* c) {
  CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_done, 0));
  return HPG_OK;
}

bool overlapped(hpg_ctx* c, int l) {
  return c->nranks > 1 && c->overlap && !c->lev[l].nbrs.empty() && c->lev[l].n >= c->overlap_rows;
}

// rank-ordered allreduce of cnt device scalars in place (ref: comm.py:97-108)
hpg::P2PAr p2p_ar(hpg_ctx* c) {
  hpg::P2PAr ar;
  ar.peer = c->d_peer;
  ar.me = c->rank;
  ar.nranks = c->p2p ? c->nranks : 1;
  return ar;
}

template <typename T>
int allreduce_scal(hpg_ctx* c, T* buf, int cnt) {
  if (c->nranks == 1) return HPG_OK;
  if (c->p2p) {
    hpg::k_p2p_allreduce<T><<<1, 64, 0, c->stream>>>(buf, cnt, p2p_ar(c), ++c->ar_seq, 0);
    LAUNCH_CHECK();
    ++c->launches;
    return HPG_OK;
  }
  if (!c->comm) return fail(HPG_E_NCCL, "no NCCL communicator (P2P-only context) and peer memory is off");
  NCCL_TRY(ncclAllGather(buf, c->gather, cnt, sizeof(T) == 8 ? ncclFloat64 : ncclFloat32, c->comm, c->stream));
  hpg::k_fold_ranks<T><<<1, 64, 0, c->stream>>>((const T*)c->gather, c->nranks, cnt, buf, 0);
  LAUNCH_CHECK();
  ++c->launches;
  return HPG_OK;
}

template <typename T>
int gs_pass_launch(hpg_ctx* c, Level& L, int64_t a, int64_t cnt, const T* r, T* z, const uint8_t* skip,
                   const int32_t* list, int64_t known0 = -1, int rev = 0) {
  const T* vals = vals_of<T>(L);
  if (skip || list)
    CUDA_TRY(launch_pdl(c, hpg::k_gs_pass<T, 3, true>, grid_for(cnt), 256, L.cols, vals, L.ld, a, cnt, r, z, skip,
                        list, known0, 0, stencil_of(c, L)));
  else if (c->gs_minb == 3)
    CUDA_TRY(launch_pdl(c, hpg::k_gs_pass<T, 3>, grid_for(cnt, HPG_GS_BLOCK), HPG_GS_BLOCK, L.cols, vals, L.ld, a, cnt, r, z, skip, list,
                        known0, rev, stencil_of(c, L)));
  else if (c->gs_minb == 4)
    CUDA_TRY(launch_pdl(c, hpg::k_gs_pass<T, 4>, grid_for(cnt, HPG_GS_BLOCK), HPG_GS_BLOCK, L.cols, vals, L.ld, a, cnt, r, z, skip, list,
                        known0, rev, stencil_of(c, L)));
  else
    CUDA_TRY(launch_pdl(c, hpg::k_gs_pass<T, 2>, grid_for(cnt, HPG_GS_BLOCK), HPG_GS_BLOCK, L.cols, vals, L.ld, a, cnt, r, z, skip, list,
                        known0, rev, stencil_of(c, L)));
  ++c->launches;
  return HPG_OK;
}

template <typename T>
int gs_lower_launch(hpg_ctx* c, Level& L, int col, const T* r, T* z) {
  const hpg::LowerColor& lc = L.lc[col];
  const int64_t a = L.g.off[col], cnt = L.g.off[col + 1] - a;
  if (cnt <= 0) return HPG_OK;
  const int32_t* lcols = L.lcols + lc.base;
  const T* lv = (sizeof(T) == 8 ? (const T*)L.lv64 : (const T*)L.lv32) + lc.base;
  const T* dg = sizeof(T) == 8 ? (const T*)L.dg64 : (const T*)L.dg32;
  const int rev = c->gs_rev && (col & 1);
  cudaError_t e =
      c->stencil && L.st.on && L.st_lower
          ? launch_pdl(c, hpg::lower_st_kernel<T>(col), grid_for(cnt, HPG_LOWER_BLOCK), HPG_LOWER_BLOCK, lcols, lv,
                       lc.ldc, a, cnt, dg, r, z, rev,
                       L.st)
          : launch_pdl(c, hpg::lower_kernel<T>(lc.w), grid_for(cnt), 256, lcols, lv, lc.ldc, a, cnt, dg, r, z, rev);
  CUDA_TRY(e);
  ++c->launches;
  return HPG_OK;
}

template <typename T>
const void* wave_fn(bool coh) {
  return coh ? (const void*)hpg::k_gs_wave<T, true> : (const void*)hpg::k_gs_wave<T, false>;
}

template <typename T>
int gs_wave_launch(hpg_ctx* c, Level& L, const T* r, T* z, int zero) {
  const int blocks = c->wave_blocks[sizeof(T) == 4];
  const int32_t* cols = L.cols;
  const T* vals = vals_of<T>(L);
  int64_t ld = L.ld;
  // (no implicit-index rows here: the extra kernel argument made the fp64 item
  // loop spill, level-0 fp64 sweep 1028 -> 1223 us)
  void* args[] = {(void*)&cols, (void*)&vals, (void*)&ld, (void*)&r, (void*)&z, (void*)&L.wave, (void*)&zero};
  const void* fn = wave_fn<T>(c->wave_coh);
  CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3(blocks), dim3(hpg::kWaveRows), args, 0,
                                       c->stream));
  ++c->launches;
  return HPG_OK;
}

// One forward multicolor sweep (ref: smoother.py:78-114).  Multi-rank: the
// Persistent bulk-copy pipelined sweep (hpg_tma.cuh): tile rows / ring depth
template <typename T>
struct TmaCfg;
template <>
struct TmaCfg<float> {
  static constexpr int kRows = 256, kStages = 4;
};
template <>
struct TmaCfg<double> {
  static constexpr int kRows = 128, kStages = 4;
};

template <typename T>
size_t tma_smem() {
  return (size_t)TmaCfg<T>::kStages * hpg::TmaTile<T, TmaCfg<T>::kRows>::kBytes + 2 * TmaCfg<T>::kStages * 8;
}

template <typename T>
bool tma_ok(hpg_ctx* c, const Level& L) {
  if (!((c->tma >> (sizeof(T) == 4)) & 1) || L.n < c->tma_min_rows || c->tma_blocks[sizeof(T) == 4] <= 0) return false;
  // tensor map: 16-byte aligned base and row pitch; every tile starts 16-byte aligned
  // (tile starts are colour offsets plus multiples of 32 rows)
  if ((L.ld * (int64_t)sizeof(T)) % 16 || ((uintptr_t)vals_of<T>(L)) % 16 || L.ld >= (int64_t{1} << 31)) return false;
  if (L.ld < std::max(TmaCfg<T>::kRows, c->tma_cfg[sizeof(T) == 4] / 100)) return false;  // the box fits the tensor
  for (int k = 0; k <= L.g.ncolors; ++k)
    if ((L.g.off[k] * (int64_t)sizeof(T)) % 16) return false;
  return true;
}

// The value planes [27][ld] of T as a 2-D tensor map, box {rows, 27}
// (cuTensorMapEncodeTiled through the runtime's driver entry point: no -lcuda).
template <typename T>
int encode_value_map(hpg_ctx* c, const Level& L, int rows, CUtensorMap* map) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !fn) return fail(HPG_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }
  const cuuint64_t dims[2] = {(cuuint64_t)L.ld, 27};
  const cuuint64_t strides[1] = {(cuuint64_t)L.ld * sizeof(T)};
  const cuuint32_t box[2] = {(cuuint32_t)rows, 27};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(map, sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                      (void*)vals_of<T>(L), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(HPG_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return HPG_OK;
}

void stencil_offsets(const hpg::Stencil& st, int col, int32_t* doff, uint32_t* kmask);

template <typename T>
int gs_sweep_tma(hpg_ctx* c, Level& L, const T* r, T* z, int zero) {
  hpg::SweepPlan p;
  memset(&p, 0, sizeof p);
  int rc0 = encode_value_map<T>(c, L, TmaCfg<T>::kRows, &p.vmap);
  if (rc0) return rc0;
  p.cols = L.cols;
  p.vals = vals_of<T>(L);
  p.ld = L.ld;
  p.ncolors = L.g.ncolors;
  for (int k = 0; k <= L.g.ncolors; ++k) p.off[k] = L.g.off[k];
  p.zero = zero;
  p.rev_odd = c->gs_rev ? 1 : 0;
  p.contiguous = c->tma_contig;
  p.done = c->sweep_done;
  p.st = stencil_of(c, L);
  if (p.st.on)  // per-colour column offsets of implicit-index rows (see hpg_tma.cuh SweepPlan)
    for (int col = 0; col < 8; ++col) stencil_offsets(p.st, col, p.doff[col], &p.kmask[col]);
  constexpr int R = TmaCfg<T>::kRows, S = TmaCfg<T>::kStages;
  CUDA_TRY(launch_pdl_smem(c, hpg::k_gs_sweep_tma<T, R, S>, c->tma_blocks[sizeof(T) == 4], 32 + R, tma_smem<T>(), p, r,
                           z));
  ++c->launches;
  return HPG_OK;
}

// per-pass TMA-fed colour pass: (rows per CTA, CTAs per SM) chosen per precision
// by the option "tma_cfg32" / "tma_cfg64" = rows * 100 + CTAs per SM
#define HPG_PASS_CFGS(X) X(float, 256, 5) X(float, 256, 4) X(float, 128, 10) X(float, 128, 8) X(float, 64, 16) X(float, 32, 32) \
  X(float, 128, 6) X(float, 128, 7) X(float, 192, 5) X(float, 96, 10) X(double, 64, 6) X(double, 96, 6) \
  X(float, 64, 12) X(double, 128, 6) X(double, 128, 4) X(double, 64, 12) X(double, 64, 10) X(double, 64, 8) \
  X(double, 32, 20)
template <typename T, int R>
size_t pass_smem() {
  return (size_t)27 * R * sizeof(T) + 16;
}

// the per-colour constants of implicit-index rows (see hpg_tma.cuh SweepPlan)
void stencil_offsets(const hpg::Stencil& st, int col, int32_t* doff, uint32_t* kmask) {
  const int pxyz[3] = {(col >> st.bx) & 1, (col >> st.by) & 1, (col >> st.bz) & 1};
  const int bits[3] = {st.bx, st.by, st.bz};
  const int64_t stride[3] = {1, st.hx, st.hxy};
  uint32_t km = 0;
  for (int s = 0; s < 27; ++s) {
    const int d[3] = {s % 3 - 1, (s / 3) % 3 - 1, s / 9 - 1};
    int c2 = 0;
    int64_t shift = 0;
    for (int a = 0; a < 3; ++a) {
      const int ax = pxyz[a] + d[a];  // in [-1, 2]
      c2 |= (ax & 1) << bits[a];
      shift += (int64_t)(ax >= 0 ? ax / 2 : -1) * stride[a];
    }
    doff[s] = (int32_t)((int64_t)(c2 - col) * st.n8 + shift);
    if (c2 >= col) km |= 1u << s;
  }
  *kmask = km;
}

template <typename T, int R, int MB>
int gs_pass_tma_t(hpg_ctx* c, Level& L, int col, const T* r, T* z, int zero, int rev) {
  hpg::PassPlan p;
  memset(&p, 0, sizeof p);
  int rc0 = encode_value_map<T>(c, L, R, &p.vmap);
  if (rc0) return rc0;
  p.cols = L.cols;
  p.ld = L.ld;
  p.row0 = L.g.off[col];
  p.nrows = L.g.off[col + 1] - p.row0;
  p.known0 = zero ? p.row0 : -1;
  p.rev = rev;
  p.color = col;
  p.skip = c->pass_skip;
  p.st = stencil_of(c, L);
  if (p.st.on) {
    stencil_offsets(p.st, col, p.doff, &p.kmask);
    if (!zero) p.kmask = 0;
    p.xface = (c->face_cols & 8) ? 1 : 0;
    if (!(c->face_cols & (sizeof(T) == 4 ? 4 : 2))) p.st.ifc = 63;  // other face rows read the index plane
  }
  if (p.nrows <= 0) return HPG_OK;
  if (c->l2_window > 0 && L.n >= c->tma_min_rows) {
    // keep the smoothed vector resident in L2 across the colour passes: the
    // other colours' z lines are re-read by every pass (option "l2_window")
    if (!c->l2_limit_set) {
      cudaDeviceProp prop;
      CUDA_TRY(cudaGetDeviceProperties(&prop, c->device));
      c->l2_setaside = std::min<size_t>((size_t)c->l2_window, (size_t)prop.persistingL2CacheMaxSize);
      c->l2_maxwin = (size_t)prop.accessPolicyMaxWindowSize;
      CUDA_TRY(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, c->l2_setaside));
      c->l2_limit_set = true;
    }
    const size_t bytes = std::min<size_t>((size_t)L.n * sizeof(T), c->l2_maxwin);
    const float hit = std::min(1.0f, (float)c->l2_setaside / (float)bytes);
    CUDA_TRY(launch_pdl_smem_win(c, (const void*)z, bytes, hit, hpg::k_gs_pass_tma<T, R, MB>, (int)cdiv(p.nrows, R), R,
                                 pass_smem<T, R>(), p, r, z));
  } else {
    CUDA_TRY(launch_pdl_smem(c, hpg::k_gs_pass_tma<T, R, MB>, (int)cdiv(p.nrows, R), R, pass_smem<T, R>(), p, r, z));
  }
  ++c->launches;
  return HPG_OK;
}

template <typename T>
int gs_pass_tma(hpg_ctx* c, Level& L, int col, const T* r, T* z, int zero, int rev) {
  const int code = c->tma_cfg[sizeof(T) == 4];
#define HPG_PASS_CASE(TT, R, MB)                                                          \
  if (std::is_same<T, TT>::value && code == R * 100 + MB)                                  \
    return gs_pass_tma_t<TT, R, MB>(c, L, col, (const TT*)r, (TT*)z, zero, rev);
  HPG_PASS_CFGS(HPG_PASS_CASE)
#undef HPG_PASS_CASE
  return fail(HPG_E_ARG, "unknown colour-pass configuration %d", code);
}

int pass_rows(int code) { return code / 100; }

// ---- brick colour pass (hpg_brick.cuh): values AND neighbour z staged by tensor copies
#define HPG_SPMV_CFGS(X) X(float, 64, 16, 0) X(float, 128, 8, 0) X(float, 32, 32, 0) X(double, 32, 20, 0) \
  X(double, 64, 10, 0) X(double, 64, 8, 0) X(double, 32, 20, 1) X(double, 64, 10, 1) X(double, 64, 8, 1) \
  X(float, 64, 16, 2) X(float, 128, 8, 2) X(double, 32, 20, 2) X(double, 64, 10, 2)
#define HPG_BRICK_CFGS(X) X(float, 256, 5) X(float, 256, 4) X(float, 128, 8) X(double, 128, 4) X(double, 128, 3) \
  X(double, 64, 8)

template <typename T>
PFN_cuTensorMapEncodeTiled_v12000 tensor_encoder(hpg_ctx* c) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }
  return encode;
}

// the brick tiling applies: implicit-index layout, ROWS whole x-lines of one plane,
// every box within the tensor-copy limits
template <typename T>
bool brick_ok(hpg_ctx* c, const Level& L, int rows, bool any = false) {
  const hpg::Stencil st = stencil_of(c, L);
  if (!st.on || (!any && !((c->brick >> (sizeof(T) == 4)) & 1))) return false;
  const int pad = 16 / (int)sizeof(T);
  const int hx = (int)st.hx, hy = (int)st.hy;
  if (hx % pad || rows % hx || hy % (rows / hx) || hx + pad > 256 || rows / hx + 1 > 256) return false;
  return true;
}

// The brick plan of colour col (value map, z box maps and offsets, slot table)
template <typename T>
int brick_plan(hpg_ctx* c, Level& L, int col, T* z, int zero, int rev, int R, hpg::BrickPlan& p, int* zelems) {
  memset(&p, 0, sizeof p);
  int rc0 = encode_value_map<T>(c, L, R, &p.vmap);
  if (rc0) return rc0;
  const hpg::Stencil st = stencil_of(c, L);
  const int w = (int)sizeof(T), pad = 16 / w;
  const int hx = (int)st.hx, hy = (int)st.hy, hz = (int)(st.n8 / st.hxy), BY = R / hx;
  p.cols = L.cols;
  p.ld = L.ld;
  p.row0 = L.g.off[col];
  p.nrows = L.g.off[col + 1] - p.row0;
  p.known0 = zero ? p.row0 : -1;
  p.rev = rev;
  p.color = col;
  p.hx = hx;
  p.hxy = (int)st.hxy;
  p.pad = pad;
  p.st = st;
  const int par[3] = {(col >> st.bx) & 1, (col >> st.by) & 1, (col >> st.bz) & 1};
  const int bits[3] = {st.bx, st.by, st.bz};
  int xe[8], ye[8];
  int off = 0;
  auto encode = tensor_encoder<T>(c);
  if (!encode) return fail(HPG_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  for (int am = 1; am < 8; ++am) {
    const int xb = am & 1, yb = (am >> 1) & 1, zb = (am >> 2) & 1;
    xe[am] = hx + (xb ? pad : 0);
    ye[am] = BY + yb;
    const int ze = 1 + zb;
    // the innermost start coordinate of a tensor copy must be 16-byte aligned (x = -1
    // faults: tools/tma4d_test.cu), so a box reaching one column left starts at -pad
    p.box_x[am] = (xb && par[0] == 0) ? -pad : 0;
    p.box_y[am] = (yb && par[1] == 0) ? -1 : 0;
    p.box_z[am] = (zb && par[2] == 0) ? -1 : 0;
    p.box_c[am] = col ^ ((xb << bits[0]) | (yb << bits[1]) | (zb << bits[2]));
    p.box_off[am] = off;
    p.box_bytes[am] = (uint32_t)(xe[am] * ye[am] * ze * w);
    off += (xe[am] * ye[am] * ze * w + 127) / 128 * 128 / w;
    if (!zero || p.box_c[am] < col) p.load_mask |= 1u << am;
    // X extent hx + pad: a box may not be wider than its tensor (entries past hx alias the next
    // line and are never read by an interior row)
    const cuuint64_t dims[4] = {(cuuint64_t)(hx + pad), (cuuint64_t)hy, (cuuint64_t)hz, 8};
    const cuuint64_t strides[3] = {(cuuint64_t)hx * w, (cuuint64_t)st.hxy * w, (cuuint64_t)st.n8 * w};
    const cuuint32_t box[4] = {(cuuint32_t)xe[am], (cuuint32_t)ye[am], (cuuint32_t)ze, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult er = encode(&p.zmap[am], w == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
                         (void*)z, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (er != CUDA_SUCCESS) return fail(HPG_E_CUDA, "z tensor map encode failed (%d)", (int)er);
  }
  p.box_off[0] = off;  // end of the boxes: the mbarriers follow
  for (int s = 0; s < 27; ++s) {
    const int d[3] = {s % 3 - 1, (s / 3) % 3 - 1, s / 9 - 1};
    const int am = (d[0] != 0) | ((d[1] != 0) << 1) | ((d[2] != 0) << 2);
    if (!am) continue;  // the diagonal
    int e[3];
    for (int a = 0; a < 3; ++a) {
      const int ax = par[a] + d[a];
      e[a] = ax >= 0 ? ax / 2 : -1;
    }
    const int xl = e[0] - p.box_x[am], yl = e[1] - p.box_y[am], zl = e[2] - p.box_z[am];
    p.sconst[s] = p.box_off[am] + xl + xe[am] * yl + xe[am] * ye[am] * zl;
    if (am & 1) p.xsel |= 1u << s;
    if (zero && p.box_c[am] >= col) p.kmask |= 1u << s;
  }
  *zelems = off;
  return HPG_OK;
}

template <typename T, int R, int MB>
int gs_pass_brick_t(hpg_ctx* c, Level& L, int col, const T* r, T* z, int zero, int rev) {
  hpg::BrickPlan p;
  int off = 0;
  int rc0 = brick_plan<T>(c, L, col, z, zero, rev, R, p, &off);
  if (rc0) return rc0;
  const int w = (int)sizeof(T);
  if (p.nrows <= 0) return HPG_OK;
  const size_t zoff = (hpg::BrickSmem<T, R>::kValBytes + 127) / 128 * 128;
  const size_t smem = zoff + (size_t)off * w + 16;
  if (smem > c->brick_smem_max) return fail(HPG_E_ARG, "brick tile needs %zu B of shared memory", smem);
  CUDA_TRY(launch_pdl_smem(c, hpg::k_gs_pass_brick<T, R, MB>, (int)cdiv(p.nrows, R), R, smem, p, r, z, zoff));
  ++c->launches;
  return HPG_OK;
}

template <typename T>
int gs_pass_brick(hpg_ctx* c, Level& L, int col, const T* r, T* z, int zero, int rev) {
  const int code = c->brick_cfg[sizeof(T) == 4];
#define HPG_BRICK_CASE(TT, R, MB)                                                     \
  if (std::is_same<T, TT>::value && code == R * 100 + MB)                              \
    return gs_pass_brick_t<TT, R, MB>(c, L, col, (const TT*)r, (TT*)z, zero, rev);
  HPG_BRICK_CFGS(HPG_BRICK_CASE)
#undef HPG_BRICK_CASE
  return fail(HPG_E_ARG, "unknown brick-pass configuration %d", code);
}

// pipelined persistent brick pass (hpg_brick.cuh k_gs_brick_pp): (rows, stages)
#define HPG_BPP_CFGS(X) X(float, 128, 3) X(float, 128, 2) X(float, 256, 2) X(double, 128, 2) X(double, 64, 3)

template <typename T, int R, int S>
int gs_pass_bpp_t(hpg_ctx* c, Level& L, int col, const T* r, T* z, int zero, int rev) {
  hpg::BrickPlan p;
  int zel = 0;
  int rc0 = brick_plan<T>(c, L, col, z, zero, rev, R, p, &zel);
  if (rc0) return rc0;
  if (getenv("HPG_BPP_NOZ")) p.load_mask = 0;  // timing experiment only (wrong results)
  hpg::BrickPipe q;
  q.vbytes = (uint32_t)(27 * R * sizeof(T));
  q.zoff = (q.vbytes + 127) / 128 * 128;
  q.roff = (uint32_t)((q.zoff + (size_t)zel * sizeof(T) + 127) / 128 * 128);
  q.stage_bytes = (uint32_t)((q.roff + 2 * R * sizeof(T) + 127) / 128 * 128);
  q.ntiles = p.nrows / R;
  if (p.nrows <= 0) return HPG_OK;
  const size_t smem = (size_t)S * q.stage_bytes + 2 * S * 8;
  auto fn = hpg::k_gs_brick_pp<T, R, S>;
  const int key = (sizeof(T) == 4 ? 1000000 : 0) + R * 10 + S;
  int& blocks = c->bpp_blocks[key];
  if (blocks == 0 || c->bpp_smem[key] != smem) {
    CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    int per = 0;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, 32 + R, smem));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
    blocks = std::max(1, per) * sms;
    c->bpp_smem[key] = smem;
    if (getenv("HPG_DEBUG")) fprintf(stderr, "bpp R=%d S=%d smem=%zu per_sm=%d\n", R, S, smem, per);
  }
  const int grid = (int)std::min<int64_t>(blocks, q.ntiles);
  CUDA_TRY(launch_pdl_smem(c, fn, grid, 32 + R, smem, p, q, r, z));
  ++c->launches;
  return HPG_OK;
}

template <typename T>
int gs_pass_bpp(hpg_ctx* c, Level& L, int col, const T* r, T* z, int zero, int rev) {
  const int code = c->bpp_cfg[sizeof(T) == 4];
#define HPG_BPP_CASE(TT, R, S)                                                        \
  if (std::is_same<T, TT>::value && code == R * 10 + S)                                \
    return gs_pass_bpp_t<TT, R, S>(c, L, col, (const TT*)r, (TT*)z, zero, rev);
  HPG_BPP_CFGS(HPG_BPP_CASE)
#undef HPG_BPP_CASE
  return fail(HPG_E_ARG, "unknown pipelined brick configuration %d", code);
}

template <typename T>
int tma_setup(hpg_ctx* c, int sms) {
#define HPG_BRICK_ATTR(TT, R, MB)                                                                           \
  if (std::is_same<T, TT>::value)                                                                           \
    CUDA_TRY(cudaFuncSetAttribute(hpg::k_gs_pass_brick<TT, R, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                  (int)c->brick_smem_max));
  HPG_BRICK_CFGS(HPG_BRICK_ATTR)
#undef HPG_BRICK_ATTR
#define HPG_SPMV_ATTR(TT, R, MB, MD)                                                                   \
  if (std::is_same<T, TT>::value)                                                                      \
    CUDA_TRY(cudaFuncSetAttribute(hpg::k_spmv_tma<TT, R, MB, MD>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                  (int)((size_t)27 * R * sizeof(TT) + 16)));
  HPG_SPMV_CFGS(HPG_SPMV_ATTR)
#undef HPG_SPMV_ATTR
#define HPG_PASS_ATTR(TT, R, MB)                                                                         \
  if (std::is_same<T, TT>::value)                                                                        \
    CUDA_TRY(cudaFuncSetAttribute(hpg::k_gs_pass_tma<TT, R, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                  (int)pass_smem<TT, R>()));
  HPG_PASS_CFGS(HPG_PASS_ATTR)
#undef HPG_PASS_ATTR
  constexpr int R = TmaCfg<T>::kRows, S = TmaCfg<T>::kStages;
  auto fn = hpg::k_gs_sweep_tma<T, R, S>;
  CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tma_smem<T>()));
  int per = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, 32 + R, tma_smem<T>()));
  c->tma_blocks[sizeof(T) == 4] = per * sms;
  return HPG_OK;
}

// exchange of z overlaps color 0's interior rows, then color 0's boundary rows,
// then colors 1.. (block-Jacobi across ranks: one exchange per sweep).
template <typename T>
int gs_sweep(hpg_ctx* c, int l, const T* r, T* z, int zero) {
  Timed tm(c, M_GS);
  Level& L = c->lev[l];
  // level-0 sweeps also timed alone (bench roofline): full sweeps and zero-guess
  // (strictly-lower) sweeps apart, they run different kernels
  Timed tm0(c, l != 0 ? -1 : (zero && c->lower && L.lower_ok) ? M_GS_L0Z : M_GS_L0);
  const int prec = sizeof(T) == 8 ? HPG_F64 : HPG_F32;
  int first = 0, rc;
  if (zero && c->lower && L.lower_ok) {
    // zero initial guess: only the strictly-lower part of each color contributes
    // (hpg_lower.cuh, bitwise equal); the halo tail is still cleared for later users
    if (L.n_ext > L.n) {
      CUDA_TRY(launch_pdl(c, hpg::k_zero<T>, grid_for(cdiv(L.n_ext - L.n, 4)), 256, z + L.n, L.n_ext - L.n));
      ++c->launches;
    }
    for (int col = 0; col < L.g.ncolors; ++col)
      if ((rc = gs_lower_launch<T>(c, L, col, r, z))) return rc;
    return HPG_OK;
  }
  if (tma_ok<T>(c, L) && !(overlapped(c, l) && !zero && !c->overlap_tma)) {
    if (zero) {
      if (L.n_ext > L.n) {  // zero initial guess: clear the halo tail; rows are all written
        CUDA_TRY(launch_pdl(c, hpg::k_zero<T>, grid_for(cdiv(L.n_ext - L.n, 4)), 256, z + L.n, L.n_ext - L.n));
        ++c->launches;
      }
      if (!c->known_zero) {
        CUDA_TRY(launch_pdl(c, hpg::k_zero<T>, grid_for(cdiv(L.n, 4)), 256, z, L.n));
        ++c->launches;
      }
    } else if (overlapped(c, l)) {
      // the exchange runs on the halo stream while colour 0's rows that neither read
      // a halo slot nor are sent run here; those rows follow once it has landed
      if ((rc = exchange_begin(c, l, prec, z))) return rc;
      c->pass_skip = L.hflag;
      rc = gs_pass_tma<T>(c, L, 0, r, z, 0, 0);
      c->pass_skip = nullptr;
      if (rc) return rc;
      if ((rc = exchange_end(c))) return rc;
      if (L.nbnd0 && (rc = gs_pass_launch<T>(c, L, 0, L.nbnd0, r, z, nullptr, L.bnd0))) return rc;
      for (int col = 1; col < L.g.ncolors; ++col)
        if ((rc = gs_pass_tma<T>(c, L, col, r, z, 0, c->gs_rev && (col & 1)))) return rc;
      return HPG_OK;
    } else if ((rc = do_exchange(c, l, prec, z))) {
      return rc;
    }
    if (c->tma_sweep) return gs_sweep_tma<T>(c, L, r, z, zero && c->known_zero);
    const bool bpp = ((c->bpp >> (sizeof(T) == 4)) & 1) && brick_ok<T>(c, L, c->bpp_cfg[sizeof(T) == 4] / 10, true);
    const bool brick = !bpp && brick_ok<T>(c, L, c->brick_cfg[sizeof(T) == 4] / 100);
    for (int col = 0; col < L.g.ncolors; ++col) {
      const int zz = zero && c->known_zero, rv = c->gs_rev && (col & 1);
      if ((rc = bpp     ? gs_pass_bpp<T>(c, L, col, r, z, zz, rv)
                : brick ? gs_pass_brick<T>(c, L, col, r, z, zz, rv)
                        : gs_pass_tma<T>(c, L, col, r, z, zz, rv)))
        return rc;
    }
    return HPG_OK;
  }
  const bool use_wave = (c->wave >> (sizeof(T) == 4)) & 1 && L.wave_ok && L.n >= c->wave_min_rows && c->wave_blocks[sizeof(T) == 4] > 0 &&
                        !(overlapped(c, l) && !zero);
  if (use_wave) {
    if (zero) {
      if (L.n_ext > L.n) {  // zero initial guess: clear the halo tail; rows are all written
        CUDA_TRY(launch_pdl(c, hpg::k_zero<T>, grid_for(cdiv(L.n_ext - L.n, 4)), 256, z + L.n, L.n_ext - L.n));
        ++c->launches;
      }
      if (!c->known_zero) {
        CUDA_TRY(launch_pdl(c, hpg::k_zero<T>, grid_for(cdiv(L.n, 4)), 256, z, L.n));
        ++c->launches;
      }
    } else if ((rc = do_exchange(c, l, prec, z))) {
      return rc;
    }
    return gs_wave_launch<T>(c, L, r, z, zero && c->known_zero);
  }
  if (zero && c->known_zero) {
    // zero initial guess (ref: smoother.py:95-96): only the halo tail is cleared;
    // every owned row is written by its color pass, which forms v * 0 for the
    // colors not yet updated instead of loading zeros (same arithmetic)
    if (L.n_ext > L.n)
      CUDA_TRY(launch_pdl(c, hpg::k_zero<T>, grid_for(cdiv(L.n_ext - L.n, 4)), 256, z + L.n, L.n_ext - L.n));
    for (int col = 0; col < L.g.ncolors; ++col) {
      const int64_t a = L.g.off[col], b = L.g.off[col + 1];
      if (b > a && (rc = gs_pass_launch<T>(c, L, a, b - a, r, z, nullptr, nullptr, a, c->gs_rev && (col & 1))))
        return rc;
    }
    return HPG_OK;
  }
  if (zero) {
    CUDA_TRY(launch_pdl(c, hpg::k_zero<T>, grid_for(cdiv(L.n_ext, 4)), 256, z, L.n_ext));
    ++c->launches;
  } else if (overlapped(c, l) && L.g.ncolors > 0) {
    if ((rc = exchange_begin(c, l, prec, z))) return rc;
    const int64_t a = L.g.off[0], b = L.g.off[1];
    if (b > a && (rc = gs_pass_launch<T>(c, L, a, b - a, r, z, L.hflag, nullptr))) return rc;
    if ((rc = exchange_end(c))) return rc;
    if (L.nbnd0 && (rc = gs_pass_launch<T>(c, L, 0, L.nbnd0, r, z, nullptr, L.bnd0))) return rc;
    first = 1;
  } else {
    if ((rc = do_exchange(c, l, prec, z))) return rc;
  }
  for (int col = first; col < L.g.ncolors; ++col) {
    const int64_t a = L.g.off[col], b = L.g.off[col + 1];
    if (b <= a) continue;
    if ((rc = gs_pass_launch<T>(c, L, a, b - a, r, z, nullptr, nullptr, -1, c->gs_rev && (col & 1)))) return rc;
  }
  return HPG_OK;
}

template <typename T>
bool spmv_tma_ok(hpg_ctx* c, const Level& L, int rows);
template <typename T, int MODE>
int spmv_tma(hpg_ctx* c, Level& L, const T* x, const T* b, T* y, double* partial, int64_t* nblocks,
             const int32_t* dst = nullptr, int64_t rows = -1);

template <typename T>
int restrict_(hpg_ctx* c, int l, const T* rf, const T* zf, T* rcoarse) {
  Timed tm(c, M_RESTRICT);
  Level& F = c->lev[l];
  Level& C = c->lev[l + 1];
  if (!C.f2c && spmv_tma_ok<T>(c, F, c->restr_cfg[sizeof(T) == 4] / 100)) {
    // the fine colour-0 rows [0, C.n) with staged values; rc[inj[j]] = r[j] - (A z)[j]
    return spmv_tma<T, 2>(c, F, zf, rf, rcoarse, nullptr, nullptr, (const int32_t*)C.inj, C.n);
  }
  if (C.f2c)
    CUDA_TRY(launch_pdl(c, hpg::k_restrict_gen<T>, grid_for(C.n), 256, F.cols, (const T*)vals_of<T>(F), F.ld, C.n,
                        (const int32_t*)C.f2c, rf, zf, rcoarse));
  else
    CUDA_TRY(launch_pdl(c, hpg::k_restrict<T>, grid_for(C.n), 256, F.cols, (const T*)vals_of<T>(F), F.ld, C.n,
                        (const int32_t*)C.inj, rf, zf, rcoarse, stencil_of(c, F)));
  ++c->launches;
  return HPG_OK;
}

template <typename T>
int prolong_(hpg_ctx* c, int l, T* zf, const T* zc) {
  Timed tm(c, M_PROLONG);
  Level& C = c->lev[l + 1];
  if (C.f2c)
    CUDA_TRY(launch_pdl(c, hpg::k_prolong_gen<T>, grid_for(C.n), 256, C.n, (const int32_t*)C.f2c, zf, zc));
  else
    CUDA_TRY(launch_pdl(c, hpg::k_prolong<T>, grid_for(C.n), 256, C.n, (const int32_t*)C.inj, zf, zc));
  ++c->launches;
  return HPG_OK;
}

template <typename T>
T* lev_z(Level& L);
template <>
double* lev_z<double>(Level& L) { return L.z64; }
template <>
float* lev_z<float>(Level& L) { return L.z32; }
template <typename T>
T* lev_r(Level& L);
template <>
double* lev_r<double>(Level& L) { return L.r64; }
template <>
float* lev_r<float>(Level& L) { return L.r32; }

template <typename T>
int vcycle_tail(hpg_ctx* c, int l, const T* r, T* z) {
  Timed tm(c, M_GS);
  hpg::TailParams<T> p;
  memset(&p, 0, sizeof p);
  p.nl = c->nlev - l;
  p.nu1 = c->nu1;
  p.nu2 = c->nu2;
  p.nu_c = c->nu_c;
  for (int k = 0; k < p.nl; ++k) {
    Level& L = c->lev[l + k];
    hpg::TailLevel<T>& t = p.lv[k];
    t.cols = L.cols;
    t.vals = vals_of<T>(L);
    t.inj = L.inj;
    t.z = k == 0 ? z : lev_z<T>(L);
    t.r = k == 0 ? (T*)r : lev_r<T>(L);
    t.ld = L.ld;
    t.n = L.n;
    t.n_ext = L.n_ext;
    for (int q = 0; q < 9; ++q) t.off[q] = L.g.off[q];
    t.ncolors = L.g.ncolors;
  }
  if (c->tail_cluster > 0) {
    // the whole tail on ONE thread-block cluster (hardware cluster barrier)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c->tail_cluster);
    cfg.blockDim = dim3(256);
    cfg.stream = c->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = c->tail_cluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CUDA_TRY(cudaLaunchKernelEx(&cfg, hpg::k_vcycle_tail<T, true>, p));
  } else {
    const int blocks = c->tail_blocks[sizeof(T) == 4];
    void* args[] = {(void*)&p};
    CUDA_TRY(cudaLaunchCooperativeKernel((const void*)hpg::k_vcycle_tail<T, false>, dim3(blocks), dim3(256), args,
                                         0, c->stream));
  }
  ++c->launches;
  return HPG_OK;
}

void set_tail_cluster(hpg_ctx* c, int v) {
  c->tail_cluster = std::max(0, std::min(v, 16));
  if (c->tail_cluster > 8) {  // non-portable cluster sizes (up to 16) must be opted into
    cudaFuncSetAttribute(hpg::k_vcycle_tail<double, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(hpg::k_vcycle_tail<float, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  }
}

// V-cycle with zero initial guess (ref: multigrid.py:140-171)
template <typename T>
int vcycle(hpg_ctx* c, int l, const T* r, T* z) {
  if (c->nranks == 1 && l > 0 && c->lev[l].n <= c->tail_rows && c->nlev - l <= hpg::kMaxTail && !c->general)
    return vcycle_tail<T>(c, l, r, z);
  const bool last = l == c->nlev - 1;
  const int sweeps = last ? c->nu_c : c->nu1;
  int rc;
  for (int s = 0; s < sweeps; ++s)
    if ((rc = gs_sweep<T>(c, l, r, z, s == 0))) return rc;
  if (last) return HPG_OK;
  if ((rc = do_exchange(c, l, sizeof(T) == 8 ? HPG_F64 : HPG_F32, z))) return rc;
  Level& C = c->lev[l + 1];
  if ((rc = restrict_<T>(c, l, r, z, lev_r<T>(C)))) return rc;
  if ((rc = vcycle<T>(c, l + 1, lev_r<T>(C), lev_z<T>(C)))) return rc;
  if ((rc = prolong_<T>(c, l, z, lev_z<T>(C)))) return rc;
  for (int s = 0; s < c->nu2; ++s)
    if ((rc = gs_sweep<T>(c, l, r, z, 0))) return rc;
  return HPG_OK;
}

// Fixed-order fold of fp64 dot partials [cnt][nb] -> scal[0..cnt), the
// rank-ordered all-reduce, then one rounding to T (+ sqrt for beta).
template <typename T>
int fold_dots(hpg_ctx* c, const double* part, int nb, int cnt, double* out, bool do_sqrt) {
  hpg::k_fold<double><<<1, 1024, 0, c->stream>>>(part, nb, cnt, out, 0);
  LAUNCH_CHECK();
  ++c->launches;
  int rc = allreduce_scal<double>(c, out, cnt);
  if (rc) return rc;
  hpg::k_round_dots<T><<<1, 64, 0, c->stream>>>(out, cnt, do_sqrt ? 1 : 0);
  LAUNCH_CHECK();
  ++c->launches;
  return HPG_OK;
}

template <typename T, int KB>
int cgs2_kb(hpg_ctx* c, T* Q, int64_t ldq, int kb, T* w, T* qnext) {
  const int64_t n = c->lev[0].n;
  double* part = (double*)c->partial;
  double* scal = (double*)c->scal;
  const int nb = c->nb;
  int rc;
  hpg::k_dots<T, KB><<<nb, 256, 0, c->stream>>>(Q, ldq, kb, w, n, part);
  if ((rc = fold_dots<T>(c, part, nb, kb, scal, false))) return rc;
  hpg::k_cgs_sub_dots<T, KB><<<nb, 256, 0, c->stream>>>(Q, ldq, kb, w, n, scal, part);
  if ((rc = fold_dots<T>(c, part, nb, kb, scal + 64, false))) return rc;
  hpg::k_cgs_sub_norm<T, KB><<<nb, 256, 0, c->stream>>>(Q, ldq, kb, w, n, scal + 64, part);
  LAUNCH_CHECK();
  c->launches += 3;
  if (qnext) {
    if ((rc = fold_dots<T>(c, part, nb, 1, scal + 128, true))) return rc;
    hpg::k_scale<T><<<grid_for(n), 256, 0, c->stream>>>(w, scal + 128, qnext, n);
    LAUNCH_CHECK();
    c->launches += 1;
  }
  return HPG_OK;
}

// single-rank CGS2: one cooperative launch (csrc/hpg_cgs.cuh)
template <typename T, int WR, int RPW, int U, int MINB = 2>
int cgs2_fused(hpg_ctx* c, T* Q, int64_t ldq, int kb, T* w, T* qnext) {
  hpg::CgsParams<T> p;
  memset(&p, 0, sizeof p);
  p.Q = Q;
  p.w = w;
  p.qnext = qnext;
  p.partial = (double*)c->partial;
  p.scal = (double*)c->scal;
  p.ldq = ldq;
  p.n = c->lev[0].n;
  p.kb = kb;
  p.zigzag = c->cgs_zigzag;
  p.solo_fold = c->cgs_solo;
  p.ar = p2p_ar(c);
  p.seq0 = c->ar_seq + 1;
  if (c->nranks > 1) c->ar_seq += qnext ? 3 : 2;
  if (ldq % 32) return fail(HPG_E_ARG, "basis row stride must be a multiple of 32 elements");
  auto fn = hpg::k_cgs2_fused<T, WR, RPW, U, MINB>;
  int per = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, hpg::kCgsThreads, 0));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  const int blocks = std::min(std::max(1, per), 8) * sms;
  void* args[] = {(void*)&p};
  CUDA_TRY(cudaLaunchCooperativeKernel((const void*)fn, dim3(blocks), dim3(hpg::kCgsThreads), args, 0, c->stream));
  ++c->launches;
  return HPG_OK;
}

// multi-rank CGS2: the same streaming passes, one launch each, with the
// rank-ordered all-reduce (NCCL all-gather + ordered fold) between them
template <typename T, int WR, int RPW, int U>
int cgs2_passes(hpg_ctx* c, T* Q, int64_t ldq, int kb, T* w, T* qnext) {
  hpg::CgsParams<T> p;
  memset(&p, 0, sizeof p);
  p.Q = Q;
  p.w = w;
  p.qnext = qnext;
  p.partial = (double*)c->partial;
  p.scal = (double*)c->scal;
  p.ldq = ldq;
  p.n = c->lev[0].n;
  p.kb = kb;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  const int grid = 2 * sms;
  double* scal = (double*)c->scal;
  int rc;
  hpg::k_cgs_onepass<T, WR, RPW, U, 0><<<grid, hpg::kCgsThreads, 0, c->stream>>>(p, (const double*)nullptr);
  if ((rc = fold_dots<T>(c, p.partial, grid, kb, scal, false))) return rc;
  hpg::k_cgs_onepass<T, WR, RPW, U, 1><<<grid, hpg::kCgsThreads, 0, c->stream>>>(p, (const double*)scal);
  if ((rc = fold_dots<T>(c, p.partial, grid, kb, scal + 64, false))) return rc;
  hpg::k_cgs_onepass<T, WR, RPW, U, 2><<<grid, hpg::kCgsThreads, 0, c->stream>>>(p, (const double*)(scal + 64));
  LAUNCH_CHECK();
  c->launches += 3;
  if (qnext) {
    if ((rc = fold_dots<T>(c, p.partial, grid, 1, scal + 128, true))) return rc;
    hpg::k_scale<T><<<grid_for(p.n), 256, 0, c->stream>>>(w, scal + 128, qnext, p.n);
    LAUNCH_CHECK();
    c->launches += 1;
  }
  return HPG_OK;
}

// Enqueue one CGS2 step (+ norm + normalise when qnext) and the async copy of
// (h1, h2, beta) to pinned host memory; cgs2_finish waits for it.  Splitting
// the two lets the host enqueue the next Arnoldi step's V-cycle and SpMV
// before it blocks on this step's coefficients.
// (WR, RPW, U) of the fused kernel per basis size: encoded WR*100 + RPW*10 + U
// (RPW < 10).  HPG_CGS_CFG="kbmax:code,kbmax:code,..." overrides (tuning).
int cgs_config(hpg_ctx* c, int kb) {
  // code: [MINB * 1000 +] WR * 100 + RPW * 10 + U (MINB: CTAs per SM the kernel is built for, default 2)
  if (c->cgs_force > 0 && ((c->cgs_force % 1000) / 100) * ((c->cgs_force / 10) % 10) >= kb) return c->cgs_force;
  if (c->cgs_cfg.empty()) {
    const char* e = getenv("HPG_CGS_CFG");
    if (e) {
      int kbm, code, off = 0, used = 0;
      while (sscanf(e + off, "%d:%d%n", &kbm, &code, &used) == 2) {
        c->cgs_cfg.push_back({kbm, code});
        off += used;
        if (e[off] == ',') ++off;
      }
    }
    if (c->cgs_cfg.empty())
      // r02 re-sweeps (tools/cgs_sweep.py): kb 5-8 with 2 row groups x 4 rows (kb 6: 396 -> 354 us);
      // kb 9-14 with 2 x 8 rows (kb 12: 579 -> 549 us); kb 15-16 with 4 x 4 rows built for 3 CTAs
      // per SM (kb 16: 677 -> 643 us)
      c->cgs_cfg = {{1, 118}, {2, 218}, {4, 418}, {8, 242}, {14, 281}, {16, 3441}, {24, 461}, {32, 481}, {64, 881}};
  }
  for (const auto& e : c->cgs_cfg)  // a configuration must hold all kb rows (WR * RPW >= kb)
    if (kb <= e.first && ((e.second % 1000) / 100) * ((e.second / 10) % 10) >= kb) return e.second;
  return 881;
}

template <typename T>
int cgs2_fused_dispatch(hpg_ctx* c, int code, T* Q, int64_t ldq, int kb, T* w, T* qnext) {
  switch (code) {
#define HPG_CGS_CASE(WR, RPW, U) \
  case WR * 100 + RPW * 10 + U:  \
    return cgs2_fused<T, WR, RPW, U>(c, Q, ldq, kb, w, qnext);
    HPG_CGS_CASE(1, 1, 8)
    HPG_CGS_CASE(2, 1, 8)
    HPG_CGS_CASE(4, 1, 8)
    HPG_CGS_CASE(8, 1, 8)
    HPG_CGS_CASE(4, 2, 4)
    HPG_CGS_CASE(8, 2, 4)
    HPG_CGS_CASE(4, 2, 2)
    HPG_CGS_CASE(4, 3, 2)
    HPG_CGS_CASE(8, 3, 2)
    HPG_CGS_CASE(4, 4, 2)
    HPG_CGS_CASE(8, 4, 2)
    HPG_CGS_CASE(4, 4, 1)
    HPG_CGS_CASE(2, 4, 2)
    HPG_CGS_CASE(2, 8, 1)
    HPG_CGS_CASE(4, 6, 1)
    HPG_CGS_CASE(8, 6, 1)
    HPG_CGS_CASE(4, 8, 1)
    HPG_CGS_CASE(8, 8, 1)
#undef HPG_CGS_CASE
#define HPG_CGS3_CASE(WR, RPW, U)        \
  case 3000 + WR * 100 + RPW * 10 + U:  \
    return cgs2_fused<T, WR, RPW, U, 3>(c, Q, ldq, kb, w, qnext);
    HPG_CGS3_CASE(4, 4, 1)
    HPG_CGS3_CASE(8, 4, 1)
    HPG_CGS3_CASE(8, 3, 1)
    HPG_CGS3_CASE(4, 2, 2)
    HPG_CGS3_CASE(8, 2, 2)
#undef HPG_CGS3_CASE
  }
  return fail(HPG_E_ARG, "unknown CGS2 configuration %d", code);
}

template <typename T>
int cgs2_launch_t(hpg_ctx* c, T* Q, int64_t ldq, int k, T* w, T* qnext) {
  const int kb = k + 1;
  if (kb > 64) return fail(HPG_E_UNSUPPORTED, "restart basis of %d vectors exceeds 64", kb);
  const bool vec_ok = c->lev[0].n % (16 / (int)sizeof(T)) == 0 && ldq % 32 == 0;
  int rc;
  {
    Timed tm(c, M_ORTHO);
    if (c->nranks > 1 && !c->p2p && c->cgs_fused && vec_ok) {
      if (kb <= 1) rc = cgs2_passes<T, 1, 1, 8>(c, Q, ldq, kb, w, qnext);
      else if (kb <= 2) rc = cgs2_passes<T, 2, 1, 8>(c, Q, ldq, kb, w, qnext);
      else if (kb <= 4) rc = cgs2_passes<T, 4, 1, 8>(c, Q, ldq, kb, w, qnext);
      else if (kb <= 8) rc = cgs2_passes<T, 4, 2, 4>(c, Q, ldq, kb, w, qnext);
      else if (kb <= 16) rc = cgs2_passes<T, 8, 2, 4>(c, Q, ldq, kb, w, qnext);
      else if (kb <= 32) rc = cgs2_passes<T, 8, 4, 2>(c, Q, ldq, kb, w, qnext);
      else rc = cgs2_passes<T, 8, 8, 1>(c, Q, ldq, kb, w, qnext);
    } else if ((c->nranks == 1 || c->p2p) && c->cgs_fused && vec_ok) {
      rc = cgs2_fused_dispatch<T>(c, cgs_config(c, kb), Q, ldq, kb, w, qnext);
    } else {
      if (kb <= 4) rc = cgs2_kb<T, 4>(c, Q, ldq, kb, w, qnext);
      else if (kb <= 8) rc = cgs2_kb<T, 8>(c, Q, ldq, kb, w, qnext);
      else if (kb <= 16) rc = cgs2_kb<T, 16>(c, Q, ldq, kb, w, qnext);
      else if (kb <= 32) rc = cgs2_kb<T, 32>(c, Q, ldq, kb, w, qnext);
      else rc = cgs2_kb<T, 64>(c, Q, ldq, kb, w, qnext);
    }
    if (rc) return rc;
  }
  CUDA_TRY(cudaMemcpyAsync(c->pinned, c->scal, 129 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaEventRecord(c->ev_cgs, c->stream));
  c->cgs_pending_kb = kb;
  c->cgs_pending_es = (int)sizeof(T);
  c->cgs_pending_norm = qnext != nullptr;
  return HPG_OK;
}

int cgs2_finish(hpg_ctx* c, double* out) {
  if (c->cgs_pending_kb <= 0) return fail(HPG_E_ARG, "no CGS2 step in flight");
  if (getenv("HPG_CGS_STREAMSYNC")) CUDA_TRY(cudaStreamSynchronize(c->stream));
  else CUDA_TRY(cudaEventSynchronize(c->ev_cgs));
  const int kb = c->cgs_pending_kb;
  // fp64 slots holding values rounded to the solve's precision
  for (int j = 0; j < kb; ++j) {
    out[j] = c->pinned[j];
    out[kb + j] = c->pinned[64 + j];
  }
  out[2 * kb] = c->cgs_pending_norm ? c->pinned[128] : 0.0;
  c->cgs_pending_kb = 0;
  return HPG_OK;
}

template <typename T>
int cgs2_t(hpg_ctx* c, T* Q, int64_t ldq, int k, T* w, T* qnext, double* out) {
  int rc = cgs2_launch_t<T>(c, Q, ldq, k, w, qnext);
  return rc ? rc : cgs2_finish(c, out);
}

template <typename T, int WR, int RPW, int U>
int gemv_launch(hpg_ctx* c, const T* Q, int64_t ldq, int k, T* out) {
  hpg::CgsParams<T> p;
  memset(&p, 0, sizeof p);
  p.Q = Q;
  p.w = out;
  p.scal = (double*)c->scal + 320;
  p.ldq = ldq;
  p.n = c->lev[0].n;
  p.kb = k;
  int per = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, hpg::k_gemv_combine<T, WR, RPW, U>, hpg::kCgsThreads, 0));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  hpg::k_gemv_combine<T, WR, RPW, U><<<std::max(1, per) * sms, hpg::kCgsThreads, 0, c->stream>>>(p);
  LAUNCH_CHECK();
  ++c->launches;
  return HPG_OK;
}

// out = Q[0:k]^T y with y narrowed to T on the host first (ref: krylov.py:288-289)
template <typename T>
int gemv_t(hpg_ctx* c, const T* Q, int64_t ldq, int k, const double* y, T* out) {
  Timed tm(c, M_ORTHO);
  if (k > 64) return fail(HPG_E_UNSUPPORTED, "restart length %d exceeds 64", k);
  if (ldq % 32 || c->lev[0].n % (16 / (int)sizeof(T))) return fail(HPG_E_ARG, "unaligned basis for gemv");
  double ys[64];
  for (int j = 0; j < k; ++j) ys[j] = (double)(T)y[j];
  CUDA_TRY(cudaMemcpyAsync((double*)c->scal + 320, ys, k * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  if (k <= 1) return gemv_launch<T, 1, 1, 8>(c, Q, ldq, k, out);
  if (k <= 2) return gemv_launch<T, 2, 1, 8>(c, Q, ldq, k, out);
  if (k <= 4) return gemv_launch<T, 4, 1, 8>(c, Q, ldq, k, out);
  if (k <= 8) return gemv_launch<T, 4, 2, 4>(c, Q, ldq, k, out);
  if (k <= 16) return gemv_launch<T, 8, 2, 4>(c, Q, ldq, k, out);
  if (k <= 32) return gemv_launch<T, 8, 4, 2>(c, Q, ldq, k, out);
  return gemv_launch<T, 8, 8, 1>(c, Q, ldq, k, out);
}

void free_level(Level& L) {
  for (void* p : {(void*)L.cols, (void*)L.v64, (void*)L.v32, (void*)L.inj, (void*)L.send_idx, L.send_buf,
                  (void*)L.z64, (void*)L.z32, (void*)L.r64, (void*)L.r32, (void*)L.hflag, (void*)L.bnd,
                  (void*)L.bnd0, (void*)L.f2c, (void*)L.perm_d, (void*)L.iperm_d, (void*)L.wave_items,
                  (void*)L.wave_done, (void*)L.lcols, (void*)L.lv64, (void*)L.lv32, (void*)L.dg64, (void*)L.dg32})
    if (p) cudaFree(p);
  L = Level();
}

template <typename P>
int dmalloc(P** p, size_t bytes, size_t* acc) {
  void* q = nullptr;
  CUDA_TRY(cudaMalloc(&q, std::max<size_t>(bytes, 16)));
  *p = (P*)q;
  if (acc) *acc += bytes;
  return HPG_OK;
}

// Strictly-lower part of every color block (hpg_lower.cuh), from the ELL rows.
int build_lower(hpg_ctx* c, Level& L) {
  L.lower_ok = false;
  for (void* p : {(void*)L.lcols, (void*)L.lv64, (void*)L.lv32, (void*)L.dg64, (void*)L.dg32})
    if (p) cudaFree(p);
  L.lcols = nullptr, L.lv64 = nullptr, L.lv32 = nullptr, L.dg64 = nullptr, L.dg32 = nullptr;
  const int nc = L.g.ncolors;
  char* scratch = nullptr;  // setup-time scratch: widths, then the per-color table
  CUDA_TRY(cudaMalloc(&scratch, 4096));
  int* wd = (int*)scratch;
  CUDA_TRY(cudaMemsetAsync(wd, 0, hpg::kMaxColors * sizeof(int), c->stream));
  hpg::k_lower_count<<<grid_for(L.n), 256, 0, c->stream>>>(L.g, L.ld, L.cols, L.v64, wd);
  LAUNCH_CHECK();
  int w[hpg::kMaxColors] = {0};
  CUDA_TRY(cudaMemcpyAsync(w, wd, sizeof w, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  int64_t tot = 0;
  for (int k = 0; k < nc; ++k) {
    if (w[k] > 27) return fail(HPG_E_ARG, "lower width %d", w[k]);
    L.lc[k].w = w[k];
    L.lc[k].ldc = pad_ld(L.g.off[k + 1] - L.g.off[k]);  // odd multiple of 128 B: no L2-slice aliasing
    L.lc[k].base = tot;
    tot += (int64_t)w[k] * L.lc[k].ldc;
  }
  int rc;
  size_t* acc = nullptr;  // accounted in L.bytes below
  if ((rc = dmalloc(&L.lcols, std::max<int64_t>(1, tot) * 4, acc))) return rc;
  if ((rc = dmalloc(&L.lv64, std::max<int64_t>(1, tot) * 8, acc))) return rc;
  if ((rc = dmalloc(&L.lv32, std::max<int64_t>(1, tot) * 4, acc))) return rc;
  if ((rc = dmalloc(&L.dg64, L.n * 8, acc))) return rc;
  if ((rc = dmalloc(&L.dg32, L.n * 4, acc))) return rc;
  L.bytes += tot * 16 + L.n * 12;
  hpg::LowerColor* lcd = (hpg::LowerColor*)(scratch + 1024);
  CUDA_TRY(cudaMemcpyAsync(lcd, L.lc, nc * sizeof(hpg::LowerColor), cudaMemcpyHostToDevice, c->stream));
  hpg::k_lower_fill<<<grid_for(L.n), 256, 0, c->stream>>>(L.g, L.ld, L.cols, L.v64, lcd, L.lcols, L.lv64, L.lv32,
                                                           L.dg64, L.dg32);
  LAUNCH_CHECK();
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  cudaFree(scratch);
  L.lower_ok = true;
  return HPG_OK;
}

// Implicit-index rows (hpg_kernels.cuh Stencil): eligible for the greedy
// layout with even local extents (8 equal color blocks); every row that takes
// the closed form is compared with its stored ELL columns, and any mismatch
// leaves the level on the index stream.
int build_stencil(hpg_ctx* c, Level& L) {
  L.st = hpg::Stencil{};
  L.st_rows = 0;
  L.st_lower = false;
  const Geom& g = L.g;
  if (!L.n || g.perm_tab || g.ncolors != 8 || ((g.lx | g.ly | g.lz) & 1) || g.lx < 2 || g.ly < 2 || g.lz < 2 ||
      L.n >= (int64_t{1} << 31))
    return HPG_OK;
  const int64_t n8 = L.n / 8;
  for (int k = 0; k <= 8; ++k)
    if (g.off[k] != k * n8) return HPG_OK;
  hpg::Stencil st{};
  st.on = 1;
  st.n8 = (uint32_t)n8;
  st.hx = (uint32_t)(g.lx / 2);
  st.hy = (uint32_t)(g.ly / 2);
  st.hxy = st.hx * st.hy;
  st.lx = g.lx;
  st.ly = g.ly;
  st.lz = g.lz;
  st.bx = g.bit[0];
  st.by = g.bit[1];
  st.bz = g.bit[2];
  st.cx = st.n8 << st.bx;
  st.cy = st.n8 << st.by;
  st.cz = st.n8 << st.bz;
  st.ifc = (g.ox > 0) | ((g.ox + g.lx < g.gx) << 1) | ((g.oy > 0) << 2) | ((g.oy + g.ly < g.gy) << 3) |
           ((g.oz > 0) << 4) | ((g.oz + g.lz < g.gz) << 5);
  auto magic = [](uint64_t d) { return d == 1 ? uint64_t{0} : ~uint64_t{0} / d + 1; };  // ceil(2^64 / d); d = 1 special-cased
  st.mn8 = magic(st.n8);
  st.mhxy = magic(st.hxy);
  st.mhx = magic(st.hx);
  void* scratch = nullptr;
  CUDA_TRY(cudaMalloc(&scratch, 16));
  CUDA_TRY(cudaMemsetAsync(scratch, 0, 16, c->stream));
  unsigned long long* rows = (unsigned long long*)scratch;
  unsigned int* bad = (unsigned int*)((char*)scratch + 8);
  hpg::k_check_stencil<<<grid_for(L.n), 256, 0, c->stream>>>(L.cols, L.ld, L.n, st, bad, rows);
  LAUNCH_CHECK();
  // lower ELL (zero-guess sweeps): the compile-time offset lists of
  // k_gs_lower_st assume parity bits x->0, y->1, z->2 and W_c = lower_width(c)
  bool lower = L.lower_ok && st.bx == 0 && st.by == 1 && st.bz == 2;
  for (int k = 0; lower && k < 8; ++k) lower = L.lc[k].w == hpg::lower_width(k);
  unsigned int* bad_lower = (unsigned int*)((char*)scratch + 12);
  if (lower)
    for (int k = 0; k < 8; ++k) {
      hpg::check_lower_st_kernel(k)<<<grid_for(n8), 256, 0, c->stream>>>(L.lcols + L.lc[k].base, L.lc[k].ldc, n8, st,
                                                                          bad_lower);
      LAUNCH_CHECK();
    }
  unsigned long long h[2] = {0, 0};
  CUDA_TRY(cudaMemcpyAsync(h, scratch, 16, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  cudaFree(scratch);
  if ((unsigned int)h[1] == 0) {
    L.st = st;
    L.st_rows = (int64_t)h[0];
    L.st_lower = lower && (unsigned int)(h[1] >> 32) == 0;
  }
  return HPG_OK;
}

// (Re)build a level's permutation-dependent structure: ELL rows, send lists and
// the interior/boundary split.  `first` allocates the send/split buffers.
int build_structure(hpg_ctx* c, Level& L, bool first) {
  int rc;
  if (L.n) {
    hpg::k_build_level<<<grid_for(L.n, 128), 128, 0, c->stream>>>(L.g, L.ld, L.cols, L.v64, L.v32);
    LAUNCH_CHECK();
    if ((rc = build_lower(c, L))) return rc;
    if ((rc = build_stencil(c, L))) return rc;
  }
  // halo plan: one send list per neighbour, in ascending neighbour rank
  struct Tmp {
    int rank, idx, sx, sy, sz;
  };
  std::vector<Tmp> t;
  for (int i = 0; i < 27; ++i)
    if (L.g.nbr_rank[i] >= 0) t.push_back({L.g.nbr_rank[i], i, i % 3 - 1, (i / 3) % 3 - 1, i / 9 - 1});
  std::sort(t.begin(), t.end(), [](const Tmp& a, const Tmp& b) { return a.rank < b.rank; });
  if (first) {
    int64_t off = 0;
    for (auto& e : t) {
      const int64_t cnt = hpg::region_size(L.g, e.sx, e.sy, e.sz);
      L.nbrs.push_back({e.rank, e.idx, off, cnt, L.g.halo_base[e.idx]});
      off += cnt;
    }
    L.send_total = off;
    if (off) {
      if ((rc = dmalloc(&L.send_idx, off * 4, &L.bytes))) return rc;
      if ((rc = dmalloc((char**)&L.send_buf, off * 8, &L.bytes))) return rc;
    }
  }
  for (size_t i = 0; i < t.size(); ++i) {
    const Nbr& nb = L.nbrs[i];
    hpg::k_build_send<<<grid_for(nb.cnt), 256, 0, c->stream>>>(L.g, t[i].sx, t[i].sy, t[i].sz, nb.cnt,
                                                                L.send_idx + nb.send_off);
    LAUNCH_CHECK();
  }
  if (!L.nbrs.empty() && L.n) {
    // interior / boundary split for the overlapped exchange
    if (first && (rc = dmalloc(&L.hflag, L.n, &L.bytes))) return rc;
    hpg::k_build_halo_flags<<<grid_for(L.n), 256, 0, c->stream>>>(L.g, L.hflag);
    LAUNCH_CHECK();
    std::vector<uint8_t> f(L.n);
    CUDA_TRY(cudaMemcpyAsync(f.data(), L.hflag, L.n, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    std::vector<int32_t> all, c0;
    for (int64_t i = 0; i < L.n; ++i)
      if (f[i]) {
        all.push_back((int32_t)i);
        if (i < L.g.off[1]) c0.push_back((int32_t)i);
      }
    L.nbnd = (int64_t)all.size();
    L.nbnd0 = (int64_t)c0.size();
    if (L.bnd) cudaFree(L.bnd);
    if (L.bnd0) cudaFree(L.bnd0);
    L.bnd = L.bnd0 = nullptr;
    if ((rc = dmalloc(&L.bnd, std::max<int64_t>(1, L.nbnd) * 4, &L.bytes))) return rc;
    if ((rc = dmalloc(&L.bnd0, std::max<int64_t>(1, L.nbnd0) * 4, &L.bytes))) return rc;
    if (L.nbnd) CUDA_TRY(cudaMemcpy(L.bnd, all.data(), L.nbnd * 4, cudaMemcpyHostToDevice));
    if (L.nbnd0) CUDA_TRY(cudaMemcpy(L.bnd0, c0.data(), L.nbnd0 * 4, cudaMemcpyHostToDevice));
  }
  return HPG_OK;
}

// Dataflow sweep plan for a greedy (closed-form) level with every extent >= 2:
// color c = px + 2 py + 4 pz; its half-plane Z holds hx(px) * hy(py) rows.
int build_wave(hpg_ctx* c, Level& L) {
  L.wave_ok = false;
  const Geom& g = L.g;
  if (g.perm_tab || g.ncolors != 8 || g.lx < 2 || g.ly < 2 || g.lz < 2 || !L.n) return HPG_OK;
  hpg::WaveLevel& w = L.wave;
  memset(&w, 0, sizeof w);
  w.ncolors = 8;
  for (int k = 0; k <= hpg::kMaxColors; ++k) w.off[k] = g.off[k];
  int maxp = 0;
  for (int col = 0; col < 8; ++col) {
    const int px = col & 1, py = (col >> 1) & 1, pz = (col >> 2) & 1;
    w.planes[col] = (g.lz - pz + 1) / 2;
    w.plane[col] = (int64_t)((g.lx - px + 1) / 2) * ((g.ly - py + 1) / 2);
    w.chunks[col] = (int)cdiv(w.plane[col], hpg::kWaveRows);
    if (w.chunks[col] > 255 || w.planes[col] > 65535) return HPG_OK;
    maxp = std::max(maxp, w.planes[col]);
  }
  w.maxplanes = maxp;
  // wavefront order t = Z + lag * c: a larger lag puts an item's producers
  // (color c-1, planes Z-1..Z+1) further ahead in the deal, so co-resident
  // blocks rarely wait; the live window of z grows as lag * 8 half-planes
  const int lag = c->wave_lag;
  std::vector<int32_t> items;
  for (int t = 0; t < maxp + lag * 8; ++t)
    for (int col = 0; col < 8; ++col) {
      const int Z = t - lag * col;
      if (Z < 0 || Z >= w.planes[col]) continue;
      for (int q = 0; q < w.chunks[col]; ++q) items.push_back((col << 24) | (Z << 8) | q);
    }
  w.nitems = (int64_t)items.size();
  int rc;
  if ((rc = dmalloc(&L.wave_items, items.size() * 4, &L.bytes))) return rc;
  if ((rc = dmalloc(&L.wave_done, ((size_t)8 * maxp + 2) * 4, &L.bytes))) return rc;
  CUDA_TRY(cudaMemcpy(L.wave_items, items.data(), items.size() * 4, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemset(L.wave_done, 0, ((size_t)8 * maxp + 2) * 4));
  w.items = L.wave_items;
  w.done = L.wave_done;
  w.ctl = L.wave_done + (size_t)8 * maxp;
  L.wave_ok = true;
  return HPG_OK;
}

int build_level(hpg_ctx* c, Level& L, const int dims[3]) {
  L.g = make_geom(dims, c->coords, c->procs);
  L.n = L.g.n;
  L.n_ext = L.n + L.g.halo_size;
  L.ld = pad_ld(L.n);
  L.nnz = geom_nnz(L.g);
  if (L.n_ext >= (int64_t)1 << 31) return fail(HPG_E_ARG, "level too large for int32 columns");
  int rc;
  const size_t slots = (size_t)27 * L.ld;
  if ((rc = dmalloc(&L.cols, slots * 4, &L.bytes))) return rc;
  if ((rc = dmalloc(&L.v64, slots * 8, &L.bytes))) return rc;
  if ((rc = dmalloc(&L.v32, slots * 4, &L.bytes))) return rc;
  CUDA_TRY(cudaMemsetAsync(L.cols, 0, slots * 4, c->stream));
  CUDA_TRY(cudaMemsetAsync(L.v64, 0, slots * 8, c->stream));
  CUDA_TRY(cudaMemsetAsync(L.v32, 0, slots * 4, c->stream));
  if ((rc = build_structure(c, L, true))) return rc;
  if ((rc = build_wave(c, L))) return rc;
  if ((rc = dmalloc(&L.z64, L.n_ext * 8, &L.bytes))) return rc;
  if ((rc = dmalloc(&L.z32, L.n_ext * 4, &L.bytes))) return rc;
  if ((rc = dmalloc(&L.r64, L.n * 8, &L.bytes))) return rc;
  if ((rc = dmalloc(&L.r32, L.n * 4, &L.bytes))) return rc;
  CUDA_TRY(cudaMemsetAsync(L.z64, 0, L.n_ext * 8, c->stream));
  CUDA_TRY(cudaMemsetAsync(L.z32, 0, L.n_ext * 4, c->stream));
  return HPG_OK;
}

int check_prec(int prec) { return prec == HPG_F64 || prec == HPG_F32 ? HPG_OK : fail(HPG_E_ARG, "bad prec %d", prec); }
int check_level(hpg_ctx* c, int l) {
  if (!c) return fail(HPG_E_ARG, "null context");
  return l >= 0 && l < c->nlev ? HPG_OK : fail(HPG_E_ARG, "level %d out of range", l);
}

// ---- SpMV / residual with tensor-copy staged values (hpg_tma.cuh k_spmv_tma)

template <typename T, int R, int MB, int MODE>
int spmv_tma_t(hpg_ctx* c, Level& L, const T* x, const T* b, T* y, double* partial, int64_t* nblocks,
               const int32_t* dst = nullptr, int64_t rows = -1) {
  hpg::SpmvPlan p;
  memset(&p, 0, sizeof p);
  int rc0 = encode_value_map<T>(c, L, R, &p.vmap);
  if (rc0) return rc0;
  p.cols = L.cols;
  p.ld = L.ld;
  p.n = L.n;
  p.st = stencil_of(c, L);
  if (p.st.on && p.st.n8 % R == 0) {
    p.n8 = p.st.n8;
    uint32_t km;
    for (int col = 0; col < 8; ++col) stencil_offsets(p.st, col, p.doff[col], &km);
    p.xface = (c->face_cols & 16) ? 1 : 0;
    if (!(c->face_cols & 1)) p.st.ifc = 63;  // face rows read the index plane
  } else {
    p.st.on = 0;
  }
  const int ilv = MODE == 2 ? 1 : std::max(1, c->spmv_ilv[sizeof(T) == 4]);
  p.ilv = ilv;
  p.skip = MODE == 0 ? c->pass_skip : nullptr;
  if (rows >= 0) p.n = rows;  // MODE 2: the fine colour-0 rows
  const int64_t nbk = cdiv(p.n, R);
  if (nblocks) *nblocks = nbk;
  const int grid = (int)(cdiv(nbk, ilv) * ilv);
  CUDA_TRY(launch_pdl_smem(c, hpg::k_spmv_tma<T, R, MB, MODE>, grid, R, (size_t)27 * R * sizeof(T) + 16, p, x, b, y,
                           partial, dst));
  ++c->launches;
  return HPG_OK;
}

template <typename T, int MODE>
int spmv_tma(hpg_ctx* c, Level& L, const T* x, const T* b, T* y, double* partial, int64_t* nblocks,
             const int32_t* dst, int64_t rows) {
  const int code = MODE == 1 ? c->resid_cfg : MODE == 2 ? c->restr_cfg[sizeof(T) == 4] : c->spmv_cfg[sizeof(T) == 4];
#define HPG_SPMV_CASE(TT, R, MB, MD)                                                                  \
  if (std::is_same<T, TT>::value && MODE == MD && code == R * 100 + MB)                                \
    return spmv_tma_t<TT, R, MB, MD>(c, L, (const TT*)x, (const TT*)b, (TT*)y, partial, nblocks, dst, rows);
  HPG_SPMV_CFGS(HPG_SPMV_CASE)
#undef HPG_SPMV_CASE
  return fail(HPG_E_ARG, "unknown SpMV configuration %d", code);
}

template <typename T>
bool spmv_tma_ok(hpg_ctx* c, const Level& L, int rows) {
  return ((c->spmv_tma >> (sizeof(T) == 4)) & 1) && L.n >= c->tma_min_rows && L.ld >= rows &&
         (L.ld * (int64_t)sizeof(T)) % 16 == 0 && ((uintptr_t)vals_of<T>(L)) % 16 == 0 && L.ld < (int64_t{1} << 31);
}

template <typename T>
int spmv_launch(hpg_ctx* c, Level& L, int64_t cnt, const T* x, T* y, const uint8_t* skip, const int32_t* list) {
  if ((!skip || c->overlap_tma) && !list && cnt == L.n && spmv_tma_ok<T>(c, L, c->spmv_cfg[sizeof(T) == 4] / 100)) {
    c->pass_skip = skip;
    const int rc = spmv_tma<T, 0>(c, L, x, nullptr, y, nullptr, nullptr);
    c->pass_skip = nullptr;
    return rc;
  }
  if (skip || list)
    CUDA_TRY(launch_pdl(c, hpg::k_spmv<T, 0, true>, grid_for(cnt), 256, (const int32_t*)L.cols,
                        (const T*)vals_of<T>(L), L.ld, (int64_t)0, cnt, x, (const T*)nullptr, y, (double*)nullptr,
                        skip, list, stencil_of(c, L), 1));
  else {
    const int ilv = std::max(1, c->spmv_ilv[sizeof(T) == 4]);
    const int grid = (int)(cdiv(grid_for(cnt, HPG_SPMV_BLOCK), ilv) * ilv);
    CUDA_TRY(launch_pdl(c, hpg::k_spmv<T, 0>, grid, HPG_SPMV_BLOCK, (const int32_t*)L.cols,
                        (const T*)vals_of<T>(L),
                        L.ld, (int64_t)0, cnt, x, (const T*)nullptr, y, (double*)nullptr, skip, list,
                        stencil_of(c, L), ilv));
  }
  ++c->launches;
  return HPG_OK;
}

// y = A x (ref: krylov.py:83-107); multi-rank: rows without halo columns run
// while the exchange is in flight, then the boundary rows
template <typename T>
int spmv_t(hpg_ctx* c, int l, T* x, T* y) {
  Level& L = c->lev[l];
  const int prec = sizeof(T) == 8 ? HPG_F64 : HPG_F32;
  int rc;
  if (overlapped(c, l)) {
    if ((rc = exchange_begin(c, l, prec, x))) return rc;
    if (L.n && (rc = spmv_launch<T>(c, L, L.n, x, y, L.hflag, nullptr))) return rc;
    if ((rc = exchange_end(c))) return rc;
    if (L.nbnd && (rc = spmv_launch<T>(c, L, L.nbnd, x, y, nullptr, L.bnd))) return rc;
    return HPG_OK;
  }
  if ((rc = do_exchange(c, l, prec, x))) return rc;
  if (!L.n) return HPG_OK;
  return spmv_launch<T>(c, L, L.n, x, y, nullptr, nullptr);
}

// Staging layout of rank R's symmetric buffer: per level, per neighbour
// (ascending rank), 2 parities x count x 8 B, 256-B aligned.  Every rank can
// evaluate it for every other rank from the geometry alone.
size_t stage_offset_geo(const int procs[3], const int local0[3], int nlev, int R, int level, int sender,
                        int64_t* cnt_out) {
  const int nranks = procs[0] * procs[1] * procs[2];
  size_t off = hpg::kSymArSlots + (size_t)2 * nranks * hpg::kArSlot * 8;
  off = (off + 255) & ~(size_t)255;
  const int coords[3] = {R % procs[0], (R / procs[0]) % procs[1], R / (procs[0] * procs[1])};
  int dims[3] = {local0[0], local0[1], local0[2]};
  for (int l = 0; l < nlev; ++l) {
    const Geom g = make_geom(dims, coords, procs);
    struct E {
      int rank;
      int64_t cnt;
    };
    std::vector<E> es;
    for (int i = 0; i < 27; ++i)
      if (g.nbr_rank[i] >= 0) es.push_back({g.nbr_rank[i], hpg::region_size(g, i % 3 - 1, (i / 3) % 3 - 1, i / 9 - 1)});
    std::sort(es.begin(), es.end(), [](const E& a, const E& b) { return a.rank < b.rank; });
    for (auto& e : es) {
      if (l == level && e.rank == sender) {
        if (cnt_out) *cnt_out = e.cnt;
        return off;
      }
      off += ((size_t)2 * e.cnt * 8 + 255) & ~(size_t)255;
    }
    for (int a = 0; a < 3; ++a) dims[a] /= 2;
  }
  if (cnt_out) *cnt_out = -1;
  return off;  // past the end: total size when sender < 0
}

// Staging layout of rank R's symmetric buffer: per level, per neighbour
// (ascending rank), 2 parities x count x 8 B, 256-B aligned.  Every rank can
// evaluate it for every other rank from the geometry alone.
size_t stage_offset(const hpg_ctx* c, int R, int level, int sender, int64_t* cnt_out) {
  const int local0[3] = {c->lev[0].g.lx, c->lev[0].g.ly, c->lev[0].g.lz};
  return stage_offset_geo(c->procs, local0, c->nlev, R, level, sender, cnt_out);
}

}  // namespace

// =============================================================== C ABI

extern "C" {

int hpg_abi_version(void) { return 1; }
const char* hpg_last_error(void) { return g_err.c_str(); }

int hpg_host_level(const int local_dims[3], const int rank_coords[3], const int proc_dims[3], double* values,
                   int32_t* col_idx, int32_t* row_nnz, int32_t* diag_pos, int64_t* info, int ninfo) {
  const Geom g = make_geom(local_dims, rank_coords, proc_dims);
  for (int64_t i = 0; i < g.n; ++i) {
    int32_t cols[27];
    double v[27];
    int diag = 0;
    const int nnz = hpg::build_row(g, i, cols, v, &diag);
    for (int s = 0; s < 27; ++s) {
      if (values) values[i * 27 + s] = s < nnz ? v[s] : 0.0;
      if (col_idx) col_idx[i * 27 + s] = s < nnz ? cols[s] : -1;
    }
    if (row_nnz) row_nnz[i] = nnz;
    if (diag_pos) diag_pos[i] = diag;
  }
  int64_t tmp[16] = {g.n, g.n + g.halo_size, geom_nnz(g), g.ncolors};
  for (int k = 0; k < 9; ++k) tmp[4 + k] = g.off[k];
  tmp[13] = g.halo_size;
  for (int k = 0; k < ninfo && k < 14; ++k) info[k] = tmp[k];
  return HPG_OK;
}

int64_t hpg_host_send_rows(const int local_dims[3], const int rank_coords[3], const int proc_dims[3], int sx, int sy,
                           int sz, int64_t* rows) {
  const Geom g = make_geom(local_dims, rank_coords, proc_dims);
  if (g.halo_base[hpg::offset_index(sx, sy, sz)] < 0) return 0;
  const int64_t cnt = hpg::region_size(g, sx, sy, sz);
  if (rows)
    for (int64_t p = 0; p < cnt; ++p) rows[p] = hpg::send_row(g, sx, sy, sz, p);
  return cnt;
}

int64_t hpg_host_stage_offset(const int local_dims[3], const int proc_dims[3], int levels, int receiver, int level,
                              int sender, int64_t* count) {
  return (int64_t)stage_offset_geo(proc_dims, local_dims, levels, receiver, level, sender, count);
}

int hpg_nccl_unique_id(void* out, int len) {
  if (len < (int)sizeof(ncclUniqueId)) return fail(HPG_E_ARG, "need %zu bytes", sizeof(ncclUniqueId));
  ncclUniqueId id;
  NCCL_TRY(ncclGetUniqueId(&id));
  memcpy(out, &id, sizeof id);
  return HPG_OK;
}

int hpg_create(hpg_ctx** out, int device, int rank, int nranks, const int proc_dims[3], const int local_dims[3],
               int levels, int nu1, int nu2, int nu_c, const void* nccl_uid, void* stream) {
  if (!out) return fail(HPG_E_ARG, "null out");
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(HPG_E_ARG, "bad rank %d of %d", rank, nranks);
  if (proc_dims[0] * proc_dims[1] * proc_dims[2] != nranks) return fail(HPG_E_ARG, "process grid != nranks");
  if (levels < 1) return fail(HPG_E_ARG, "need at least one level");
  if (std::min(nu1, std::min(nu2, nu_c)) < 1) return fail(HPG_E_ARG, "sweep counts must all be >= 1");
  int dims[3] = {local_dims[0], local_dims[1], local_dims[2]};
  for (int l = 0; l + 1 < levels; ++l)
    for (int a = 0; a < 3; ++a) {
      if (dims[a] % 2) return fail(HPG_E_COARSEN, "axis %c: local dimension %d is odd at level %d", "xyz"[a], dims[a], l);
      dims[a] /= 2;
    }
  CUDA_TRY(cudaSetDevice(device));
  hpg_ctx* c = new hpg_ctx();
  c->device = device;
  c->rank = rank;
  c->nranks = nranks;
  for (int a = 0; a < 3; ++a) c->procs[a] = proc_dims[a];
  c->coords[0] = rank % proc_dims[0];
  c->coords[1] = (rank / proc_dims[0]) % proc_dims[1];
  c->coords[2] = rank / (proc_dims[0] * proc_dims[1]);
  c->nlev = levels;
  c->nu1 = nu1;
  c->nu2 = nu2;
  c->nu_c = nu_c;
  auto bail = [&](int rc) {
    hpg_destroy(c);
    return rc;
  };
  if (stream) {
    c->stream = (cudaStream_t)stream;
    c->own_stream = false;
  } else if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
    return bail(fail(HPG_E_CUDA, "stream create failed"));
  }
  int prio_lo = 0, prio_hi = 0;  // the halo stream's CTAs are scheduled ahead of the compute stream's
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  if (cudaStreamCreateWithPriority(&c->halo, cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_ready, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_cgs, cudaEventDisableTiming) != cudaSuccess)
    return bail(fail(HPG_E_CUDA, "halo stream/event create failed"));
  c->lev.resize(levels);
  dims[0] = local_dims[0];
  dims[1] = local_dims[1];
  dims[2] = local_dims[2];
  for (int l = 0; l < levels; ++l) {
    int rc = build_level(c, c->lev[l], dims);
    if (rc) return bail(rc);
    if (l > 0) {
      Level& C = c->lev[l];
      rc = dmalloc(&C.inj, std::max<int64_t>(C.n, 1) * 4, &C.bytes);
      if (rc) return bail(rc);
      if (C.n) hpg::k_build_inject<<<grid_for(C.n), 256, 0, c->stream>>>(C.g, C.inj);
    }
    for (int a = 0; a < 3; ++a) dims[a] /= 2;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  {
    const char* e = getenv("HPG_TAIL_ROWS");
    c->tail_rows = e ? atoll(e) : (int64_t)0;  // measured: per-pass PDL kernels win at 256^3
    const char* wv = getenv("HPG_WAVE");
    if (wv) c->wave = atoi(wv);
    const char* wl = getenv("HPG_WAVE_LAG");
    if (wl) c->wave_lag = std::max(1, atoi(wl));
    const char* wc = getenv("HPG_WAVE_COH");
    if (wc) c->wave_coh = wc[0] != '0';
    const char* wm = getenv("HPG_WAVE_MIN_ROWS");
    if (wm) c->wave_min_rows = atoll(wm);
    int pw = 0;
    auto occ = [&](const void* fn) {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pw, fn, hpg::kWaveRows, 0);
      return pw * sms;
    };
    c->wave_blocks[0] = std::min(occ(wave_fn<double>(true)), occ(wave_fn<double>(false)));
    c->wave_blocks[1] = std::min(occ(wave_fn<float>(true)), occ(wave_fn<float>(false)));
    const char* tm = getenv("HPG_TMA");
    if (tm) c->tma = atoi(tm);
    const char* fc = getenv("HPG_FACE_COLS");
    if (fc) c->face_cols = atoi(fc);
    const char* t32 = getenv("HPG_TMA_CFG32");
    if (t32) c->tma_cfg[1] = atoi(t32);
    const char* tr = getenv("HPG_TMA_MIN_ROWS");
    if (tr) c->tma_min_rows = atoll(tr);
    if (tma_setup<float>(c, sms) || tma_setup<double>(c, sms)) return bail(HPG_E_CUDA);
    const char* f = getenv("HPG_CGS_FUSED");
    c->cgs_fused = !(f && f[0] == '0');
    const char* sn = getenv("HPG_STENCIL");
    if (sn) c->stencil = sn[0] != '0';
    const char* rv = getenv("HPG_GS_REV");
    if (rv) c->gs_rev = rv[0] != '0';
    const char* mb = getenv("HPG_GS_MINB");
    if (mb) c->gs_minb = atoi(mb);
    const char* lw = getenv("HPG_LOWER");
    if (lw) c->lower = lw[0] != '0';
    const char* kz = getenv("HPG_KNOWN_ZERO");
    if (kz) c->known_zero = kz[0] != '0';
    const char* gr = getenv("HPG_GRAPHS");
    if (gr) c->graphs = gr[0] != '0';
    const char* pp = getenv("HPG_P2P");
    if (pp) c->p2p_want = pp[0] != '0';
    const char* ov = getenv("HPG_OVERLAP");
    if (ov) c->overlap = ov[0] != '0';
    const char* ovr = getenv("HPG_OVERLAP_ROWS");
    if (ovr) c->overlap_rows = atoll(ovr);
    const char* si = getenv("HPG_SPMV_ILV");
    if (si) c->spmv_ilv[0] = atoi(si);
    const char* si32 = getenv("HPG_SPMV_ILV32");
    if (si32) c->spmv_ilv[1] = atoi(si32);
    const char* g = getenv("HPG_PDL");
    c->pdl = !(g && g[0] == '0');
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, hpg::k_vcycle_tail<double, false>, 256, 0);
    c->tail_blocks[0] = std::max(1, per) * sms;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, hpg::k_vcycle_tail<float, false>, 256, 0);
    c->tail_blocks[1] = std::max(1, per) * sms;
    const char* tc = getenv("HPG_TAIL_CLUSTER");
    if (tc) set_tail_cluster(c, atoi(tc));
  }
  c->nb = (int)std::min<int64_t>(8 * sms, std::max<int64_t>(1, cdiv(c->lev[0].n, 256)));
  c->spmv_partial_len = cdiv(c->lev[0].n, 32);  // one partial per row tile (>= 32 rows)
  // partials: [64][grid] for the per-pass kernels (nb CTAs) and the cooperative ones (<= 8 per SM)
  if (dmalloc((char**)&c->partial, (size_t)std::max(c->nb, 8 * sms) * 64 * 8, nullptr) ||
      dmalloc(&c->spmv_partial, c->spmv_partial_len * 8, nullptr) ||
      dmalloc((char**)&c->scal, 512 * 8, nullptr) || dmalloc((char**)&c->gather, (size_t)nranks * 256 * 8, nullptr) ||
      dmalloc((char**)&c->sweep_done, 64 * 4, nullptr))
    return bail(HPG_E_CUDA);
  if (cudaMemset(c->sweep_done, 0, 64 * 4) != cudaSuccess) return bail(fail(HPG_E_CUDA, "memset"));
  if (cudaMallocHost((void**)&c->pinned, 256 * 8) != cudaSuccess) return bail(fail(HPG_E_CUDA, "pinned alloc"));
  // nccl_uid == NULL: P2P-only context (every exchange and reduction over the
  // peer-memory path; lets several ranks share one GPU, where NCCL refuses)
  if (nranks > 1 && nccl_uid) {
    ncclUniqueId id;
    memcpy(&id, nccl_uid, sizeof id);
    ncclResult_t r = ncclCommInitRank(&c->comm, nranks, id, rank);
    if (r != ncclSuccess) return bail(fail(HPG_E_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r)));
  }
  if (cudaStreamSynchronize(c->stream) != cudaSuccess || cudaGetLastError() != cudaSuccess)
    return bail(fail(HPG_E_CUDA, "hierarchy build failed"));
  *out = c;
  return HPG_OK;
}

int hpg_destroy(hpg_ctx* c) {
  if (!c) return HPG_OK;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto& L : c->lev) free_level(L);
  for (void* p : {c->partial, (void*)c->spmv_partial, c->scal, c->gather})
    if (p) cudaFree(p);
  if (c->pinned) cudaFreeHost(c->pinned);
  if (c->comm) ncclCommDestroy(c->comm);
  for (size_t q = 0; q < c->peer_sym.size(); ++q)
    if (c->peer_sym[q] && c->peer_sym[q] != c->sym) cudaIpcCloseMemHandle(c->peer_sym[q]);
  if (c->sym) cudaFree(c->sym);
  if (c->d_peer) cudaFree(c->d_peer);
  if (c->done) cudaFree(c->done);
  if (c->sweep_done) cudaFree(c->sweep_done);
  for (auto& e : c->gcache) cudaGraphExecDestroy(e.exec);
  for (auto e : c->events) cudaEventDestroy(e);
  if (c->ev_ready) cudaEventDestroy(c->ev_ready);
  if (c->ev_done) cudaEventDestroy(c->ev_done);
  if (c->ev_cgs) cudaEventDestroy(c->ev_cgs);
  if (c->halo) cudaStreamDestroy(c->halo);
  if (c->stream && c->own_stream) cudaStreamDestroy(c->stream);
  delete c;
  return HPG_OK;
}

void* hpg_stream(hpg_ctx* c) { return c ? (void*)c->stream : nullptr; }

int hpg_level_info(hpg_ctx* c, int l, int64_t* info, int ninfo) {
  int rc = check_level(c, l);
  if (rc) return rc;
  const Level& L = c->lev[l];
  int64_t tmp[20] = {L.n, L.n_ext, L.nnz, L.g.ncolors};
  for (int k = 0; k < 9; ++k) tmp[4 + k] = L.g.off[k];
  tmp[13] = L.g.halo_size;
  tmp[14] = L.ld;
  tmp[15] = (int64_t)L.nbrs.size();
  tmp[16] = (int64_t)L.bytes;
  // slots a zero-initial-guess sweep streams: sum_c W_c * rows_c (27 n without the lower split)
  int64_t ls = 0;
  for (int k = 0; k < L.g.ncolors; ++k)
    ls += (L.lower_ok ? L.lc[k].w : hpg::kWidth) * (L.g.off[k + 1] - L.g.off[k]);
  tmp[17] = ls;
  tmp[18] = L.st.on ? L.st_rows : 0;  // rows on the implicit-index path
  tmp[19] = L.st_lower ? 1 : 0;        // zero-guess sweeps on the implicit-index path
  for (int k = 0; k < ninfo && k < 20; ++k) info[k] = tmp[k];
  return HPG_OK;
}

int hpg_export_level(hpg_ctx* c, int l, double* values, int32_t* col_idx, int32_t* row_nnz, int32_t* diag_pos) {
  int rc = check_level(c, l);
  if (rc) return rc;
  const Level& L = c->lev[l];
  CUDA_TRY(cudaSetDevice(c->device));
  std::vector<int32_t> cols((size_t)27 * L.ld);
  std::vector<double> v((size_t)27 * L.ld);
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  CUDA_TRY(cudaMemcpy(cols.data(), L.cols, cols.size() * 4, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(v.data(), L.v64, v.size() * 8, cudaMemcpyDeviceToHost));
  for (int64_t i = 0; i < L.n; ++i) {
    int nnz = 0, diag = -1;
    for (int s = 0; s < 27; ++s) {
      int32_t cc = cols[s * L.ld + i];
      const double vv = v[s * L.ld + i];
      if (cc < 0) {
        diag = s;
        cc = ~cc;
      }
      if (vv != 0.0) nnz = s + 1;
      if (values) values[i * 27 + s] = vv;
      if (col_idx) col_idx[i * 27 + s] = cc;
    }
    for (int s = nnz; s < 27; ++s)
      if (col_idx) col_idx[i * 27 + s] = -1;
    if (row_nnz) row_nnz[i] = nnz;
    if (diag_pos) diag_pos[i] = diag;
  }
  return HPG_OK;
}

int hpg_export_f2c(hpg_ctx* c, int l, int64_t* f2c) {
  int rc = check_level(c, l);
  if (rc) return rc;
  if (l == 0) return fail(HPG_E_ARG, "level 0 has no injection map");
  const Level& C = c->lev[l];
  std::vector<int32_t> dst(C.n);
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  if (C.f2c) {
    CUDA_TRY(cudaMemcpy(dst.data(), C.f2c, C.n * 4, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < C.n; ++i) f2c[i] = dst[i];
    return HPG_OK;
  }
  CUDA_TRY(cudaMemcpy(dst.data(), C.inj, C.n * 4, cudaMemcpyDeviceToHost));
  for (int64_t j = 0; j < C.n; ++j) f2c[dst[j]] = j;  // fine color-0 row j feeds coarse row dst[j]
  return HPG_OK;
}

int hpg_set_coloring(hpg_ctx* c, int l, int ncolors, const int64_t* offsets, const int64_t* perm) {
  int rc = check_level(c, l);
  if (rc) return rc;
  Level& L = c->lev[l];
  if (ncolors < 1 || ncolors > hpg::kMaxColors) return fail(HPG_E_ARG, "ncolors %d out of [1, 27]", ncolors);
  if (offsets[0] != 0 || offsets[ncolors] != L.n) return fail(HPG_E_ARG, "color offsets must span [0, n)");
  for (int k = 0; k < ncolors; ++k)
    if (offsets[k + 1] < offsets[k]) return fail(HPG_E_ARG, "color offsets must be non-decreasing");
  std::vector<int32_t> p32(L.n), ip32(L.n, -1);
  for (int64_t i = 0; i < L.n; ++i) {
    if (perm[i] < 0 || perm[i] >= L.n || ip32[perm[i]] >= 0) return fail(HPG_E_ARG, "perm is not a permutation");
    p32[i] = (int32_t)perm[i];
    ip32[perm[i]] = (int32_t)i;
  }
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  if (!L.perm_d && (rc = dmalloc(&L.perm_d, std::max<int64_t>(1, L.n) * 4, &L.bytes))) return rc;
  if (!L.iperm_d && (rc = dmalloc(&L.iperm_d, std::max<int64_t>(1, L.n) * 4, &L.bytes))) return rc;
  CUDA_TRY(cudaMemcpy(L.perm_d, p32.data(), L.n * 4, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(L.iperm_d, ip32.data(), L.n * 4, cudaMemcpyHostToDevice));
  L.g.perm_tab = L.perm_d;
  L.g.iperm_tab = L.iperm_d;
  L.g.ncolors = ncolors;
  for (int k = 0; k <= hpg::kMaxColors; ++k) L.g.off[k] = k <= ncolors ? offsets[k] : L.n;
  c->general = true;
  L.wave_ok = false;  // the dataflow plan needs the closed-form (greedy) layout
  if ((rc = build_structure(c, L, false))) return rc;
  // injection maps of the coarse levels that touch this one
  for (int cl = std::max(1, l); cl <= std::min(l + 1, c->nlev - 1); ++cl) {
    Level& C = c->lev[cl];
    if (!C.f2c && (rc = dmalloc(&C.f2c, std::max<int64_t>(1, C.n) * 4, &C.bytes))) return rc;
    if (C.n) hpg::k_build_f2c<<<grid_for(C.n), 256, 0, c->stream>>>(C.g, c->lev[cl - 1].g, C.f2c);
    LAUNCH_CHECK();
  }
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return HPG_OK;
}

int hpg_spmv(hpg_ctx* c, int l, int prec, void* x, void* y) {
  int rc = check_level(c, l);
  if (rc || (rc = check_prec(prec))) return rc;
  Timed tm(c, M_SPMV);
  return prec == HPG_F64 ? spmv_t<double>(c, l, (double*)x, (double*)y) : spmv_t<float>(c, l, (float*)x, (float*)y);
}

int hpg_exchange(hpg_ctx* c, int l, int prec, void* v) {
  int rc = check_level(c, l);
  if (rc || (rc = check_prec(prec))) return rc;
  return do_exchange(c, l, prec, v);
}

int hpg_gs_sweep(hpg_ctx* c, int l, int prec, const void* r, void* z, int z_is_zero) {
  int rc = check_level(c, l);
  if (rc || (rc = check_prec(prec))) return rc;
  return prec == HPG_F64 ? gs_sweep<double>(c, l, (const double*)r, (double*)z, z_is_zero)
                         : gs_sweep<float>(c, l, (const float*)r, (float*)z, z_is_zero);
}

int hpg_restrict(hpg_ctx* c, int l, int prec, const void* rf, const void* zf, void* rcoarse) {
  int rc = check_level(c, l);
  if (rc || (rc = check_prec(prec))) return rc;
  if (l + 1 >= c->nlev) return fail(HPG_E_ARG, "level %d has no coarser level", l);
  return prec == HPG_F64 ? restrict_<double>(c, l, (const double*)rf, (const double*)zf, (double*)rcoarse)
                         : restrict_<float>(c, l, (const float*)rf, (const float*)zf, (float*)rcoarse);
}

int hpg_prolong(hpg_ctx* c, int l, int prec, void* zf, const void* zc) {
  int rc = check_level(c, l);
  if (rc || (rc = check_prec(prec))) return rc;
  if (l + 1 >= c->nlev) return fail(HPG_E_ARG, "level %d has no coarser level", l);
  return prec == HPG_F64 ? prolong_<double>(c, l, (double*)zf, (const double*)zc)
                         : prolong_<float>(c, l, (float*)zf, (const float*)zc);
}

int hpg_vcycle(hpg_ctx* c, int prec, const void* r, void* z) {
  int rc = check_level(c, 0);
  if (rc || (rc = check_prec(prec))) return rc;
  // Single rank, no motif timers: replay a CUDA graph of the whole V-cycle
  // (~60 dependent launches) captured once per (precision, r, z).
  if (c->graphs && c->nranks == 1 && !c->timing) {
    const GraphKey key{prec, r, z};
    for (auto& e : c->gcache)
      if (e.key == key) {
        e.stamp = ++c->gclock;
        CUDA_TRY(cudaGraphLaunch(e.exec, c->stream));
        c->launches += e.kernels;
        return HPG_OK;
      }
    cudaGraph_t g = nullptr;
    const int64_t l0 = c->launches;
    CUDA_TRY(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    rc = prec == HPG_F64 ? vcycle<double>(c, 0, (const double*)r, (double*)z)
                         : vcycle<float>(c, 0, (const float*)r, (float*)z);
    cudaError_t ce = cudaStreamEndCapture(c->stream, &g);
    if (rc) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    if (ce != cudaSuccess) return fail(HPG_E_CUDA, "V-cycle capture: %s", cudaGetErrorString(ce));
    cudaGraphExec_t exec = nullptr;
    ce = cudaGraphInstantiate(&exec, g, 0);
    cudaGraphDestroy(g);
    if (ce != cudaSuccess) return fail(HPG_E_CUDA, "V-cycle instantiate: %s", cudaGetErrorString(ce));
    if (c->gcache.size() >= 96) {  // evict the least recently used
      size_t lru = 0;
      for (size_t q = 1; q < c->gcache.size(); ++q)
        if (c->gcache[q].stamp < c->gcache[lru].stamp) lru = q;
      cudaGraphExecDestroy(c->gcache[lru].exec);
      c->gcache.erase(c->gcache.begin() + lru);
    }
    c->gcache.push_back({key, exec, ++c->gclock, c->launches - l0});
    CUDA_TRY(cudaGraphLaunch(exec, c->stream));
    return HPG_OK;
  }
  return prec == HPG_F64 ? vcycle<double>(c, 0, (const double*)r, (double*)z)
                         : vcycle<float>(c, 0, (const float*)r, (float*)z);
}

int hpg_cgs2(hpg_ctx* c, int prec, void* Q, int64_t ldq, int k, void* w, void* qnext, double* out) {
  int rc = check_level(c, 0);
  if (rc || (rc = check_prec(prec))) return rc;
  if (k < 0) return fail(HPG_E_ARG, "bad k");
  return prec == HPG_F64 ? cgs2_t<double>(c, (double*)Q, ldq, k, (double*)w, (double*)qnext, out)
                         : cgs2_t<float>(c, (float*)Q, ldq, k, (float*)w, (float*)qnext, out);
}

int hpg_cgs2_begin(hpg_ctx* c, int prec, void* Q, int64_t ldq, int k, void* w, void* qnext) {
  int rc = check_level(c, 0);
  if (rc || (rc = check_prec(prec))) return rc;
  if (k < 0) return fail(HPG_E_ARG, "bad k");
  return prec == HPG_F64 ? cgs2_launch_t<double>(c, (double*)Q, ldq, k, (double*)w, (double*)qnext)
                         : cgs2_launch_t<float>(c, (float*)Q, ldq, k, (float*)w, (float*)qnext);
}

int hpg_cgs2_end(hpg_ctx* c, double* out) {
  if (!c) return fail(HPG_E_ARG, "null context");
  return cgs2_finish(c, out);
}

int hpg_gemv_combine(hpg_ctx* c, int prec, const void* Q, int64_t ldq, int k, const double* y, void* out) {
  int rc = check_level(c, 0);
  if (rc || (rc = check_prec(prec))) return rc;
  if (k < 1) return fail(HPG_E_ARG, "bad k");
  return prec == HPG_F64 ? gemv_t<double>(c, (const double*)Q, ldq, k, y, (double*)out)
                         : gemv_t<float>(c, (const float*)Q, ldq, k, y, (float*)out);
}

int hpg_axpy_mixed(hpg_ctx* c, int prec, double* x, const void* z, int64_t n) {
  int rc = check_level(c, 0);
  if (rc || (rc = check_prec(prec))) return rc;
  Timed tm(c, M_VEC);
  if (prec == HPG_F64)
    hpg::k_axpy_mixed<double><<<grid_for(n), 256, 0, c->stream>>>(x, (const double*)z, n);
  else
    hpg::k_axpy_mixed<float><<<grid_for(n), 256, 0, c->stream>>>(x, (const float*)z, n);
  LAUNCH_CHECK();
  ++c->launches;
  return HPG_OK;
}

int hpg_residual(hpg_ctx* c, const double* b, double* x, double* r, double* rho2) {
  int rc = check_level(c, 0);
  if (rc) return rc;
  {
  Timed tm(c, M_SPMV);
  if ((rc = do_exchange(c, 0, HPG_F64, x))) return rc;
  Level& L = c->lev[0];
  double* scal = (double*)c->scal;
  int64_t nbk = grid_for(L.n);
  if (spmv_tma_ok<double>(c, L, c->resid_cfg / 100) && cdiv(L.n, c->resid_cfg / 100) <= c->spmv_partial_len) {
    if ((rc = spmv_tma<double, 1>(c, L, x, b, r, c->spmv_partial, &nbk))) return rc;
  } else {
    const int ilv = std::max(1, c->spmv_ilv[0]);
    hpg::k_spmv<double, 1><<<(int)(cdiv(nbk, ilv) * ilv), 256, 0, c->stream>>>(
        L.cols, L.v64, L.ld, 0, L.n, x, b, r, c->spmv_partial, nullptr, nullptr, stencil_of(c, L), ilv);
    ++c->launches;
  }
  hpg::k_fold<double><<<1, 1024, 0, c->stream>>>(c->spmv_partial, (int)nbk, 1, scal + 200, 0);
  LAUNCH_CHECK();
  c->launches += 1;
  if ((rc = allreduce_scal<double>(c, scal + 200, 1))) return rc;
  }
  CUDA_TRY(cudaMemcpyAsync(c->pinned + 200, (double*)c->scal + 200, 8, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  *rho2 = c->pinned[200];
  return HPG_OK;
}

int hpg_scale_cast(hpg_ctx* c, int prec, const double* r, double rho, void* q0, int64_t n) {
  int rc = check_level(c, 0);
  if (rc || (rc = check_prec(prec))) return rc;
  Timed tm(c, M_VEC);
  if (prec == HPG_F64)
    hpg::k_scale_cast<double><<<grid_for(n), 256, 0, c->stream>>>(r, rho, (double*)q0, n);
  else
    hpg::k_scale_cast<float><<<grid_for(n), 256, 0, c->stream>>>(r, rho, (float*)q0, n);
  LAUNCH_CHECK();
  ++c->launches;
  return HPG_OK;
}

int hpg_sumsq(hpg_ctx* c, int prec, const void* x, int64_t n, double* out) {
  int rc = check_level(c, 0);
  if (rc || (rc = check_prec(prec))) return rc;
  const int nb = (int)std::min<int64_t>(c->nb, std::max<int64_t>(1, cdiv(n, 256)));
  Timed tm(c, M_VEC);
  if (prec == HPG_F64) {
    double* scal = (double*)c->scal;
    hpg::k_sumsq<double><<<nb, 256, 0, c->stream>>>((const double*)x, n, (double*)c->partial);
    hpg::k_fold<double><<<1, 1024, 0, c->stream>>>((const double*)c->partial, nb, 1, scal + 210, 0);
    LAUNCH_CHECK();
    if ((rc = allreduce_scal<double>(c, scal + 210, 1))) return rc;
    CUDA_TRY(cudaMemcpyAsync(c->pinned + 210, scal + 210, 8, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    *out = c->pinned[210];
  } else {
    float* scal = (float*)c->scal;
    hpg::k_sumsq<float><<<nb, 256, 0, c->stream>>>((const float*)x, n, (float*)c->partial);
    hpg::k_fold<float><<<1, 1024, 0, c->stream>>>((const float*)c->partial, nb, 1, scal + 420, 0);
    LAUNCH_CHECK();
    if ((rc = allreduce_scal<float>(c, scal + 420, 1))) return rc;
    CUDA_TRY(cudaMemcpyAsync(c->pinned + 210, scal + 420, 4, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    *out = (double)*(float*)(c->pinned + 210);
  }
  c->launches += 2;
  return HPG_OK;
}

int hpg_sync(hpg_ctx* c) {
  if (!c) return fail(HPG_E_ARG, "null context");
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return HPG_OK;
}

int hpg_allreduce_host(hpg_ctx* c, double* vals, int n) {
  if (!c) return fail(HPG_E_ARG, "null context");
  if (c->nranks == 1) return HPG_OK;
  if (n > 32) return fail(HPG_E_ARG, "at most 32 values");
  double* scal = (double*)c->scal;
  CUDA_TRY(cudaMemcpyAsync(scal + 220, vals, n * 8, cudaMemcpyHostToDevice, c->stream));
  int rc = allreduce_scal<double>(c, scal + 220, n);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(vals, scal + 220, n * 8, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return HPG_OK;
}

int64_t hpg_launch_count(hpg_ctx* c) { return c ? c->launches : -1; }

int hpg_p2p_handle(hpg_ctx* c, void* out, int len) {
  if (!c || !out) return fail(HPG_E_ARG, "null argument");
  if (len < (int)sizeof(cudaIpcMemHandle_t)) return fail(HPG_E_ARG, "need %zu bytes", sizeof(cudaIpcMemHandle_t));
  if (c->nranks == 1) return fail(HPG_E_ARG, "peer memory needs more than one rank");
  CUDA_TRY(cudaSetDevice(c->device));
  if (!c->sym) {
    c->sym_bytes = stage_offset(c, c->rank, -1, -1, nullptr);
    CUDA_TRY(cudaMalloc((void**)&c->sym, c->sym_bytes));
    CUDA_TRY(cudaMemset(c->sym, 0, c->sym_bytes));
    CUDA_TRY(cudaMalloc((void**)&c->done, 64));
    CUDA_TRY(cudaMemset(c->done, 0, 64));
    CUDA_TRY(cudaDeviceSynchronize());
  }
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, c->sym));
  memcpy(out, &h, sizeof h);
  return HPG_OK;
}

int hpg_p2p_open(hpg_ctx* c, const void* handles, int stride) {
  if (!c || !handles) return fail(HPG_E_ARG, "null argument");
  if (!c->sym) return fail(HPG_E_ARG, "call hpg_p2p_handle first");
  CUDA_TRY(cudaSetDevice(c->device));
  c->peer_sym.assign(c->nranks, nullptr);
  for (int q = 0; q < c->nranks; ++q) {
    if (q == c->rank) {
      c->peer_sym[q] = c->sym;
      continue;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, (const char*)handles + (size_t)q * stride, sizeof h);
    void* p = nullptr;
    CUDA_TRY(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    c->peer_sym[q] = (char*)p;
  }
  CUDA_TRY(cudaMalloc((void**)&c->d_peer, sizeof(char*) * c->nranks));
  CUDA_TRY(cudaMemcpy(c->d_peer, c->peer_sym.data(), sizeof(char*) * c->nranks, cudaMemcpyHostToDevice));
  for (int l = 0; l < c->nlev; ++l) {
    Level& L = c->lev[l];
    memset(&L.p2p, 0, sizeof L.p2p);
    if ((int)L.nbrs.size() > hpg::kMaxNbr) return fail(HPG_E_ARG, "too many neighbours");
    L.p2p.nn = (int)L.nbrs.size();
    for (size_t k = 0; k < L.nbrs.size(); ++k) {
      const Nbr& nb = L.nbrs[k];
      int64_t cnt_r = 0, cnt_l = 0;
      const size_t roff = stage_offset(c, nb.rank, l, c->rank, &cnt_r);
      const size_t loff = stage_offset(c, c->rank, l, nb.rank, &cnt_l);
      if (cnt_r != nb.cnt || cnt_l != nb.cnt) return fail(HPG_E_ARG, "asymmetric halo plan");
      hpg::P2PNbr& d = L.p2p.nb[k];
      d.remote_stage = c->peer_sym[nb.rank] + roff;
      d.local_stage = c->sym + loff;
      d.remote_flag = (uint64_t*)(c->peer_sym[nb.rank] + hpg::kSymHaloFlags) + c->rank;
      d.local_flag = (const uint64_t*)(c->sym + hpg::kSymHaloFlags) + nb.rank;
      d.send_off = nb.send_off;
      d.cnt = nb.cnt;
      d.recv_base = nb.recv_base;
      L.p2p.total += nb.cnt;
    }
  }
  c->p2p = c->p2p_want;
  return HPG_OK;
}

// Captured V-cycle graphs bake in the kernel choice and launch arguments that
// the options select, so every option change drops them (they are re-captured
// on the next V-cycle).
static void drop_graphs(hpg_ctx* c) {
  if (!c->gcache.empty()) cudaStreamSynchronize(c->stream);
  for (auto& e : c->gcache) cudaGraphExecDestroy(e.exec);
  c->gcache.clear();
}

int hpg_set_option(hpg_ctx* c, const char* key, int64_t value) {
  if (!c || !key) return fail(HPG_E_ARG, "null argument");
  if (!strcmp(key, "cgs_fused")) c->cgs_fused = value != 0;
  else if (!strcmp(key, "cgs_cfg")) c->cgs_force = (int)value;
  else if (!strcmp(key, "overlap_tma")) c->overlap_tma = value != 0;
  else if (!strcmp(key, "cgs_solo")) c->cgs_solo = value != 0;
  else if (!strcmp(key, "cgs_zigzag")) c->cgs_zigzag = value != 0;
  else if (!strcmp(key, "pdl")) c->pdl = value != 0;
  else if (!strcmp(key, "overlap")) c->overlap = value != 0;
  else if (!strcmp(key, "p2p")) c->p2p = value != 0 && !c->peer_sym.empty();
  else if (!strcmp(key, "overlap_rows")) c->overlap_rows = value;
  else if (!strcmp(key, "gs_minb")) c->gs_minb = (int)value;
  else if (!strcmp(key, "spmv_ilv")) c->spmv_ilv[0] = (int)value;
  else if (!strcmp(key, "spmv_ilv32")) c->spmv_ilv[1] = (int)value;
  else if (!strcmp(key, "wave")) c->wave = (int)value;
  else if (!strcmp(key, "wave_min_rows")) c->wave_min_rows = value;
  else if (!strcmp(key, "known_zero")) c->known_zero = value != 0;
  else if (!strcmp(key, "lower")) c->lower = value != 0;
  else if (!strcmp(key, "graphs")) c->graphs = value != 0;
  else if (!strcmp(key, "tail_rows")) c->tail_rows = value;
  else if (!strcmp(key, "tail_cluster")) set_tail_cluster(c, (int)value);
  else if (!strcmp(key, "gs_rev")) c->gs_rev = value != 0;
  else if (!strcmp(key, "stencil")) c->stencil = value != 0;
  else if (!strcmp(key, "tma")) c->tma = (int)value;
  else if (!strcmp(key, "tma_min_rows")) c->tma_min_rows = value;
  else if (!strcmp(key, "tma_contig")) c->tma_contig = (int)value;
  else if (!strcmp(key, "tma_sweep")) c->tma_sweep = (int)value;
  else if (!strcmp(key, "tma_cfg64")) c->tma_cfg[0] = (int)value;
  else if (!strcmp(key, "tma_cfg32")) c->tma_cfg[1] = (int)value;
  else if (!strcmp(key, "brick")) c->brick = (int)value;
  else if (!strcmp(key, "bpp")) c->bpp = (int)value;
  else if (!strcmp(key, "bpp_cfg64")) c->bpp_cfg[0] = (int)value;
  else if (!strcmp(key, "bpp_cfg32")) c->bpp_cfg[1] = (int)value;
  else if (!strcmp(key, "spmv_tma")) c->spmv_tma = (int)value;
  else if (!strcmp(key, "spmv_cfg64")) c->spmv_cfg[0] = (int)value;
  else if (!strcmp(key, "spmv_cfg32")) c->spmv_cfg[1] = (int)value;
  else if (!strcmp(key, "resid_cfg")) c->resid_cfg = (int)value;
  else if (!strcmp(key, "restr_cfg64")) c->restr_cfg[0] = (int)value;
  else if (!strcmp(key, "l2_window")) c->l2_window = value;
  else if (!strcmp(key, "face_cols")) c->face_cols = (int)value;
  else if (!strcmp(key, "restr_cfg32")) c->restr_cfg[1] = (int)value;
  else if (!strcmp(key, "brick_cfg64")) c->brick_cfg[0] = (int)value;
  else if (!strcmp(key, "brick_cfg32")) c->brick_cfg[1] = (int)value;
  else return fail(HPG_E_ARG, "unknown option %s", key);
  drop_graphs(c);
  return HPG_OK;
}

// mode 1: enable, 0: disable, 2: synchronise, add each motif's seconds into
// seconds[8] (GS, SpMV, Ortho, Restriction, Prolongation, Vector ops, GS at level 0
// (a subset of GS), reserved) and reset.
int hpg_timers(hpg_ctx* c, int mode, double* seconds) {
  if (!c) return fail(HPG_E_ARG, "null context");
  if (mode == 0 || mode == 1) {
    c->timing = mode == 1;
    return HPG_OK;
  }
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  for (auto& m : c->marks) {
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, c->events[m.second], c->events[m.second + 1]));
    if (seconds) seconds[m.first] += ms * 1e-3;
  }
  c->marks.clear();
  c->ev_used = 0;
  return HPG_OK;
}

}  // extern "C"


// Jones-Plassmann-Luby colouring of an lx x ly x lz box on the device, bit-identical to
// the reference's numpy loop (ref: coloring.py:56-70; csrc/hpg_jpl.cuh).  state / inc:
// numpy's PCG64 state (low, high 64-bit words) of default_rng(seed).
int hpg_jpl_color(int device, int lx, int ly, int lz, const uint64_t* state, const uint64_t* inc, int32_t* colors,
                  int* rounds) {
  if (lx < 0 || ly < 0 || lz < 0 || !state || !inc || !colors) return fail(HPG_E_ARG, "bad JPL arguments");
  const int64_t n = (int64_t)lx * ly * lz;
  if (rounds) *rounds = 0;
  if (n == 0) return HPG_OK;
  CUDA_TRY(cudaSetDevice(device));
  cudaStream_t st;
  CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  double* w = nullptr;
  int32_t* col = nullptr;
  uint8_t* sel = nullptr;
  unsigned long long* cnt = nullptr;
  int rc = HPG_OK;
  if (cudaMalloc(&w, n * 8) != cudaSuccess || cudaMalloc(&col, n * 4) != cudaSuccess ||
      cudaMalloc(&sel, n) != cudaSuccess || cudaMalloc(&cnt, 8) != cudaSuccess) {
    rc = fail(HPG_E_CUDA, "JPL buffers");
  }
  hpg::U128 base{state[0], state[1]};
  const hpg::U128 inc128{inc[0], inc[1]};
  int64_t colored = 0;
  int r = 0;
  if (!rc && cudaMemsetAsync(col, 0xff, n * 4, st) != cudaSuccess) rc = fail(HPG_E_CUDA, "JPL memset");
  while (!rc && colored < n) {
    const int grid = (int)cdiv(n, 256);
    hpg::k_jpl_weights<<<grid, 256, 0, st>>>(n, base, inc128, w);
    hpg::k_jpl_select<<<grid, 256, 0, st>>>(lx, ly, lz, w, col, sel);
    cudaMemsetAsync(cnt, 0, 8, st);
    hpg::k_jpl_color<<<grid, 256, 0, st>>>(lx, ly, lz, sel, col, cnt);
    unsigned long long got = 0;
    if (cudaMemcpyAsync(&got, cnt, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess) {
      rc = fail(HPG_E_CUDA, "JPL round: %s", cudaGetErrorString(cudaGetLastError()));
      break;
    }
    if (got == 0) {
      rc = fail(HPG_E_CUDA, "JPL made no progress");
      break;
    }
    colored += (int64_t)got;
    base = hpg::pcg_advance(base, inc128, (uint64_t)n);  // the next round's rng.random(n)
    ++r;
  }
  if (!rc && (cudaMemcpyAsync(colors, col, n * 4, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
              cudaStreamSynchronize(st) != cudaSuccess))
    rc = fail(HPG_E_CUDA, "JPL copy-out");
  cudaFree(w);
  cudaFree(col);
  cudaFree(sel);
  cudaFree(cnt);
  cudaStreamDestroy(st);
  if (rounds) *rounds = r;
  return rc;
}
