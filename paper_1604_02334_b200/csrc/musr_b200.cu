// musr_b200.cu -- host runtime of libmusr_b200.so (C ABI in include/musr_b200.h).
//
// Responsibilities:
//   * NVRTC JIT of (theory fragment + kernel template) for sm_100a, cached by
//     source hash (the paper's runtime kernel generation);
//   * device layout: per-dataset in-range segments packed into aligned
//     4096-term tiles, 16-byte-group transposed; formats c32 (integer counts
//     < 2^23 as fp32 + fp64 envelope, {err, 1/err} from a count-indexed table,
//     in-kernel beyond it) and f64 (counts and envelope as fp64, err and 1/err
//     in-kernel) -- musr_layout.h, musr_kernel.cuh;
//   * the direct path (one GPU, the default): one launch of the persistent
//     objective kernel per evaluation, p inside the kernel parameters, results
//     returned as epoch-tagged 8-byte words in mapped host memory (no graph,
//     no copy, no stream sync);
//   * multi-GPU: the shared-results path (every rank's kernel writes its
//     datasets' words into one host buffer all ranks map) or the NCCL path
//     (one CUDA graph per kind: objective kernel -> fp64 ncclAllReduce of the
//     2*n_global result vector -> D2H);
//   * the ordered left fold of per-dataset sums (musr.py:190-201).
//
// The handle is single-threaded, like the reference orchestration.

#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvrtc.h>
#include <signal.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cerrno>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <chrono>
#include <map>
#include <mutex>
#include <string>
#include <unordered_map>
#include <thread>
#include <vector>

#include "../../include/musr_b200.h"
#include "musr_layout.h"
#include "musr_embedded.inc"  // kMusrLayoutSrc, kMusrPreludeSrc, kMusrKernelSrc (generated at build time)

static_assert(sizeof(MusrHist) == 64, "MusrHist layout");

namespace {

thread_local std::string g_error;

// ---- minimal NCCL surface, resolved with dlopen (only sharded handles) ------
struct NcclId { unsigned char bytes[128]; };
typedef void* NcclComm;
struct NcclApi {
  void* lib = nullptr;
  int (*GetUniqueId)(NcclId*) = nullptr;
  int (*CommInitRank)(NcclComm*, int, NcclId, int) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
  int (*CommDestroy)(NcclComm) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
};
constexpr int kNcclFloat64 = 8;
constexpr int kNcclSum = 0;

std::mutex g_nccl_mu;
NcclApi g_nccl;

bool load_nccl(const char* path, std::string* err) {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (g_nccl.lib) return true;
  void* h = dlopen(path && *path ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    *err = std::string("cannot load NCCL: ") + dlerror();
    return false;
  }
  NcclApi api;
  api.lib = h;
  api.GetUniqueId = (int (*)(NcclId*))dlsym(h, "ncclGetUniqueId");
  api.CommInitRank = (int (*)(NcclComm*, int, NcclId, int))dlsym(h, "ncclCommInitRank");
  api.AllReduce = (int (*)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t))dlsym(
      h, "ncclAllReduce");
  api.CommDestroy = (int (*)(NcclComm))dlsym(h, "ncclCommDestroy");
  api.GetErrorString = (const char* (*)(int))dlsym(h, "ncclGetErrorString");
  if (!api.GetUniqueId || !api.CommInitRank || !api.AllReduce || !api.CommDestroy ||
      !api.GetErrorString) {
    *err = "NCCL library lacks required symbols";
    dlclose(h);
    return false;
  }
  g_nccl = api;
  return true;
}

// ---- driver API resolved through the runtime (no link-time libcuda) -----------
struct DriverApi {
  bool ok = false;
  CUresult (*ModuleLoadData)(CUmodule*, const void*) = nullptr;
  CUresult (*ModuleGetFunction)(CUfunction*, CUmodule, const char*) = nullptr;
  CUresult (*ModuleUnload)(CUmodule) = nullptr;
  CUresult (*LaunchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned,
                           unsigned, unsigned, CUstream, void**, void**) = nullptr;
  CUresult (*GetErrorString)(CUresult, const char**) = nullptr;
  CUresult (*OccupancyMaxActiveBlocksPerMultiprocessor)(int*, CUfunction, int, size_t) = nullptr;
  CUresult (*FuncSetAttribute)(CUfunction, CUfunction_attribute, int) = nullptr;
  CUresult (*ModuleGetGlobal)(CUdeviceptr*, size_t*, CUmodule, const char*) = nullptr;
  CUresult (*FuncGetAttribute)(int*, CUfunction_attribute, CUfunction) = nullptr;
};
std::mutex g_drv_mu;
DriverApi g_drv;

bool load_driver(std::string* err) {
  std::lock_guard<std::mutex> lk(g_drv_mu);
  if (g_drv.ok) return true;
  DriverApi d;
  struct { const char* name; void** slot; } syms[] = {
      {"cuModuleLoadData", (void**)&d.ModuleLoadData},
      {"cuModuleGetFunction", (void**)&d.ModuleGetFunction},
      {"cuModuleUnload", (void**)&d.ModuleUnload},
      {"cuLaunchKernel", (void**)&d.LaunchKernel},
      {"cuGetErrorString", (void**)&d.GetErrorString},
      {"cuOccupancyMaxActiveBlocksPerMultiprocessor",
       (void**)&d.OccupancyMaxActiveBlocksPerMultiprocessor},
      {"cuFuncSetAttribute", (void**)&d.FuncSetAttribute},
      {"cuModuleGetGlobal", (void**)&d.ModuleGetGlobal},
      {"cuFuncGetAttribute", (void**)&d.FuncGetAttribute},
  };
  for (auto& s : syms) {
    cudaDriverEntryPointQueryResult q;
    cudaError_t ce = cudaGetDriverEntryPoint(s.name, s.slot, cudaEnableDefault, &q);
    if (ce != cudaSuccess || q != cudaDriverEntryPointSuccess || !*s.slot) {
      *err = std::string("driver entry point ") + s.name + " unavailable";
      return false;
    }
  }
  d.ok = true;
  g_drv = d;
  return true;
}

// ---- JIT cache ---------------------------------------------------------------
std::mutex g_jit_mu;
std::unordered_map<std::string, std::vector<std::string>> g_cubin_cache;  // source -> per-entry cubins
constexpr int kEntries = 10;  // musr_kernel.cuh: MUSR_ONLY = 1 .. 10

uint64_t fnv1a(const std::string& s) {
  uint64_t h = 1469598103934665603ull;
  for (unsigned char c : s) { h ^= c; h *= 1099511628211ull; }
  return h;
}

std::string fmt(const char* f, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, f);
  vsnprintf(buf, sizeof(buf), f, ap);
  va_end(ap);
  return buf;
}

}  // namespace

struct musr_ctx {
  int device = 0;
  int rank = 0, world = 1;
  cudaStream_t stream = nullptr;
  std::string err;

  // theory module
  CUmodule mods[kEntries + 1] = {};  // per entry point (index 1..kEntries; see MUSR_ONLY)
  CUfunction fn[2][3] = {};  // [kind][kernel format: 0 f64, 1 c32, 2 c32 + counts beyond the table]
  CUfunction fn_utab = nullptr;
  CUfunction fn_batch[2][3] = {};  // musr_eval_batch
  bool have_theory = false;
  int n_uniform = 1;            // MUSR_NU of the loaded theory
  int nu_reg = 1, n_rot = 0;    // its MUSR_NU_REG, MUSR_NROT
  // host uniform program (musr_set_uniform_program): int32 (op, dst, a, b) + literals
  std::vector<int32_t> ucode;
  std::vector<double> ulits;
  int u_nreg = 0;
  bool device_rows = false;     // MUSR_DEVICE_ROWS (at open): rows in the CTA prologue always
  int sms = 0;                  // multiprocessors on the device
  int per_thread = 8;           // MUSR_PT: terms per consumer thread
  int cwarps = 16;              // MUSR_CWARPS: consumer warps per CTA; tile = 32*cwarps*per_thread
  int stages = 3;               // MUSR_STAGES: deepest TMA pipeline compiled in
  int stages_used[2] = {0, 0};  // depth that fits per kind (plan_launch)
  int stages_batch[2] = {0, 0};
  int min_blocks = 1;           // MUSR_MIN_BLOCKS: register budget target
  double* utab = nullptr;       // uniform table (sized at graph build)
  size_t utab_rows = 0;
  unsigned long long* trace = nullptr;  // MUSR_TRACE=1: per-CTA timeline
  unsigned* sched = nullptr;    // [2] dynamic tile scheduler: next tile, spare (self-resetting)
  unsigned grid[2] = {0, 0};    // persistent grid per kind
  size_t dyn_smem[2] = {0, 0};  // dynamic shared memory per kind
  unsigned grid_batch[2] = {0, 0};
  size_t dyn_smem_batch[2] = {0, 0};
  int per_thread_data = 8;      // per_thread the uploaded layout was padded for

  // data
  bool have_data = false;
  bool have_errors = false;
  int n_global = 0, n_local = 0;
  int64_t n_tiles = 0;
  int p_capacity = 0;
  void* d = nullptr;            // fp64, or fp32 (c32 format, exact integers)
  double* env = nullptr;
  double2* table = nullptr;
  int table_size = 0;
  bool big_counts = false;      // c32: some count >= table_size
  int fmt = 0;                  // 0: f64 streams, 1: c32 (fp32 counts + err/rcp table)
  int* tile_hist = nullptr;
  MusrHist* hist = nullptr;
  double* P = nullptr;
  int* maps = nullptr;
  double* fvals = nullptr;
  double* partial = nullptr;
  unsigned* count = nullptr;
  unsigned long long* bad = nullptr;
  double* out_send = nullptr;
  double* out_recv = nullptr;
  double* h_p = nullptr;    // pinned
  double* P_batch = nullptr;    // [MUSR_KMAX][p_capacity] (musr_eval_batch)
  double* h_p_batch = nullptr;  // pinned staging of P_batch
  double* h_out_batch = nullptr;  // pinned + mapped, [MUSR_KMAX][2 * n_global]
  double* h_out_batch_dev = nullptr;  // device alias of h_out_batch (host-row batches write here)
  double* h_utab = nullptr;     // pinned: host-evaluated rows of a batch, [MUSR_KMAX][n_local][row]
  size_t h_utab_rows = 0;
  double* h_out = nullptr;  // pinned + mapped, 2 * n_global
  double* h_out_dev = nullptr;  // device alias of h_out (direct path writes here)
  std::vector<double> last_p;   // parameter vector of the last evaluation (timing replays)
  MusrArgs direct_args;         // prebuilt direct-launch arguments (only pin[]/epoch change)
  unsigned long long* ll_host = nullptr;  // mapped LL result words (direct path), 4 per dataset
  unsigned long long* ll_dev = nullptr;
  // Shared results (musr_open_shared): every rank's kernel writes its datasets'
  // LL words into one host buffer mapped by all ranks' processes (double-
  // buffered by epoch parity), so each host reads every dataset's result
  // without a device collective.
  unsigned long long* shared_host = nullptr;  // caller-owned, registered mapped
  unsigned long long* shared_dev = nullptr;
  size_t shared_bytes = 0;
  unsigned long long epoch_base = 0;
  unsigned long long epoch = 0;
  bool direct_args_ok = false;
  bool direct_args_rows = false;  // direct_args.u holds host rows (not pin / min / fin)
  bool h_inline = false;        // metadata small enough for kernel-parameter space
  std::vector<MusrHist> hist_host;
  std::vector<int32_t> maps_host;
  std::vector<double> fvals_host;
  int map_stride = 1, f_stride = 1;
  int last_np = -1;

  // graphs (one per kind), with event nodes around the objective kernel
  cudaGraphExec_t gexec[2] = {nullptr, nullptr};
  cudaEvent_t kev[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};

  // sharding
  NcclComm comm = nullptr;

  // L2 flush scratch for timing
  void* flush = nullptr;
  size_t flush_bytes = 0;
};

// Tile layout of one stream (musr_kernel.cuh): tiles of cthreads*pt terms; inside
// a tile the 16-byte group k*cthreads + t holds thread t's elements g*k .. g*k+g-1
// (g = 16 / element size), so consumer reads are conflict-free LDS.128.
// mode 0: fp64 copy, 1: fp32 (the c32 format: integer counts < 2^23, exact).
__global__ void musr_layout_stream(const double* __restrict__ src, void* __restrict__ dst,
                                   size_t terms, unsigned pt, unsigned cthreads, int mode) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= terms) return;
  const size_t tile_terms = (size_t)cthreads * pt;
  const size_t tile = i / tile_terms;
  const unsigned r = (unsigned)(i - tile * tile_terms);
  const unsigned g = (mode == 1) ? 4u : 2u;
  const unsigned grp = r / g, e = r - grp * g, k = grp / cthreads, t = grp % cthreads;
  const double v = src[tile * tile_terms + (size_t)t * pt + g * k + e];
  if (mode == 1)
    static_cast<float*>(dst)[i] = (float)v;
  else
    static_cast<double*>(dst)[i] = v;
}

// L2 flush for timing (writes > 126 MB).  A kernel rather than cudaMemset so
// it can prefer the same max-shared carveout as the objective kernels: a
// carveout change forces the SMs to drain and reconfigure at the next launch.
__global__ void musr_l2_flush(double4* buf, size_t n, double v) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    buf[i] = make_double4(v, v, v, v);
}

// flush_l2 == 2: after the write pass, read the first half of the flush buffer
// so the L2 holds clean lines only (no write-back of the flush's dirty lines
// inside the timed kernel).  The values written are >= 0, so the sink store
// never happens; it only keeps the loads alive.
__global__ void musr_l2_clean(const double4* buf, size_t n, double* sink) {
  double acc = 0.0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    acc += __ldcg(reinterpret_cast<const double2*>(buf + i)).x;
  if (acc < 0.0) *sink = acc;
}

// c32 table: {max(1, sqrt(k)), 1 / that}, both correctly rounded like numpy's
// np.maximum(1.0, np.sqrt(d)) and 1.0 / err.
__global__ void musr_build_table(double2* table, int n) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const double s = __dsqrt_rn((double)k);
  const double e = s < 1.0 ? 1.0 : s;
  table[k] = make_double2(e, __drcp_rn(e));
}

namespace {

constexpr int kMaxStaged = 64;         // MUSR_MAX_STAGED

int set_err(musr_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg; else g_error = msg;
  return code;
}

#define CUDA_TRY(ctx, expr)                                                           \
  do {                                                                                \
    cudaError_t e_ = (expr);                                                          \
    if (e_ != cudaSuccess)                                                            \
      return set_err(ctx, MUSR_ERR_CUDA,                                              \
                     fmt("%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, __LINE__)); \
  } while (0)

#define CU_TRY(ctx, expr)                                                             \
  do {                                                                                \
    CUresult r_ = (expr);                                                             \
    if (r_ != CUDA_SUCCESS) {                                                         \
      const char* s_ = nullptr;                                                       \
      if (g_drv.GetErrorString) g_drv.GetErrorString(r_, &s_);                       \
      return set_err(ctx, MUSR_ERR_CUDA, fmt("%s: %s", #expr, s_ ? s_ : "?"));       \
    }                                                                                 \
  } while (0)

void free_graphs(musr_ctx* c) {
  c->direct_args_ok = false;
  for (auto& g : c->gexec) {
    if (g) cudaGraphExecDestroy(g);
    g = nullptr;
  }
}

void free_data(musr_ctx* c) {
  free_graphs(c);
  void* dev[] = {c->d, c->env, c->table, c->tile_hist, c->hist, c->P, c->maps,
                 c->fvals, c->partial, c->count, c->bad, c->out_send, c->out_recv, c->utab,
                 c->sched, c->P_batch};
  for (void* p : dev)
    if (p) cudaFree(p);
  c->d = nullptr;
  c->env = nullptr;
  c->table = nullptr;
  c->table_size = 0;
  c->tile_hist = nullptr;
  c->hist = nullptr;
  c->P = nullptr;
  c->maps = nullptr;
  c->fvals = nullptr;
  c->partial = nullptr;
  c->count = nullptr;
  c->bad = nullptr;
  c->out_send = c->out_recv = nullptr;
  c->utab = nullptr;
  c->utab_rows = 0;
  c->sched = nullptr;
  c->P_batch = nullptr;
  if (c->h_p_batch) cudaFreeHost(c->h_p_batch);
  if (c->h_out_batch) cudaFreeHost(c->h_out_batch);
  c->h_p_batch = c->h_out_batch = c->h_out_batch_dev = nullptr;
  if (c->h_utab) cudaFreeHost(c->h_utab);
  c->h_utab = nullptr;
  c->h_utab_rows = 0;
  if (c->ll_host && c->ll_host != c->shared_host) cudaFreeHost(c->ll_host);
  c->ll_host = c->ll_dev = nullptr;
  if (c->h_p) cudaFreeHost(c->h_p);
  if (c->h_out) cudaFreeHost(c->h_out);
  c->h_p = c->h_out = nullptr;
  c->h_out_dev = nullptr;
  c->have_data = false;
  c->last_np = -1;
}

// Direct-launch path: single GPU, per-dataset rows staged per CTA.  One
// kernel launch per evaluation, parameters inline in the kernel parameters,
// results written straight to mapped pinned host memory.
// (Any number of datasets: beyond kMaxStaged the launch is preceded by the
// uniform-table kernel, since the per-CTA rows no longer fit shared memory.)
bool direct_mode(const musr_ctx* c) { return c->comm == nullptr; }

// Kernel variant for the data format: chi2 on c32 data with counts beyond the
// {err, 1/err} table has its own entry point (the in-kernel sqrt / reciprocal
// path would otherwise cost the common table-only kernel registers).
int kfmt(const musr_ctx* c, int kind) { return (kind == 0 && c->fmt == 1 && c->big_counts) ? 2 : c->fmt; }

MusrArgs make_args(const musr_ctx* c, bool direct = false) {
  MusrArgs a;
  std::memset(&a, 0, sizeof(a));
  a.d = c->d;
  a.env = c->env;
  a.table = c->table;
  a.table_size = c->table_size;
  a.tile_hist = c->tile_hist;
  a.hist = c->hist;
  a.P = c->P;
  a.maps = c->maps;
  a.fvals = c->fvals;
  a.partial = c->partial;
  a.count = c->count;
  a.bad = c->bad;
  a.out = direct ? c->h_out_dev : c->out_send;
  a.h_inline = c->h_inline ? 1 : 0;
  if (c->h_inline) {
    for (int i = 0; i < c->n_local; ++i) {
      a.hin[i] = c->hist_host[i];
      for (int k = 0; k < c->map_stride; ++k)
        a.u.dev.min[i][k] = c->maps_host[(size_t)i * c->map_stride + k];
      for (int k = 0; k < c->f_stride; ++k)
        a.u.dev.fin[i][k] = c->fvals_host[(size_t)i * c->f_stride + k];
    }
  }
  a.ll = c->ll_dev;
  a.utab = c->utab;
  a.trace = c->trace;
  a.sched = c->sched;
  a.n_tiles = (int)c->n_tiles;
  a.n_global = c->n_global;
  a.n_local = c->n_local;
  a.n_points = 1;
  a.p_stride = c->p_capacity;
  return a;
}

// Host uniform rows (the reference evaluates these parameter-only values as numpy
// float64 scalars on the host, theory.py:409-464): direct path, inline metadata,
// and all local rows within MUSR_R_INLINE doubles.
bool host_rows_ok(const musr_ctx* c) {
  return !c->device_rows && !c->ucode.empty() && c->h_inline && direct_mode(c) &&
         (size_t)c->n_local * (size_t)(c->n_uniform + 2) <= MUSR_R_INLINE;
}

// Evaluate every local dataset's row [U (nu_reg) | rotation tables | N0 | Nbkg]
// with the theory's uniform program (codegen.py: _UniformProgram) -- the same
// operations as the device prologue (musr_uniform / musr_rot_entry) in IEEE double
// arithmetic, exp / log / cos / sin / pow from the host libm.
int eval_uniform_rows(musr_ctx* c, const double* p, int n_p, double* rows) {
  const int row = c->n_uniform + 2, pt = c->per_thread;
  static thread_local std::vector<double> R, last_w;
  R.assign((size_t)std::max(c->u_nreg, 1), 0.0);
  last_w.assign((size_t)std::max(c->n_rot, 1), 0.0);
  const int32_t* code = c->ucode.data();
  const int n_ins = (int)c->ucode.size() / 4;
  for (int i = 0; i < c->n_local; ++i) {
    const int32_t* M = c->maps_host.data() + (size_t)i * c->map_stride;
    const double* F = c->fvals_host.data() + (size_t)i * c->f_stride;
    const MusrHist& H = c->hist_host[i];
    double* U = rows + (size_t)i * row;
    std::fill(U, U + row, 0.0);
    for (int k = 0; k < n_ins; ++k) {
      const int op = code[4 * k], d = code[4 * k + 1], x = code[4 * k + 2], y = code[4 * k + 3];
      switch (op) {
        case 0: R[d] = c->ulits[x]; break;
        case 1:
          if (x >= c->map_stride || M[x] >= n_p)
            return set_err(c, MUSR_ERR_ARG, "p[m[k]] out of range");
          R[d] = p[M[x]];
          break;
        case 2:
          if (x >= c->map_stride || M[x] >= c->f_stride)
            return set_err(c, MUSR_ERR_ARG, "f[m[k]] out of range");
          R[d] = F[M[x]];
          break;
        case 3: R[d] = -R[x]; break;
        case 4: R[d] = R[x] + R[y]; break;
        case 5: R[d] = R[x] - R[y]; break;
        case 6: R[d] = R[x] * R[y]; break;
        case 7: R[d] = R[x] / R[y]; break;
        case 8: R[d] = R[x] * R[x]; break;
        case 9: R[d] = std::sqrt(R[x]); break;
        case 10: R[d] = 1.0 / R[x]; break;
        case 11: {  // np.power, bin-uniform exponent (musr_npy_pow_u)
          const double b = R[y], v = R[x];
          R[d] = b == 2.0 ? v * v : b == 0.5 ? std::sqrt(v) : b == -1.0 ? 1.0 / v
               : b == 1.0 ? v : b == 0.0 ? 1.0 : std::pow(v, b);
          break;
        }
        case 12: R[d] = std::pow(R[x], R[y]); break;
        case 13: R[d] = std::exp(R[x]); break;
        case 14: R[d] = std::log(R[x]); break;
        case 15: R[d] = std::cos(R[x]); break;
        case 16: R[d] = std::sin(R[x]); break;
        case 17: U[d] = R[x]; break;
        case 18: {  // rotation table d: D_j = W * (j * dt), cos D_j, sin D_j (musr_rot_entry)
          const double W = R[x];
          double* T = U + c->nu_reg + 4 * pt * d;
          const double* prev = i ? rows + (size_t)(i - 1) * row + c->nu_reg + 4 * pt * d : nullptr;
          if (prev && c->hist_host[i - 1].dt == H.dt && last_w[d] == W) {
            std::memcpy(T, prev, sizeof(double) * 4 * pt);  // same slope and bin width
            break;
          }
          last_w[d] = W;
          for (int j = 1; j < pt; ++j) {
            const double D = W * ((double)j * H.dt);
            T[4 * j] = D;
            T[4 * j + 1] = std::cos(D);
            T[4 * j + 2] = std::sin(D);
          }
          break;
        }
        default: break;
      }
      (void)y;
    }
    if (H.n0_slot >= n_p || H.nbkg_slot >= n_p)
      return set_err(c, MUSR_ERR_ARG, "N0 / Nbkg slot out of range");
    U[c->n_uniform] = p[H.n0_slot];
    U[c->n_uniform + 1] = p[H.nbkg_slot];
  }
  return MUSR_OK;
}

// The evaluation's kernels: [uniform table,] objective tiles.  `a` carries
// the parameter vector inline when `pinl` is given (direct path).
int launch_kernels(musr_ctx* c, int kind, bool with_table, bool direct = false,
                   const double* pinl = nullptr, int n_p = -1, unsigned long long epoch = 0) {
  if (c->n_tiles == 0) return MUSR_OK;  // rank without datasets
  MusrArgs local;
  MusrArgs* ap = &local;
  if (direct) {  // reuse the prebuilt block; only the inline parameters change per call
    const bool rows = host_rows_ok(c);
    if (!c->direct_args_ok || c->direct_args_rows != rows) {
      c->direct_args = make_args(c, true);
      c->direct_args_ok = true;
      c->direct_args_rows = rows;
    }
    ap = &c->direct_args;
    ap->p_inline = n_p >= 0 ? 1 : 0;
    ap->r_inline = 0;
    if (rows) {  // the uniform rows from the host program, in place of pin / min / fin
      const int rc = eval_uniform_rows(c, c->last_p.data(), (int)c->last_p.size(), ap->u.rin);
      if (rc != MUSR_OK) return rc;
      ap->r_inline = 1;
      ap->p_inline = 0;
      n_p = -1;  // (pin shares the space)
    }
  } else {
    local = make_args(c, false);
  }
  MusrArgs& a = *ap;
  a.epoch = epoch;
  if (c->shared_host)  // double-buffered by epoch parity: a rank running one evaluation
    a.ll = c->ll_dev + (size_t)(epoch & 1ull) * 4 * c->n_global;  // ahead never overwrites

  a.stages = c->stages_used[kind];
  if (n_p >= 0) {
    a.p_inline = 1;
    if (n_p) std::memcpy(a.u.dev.pin, pinl, sizeof(double) * (size_t)n_p);
  }
  void* params[] = {&a};
  with_table = with_table && c->n_local > kMaxStaged;
  if (with_table)
    CU_TRY(c, g_drv.LaunchKernel(c->fn_utab, (unsigned)((c->n_local + 3) / 4), 1, 1, 128, 1,
                                 1, 0, (CUstream)c->stream, params, nullptr));
  CU_TRY(c, g_drv.LaunchKernel(c->fn[kind][kfmt(c, kind)], c->grid[kind], 1, 1, 32 * (c->cwarps + 1), 1, 1,
                               (unsigned)c->dyn_smem[kind], (CUstream)c->stream, params, nullptr));
  return MUSR_OK;
}

constexpr int kTableMax = 4096;          // c32 chi2: {err, 1/err} table entries (64 KB)
constexpr double kCompactMax = 8388608.0;  // c32 format: counts are integers < 2^23 (fp32-exact table index)

// Deepest TMA pipeline (<= max_stages) whose shared memory fits one CTA per SM:
// `stage` bytes per stage plus `extra` (table, staged rows); `per_stage`
// bytes of extra per stage (batched thread-node blocks).  0 if none fits.
int fit_stages(CUfunction fn, int threads, size_t stage, size_t per_stage, size_t extra,
               int max_stages, size_t* smem_out, int* occ_out) {
  // candidates beyond the opt-in limit (minus the kernel's static shared
  // memory) are skipped without asking the driver (no failing API calls)
  int dev = 0, optin = 0, stat = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  g_drv.FuncGetAttribute(&stat, CU_FUNC_ATTRIBUTE_SHARED_SIZE_BYTES, fn);
  for (int st = max_stages; st >= 1; --st) {
    const size_t smem = (size_t)st * (stage + per_stage) + extra;
    if (optin > 0 && smem + (size_t)stat > (size_t)optin) continue;
    if (g_drv.FuncSetAttribute(fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)smem) !=
        CUDA_SUCCESS)
      continue;
    int occ = 0;
    if (g_drv.OccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem) != CUDA_SUCCESS ||
        occ < 1)
      continue;
    g_drv.FuncSetAttribute(fn, CU_FUNC_ATTRIBUTE_PREFERRED_SHARED_MEMORY_CARVEOUT, 100);
    *smem_out = smem;
    *occ_out = occ;
    return st;
  }
  return 0;
}

// Persistent grid, TMA pipeline depth and dynamic shared memory per objective
// kind.  The kernel is compiled for up to MUSR_STAGES stages and takes the
// depth that fits at run time (MusrArgs::stages): a large count table or many
// staged datasets cost a stage instead of failing the launch.
int plan_launch(musr_ctx* c) {
  const size_t tile = (size_t)32 * c->cwarps * c->per_thread;  // terms per tile
  const int threads = 32 * (c->cwarps + 1);
  for (int kind = 0; kind < 2; ++kind) {
    // MusrGeom in musr_kernel.cuh: d | env
    const size_t stage = tile * (c->fmt ? 4 : 8) + tile * 8;
    const int max_st = c->stages;
    size_t extra = 0;
    if (kind == 0 && c->fmt == 1) extra += (size_t)c->table_size * 16;
    size_t extra_rows = 0;
    if (c->n_local <= kMaxStaged) extra_rows = (size_t)c->n_local * (c->n_uniform + 2) * sizeof(double);
    int occ = 0;
    const int st = fit_stages(c->fn[kind][kfmt(c, kind)], threads, stage, 0, extra + extra_rows, max_st,
                              &c->dyn_smem[kind], &occ);
    if (st < 1) return set_err(c, MUSR_ERR_CUDA, "objective kernel does not fit on an SM");
    c->stages_used[kind] = st;
    c->grid[kind] = (unsigned)std::max<int64_t>(1, std::min<int64_t>(c->n_tiles, (int64_t)c->sms * occ));

    // batched variant: rows come from the global table; the per-point thread
    // nodes take the place of the staged rows (musr_kernel.cuh: s_tn)
    const size_t tn_block = (size_t)MUSR_KMAX * c->cwarps * 33 * sizeof(double);  // [KMAX][TN_K * 33]
    int occ_b = 0;
    const int st_b = fit_stages(c->fn_batch[kind][kfmt(c, kind)], threads, stage, tn_block, extra, max_st,
                                &c->dyn_smem_batch[kind], &occ_b);
    c->stages_batch[kind] = st_b;
    // 0: the batched kernel does not fit (musr_eval_batch then evaluates the
    // points one launch at a time)
    c->grid_batch[kind] =
        st_b < 1 ? 0u
                 : (unsigned)std::max<int64_t>(1, std::min<int64_t>(c->n_tiles, (int64_t)c->sms * occ_b));
  }
  if (std::getenv("MUSR_TRACE") && !c->trace) {
    // per-CTA blocks (sms * 32 words), then [tile][3] stamps for up to 2^16 tiles
    const size_t words = (size_t)c->sms * 32 + 3 * 65536;
    CUDA_TRY(c, cudaMalloc(&c->trace, words * sizeof(unsigned long long)));
    CUDA_TRY(c, cudaMemset(c->trace, 0, words * sizeof(unsigned long long)));
  }
  return MUSR_OK;
}

// Uniform table sized for the loaded theory and data.
int ensure_utab(musr_ctx* c) {
  const size_t rows = (size_t)MUSR_KMAX * std::max(1, c->n_local) * (size_t)(c->n_uniform + 2);
  if (c->utab && c->utab_rows >= rows) return MUSR_OK;
  if (c->utab) cudaFree(c->utab);
  c->utab = nullptr;
  CUDA_TRY(c, cudaMalloc(&c->utab, rows * sizeof(double)));
  CUDA_TRY(c, cudaMemset(c->utab, 0, rows * sizeof(double)));
  c->utab_rows = rows;
  return MUSR_OK;
}

int build_graphs(musr_ctx* c) {
  free_graphs(c);
  if (!c->have_theory || !c->have_data) return MUSR_OK;
  int prc = ensure_utab(c);
  if (prc == MUSR_OK) prc = plan_launch(c);
  if (prc != MUSR_OK) return prc;

  for (int kind = 0; kind < 2; ++kind) {
    if (kind == 0 && !c->have_errors) continue;
    cudaGraph_t g = nullptr;
    CUDA_TRY(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    cudaMemcpyAsync(c->P, c->h_p, sizeof(double) * c->p_capacity, cudaMemcpyHostToDevice,
                    c->stream);
    MusrArgs a = make_args(c);
    a.stages = c->stages_used[kind];
    void* params[] = {&a};
    CUresult lr = CUDA_SUCCESS;
    if (c->n_tiles > 0) {
      if (c->n_local > kMaxStaged)
        lr = g_drv.LaunchKernel(c->fn_utab, (unsigned)((c->n_local + 3) / 4), 1, 1, 128, 1,
                                1, 0, (CUstream)c->stream, params, nullptr);
      cudaEventRecordWithFlags(c->kev[kind][0], c->stream, cudaEventRecordExternal);
      if (lr == CUDA_SUCCESS)
        lr = g_drv.LaunchKernel(c->fn[kind][kfmt(c, kind)], c->grid[kind], 1, 1, 32 * (c->cwarps + 1), 1, 1,
                                (unsigned)c->dyn_smem[kind], (CUstream)c->stream, params,
                                nullptr);
      cudaEventRecordWithFlags(c->kev[kind][1], c->stream, cudaEventRecordExternal);
    }
    int nr = 0;
    if (c->comm)
      nr = g_nccl.AllReduce(c->out_send, c->out_recv, (size_t)2 * c->n_global, kNcclFloat64,
                            kNcclSum, c->comm, c->stream);
    cudaMemcpyAsync(c->h_out, c->comm ? c->out_recv : c->out_send,
                    sizeof(double) * 2 * c->n_global, cudaMemcpyDeviceToHost, c->stream);
    cudaError_t ce = cudaStreamEndCapture(c->stream, &g);
    if (lr != CUDA_SUCCESS) {
      if (g) cudaGraphDestroy(g);
      const char* s = nullptr;
      if (g_drv.GetErrorString) g_drv.GetErrorString(lr, &s);
      return set_err(c, MUSR_ERR_CUDA, fmt("cuLaunchKernel during capture: %s", s ? s : "?"));
    }
    if (nr != 0) {
      if (g) cudaGraphDestroy(g);
      return set_err(c, MUSR_ERR_NCCL,
                     fmt("ncclAllReduce during capture: %s", g_nccl.GetErrorString(nr)));
    }
    CUDA_TRY(c, ce);
    cudaError_t ie = cudaGraphInstantiate(&c->gexec[kind], g, 0);
    cudaGraphDestroy(g);
    CUDA_TRY(c, ie);
  }
  return MUSR_OK;
}

int open_common(int device, musr_ctx** out, musr_ctx** made) {
  if (!out) return set_err(nullptr, MUSR_ERR_ARG, "out is NULL");
  int n = 0;
  cudaError_t ce = cudaGetDeviceCount(&n);
  if (ce != cudaSuccess || n == 0)
    return set_err(nullptr, MUSR_ERR_CUDA,
                   fmt("no CUDA device available (%s)", cudaGetErrorString(ce)));
  if (device < 0 || device >= n)
    return set_err(nullptr, MUSR_ERR_ARG, fmt("device %d out of range [0, %d)", device, n));
  ce = cudaSetDevice(device);
  if (ce == cudaSuccess) ce = cudaFree(nullptr);  // create the primary context
  if (ce != cudaSuccess)
    return set_err(nullptr, MUSR_ERR_CUDA, fmt("cudaSetDevice: %s", cudaGetErrorString(ce)));
  std::string derr;
  if (!load_driver(&derr)) return set_err(nullptr, MUSR_ERR_CUDA, derr);
  musr_ctx* c = new musr_ctx();
  c->device = device;
  cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
  if (c->sms < 1) c->sms = 1;
  // tuning overrides (defaults are the measured best on B200)
  if (const char* v = std::getenv("MUSR_PT")) {
    const int pt = std::atoi(v);
    c->per_thread = (pt == 4 || pt == 16) ? pt : 8;
  }
  c->device_rows = std::getenv("MUSR_DEVICE_ROWS") != nullptr;
  // (5+ stages overflow the 48 KB static shared memory of the f64 MLH entry point)
  if (const char* v = std::getenv("MUSR_STAGES")) c->stages = std::max(1, std::min(4, std::atoi(v)));
  if (const char* v = std::getenv("MUSR_MIN_BLOCKS")) c->min_blocks = std::max(1, std::min(4, std::atoi(v)));
  if (const char* v = std::getenv("MUSR_CWARPS")) {
    const int w = std::atoi(v);
    c->cwarps = (w == 4 || w == 8) ? w : 16;  // 32 + the producer would exceed 1024 threads
  }
  if (c->cwarps >= 16) c->min_blocks = std::min(c->min_blocks, 1);  // >= 544 threads: one CTA per SM
  ce = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  for (auto& pair : c->kev)
    for (auto& ev : pair)
      if (ce == cudaSuccess) ce = cudaEventCreate(&ev);
  if (ce != cudaSuccess) {
    delete c;
    return set_err(nullptr, MUSR_ERR_CUDA, fmt("stream/events: %s", cudaGetErrorString(ce)));
  }
  *made = c;
  return MUSR_OK;
}

}  // namespace

extern "C" {

int musr_version(void) { return 100; }

const char* musr_global_error(void) { return g_error.c_str(); }

int musr_device_count(int* n) {
  if (!n) return set_err(nullptr, MUSR_ERR_ARG, "n is NULL");
  cudaError_t ce = cudaGetDeviceCount(n);
  if (ce != cudaSuccess) *n = 0;
  return MUSR_OK;
}

int musr_open(int device, musr_ctx** out) {
  musr_ctx* c = nullptr;
  int rc = open_common(device, out, &c);
  if (rc != MUSR_OK) return rc;
  *out = c;
  return MUSR_OK;
}

int musr_nccl_unique_id(const char* nccl_lib, unsigned char out_id[128]) {
  std::string err;
  if (!load_nccl(nccl_lib, &err)) return set_err(nullptr, MUSR_ERR_NCCL, err);
  NcclId id;
  int r = g_nccl.GetUniqueId(&id);
  if (r != 0) return set_err(nullptr, MUSR_ERR_NCCL, g_nccl.GetErrorString(r));
  std::memcpy(out_id, id.bytes, 128);
  return MUSR_OK;
}

int musr_open_sharded(int device, int rank, int world, const char* nccl_lib,
                      const unsigned char unique_id[128], musr_ctx** out) {
  if (world < 1 || rank < 0 || rank >= world)
    return set_err(nullptr, MUSR_ERR_ARG, fmt("bad rank %d / world %d", rank, world));
  std::string err;
  if (!load_nccl(nccl_lib, &err)) return set_err(nullptr, MUSR_ERR_NCCL, err);
  musr_ctx* c = nullptr;
  int rc = open_common(device, out, &c);
  if (rc != MUSR_OK) return rc;
  NcclId id;
  std::memcpy(id.bytes, unique_id, 128);
  int r = g_nccl.CommInitRank(&c->comm, world, id, rank);
  if (r != 0) {
    cudaStreamDestroy(c->stream);
    delete c;
    return set_err(nullptr, MUSR_ERR_NCCL,
                   fmt("ncclCommInitRank: %s", g_nccl.GetErrorString(r)));
  }
  c->rank = rank;
  c->world = world;
  *out = c;
  return MUSR_OK;
}

// Shared result buffers are registered once per process (several handles of
// one backend share a buffer).
static std::mutex g_shared_mu;
static std::map<void*, int> g_shared_refs;

// Liveness table at the end of a shared result buffer: one 8-byte word per
// rank holding its process id while the rank has a handle open on the buffer
// (0 = none).  A rank waiting for another rank's results checks it, so a peer
// that died or closed its handle is reported at once instead of after the
// timeout.
static volatile unsigned long long* shared_pids(void* buf, size_t bytes, int world) {
  return reinterpret_cast<volatile unsigned long long*>(static_cast<char*>(buf) + bytes) - world;
}

// 0: rank `r`'s process is alive with a handle on the buffer; else a reason.
static const char* peer_gone(const musr_ctx* c, int r) {
  const unsigned long long pid = shared_pids(c->shared_host, c->shared_bytes, c->world)[r];
  if (pid == 0) return "has no open handle on the shared result buffer";
  if (kill((pid_t)pid, 0) != 0 && errno == ESRCH) return "has exited";
  char path[64], buf[256];
  std::snprintf(path, sizeof(path), "/proc/%llu/stat", pid);
  if (FILE* f = std::fopen(path, "r")) {
    const size_t n = std::fread(buf, 1, sizeof(buf) - 1, f);
    std::fclose(f);
    buf[n] = 0;
    const char* q = std::strrchr(buf, ')');
    if (q && q[1] == ' ' && (q[2] == 'Z' || q[2] == 'X')) return "has exited (zombie)";
  }
  return nullptr;
}

int musr_open_shared(int device, int rank, int world, void* buf, size_t bytes,
                     unsigned long long epoch_base, musr_ctx** out) {
  if (world < 1 || rank < 0 || rank >= world)
    return set_err(nullptr, MUSR_ERR_ARG, fmt("bad rank %d / world %d", rank, world));
  if (!buf || bytes < 64 + (size_t)8 * world || (reinterpret_cast<uintptr_t>(buf) & 63) ||
      (bytes & 7))
    return set_err(nullptr, MUSR_ERR_ARG,
                   "shared result buffer must be 64-byte aligned, a multiple of 8 bytes and hold "
                   ">= 64 bytes plus one 8-byte word per rank");
  musr_ctx* c = nullptr;
  int rc = open_common(device, out, &c);
  if (rc != MUSR_OK) return rc;
  {
    std::lock_guard<std::mutex> lk(g_shared_mu);
    if (g_shared_refs[buf]++ == 0) {
      const cudaError_t ce = cudaHostRegister(buf, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable);
      if (ce != cudaSuccess) {
        g_shared_refs.erase(buf);
        cudaStreamDestroy(c->stream);
        delete c;
        return set_err(nullptr, MUSR_ERR_CUDA, fmt("cudaHostRegister: %s", cudaGetErrorString(ce)));
      }
    }
  }
  void* dev = nullptr;
  const cudaError_t dce = cudaHostGetDevicePointer(&dev, buf, 0);
  c->shared_host = static_cast<unsigned long long*>(buf);  // (released by musr_close)
  if (dce != cudaSuccess) {
    musr_close(c);
    return set_err(nullptr, MUSR_ERR_CUDA,
                   fmt("cudaHostGetDevicePointer: %s", cudaGetErrorString(dce)));
  }
  c->shared_dev = static_cast<unsigned long long*>(dev);
  c->shared_bytes = bytes;
  c->epoch_base = epoch_base;
  c->rank = rank;
  c->world = world;
  shared_pids(buf, bytes, world)[rank] = (unsigned long long)getpid();
  *out = c;
  return MUSR_OK;
}

void musr_close(musr_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  free_data(c);
  if (c->shared_host) {
    std::lock_guard<std::mutex> lk(g_shared_mu);
    if (--g_shared_refs[c->shared_host] == 0) {
      g_shared_refs.erase(c->shared_host);
      if (c->shared_bytes) shared_pids(c->shared_host, c->shared_bytes, c->world)[c->rank] = 0;
      cudaHostUnregister(c->shared_host);
    }
  }
  for (auto& m : c->mods)
    if (m) g_drv.ModuleUnload(m);
  if (c->comm) g_nccl.CommDestroy(c->comm);
  if (c->flush) cudaFree(c->flush);
  if (c->trace) cudaFree(c->trace);
  for (auto& pair : c->kev)
    for (auto& ev : pair)
      if (ev) cudaEventDestroy(ev);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

const char* musr_last_error(const musr_ctx* c) { return c ? c->err.c_str() : g_error.c_str(); }

}  // extern "C"

namespace {

// NVRTC: (prelude + fragment + kernel template) -> sm_100a CUBIN, cached by source.
// One NVRTC build of `src` with `opt_s`; the compiler log goes to *plog.
int nvrtc_build(musr_ctx* c, const std::string& src, const std::vector<std::string>& opt_s,
                const std::string& key, std::string* cubin, std::string* plog) {
  std::vector<const char*> opts;
  for (auto& o : opt_s) opts.push_back(o.c_str());
  const char* hdr_src[] = {kMusrLayoutSrc, kMusrMathSrc, kMusrPreludeSrc, kMusrKernelSrc};
  const char* hdr_name[] = {"musr_layout.h", "musr_math.cuh", "musr_prelude.cuh",
                            "musr_kernel.cuh"};
  const int n_hdr = sizeof(hdr_src) / sizeof(hdr_src[0]);
  nvrtcProgram prog;
  std::string pname = fmt("musr_theory_%016llx.cu", (unsigned long long)fnv1a(key));
  nvrtcResult nr = nvrtcCreateProgram(&prog, src.c_str(), pname.c_str(), n_hdr, hdr_src, hdr_name);
  if (nr != NVRTC_SUCCESS)
    return set_err(c, MUSR_ERR_NVRTC, fmt("nvrtcCreateProgram: %s", nvrtcGetErrorString(nr)));
  nr = nvrtcCompileProgram(prog, (int)opts.size(), opts.data());
  size_t log_size = 0;
  nvrtcGetProgramLogSize(prog, &log_size);
  plog->assign(log_size, '\0');
  if (log_size) nvrtcGetProgramLog(prog, &(*plog)[0]);
  if (nr != NVRTC_SUCCESS) {
    nvrtcDestroyProgram(&prog);
    return set_err(c, MUSR_ERR_NVRTC,
                   fmt("NVRTC compile failed: %s\n", nvrtcGetErrorString(nr)) + *plog);
  }
  size_t n = 0;
  nvrtcGetCUBINSize(prog, &n);
  cubin->resize(n);
  nvrtcGetCUBIN(prog, &(*cubin)[0]);
  nvrtcDestroyProgram(&prog);
  return MUSR_OK;
}

// Spill-store bytes ptxas -v reported for entry point `fn` (-1 if absent).
long spill_stores(const std::string& plog, const char* fn) {
  const std::string tag = std::string("Function properties for ") + fn + "\n";
  const size_t at = plog.find(tag);
  if (at == std::string::npos) return -1;
  const size_t eol = plog.find('\n', at + tag.size());
  const std::string line = plog.substr(at + tag.size(), eol - at - tag.size());
  const size_t k = line.find(" bytes spill stores");
  if (k == std::string::npos) return -1;
  size_t b = line.rfind(',', k);
  b = (b == std::string::npos) ? 0 : b + 1;
  return std::atol(line.substr(b, k - b).c_str());
}

// On-disk cubin cache ($MUSR_CACHE_DIR, default ~/.cache/musr_b200; MUSR_CACHE_DIR=""
// disables it): a theory compiled once loads in milliseconds in later processes.
std::string cache_path(const std::string& key, int k) {
  const char* dir = std::getenv("MUSR_CACHE_DIR");
  std::string d;
  if (dir) {
    d = dir;
  } else if (const char* home = std::getenv("HOME")) {
    d = std::string(home) + "/.cache/musr_b200";
  }
  if (d.empty()) return "";
  return d + fmt("/%016llx_%02d.cubin", (unsigned long long)fnv1a(key), k);
}
bool cache_read(const std::string& path, std::string* out) {
  if (path.empty()) return false;
  FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) return false;
  std::fseek(f, 0, SEEK_END);
  const long n = std::ftell(f);
  std::fseek(f, 0, SEEK_SET);
  bool ok = n > 0;
  if (ok) {
    out->resize((size_t)n);
    ok = std::fread(&(*out)[0], 1, (size_t)n, f) == (size_t)n;
  }
  std::fclose(f);
  return ok;
}
void cache_write(const std::string& path, const std::string& data) {
  if (path.empty()) return;
  const size_t slash = path.rfind('/');
  std::string dir = path.substr(0, slash);
  for (size_t i = 1; i <= dir.size(); ++i)  // mkdir -p
    if (i == dir.size() || dir[i] == '/') mkdir(dir.substr(0, i).c_str(), 0755);
  const std::string tmp = path + fmt(".%d.tmp", (int)getpid());
  if (FILE* f = std::fopen(tmp.c_str(), "wb")) {
    const bool ok = std::fwrite(data.data(), 1, data.size(), f) == data.size();
    std::fclose(f);
    if (ok) std::rename(tmp.c_str(), path.c_str());
    else std::remove(tmp.c_str());
  }
}

// NVRTC: (prelude + fragment + kernel template) -> one sm_100a CUBIN per entry point,
// the ten programs (-DMUSR_ONLY=k) built in parallel threads; cached by source and
// options in memory and on disk.
int jit_compile(musr_ctx* c, int per_thread, int stages, int min_blocks, int cwarps,
                const char* fragment, char* log, size_t log_cap, std::vector<std::string>* cubins) {
  std::string src = std::string("#include \"musr_prelude.cuh\"\n// generated theory\n") + fragment +
                    "\n#include \"musr_kernel.cuh\"\n";
  std::vector<std::string> opt_s = {"--gpu-architecture=sm_100a", "--fmad=false", "--std=c++17",
                                    "-lineinfo", "--prec-div=true", "--prec-sqrt=true",
                                    "--ftz=false", "-DMUSR_PT=" + std::to_string(per_thread),
                                    "-DMUSR_STAGES=" + std::to_string(stages),
                                    "-DMUSR_MIN_BLOCKS=" + std::to_string(min_blocks),
                                    "-DMUSR_CWARPS=" + std::to_string(cwarps)};
  if (std::getenv("MUSR_TRACE")) opt_s.push_back("-DMUSR_TRACE");
  // tuning hook: extra NVRTC options (e.g. "-DMUSR_PREFETCH=0 -DMUSR_MIN_BLOCKS=3")
  if (const char* extra = std::getenv("MUSR_NVRTC_OPTS")) {
    std::string s(extra), tok;
    for (size_t i = 0; i <= s.size(); ++i) {
      if (i == s.size() || s[i] == ' ') {
        if (!tok.empty()) opt_s.push_back(tok);
        tok.clear();
      } else {
        tok += s[i];
      }
    }
  }
  int nvrtc_major = 0, nvrtc_minor = 0;
  nvrtcVersion(&nvrtc_major, &nvrtc_minor);
  std::string key = src + fmt("\n//nvrtc %d.%d", nvrtc_major, nvrtc_minor);
  for (auto& o : opt_s) key += "\n//opt " + o;
  {
    std::lock_guard<std::mutex> lk(g_jit_mu);
    auto it = g_cubin_cache.find(key);
    if (it != g_cubin_cache.end()) {
      *cubins = it->second;
      if (log && log_cap) log[0] = 0;
      return MUSR_OK;
    }
  }
  // The MLH c32 kernels' lean per-bin checks (MUSR_MLH_LEAN) pay off only while the
  // theory leaves registers to spare: build with them, and if ptxas reports the
  // kernel spilling more than 32 bytes (a register-heavy theory, e.g. C3's
  // KT x exp + ge), build it again without (measured: C4 MLH -2.5 %, C3 MLH +11 %).
  const bool auto_lean = key.find("MUSR_MLH_LEAN") == std::string::npos;
  static const char* kName[kEntries + 1] = {"",
      "musr_chi2_f64", "musr_chi2_c32", "musr_chi2_c32big", "musr_mlh_f64", "musr_mlh_c32",
      "musr_chi2_f64_batch", "musr_chi2_c32_batch", "musr_chi2_c32big_batch", "musr_mlh_f64_batch",
      "musr_mlh_c32_batch"};
  cubins->assign(kEntries + 1, std::string());
  std::vector<std::string> logs(kEntries + 1);
  std::vector<int> rcs(kEntries + 1, MUSR_OK);
  std::vector<std::string> errs(kEntries + 1);
  auto build_one = [&](int k) {
    const std::string path = cache_path(key, k);
    if (cache_read(path, &(*cubins)[k])) return;
    const bool lean_entry = auto_lean && (k == 5 || k == 10);  // MLH on c32 data
    std::vector<std::string> o = opt_s;
    o.push_back("-DMUSR_ONLY=" + std::to_string(k));
    if (lean_entry) {
      o.push_back("-DMUSR_MLH_LEAN=1");
      o.push_back("--ptxas-options=-v");
    }
    musr_ctx scratch;  // per-thread error sink (set_err is not thread-safe on c)
    int rc = nvrtc_build(&scratch, src, o, key, &(*cubins)[k], &logs[k]);
    if (rc == MUSR_OK && lean_entry && spill_stores(logs[k], kName[k]) > 32) {
      o.pop_back();
      o.back() = "-DMUSR_MLH_LEAN=0";
      rc = nvrtc_build(&scratch, src, o, key, &(*cubins)[k], &logs[k]);
    }
    rcs[k] = rc;
    errs[k] = scratch.err;
    if (rc == MUSR_OK) cache_write(path, (*cubins)[k]);
  };
  std::vector<std::thread> pool;
  for (int k = 1; k <= kEntries; ++k) pool.emplace_back(build_one, k);
  for (auto& t : pool) t.join();
  std::string all_logs;
  for (int k = 1; k <= kEntries; ++k) all_logs += logs[k];
  if (log && log_cap) {
    size_t n = std::min(log_cap - 1, all_logs.size());
    std::memcpy(log, all_logs.data(), n);
    log[n] = 0;
  }
  for (int k = 1; k <= kEntries; ++k)
    if (rcs[k] != MUSR_OK) return set_err(c, rcs[k], errs[k]);
  if (const char* path = std::getenv("MUSR_DUMP_CUBIN")) {  // developer hook: the product SASS
    for (int k = 1; k <= kEntries; ++k)
      if (FILE* f = std::fopen(fmt("%s.%s", path, kName[k]).c_str(), "wb")) {
        std::fwrite((*cubins)[k].data(), 1, (*cubins)[k].size(), f);
        std::fclose(f);
      }
  }
  std::lock_guard<std::mutex> lk(g_jit_mu);
  g_cubin_cache[key] = *cubins;
  return MUSR_OK;
}

}  // namespace

extern "C" {

int musr_compile_theory(const char* fragment, char* log, size_t log_cap, size_t* cubin_bytes) {
  if (!fragment) return set_err(nullptr, MUSR_ERR_ARG, "NULL fragment");
  std::vector<std::string> cubins;
  int rc = jit_compile(nullptr, 8, 3, 1, 16, fragment, log, log_cap, &cubins);  // the defaults
  if (rc != MUSR_OK) return rc;
  size_t total = 0;
  for (auto& cb : cubins) total += cb.size();
  if (cubin_bytes) *cubin_bytes = total;
  return MUSR_OK;
}

int musr_set_tile_shape(musr_ctx* c, int per_thread, int cwarps) {
  if (!c) return set_err(c, MUSR_ERR_ARG, "NULL handle");
  // (32 consumer warps + the producer would exceed 1024 threads per CTA)
  if ((per_thread != 4 && per_thread != 8 && per_thread != 16) ||
      (cwarps != 4 && cwarps != 8 && cwarps != 16))
    return set_err(c, MUSR_ERR_ARG,
                   fmt("tile shape (%d terms/thread, %d warps) not in {4,8,16} x {4,8,16}",
                       per_thread, cwarps));
  if (c->have_theory || c->have_data)
    return set_err(c, MUSR_ERR_ARG, "the tile shape must be set before the theory and data");
  c->per_thread = per_thread;
  c->cwarps = cwarps;
  if (c->cwarps >= 16) c->min_blocks = std::min(c->min_blocks, 1);
  return MUSR_OK;
}

int musr_set_theory(musr_ctx* c, const char* fragment, char* log, size_t log_cap) {
  if (!c || !fragment) return set_err(c, MUSR_ERR_ARG, "NULL argument");
  CUDA_TRY(c, cudaSetDevice(c->device));
  // row length MUSR_NU = MUSR_NU_REG + 4 * MUSR_PT * MUSR_NROT (codegen.py)
  int nu_reg = 0, nrot = -1;
  const char* def = std::strstr(fragment, "#define MUSR_NU_REG ");
  const char* rot = std::strstr(fragment, "#define MUSR_NROT ");
  if (!def || std::sscanf(def + 20, "%d", &nu_reg) != 1 || nu_reg < 1 || !rot ||
      std::sscanf(rot + 18, "%d", &nrot) != 1 || nrot < 0)
    return set_err(c, MUSR_ERR_ARG,
                   "theory fragment must #define MUSR_NU_REG (>= 1) and MUSR_NROT (>= 0)");
  const int nu = nu_reg + 4 * c->per_thread * nrot;
  std::vector<std::string> cubins;
  if (c->have_data && c->per_thread_data != c->per_thread * 100 + c->cwarps)  // layout <-> tile
    return set_err(c, MUSR_ERR_ARG, "tile size changed after upload");
  int rc = jit_compile(c, c->per_thread, c->stages, c->min_blocks, c->cwarps, fragment, log,
                       log_cap, &cubins);
  if (rc != MUSR_OK) return rc;
  c->n_uniform = nu;
  c->nu_reg = nu_reg;
  c->n_rot = nrot;
  c->ucode.clear();  // a new theory: its uniform program (if any) comes next
  c->ulits.clear();
  free_graphs(c);
  for (auto& m : c->mods)
    if (m) {
      g_drv.ModuleUnload(m);
      m = nullptr;
    }
  c->have_theory = false;
  for (int k = 1; k <= kEntries; ++k) CU_TRY(c, g_drv.ModuleLoadData(&c->mods[k], cubins[k].data()));
  CU_TRY(c, g_drv.ModuleGetFunction(&c->fn[0][0], c->mods[1], "musr_chi2_f64"));
  CU_TRY(c, g_drv.ModuleGetFunction(&c->fn[0][1], c->mods[2], "musr_chi2_c32"));
  CU_TRY(c, g_drv.ModuleGetFunction(&c->fn[0][2], c->mods[3], "musr_chi2_c32big"));
  CU_TRY(c, g_drv.ModuleGetFunction(&c->fn[1][0], c->mods[4], "musr_mlh_f64"));
  CU_TRY(c, g_drv.ModuleGetFunction(&c->fn[1][1], c->mods[5], "musr_mlh_c32"));
  c->fn[1][2] = c->fn[1][1];
  CU_TRY(c, g_drv.ModuleGetFunction(&c->fn_utab, c->mods[1], "musr_uniform_table"));
  CU_TRY(c, g_drv.ModuleGetFunction(&c->fn_batch[0][0], c->mods[6], "musr_chi2_f64_batch"));
  CU_TRY(c, g_drv.ModuleGetFunction(&c->fn_batch[0][1], c->mods[7], "musr_chi2_c32_batch"));
  CU_TRY(c, g_drv.ModuleGetFunction(&c->fn_batch[0][2], c->mods[8], "musr_chi2_c32big_batch"));
  CU_TRY(c, g_drv.ModuleGetFunction(&c->fn_batch[1][0], c->mods[9], "musr_mlh_f64_batch"));
  CU_TRY(c, g_drv.ModuleGetFunction(&c->fn_batch[1][1], c->mods[10], "musr_mlh_c32_batch"));
  c->fn_batch[1][2] = c->fn_batch[1][1];
  for (int k : {4, 5, 9, 10}) {  // the MLH modules' exponent-folded log tables (stream-ordered)
    CUfunction init = nullptr;
    CU_TRY(c, g_drv.ModuleGetFunction(&init, c->mods[k], "musr_logk_init"));
    CU_TRY(c, g_drv.LaunchKernel(init, 8, 1, 1, 128, 1, 1, 0, (CUstream)c->stream, nullptr, nullptr));
  }
  c->have_theory = true;
  return build_graphs(c);
}

int musr_set_uniform_program(musr_ctx* c, const int32_t* code, int n_words, const double* lits,
                              int n_lits) {
  if (!c) return set_err(c, MUSR_ERR_ARG, "NULL handle");
  if (!c->have_theory) return set_err(c, MUSR_ERR_ARG, "set the theory before its uniform program");
  if (n_words < 0 || n_words % 4 || (n_words && !code) || n_lits < 0 || (n_lits && !lits))
    return set_err(c, MUSR_ERR_ARG, "uniform program: bad arguments");
  int nreg = 0;
  for (int k = 0; k < n_words / 4; ++k) {  // validate once: every operand defined before use
    const int op = code[4 * k], d = code[4 * k + 1], x = code[4 * k + 2], y = code[4 * k + 3];
    const bool bin = op == 4 || op == 5 || op == 6 || op == 7 || op == 11 || op == 12;
    bool ok = op >= 0 && op <= 18;
    if (op <= 16) {
      ok = ok && d == nreg;
      if (op == 0) ok = ok && x >= 0 && x < n_lits;
      else if (op <= 2) ok = ok && x >= 0 && x < MUSR_M_INLINE;  // map slot (checked per row)
      else ok = ok && x >= 0 && x < nreg && (!bin || (y >= 0 && y < nreg));
      ++nreg;
    } else if (op == 17) {
      ok = ok && d >= 0 && d < c->nu_reg && x >= 0 && x < nreg;
    } else {
      ok = ok && d >= 0 && d < c->n_rot && x >= 0 && x < nreg;
    }
    if (!ok) return set_err(c, MUSR_ERR_ARG, fmt("uniform program: bad instruction %d", k));
  }
  c->ucode.assign(code, code + n_words);
  c->ulits.assign(lits, lits + n_lits);
  c->u_nreg = nreg;
  c->direct_args_ok = false;
  return MUSR_OK;
}

int musr_eval_uniform_rows(musr_ctx* c, const double* p, int n_p, double* rows) {
  if (!c || (n_p && !p) || !rows) return set_err(c, MUSR_ERR_ARG, "NULL argument");
  if (c->ucode.empty() || !c->have_data)
    return set_err(c, MUSR_ERR_ARG, "uniform program and data must be set");
  return eval_uniform_rows(c, p, n_p, rows);
}

int musr_upload(musr_ctx* c, int n_global, int n_local, const int32_t* out_index,
                const int64_t* n_terms, const int64_t* first_bin, const int64_t* t0_bin,
                const double* dt, const double* const* counts, const double* const* errors,
                const double* const* envelope, const int32_t* n0_slot, const int32_t* nbkg_slot,
                const int32_t* maps, int map_stride, const double* fvals, int f_stride,
                int p_capacity) {
  if (!c) return set_err(c, MUSR_ERR_ARG, "NULL handle");
  if (n_global < 1 || n_local < 0 || n_local > n_global)
    return set_err(c, MUSR_ERR_ARG, fmt("bad dataset counts %d/%d", n_local, n_global));
  if (c->shared_host) {
    if ((size_t)2 * 4 * 8 * n_global + (size_t)8 * c->world > c->shared_bytes)
      return set_err(c, MUSR_ERR_ARG, fmt("shared result buffer of %zu bytes is too small for "
                                          "%d datasets", c->shared_bytes, n_global));
  }
  if (map_stride < 1 || f_stride < 1 || p_capacity < 1)
    return set_err(c, MUSR_ERR_ARG, "strides and p_capacity must be >= 1");
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  free_data(c);

  const int64_t tile_terms = (int64_t)32 * c->cwarps * c->per_thread;
  c->per_thread_data = c->per_thread * 100 + c->cwarps;

  std::vector<MusrHist> hv(n_local);
  std::vector<int> th;
  int64_t tiles = 0;
  bool all_err = true;  // chi2 needs errors for every local dataset
  for (int i = 0; i < n_local; ++i) {
    if (n_terms[i] < 1) return set_err(c, MUSR_ERR_ARG, fmt("dataset %d has no terms", i));
    if (!counts[i] || !envelope[i]) return set_err(c, MUSR_ERR_ARG, "NULL data array");
    if (!errors || !errors[i]) all_err = false;
    if (out_index[i] < 0 || out_index[i] >= n_global)
      return set_err(c, MUSR_ERR_ARG, "out_index out of range");
    if (n0_slot[i] < 0 || n0_slot[i] >= p_capacity || nbkg_slot[i] < 0 ||
        nbkg_slot[i] >= p_capacity)
      return set_err(c, MUSR_ERR_ARG, "N0/Nbkg slot outside p_capacity");
    const int64_t nt = (n_terms[i] + tile_terms - 1) / tile_terms;
    MusrHist& H = hv[i];
    std::memset(&H, 0, sizeof(H));
    H.n_terms = n_terms[i];
    H.first_rel = first_bin[i] - t0_bin[i];
    H.first_bin = first_bin[i];
    H.dt = dt[i];
    H.tile_start = (int)tiles;
    H.n_tiles = (int)nt;
    H.n0_slot = n0_slot[i];
    H.nbkg_slot = nbkg_slot[i];
    H.out_index = out_index[i];
    H.map_off = i * map_stride;
    H.f_off = i * f_stride;
    for (int64_t k = 0; k < nt; ++k) th.push_back(i);
    tiles += nt;
  }
  if (tiles > 0x7fffffff) return set_err(c, MUSR_ERR_ARG, "too many tiles");
  for (int i = 0; i < n_local * map_stride; ++i)
    if (maps[i] < 0)
      return set_err(c, MUSR_ERR_ARG, "negative map entry");

  // Format: c32 when every in-range count is an integer in [0, 2^23) (exact in
  // fp32, and its table index by the 2^23 bias); the chi2 table covers counts below min(max count + 1, 4096) rounded
  // up to a power of two, larger counts get err and 1/err in-kernel.
  double max_count = 0.0;
  bool compact = n_local > 0;
  for (int i = 0; compact && i < n_local; ++i) {
    const double* x = counts[i];
    for (int64_t k = 0; k < n_terms[i]; ++k) {
      const double v = x[k];
      if (!(v >= 0.0 && v < kCompactMax && v == (double)(int)v)) { compact = false; break; }
      if (v > max_count) max_count = v;
    }
  }
  if (const char* f = std::getenv("MUSR_FORMAT")) compact = compact && std::strcmp(f, "f64") != 0;
  c->fmt = compact ? 1 : 0;
  c->table_size = 0;
  c->big_counts = false;
  if (compact) {
    int ts = 16;
    while (ts < kTableMax && ts <= (int)max_count) ts <<= 1;
    c->table_size = ts;
    c->big_counts = max_count >= (double)ts;
  }

  c->n_global = n_global;
  c->n_local = n_local;
  c->n_tiles = tiles;
  c->hist_host = hv;
  c->maps_host.assign(maps, maps + (size_t)n_local * map_stride);
  c->fvals_host.assign(fvals, fvals + (size_t)n_local * f_stride);
  c->map_stride = map_stride;
  c->f_stride = f_stride;
  c->h_inline = n_local >= 1 && n_local <= MUSR_H_INLINE && map_stride <= MUSR_M_INLINE &&
                f_stride <= MUSR_F_INLINE;
  c->p_capacity = p_capacity;
  c->have_errors = all_err || compact;
  const size_t terms = (size_t)tiles * tile_terms;

  auto dalloc = [&](void** p, size_t bytes) -> int {
    if (bytes == 0) bytes = 8;
    cudaError_t ce = cudaMalloc(p, bytes);
    if (ce != cudaSuccess) {
      free_data(c);
      return set_err(c, MUSR_ERR_NOMEM,
                     fmt("cudaMalloc(%zu): %s", bytes, cudaGetErrorString(ce)));
    }
    return MUSR_OK;
  };
  int rc;
#define ALLOC(ptr, bytes) \
  if ((rc = dalloc((void**)&(ptr), (bytes))) != MUSR_OK) return rc
  ALLOC(c->d, terms * (compact ? 4 : 8));
  if (compact) ALLOC(c->table, (size_t)c->table_size * 16);
  ALLOC(c->env, terms * 8);
  ALLOC(c->tile_hist, (size_t)tiles * 4);
  ALLOC(c->hist, (size_t)n_local * sizeof(MusrHist));
  ALLOC(c->P, (size_t)p_capacity * 8);
  ALLOC(c->maps, (size_t)n_local * map_stride * 4);
  ALLOC(c->fvals, (size_t)n_local * f_stride * 8);
  ALLOC(c->partial, (size_t)MUSR_KMAX * tiles * 8);
  ALLOC(c->count, (size_t)n_local * 4);
  ALLOC(c->sched, 2 * sizeof(unsigned));
  ALLOC(c->bad, (size_t)MUSR_KMAX * n_local * 8);
  ALLOC(c->out_send, (size_t)MUSR_KMAX * 2 * n_global * 8);
  ALLOC(c->out_recv, (size_t)MUSR_KMAX * 2 * n_global * 8);
  ALLOC(c->P_batch, (size_t)MUSR_KMAX * p_capacity * 8);
#undef ALLOC
  if (cudaHostAlloc((void**)&c->h_p, (size_t)p_capacity * 8, cudaHostAllocDefault) !=
          cudaSuccess ||
      cudaHostAlloc((void**)&c->h_out, (size_t)2 * n_global * 8, cudaHostAllocMapped) !=
          cudaSuccess ||
      cudaHostGetDevicePointer((void**)&c->h_out_dev, c->h_out, 0) != cudaSuccess ||
      (!c->shared_host &&
       (cudaHostAlloc((void**)&c->ll_host, (size_t)4 * n_global * 8, cudaHostAllocMapped) !=
            cudaSuccess ||
        cudaHostGetDevicePointer((void**)&c->ll_dev, c->ll_host, 0) != cudaSuccess)) ||
      cudaHostAlloc((void**)&c->h_p_batch, (size_t)MUSR_KMAX * p_capacity * 8,
                    cudaHostAllocDefault) != cudaSuccess ||
      cudaHostAlloc((void**)&c->h_out_batch, (size_t)MUSR_KMAX * 2 * n_global * 8,
                    cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer((void**)&c->h_out_batch_dev, c->h_out_batch, 0) != cudaSuccess) {
    free_data(c);
    return set_err(c, MUSR_ERR_NOMEM, "pinned host allocation failed");
  }
  std::memset(c->h_p, 0, (size_t)p_capacity * 8);

  // Streams: dataset segments are copied into a zero-padded natural-order
  // staging buffer, then laid out per tile for the kernel (musr_layout_stream).
  {
    double* stage = nullptr;
    CUDA_TRY(c, cudaMalloc(&stage, terms * 8 + 8));
    struct Job { void* dst; const double* const* src; int mode; };
    const Job jobs[2] = {{c->d, counts, compact ? 1 : 0}, {c->env, envelope, 0}};
    int rc2 = MUSR_OK;
    for (const Job& job : jobs) {
      if (!job.dst) continue;
      cudaError_t ce = cudaMemsetAsync(stage, 0, terms * 8, c->stream);
      for (int i = 0; ce == cudaSuccess && i < n_local; ++i) {
        const size_t off = (size_t)hv[i].tile_start * tile_terms;
        ce = cudaMemcpyAsync(stage + off, job.src[i], (size_t)n_terms[i] * 8,
                             cudaMemcpyHostToDevice, c->stream);
      }
      if (ce == cudaSuccess && terms > 0) {
        musr_layout_stream<<<(unsigned)((terms + 255) / 256), 256, 0, c->stream>>>(
            stage, job.dst, terms, (unsigned)c->per_thread, (unsigned)(32 * c->cwarps), job.mode);
        ce = cudaGetLastError();
      }
      if (ce == cudaSuccess) ce = cudaStreamSynchronize(c->stream);
      if (ce != cudaSuccess) {
        rc2 = set_err(c, MUSR_ERR_CUDA, fmt("stream upload: %s", cudaGetErrorString(ce)));
        break;
      }
    }
    cudaFree(stage);
    if (rc2 != MUSR_OK) return rc2;
    if (compact) {
      musr_build_table<<<(c->table_size + 255) / 256, 256, 0, c->stream>>>(c->table,
                                                                             c->table_size);
      CUDA_TRY(c, cudaGetLastError());
      CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    }
  }
  if (!th.empty())
    CUDA_TRY(c, cudaMemcpy(c->tile_hist, th.data(), th.size() * 4, cudaMemcpyHostToDevice));
  if (!hv.empty())
    CUDA_TRY(c, cudaMemcpy(c->hist, hv.data(), hv.size() * sizeof(MusrHist),
                           cudaMemcpyHostToDevice));
  CUDA_TRY(c, cudaMemset(c->P, 0, (size_t)p_capacity * 8));
  if (n_local) {
    CUDA_TRY(c, cudaMemcpy(c->maps, maps, (size_t)n_local * map_stride * 4,
                           cudaMemcpyHostToDevice));
    CUDA_TRY(c, cudaMemcpy(c->fvals, fvals, (size_t)n_local * f_stride * 8,
                           cudaMemcpyHostToDevice));
  }
  CUDA_TRY(c, cudaMemset(c->count, 0, (size_t)n_local * 4));
  CUDA_TRY(c, cudaMemset(c->sched, 0, 2 * sizeof(unsigned)));
  if (c->shared_host) {  // epochs unique per session: stale words never match, no clearing
    c->ll_host = c->shared_host;
    c->ll_dev = c->shared_dev;
    c->epoch = c->epoch_base;
  } else {
    std::memset(c->ll_host, 0, (size_t)4 * n_global * 8);
    c->epoch = 0;
  }
  std::memset(c->h_out, 0, (size_t)2 * n_global * 8);
  CUDA_TRY(c, cudaMemset(c->bad, 0xff, (size_t)MUSR_KMAX * n_local * 8));
  CUDA_TRY(c, cudaMemset(c->out_send, 0, (size_t)MUSR_KMAX * 2 * n_global * 8));
  CUDA_TRY(c, cudaMemset(c->out_recv, 0, (size_t)MUSR_KMAX * 2 * n_global * 8));
  c->have_data = true;
  return build_graphs(c);
}

}  // extern "C"

namespace {

// One dataset's four LL words (sum hi, lo, bad hi, lo; musr_kernel.cuh
// musr_ll_put) -> its sum and (first bad bin + 1, 0 = none).
void ll_decode(const unsigned long long* x, double* sum, double* bad) {
  const unsigned long long s = ((x[0] >> 32) << 32) | (x[1] >> 32);
  const unsigned long long b = ((x[2] >> 32) << 32) | (x[3] >> 32);
  std::memcpy(sum, &s, 8);
  std::memcpy(bad, &b, 8);
}

// Per-dataset outputs and the total: the left fold of musr.py:190-201
// (total = 0.0; total += s_j in dataset order).  h = [sums | bad + 1].
void fold_results(const double* h, int G, double* per_dataset, int64_t* first_bad_bin,
                  double* total) {
  double acc = 0.0;
  for (int i = 0; i < G; ++i) {
    const double s = h[i];
    if (per_dataset) per_dataset[i] = s;
    if (first_bad_bin) {
      const double b = h[G + i];
      first_bad_bin[i] = (b == 0.0) ? -1 : (int64_t)b - 1;
    }
    acc = acc + s;
  }
  if (total) *total = acc;
}

// Device work of one evaluation on the handle's stream (no host sync).
//   direct path: [H2D p if it does not fit inline] + one objective launch
//   graph path : one graph replay (H2D p, [uniform table], objective,
//                [ncclAllReduce], D2H results)
int launch_eval(musr_ctx* c, int kind, unsigned long long epoch = 0) {
  if (direct_mode(c)) {
    const int n_p = (int)c->last_p.size();
    const bool inline_p = n_p <= MUSR_P_INLINE;
    if (!inline_p)
      CUDA_TRY(c, cudaMemcpyAsync(c->P, c->h_p, sizeof(double) * c->p_capacity,
                                  cudaMemcpyHostToDevice, c->stream));
    return launch_kernels(c, kind, true, true, c->last_p.data(), inline_p ? n_p : -1, epoch);
  }
  CUDA_TRY(c, cudaGraphLaunch(c->gexec[kind], c->stream));
  return MUSR_OK;
}

}  // namespace

extern "C" {

int musr_eval(musr_ctx* c, int kind, const double* p, int n_p, double* per_dataset,
              int64_t* first_bad_bin, double* total) {
  if (!c) return set_err(c, MUSR_ERR_ARG, "NULL handle");
  if (kind != MUSR_KIND_CHI2 && kind != MUSR_KIND_MLH)
    return set_err(c, MUSR_ERR_ARG, fmt("unknown objective kind %d", kind));
  if (!c->have_theory || !c->have_data)
    return set_err(c, MUSR_ERR_ARG, "theory and data must be set before musr_eval");
  if (!c->gexec[kind])
    return set_err(c, MUSR_ERR_ARG, "chi2 needs the error histograms (upload errors)");
  if (n_p < 0 || n_p > c->p_capacity)
    return set_err(c, MUSR_ERR_ARG, fmt("parameter vector length %d exceeds capacity %d", n_p,
                                        c->p_capacity));
  if (n_p && !p) return set_err(c, MUSR_ERR_ARG, "p is NULL");
  CUDA_TRY(c, cudaSetDevice(c->device));
  const bool inline_p = n_p <= MUSR_P_INLINE;
  if (!inline_p || !direct_mode(c)) {
    if (n_p) std::memcpy(c->h_p, p, (size_t)n_p * 8);
    if (n_p != c->last_np) {
      if (n_p < c->p_capacity) std::memset(c->h_p + n_p, 0, (size_t)(c->p_capacity - n_p) * 8);
      c->last_np = n_p;
    }
  }
  c->last_p.assign(p, p + n_p);
  static const bool no_flag = std::getenv("MUSR_NO_FLAG") != nullptr;
  // (shared results exist only as LL words: MUSR_NO_FLAG does not apply there)
  const bool flagged = direct_mode(c) && (c->n_tiles > 0 || c->shared_host) &&
                       (!no_flag || c->shared_host);
  if (flagged) {
    c->epoch += 1;
    if ((uint32_t)c->epoch == 0) c->epoch += 1;  // 0 marks "never written"
  }
  int rc = (c->n_tiles > 0 || !c->shared_host) ? launch_eval(c, kind, flagged ? c->epoch : 0)
                                                : MUSR_OK;  // a rank without datasets only reads
  if (rc != MUSR_OK) return rc;
  const int G = c->n_global;
  if (flagged) {
    // Each local dataset's stage-2 writer stores its results as LL words
    // carrying this evaluation's epoch; the host reads them as they land
    // (no completion flag, no device-side fence), typically before the kernel
    // has retired.  Bounded: after 1 s a stream sync (which reports this
    // rank's errors), after which every word of this rank is current.  Other
    // ranks' words (shared results) are then awaited while their processes are
    // alive with a handle open on the buffer, up to MUSR_PEER_TIMEOUT_S
    // (default 60 s) -- a peer that exited or closed is reported at once.
    const uint32_t e32 = (uint32_t)c->epoch;
    // shared results: every rank's datasets, in this epoch's half of the buffer
    const bool shared = c->shared_host != nullptr;
    const int n_read = shared ? G : c->n_local;
    auto out_of = [&](int j) { return shared ? j : c->hist_host[j].out_index; };
    volatile unsigned long long* ll = c->ll_host + (shared ? (size_t)(c->epoch & 1ull) * 4 * G : 0);
    int i = 0, w = 0;
    auto t_start = std::chrono::steady_clock::now();
    bool synced = false;
    static const double peer_s = [] {
      const char* v = std::getenv("MUSR_PEER_TIMEOUT_S");
      return v ? std::max(0.0, std::atof(v)) : 60.0;
    }();
    for (long spin = 0; i < n_read; ++spin) {
      const int o = out_of(i);
      while (w < 4 && (uint32_t)ll[4 * o + w] == e32) ++w;
      if (w == 4) { ++i; w = 0; continue; }
      if ((spin & 4095) != 4095) continue;
      const double waited =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
      if (!synced && waited > 1.0) {
        CUDA_TRY(c, cudaStreamSynchronize(c->stream));  // this rank's words are now final
        synced = true;
        t_start = std::chrono::steady_clock::now();
        continue;
      }
      if (!synced) continue;
      // the word still missing belongs to another rank (or the kernel failed silently)
      bool mine = !shared;
      for (int k = 0; shared && k < c->n_local; ++k) mine = mine || c->hist_host[k].out_index == o;
      if (mine)
        return set_err(c, MUSR_ERR_CUDA,
                       fmt("evaluation finished without the result of dataset %d", o));
      if ((spin & 65535) == 65535)
        for (int r = 0; r < c->world; ++r)
          if (r != c->rank)
            if (const char* why = peer_gone(c, r))
              return set_err(c, MUSR_ERR_PEER,
                             fmt("rank %d %s: the result of dataset %d (epoch %u) never "
                                 "arrived", r, why, o, e32));
      if (waited > peer_s)
        return set_err(c, MUSR_ERR_PEER,
                       fmt("the result of dataset %d (epoch %u) did not arrive within %.0f s "
                           "(MUSR_PEER_TIMEOUT_S): is every rank evaluating the same problem?",
                           o, e32, peer_s));
    }
    for (int j = 0; j < n_read; ++j) {
      const int o = out_of(j);
      ll_decode((const unsigned long long*)ll + 4 * o, &c->h_out[o], &c->h_out[G + o]);
    }
  } else {
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  }
  fold_results(c->h_out, G, per_dataset, first_bad_bin, total);
  return MUSR_OK;
}

int musr_collect_results(const unsigned long long* words, int n_global, unsigned epoch,
                         double* per_dataset, int64_t* first_bad_bin, double* total) {
  if (!words || n_global < 0) return set_err(nullptr, MUSR_ERR_ARG, "bad arguments");
  std::vector<double> h((size_t)2 * n_global);
  for (int o = 0; o < n_global; ++o) {
    for (int w = 0; w < 4; ++w)
      if ((uint32_t)words[4 * o + w] != (uint32_t)epoch)
        return set_err(nullptr, MUSR_ERR_PEER,
                       fmt("the result of dataset %d does not carry epoch %u", o, epoch));
    ll_decode(words + 4 * o, &h[o], &h[n_global + o]);
  }
  fold_results(h.data(), n_global, per_dataset, first_bad_bin, total);
  return MUSR_OK;
}

int musr_debug_trace(musr_ctx* c, int kind, uint64_t* out, int cap, int* n_ctas) {
  if (!c || !out || !n_ctas) return set_err(c, MUSR_ERR_ARG, "NULL argument");
  if (!c->trace) return set_err(c, MUSR_ERR_ARG, "handle not built with MUSR_TRACE=1");
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  // [grid][4] basic stamps, then (if cap allows) [grid][4] prologue / first-tile stamps
  const int n = std::min<int>(cap / 4, (int)c->grid[kind]);
  if (cap >= c->sms * 32 + 3 * (int)std::min<int64_t>(c->n_tiles, 65536)) {  // everything
    const size_t all = (size_t)c->sms * 32 + 3 * (size_t)std::min<int64_t>(c->n_tiles, 65536);
    CUDA_TRY(c, cudaMemcpy(out, c->trace, all * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    *n_ctas = n;
    return MUSR_OK;
  }
  const size_t words = (cap >= 20 * (int)c->grid[kind]) ? (size_t)20 * n
                       : (cap >= 16 * (int)c->grid[kind]) ? (size_t)16 * n
                       : (cap >= 8 * (int)c->grid[kind]) ? (size_t)8 * n : (size_t)4 * n;
  CUDA_TRY(c, cudaMemcpy(out, c->trace, words * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  *n_ctas = n;
  return MUSR_OK;
}

int musr_format(const musr_ctx* c, int* format, int* table_size) {
  if (!c || !format) return MUSR_ERR_ARG;
  *format = c->fmt;
  if (table_size) *table_size = c->table_size;
  return MUSR_OK;
}

int musr_n_datasets(const musr_ctx* c, int* n_global) {
  if (!c || !n_global) return MUSR_ERR_ARG;
  if (!c->have_data) return set_err(const_cast<musr_ctx*>(c), MUSR_ERR_ARG, "no data uploaded");
  *n_global = c->n_global;
  return MUSR_OK;
}

int musr_tiles(const musr_ctx* c, int64_t* n_tiles) {
  if (!c || !n_tiles) return MUSR_ERR_ARG;
  *n_tiles = c->n_tiles;
  return MUSR_OK;
}

// Batched evaluation: up to MUSR_KMAX parameter vectors per launch pair
// (uniform table over points x datasets, then one pass over the tiles that
// evaluates every point), larger batches in chunks.  Each point's results are
// bit-identical to musr_eval at that point.
int musr_eval_batch(musr_ctx* c, int kind, const double* p, int n_points, int n_p,
                    double* per_dataset, int64_t* first_bad_bin, double* totals) {
  if (!c) return set_err(c, MUSR_ERR_ARG, "NULL handle");
  if (kind != MUSR_KIND_CHI2 && kind != MUSR_KIND_MLH)
    return set_err(c, MUSR_ERR_ARG, fmt("unknown objective kind %d", kind));
  if (!c->have_theory || !c->have_data)
    return set_err(c, MUSR_ERR_ARG, "theory and data must be set before musr_eval_batch");
  if (!c->gexec[kind])
    return set_err(c, MUSR_ERR_ARG, "chi2 needs the error histograms (upload errors)");
  if (n_points < 0) return set_err(c, MUSR_ERR_ARG, "negative n_points");
  if (n_p < 0 || n_p > c->p_capacity)
    return set_err(c, MUSR_ERR_ARG, fmt("parameter vector length %d exceeds capacity %d", n_p,
                                        c->p_capacity));
  if (n_points && n_p && !p) return set_err(c, MUSR_ERR_ARG, "p is NULL");
  CUDA_TRY(c, cudaSetDevice(c->device));
  const int G = c->n_global, cap = c->p_capacity;
  // point by point when the batched kernel does not fit, and with shared results
  // (each point's results come back through the ranks' shared LL words)
  if ((c->n_tiles > 0 && c->grid_batch[kind] == 0) || c->shared_host) {
    for (int k = 0; k < n_points; ++k) {
      const int rc = musr_eval(c, kind, p + (size_t)k * n_p, n_p,
                               per_dataset ? per_dataset + (size_t)k * G : nullptr,
                               first_bad_bin ? first_bad_bin + (size_t)k * G : nullptr,
                               totals ? totals + k : nullptr);
      if (rc != MUSR_OK) return rc;
    }
    return MUSR_OK;
  }
  // Host rows (the single-evaluation path's rows, host_rows_ok): the batch's
  // uniform rows are evaluated on the host like a single call's and copied in
  // with one H2D; the kernel writes its results straight into mapped host memory.
  // One copy + one launch + a sync instead of p upload, uniform-table kernel,
  // objective, D2H and a sync -- and every point's rows are the very rows its
  // single evaluation uses.
  if (host_rows_ok(c) && c->n_tiles > 0) {
    const size_t row = (size_t)c->n_uniform + 2, per_point = (size_t)c->n_local * row;
    if (c->h_utab_rows < (size_t)MUSR_KMAX * per_point) {
      if (c->h_utab) cudaFreeHost(c->h_utab);
      c->h_utab = nullptr;
      c->h_utab_rows = 0;
      CUDA_TRY(c, cudaHostAlloc((void**)&c->h_utab, (size_t)MUSR_KMAX * per_point * 8,
                                cudaHostAllocDefault));
      c->h_utab_rows = (size_t)MUSR_KMAX * per_point;
    }
    for (int base = 0; base < n_points; base += MUSR_KMAX) {
      const int K = std::min(MUSR_KMAX, n_points - base);
      for (int k = 0; k < K; ++k)
        if (const int rc = eval_uniform_rows(c, p + (size_t)(base + k) * n_p, n_p,
                                             c->h_utab + (size_t)k * per_point))
          return rc;
      CUDA_TRY(c, cudaMemcpyAsync(c->utab, c->h_utab, (size_t)K * per_point * 8,
                                  cudaMemcpyHostToDevice, c->stream));
      MusrArgs a = make_args(c, false);
      a.P = c->P_batch;  // not read: the rows carry every parameter-dependent value
      a.p_stride = cap;
      a.p_inline = 0;
      a.n_points = K;
      a.epoch = 0;
      a.out = c->h_out_batch_dev;
      a.stages = c->stages_batch[kind];
      void* params[] = {&a};
      CU_TRY(c, g_drv.LaunchKernel(c->fn_batch[kind][kfmt(c, kind)], c->grid_batch[kind], 1, 1,
                                   32 * (c->cwarps + 1), 1, 1, (unsigned)c->dyn_smem_batch[kind],
                                   (CUstream)c->stream, params, nullptr));
      CUDA_TRY(c, cudaStreamSynchronize(c->stream));
      for (int k = 0; k < K; ++k)
        fold_results(c->h_out_batch + (size_t)k * 2 * G, G,
                     per_dataset ? per_dataset + (size_t)(base + k) * G : nullptr,
                     first_bad_bin ? first_bad_bin + (size_t)(base + k) * G : nullptr,
                     totals ? totals + base + k : nullptr);
    }
    return MUSR_OK;
  }
  for (int base = 0; base < n_points; base += MUSR_KMAX) {
    const int K = std::min(MUSR_KMAX, n_points - base);
    std::memset(c->h_p_batch, 0, (size_t)K * cap * 8);
    for (int k = 0; k < K; ++k)
      if (n_p) std::memcpy(c->h_p_batch + (size_t)k * cap, p + (size_t)(base + k) * n_p,
                           (size_t)n_p * 8);
    CUDA_TRY(c, cudaMemcpyAsync(c->P_batch, c->h_p_batch, (size_t)K * cap * 8,
                                cudaMemcpyHostToDevice, c->stream));
    if (c->n_tiles > 0) {
      MusrArgs a = make_args(c, false);
      a.P = c->P_batch;
      a.p_stride = cap;
      a.p_inline = 0;
      a.n_points = K;
      a.epoch = 0;
      a.stages = c->stages_batch[kind];
      void* params[] = {&a};
      const unsigned rows = (unsigned)(K * c->n_local);
      CU_TRY(c, g_drv.LaunchKernel(c->fn_utab, (rows + 3) / 4, 1, 1, 128, 1, 1, 0,
                                   (CUstream)c->stream, params, nullptr));  // a warp per row
      CU_TRY(c, g_drv.LaunchKernel(c->fn_batch[kind][kfmt(c, kind)], c->grid_batch[kind], 1, 1,
                                   32 * (c->cwarps + 1), 1, 1, (unsigned)c->dyn_smem_batch[kind],
                                   (CUstream)c->stream, params, nullptr));
    }
    if (c->comm) {
      const int nr = g_nccl.AllReduce(c->out_send, c->out_recv, (size_t)K * 2 * G, kNcclFloat64,
                                      kNcclSum, c->comm, c->stream);
      if (nr != 0)
        return set_err(c, MUSR_ERR_NCCL, fmt("ncclAllReduce: %s", g_nccl.GetErrorString(nr)));
    }
    CUDA_TRY(c, cudaMemcpyAsync(c->h_out_batch, c->comm ? c->out_recv : c->out_send,
                                (size_t)K * 2 * G * 8, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    for (int k = 0; k < K; ++k) {
      const double* o = c->h_out_batch + (size_t)k * 2 * G;
      const size_t row = (size_t)(base + k) * G;
      double acc = 0.0;
      for (int i = 0; i < G; ++i) {
        if (per_dataset) per_dataset[row + i] = o[i];
        if (first_bad_bin) first_bad_bin[row + i] = (o[G + i] == 0.0) ? -1 : (int64_t)o[G + i] - 1;
        acc = acc + o[i];  // musr.py:190-201, per point
      }
      if (totals) totals[base + k] = acc;
    }
  }
  return MUSR_OK;
}

int musr_time_evals(musr_ctx* c, int kind, int iters, int mode, int flush_l2, double* ms,
                    double* kernel_ms) {
  if (!c || !ms || iters < 1) return set_err(c, MUSR_ERR_ARG, "bad timing arguments");
  if (kind != 0 && kind != 1) return set_err(c, MUSR_ERR_ARG, "bad kind");
  if (!c->gexec[kind]) return set_err(c, MUSR_ERR_ARG, "objective not ready");
  CUDA_TRY(c, cudaSetDevice(c->device));
  cudaEvent_t e0, e1;
  CUDA_TRY(c, cudaEventCreate(&e0));
  CUDA_TRY(c, cudaEventCreate(&e1));
  double total = 0.0, ktotal = 0.0;
  if (mode < 0 || mode > 4) return set_err(c, MUSR_ERR_ARG, "bad timing mode");
  if (mode == 4 && c->last_p.empty() && c->p_capacity > 0)
    c->last_p.assign((size_t)c->p_capacity, 0.0);
  if ((mode == 1 || mode == 2 || mode == 3 || mode == 4) && flush_l2 && !c->flush) {
    c->flush_bytes = (size_t)512 << 20;  // > 126 MB L2
    CUDA_TRY(c, cudaMalloc(&c->flush, c->flush_bytes));
    CUDA_TRY(c, cudaFuncSetAttribute(musr_l2_flush, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     cudaSharedmemCarveoutMaxShared));
    CUDA_TRY(c, cudaFuncSetAttribute(musr_l2_clean, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     cudaSharedmemCarveoutMaxShared));
  }
  auto flush = [&](int i) -> cudaError_t {
    musr_l2_flush<<<c->sms * 4, 512, 0, c->stream>>>(static_cast<double4*>(c->flush),
                                                     c->flush_bytes / sizeof(double4), (double)i);
    if (flush_l2 == 2)
      musr_l2_clean<<<c->sms * 4, 512, 0, c->stream>>>(static_cast<const double4*>(c->flush),
                                                       c->flush_bytes / 2 / sizeof(double4),
                                                       static_cast<double*>(c->flush));
    return cudaGetLastError();
  };
  const bool direct = direct_mode(c);
  if (mode == 3) {  // L2 flush only (before an end-to-end call timed by the caller)
    if (flush_l2) CUDA_TRY(c, flush(0));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  } else if (mode == 2) {  // evaluations, each bracketed by events, L2 flushed (untimed) before each
    for (int i = 0; i < iters; ++i) {
      if (flush_l2) CUDA_TRY(c, flush(i));
      CUDA_TRY(c, cudaEventRecord(e0, c->stream));
      int rc = launch_eval(c, kind);
      if (rc != MUSR_OK) return rc;
      CUDA_TRY(c, cudaEventRecord(e1, c->stream));
      CUDA_TRY(c, cudaEventSynchronize(e1));
      float f = 0.f, fk = 0.f;
      CUDA_TRY(c, cudaEventElapsedTime(&f, e0, e1));
      if (direct)
        fk = f;  // the evaluation is the objective kernel
      else if (c->n_tiles > 0)
        CUDA_TRY(c, cudaEventElapsedTime(&fk, c->kev[kind][0], c->kev[kind][1]));
      total += f;
      ktotal += fk;
    }
  } else if (mode == 4) {
    // `iters` synchronous evaluations (musr_eval at the last parameter vector:
    // launch, then the host waits for every dataset's result -- with shared
    // results every rank's -- and folds).  Without a flush: one event before the
    // first launch and one after the last evaluation, so the interval covers
    // the launches, the kernels and the host waits between them.  With a flush
    // (inputs smaller than L2): the flush runs untimed before each evaluation,
    // which is bracketed by its own events.
    const std::vector<double> p = c->last_p;
    if (!flush_l2) CUDA_TRY(c, cudaEventRecord(e0, c->stream));
    for (int i = 0; i < iters; ++i) {
      if (flush_l2) {
        CUDA_TRY(c, flush(i));
        CUDA_TRY(c, cudaEventRecord(e0, c->stream));
      }
      const int rc = musr_eval(c, kind, p.data(), (int)p.size(), nullptr, nullptr, nullptr);
      if (rc != MUSR_OK) return rc;
      if (flush_l2) {
        CUDA_TRY(c, cudaEventRecord(e1, c->stream));
        CUDA_TRY(c, cudaEventSynchronize(e1));
        float f = 0.f;
        CUDA_TRY(c, cudaEventElapsedTime(&f, e0, e1));
        total += f;
      }
    }
    if (!flush_l2) {
      CUDA_TRY(c, cudaEventRecord(e1, c->stream));
      CUDA_TRY(c, cudaEventSynchronize(e1));
      float f = 0.f;
      CUDA_TRY(c, cudaEventElapsedTime(&f, e0, e1));
      total = f;
    }
    ktotal = total;
  } else if (mode == 0) {
    CUDA_TRY(c, cudaEventRecord(e0, c->stream));
    for (int i = 0; i < iters; ++i) {
      int rc = launch_eval(c, kind);
      if (rc != MUSR_OK) return rc;
    }
    CUDA_TRY(c, cudaEventRecord(e1, c->stream));
    CUDA_TRY(c, cudaEventSynchronize(e1));
    float f = 0.f;
    CUDA_TRY(c, cudaEventElapsedTime(&f, e0, e1));
    total = f;
  } else {
    for (int i = 0; i < iters; ++i) {
      if (flush_l2) CUDA_TRY(c, flush(i));
      CUDA_TRY(c, cudaEventRecord(e0, c->stream));
      int rc = direct ? launch_eval(c, kind) : launch_kernels(c, kind, false);
      if (rc != MUSR_OK) return rc;
      CUDA_TRY(c, cudaEventRecord(e1, c->stream));
      CUDA_TRY(c, cudaEventSynchronize(e1));
      float f = 0.f;
      CUDA_TRY(c, cudaEventElapsedTime(&f, e0, e1));
      total += f;
    }
    ktotal = total;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *ms = total;
  if (kernel_ms) *kernel_ms = ktotal;
  return MUSR_OK;
}

}  // extern "C"

// ---- fp64 DFMA throughput probe --------------------------------------------------
__global__ void __launch_bounds__(256) musr_fp64_probe(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = __fma_rn(x[k], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 1234.5678) out[0] = s;  // keep the chain alive
}

extern "C" int musr_fp64_peak(int device, double* tflops) {
  if (!tflops) return set_err(nullptr, MUSR_ERR_ARG, "tflops is NULL");
  CUDA_TRY(nullptr, cudaSetDevice(device));
  int sms = 0;
  CUDA_TRY(nullptr, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  double* out = nullptr;
  CUDA_TRY(nullptr, cudaMalloc(&out, 8));
  const int blocks = sms * 8, threads = 256, iters = 1 << 14;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    musr_fp64_probe<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  cudaError_t ce = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  CUDA_TRY(nullptr, ce);
  const double flops = 2.0 * 8.0 * (double)iters * blocks * threads;
  *tflops = flops / (best * 1e-3) / 1e12;
  return MUSR_OK;
}
