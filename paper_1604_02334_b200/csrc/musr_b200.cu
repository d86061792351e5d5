// musr_b200.cu -- host runtime of libmusr_b200.so (C ABI in include/musr_b200.h).
//
// Responsibilities:
//   * NVRTC JIT of (theory fragment + kernel template) for sm_100a, cached by
//     source hash (the paper's runtime kernel generation);
//   * device layout: per-dataset in-range segments packed into aligned
//     2048-term tiles of three fp64 streams (counts, errors, envelope);
//   * one CUDA graph per objective kind: H2D p -> objective kernel ->
//     [ncclAllReduce of the 2*n_global result vector] -> D2H results,
//     replayed once per evaluation (hides the per-call launch/upload latency
//     the paper identifies);
//   * the ordered left fold of per-dataset sums (musr.py:190-201).
//
// The handle is single-threaded, like the reference orchestration.

#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvrtc.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/musr_b200.h"
#include "musr_layout.h"
#include "musr_embedded.inc"  // kMusrLayoutSrc, kMusrPreludeSrc, kMusrKernelSrc (generated at build time)

static_assert(sizeof(MusrHist) == 64, "MusrHist layout");
static_assert(MUSR_TILE_TERMS == 2048, "tile size must match musr_kernel.cuh");

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
std::unordered_map<std::string, std::string> g_cubin_cache;  // source -> cubin

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
  CUmodule mod = nullptr;
  CUfunction fn[2] = {nullptr, nullptr};
  bool have_theory = false;

  // data
  bool have_data = false;
  bool have_errors = false;
  int n_global = 0, n_local = 0;
  int64_t n_tiles = 0;
  int p_capacity = 0;
  double* d = nullptr;
  double* e = nullptr;
  double* env = nullptr;
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
  double* h_out = nullptr;  // pinned, 2 * n_global
  int last_np = -1;

  // graphs (one per kind)
  cudaGraphExec_t gexec[2] = {nullptr, nullptr};

  // sharding
  NcclComm comm = nullptr;

  // L2 flush scratch for timing
  void* flush = nullptr;
  size_t flush_bytes = 0;
};

namespace {

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
  for (auto& g : c->gexec) {
    if (g) cudaGraphExecDestroy(g);
    g = nullptr;
  }
}

void free_data(musr_ctx* c) {
  free_graphs(c);
  void* dev[] = {c->d, c->e, c->env, c->tile_hist, c->hist, c->P, c->maps, c->fvals,
                 c->partial, c->count, c->bad, c->out_send, c->out_recv};
  for (void* p : dev)
    if (p) cudaFree(p);
  c->d = c->e = c->env = nullptr;
  c->tile_hist = nullptr;
  c->hist = nullptr;
  c->P = nullptr;
  c->maps = nullptr;
  c->fvals = nullptr;
  c->partial = nullptr;
  c->count = nullptr;
  c->bad = nullptr;
  c->out_send = c->out_recv = nullptr;
  if (c->h_p) cudaFreeHost(c->h_p);
  if (c->h_out) cudaFreeHost(c->h_out);
  c->h_p = c->h_out = nullptr;
  c->have_data = false;
  c->last_np = -1;
}

MusrArgs make_args(const musr_ctx* c) {
  MusrArgs a;
  a.d = c->d;
  a.e = c->have_errors ? c->e : c->d;
  a.env = c->env;
  a.tile_hist = c->tile_hist;
  a.hist = c->hist;
  a.P = c->P;
  a.maps = c->maps;
  a.fvals = c->fvals;
  a.partial = c->partial;
  a.count = c->count;
  a.bad = c->bad;
  a.out = c->out_send;
  a.n_global = c->n_global;
  return a;
}

int launch_kernel(musr_ctx* c, int kind) {
  if (c->n_tiles == 0) return MUSR_OK;  // rank without datasets
  MusrArgs a = make_args(c);
  void* params[] = {&a};
  CU_TRY(c, g_drv.LaunchKernel(c->fn[kind], (unsigned)c->n_tiles, 1, 1, 256, 1, 1, 0,
                           (CUstream)c->stream, params, nullptr));
  return MUSR_OK;
}

int build_graphs(musr_ctx* c) {
  free_graphs(c);
  if (!c->have_theory || !c->have_data) return MUSR_OK;
  for (int kind = 0; kind < 2; ++kind) {
    if (kind == 0 && !c->have_errors) continue;
    cudaGraph_t g = nullptr;
    CUDA_TRY(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    cudaMemcpyAsync(c->P, c->h_p, sizeof(double) * c->p_capacity, cudaMemcpyHostToDevice,
                    c->stream);
    MusrArgs a = make_args(c);
    void* params[] = {&a};
    CUresult lr = CUDA_SUCCESS;
    if (c->n_tiles > 0)
      lr = g_drv.LaunchKernel(c->fn[kind], (unsigned)c->n_tiles, 1, 1, 256, 1, 1, 0,
                          (CUstream)c->stream, params, nullptr);
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
  ce = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (ce != cudaSuccess) {
    delete c;
    return set_err(nullptr, MUSR_ERR_CUDA, fmt("stream: %s", cudaGetErrorString(ce)));
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

void musr_close(musr_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  free_data(c);
  if (c->mod) g_drv.ModuleUnload(c->mod);
  if (c->comm) g_nccl.CommDestroy(c->comm);
  if (c->flush) cudaFree(c->flush);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

const char* musr_last_error(const musr_ctx* c) { return c ? c->err.c_str() : g_error.c_str(); }

}  // extern "C"

namespace {

// NVRTC: (prelude + fragment + kernel template) -> sm_100a CUBIN, cached by source.
int jit_compile(musr_ctx* c, const char* fragment, char* log, size_t log_cap, std::string* cubin) {
  std::string src = std::string("#include \"musr_prelude.cuh\"\n// generated theory\n") + fragment +
                    "\n#include \"musr_kernel.cuh\"\n";
  const char* opts[] = {"--gpu-architecture=sm_100a", "--fmad=false", "--std=c++17",
                        "-lineinfo", "--prec-div=true", "--prec-sqrt=true", "--ftz=false"};
  const int n_opts = sizeof(opts) / sizeof(opts[0]);
  std::string key = src;
  for (const char* o : opts) key += std::string("\n//opt ") + o;
  {
    std::lock_guard<std::mutex> lk(g_jit_mu);
    auto it = g_cubin_cache.find(key);
    if (it != g_cubin_cache.end()) {
      *cubin = it->second;
      if (log && log_cap) log[0] = 0;
      return MUSR_OK;
    }
  }
  const char* hdr_src[] = {kMusrLayoutSrc, kMusrPreludeSrc, kMusrKernelSrc};
  const char* hdr_name[] = {"musr_layout.h", "musr_prelude.cuh", "musr_kernel.cuh"};
  nvrtcProgram prog;
  std::string pname = fmt("musr_theory_%016llx.cu", (unsigned long long)fnv1a(key));
  nvrtcResult nr = nvrtcCreateProgram(&prog, src.c_str(), pname.c_str(), 3, hdr_src, hdr_name);
  if (nr != NVRTC_SUCCESS)
    return set_err(c, MUSR_ERR_NVRTC, fmt("nvrtcCreateProgram: %s", nvrtcGetErrorString(nr)));
  nr = nvrtcCompileProgram(prog, n_opts, opts);
  size_t log_size = 0;
  nvrtcGetProgramLogSize(prog, &log_size);
  std::string plog(log_size, '\0');
  if (log_size) nvrtcGetProgramLog(prog, &plog[0]);
  if (log && log_cap) {
    size_t n = std::min(log_cap - 1, plog.size());
    std::memcpy(log, plog.data(), n);
    log[n] = 0;
  }
  if (nr != NVRTC_SUCCESS) {
    nvrtcDestroyProgram(&prog);
    return set_err(c, MUSR_ERR_NVRTC,
                   fmt("NVRTC compile failed: %s\n", nvrtcGetErrorString(nr)) + plog);
  }
  size_t n = 0;
  nvrtcGetCUBINSize(prog, &n);
  cubin->resize(n);
  nvrtcGetCUBIN(prog, &(*cubin)[0]);
  nvrtcDestroyProgram(&prog);
  std::lock_guard<std::mutex> lk(g_jit_mu);
  g_cubin_cache[key] = *cubin;
  return MUSR_OK;
}

}  // namespace

extern "C" {

int musr_compile_theory(const char* fragment, char* log, size_t log_cap, size_t* cubin_bytes) {
  if (!fragment) return set_err(nullptr, MUSR_ERR_ARG, "NULL fragment");
  std::string cubin;
  int rc = jit_compile(nullptr, fragment, log, log_cap, &cubin);
  if (rc != MUSR_OK) return rc;
  if (cubin_bytes) *cubin_bytes = cubin.size();
  return MUSR_OK;
}

int musr_set_theory(musr_ctx* c, const char* fragment, char* log, size_t log_cap) {
  if (!c || !fragment) return set_err(c, MUSR_ERR_ARG, "NULL argument");
  CUDA_TRY(c, cudaSetDevice(c->device));
  std::string cubin;
  int rc = jit_compile(c, fragment, log, log_cap, &cubin);
  if (rc != MUSR_OK) return rc;
  free_graphs(c);
  if (c->mod) {
    g_drv.ModuleUnload(c->mod);
    c->mod = nullptr;
  }
  c->have_theory = false;
  CU_TRY(c, g_drv.ModuleLoadData(&c->mod, cubin.data()));
  CU_TRY(c, g_drv.ModuleGetFunction(&c->fn[0], c->mod, "musr_chi2"));
  CU_TRY(c, g_drv.ModuleGetFunction(&c->fn[1], c->mod, "musr_mlh"));
  c->have_theory = true;
  return build_graphs(c);
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
  if (map_stride < 1 || f_stride < 1 || p_capacity < 1)
    return set_err(c, MUSR_ERR_ARG, "strides and p_capacity must be >= 1");
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  free_data(c);

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
    const int64_t nt = (n_terms[i] + MUSR_TILE_TERMS - 1) / MUSR_TILE_TERMS;
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

  c->n_global = n_global;
  c->n_local = n_local;
  c->n_tiles = tiles;
  c->p_capacity = p_capacity;
  c->have_errors = all_err;
  const size_t terms = (size_t)tiles * MUSR_TILE_TERMS;

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
  ALLOC(c->d, terms * 8);
  if (all_err) ALLOC(c->e, terms * 8);
  ALLOC(c->env, terms * 8);
  ALLOC(c->tile_hist, (size_t)tiles * 4);
  ALLOC(c->hist, (size_t)n_local * sizeof(MusrHist));
  ALLOC(c->P, (size_t)p_capacity * 8);
  ALLOC(c->maps, (size_t)n_local * map_stride * 4);
  ALLOC(c->fvals, (size_t)n_local * f_stride * 8);
  ALLOC(c->partial, (size_t)tiles * 8);
  ALLOC(c->count, (size_t)n_local * 4);
  ALLOC(c->bad, (size_t)n_local * 8);
  ALLOC(c->out_send, (size_t)2 * n_global * 8);
  ALLOC(c->out_recv, (size_t)2 * n_global * 8);
#undef ALLOC
  if (cudaHostAlloc((void**)&c->h_p, (size_t)p_capacity * 8, cudaHostAllocDefault) !=
          cudaSuccess ||
      cudaHostAlloc((void**)&c->h_out, (size_t)2 * n_global * 8, cudaHostAllocDefault) !=
          cudaSuccess) {
    free_data(c);
    return set_err(c, MUSR_ERR_NOMEM, "pinned host allocation failed");
  }
  std::memset(c->h_p, 0, (size_t)p_capacity * 8);

  // zero padding of the streams: padded terms are masked in-kernel, zero keeps
  // them finite and deterministic
  CUDA_TRY(c, cudaMemsetAsync(c->d, 0, terms * 8, c->stream));
  if (all_err) CUDA_TRY(c, cudaMemsetAsync(c->e, 0, terms * 8, c->stream));
  CUDA_TRY(c, cudaMemsetAsync(c->env, 0, terms * 8, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  for (int i = 0; i < n_local; ++i) {
    const size_t off = (size_t)hv[i].tile_start * MUSR_TILE_TERMS;
    const size_t bytes = (size_t)n_terms[i] * 8;
    CUDA_TRY(c, cudaMemcpy(c->d + off, counts[i], bytes, cudaMemcpyHostToDevice));
    if (all_err) CUDA_TRY(c, cudaMemcpy(c->e + off, errors[i], bytes, cudaMemcpyHostToDevice));
    CUDA_TRY(c, cudaMemcpy(c->env + off, envelope[i], bytes, cudaMemcpyHostToDevice));
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
  CUDA_TRY(c, cudaMemset(c->bad, 0xff, (size_t)n_local * 8));
  CUDA_TRY(c, cudaMemset(c->out_send, 0, (size_t)2 * n_global * 8));
  CUDA_TRY(c, cudaMemset(c->out_recv, 0, (size_t)2 * n_global * 8));
  c->have_data = true;
  return build_graphs(c);
}

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
  if (n_p) std::memcpy(c->h_p, p, (size_t)n_p * 8);
  if (n_p != c->last_np) {
    if (n_p < c->p_capacity) std::memset(c->h_p + n_p, 0, (size_t)(c->p_capacity - n_p) * 8);
    c->last_np = n_p;
  }
  CUDA_TRY(c, cudaGraphLaunch(c->gexec[kind], c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  const int G = c->n_global;
  double acc = 0.0;
  for (int i = 0; i < G; ++i) {
    const double s = c->h_out[i];
    if (per_dataset) per_dataset[i] = s;
    if (first_bad_bin) {
      const double b = c->h_out[G + i];
      first_bad_bin[i] = (b == 0.0) ? -1 : (int64_t)b - 1;
    }
    acc = acc + s;  // musr.py:190-201: total = 0.0; total += s_j in dataset order
  }
  if (total) *total = acc;
  return MUSR_OK;
}

int musr_tiles(const musr_ctx* c, int64_t* n_tiles) {
  if (!c || !n_tiles) return MUSR_ERR_ARG;
  *n_tiles = c->n_tiles;
  return MUSR_OK;
}

int musr_time_evals(musr_ctx* c, int kind, int iters, int mode, int flush_l2, double* ms) {
  if (!c || !ms || iters < 1) return set_err(c, MUSR_ERR_ARG, "bad timing arguments");
  if (kind != 0 && kind != 1) return set_err(c, MUSR_ERR_ARG, "bad kind");
  if (!c->gexec[kind]) return set_err(c, MUSR_ERR_ARG, "objective not ready");
  CUDA_TRY(c, cudaSetDevice(c->device));
  cudaEvent_t e0, e1;
  CUDA_TRY(c, cudaEventCreate(&e0));
  CUDA_TRY(c, cudaEventCreate(&e1));
  double total = 0.0;
  if (mode == 0) {
    CUDA_TRY(c, cudaEventRecord(e0, c->stream));
    for (int i = 0; i < iters; ++i) CUDA_TRY(c, cudaGraphLaunch(c->gexec[kind], c->stream));
    CUDA_TRY(c, cudaEventRecord(e1, c->stream));
    CUDA_TRY(c, cudaEventSynchronize(e1));
    float f = 0.f;
    CUDA_TRY(c, cudaEventElapsedTime(&f, e0, e1));
    total = f;
  } else {
    if (flush_l2 && !c->flush) {
      c->flush_bytes = (size_t)512 << 20;  // > 126 MB L2
      CUDA_TRY(c, cudaMalloc(&c->flush, c->flush_bytes));
    }
    for (int i = 0; i < iters; ++i) {
      if (flush_l2) CUDA_TRY(c, cudaMemsetAsync(c->flush, i & 0xff, c->flush_bytes, c->stream));
      CUDA_TRY(c, cudaEventRecord(e0, c->stream));
      int rc = launch_kernel(c, kind);
      if (rc != MUSR_OK) return rc;
      CUDA_TRY(c, cudaEventRecord(e1, c->stream));
      CUDA_TRY(c, cudaEventSynchronize(e1));
      float f = 0.f;
      CUDA_TRY(c, cudaEventElapsedTime(&f, e0, e1));
      total += f;
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *ms = total;
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
