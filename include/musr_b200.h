/* musr_b200.h -- C ABI of libmusr_b200.so, the DKS-style GPU layer for the
 * uSR fit objective (chi2 / maximum log-likelihood) on NVIDIA B200 (sm_100a).
 *
 * Every entry point is plain C: int status (0 = MUSR_OK), no exceptions across
 * the boundary, a per-handle last-error string.  A handle is driven by one
 * host thread (the reference orchestration is single-threaded).
 *
 * Reference interfaces replaced (paths under the reference tree, pkg/src/blk):
 *   musr_open / musr_open_sharded / musr_close
 *       Backend construction + worker pool, backend.py:98-155 (DKS setAPI /
 *       initDevice).  One handle = one GPU; sharded handles
 *       additionally own an NCCL communicator (one rank per process).
 *   musr_set_theory
 *       theory.evaluate's bytecode interpreter, theory.py:409-464, replaced by
 *       CUDA source generated from the AST (codegen.py) and compiled with
 *       NVRTC for sm_100a (paper's runtime kernel generation).
 *   musr_upload
 *       Backend.allocate + DeviceBuffer.write, backend.py:44-76, 127-143, fed
 *       with MusrDataset.counts / errors() / range_mask(), musr.py:66-101, and
 *       the parameter-independent envelope exp(-t/tau_mu) of musr.py:162.
 *   musr_eval
 *       musr.chi2 / musr.mlh, musr.py:181-232, including model_expected
 *       (musr.py:150-162) and Backend.map_reduce + pairwise_sum
 *       (backend.py:79-95, 174-207).  Returns per-dataset sums, the left-folded
 *       total (musr.py:190-201) and the MLH first non-positive bin per dataset.
 *   musr_eval_batch
 *       n_points calls of musr.chi2 / musr.mlh at different p in one pass over
 *       the histograms (Nelder-Mead simplex / shrink points, optimize.py:89-135;
 *       profile scans, test_acceptance.py:135-157).
 *   musr_time_evals / musr_fp64_peak
 *       measurement helpers for bench.py (no reference counterpart).
 */
#ifndef MUSR_B200_H
#define MUSR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MUSR_OK 0
#define MUSR_ERR_ARG 1      /* bad argument / state                       */
#define MUSR_ERR_CUDA 2     /* CUDA runtime or driver failure            */
#define MUSR_ERR_NVRTC 3    /* theory source failed to compile           */
#define MUSR_ERR_NCCL 4     /* NCCL failure (sharded handles)            */
#define MUSR_ERR_NOMEM 5    /* device or pinned allocation failed        */

#define MUSR_ERR_IO 6       /* muSR data file: see musr_io_error.code     */
#define MUSR_ERR_PEER 7     /* shared results: a peer rank died, closed or timed out */

#define MUSR_KIND_CHI2 0
#define MUSR_KIND_MLH 1

#define MUSR_ROUND_TERMS 256  /* terms per warp round; tiles are 1-8 rounds */

typedef struct musr_ctx musr_ctx;

/* Library version (major*10000 + minor*100 + patch). */
int musr_version(void);

/* Number of visible CUDA devices (0 when none). */
int musr_device_count(int* n);

/* Message of the last failure of a call that had no handle (musr_open*). */
const char* musr_global_error(void);

/* One GPU, no collective. */
int musr_open(int device, musr_ctx** out);

/* Sharded handle: this process is rank `rank` of `world`, each rank owning a
 * disjoint set of datasets; results are combined with one fp64 ncclAllReduce
 * per evaluation, captured in the evaluation's CUDA graph.  `nccl_lib` is the
 * path of libnccl.so.2 (NULL: default dlopen search); `unique_id` is the
 * 128-byte ncclUniqueId made by rank 0 with musr_nccl_unique_id. */
int musr_nccl_unique_id(const char* nccl_lib, unsigned char out_id[128]);
int musr_open_sharded(int device, int rank, int world, const char* nccl_lib,
                      const unsigned char unique_id[128], musr_ctx** out);

/* Multi-GPU without a device collective: rank `rank`
 * of `world` processes on one node, each owning a contiguous shard of the
 * datasets (musr_upload's out_index gives every local dataset its global
 * slot).  `buf` is host memory shared by all ranks' processes (e.g. one
 * /dev/shm mapping, zero-filled, 64-byte aligned, >= 64 * n_global bytes);
 * the library registers it as mapped memory and every rank's objective kernel
 * writes its datasets' results there as epoch-tagged 8-byte words, so each
 * host reads every dataset's result directly -- the per-evaluation exchange
 * rides on the stage-2 stores, no ncclAllReduce and no device sync.  Double-
 * buffered by epoch parity.  `epoch_base` must differ between the handles
 * sharing a buffer (same value on every rank).  The last 8 * world bytes of
 * `buf` hold each rank's process id while it has a handle open: a rank waiting
 * for a peer's results fails with MUSR_ERR_PEER as soon as that peer exited or
 * closed, or after MUSR_PEER_TIMEOUT_S seconds (environment, default 60).
 * Replaces the reference's single-process dataset loop (musr.py:190-201) for
 * sharded runs; values are bitwise identical to one GPU. */
int musr_open_shared(int device, int rank, int world, void* buf, size_t bytes,
                     unsigned long long epoch_base, musr_ctx** out);

/* Host half of the shared-results exchange, exposed for host-only tests: decode
 * n_global datasets' LL words (4 per dataset, (32-bit half << 32) | epoch, as the
 * objective kernel writes them) of evaluation `epoch` and fold them exactly as
 * musr_eval does (musr.py:190-201).  MUSR_ERR_PEER if any word is stale. */
int musr_collect_results(const unsigned long long* words, int n_global, unsigned epoch,
                         double* per_dataset, int64_t* first_bad_bin, double* total);

void musr_close(musr_ctx* ctx);
const char* musr_last_error(const musr_ctx* ctx);

/* Compile the theory fragment produced by codegen.lower() (defines MUSR_NU,
 * musr_uniform, musr_theory) into the objective kernels.  Cached by source
 * hash.  On MUSR_ERR_NVRTC the compiler log is copied into `log`. */
int musr_set_theory(musr_ctx* ctx, const char* fragment, char* log, size_t log_cap);

/* Compile-only check of a theory fragment (no device needed).  Returns the
 * size of the sm_100a CUBIN NVRTC produced; the log as in musr_set_theory. */
int musr_compile_theory(const char* fragment, char* log, size_t log_cap, size_t* cubin_bytes);

/* Upload the local datasets (copied; the device owns them afterwards).
 *   n_global       datasets over all ranks (length of per-dataset outputs)
 *   n_local        datasets owned by this handle
 *   out_index[i]   global index of local dataset i
 *   n_terms[i]     in-range bin count (> 0)
 *   first_bin[i]   first in-range bin; t0_bin[i]; dt[i]
 *   counts[i], errors[i], envelope[i]
 *                  host arrays of n_terms[i] doubles starting at first_bin[i]
 *                  (errors may be NULL: MLH-only handle).  errors[i] must be
 *                  the reference's MusrDataset.errors() = max(1, sqrt(counts))
 *                  (musr.py:95-96): it marks the handle chi2-capable, and the
 *                  device recomputes it bit for bit (correctly rounded sqrt)
 *                  instead of streaming it.
 *   n0_slot[i], nbkg_slot[i]   parameter indices (already wrapped)
 *   maps           n_local * map_stride int32 (per-dataset map rows)
 *   fvals          n_local * f_stride doubles (per-dataset function values)
 *   p_capacity     maximum parameter-vector length accepted by musr_eval */
int musr_upload(musr_ctx* ctx, int n_global, int n_local, const int32_t* out_index,
                const int64_t* n_terms, const int64_t* first_bin, const int64_t* t0_bin,
                const double* dt, const double* const* counts, const double* const* errors,
                const double* const* envelope, const int32_t* n0_slot, const int32_t* nbkg_slot,
                const int32_t* maps, int map_stride, const double* fvals, int f_stride,
                int p_capacity);

/* One synchronous objective evaluation: copy p (n_p <= p_capacity) to pinned
 * staging, replay the CUDA graph (H2D p -> kernel -> [allreduce] -> D2H),
 * wait, then fold.  per_dataset / first_bad_bin have n_global entries
 * (first_bad_bin = -1: none).  total = left fold of per_dataset in global
 * order (may be NULL). */
int musr_eval(musr_ctx* ctx, int kind, const double* p, int n_p, double* per_dataset,
              int64_t* first_bad_bin, double* total);

/* Batched evaluation: n_points parameter vectors,
 * row-major in p (n_points x n_p).  Each tile of the histograms is streamed
 * once per MUSR_KMAX (8) points and evaluated at all of them; larger batches
 * run in chunks.  Outputs are row-major per point: per_dataset and
 * first_bad_bin n_points x n_global, totals n_points.  Every point's values are
 * bit-identical to musr_eval at that point.  Replaces n_points calls of the
 * reference objective (musr.py:181-232) -- e.g. the Nelder-Mead initial
 * simplex and shrink steps (optimize.py:89-96, optimize.py:133-135). */
int musr_eval_batch(musr_ctx* ctx, int kind, const double* p, int n_points, int n_p,
                    double* per_dataset, int64_t* first_bad_bin, double* totals);

/* Datasets of the whole (possibly sharded) problem after musr_upload. */
int musr_n_datasets(const musr_ctx* ctx, int* n_global);

/* Native bounded Nelder-Mead (restates optimize.py:41-146, bitwise-identical
 * iterates) driving musr_eval / musr_eval_batch directly, so a fit does not
 * return to the host language between evaluations.  p_full: the full
 * parameter vector (fixed values); free_idx[n_free]: the optimised slots;
 * x0: the clamped start in free coordinates and f0 its objective value
 * (evaluated by the caller, which raises the reference's errors there);
 * step/lo/hi: per free coordinate; budget: maximum evaluations including the
 * start.  Returns MUSR_OK with best_x[n_free] etc., or MUSR_NM_RAISED when an
 * evaluation hit a reference error (an MLH non-positive model): fail_x[n_free]
 * is that point, for the caller to re-evaluate with the reference semantics.
 * Replaces the minimize -> nelder_mead loop of musr.py:246-296 /
 * optimize.py:41-146 for the built-in objectives. */
#define MUSR_NM_RAISED 100
int musr_minimize(musr_ctx* ctx, int kind, const double* p_full, int n_p, const int32_t* free_idx,
                  int n_free, const double* x0, double f0, const double* step, const double* lo,
                  const double* hi, double tol_f, int64_t budget, int restarts, double* best_x,
                  double* best_f, int64_t* iterations, int64_t* evaluations, int* converged,
                  double* fail_x);

/* The same loop over a caller-supplied objective (tests: checks the native
 * loop against optimize.py without a GPU).  eval(user, xs, k, n, fs) fills
 * fs[0..k) for the k rows of xs; a nonzero return aborts with that status
 * (fail_x = the point). */
typedef int (*musr_nm_eval_fn)(void* user, const double* xs, int k, int n, double* fs);
int musr_nm_run(int n, const double* x0, double f0, const double* step, const double* lo,
                const double* hi, double tol_f, int64_t budget, int restarts, musr_nm_eval_fn eval,
                void* user, double* best_x, double* best_f, int64_t* iterations,
                int64_t* evaluations, int* converged, double* fail_x);

/* Timing helpers (CUDA events on the handle's stream).
 *   mode 0: `iters` back-to-back graph replays (full evaluation incl. H2D p and
 *           D2H results, no host sync in between) -> *ms = total elapsed.
 *   mode 1: `iters` objective-kernel launches, each bracketed by its own
 *           events -> *ms = *kernel_ms = summed kernel time.
 *   mode 2: `iters` graph replays, each bracketed by events -> *ms = summed
 *           evaluation time, *kernel_ms = summed time of the objective kernel
 *           inside those same replays (event nodes captured in the graph).
 *   mode 3: no evaluation -- only the L2 flush below, then a stream sync (the
 *           caller times an end-to-end call right after it).
 *   mode 4: `iters` synchronous evaluations at the last parameter vector
 *           (musr_eval: launch, host waits for every dataset's result -- all
 *           ranks' with shared results -- and folds).  Without a flush one event
 *           pair spans all of them (launches, kernels and host waits); with a
 *           flush each evaluation has its own pair and *ms is their sum.
 *   flush_l2 (modes 1-4): 1 = write 512 MiB before each iteration, outside the
 *   timed interval, so inputs never start L2-resident; 2 = that, then read
 *   256 MiB of it back, so the L2 also holds no dirty lines whose write-back
 *   would land inside the timed interval. */
int musr_time_evals(musr_ctx* ctx, int kind, int iters, int mode, int flush_l2, double* ms,
                    double* kernel_ms);

/* The theory's uniform row as a host program (codegen.py: _UniformProgram;
 * int32 quadruples (op, dst, a, b) and literals), set after musr_set_theory.
 * On the direct path with <= 16 local datasets the library then evaluates every
 * dataset's parameter-only values, rotation tables, N0 and Nbkg on the host per
 * call -- as the reference evaluates them as numpy float64 scalars on the CPU
 * (theory.py:409-464, musr.py:150-162) -- and passes them inline with the launch,
 * so the CTA prologue only copies them.  Optional: without it the prologue
 * computes the rows on the device. */
int musr_set_uniform_program(musr_ctx* ctx, const int32_t* code, int n_words, const double* lits,
                              int n_lits);

/* Tile shape (extension, no reference counterpart): terms per consumer
 * thread (4, 8, 16) and consumer warps per CTA (4, 8, 16); a tile is
 * 32 * cwarps * per_thread terms.  Default 8 x 16 (4096-term tiles, the best
 * for problems that fill the GPU); problems of at most 64 such tiles use 8 x 8
 * (at most 16: 8 x 4) so more SMs share the work (Session picks it).  Must precede musr_set_theory
 * and musr_upload.  The reduction is the same pairwise tree for every shape;
 * with the same per_thread the values are bit-identical (the theory's anchored
 * recurrences restart every per_thread bins). */
int musr_set_tile_shape(musr_ctx* ctx, int per_thread, int cwarps);

/* The rows the host program gives for p ([n_local][row length], test hook). */
int musr_eval_uniform_rows(musr_ctx* ctx, const double* p, int n_p, double* rows);

/* Data format chosen at upload: 0 = f64 (counts + envelope as fp64, 16 B/bin;
 * chi2 computes err and 1/err per bin), 1 = c32 (integral counts < 2^23: fp32
 * counts + fp64 envelope, 12 B/bin, with a {err, 1/err} table of `table_size`
 * (<= 4096) entries in shared memory; larger counts computed per bin). */
int musr_format(const musr_ctx* ctx, int* format, int* table_size);

/* Number of tiles (units of 256*R terms) one evaluation processes here. */
int musr_tiles(const musr_ctx* ctx, int64_t* n_tiles);

/* Developer timeline (handles opened with MUSR_TRACE=1 in the environment):
 * copies 4 %globaltimer stamps per CTA of the last objective launch of `kind`
 * (CTA start, first tile landed, stage-2 done, producer exit; 0 = not reached). */
int musr_debug_trace(musr_ctx* ctx, int kind, uint64_t* out, int cap, int* n_ctas);

/* DFMA throughput probe: returns measured fp64 TFLOP/s (2 flops per DFMA). */
int musr_fp64_peak(int device, double* tflops);

/* ---- muSR data file (fast ingest) --------------------
 * Native, multi-threaded reader / writer of the reference's text format
 * (pkg/src/blk/io.py:109-140 store_musr_data, io.py:143-212 load_musr_data),
 * replacing both.  The reader reproduces load_musr_data's decisions line by
 * line; on failure it reports which error the reference raises first, and
 * where, and the caller formats the reference's message from it
 * (paper_1604_02334_b200/musrio.py). */
#define MUSR_IO_OS 1             /* open/read/write failed; errno in `bin`          */
#define MUSR_IO_MALFORMED 2      /* "{path}:{line}: malformed line: {text!r}"       */
#define MUSR_IO_BEFORE_HEADER 3  /* "{path}:{line}: data before any DETECTOR header" */
#define MUSR_IO_UNKNOWN_KEY 4    /* "{path}:{line}: unknown key {first token!r}"    */
#define MUSR_IO_MISSING 5        /* "{path}: detector {d} is missing {missing}"     */
#define MUSR_IO_NEGATIVE 6       /* "{path}: detector {d} has a negative count at bin {bin}" */
#define MUSR_IO_BAD_MAP 7        /* TheoryError "map entries must be non-negative integers" */
#define MUSR_IO_EMPTY_HIST 8     /* "{path}: detector {d}: empty histogram"         */
#define MUSR_IO_BAD_DT 9         /* "{path}: detector {d}: dt must be positive"     */
#define MUSR_IO_NO_BLOCKS 10     /* "{path}: no detector blocks found"              */
#define MUSR_IO_UNSUPPORTED 11   /* non-ASCII bytes or integers beyond int64: the
                                    caller parses the file with the Python rules   */
typedef struct musr_io_error {
  int code;
  int64_t line;       /* 1-based line of a line error, else -1                     */
  int64_t text_off;   /* byte offset / length of that (stripped) line in the file  */
  int64_t text_len;
  int64_t detector;   /* DETECTOR index of a block error, else -1                  */
  int64_t bin;        /* negative-count bin, or errno for MUSR_IO_OS              */
  char missing[96];   /* MUSR_IO_MISSING: "dt, t0, ..." in the reference's order  */
} musr_io_error;

typedef struct musr_file musr_file;
typedef struct musr_detector_info {
  int64_t index;      /* DETECTOR value                                             */
  double dt;
  int64_t t0_bin, n0_slot, nbkg_slot;
  int64_t n_map, n_func, n_counts;
} musr_detector_info;

/* Parse a muSR data file with `n_threads` threads (<= 0: all cores). */
int musr_file_load(const char* path, int n_threads, musr_file** out, musr_io_error* err);
int musr_file_n_detectors(const musr_file* f);
int musr_file_detector(const musr_file* f, int i, musr_detector_info* info);
/* Copy detector i's map (int64), func (double) and counts (as float64 like
 * MusrDataset.counts, and/or int64); any pointer may be NULL. */
int musr_file_copy(const musr_file* f, int i, int64_t* map, double* func, double* counts_f64,
                   int64_t* counts_i64);
void musr_file_free(musr_file* f);

/* Write a muSR data file: headers[d] is detector d's "DETECTOR ... func ..."
 * text (one '\n'-terminated line per key, formatted like store_musr_data);
 * its counts are truncated to int64 (ndarray.astype) and written 16 per line,
 * detectors separated by an empty line, exactly as store_musr_data. */
int musr_file_store(const char* path, int n_det, const char* const* headers,
                    const double* const* counts, const int64_t* n_counts, int n_threads,
                    musr_io_error* err);

#ifdef __cplusplus
}
#endif
#endif /* MUSR_B200_H */
