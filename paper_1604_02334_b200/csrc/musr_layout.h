// musr_layout.h -- device-side data layout shared by the host runtime
// (musr_b200.cu) and the JIT-compiled kernel (musr_kernel.cuh).  Plain C
// structs, identical layout on host and device.
#ifndef MUSR_LAYOUT_H
#define MUSR_LAYOUT_H

// Parameter vectors up to this length travel inside the kernel parameters
// (no H2D copy per evaluation); longer ones use the device buffer `P`.
#define MUSR_P_INLINE 64
// Small problems (<= MUSR_H_INLINE datasets, short map / f rows) also carry
// their per-dataset metadata, maps and function values inline, so the CTA
// prologue reads only kernel-parameter space (no dependent global loads).
#define MUSR_H_INLINE 16
#define MUSR_M_INLINE 12
#define MUSR_F_INLINE 4
// Uniform rows computed on the host (musr_set_uniform_program): up to this many
// doubles (n_local * row length) travel inline in place of pin / min / fin, and
// the CTA prologue only copies them (no dependent loads, no per-CTA arithmetic).
#define MUSR_R_INLINE 320
// Batched evaluation (musr_eval_batch): parameter vectors per objective launch.
#define MUSR_KMAX 8

struct MusrHist {
  long long n_terms;    // in-range bins
  long long first_rel;  // first_bin - t0_bin
  long long first_bin;  // absolute first in-range bin (MLH error report)
  double dt;            // bin width (us)
  int tile_start;       // first tile of this dataset
  int n_tiles;
  int n0_slot;          // index of N0 in P (already wrapped like numpy)
  int nbkg_slot;
  int out_index;        // dataset index in the global (all-rank) order
  int map_off;          // offset of this histogram's map row in maps[]
  int f_off;            // offset of this histogram's f row in fvals[]
  int pad_;
};

struct MusrArgs {
  const void* d;              // counts, packed tiles (fp64, or fp32 in the c32 format)
  const double* env;          // exp(-t / tau_mu), packed tiles
  const double2* table;       // c32 chi2: {max(1, sqrt(k)), 1 / that} for k < table_size
  const int* tile_hist;       // tile -> local histogram
  const MusrHist* hist;       // [n_local]
  const double* P;            // parameter vector
  const int* maps;            // map rows
  const double* fvals;        // function-value rows
  double* partial;            // [n_points][n_tiles] tile nodes
  unsigned int* count;        // [n_local] tiles finished (self-resetting)
  unsigned long long* bad;    // [n_points][n_local] first non-positive bin (self-resetting)
  double* out;                // [n_points][2 * n_global]: sums | (bad bin + 1), 0 = none
  double* utab;               // [n_points][n_local][MUSR_NU + 2] uniform values, N0, Nbkg
  int n_global;               // datasets over all ranks
  int n_local;                // datasets on this device
  int n_tiles;                // tiles on this device
  int table_size;             // entries of `table` (c32 format)
  unsigned long long* trace;  // MUSR_TRACE builds: per-CTA %globaltimer stamps
  unsigned int* sched;        // [2] dynamic tile scheduler: next tile (self-resetting), spare
  // Direct path: results go to mapped host memory as "LL" words -- each
  // 32-bit half of a result travels with the evaluation's 32-bit epoch in one
  // 8-byte store ((half << 32) | epoch), so the host knows a word is current
  // without any fence or completion flag.  [n_global][4]: sum hi, lo, bad hi, lo.
  unsigned long long* ll;
  unsigned long long epoch;   // evaluation sequence number (direct path), 0 = write `out`
  int n_points;               // parameter vectors in this launch (1, or <= MUSR_KMAX batched)
  int p_stride;               // batched: P holds n_points rows of p_stride doubles
  int p_inline;               // 1: parameters are in `pin` (kernel parameter space)
  int h_inline;               // 1: hin/min/fin hold all datasets' metadata
  int stages;                 // TMA pipeline depth of this launch (<= MUSR_STAGES)
  int r_inline;               // 1: `rin` holds every local dataset's uniform row (host-computed)
  // Small-problem metadata inline in the kernel parameters: they arrive with
  // the launch, so the CTA prologue issues no dependent global/constant misses.
  MusrHist hin[MUSR_H_INLINE];
  union {
    struct {                  // rows computed in the CTA prologue from p, maps, f values
      double pin[MUSR_P_INLINE];  // inline parameter vector (direct-launch path)
      int min[MUSR_H_INLINE][MUSR_M_INLINE];
      double fin[MUSR_H_INLINE][MUSR_F_INLINE];
    } dev;
    double rin[MUSR_R_INLINE];    // r_inline: [n_local][MUSR_NU + 2] rows from the host
  } u;
};

#endif  // MUSR_LAYOUT_H
