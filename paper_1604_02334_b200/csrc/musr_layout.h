// musr_layout.h -- device-side data layout shared by the host runtime
// (musr_b200.cu) and the JIT-compiled kernel (musr_kernel.cuh).  Plain C
// structs, identical layout on host and device.
#ifndef MUSR_LAYOUT_H
#define MUSR_LAYOUT_H

struct MusrHist {
  long long n_terms;    // in-range bins
  long long first_rel;  // first_bin - t0_bin
  long long first_bin;  // absolute first in-range bin (MLH error report)
  double dt;            // bin width (us)
  int tile_start;       // first global tile of this histogram
  int n_tiles;
  int n0_slot;          // index of N0 in P (already wrapped like numpy)
  int nbkg_slot;
  int out_index;        // dataset index in the global (all-rank) order
  int map_off;          // offset of this histogram's map row in maps[]
  int f_off;            // offset of this histogram's f row in fvals[]
  int pad_;
};

struct MusrArgs {
  const double* d;            // counts, packed tiles
  const double* e;            // max(1, sqrt(d)), packed tiles (chi2 only)
  const double* env;          // exp(-t / tau_mu), packed tiles
  const int* tile_hist;       // tile -> local histogram
  const MusrHist* hist;       // [n_local]
  const double* P;            // parameter vector
  const int* maps;            // map rows
  const double* fvals;        // function-value rows
  double* partial;            // [n_tiles] tile nodes
  unsigned int* count;        // [n_local] tiles finished (self-resetting)
  unsigned long long* bad;    // [n_local] first non-positive bin (self-resetting)
  double* out;                // [2 * n_global]: sums | (bad bin + 1), 0 = none
  int n_global;
};

#endif  // MUSR_LAYOUT_H
