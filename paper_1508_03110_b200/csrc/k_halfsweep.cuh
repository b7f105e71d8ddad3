// k_halfsweep.cu -- K1-K4: one ALS half-sweep (als.cpp:40-121,
// parallel.cpp:144-185).  For every destination row c with ratings
// {(j_t, r_t)}:
//      (sum_t m_t m_t^T + lambda*n_c*I) u_c = sum_t r_t m_t ,  m_t = src row j_t
// empty rows -> 0; unregularised or non-SPD systems -> least-norm solve.
//
// Design:
//  * Rows are cut into segments of <= S ratings (SegPlan, heavy rows first).
//    One group of GW warps owns a segment.  Gathered source rows are staged
//    into shared memory with cp.async (16-byte, double-buffered, CH ratings
//    per stage) as the augmented vector m' = [m, r] (rhs folded into the Gram).
//  * Gram of m' on the FP64 tensor cores: mma.sync m8n8k4 f64 (SASS
//    DMMA.8x8x4) over the NB(NB+1)/2 lower-triangular 8x8 blocks, k = 4
//    ratings per MMA; block pairs are distributed round-robin over the warps,
//    accumulators live in registers.
//  * Single-segment rows finish in the same CTA: the Gram goes to shared
//    memory, lambda*n_c is added to the diagonal and an in-place symmetric
//    elimination (LDL^T form of Cholesky: a pivot <= 0 means "not SPD", as
//    Eigen's LLT) runs on the augmented matrix, so the forward substitution
//    falls out of the rhs row; one warp back-substitutes.
//  * Multi-segment (heavy) rows write register partials per segment; a
//    second kernel sums them in segment order (deterministic) and solves.
//  * Fallback columns (lambda*n_c == 0 or a non-positive pivot) are listed
//    and solved by k_hs_fallback: exact reference-order Gram, cyclic Jacobi
//    eigen-decomposition, pseudo-inverse solve + one refinement step
//    (als.cpp:71-81 semantics).
//
// k_halfsweep.cuh: argument blocks shared by the per-rank instantiation units
// (k_hs_inst.cu, compiled once per 8x8 block count NB) and the dispatcher
// (k_halfsweep.cu: NB switch + least-norm fallback).
#pragma once

#include "common.cuh"

namespace ab2 {
namespace hs {

struct HsArgs {
  const int64_t* ptr;
  const int* idx;
  const double* val;
  int row0;            // flat-vector row of local row 0 (output side)
  const double* src;   // flat-vector row 0 of the source side
  double* out;         // flat vector base (rows indexed by row0 + local row)
  int n_f, ld;
  double lambda;
  const int* seg_row;
  const int64_t* seg_beg;
  const int* seg_len;
  const int* seg_slot;
  int n_seg;
  const int* m_row;
  const int* m_slot0;
  const int* m_nslot;
  int n_multi;
  double* partial;
  int* fb_list;
  unsigned* fb_count;
  unsigned* fb_total;
};

struct SolveArgs {
  int row0;     // first local row of the batch
  int nrows;    // rows in the batch
  const int* row_slot0;
  const int* row_nslot;
  const double* G;
};

// Gram + solve of one half-sweep for 8*NB-1 >= ld; defined in k_hs_inst.cu
// (one translation unit per NB so the heavy template bodies build in parallel).
template <int NB>
void run_hs(Ctx* ctx, DevRatings& R, int kind, HsArgs& a, int S);

}  // namespace hs
}  // namespace ab2
