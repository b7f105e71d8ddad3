// k_halfsweep.cu -- K1-K4: one ALS half-sweep (als.cpp:40-121,
// parallel.cpp:144-185).  For every destination row c with ratings
// {(j_t, r_t)}:
//      (sum_t m_t m_t^T + lambda*n_c*I) u_c = sum_t r_t m_t ,  m_t = src row j_t
// empty rows -> 0; unregularised or non-SPD systems -> least-norm solve.
//
// Design (K1-K4):
//  * Rows are cut into segments of <= S ratings (heavy rows first); the
//    Gram of the augmented vector m' = [m, r] (rhs folded in) is accumulated
//    on the FP64 tensor cores (mma.sync m8n8k4 f64, SASS DMMA.8x8x4) over the
//    NB(NB+1)/2 lower-triangular 8x8 blocks.
//  * Small ranks (NB <= 4): k_hs_main, one warp per segment -- cp.async
//    staging, DMMA Gram, then the shifted symmetric elimination in shared
//    memory (LDL^T; a pivot <= 0 means "not SPD", as Eigen's LLT); heavy rows
//    write per-segment partials that k_hs_reduce sums in order and solves.
//  * Larger ranks (split path): k_hs_gram_ws (persistent, warp-specialised:
//    a TMA producer warp feeds a ring of stages, consumer warps own fixed
//    block ranges) writes one partial Gram slot per segment;
//    k_hs_slot_reduce folds heavy rows' slots in slot order; k_hs_solve_ws
//    (persistent, one CTA per SM, teams of four warps split by SM
//    sub-partition: a pivot warp inverts the 8x8 diagonal blocks and runs the
//    back substitution, three DMMA warps do the block TRSM and trailing
//    updates) solves each column.  NB > 20 uses the non-persistent k_hs_gram.
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
