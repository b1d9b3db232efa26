// =====================================================================================================
// TurboReg hot-path kernels for sm_100a (B200).  Included once, by turboreg_runtime.cu.
//
// Every kernel takes a batch of independent registration pairs (grid.y / grid.z = pair) and reads its
// pair's geometry from a PairDesc.  Data layout per pair:
//   src4/dst4  float4[n]          correspondences (x, y, z, 0)
//   bits       uint32[n][W]       rows of C(τ); bit c of word c/32 = C_rc; W = ceil(n/32) rounded up to 4
//   edges      uint32[E]          compact CSR of the O2 rows: row i's upper edges (j > i) in increasing j at
//                                 rowptr[i]: (j << 16) | Ĝ_ij   ("rank-indexed" O2 weights, Def. 2)
//   rowptr     int32[n+1]         exclusive scan of the upper degrees
//   deg        int32[n]           upper degree of row i
//   piv        int4[K1]           (i, j, Ĝ_ij, 0) in (Ĝ desc, i asc, j asc) order (lexicographic when more
//                                 than PIV_CAP edges reach the cut weight)
//   cliq       int4[K1*K2]        (i, j, z, S) per slot pivot*K2 + r; empty (-1,-1,-1,0)
//   hyp        float[K1*K2][16]   R[9], t[3], count, flag, S, 0
// Float32 arithmetic that decides an integer is bit-identical to the oracle's: the inlier test uses explicit
// _rn intrinsics in the reading-r13 FMA tree; Eq. 1 edges come from a certified square-root-free filter whose
// decisions provably equal the oracle's float32 tree, with that exact tree (r1) evaluated for
// every test the filter cannot certify.
// =====================================================================================================
#pragma once
// Stage headers (each includes the previous one, so definitions keep their order):
//   turboreg_common.cuh  types, workspace views, warp helpers
//   turboreg_compat.cuh  a1 ingest, a2 compat
//   turboreg_sc2.cuh     a3 degrees, heavy/sparse split, SC^2 assembly
//   turboreg_select.cuh  a4 pivots
//   turboreg_pgs.cuh     a5 PGS, SC^2-mode canonical list
//   turboreg_model.cuh   a6 Kabsch, a7 scoring, a8 argmax
//   turboreg_rank.cuh    optional outputs: per-row SC^2 sums r_i, the ranked hypothesis list
#include "turboreg_rank.cuh"
