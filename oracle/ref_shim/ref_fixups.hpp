// SPDX-License-Identifier: Apache-2.0
//
// TEST INFRASTRUCTURE ONLY -- force-included (-include) when oracle/Makefile compiles the
// reference's proj/src/attention.cpp, so that file builds UNMODIFIED. It supplies the two
// names AttentionLayer::backward uses but the reference never declares (SURVEY.md section 0:
// "attention.cpp:152,180-183,194 are hard compile errors"), with the intended math:
//
//  * attention.cpp:152 stores, and :194 adds, the gate path's d(xq) in
//    `dout_pre_gate_gate_dxq_`, which is not a member of AttentionLayer (attention.hpp:51-73).
//    Unqualified lookup from the const member function falls through to namespace
//    rankformer, where this per-thread scratch matrix lives (per thread: the reference's
//    forward/backward are called concurrently on shared const layers, params.hpp:12-14).
//
//  * attention.cpp:180-183 call a 5-argument rmsnorm_backward(dy, cache, gain_row,
//    dgain_matrix, head): the QKNorm gains are a [heads, head_dim] parameter
//    (attention.cpp:43-44) and head i's gain gradient belongs in row i. norm.hpp:32 only
//    defines the 4-argument form (which accumulates into row 0). The overload below runs that
//    4-argument form on a 1-row scratch and adds the result into row `row`.
#pragma once

#include "rankformer/norm.hpp"

namespace rankformer {

inline thread_local Mat dout_pre_gate_gate_dxq_;

inline Mat rmsnorm_backward(const Mat& dy, const RmsNormCache& cache, const Mat& gain, Mat& dgain, int row) {
  Mat dg = Mat::Zero(1, gain.cols());
  Mat dx = rmsnorm_backward(dy, cache, gain, dg);
  dgain.row(row) += dg.row(0);
  return dx;
}

}  // namespace rankformer
