// SPDX-License-Identifier: Apache-2.0
// Host-side structural planner: sequence layout, per-layer retained rows, the
// compact row-interval mask and the attention kernel's 128x128 tile lists.
// All integer rules restate the reference (file:line in plan.cpp).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/sort_b200.h"

namespace sortk {

struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct RuntimeFailure : std::runtime_error {
  using std::runtime_error::runtime_error;
};

constexpr int kAttnTile = 128;

struct LayerPlan {
  int l_q = 0, l_kv = 0;
  bool q_identity = false;  // query rows == all kv rows, in order
  std::vector<int32_t> query_rows, lo, hi, self_idx;
  std::vector<int32_t> roles_kv, pos_kv, pos_q;
  int64_t visible = 0;
  // attention tile lists (q-tiles of kAttnTile rows x kv-tiles of kAttnTile cols)
  int n_qtiles = 0;
  std::vector<int32_t> tile_off;    // [n_qtiles + 1]
  std::vector<int32_t> tile_code;   // pairs {kv_tile, chunk classes}: for row quarter q and
                                    // 32-column chunk c, bit 2(4q+c) = fully visible to every
                                    // valid row, bit 2(4q+c)+1 = visible to none
  std::vector<int32_t> qtile_order; // q-tiles, heaviest first
  int64_t tiles_issued = 0, tiles_total = 0;
};

struct Plan {
  int L0 = 0, prefix = 0;
  std::vector<int32_t> roles0, pos0, cand_index0;
  std::vector<LayerPlan> layers;
  int max_pos = 0;
};

int time_bucket_int(int64_t delta, int n_buckets);
std::vector<int32_t> geometric_schedule(int prefix_len, int depth, int target);
std::vector<int32_t> retained_rows(const std::vector<int32_t>& roles, int keep, bool keep_specials);
void mask_intervals(int l_q, int l_kv, int window, int full_suffix, const int32_t* roles,
                    const int32_t* pos, const int32_t* query_rows, int32_t* lo, int32_t* hi,
                    int32_t* self_idx);
void build_tiles(LayerPlan& p);
void validate_config(const SortConfig& c);
Plan make_plan(const SortConfig& c);

}  // namespace sortk
