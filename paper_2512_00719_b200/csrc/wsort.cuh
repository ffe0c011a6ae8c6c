// wsort.cuh — register-resident warp sorting networks for the per-row final
// stage: sorted top-64 of a candidate stream with one warp and no shared
// memory traffic inside the network (bitonic sort of 64 = 21 compare-exchange
// stages, bitonic merge of two sorted 64-lists = 1 + 6 stages).
//
// Items are (key desc, pos asc) pairs — the canonical (value desc, index asc)
// order of filtering.py:83 once `key` is an order-preserving value key.  A
// list of 64 lives two per lane: rank r sits in lane r % 32, register r / 32.
#pragma once

#include "common.cuh"

namespace dp {

struct Item {
  uint64_t k;
  uint32_t p;
};

DP_DEV Item item_worst() { return Item{0ull, 0xFFFFFFFFu}; }
DP_DEV bool item_before(const Item& a, const Item& b) { return a.k > b.k || (a.k == b.k && a.p < b.p); }
DP_DEV Item item_shfl_xor(const Item& x, int m) {
  Item r;
  r.k = __shfl_xor_sync(0xffffffffu, x.k, m);
  r.p = __shfl_xor_sync(0xffffffffu, x.p, m);
  return r;
}
DP_DEV Item item_shfl(const Item& x, int src) {
  Item r;
  r.k = __shfl_sync(0xffffffffu, x.k, src);
  r.p = __shfl_sync(0xffffffffu, x.p, src);
  return r;
}
// keep the item that belongs at this position: `first` = this position is the
// lower index of the pair, `desc` = the pair is ordered descending
DP_DEV void item_cx(Item& mine, const Item& other, bool first, bool desc) {
  const bool mine_first = item_before(mine, other);
  if (mine_first != (first == desc)) mine = other;
}

// Bitonic merge stages strides 16..1 across lanes (both registers descending).
DP_DEV void warp_merge_lanes_desc(Item& a, Item& b) {
  const uint32_t lane = lane_id();
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) {
    const bool first = (lane & (uint32_t)s) == 0u;
    const Item oa = item_shfl_xor(a, s), ob = item_shfl_xor(b, s);
    item_cx(a, oa, first, true);
    item_cx(b, ob, first, true);
  }
}

// Sort 64 items (a = element lane, b = element 32 + lane) descending.
DP_DEV void warp_sort64_desc(Item& a, Item& b) {
  const uint32_t lane = lane_id();
#pragma unroll 1
  for (int size = 2; size <= 32; size <<= 1) {
    // within-32 stages: element i = lane (a) and 32 + lane (b); the two
    // 32-halves sort in opposite directions so that they form a bitonic 64
    const bool desc_a = (lane & (uint32_t)size) == 0u || size == 32;
    const bool desc_b = size == 32 ? false : desc_a;
#pragma unroll 1
    for (int s = size >> 1; s > 0; s >>= 1) {
      const bool first = (lane & (uint32_t)s) == 0u;
      const Item oa = item_shfl_xor(a, s), ob = item_shfl_xor(b, s);
      item_cx(a, oa, first, desc_a);
      item_cx(b, ob, first, desc_b);
    }
  }
  // a: 32 sorted descending, b: 32 sorted ascending -> bitonic 64; stride 32
  // pairs a[lane] with b[lane], then strides 16..1 within each half
  if (item_before(b, a)) {
    const Item t = a;
    a = b;
    b = t;
  }
  warp_merge_lanes_desc(a, b);
}

// (a, b) <- top 64 of two descending lists (a, b) and (c, d), descending.
DP_DEV void warp_merge64_desc(Item& a, Item& b, const Item& c, const Item& d) {
  const uint32_t lane = lane_id();
  // reverse (c, d) to ascending: asc[i] = desc[63 - i]
  const Item ra = item_shfl(d, 31 - (int)lane);   // element lane       <- rank 63 - lane
  const Item rb = item_shfl(c, 31 - (int)lane);   // element 32 + lane  <- rank 31 - lane
  // elementwise max of a descending and an ascending list: a bitonic
  // sequence holding the top 64 of the union
  if (item_before(ra, a)) a = ra;
  if (item_before(rb, b)) b = rb;
  // bitonic merge, descending: stride 32 (register pair), then 16..1
  if (item_before(b, a)) {
    const Item t = a;
    a = b;
    b = t;
  }
  warp_merge_lanes_desc(a, b);
}

}  // namespace dp
