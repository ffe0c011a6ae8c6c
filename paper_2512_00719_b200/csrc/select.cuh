// select.cuh — exact radix selection on unique 64-bit composite keys
// (value desc, position asc), the tie rule of _top_k_ids (filtering.py:38-58).
//
// Keys are unique (they embed the position), so "the `need` largest keys" is
// a well-defined set and a most-significant-digit radix walk finds the cut in
// at most 8 rounds of 8-bit digits, usually 2-4 because the walk stops as soon
// as a whole digit bucket is selected.
#pragma once

#include "common.cuh"

namespace dp {

// Per-digit descending search over a 256-bin histogram, done by one warp.
// Lane l owns bins 255-8l .. 248-8l.  Returns (digit, count strictly above
// digit, count in digit) for the bucket where the running count reaches need.
struct DigitHit {
  uint32_t digit, above, inbin;
};
DP_DEV DigitHit warp_find_digit(const uint32_t* hist, uint32_t need) {
  const uint32_t lane = lane_id();
  uint32_t c[8], s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    c[j] = hist[255 - 8 * lane - j];
    s += c[j];
  }
  const uint32_t incl = warp_incl_scan(s);
  const uint32_t excl = incl - s;
  const uint32_t hit = __ballot_sync(0xffffffffu, excl < need && need <= incl);
  const int L = __ffs(hit) - 1;
  uint32_t d = 0, above = 0, inbin = 0;
  if ((int)lane == L) {
    uint32_t acc = excl;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (inbin == 0 && acc + c[j] >= need) {
        d = 255 - 8 * lane - j;
        above = acc;
        inbin = c[j];
      }
      acc += c[j];
    }
  }
  DigitHit r;
  r.digit = __shfl_sync(0xffffffffu, d, L);
  r.above = __shfl_sync(0xffffffffu, above, L);
  r.inbin = __shfl_sync(0xffffffffu, inbin, L);
  return r;
}

// Warp-level: threshold t such that exactly min(cnt, need) keys of buf[0,cnt)
// are >= t.  hist: 256 u32 of warp-private shared memory.
DP_DEV uint64_t warp_select_threshold(const uint64_t* buf, uint32_t cnt, uint32_t need,
                                      uint32_t* hist) {
  if (cnt <= need || need == 0) return need == 0 ? ~0ull : 0ull;
  const uint32_t lane = lane_id();
  uint64_t prefix = 0, mask = 0;
  for (int shift = 56; shift >= 0; shift -= 8) {
#pragma unroll
    for (int i = 0; i < 8; ++i) hist[lane + 32 * i] = 0u;
    __syncwarp();
    for (uint32_t i = lane; i < cnt; i += 32) {
      const uint64_t k = buf[i];
      if ((k & mask) == prefix) atomicAdd(&hist[(uint32_t)(k >> shift) & 255u], 1u);
    }
    __syncwarp();
    const DigitHit h = warp_find_digit(hist, need);
    prefix |= (uint64_t)h.digit << shift;
    mask |= 255ull << shift;
    need -= h.above;
    __syncwarp();
    if (h.inbin == need) break;
  }
  return prefix;
}

// Warp-level: the r-th largest (1-based) of n u32 keys (duplicates allowed),
// or a value t below it with exactly r keys >= t (the walk stops once a whole
// digit bucket is taken).  Either way at least r keys are >= the result.
DP_DEV uint32_t warp_kth_u32(const uint32_t* keys, uint32_t n, uint32_t r, uint32_t* hist) {
  if (r == 0u) return 0xFFFFFFFFu;
  if (r > n) return 0u;
  const uint32_t lane = lane_id();
  uint32_t prefix = 0u, mask = 0u, need = r;
  for (int shift = 24; shift >= 0; shift -= 8) {
#pragma unroll
    for (int i = 0; i < 8; ++i) hist[lane + 32 * i] = 0u;
    __syncwarp();
    for (uint32_t i = lane; i < n; i += 32) {
      const uint32_t k = keys[i];
      if ((k & mask) == prefix) atomicAdd(&hist[(k >> shift) & 255u], 1u);
    }
    __syncwarp();
    const DigitHit h = warp_find_digit(hist, need);
    prefix |= h.digit << shift;
    mask |= 255u << shift;
    need -= h.above;
    __syncwarp();
    if (h.inbin == need) break;
  }
  return prefix;
}

// In-place stable compaction of buf[0,cnt) keeping keys >= t; returns new count.
DP_DEV uint32_t warp_compact(uint64_t* buf, uint32_t cnt, uint64_t t) {
  const uint32_t lane = lane_id();
  uint32_t out = 0;
  for (uint32_t base = 0; base < cnt; base += 32) {
    const uint32_t i = base + lane;
    const uint64_t k = i < cnt ? buf[i] : 0ull;
    const bool keep = i < cnt && k >= t;
    const uint32_t m = __ballot_sync(0xffffffffu, keep);
    __syncwarp();
    if (keep) buf[out + __popc(m & lanemask_lt())] = k;
    out += __popc(m);
    __syncwarp();
  }
  return out;
}

// Block-level threshold over an indexed source: get(i, &key) returns false for
// empty slots, i in [0, n_slots).  NT cooperating threads (index t) with
// barrier `sync`; hist: 256 u32 shared; bcast: 4 u32 shared.  Returns the
// threshold to all.
// kvar: the key bits that vary among the candidates (OR ^ AND over them, ~0
// when unknown); a digit with no varying bit is the same for every key, so
// its round is skipped (bf16 values: two of the four value digits are
// constant, and positions < 2^24 leave the top position digit constant).
template <int NT, typename Get, typename Sync>
DP_DEV uint64_t group_select_threshold(Get get, uint32_t n_slots, uint32_t cnt, uint32_t need, uint32_t* hist,
                                       uint32_t* bcast, uint32_t t, Sync sync, uint64_t kvar = ~0ull,
                                       uint64_t kconst = 0ull) {
  if (cnt <= need || need == 0) return need == 0 ? ~0ull : 0ull;
  uint64_t prefix = 0, mask = 0;
  for (int shift = 56; shift >= 0; shift -= 8) {
    if (((kvar >> shift) & 255ull) == 0ull) {
      prefix |= kconst & (255ull << shift);
      mask |= 255ull << shift;
      continue;
    }
    for (uint32_t i = t; i < 256; i += NT) hist[i] = 0u;
    sync();
    for (uint32_t i = t; i < n_slots; i += NT) {
      uint64_t k;
      if (get(i, k) && (k & mask) == prefix) atomicAdd(&hist[(uint32_t)(k >> shift) & 255u], 1u);
    }
    sync();
    if (t < 32) {
      const DigitHit h = warp_find_digit(hist, need);
      if (t == 0) {
        bcast[0] = h.digit;
        bcast[1] = h.above;
        bcast[2] = h.inbin;
      }
    }
    sync();
    const uint32_t d = bcast[0], above = bcast[1], inbin = bcast[2];
    prefix |= (uint64_t)d << shift;
    mask |= 255ull << shift;
    need -= above;
    sync();
    if (inbin == need) break;
  }
  return prefix;
}

template <int NT, typename Get>
DP_DEV uint64_t block_select_threshold(Get get, uint32_t n_slots, uint32_t cnt, uint32_t need, uint32_t* hist,
                                       uint32_t* bcast, uint64_t kvar = ~0ull, uint64_t kconst = 0ull) {
  return group_select_threshold<NT>(get, n_slots, cnt, need, hist, bcast, threadIdx.x, [] { __syncthreads(); }, kvar,
                                    kconst);
}

// The valid keys of an indexed candidate source, compacted (any order) into
// dense[0, dcap) — the candidates' spare shared memory — with their count
// and the OR / AND of the keys (constant-digit skipping above).  Every
// later select round then reads n_valid dense keys instead of re-decoding
// every element slot of the admitted vectors.  NT threads, index t; all of
// them call it (warp ballots).  Returns the count; keys past dcap are not
// stored (the caller then keeps the indexed source).
struct DenseStats {
  uint32_t n;
  uint64_t kor, kand;
};
template <int NT, typename Get, typename Sync>
DP_DEV DenseStats group_compact_valid(Get get, uint32_t n_slots, uint64_t* dense, uint32_t dcap, uint32_t* counter,
                                      unsigned long long* kor_s, unsigned long long* kand_s, uint32_t t, Sync sync) {
  const uint32_t lane = t & 31u;
  if (t == 0) {
    *counter = 0u;
    *kor_s = 0ull;
    *kand_s = ~0ull;
  }
  sync();
  uint64_t o = 0ull, an = ~0ull;
  for (uint32_t b0 = 0; b0 < n_slots; b0 += NT) {
    const uint32_t i = b0 + t;
    uint64_t kk = 0ull;
    const bool v = i < n_slots && get(i, kk);
    const uint32_t m = __ballot_sync(0xffffffffu, v);
    uint32_t base = 0u;
    if (lane == 0 && m) base = atomicAdd(counter, (uint32_t)__popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (v) {
      const uint32_t s = base + (uint32_t)__popc(m & lanemask_lt());
      if (s < dcap) dense[s] = kk;
      o |= kk;
      an &= kk;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    o |= __shfl_xor_sync(0xffffffffu, o, off);
    an &= __shfl_xor_sync(0xffffffffu, an, off);
  }
  if (lane == 0) {
    atomicOr(kor_s, (unsigned long long)o);
    atomicAnd(kand_s, (unsigned long long)an);
  }
  sync();
  DenseStats r;
  r.n = *counter;
  r.kor = *kor_s;
  r.kand = *kand_s;
  sync();
  return r;
}

}  // namespace dp
