// mods.cuh — mask_mod / score_mod as device functors inlined into the
// templated kernels (the reference's std::function callables,
// modifiers.hpp:17-40, evaluated in double; here fp32 on device).
//
// A mask functor is any type with
//     __device__ bool operator()(int b, int h, int q, int kv) const;
// A score functor is any type with
//     static constexpr bool kIdentity;
//     __device__ float apply(float s, int b, int h, int q, int kv) const;  // s = scaled score
//     __device__ float grad (float s, int b, int h, int q, int kv) const;  // d apply / d s
// The built-in ones below cover the reference mask library
// (mask_library.cpp) and are what the C ABI dispatches to.
#pragma once

#include <limits.h>
#include <stdint.h>

#include "sm100_ptx.cuh"

namespace fa {

struct MaskParams {
  uint32_t terms;
  int32_t hash_density;
  int32_t window;
  int32_t prefix;
  int32_t q_offset;
  int32_t doc_len;
  uint64_t hash_seed;
  const int32_t* doc_ids;
  uint32_t or_terms;       // second AND-group (or_mask)
  int32_t na_w, na_n, na_radius;  // neighbourhood attention canvas (width, tokens, kernel / 2)
  const int32_t* remap;    // slot -> token (remap_mask), or null
  const int32_t* remap_rc; // slot -> (row << 16) | col of its token (remapped na_naive), or null
};

struct ScoreParams {
  uint32_t terms;
  int32_t q_offset;
  float cap;
  float inv_cap;
  const float* slopes;
};

enum : uint32_t {
  kMaskCausal = 1u << 0,
  kMaskSliding = 1u << 1,
  kMaskDocument = 1u << 2,
  kMaskPrefix = 1u << 3,
  kMaskHash = 1u << 4,
  kMaskNever = 1u << 5,
  kMaskNatten = 1u << 6,
};

// Specialised mask kinds the kernels are instantiated for; kMaskDynamic
// evaluates any AND-combination of terms from the runtime bit set.
enum MaskKind : int { kMaskDynamic = 0, kMaskNoop = 1, kMaskCausalOnly = 2, kMaskSlidingOnly = 3,
                      kMaskDocCausal = 4 };

__device__ __forceinline__ bool hash_mask_eval(uint64_t seed, int density, int b, int h, int q,
                                               int kv) {
  // tests/test_support.hpp:16-29
  uint64_t x = seed;
  x ^= 0x9e3779b97f4a7c15ull * static_cast<uint64_t>(b + 1);
  x ^= 0xc2b2ae3d27d4eb4full * static_cast<uint64_t>(h + 1);
  x ^= 0x165667b19e3779f9ull * static_cast<uint64_t>(q + 1);
  x ^= 0x27d4eb2f165667c5ull * static_cast<uint64_t>(kv + 1);
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  x ^= x >> 31;
  return static_cast<int>(x & 0xff) < density;
}

// Bit i of the result = mask(b, h, q, kv0 + i) for i in [0, 32); positions kv >= kv_lim are
// not evaluated (0), so table-backed masks never read past their tables.
template <class MaskT>
__device__ __forceinline__ uint32_t mask_bits32_generic(const MaskT& m, int b, int h, int q, int kv0,
                                                        int kv_lim) {
  uint32_t bits = 0;
#pragma unroll 4
  for (int i = 0; i < 32; ++i)
    if (kv0 + i < kv_lim) bits |= static_cast<uint32_t>(m(b, h, q, kv0 + i)) << i;
  return bits;
}
// Bits set for kv0 + i in [lo, hi] (inclusive), i in [0, 32).
__device__ __forceinline__ uint32_t range_bits32(int kv0, int lo, int hi) {
  const int a = max(lo - kv0, 0), e = min(hi - kv0, 31);
  if (a > e) return 0u;
  const uint32_t upto = (e >= 31) ? 0xffffffffu : ((2u << e) - 1u);
  return upto & ~((1u << a) - 1u);
}

// Bit i = (ids[x0 + i] == doc) for i in [0, 32); vectorised 16-byte loads (the ids of a
// 32-wide chunk are shared by every thread of the warp, so the loads broadcast).
__device__ __forceinline__ uint32_t doc_match_bits32(const int32_t* ids, int len, int x0, int doc) {
  uint32_t bits = 0;
  if (x0 >= 0 && x0 + 32 <= len && (x0 & 3) == 0) {
    const int4* v = reinterpret_cast<const int4*>(ids + x0);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int4 d = __ldg(v + k);
      bits |= (static_cast<uint32_t>(d.x == doc) | (static_cast<uint32_t>(d.y == doc) << 1) |
               (static_cast<uint32_t>(d.z == doc) << 2) | (static_cast<uint32_t>(d.w == doc) << 3))
              << (4 * k);
    }
  } else {
    for (int i = 0; i < 32; ++i)
      if (x0 + i >= 0 && x0 + i < len) bits |= static_cast<uint32_t>(__ldg(ids + x0 + i) == doc) << i;
  }
  return bits;
}

// Tile classes of a mask term over a whole tile (the BlockMask builder's closed forms):
// the AND of terms is the min, the OR of groups the max.
enum : int { kTileNone = 0, kTileMixed = 1, kTileAll = 2 };
// q in [a0, a1], kv in [c0, c1] (inclusive, offsets applied)
__device__ __forceinline__ int tile_causal(int a0, int a1, int c0, int c1) {
  if (a0 >= c1) return kTileAll;
  if (a1 < c0) return kTileNone;
  return kTileMixed;
}
__device__ __forceinline__ int tile_sliding(int a0, int a1, int c0, int c1, int w) {
  if (a1 < c0 || a0 - c1 > w) return kTileNone;  // no q >= kv, or every q - kv > w
  if (a0 >= c1 && a1 - c0 <= w) return kTileAll;
  return kTileMixed;
}
__device__ __forceinline__ int tile_prefix(int a0, int a1, int c0, int c1, int prefix) {
  if (c1 < prefix || a0 >= c1) return kTileAll;
  if (c0 >= prefix && a1 < c0) return kTileNone;
  return kTileMixed;
}
// document ids over q in [a0, a1] and kv in [c0, c1]: all equal -> all; disjoint id ranges ->
// none (warp-collective: every lane passes the same arguments)
__device__ __forceinline__ int tile_document(const int32_t* ids, int a0, int a1, int c0, int c1, int lane) {
  int qmin = INT_MAX, qmax = INT_MIN, kmin = INT_MAX, kmax = INT_MIN;
  for (int i = a0 + lane; i <= a1; i += 32) {
    const int d = __ldg(ids + i);
    qmin = min(qmin, d);
    qmax = max(qmax, d);
  }
  for (int i = c0 + lane; i <= c1; i += 32) {
    const int d = __ldg(ids + i);
    kmin = min(kmin, d);
    kmax = max(kmax, d);
  }
  qmin = __reduce_min_sync(0xffffffffu, qmin);
  qmax = __reduce_max_sync(0xffffffffu, qmax);
  kmin = __reduce_min_sync(0xffffffffu, kmin);
  kmax = __reduce_max_sync(0xffffffffu, kmax);
  if (qmax < kmin || kmax < qmin) return kTileNone;
  if (qmin == qmax && kmin == kmax && qmin == kmin) return kTileAll;
  return kTileMixed;
}
// na_naive: no pair within the radius when the canvas rows (or, for single-row ranges, the
// columns) are farther apart than the radius
__device__ __forceinline__ int tile_natten(int a0, int a1, int c0, int c1, int w, int rad) {
  const int rq0 = a0 / w, rq1 = a1 / w, rk0 = c0 / w, rk1 = c1 / w;
  if (max(0, max(rq0 - rk1, rk0 - rq1)) > rad) return kTileNone;
  if (rq0 == rq1 && rk0 == rk1) {
    const int cq0 = a0 % w, cq1 = a1 % w, ck0 = c0 % w, ck1 = c1 % w;
    if (max(0, max(cq0 - ck1, ck0 - cq1)) > rad) return kTileNone;
  }
  return kTileMixed;
}

// Remapped na_naive from the slot -> (row << 16 | col) table: the Chebyshev distance of the
// two tokens' canvas positions (mask_library.cpp:137-149 after remap_mask :203-215).
__device__ __forceinline__ bool natten_rc(int a, int c, int rad) {
  return max(abs((a >> 16) - (c >> 16)), abs((a & 0xffff) - (c & 0xffff))) <= rad;
}
// bit i = natten_rc(rc[x], rc[y0 + i]) for y0 + i < lim (the other operand fixed)
__device__ __forceinline__ uint32_t natten_rc_bits32(const int32_t* rc, int x, int y0, int lim, int rad) {
  const int a = __ldg(rc + x);
  uint32_t bits = 0;
  if (y0 + 32 <= lim && (y0 & 3) == 0) {
    const int4* v = reinterpret_cast<const int4*>(rc + y0);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int4 c = __ldg(v + k);
      bits |= (static_cast<uint32_t>(natten_rc(a, c.x, rad)) | (static_cast<uint32_t>(natten_rc(a, c.y, rad)) << 1) |
               (static_cast<uint32_t>(natten_rc(a, c.z, rad)) << 2) | (static_cast<uint32_t>(natten_rc(a, c.w, rad)) << 3))
              << (4 * k);
    }
  } else {
    for (int i = 0; i < 32; ++i)
      if (y0 + i < lim) bits |= static_cast<uint32_t>(natten_rc(a, __ldg(rc + y0 + i), rad)) << i;
  }
  return bits;
}
// tile class from the canvas bounding boxes of the tile's q slots [a0, a1] and kv slots
// [c0, c1] (warp-collective)
__device__ __forceinline__ int tile_natten_rc(const int32_t* rc, int a0, int a1, int c0, int c1, int rad, int lane) {
  int qr0 = INT_MAX, qr1 = INT_MIN, qc0 = INT_MAX, qc1 = INT_MIN;
  int kr0 = INT_MAX, kr1 = INT_MIN, kc0 = INT_MAX, kc1 = INT_MIN;
  for (int i = a0 + lane; i <= a1; i += 32) {
    const int v = __ldg(rc + i);
    qr0 = min(qr0, v >> 16); qr1 = max(qr1, v >> 16); qc0 = min(qc0, v & 0xffff); qc1 = max(qc1, v & 0xffff);
  }
  for (int i = c0 + lane; i <= c1; i += 32) {
    const int v = __ldg(rc + i);
    kr0 = min(kr0, v >> 16); kr1 = max(kr1, v >> 16); kc0 = min(kc0, v & 0xffff); kc1 = max(kc1, v & 0xffff);
  }
  qr0 = __reduce_min_sync(0xffffffffu, qr0); qr1 = __reduce_max_sync(0xffffffffu, qr1);
  qc0 = __reduce_min_sync(0xffffffffu, qc0); qc1 = __reduce_max_sync(0xffffffffu, qc1);
  kr0 = __reduce_min_sync(0xffffffffu, kr0); kr1 = __reduce_max_sync(0xffffffffu, kr1);
  kc0 = __reduce_min_sync(0xffffffffu, kc0); kc1 = __reduce_max_sync(0xffffffffu, kc1);
  // no pair is within the radius when the boxes are farther apart along rows or columns
  if (max(qr0 - kr1, kr0 - qr1) > rad || max(qc0 - kc1, kc0 - qc1) > rad) return kTileNone;
  // every pair is within the radius when the farthest corners are
  if (max(qr1 - kr0, kr1 - qr0) <= rad && max(qc1 - kc0, kc1 - qc0) <= rad) return kTileAll;
  return kTileMixed;
}

template <int K>
struct MaskFn {
  MaskParams p;
  // Class of the tile q in [q0, q1), kv in [k0, k1) (non-empty, in bounds): kTileAll /
  // kTileNone when decidable in closed form, else kTileMixed (the builder then evaluates it).
  // Warp-collective (every lane passes the same tile).
  __device__ __forceinline__ int tile_class(int b, int h, int q0, int q1, int k0, int k1, int lane) const {
    (void)b; (void)h;
    const int a0 = q0 + p.q_offset, a1 = q1 - 1 + p.q_offset, c0 = k0, c1 = k1 - 1;
    if constexpr (K == kMaskNoop) {
      return kTileAll;
    } else if constexpr (K == kMaskCausalOnly) {
      return tile_causal(a0, a1, c0, c1);
    } else if constexpr (K == kMaskSlidingOnly) {
      return tile_sliding(a0, a1, c0, c1, p.window);
    } else if constexpr (K == kMaskDocCausal) {
      const int c = tile_causal(a0, a1, c0, c1);
      if (c == kTileNone) return c;
      return min(c, tile_document(p.doc_ids, a0, a1, c0, c1, lane));
    } else {
      if (p.remap != nullptr)
        return p.remap_rc != nullptr ? tile_natten_rc(p.remap_rc, a0, a1, c0, c1, p.na_radius, lane) : kTileMixed;
      int g = group_class(p.terms, a0, a1, c0, c1, lane);
      if (p.or_terms != 0u && g != kTileAll) g = max(g, group_class(p.or_terms, a0, a1, c0, c1, lane));
      return g;
    }
  }
  __device__ __forceinline__ int group_class(uint32_t t, int a0, int a1, int c0, int c1, int lane) const {
    if (t & kMaskNever) return kTileNone;
    int c = kTileAll;
    if (t & kMaskCausal) c = min(c, tile_causal(a0, a1, c0, c1));
    if (t & kMaskSliding) c = min(c, tile_sliding(a0, a1, c0, c1, p.window));
    if (t & kMaskPrefix) c = min(c, tile_prefix(a0, a1, c0, c1, p.prefix));
    if (t & kMaskNatten) c = min(c, tile_natten(a0, a1, c0, c1, p.na_w, p.na_radius));
    if (t & kMaskHash) c = min(c, p.hash_density <= 0 ? kTileNone : (p.hash_density >= 256 ? kTileAll : kTileMixed));
    if ((t & kMaskDocument) && c != kTileNone) c = min(c, tile_document(p.doc_ids, a0, a1, c0, c1, lane));
    return c;
  }
  // kv positions >= kv_lim are reported as 0 (bounds of bound_mask, block_mask.cpp:14-19)
  __device__ __forceinline__ uint32_t bits32(int b, int h, int q, int kv0, int kv_lim) const {
    const int qq = q + p.q_offset;
    if constexpr (K == kMaskNoop) {
      return range_bits32(kv0, INT_MIN / 2, kv_lim - 1);
    } else if constexpr (K == kMaskCausalOnly) {
      return range_bits32(kv0, INT_MIN / 2, min(qq, kv_lim - 1));
    } else if constexpr (K == kMaskSlidingOnly) {
      return range_bits32(kv0, qq - p.window, min(qq, kv_lim - 1));
    } else if constexpr (K == kMaskDocCausal) {
      uint32_t bits = range_bits32(kv0, INT_MIN / 2, min(qq, kv_lim - 1));
      if (bits == 0u) return 0u;
      const int dq = __ldg(p.doc_ids + qq);
      return bits & doc_match_bits32(p.doc_ids, p.doc_len, kv0, dq);
    } else {
      // word-level evaluation of the term groups (one range / vector compare per term); only
      // remapped positions (non-affine) and the per-element terms (natten, hash) fall back
      if (p.remap_rc != nullptr) return natten_rc_bits32(p.remap_rc, qq, kv0, kv_lim, p.na_radius);
      if (p.remap != nullptr) return mask_bits32_generic(*this, b, h, q, kv0, kv_lim);
      const uint32_t in = range_bits32(kv0, INT_MIN / 2, kv_lim - 1);
      uint32_t bits = group_bits32(p.terms, b, h, qq, kv0, in);
      if (p.or_terms != 0u && bits != in) bits |= group_bits32(p.or_terms, b, h, qq, kv0, in & ~bits);
      return bits;
    }
  }
  // na_naive over x0 + i (i in [0, 32)) around pixel c: per canvas row within the radius, one
  // contiguous column range (mask_library.cpp:137-149 is symmetric in q and kv)
  __device__ __forceinline__ uint32_t natten_bits32(int c, int x0) const {
    const int w = p.na_w, rad = p.na_radius;
    const int cr = c / w, cc = c % w;
    const int c_lo = max(cc - rad, 0), c_hi = min(cc + rad, w - 1);
    uint32_t nb = 0u;
    for (int r = max(x0 / w, cr - rad); r <= min((x0 + 31) / w, cr + rad); ++r)
      nb |= range_bits32(x0, r * w + c_lo, r * w + c_hi);
    return nb;
  }
  // AND of the terms in t over kv0 + i (i in [0, 32)) at query position q, within `in`
  __device__ __forceinline__ uint32_t group_bits32(uint32_t t, int b, int h, int q, int kv0, uint32_t in) const {
    uint32_t bits = in;
    if (t & kMaskNever) return 0u;
    if (t & kMaskCausal) bits &= range_bits32(kv0, INT_MIN / 2, q);
    if (t & kMaskSliding) bits &= range_bits32(kv0, q - p.window, q);
    if (t & kMaskPrefix) bits &= range_bits32(kv0, INT_MIN / 2, max(p.prefix - 1, q));
    if ((t & kMaskNatten) && bits != 0u) bits &= natten_bits32(q, kv0);
    if ((t & kMaskDocument) && bits != 0u) bits &= doc_match_bits32(p.doc_ids, p.doc_len, kv0, __ldg(p.doc_ids + q));
    if ((t & kMaskHash) && bits != 0u) {
      for (uint32_t m = bits; m != 0u; m &= m - 1u) {
        const int i = __ffs(m) - 1;
        if (!group(kMaskHash, b, h, q, kv0 + i)) bits &= ~(1u << i);
      }
    }
    return bits;
  }
  // the same over q0 + i at a fixed kv (the backward's view)
  __device__ __forceinline__ uint32_t group_bits32_q(uint32_t t, int b, int h, int q0, int kv, uint32_t in) const {
    uint32_t bits = in;
    if (t & kMaskNever) return 0u;
    if (t & kMaskCausal) bits &= range_bits32(q0, kv, INT_MAX / 2);
    if (t & kMaskSliding) bits &= range_bits32(q0, kv, kv + p.window);
    if ((t & kMaskPrefix) && kv >= p.prefix) bits &= range_bits32(q0, kv, INT_MAX / 2);
    if ((t & kMaskNatten) && bits != 0u) bits &= natten_bits32(kv, q0);  // the window is symmetric
    if ((t & kMaskDocument) && bits != 0u) bits &= doc_match_bits32(p.doc_ids, p.doc_len, q0, __ldg(p.doc_ids + kv));
    if ((t & kMaskHash) && bits != 0u) {
      for (uint32_t m = bits; m != 0u; m &= m - 1u) {
        const int i = __ffs(m) - 1;
        if (!group(kMaskHash, b, h, q0 + i, kv)) bits &= ~(1u << i);
      }
    }
    return bits;
  }
  // Bit i = mask(b, h, q0 + i, kv) for i in [0, 32): the backward's (kv row, q columns) view.
  // q positions >= q_lim are reported as 0 and not evaluated.
  __device__ __forceinline__ uint32_t bits32_q(int b, int h, int q0, int kv, int q_lim) const {
    const int qq0 = q0 + p.q_offset;
    const uint32_t in = range_bits32(q0, INT_MIN / 2, q_lim - 1);
    if constexpr (K == kMaskNoop) {
      return in;
    } else if constexpr (K == kMaskCausalOnly) {
      return in & range_bits32(qq0, kv, INT_MAX / 2);
    } else if constexpr (K == kMaskSlidingOnly) {
      return in & range_bits32(qq0, kv, kv + p.window);
    } else if constexpr (K == kMaskDocCausal) {
      const uint32_t bits = in & range_bits32(qq0, kv, INT_MAX / 2);
      if (bits == 0u) return 0u;
      return bits & doc_match_bits32(p.doc_ids, p.doc_len, qq0, __ldg(p.doc_ids + kv));
    } else {
      if (p.remap_rc != nullptr)  // the window is symmetric: q slots vary at a fixed kv slot
        return q0 >= q_lim ? 0u : natten_rc_bits32(p.remap_rc, kv, qq0, q_lim + p.q_offset, p.na_radius);
      if (p.remap != nullptr) {
        uint32_t bits = 0;
#pragma unroll 4
        for (int i = 0; i < 32; ++i)
          if (q0 + i < q_lim) bits |= static_cast<uint32_t>((*this)(b, h, q0 + i, kv)) << i;
        return bits;
      }
      uint32_t bits = group_bits32_q(p.terms, b, h, qq0, kv, in);
      if (p.or_terms != 0u && bits != in) bits |= group_bits32_q(p.or_terms, b, h, qq0, kv, in & ~bits);
      return bits;
    }
  }
  __device__ __forceinline__ bool operator()(int b, int h, int q, int kv) const {
    const int qq = q + p.q_offset;  // offset_mask, mask_library.cpp:106-110
    if constexpr (K == kMaskNoop) {
      return true;
    } else if constexpr (K == kMaskCausalOnly) {
      return qq >= kv;  // causal, mask_library.cpp:13-15
    } else if constexpr (K == kMaskSlidingOnly) {
      return qq >= kv && qq - kv <= p.window;  // sliding_window, :17-22
    } else if constexpr (K == kMaskDocCausal) {
      // and_mask(document_mask(ids), causal()), :24-34 + :94-98. Index range is
      // validated on the host before launch (the reference throws IndexOutOfRange).
      return qq >= kv && __ldg(p.doc_ids + qq) == __ldg(p.doc_ids + kv);
    } else {
      if (p.remap_rc != nullptr) return natten_rc(__ldg(p.remap_rc + qq), __ldg(p.remap_rc + kv), p.na_radius);
      int qs = qq, ks = kv;
      if (p.remap != nullptr) {  // remap_mask, mask_library.cpp:203-215
        qs = __ldg(p.remap + qq);
        ks = __ldg(p.remap + kv);
      }
      bool ok = group(p.terms, b, h, qs, ks);
      if (p.or_terms != 0u && !ok) ok = group(p.or_terms, b, h, qs, ks);  // or_mask :100-104
      return ok;
    }
  }
  // AND of the primitive terms in t at (already offset / remapped) positions q, kv
  __device__ __forceinline__ bool group(uint32_t t, int b, int h, int q, int kv) const {
    bool ok = true;
    if (t & kMaskNever) ok = false;
    if (t & kMaskCausal) ok = ok && (q >= kv);
    if (t & kMaskSliding) ok = ok && (q >= kv && q - kv <= p.window);
    if (t & kMaskPrefix) ok = ok && (kv < p.prefix || q >= kv);  // prefix_lm :36-41
    if ((t & kMaskNatten) && ok) {  // na_naive, mask_library.cpp:137-149
      const int dr = q / p.na_w - kv / p.na_w, dc = q % p.na_w - kv % p.na_w;
      ok = max(abs(dr), abs(dc)) <= p.na_radius;
    }
    if ((t & kMaskDocument) && ok) ok = __ldg(p.doc_ids + q) == __ldg(p.doc_ids + kv);
    if ((t & kMaskHash) && ok) ok = hash_mask_eval(p.hash_seed, p.hash_density, b, h, q, kv);
    return ok;
  }
};

enum : uint32_t { kScoreAlibi = 1u << 0, kScoreSoftCap = 1u << 1 };

// K is the exact term set: 0 noop, 1 alibi, 2 soft_cap, 3 soft_cap(alibi(s)).
// Precise selects tanhf (fp32 paths) over the MUFU tanh.approx (bf16 paths).
template <int K, bool Precise = false>
struct ScoreFn {
  ScoreParams p;
  static constexpr bool kIdentity = (K == 0);
  static constexpr int kKind = K;
  static constexpr bool kUnitGrad = (K & kScoreSoftCap) == 0;  // d apply / d s == 1
  __device__ __forceinline__ float apply(float s, int b, int h, int q, int kv) const {
    (void)b;
    if constexpr (K & kScoreAlibi) {  // alibi, mask_library.cpp:61-63 (slope of q-head h)
      s = fmaf(__ldg(p.slopes + h), static_cast<float>(q + p.q_offset - kv), s);
    }
    if constexpr (K & kScoreSoftCap) {  // soft_cap, :88
      s = p.cap * (Precise ? tanhf(s * p.inv_cap) : tanh_fast(s * p.inv_cap));
    }
    return s;
  }
  // Row context: log2e * apply(s_raw * scale, b, h, q, kv0 + i) for a fixed (b, h, q, kv0),
  // with every per-row constant hoisted (ALiBi folds into two FFMAs per score).
  struct Row {
    float c;      // multiplier of the raw score
    float base;   // additive term at i = 0 (alibi), pre-scaled
    float step;   // additive change per kv step (alibi), pre-scaled
    float outer;  // soft-cap output multiplier (cap * log2e)
    // the same row context advanced by `off` kv positions (keeps per-score i immediate)
    __device__ __forceinline__ Row shifted(int off) const {
      Row r = *this;
      r.base = fmaf(step, static_cast<float>(off), base);
      return r;
    }
    // log2-domain score and d apply / d s (1 unless soft-capped)
    __device__ __forceinline__ float log2_grad(float s_raw, int i, float& g) const {
      if constexpr (K == 0 || K == 1) {
        g = 1.0f;
        return log2(s_raw, i);
      } else {
        const float u = (K == 2) ? s_raw * c : fmaf(s_raw, c, fmaf(step, static_cast<float>(i), base));
        const float t = Precise ? tanhf(u) : tanh_fast(u);
        g = fmaf(-t, t, 1.0f);
        return outer * t;
      }
    }
    __device__ __forceinline__ float log2(float s_raw, int i) const {
      if constexpr (K == 0) {
        return s_raw * c;
      } else if constexpr (K == 1) {
        return fmaf(s_raw, c, fmaf(step, static_cast<float>(i), base));
      } else if constexpr (K == 2) {
        return outer * (Precise ? tanhf(s_raw * c) : tanh_fast(s_raw * c));
      } else {
        const float t = fmaf(s_raw, c, fmaf(step, static_cast<float>(i), base));
        return outer * (Precise ? tanhf(t) : tanh_fast(t));
      }
    }
  };
  // Column context for the backward's (kv row, q columns) view: the same affine form with q
  // varying (q = q0 + i) at a fixed kv.
  __device__ __forceinline__ Row col(int b, int h, int q0, int kv, float scale) const {
    Row r = row(b, h, q0, kv, scale);
    r.step = -r.step;
    return r;
  }
  __device__ __forceinline__ Row row(int b, int h, int q, int kv0, float scale) const {
    (void)b;
    constexpr float kL2e = 1.4426950408889634f;
    Row r{};
    float slope = 0.f;
    if constexpr ((K & kScoreAlibi) != 0) slope = __ldg(p.slopes + h);
    const float dq = static_cast<float>(q + p.q_offset - kv0);
    if constexpr (K == 0) {
      r.c = scale * kL2e;
    } else if constexpr (K == 1) {
      r.c = scale * kL2e;
      r.base = slope * dq * kL2e;
      r.step = -slope * kL2e;
    } else if constexpr (K == 2) {
      r.c = scale * p.inv_cap;
      r.outer = p.cap * kL2e;
    } else {
      r.c = scale * p.inv_cap;
      r.base = slope * dq * p.inv_cap;
      r.step = -slope * p.inv_cap;
      r.outer = p.cap * kL2e;
    }
    return r;
  }
  // apply() and its derivative in one evaluation (one tanh for soft_cap).
  __device__ __forceinline__ float apply_grad(float s, int b, int h, int q, int kv, float& g) const {
    (void)b;
    if constexpr (K & kScoreAlibi) s = fmaf(__ldg(p.slopes + h), static_cast<float>(q + p.q_offset - kv), s);
    if constexpr (K & kScoreSoftCap) {
      const float t = Precise ? tanhf(s * p.inv_cap) : tanh_fast(s * p.inv_cap);
      g = fmaf(-t, t, 1.0f);
      return p.cap * t;
    } else {
      g = 1.0f;
      return s;
    }
  }
  __device__ __forceinline__ float grad(float s, int b, int h, int q, int kv) const {
    (void)b;
    if constexpr (K & kScoreSoftCap) {  // 1 - tanh^2 (:89-91) through compose (modifiers.hpp:61-65)
      if constexpr (K & kScoreAlibi) {
        s = fmaf(__ldg(p.slopes + h), static_cast<float>(q + p.q_offset - kv), s);
      }
      const float t = Precise ? tanhf(s * p.inv_cap) : tanh_fast(s * p.inv_cap);
      return fmaf(-t, t, 1.0f);
    } else {
      return 1.0f;
    }
  }
};

}  // namespace fa
