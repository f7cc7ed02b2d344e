// C++ host API test (include/flexattn_b200.hpp over the C ABI), mirroring the reference's
// own C++ tests: BlockMask structure (test_block_mask.cpp:40-92) bit-exact vs the oracle port,
// forward/backward vs the oracle (SURVEY.md §8d tolerances), error taxonomy (errors.hpp).
// Built by tests/test_cpp_api.py; runs on a GPU box.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "flexattn_b200.hpp"
#include "flex_oracle.h"

using namespace flexattn;

static int failures = 0;
#define EXPECT(cond)                                                   \
  do {                                                                 \
    if (!(cond)) {                                                     \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                      \
    }                                                                  \
  } while (0)

static std::vector<float> to_host_f32(const DeviceTensor4& t) {
  std::vector<float> out(static_cast<size_t>(t.size()));
  if (t.dtype == DType::F32) {
    check_cuda(cudaMemcpy(out.data(), t.buf.get(), out.size() * 4, cudaMemcpyDeviceToHost), "d2h");
  } else {
    std::vector<uint16_t> raw(out.size());
    check_cuda(cudaMemcpy(raw.data(), t.buf.get(), raw.size() * 2, cudaMemcpyDeviceToHost), "d2h");
    for (size_t i = 0; i < raw.size(); ++i) {
      uint32_t u = static_cast<uint32_t>(raw[i]) << 16;
      std::memcpy(&out[i], &u, 4);
    }
  }
  return out;
}

int main() {
  // ---- BlockMask: causal 256/64 structure and 1024/128 counts -------------------------------
  {
    BlockMask bm = create_block_mask(causal(), 1, 1, 256, 256, 64, 64);
    HostBlockMask h = to_host(bm);
    for (int r = 0; r < 4; ++r) {
      EXPECT(h.full_num[r] == r && h.partial_num[r] == 1 && h.partial_idx[r * 4] == r);
    }
    BlockMask c = create_block_mask(causal(), 1, 1, 1024, 1024);
    HostBlockMask hc = to_host(c);
    long full = 0, part = 0;
    for (auto x : hc.full_num) full += x;
    for (auto x : hc.partial_num) part += x;
    EXPECT(full == 28 && part == 8);
    // bit-exact vs the oracle port, all four kv-side arrays incl. zero tails
    fo_mask om{};
    om.terms = 1;
    std::vector<int64_t> pn(8), pi(64), fn(8), fi(64);
    EXPECT(fo_create_block_mask(&om, 1, 1, 1024, 1024, 128, 128, pn.data(), pi.data(), fn.data(), fi.data()) == 0);
    EXPECT(hc.partial_num == pn && hc.partial_idx == pi && hc.full_num == fn && hc.full_idx == fi);
    // transpose view: q side of causal 1024 is the mirror (column c visits rows >= c)
    BlockMask t = transpose(c);
    HostBlockMask ht = to_host(t);
    EXPECT(ht.full_num[0] == 7 && ht.partial_num[7] == 1);
  }
  // ---- neighbourhood attention + pixel reorderings: the reference's block-count KATs ---------
  // (test_block_mask.cpp:267-309): 32x32 canvas, kernel 5, block size 32 and 16
  {
    const NAGeometry g(32, 32, 5);
    auto computed = [](const BlockMask& bm) {
      HostBlockMask h = to_host(bm);
      long n = 0;
      for (auto x : h.full_num) n += x;
      for (auto x : h.partial_num) n += x;
      return n;
    };
    const i64 n = g.tokens();
    EXPECT(computed(create_block_mask(na_naive(g), 1, 1, n, n, 32, 32)) == 154);
    EXPECT(computed(create_block_mask(remap_mask(na_naive(g), tile_permutation(g, 2)), 1, 1, n, n, 32, 32)) == 184);
    EXPECT(computed(create_block_mask(remap_mask(na_naive(g), morton_permutation(g)), 1, 1, n, n, 32, 32)) == 220);
    EXPECT(computed(create_block_mask(remap_mask(na_naive(g), tile_permutation(g, 2)), 1, 1, n, n, 16, 16)) == 460);
    // or_mask: sliding window OR prefix (bit-exact vs the oracle port)
    BlockMask bo = create_block_mask(or_mask(sliding_window(100), prefix_lm(300)), 1, 1, 1000, 1000, 64, 64);
    HostBlockMask ho = to_host(bo);
    fo_mask om{};
    om.terms = 2;
    om.or_terms = 8;
    om.window = 100;
    om.prefix = 300;
    std::vector<int64_t> pn(16), pi(256), fn(16), fi(256);
    EXPECT(fo_create_block_mask(&om, 1, 1, 1000, 1000, 64, 64, pn.data(), pi.data(), fn.data(), fi.data()) == 0);
    EXPECT(ho.partial_num == pn && ho.partial_idx == pi && ho.full_num == fn && ho.full_idx == fi);
    bool threw = false;
    try {
      NAGeometry bad(8, 8, 4);
    } catch (const GeometryMismatch&) {
      threw = true;
    }
    EXPECT(threw);
  }
  // ---- forward + backward vs the oracle, sliding window + ALiBi, bf16 tcgen05 path ----------
  {
    const i64 B = 1, H = 2, L = 384, D = 128;
    DeviceTensor4 q = random_tensor(11, B, H, L, D), k = random_tensor(12, B, H, L, D),
                  v = random_tensor(13, B, H, L, D), dout = random_tensor(14, B, H, L, D);
    const auto slopes = alibi_slopes(H);
    ScoreMod s = alibi(slopes);
    BlockMask bm = create_block_mask(sliding_window(200), 1, 1, L, L);
    AttentionOutput fwd = forward(q, k, v, s, bm);
    Gradients g = backward(q, k, v, fwd, dout, s, bm, transpose(bm));
    check_cuda(cudaDeviceSynchronize(), "sync");
    std::vector<float> qf = to_host_f32(q), kf = to_host_f32(k), vf = to_host_f32(v), df = to_host_f32(dout);
    std::vector<float> of = to_host_f32(fwd.out), lse(static_cast<size_t>(B * H * L));
    check_cuda(cudaMemcpy(lse.data(), fwd.lse.get(), lse.size() * 4, cudaMemcpyDeviceToHost), "lse");
    fo_mask om{};
    om.terms = 2;
    om.window = 200;
    om.bound_q = L;
    om.bound_kv = L;
    fo_score os{};
    os.terms = 1;
    os.slopes = slopes.data();
    os.num_slopes = static_cast<int32_t>(H);
    const i64 R = 3;
    std::vector<int64_t> pn(R), pi(R * R), fn(R), fi(R * R);
    fo_create_block_mask(&om, 1, 1, L, L, 128, 128, pn.data(), pi.data(), fn.data(), fi.data());
    fo_bm obm{1, 1, R, R, 128, 128, pn.data(), pi.data(), fn.data(), fi.data()};
    std::vector<float> ro(of.size()), rl(lse.size());
    EXPECT(fo_forward_f32(qf.data(), kf.data(), vf.data(), B, H, H, B, L, L, D, 1.0 / std::sqrt(128.0), 1,
                          &os, &om, &obm, ro.data(), rl.data()) == 0);
    double eo = 0, el = 0;
    for (size_t i = 0; i < ro.size(); ++i) eo = std::fmax(eo, std::fabs(ro[i] - of[i]));
    for (size_t i = 0; i < rl.size(); ++i) el = std::fmax(el, std::fabs(rl[i] - lse[i]));
    EXPECT(eo <= 2e-2 && el <= 2e-2);
    std::vector<int64_t> tpn(R), tpi(R * R), tfn(R), tfi(R * R);
    fo_transpose(1, 1, R, R, pn.data(), pi.data(), fn.data(), fi.data(), tpn.data(), tpi.data(), tfn.data(), tfi.data());
    fo_bm obt{1, 1, R, R, 128, 128, tpn.data(), tpi.data(), tfn.data(), tfi.data()};
    std::vector<float> rdq(qf.size()), rdk(kf.size()), rdv(vf.size());
    EXPECT(fo_backward_f32(qf.data(), kf.data(), vf.data(), of.data(), lse.data(), df.data(), B, H, H, B, L, L, D,
                           1.0 / std::sqrt(128.0), 1, &os, &om, &obm, &obt, rdq.data(), rdk.data(), rdv.data()) == 0);
    auto rel = [](const std::vector<float>& got, const std::vector<float>& want) {
      double m = 0, w = 0;
      for (size_t i = 0; i < got.size(); ++i) {
        m = std::fmax(m, std::fabs(got[i] - want[i]));
        w = std::fmax(w, std::fabs(want[i]));
      }
      return m / std::fmax(1.0, w);
    };
    EXPECT(rel(to_host_f32(g.dq), rdq) <= 2e-2);
    EXPECT(rel(to_host_f32(g.dk), rdk) <= 2e-2);
    EXPECT(rel(to_host_f32(g.dv), rdv) <= 2e-2);
    std::printf("forward max|dO| %.3g lse %.3g\n", eo, el);
  }
  // ---- error taxonomy ---------------------------------------------------------------------------
  {
    bool thrown = false;
    try { sliding_window(-1); } catch (const IndexOutOfRange&) { thrown = true; }
    EXPECT(thrown);
    thrown = false;
    try { soft_cap(0.0); } catch (const NonPositiveCap&) { thrown = true; }
    EXPECT(thrown);
    thrown = false;
    try {
      DeviceTensor4 q = random_tensor(1, 1, 2, 256, 128), k = random_tensor(2, 1, 2, 256, 64);
      BlockMask bm = create_block_mask(causal(), 1, 1, 256, 256);
      forward(q, k, k, noop_score(), bm);
    } catch (const ShapeMismatch&) { thrown = true; }
    EXPECT(thrown);
    thrown = false;
    try {
      DeviceTensor4 q = random_tensor(1, 1, 2, 256, 128);
      BlockMask bm = create_block_mask(causal(), 1, 1, 512, 256);
      forward(q, q, q, noop_score(), bm);
    } catch (const BlockMaskMismatch&) { thrown = true; }
    EXPECT(thrown);
  }
  // ---- OpCounters (test_engine.cpp:273-326) -----------------------------------------------------
  {
    const i64 L = 512, D = 64;
    DeviceTensor4 q = random_tensor(701, 1, 1, L, D, DType::F32), k = random_tensor(702, 1, 1, L, D, DType::F32),
                  v = random_tensor(703, 1, 1, L, D, DType::F32);
    OpCounters causal_ops, dense_ops;
    forward(q, k, v, noop_score(), create_block_mask(causal(), 1, 1, L, L), {}, &causal_ops);
    forward(q, k, v, noop_score(), create_block_mask(noop_mask(), 1, 1, L, L), {}, &dense_ops);
    EXPECT(causal_ops.mask_evals == 4ull * 128 * 128);
    EXPECT(dense_ops.mask_evals == 0);
    EXPECT(causal_ops.score_evals == std::uint64_t(L) * (L + 1) / 2);
    EXPECT(dense_ops.score_evals == std::uint64_t(L) * L);
    const double ratio = double(causal_ops.madds) / double(dense_ops.madds);
    EXPECT(ratio > 0.40 && ratio <= 0.60);
  }
  // ---- validation: NonFiniteInput, deterministic backward ------------------------------------------
  {
    DeviceTensor4 q = random_tensor(11, 1, 2, 256, 128), k = random_tensor(12, 1, 2, 256, 128);
    BlockMask bm = create_block_mask(causal(), 1, 1, 256, 256);
    const uint16_t nan_bf16 = 0x7fc0;
    check_cuda(cudaMemcpy(k.buf.as<uint16_t>() + 777, &nan_bf16, 2, cudaMemcpyHostToDevice), "poke");
    AttentionConfig cfg;
    cfg.validate = true;
    bool thrown = false;
    try { forward(q, k, q, noop_score(), bm, cfg); } catch (const NonFiniteInput& e) {
      thrown = std::strstr(e.what(), "k") != nullptr;
    }
    EXPECT(thrown);
    thrown = false;
    try { check_finite({{"q", &q}, {"k", &k}}); } catch (const NonFiniteInput&) { thrown = true; }
    EXPECT(thrown);
    // d_out checked by the backward (engine.cpp:196)
    AttentionOutput f = forward(q, q, q, noop_score(), bm);
    thrown = false;
    try { backward(q, q, q, f, k, noop_score(), bm, bm, cfg); } catch (const NonFiniteInput& e) {
      thrown = std::strstr(e.what(), "d_out") != nullptr;
    }
    EXPECT(thrown);
    AttentionConfig det;
    det.deterministic = true;
    DeviceTensor4 dout = random_tensor(13, 1, 2, 256, 128);
    Gradients g1 = backward(q, q, q, f, dout, noop_score(), bm, bm, det);
    Gradients g2 = backward(q, q, q, f, dout, noop_score(), bm, bm, det);
    const auto a1 = to_host_f32(g1.dq), a2 = to_host_f32(g2.dq);
    EXPECT(std::memcmp(a1.data(), a2.data(), a1.size() * 4) == 0);
  }
  // ---- PagedKVCache + convert_mods: paged decode == unpaged, foreign page -> UnmappedPhysicalIndex
  {
    const i64 B = 2, H = 2, L = 640, D = 128, ps = 128;
    PagedKVCache cache(B, B * (L / ps) + B, ps, H, D);
    cache.shuffle_free_pages(0xFA6E5);
    DeviceTensor4 kl = random_tensor(31, B, H, L, D), vl = random_tensor(32, B, H, L, D);
    for (i64 b = 0; b < B; ++b) {
      DeviceTensor4 kb(1, H, L, D), vb(1, H, L, D);
      const size_t bytes = static_cast<size_t>(H * L * D * 2);
      check_cuda(cudaMemcpy(kb.buf.get(), kl.buf.as<char>() + b * bytes, bytes, cudaMemcpyDeviceToDevice), "slice");
      check_cuda(cudaMemcpy(vb.buf.get(), vl.buf.as<char>() + b * bytes, bytes, cudaMemcpyDeviceToDevice), "slice");
      cache.assign(b, kb, vb);
    }
    EXPECT(cache.seq_len(0) == L && cache.free_pages() == B);
    DeviceTensor4 q = random_tensor(33, B, H, 1, D);
    const i64 off = L - 1;
    BlockMask lbm = create_block_mask(offset_mask(causal(), off), 1, 1, 1, L);
    BlockMask pbm = convert_block_mask(lbm, cache.table());
    ConvertedMods cm = convert_mods(causal(), noop_score(), cache.table());
    AttentionConfig vcfg;
    vcfg.validate = true;
    OpCounters ctr;
    AttentionOutput paged = decode(q, cache, off, cm, pbm, vcfg, &ctr);
    AttentionOutput unpaged = decode(q, kl, vl, off, causal(), noop_score(), lbm);
    const auto p1 = to_host_f32(paged.out), u1 = to_host_f32(unpaged.out);
    EXPECT(std::memcmp(p1.data(), u1.data(), p1.size() * 4) == 0);
    EXPECT(ctr.score_evals == std::uint64_t(B * H * L));          // every cached token is live
    EXPECT(ctr.mask_evals == std::uint64_t(B * H * L));           // all tiles partial (q_len 1)
    // a mask that points batch 1's rows at batch 0's pages: foreign pages
    fa_block_mask bad = pbm.c;
    std::vector<int32_t> idx(static_cast<size_t>(B * pbm.c.cols));
    check_cuda(cudaMemcpy(idx.data(), pbm.c.kv_indices, idx.size() * 4, cudaMemcpyDeviceToHost), "idx");
    std::vector<int32_t> swapped = idx;
    for (i64 c = 0; c < pbm.c.cols; ++c) swapped[static_cast<size_t>(pbm.c.cols + c)] = idx[static_cast<size_t>(c)];
    DeviceBuffer sidx(swapped.size() * 4);
    check_cuda(cudaMemcpy(sidx.get(), swapped.data(), swapped.size() * 4, cudaMemcpyHostToDevice), "idx");
    BlockMask pbad = pbm;
    pbad.c.kv_indices = sidx.as<int32_t>();
    (void)bad;
    bool thrown = false;
    try { decode(q, cache, off, cm, pbad, vcfg); } catch (const UnmappedPhysicalIndex&) { thrown = true; }
    EXPECT(thrown);
    thrown = false;
    try {
      PagedKVCache small(1, 2, ps, H, D);
      DeviceTensor4 big(1, H, 3 * ps, D);
      small.assign(0, big, big);
    } catch (const OutOfPages&) { thrown = true; }
    EXPECT(thrown);
    // batched device-side appends: one token for each sequence, no host sync, then status()
    {
      PagedKVCache pool(3, 6, 4, 1, 8);
      const int32_t ids[3] = {2, 0, 1}, nt[3] = {5, 4, 13};
      DeviceBuffer dids(12), dnt(12);
      check_cuda(cudaMemcpy(dids.get(), ids, 12, cudaMemcpyHostToDevice), "ids");
      check_cuda(cudaMemcpy(dnt.get(), nt, 12, cudaMemcpyHostToDevice), "nt");
      pool.update_batch(FA_PAGE_APPEND, dids.as<int32_t>(), dnt.as<int32_t>(), 3, nullptr, nullptr, false);
      // 2 + 1 of 6 pages fit; the third request needs 4 of the 3 left: status() raises it
      thrown = false;
      try { pool.status(); } catch (const OutOfPages&) { thrown = true; }
      EXPECT(thrown);
      EXPECT(pool.seq_len(2) == 5 && pool.seq_len(0) == 4 && pool.seq_len(1) == 0);
      thrown = false;
      try { pool.update_batch(FA_PAGE_APPEND, dids.as<int32_t>(), dnt.as<int32_t>(), 3, nullptr, nullptr); }
      catch (const OutOfPages&) { thrown = true; }
      EXPECT(thrown);
      EXPECT(pool.seq_len(2) == 10 && pool.seq_len(0) == 8 && pool.seq_len(1) == 0 && pool.free_pages() == 1);
    }
    std::printf("paged decode == unpaged; counters score_evals %llu\n",
                static_cast<unsigned long long>(ctr.score_evals));
  }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
