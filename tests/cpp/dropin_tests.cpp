// The reference's hot-path test cases (proj/tests/test_fp8.cpp,
// test_codec.cpp, test_collective.cpp, test_dbca.cpp), re-expressed against
// the B200 drop-in headers (include/agq_b200/), i.e. the same agq:: API but
// executing on the GPU through libagq_cuda.so; plus bit-exact comparisons
// with the CPU oracle (oracle/liboracle.so) on random inputs.
// Exit status = number of failed checks.
#include <cmath>
#include <cstdio>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/agq_b200/agq.hpp"
#include "../../oracle/agq_oracle.h"

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                          \
  do {                                                                       \
    ++g_checks;                                                              \
    if (!(cond)) {                                                           \
      ++g_fail;                                                              \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);           \
    }                                                                        \
  } while (0)
template <typename E, typename F>
static bool throws(F&& f, const char* needle = nullptr) {
  try {
    f();
  } catch (const E& e) {
    return !needle || std::string(e.what()).find(needle) != std::string::npos;
  } catch (...) {
    return false;
  }
  return false;
}

using namespace agq;

static std::vector<float> gauss(std::size_t n, std::uint64_t seed, float sd = 1.0f) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<float> g(0.0f, sd);
  std::vector<float> v(n);
  for (auto& x : v) x = g(rng);
  return v;
}
static int bits_for(CodecKind k, int lin) {
  return k == CodecKind::Fp8E4M3 ? 8 : (k == CodecKind::Fp4E2M1 ? 4 : lin);
}
static const CodecKind kKinds[] = {CodecKind::SymmetricLinear, CodecKind::Fp4E2M1,
                                   CodecKind::Fp8E4M3};

static void fp8_scalars() {
  CHECK(fp8_encode(0.0).value.byte == 0x00 && fp8_encode(-0.0).value.byte == 0x80);
  CHECK(fp8_encode(448.0).value.byte == 0x7e && !fp8_encode(448.0).overflow);
  CHECK(fp8_encode(500.0).value.byte == 0x7e && fp8_encode(500.0).overflow);
  CHECK(fp8_encode(-500.0).value.byte == 0xfe);
  for (int b = 0; b < 256; ++b)
    CHECK(fp8_encode(fp8_decode(Fp8Value{static_cast<std::uint8_t>(b)})).value.byte == b);
  CHECK(fp8_encode(432.0).value.byte == 0x7e);
  CHECK(fp8_decode(fp8_encode(431.0).value) == 416.0);
  CHECK(fp8_decode(fp8_encode(21.0).value) == 20.0);
  CHECK(fp8_encode(0x1p-10).value.byte == 0x00);
  CHECK(fp4_decode(fp4_encode(0.25)) == 0.0 && fp4_decode(fp4_encode(0.75)) == 1.0);
  CHECK(fp4_decode(fp4_encode(2.5)) == 2.0 && fp4_decode(fp4_encode(5.0)) == 4.0);
  CHECK(fp4_encode(-0.0) == 0);
  std::mt19937_64 rng(3);
  std::uniform_real_distribution<double> u(-500, 500);
  for (int i = 0; i < 20000; ++i) {
    const double v = u(rng);
    int ov = 0;
    CHECK(fp8_encode(v).value.byte == oracle_fp8_encode(v, &ov) && fp8_encode(v).overflow == (ov != 0));
    CHECK(fp4_encode(v / 60) == oracle_fp4_encode(v / 60));
  }
}

static void codec_cases() {
  const std::vector<float> zeros(300, 0.0f);  // zero payload
  for (auto k : kKinds) {
    const int b = bits_for(k, 5);
    const auto q = quantize_blockwise(zeros, b, 128, k);
    for (float s : q.scales) CHECK(s == 0.0f);
    for (float x : dequantize_blockwise(q)) CHECK(x == 0.0f);
  }
  for (auto k : kKinds) {  // absmax anchors round-trip exactly
    std::mt19937_64 rng(99);
    std::uniform_real_distribution<float> u(-1.2f, 1.2f);
    std::vector<float> x(256);
    for (auto& v : x) v = u(rng);
    x[37] = 1.25f;
    x[200] = -2.75f;
    const auto back = dequantize_blockwise(quantize_blockwise(x, bits_for(k, 6), 128, k));
    CHECK(back[37] == 1.25f && back[200] == -2.75f);
  }
  const auto x = gauss(4096, 1234);  // linear error bound
  for (int b = 4; b <= 8; ++b) {
    const auto q = quantize_blockwise(x, b, 128);
    const auto back = dequantize_blockwise(q);
    const int L = (1 << (b - 1)) - 1;
    for (std::size_t i = 0; i < x.size(); ++i) {
      const double s = q.scales[i / 128];
      CHECK(std::fabs(static_cast<double>(back[i]) - x[i]) <= s / (2.0 * L) + s * 1.2e-7);
    }
  }
  const auto y = gauss(500, 77);  // q(dq(q(x))) == q(x)
  for (auto k : kKinds) {
    const int b = bits_for(k, 7);
    const auto q1 = quantize_blockwise(y, b, 128, k);
    const auto q2 = quantize_blockwise(dequantize_blockwise(q1), b, 128, k);
    CHECK(q1.codes == q2.codes && q1.scales == q2.scales);
  }
  std::vector<float> fp8v;  // FP8 full range with scale 448 is exact
  for (int b = 0; b <= 0x7e; ++b) fp8v.push_back(static_cast<float>(fp8_decode(Fp8Value{(std::uint8_t)b})));
  for (int b = 0x81; b <= 0xfe; ++b) fp8v.push_back(static_cast<float>(fp8_decode(Fp8Value{(std::uint8_t)b})));
  const auto qf = quantize_blockwise(fp8v, 8, static_cast<std::uint32_t>(fp8v.size()), CodecKind::Fp8E4M3);
  CHECK(qf.scales.size() == 1 && qf.scales[0] == 448.0f);
  CHECK(dequantize_blockwise(qf) == fp8v);
  auto blk = gauss(384, 31);  // blocks are independent
  const auto b1 = quantize_blockwise(blk, 5, 128);
  for (std::size_t i = 128; i < 256; ++i) blk[i] *= -3.7f;
  const auto b2 = quantize_blockwise(blk, 5, 128);
  for (std::size_t i = 0; i < 128; ++i) CHECK(b1.codes[i] == b2.codes[i]);
  CHECK(b1.scales[0] == b2.scales[0] && b1.scales[2] == b2.scales[2] && b1.scales[1] != b2.scales[1]);
  auto bad = gauss(300, 8);  // non-finite -> lowest block
  bad[170] = INFINITY;
  CHECK(throws<std::invalid_argument>([&] { quantize_blockwise(bad, 4, 128); }, "block 1"));
  std::vector<float> part(130, 0.0f);  // partial final block
  for (int i = 0; i < 128; ++i) part[i] = 8.0f;
  part[128] = 0.5f;
  part[129] = -1.0f;
  const auto qp = quantize_blockwise(part, 4, 128);
  CHECK(qp.scales.size() == 2 && qp.scales[0] == 8.0f && qp.scales[1] == 1.0f);
  CHECK(dequantize_blockwise(qp)[129] == -1.0f);
  const std::vector<float> ones(16, 1.0f);  // preconditions
  CHECK(throws<std::invalid_argument>([&] { quantize_blockwise(ones, 3, 128); }));
  CHECK(throws<std::invalid_argument>([&] { quantize_blockwise(ones, 9, 128); }));
  CHECK(throws<std::invalid_argument>([&] { quantize_blockwise(ones, 4, 0); }));
  CHECK(throws<std::invalid_argument>([&] { quantize_blockwise(ones, 5, 128, CodecKind::Fp8E4M3); }));
  CHECK(throws<std::invalid_argument>([&] { quantize_blockwise(ones, 5, 128, CodecKind::Fp4E2M1); }));
  std::mt19937_64 rng(991);  // pack/unpack
  for (int b = 4; b <= 8; ++b)
    for (std::size_t n : {1u, 7u, 8u, 129u, 1000u}) {
      std::vector<std::uint8_t> c(n);
      for (auto& v : c) v = static_cast<std::uint8_t>(rng() & ((1u << b) - 1));
      const auto p = pack_codes(c, b);
      CHECK(p.size() == (n * b + 7) / 8 && unpack_codes(p, b, n) == c);
      std::vector<std::uint8_t> ref(p.size() + 1);
      ref.resize(oracle_pack_codes(c.data(), n, b, ref.data()));
      CHECK(ref == p);
    }
  for (auto k : kKinds) {  // dump/load
    const int b = bits_for(k, 6);
    const auto q = quantize_blockwise(gauss(777, 55), b, 128, k, {7, 111});
    std::stringstream ss;
    dump_tensor(q, ss);
    const auto q2 = load_tensor(ss);
    CHECK(q2.codes == q.codes && q2.scales == q.scales && q2.shape == q.shape && q2.codec_kind == k);
  }
  {
    const std::vector<float> x3 = {1.0f, -1.0f, 0.5f};
    std::stringstream ss;
    dump_tensor(quantize_blockwise(x3, 4, 2), ss);
    const std::string bytes = ss.str();
    CHECK(bytes.size() == 4 + 2 + 1 + 1 + 4 + 1 + 8 + 2 * 4 + 2 && bytes.substr(0, 4) == "AGQT");
    CHECK((unsigned char)bytes[bytes.size() - 2] == 14 && (unsigned char)bytes[bytes.size() - 1] == 14);
    std::stringstream bad_magic(std::string("BAD!") + bytes.substr(4));
    CHECK(throws<std::runtime_error>([&] { load_tensor(bad_magic); }));
  }
  // bit-exact vs the oracle on random inputs, all codecs and several blocks
  for (int trial = 0; trial < 6; ++trial) {
    const std::size_t n = 1000 + 7919 * trial * trial;
    auto v = gauss(n, 40 + trial, std::pow(10.0f, trial - 3.0f));
    for (std::uint32_t block : {2u, 16u, 128u, 1000u})
      for (auto k : kKinds)
        for (int b = 4; b <= 8; ++b) {
          if ((k != CodecKind::SymmetricLinear) && b != bits_for(k, b)) continue;
          const auto q = quantize_blockwise(v, b, block, k);
          std::vector<std::uint8_t> c(n);
          std::vector<float> s(q.scales.size());
          oracle_quantize(v.data(), n, b, block, (int)k, c.data(), s.data(), nullptr, 0);
          CHECK(q.codes == c && q.scales == s);
          std::vector<float> d(n);
          oracle_dequantize(c.data(), s.data(), n, b, block, (int)k, d.data(), nullptr, 0);
          CHECK(dequantize_blockwise(q) == d);
        }
  }
}

static QuantizedTensor fp8_tensor(const std::vector<float>& v) {
  return quantize_blockwise(v, 8, 128, CodecKind::Fp8E4M3);
}
static std::vector<WorkerState> world_of(const std::vector<std::vector<float>>& per) {
  std::vector<WorkerState> w;
  for (std::size_t r = 0; r < per.size(); ++r)
    w.push_back(WorkerState::make((int)r, (int)per.size(), fp8_tensor(per[r])));
  return w;
}
static std::vector<std::vector<float>> grads(int world, std::size_t n, std::uint64_t seed) {
  std::vector<std::vector<float>> g;
  for (int r = 0; r < world; ++r) g.push_back(gauss(n, seed * 131 + r));
  return g;
}

static void collective_cases() {
  const auto a = ChunkAssignment::block_aligned(4096, 128, 4);
  CHECK(a.ranges[0] == (std::pair<std::size_t, std::size_t>{0, 1024}));
  CHECK(a.ranges[3] == (std::pair<std::size_t, std::size_t>{3072, 4096}));
  const auto b = ChunkAssignment::block_aligned(300, 128, 2);
  CHECK(b.ranges[1] == (std::pair<std::size_t, std::size_t>{256, 300}));
  // accumulate onto zeros == quantize(g)
  const auto g = gauss(256, 2);
  const auto acc = local_accumulate(fp8_tensor(std::vector<float>(256, 0.0f)), g);
  CHECK(acc.codes == fp8_tensor(g).codes && acc.scales == fp8_tensor(g).scales);
  auto main = fp8_tensor(std::vector<float>(128, 0.0f));  // rescales instead of saturating
  for (int s = 0; s < 8; ++s) main = local_accumulate(main, std::vector<float>(128, 100.0f));
  for (float v : dequantize_blockwise(main)) CHECK(v == 800.0f);
  const auto two = fp8_tensor(std::vector<float>(128, 2.0f));
  CHECK(dequantize_blockwise(local_accumulate(two, std::vector<float>(128, 1.0f), AccumulatePrecision::Bf16))[0] == 3.0f);
  CHECK(dequantize_blockwise(local_accumulate(two, std::vector<float>(128, 1.0f), AccumulatePrecision::Fp16))[0] == 3.0f);
  CHECK(round_bf16(1.0039062f) == 1.0f && round_fp16(70000.0f) == 65504.0f && round_fp16(65504.0f) == 65504.0f);
  std::vector<float> nan_g(128, 0.0f);
  nan_g[5] = NAN;
  CHECK(throws<std::invalid_argument>([&] { local_accumulate(two, nan_g); }, "non-finite local"));
  CHECK(throws<std::invalid_argument>([&] { local_accumulate(two, std::vector<float>(64, 0.0f)); }));
  // accumulate bit-exact vs oracle, all precisions
  for (int prec = 0; prec < 3; ++prec) {
    const auto m = fp8_tensor(gauss(9000, 5, 1e-3f));
    const auto l = gauss(9000, 6, 1e-3f);
    const auto out = local_accumulate(m, l, static_cast<AccumulatePrecision>(prec));
    std::vector<std::uint8_t> oc(9000);
    std::vector<float> os(m.scales.size());
    oracle_local_accumulate(m.codes.data(), m.scales.data(), 9000, 128, l.data(), prec, oc.data(),
                            os.data(), nullptr, 0);
    CHECK(out.codes == oc && out.scales == os);
  }
  // single worker, zeros, constant-64 separation
  {
    auto w = world_of(grads(1, 512, 7));
    const auto r = allreduce_decomposed(w);
    CHECK(r.trace.events.empty() && r.outputs[0].codes == w[0].main_gradient.codes);
    auto wz = world_of(std::vector<std::vector<float>>(4, std::vector<float>(512, 0.0f)));
    for (float v : dequantize_blockwise(allreduce_decomposed(wz).outputs[0])) CHECK(v == 0.0f);
    auto wc = world_of(std::vector<std::vector<float>>(8, std::vector<float>(512, 64.0f)));
    for (float v : dequantize_blockwise(allreduce_decomposed(wc).outputs[0])) CHECK(v == 512.0f);
    auto wn = world_of(std::vector<std::vector<float>>(8, std::vector<float>(512, 64.0f)));
    const auto nr = allreduce_naive_fp8(wn);
    CHECK(nr.overflow_elements == 512);
    for (float v : dequantize_blockwise(nr.outputs[0])) CHECK(v == 64.0f);
  }
  // decomposed == quantize(oracle), within one step of the fp32 oracle
  for (int world : {2, 4, 8}) {
    auto w = world_of(grads(world, 1024, 900 + world));
    const auto oracle = allreduce_oracle(w);
    const auto r = allreduce_decomposed(w);
    const auto direct = quantize_blockwise(oracle, 8, 128, CodecKind::Fp8E4M3);
    CHECK(r.outputs[0].codes == direct.codes && r.outputs[0].scales == direct.scales);
    for (const auto& o : r.outputs) CHECK(o.codes == r.outputs[0].codes);
    const auto vals = dequantize_blockwise(r.outputs[0]);
    for (std::size_t i = 0; i < vals.size(); ++i)
      CHECK(std::fabs(vals[i] - oracle[i]) <= r.outputs[0].scales[i / 128] * (32.0 / 448.0) + 1e-6);
  }
  {  // schedule independence + trace accounting
    auto wa = world_of(grads(4, 1024, 99));
    auto wb = world_of(grads(4, 1024, 99));
    const auto ra = allreduce_decomposed(wa);
    const auto rb = allreduce_decomposed(wb, {3, 1, 0, 2});
    CHECK(ra.outputs[0].codes == rb.outputs[0].codes);
    CHECK(throws<std::invalid_argument>([&] { allreduce_decomposed(wa, {0, 1}); }));
    std::size_t a2a = 0, scale_b = 0, ag = 0;
    for (const auto& e : ra.trace.events) {
      if (e.phase == "all_to_all") {
        a2a += e.chunk_len;
        scale_b += e.payload_bytes - e.chunk_len;
      } else {
        ag += e.chunk_len;
      }
    }
    CHECK(a2a == 4 * 3 * 256 && scale_b == 4 * 3 * 2 * 4 && ag == 4 * 3 * 256);
    std::ostringstream os;
    ra.trace.write_jsonl(os);
    CHECK(os.str().find("\"phase\":\"all_to_all\"") != std::string::npos);
  }
  {  // naive ring vs oracle (codes, scales, overflow counters)
    for (int world : {2, 3, 5}) {
      auto w = world_of(grads(world, 3000, 17 + world));
      const auto r = allreduce_naive_fp8(w);
      std::vector<const std::uint8_t*> pc;
      std::vector<const float*> ps;
      for (auto& x : w) {
        pc.push_back(x.main_gradient.codes.data());
        ps.push_back(x.main_gradient.scales.data());
      }
      std::vector<std::uint8_t> oc(3000);
      std::vector<float> os(w[0].main_gradient.scales.size());
      std::uint64_t ov = 0;
      oracle_allreduce_naive(world, 3000, 128, pc.data(), ps.data(), oc.data(), os.data(), &ov,
                             nullptr, 0);
      CHECK(r.outputs[0].codes == oc && r.outputs[0].scales == os && r.overflow_elements == ov);
    }
  }
  {
    std::vector<WorkerState> w;
    w.push_back(WorkerState::make(0, 2, fp8_tensor(std::vector<float>(256, 1.0f))));
    w.push_back(WorkerState::make(1, 2, fp8_tensor(std::vector<float>(128, 1.0f))));
    CHECK(throws<std::invalid_argument>([&] { allreduce_decomposed(w); }, "shapes must match"));
  }
}

static void dbca_cases() {
  CHECK(stored_activation_counts({4, 8, 2}) == (std::vector<int>{11, 9, 7, 5}));
  CHECK(stored_activation_counts({1, 1, 2}) == (std::vector<int>{1}));
  CHECK(throws<std::invalid_argument>([] { stored_activation_counts({4, 6, 2}); }));
  CHECK(throws<std::invalid_argument>([] { stored_activation_counts({4, 8, 3}); }));
  const auto plan = plan_bit_widths({4, 8, 2});
  CHECK(plan.assigned() == (std::vector<int>{4, 5, 6, 8}));
  CHECK(plan_bit_widths({2, 4, 2}).assigned() == (std::vector<int>{4, 7}));
  CHECK(plan_bit_widths({8, 16, 2}).assigned() == (std::vector<int>{4, 4, 5, 5, 6, 7, 8, 8}));
  const auto chk = peak_memory_check(plan, 16.0);
  CHECK(chk.pass && chk.budget_bytes == 44.0 && chk.stages[1].bytes == 45.0);
  const auto reuse = plan_reuse_check({4, 8, 2}, {8, 16, 2});
  CHECK(reuse.pass && reuse.applied_bits == (std::vector<int>{4, 4, 4, 4, 4, 5, 6, 8}));
  const auto pol = stage_policy(plan, 2);
  CHECK(pol.at(LayerRole::RmsNorm).bit_width == 5);
  CHECK(pol.at(LayerRole::Attention).strategy == SaveStrategy::NoQuant);
  CHECK(throws<std::invalid_argument>([&] { stage_policy(plan, 9); }));
}

// The API's begin/finish host jobs (agq_*_host_begin + agq_host_job_finish):
// multi-chunk ragged sizes equal the oracle and the synchronous entries,
// errors surface at finish with the synchronous text, cancel leaves the
// pipeline usable, oversize calls fall back to the synchronous entry.
static void host_job_cases() {
  const std::size_t n = (5u << 20) + 77;  // 3 pipeline chunks, ragged tail
  const auto x = gauss(n, 11);
  for (CodecKind k : kKinds) {
    const int b = bits_for(k, 5);
    const auto q = quantize_blockwise(x, b, 128, k);
    std::vector<std::uint8_t> oc(n);
    std::vector<float> os(q.scales.size()), od(n), back(n);
    char err[256];
    CHECK(oracle_quantize(x.data(), n, b, 128, static_cast<int>(k), oc.data(), os.data(), err,
                          sizeof err) == 0);
    CHECK(q.codes == oc && q.scales == os);
    CHECK(oracle_dequantize(oc.data(), os.data(), n, b, 128, static_cast<int>(k), od.data(), err,
                            sizeof err) == 0);
    CHECK(dequantize_blockwise(q) == od);
    CHECK(agq_dequantize_host(q.codes.data(), q.scales.data(), n, b, 128, static_cast<int>(k),
                              back.data()) == AGQ_OK);
    CHECK(back == od);
    const auto rd = roundtrip_relative_delta(x, b, 128, k);
    CHECK(rd.size() == n && rd[n - 1] == (x[n - 1] == 0.0f ? 0.0
              : (static_cast<double>(od[n - 1]) - x[n - 1]) / static_cast<double>(x[n - 1])));
  }
  {  // FP8 local accumulate, multi-chunk
    const auto g = gauss(n, 12, 1e-3f), l = gauss(n, 13, 1e-3f);
    const auto main = quantize_blockwise(g, 8, 128, CodecKind::Fp8E4M3);
    const auto acc = local_accumulate(main, l);
    std::vector<std::uint8_t> oc(n);
    std::vector<float> os(main.scales.size());
    char err[256];
    CHECK(oracle_local_accumulate(main.codes.data(), main.scales.data(), n, 128, l.data(), 0,
                                  oc.data(), os.data(), err, sizeof err) == 0);
    CHECK(acc.codes == oc && acc.scales == os && acc.shape == main.shape &&
          acc.codec_kind == CodecKind::Fp8E4M3 && acc.bit_width == 8);
  }
  {  // errors at finish carry the synchronous entry's text
    auto q = quantize_blockwise(x, 4);
    q.scales[7] = -1.0f;
    CHECK(throws<std::invalid_argument>([&] { dequantize_blockwise(q); }, "bad scale at block 7"));
    std::vector<float> bad(x.begin(), x.begin() + 4096);
    bad[300] = NAN;
    CHECK(throws<std::invalid_argument>([&] { quantize_blockwise(bad, 4); }, "non-finite input element in block 2"));
  }
  {  // cancel, then the next call still runs
    agq_host_job* job = nullptr;
    CHECK(agq_quantize_host_begin(x.data(), n, 4, 128, 0, &job) == AGQ_OK && job != nullptr);
    CHECK(agq_host_job_finish(job, nullptr, nullptr) == AGQ_OK);
    CHECK(quantize_blockwise(x, 4).codes == quantize_blockwise(x, 4).codes);
  }
  {  // n == 0 and oversize calls: no job, nothing issued
    agq_host_job* job = reinterpret_cast<agq_host_job*>(1);
    CHECK(agq_quantize_host_begin(x.data(), 0, 4, 128, 0, &job) == AGQ_OK && job == nullptr);
    const std::size_t big = 56u << 20;  // 28 chunks x 10.06 MiB of staging > 256 MiB
    std::vector<float> xb(big, 0.5f);
    job = reinterpret_cast<agq_host_job*>(1);
    CHECK(agq_quantize_host_begin(xb.data(), big, 4, 128, 0, &job) == AGQ_OK && job == nullptr);
    const auto qb = quantize_blockwise(xb, 4);  // the synchronous fallback
    CHECK(qb.codes[big - 1] == 14 && qb.scales.back() == 0.5f);
  }
}

int main() {
  fp8_scalars();
  codec_cases();
  collective_cases();
  dbca_cases();
  host_job_cases();
  std::printf("dropin_tests: %d checks, %d failures\n", g_checks, g_fail);
  return g_fail;
}
