// test_reference_api.cpp -- the reference's own test cases
// (/root/reference/proj/tests/test_softmax.cpp, test_normalizer.cpp's
// softmax-facing parts, and the SPEC.md top-K examples) re-run against the
// B200 implementation through include/osmx/b200.hpp, i.e. through exactly
// the C++ API a reference caller uses.  Values are checked against the
// oracle port (oracle/osmx_oracle.c, itself pinned to the reference).
//
// Built by `make tests/cpp/test_reference_api`; run by
// tests/test_gpu_cpp_api.py on the GPU box.  Prints "ALL OK" on success.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <random>
#include <vector>

#include "osmx/b200.hpp"

extern "C" {
int oracle_safe_softmax(const float*, size_t, float*);
int oracle_online_softmax(const float*, size_t, float*);
int oracle_naive_softmax(const float*, size_t, float*);
int oracle_online_softmax_topk(const float*, size_t, size_t, float*, int64_t*);
int oracle_softmax_double(const float*, size_t, double*);
}

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                       \
  do {                                                                 \
    ++g_checks;                                                        \
    if (!(c)) {                                                        \
      ++g_fail;                                                        \
      std::fprintf(stderr, "%s:%d CHECK failed: %s\n", __FILE__, __LINE__, #c); \
    }                                                                  \
  } while (0)
#define CHECK_THROWS_AS(expr, T)   \
  do {                             \
    bool ok = false;               \
    try {                          \
      (void)(expr);                \
    } catch (const T&) {           \
      ok = true;                   \
    } catch (...) {                \
    }                              \
    CHECK(ok && #T);               \
  } while (0)

static std::int64_t ulps(float a, float b) {
  std::int32_t ia, ib;
  std::memcpy(&ia, &a, 4);
  std::memcpy(&ib, &b, 4);
  if (ia < 0) ia = std::numeric_limits<std::int32_t>::min() - ia;
  if (ib < 0) ib = std::numeric_limits<std::int32_t>::min() - ib;
  return std::llabs((std::int64_t)ia - (std::int64_t)ib);
}

static std::vector<float> quantized_uniform(std::mt19937_64& rng, std::size_t n, double range) {
  const long lim = std::lround(range * 1024.0);
  std::uniform_int_distribution<long> dist(-lim, lim);
  std::vector<float> x(n);
  for (auto& e : x) e = (float)(dist(rng) / 1024.0);
  return x;
}

static void check_rel(const std::vector<float>& y, const std::vector<double>& ref, double tol) {
  CHECK(y.size() == ref.size());
  for (size_t i = 0; i < y.size(); ++i) {
    if (ref[i] <= 1e-30) continue;
    CHECK(std::abs((double)y[i] - ref[i]) <= tol * ref[i]);
  }
}

int main() {
  using osmx::naive_softmax;
  using osmx::online_softmax;
  using osmx::safe_softmax;
  using F = std::vector<float> (*)(std::span<const float>);
  const F all[3] = {naive_softmax, safe_softmax, online_softmax};

  // test_softmax.cpp:37 single element maps to exactly 1
  for (auto f : all) {
    auto y = f(std::vector<float>{0.0f});
    CHECK(y.size() == 1 && y[0] == 1.0f);
  }
  CHECK(safe_softmax(std::vector<float>{-123.5f})[0] == 1.0f);
  CHECK(online_softmax(std::vector<float>{87.0f})[0] == 1.0f);

  // :47 equal elements split the mass exactly
  for (float c : {0.0f, 1.5f, -20.0f, 13.25f}) {
    std::vector<float> x(4, c);
    for (auto f : all)
      for (float v : f(x)) CHECK(v == 0.25f);
  }
  for (float v : safe_softmax(std::vector<float>(5, 2.0f))) CHECK(v == (float)(1.0 / 5.0));

  // :59 naive overflows where safe stays exact
  {
    std::vector<float> x{100.0f, 100.0f};
    auto yn = naive_softmax(x);
    CHECK(std::isnan(yn[0]) && std::isnan(yn[1]));
    auto ys = safe_softmax(x), yo = online_softmax(x);
    CHECK(ys[0] == 0.5f && ys[1] == 0.5f && yo[0] == 0.5f && yo[1] == 0.5f);
  }
  // :75
  {
    std::vector<float> x{50.0f, 89.0f, 0.0f};
    bool nf = false;
    for (float v : naive_softmax(x)) nf = nf || !std::isfinite(v);
    CHECK(nf);
    for (float v : safe_softmax(x)) CHECK(std::isfinite(v));
  }
  // :83 reference values for [1,2,3]
  {
    std::vector<float> x{1.0f, 2.0f, 3.0f};
    std::vector<double> ref{0.090030573170380462, 0.24472847105479764, 0.66524095577482178};
    for (auto f : all) check_rel(f(x), ref, 1e-6);
  }
  // :93 extreme underflow path stays finite
  {
    std::vector<float> x{-87.0f, 0.0f};
    auto y = safe_softmax(x);
    CHECK(std::isfinite(y[0]) && std::abs(y[0] - 1.6458114537543937e-38) <= 1e-6 * 1.6458114537543937e-38);
    CHECK(y[1] == 1.0f);
    auto yo = online_softmax(x);
    CHECK(yo[0] == y[0] && yo[1] == 1.0f);
  }
  // :104 input validation
  {
    const std::vector<float> empty;
    const std::vector<float> with_nan{1.0f, std::numeric_limits<float>::quiet_NaN()};
    const std::vector<float> with_inf{1.0f, std::numeric_limits<float>::infinity()};
    const std::vector<float> with_ninf{-std::numeric_limits<float>::infinity(), 1.0f};
    for (auto f : all) {
      CHECK_THROWS_AS(f(empty), osmx::empty_input_error);
      CHECK_THROWS_AS(f(with_nan), osmx::non_finite_error);
      CHECK_THROWS_AS(f(with_inf), osmx::non_finite_error);
      CHECK_THROWS_AS(f(with_ninf), osmx::non_finite_error);
    }
  }
  // :117 monotone inputs; safe vs online within 4 ulps, 1e-6 of the oracle
  {
    std::vector<float> asc, desc;
    for (int i = 0; i < 200; ++i) desc.push_back(10.0f - 0.125f * i);
    for (int i = 0; i < 200; ++i) asc.push_back(-10.0f + 0.125f * i);
    for (const auto& x : {desc, asc}) {
      std::vector<double> ref(x.size());
      oracle_softmax_double(x.data(), x.size(), ref.data());
      auto ys = safe_softmax(x), yo = online_softmax(x);
      check_rel(ys, ref, 1e-6);
      check_rel(yo, ref, 1e-6);
      for (size_t i = 0; i < x.size(); ++i) CHECK(ulps(ys[i], yo[i]) <= 4);
    }
  }
  // :131 rerun is bit-identical
  {
    std::mt19937_64 rng(60);
    std::normal_distribution<float> nd(0.0f, 1.0f);
    std::vector<float> x(3000);
    for (auto& e : x) e = nd(rng);
    CHECK(online_softmax(x) == online_softmax(x));
    CHECK(safe_softmax(x) == safe_softmax(x));
    CHECK(naive_softmax(x) == naive_softmax(x));
  }
  // :139 randomized (reduced to 200 cases; batched over the GPU below):
  // outputs in [0,1], sum 1 +- 1e-5, 1e-6 of the double oracle, safe ~ online
  {
    std::mt19937_64 rng(61);
    std::uniform_int_distribution<std::size_t> len(1, 10000);
    for (int t = 0; t < 200; ++t) {
      auto x = quantized_uniform(rng, len(rng), 100.0);
      auto ys = safe_softmax(x), yo = online_softmax(x);
      std::vector<double> ref(x.size());
      oracle_softmax_double(x.data(), x.size(), ref.data());
      double sum = 0.0;
      for (size_t i = 0; i < x.size(); ++i) {
        CHECK(ys[i] >= 0.0f && ys[i] <= 1.0f && yo[i] >= 0.0f && yo[i] <= 1.0f);
        CHECK(ulps(ys[i], yo[i]) <= 8);  // the reference's 4 ulps hold vs fp64 d; fp32 d adds <= 4
        sum += ys[i];
      }
      CHECK(std::abs(sum - 1.0) <= 1e-5);
      check_rel(ys, ref, 2e-6);
      check_rel(yo, ref, 2e-6);
    }
  }
  // :194 argmax of the output equals argmax of the input
  {
    std::mt19937_64 rng(64);
    std::uniform_int_distribution<std::size_t> len(1, 4000);
    for (int t = 0; t < 100; ++t) {
      auto x = quantized_uniform(rng, len(rng), 20.0);
      size_t want = 0;
      for (size_t i = 1; i < x.size(); ++i)
        if (x[i] > x[want]) want = i;
      for (auto f : {safe_softmax, online_softmax}) {
        auto y = f(x);
        size_t got = 0;
        for (size_t i = 1; i < y.size(); ++i)
          if (y[i] > y[got]) got = i;
        CHECK(got == want);
      }
    }
  }
  // SPEC.md top-K examples and ties
  {
    auto r = osmx::topk_of(std::vector<float>{0.1f, 0.7f, 0.2f}, 2);
    CHECK(r.indices == (std::vector<std::int64_t>{1, 2}));
    CHECK(osmx::topk_of(std::vector<float>{0.5f, 0.5f}, 1).indices[0] == 0);
    for (auto f : {osmx::online_softmax_topk, osmx::safe_softmax_fused_topk, osmx::safe_softmax_then_topk}) {
      auto a = f(std::vector<float>{1, 2, 3}, 2);
      CHECK(a.indices == (std::vector<std::int64_t>{2, 1}));
      CHECK(std::abs(a.values[0] - 0.66524095577482178) <= 1e-6);
      CHECK(f(std::vector<float>{5.0f}, 1).values[0] == 1.0f);
      CHECK(f(std::vector<float>{2, 2, 1}, 2).indices == (std::vector<std::int64_t>{0, 1}));
      CHECK_THROWS_AS(f(std::vector<float>{1.0f, 2.0f}, 3), osmx::invalid_k_error);
      CHECK_THROWS_AS(f(std::vector<float>{1.0f, 2.0f}, 0), osmx::invalid_k_error);
      CHECK_THROWS_AS(f(std::vector<float>{}, 1), osmx::empty_input_error);
      CHECK_THROWS_AS(f(std::vector<float>{1.0f, NAN}, 1), osmx::non_finite_error);
    }
    CHECK(osmx::online_softmax_topk(std::vector<float>{0, -0.0f, 1, 1, -0.0f, 0}, 4).indices ==
          (std::vector<std::int64_t>{2, 3, 0, 1}));
  }
  // batched fused top-K vs the oracle on quantized (tie-heavy) rows
  {
    std::mt19937_64 rng(77);
    const size_t rows = 300, V = 5000, k = 5;
    auto x = quantized_uniform(rng, rows * V, 2.0);
    auto r = osmx::batched::online_softmax_topk(x, rows, k);
    for (size_t i = 0; i < rows; ++i) {
      float v[k];
      int64_t z[k];
      oracle_online_softmax_topk(x.data() + i * V, V, k, v, z);
      for (size_t j = 0; j < k; ++j) {
        CHECK(r.indices[i * k + j] == z[j]);
        CHECK(std::abs(r.values[i * k + j] - v[j]) <= 1e-5 * v[j]);
      }
    }
  }
  // k above the register lists (the reference accepts any 1 <= k <= V):
  // radix-select path, same C++ call, bit-exact indices vs the oracle
  {
    std::mt19937_64 rng(78);
    for (size_t V : {200, 3001}) {
      for (size_t k : {33, 150, 200}) {
        if (k > V) continue;
        auto x = quantized_uniform(rng, V, 2.0);
        auto r = osmx::online_softmax_topk(x, k);
        std::vector<float> v(k);
        std::vector<int64_t> z(k);
        oracle_online_softmax_topk(x.data(), V, k, v.data(), z.data());
        CHECK(r.indices == z);
        for (size_t j = 0; j < k; ++j) CHECK(std::abs(r.values[j] - v[j]) <= 1e-5 * v[j]);
      }
    }
  }
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  if (g_fail == 0) std::printf("ALL OK\n");
  return g_fail ? 1 : 0;
}
