// ref_shim.cpp -- extern "C" face of the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY (the checker and the timed CPU reference arm);
// never linked into the product library.
//
// oracle/Makefile compiles /root/reference/proj/src/{softmax,topk,oracle,
// counting,bench}.cpp in place with -Dosmx=osmx_ref (so every reference
// symbol lands in osmx_ref::) and links them with this shim into
// oracle/_ref/libosmx_ref.so.  This file contains no reference code; it only
// calls the reference's public API (proj/include/osmx/*.hpp) and maps its
// exceptions (error.hpp:8-25) to status codes:
//   0 ok, 1 empty_input_error, 2 non_finite_error, 3 invalid_k_error,
//   4 invalid_chunk_error, 5 other std::exception.
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <thread>
#include <vector>

#include "osmx/bench.hpp"
#include "osmx/counting.hpp"
#include "osmx/error.hpp"
#include "osmx/normalizer.hpp"
#include "osmx/oracle.hpp"
#include "osmx/softmax.hpp"
#include "osmx/topk.hpp"

namespace {

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const osmx::empty_input_error&) {
    return 1;
  } catch (const osmx::non_finite_error&) {
    return 2;
  } catch (const osmx::invalid_k_error&) {
    return 3;
  } catch (const osmx::invalid_chunk_error&) {
    return 4;
  } catch (const std::exception&) {
    return 5;
  }
}

std::span<const float> sp(const float* x, std::int64_t n) {
  return std::span<const float>(x, static_cast<std::size_t>(n));
}

void put(const osmx::topk_result& r, float* v, std::int64_t* z) {
  std::memcpy(v, r.values.data(), r.values.size() * sizeof(float));
  std::memcpy(z, r.indices.data(), r.indices.size() * sizeof(std::int64_t));
}

// One row through one reference entry point (the switch of consume(),
// bench.cpp:34-62, but keeping the outputs).
int run_row(int op, const float* x, std::int64_t n, std::int64_t k, float* y, float* v,
            std::int64_t* z) {
  return guarded([&] {
    switch (op) {
      case 0: { auto o = osmx::naive_softmax(sp(x, n)); std::memcpy(y, o.data(), o.size() * 4); break; }
      case 1: { auto o = osmx::safe_softmax(sp(x, n)); std::memcpy(y, o.data(), o.size() * 4); break; }
      case 2: { auto o = osmx::online_softmax(sp(x, n)); std::memcpy(y, o.data(), o.size() * 4); break; }
      case 3: put(osmx::safe_softmax_then_topk(sp(x, n), static_cast<std::size_t>(k)), v, z); break;
      case 4: put(osmx::safe_softmax_fused_topk(sp(x, n), static_cast<std::size_t>(k)), v, z); break;
      case 5: put(osmx::online_softmax_topk(sp(x, n), static_cast<std::size_t>(k)), v, z); break;
      case 6: put(osmx::topk_of(sp(x, n), static_cast<std::size_t>(k)), v, z); break;
      case 7: put(osmx::oracle_topk(sp(x, n), static_cast<std::size_t>(k)), v, z); break;
      default: throw std::invalid_argument("op");
    }
  });
}

}  // namespace

extern "C" {

// Per-row reference calls.  op: 0 naive_softmax 1 safe_softmax
// 2 online_softmax 3 safe_softmax_then_topk 4 safe_softmax_fused_topk
// 5 online_softmax_topk 6 topk_of 7 oracle_topk.
int osmx_ref_row(int op, const float* x, std::int64_t n, std::int64_t k, float* y, float* v,
                 std::int64_t* z) {
  return run_row(op, x, n, k, y, v, z);
}

// Batched: rows striped over `threads` std::threads exactly like run_batch
// (bench.cpp:75-90).  y has leading dim ldy, v/z leading dim k.
int osmx_ref_batch(int op, const float* x, std::int64_t ldx, std::int64_t rows, std::int64_t n,
                   std::int64_t k, float* y, std::int64_t ldy, float* v, std::int64_t* z,
                   std::int32_t* status, int threads) {
  if (threads < 1) threads = 1;
  auto work = [&](int t) {
    for (std::int64_t r = t; r < rows; r += threads) {
      int s = run_row(op, x + r * ldx, n, k, y ? y + r * ldy : nullptr, v ? v + r * k : nullptr,
                      z ? z + r * k : nullptr);
      if (status) status[r] = s;
    }
  };
  if (threads == 1) {
    work(0);
    return 0;
  }
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) pool.emplace_back(work, t);
  for (auto& th : pool) th.join();
  return 0;
}

int osmx_ref_oracle_softmax(const float* x, std::int64_t n, double* y) {
  return guarded([&] {
    auto o = osmx::oracle_softmax(sp(x, n));
    std::memcpy(y, o.data(), o.size() * sizeof(double));
  });
}

int osmx_ref_oracle_normalizer(const float* x, std::int64_t n, double* m, double* d) {
  return guarded([&] {
    auto s = osmx::oracle_normalizer(sp(x, n));
    *m = s.max;
    *d = s.sum;
  });
}

// run_normalizer<T> / run_normalizer_chunked<T> (normalizer.hpp:61-85);
// chunk == 0 with chunked == 0 selects the sequential pass.
int osmx_ref_normalizer(const float* x, std::int64_t n, int dbl, int chunked, std::int64_t chunk,
                        double* m, double* d) {
  return guarded([&] {
    if (dbl) {
      auto s = chunked ? osmx::run_normalizer_chunked<double>(sp(x, n), static_cast<std::size_t>(chunk))
                       : osmx::run_normalizer<double>(sp(x, n));
      *m = s.max;
      *d = s.sum;
    } else {
      auto s = chunked ? osmx::run_normalizer_chunked<float>(sp(x, n), static_cast<std::size_t>(chunk))
                       : osmx::run_normalizer<float>(sp(x, n));
      *m = s.max;
      *d = s.sum;
    }
  });
}

// merge() (normalizer.hpp:52-58)
void osmx_ref_merge(int dbl, double am, double ad, double bm, double bd, double* m, double* d) {
  if (dbl) {
    auto r = osmx::merge(osmx::norm_state<double>{am, ad}, osmx::norm_state<double>{bm, bd});
    *m = r.max;
    *d = r.sum;
  } else {
    auto r = osmx::merge(osmx::norm_state<float>{static_cast<float>(am), static_cast<float>(ad)},
                         osmx::norm_state<float>{static_cast<float>(bm), static_cast<float>(bd)});
    *m = r.max;
    *d = r.sum;
  }
}

// generate_inputs (bench.cpp:162-172): batch*v floats, row-major.
int osmx_ref_generate_inputs(std::uint64_t seed, std::int64_t batch, std::int64_t v, float* out) {
  return guarded([&] {
    auto rows = osmx::generate_inputs(seed, static_cast<std::size_t>(batch), static_cast<std::size_t>(v));
    for (std::size_t r = 0; r < rows.size(); ++r)
      std::memcpy(out + r * v, rows[r].data(), static_cast<std::size_t>(v) * sizeof(float));
  });
}

// count_accesses (counting.cpp:123-140); alg in counting.hpp:17-24 order.
int osmx_ref_count_accesses(int alg, std::int64_t v, std::int64_t k, std::uint64_t* loads,
                            std::uint64_t* stores) {
  return guarded([&] {
    auto s = osmx::count_accesses(static_cast<osmx::algorithm>(alg), static_cast<std::size_t>(v),
                                  static_cast<std::size_t>(k));
    *loads = s.loads;
    *stores = s.stores;
  });
}

// log_spaced_sizes (bench.cpp:349-369); returns the count written (<= cap).
std::int64_t osmx_ref_log_spaced_sizes(std::int64_t vmin, std::int64_t vmax, std::int64_t points,
                                       std::int64_t* out, std::int64_t cap) {
  std::int64_t n = 0;
  int st = guarded([&] {
    auto s = osmx::log_spaced_sizes(static_cast<std::size_t>(vmin), static_cast<std::size_t>(vmax),
                                    static_cast<std::size_t>(points));
    for (auto e : s) {
      if (n < cap) out[n] = static_cast<std::int64_t>(e);
      ++n;
    }
  });
  return st ? -st : n;
}

// run_sweep (bench.cpp:174-221) for one algorithm and one V: the reference's
// own timing (median of repeats around run_batch); returns elements/s.
double osmx_ref_sweep_cell(int alg, std::int64_t v, std::int64_t batch, std::int64_t k,
                           std::int64_t repeats, std::int64_t warmup, std::uint64_t seed,
                           std::int64_t threads) {
  osmx::sweep_config cfg;
  cfg.algorithms = {static_cast<osmx::algorithm>(alg)};
  cfg.vector_sizes = {static_cast<std::size_t>(v)};
  cfg.batch = static_cast<std::size_t>(batch);
  cfg.k = static_cast<std::size_t>(k);
  cfg.repeats = static_cast<std::size_t>(repeats);
  cfg.warmup = static_cast<std::size_t>(warmup);
  cfg.seed = seed;
  cfg.threads = static_cast<std::size_t>(threads);
  try {
    auto rows = osmx::run_sweep(cfg);
    return rows.at(0).cells.at(0).ok ? rows[0].cells[0].elements_per_second : -1.0;
  } catch (...) {
    return -1.0;
  }
}

}  // extern "C"
