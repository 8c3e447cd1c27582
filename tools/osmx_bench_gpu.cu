// osmx-bench-gpu (tools/osmx_bench_gpu.cu): the reference's sweep driver (tools/osmx_bench.cpp:65-84)
// with the same flags, the same delimited table and the same access-count
// model (counting.hpp:83-86), timing the B200 kernels of libosmx_b200.so
// through the C-ABI instead of the CPU templates.
//
//   V, <Column> (elements/s) ..., <Column>_loads, <Column>_stores ...,
//   OnlineSoftmax_over_SafeSoftmax, OnlineSoftmaxFusedTopK_over_SafeSoftmaxUnfusedTopK
//
// exactly as bench.cpp:223-253 writes them, followed by GPU columns:
// <Column>_GBps (algorithmic bytes = 4 x (loads + stores) per vector x batch
// / median time) and <Column>_frac (of --peak-gbs, default MEASURED_PEAKS.json
// hbm_gbs).  One more algorithm, online-unfused-topk (OnlineSoftmaxUnfusedTopK,
// online softmax then topk_of: loads 3V, stores V + 2K), can be requested.
//
// Inputs: std::mt19937_64(seed) + std::normal_distribution<float>(0, 1) row
// by row -- the reference's generate_inputs (bench.cpp:162-172), same bits --
// copied to the device once per size.  A repeat is one batched launch timed
// with CUDA events; the L2 is flushed (a read of 2 x L2 bytes, outside the
// events) before each repeat.  elements/s = batch * V / median(seconds).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <ctime>
#include <fstream>
#include <iostream>
#include <optional>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include <cuda_runtime.h>
#include <sys/utsname.h>

#include "osmx_b200.h"

namespace {

enum Alg { kNaive, kSafe, kOnline, kSafeUnfused, kSafeFused, kOnlineFused, kOnlineUnfused };
const char* kColumns[] = {"NaiveSoftmax",          "SafeSoftmax",         "OnlineSoftmax",
                          "SafeSoftmaxUnfusedTopK", "SafeSoftmaxFusedTopK", "OnlineSoftmaxFusedTopK",
                          "OnlineSoftmaxUnfusedTopK"};
const char* kAliases[] = {"naive",          "safe",           "online",             "safe-unfused-topk",
                          "safe-fused-topk", "online-fused-topk", "online-unfused-topk"};
// C-ABI algorithm ids (include/osmx_b200.h osmx_algorithm)
const int kAbi[] = {OSMX_NAIVE_SOFTMAX,          OSMX_SAFE_SOFTMAX,           OSMX_ONLINE_SOFTMAX,
                    OSMX_SAFE_SOFTMAX_UNFUSED_TOPK, OSMX_SAFE_SOFTMAX_FUSED_TOPK, OSMX_ONLINE_SOFTMAX_FUSED_TOPK,
                    OSMX_ONLINE_SOFTMAX_UNFUSED_TOPK};

bool uses_topk(int a) { return a >= kSafeUnfused; }

std::optional<int> parse_algorithm(const std::string& s) {  // counting.cpp:21-32
  for (int a = 0; a < 7; ++a)
    if (s == kColumns[a] || s == kAliases[a]) return a;
  return std::nullopt;
}

// counting.hpp:83-86 (pinned against the reference in tests/test_oracle.py)
void count_accesses(int a, uint64_t v, uint64_t k, uint64_t& loads, uint64_t& stores) {
  switch (a) {
    case kNaive: loads = 2 * v, stores = v; break;
    case kSafe: loads = 3 * v, stores = v; break;
    case kOnline: loads = 2 * v, stores = v; break;
    case kSafeUnfused: loads = 4 * v, stores = v + 2 * k; break;
    case kSafeFused: loads = 3 * v, stores = 2 * k; break;
    case kOnlineFused: loads = v, stores = 2 * k; break;
    default: loads = 3 * v, stores = v + 2 * k; break;  // online softmax + topk_of
  }
}

std::vector<uint64_t> log_spaced_sizes(uint64_t vmin, uint64_t vmax, uint64_t points) {  // bench.cpp:349-369
  if (vmin == 0 || vmax < vmin || points == 0)
    throw std::invalid_argument("log_spaced_sizes: need 1 <= vmin <= vmax and points >= 1");
  std::vector<uint64_t> out;
  if (points == 1) return {vmin};
  const double lmin = std::log(double(vmin)), lmax = std::log(double(vmax));
  for (uint64_t i = 0; i < points; ++i) {
    const double f = double(i) / double(points - 1);
    const auto v = (uint64_t)std::llround(std::exp(lmin + f * (lmax - lmin)));
    out.push_back(std::clamp<uint64_t>(v, vmin, vmax));
  }
  out.back() = vmax;
  std::sort(out.begin(), out.end());
  out.erase(std::unique(out.begin(), out.end()), out.end());
  return out;
}

std::string format_double(double v) {  // bench.cpp:113-117
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

std::vector<std::string> split(const std::string& s, char d) {
  std::vector<std::string> out;
  std::stringstream ss(s);
  std::string item;
  while (std::getline(ss, item, d))
    if (!item.empty()) out.push_back(item);
  return out;
}

double measured_peak() {
  for (const char* p : {"MEASURED_PEAKS.json", "../MEASURED_PEAKS.json"}) {
    std::ifstream f(p);
    if (!f) continue;
    std::stringstream ss;
    ss << f.rdbuf();
    const std::string s = ss.str();
    const auto i = s.find("\"hbm_gbs\"");
    if (i == std::string::npos) continue;
    return std::atof(s.c_str() + s.find(':', i) + 1);
  }
  return 6650.0;  // B200_PROFILING.md fallback
}

__global__ void flush_read(const float4* p, size_t n, float* sink) {
  float acc = 0.0f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    acc += p[i].x;
  if (acc == 12345.678f) *sink = acc;  // never true; keeps the loads
}

#define CK(call)                                                                               \
  do {                                                                                         \
    cudaError_t e_ = (call);                                                                   \
    if (e_ != cudaSuccess) throw std::runtime_error(std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

struct Cell {
  bool ok = true;
  std::string error;
  double eps = NAN;
  uint64_t loads = 0, stores = 0;
};

}  // namespace

int main(int argc, char** argv) {
  std::vector<int> algs = {kNaive, kSafe, kOnline, kSafeUnfused, kSafeFused, kOnlineFused};
  std::vector<uint64_t> sizes;
  uint64_t vmin = 40, vmax = 500000, points = 12, batch = 100, k = 5, repeats = 5, warmup = 2, seed = 1,
           threads = 1;
  bool sizes_set = false, range_set = false, counts_only = false;
  std::string out_path = "-", format = "csv", plot_prefix;
  double peak = measured_peak();
  int device = 0;
  try {
    for (int i = 1; i < argc; ++i) {
      std::string a = argv[i];
      std::string val;
      const auto eq = a.find('=');
      if (eq != std::string::npos) val = a.substr(eq + 1), a = a.substr(0, eq);
      auto next = [&]() -> std::string {
        if (!val.empty()) return val;
        if (i + 1 >= argc) throw std::invalid_argument("missing value for " + a);
        return argv[++i];
      };
      if (a == "--algorithms") {
        algs.clear();
        for (const auto& n : split(next(), ',')) {
          const auto p = parse_algorithm(n);
          if (!p) throw std::invalid_argument("unknown algorithm: " + n);
          algs.push_back(*p);
        }
      } else if (a == "--sizes") {
        for (const auto& n : split(next(), ',')) sizes.push_back(std::stoull(n));
        sizes_set = true;
      } else if (a == "--vmin") {
        vmin = std::stoull(next()), range_set = true;
      } else if (a == "--vmax") {
        vmax = std::stoull(next()), range_set = true;
      } else if (a == "--points") {
        points = std::stoull(next()), range_set = true;
      } else if (a == "--batch") {
        batch = std::stoull(next());
      } else if (a == "--k") {
        k = std::stoull(next());
      } else if (a == "--repeats") {
        repeats = std::stoull(next());
      } else if (a == "--warmup") {
        warmup = std::stoull(next());
      } else if (a == "--seed") {
        seed = std::stoull(next());
      } else if (a == "--threads") {
        threads = std::stoull(next());  // host generation only; the device does the work
      } else if (a == "--out") {
        out_path = next();
      } else if (a == "--format") {
        format = next();
        if (format != "csv" && format != "tsv") throw std::invalid_argument("--format: csv or tsv");
      } else if (a == "--counts-only") {
        counts_only = true;
      } else if (a == "--plot") {
        plot_prefix = next();
      } else if (a == "--peak-gbs") {
        peak = std::atof(next().c_str());
      } else if (a == "--device") {
        device = std::stoi(next());
      } else if (a == "-h" || a == "--help") {
        std::cout << "osmx-bench-gpu [--algorithms a,b] [--sizes v,..|--vmin N --vmax N --points N] [--batch N]\n"
                     "               [--k N] [--repeats N] [--warmup N] [--seed N] [--threads N] [--out PATH]\n"
                     "               [--format csv|tsv] [--counts-only] [--plot PREFIX] [--peak-gbs X] [--device N]\n";
        return 0;
      } else {
        throw std::invalid_argument("unknown option: " + a);
      }
    }
    if (sizes_set && range_set) throw std::invalid_argument("--sizes excludes --vmin/--vmax/--points");
    if (algs.empty() || batch == 0 || repeats == 0 || threads == 0 || k == 0)
      throw std::invalid_argument("sweep config: algorithms, batch, repeats, threads, k must be non-empty / >= 1");
    if (!sizes_set) sizes = log_spaced_sizes(vmin, vmax, points);
    std::sort(sizes.begin(), sizes.end());
    sizes.erase(std::unique(sizes.begin(), sizes.end()), sizes.end());

    std::vector<std::vector<Cell>> table(sizes.size(), std::vector<Cell>(algs.size()));
    cudaStream_t st = nullptr;
    float *dx = nullptr, *dy = nullptr, *dv = nullptr, *flush = nullptr, *sink = nullptr;
    int64_t* di = nullptr;
    size_t flush_n = 0;
    if (!counts_only) {
      CK(cudaSetDevice(device));
      CK(cudaStreamCreate(&st));
      int l2 = 0;
      CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device));
      flush_n = (size_t)2 * l2 / 16;
      CK(cudaMalloc(&flush, flush_n * 16));
      CK(cudaMemset(flush, 0, flush_n * 16));
      CK(cudaMalloc(&sink, 4));
    }
    for (size_t si = 0; si < sizes.size(); ++si) {
      const uint64_t v = sizes[si];
      std::vector<float> host;
      if (!counts_only) {
        host.resize(batch * v);
        std::mt19937_64 rng(seed);  // generate_inputs, bench.cpp:162-172
        std::normal_distribution<float> normal(0.0f, 1.0f);
        for (auto& e : host) e = normal(rng);
        CK(cudaMalloc(&dx, host.size() * 4));
        CK(cudaMalloc(&dy, host.size() * 4));
        CK(cudaMalloc(&dv, batch * k * 4));
        CK(cudaMalloc(&di, batch * k * 8));
        CK(cudaMemcpy(dx, host.data(), host.size() * 4, cudaMemcpyHostToDevice));
      }
      for (size_t ai = 0; ai < algs.size(); ++ai) {
        const int a = algs[ai];
        Cell& c = table[si][ai];
        if (uses_topk(a) && (k > v)) {
          c.ok = false, c.error = "k must be in [1, V]";
          continue;
        }
        count_accesses(a, v, uses_topk(a) ? k : 0, c.loads, c.stores);
        if (counts_only) continue;
        const size_t wsb = osmx_workspace_bytes(kAbi[a], (int64_t)batch, (int64_t)v, uses_topk(a) ? (int)k : 0);
        void* ws = nullptr;
        CK(cudaMalloc(&ws, wsb));
        CK(cudaMemset(ws, 0, wsb));
        auto launch = [&]() -> osmx_status {
          if (uses_topk(a))
            return osmx_softmax_topk(kAbi[a], dx, (int64_t)v, (int64_t)batch, (int64_t)v, (int32_t)k, dv, di, ws, wsb,
                                     st);
          return osmx_softmax(kAbi[a], dx, (int64_t)v, dy, (int64_t)v, (int64_t)batch, (int64_t)v, ws, wsb, st);
        };
        osmx_status s = OSMX_OK;
        for (uint64_t w = 0; w < warmup && s == OSMX_OK; ++w) s = launch();
        std::vector<double> secs;
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        for (uint64_t r = 0; r < repeats && s == OSMX_OK; ++r) {
          flush_read<<<1184, 256, 0, st>>>(reinterpret_cast<const float4*>(flush), flush_n, sink);
          CK(cudaEventRecord(e0, st));
          s = launch();
          CK(cudaEventRecord(e1, st));
          CK(cudaEventSynchronize(e1));
          float ms = 0.0f;
          CK(cudaEventElapsedTime(&ms, e0, e1));
          secs.push_back(ms * 1e-3);
        }
        if (s == OSMX_OK) {
          int64_t bad = -1;
          s = osmx_check_status(ws, st, &bad);
        }
        CK(cudaEventDestroy(e0));
        CK(cudaEventDestroy(e1));
        CK(cudaFree(ws));
        if (s != OSMX_OK) {
          c.ok = false, c.error = osmx_status_string(s);
          continue;
        }
        std::sort(secs.begin(), secs.end());
        const size_t n = secs.size();
        const double med = n % 2 ? secs[n / 2] : 0.5 * (secs[n / 2 - 1] + secs[n / 2]);
        c.eps = double(batch) * double(v) / med;
      }
      if (!counts_only) {
        CK(cudaFree(dx));
        CK(cudaFree(dy));
        CK(cudaFree(dv));
        CK(cudaFree(di));
      }
      std::cerr << "V=" << v;
      for (size_t ai = 0; ai < algs.size(); ++ai) {
        const Cell& c = table[si][ai];
        std::cerr << "  " << kColumns[algs[ai]] << "=";
        if (!c.ok)
          std::cerr << "error(" << c.error << ")";
        else if (counts_only)
          std::cerr << c.loads + c.stores;
        else
          std::cerr << std::scientific << c.eps << std::defaultfloat;
      }
      std::cerr << '\n';
    }

    // ------------------------------------------------------------ table --
    const char d = format == "tsv" ? '\t' : ',';
    auto find = [&](int a) -> long {
      for (size_t i = 0; i < algs.size(); ++i)
        if (algs[i] == a) return (long)i;
      return -1;
    };
    std::vector<std::pair<int, int>> ratios;  // bench.cpp:124-127
    if (!counts_only) {
      for (auto r : {std::make_pair((int)kOnline, (int)kSafe), std::make_pair((int)kOnlineFused, (int)kSafeUnfused)})
        if (find(r.first) >= 0 && find(r.second) >= 0) ratios.push_back(r);
    }
    std::ostringstream out;
    {
      utsname uts{};
      uname(&uts);
      std::ostringstream cmd;
      for (int i = 0; i < argc; ++i) cmd << (i ? " " : "") << argv[i];
      char ts[32];
      const std::time_t now = std::time(nullptr);
      std::strftime(ts, sizeof ts, "%Y-%m-%dT%H:%M:%SZ", std::gmtime(&now));
      cudaDeviceProp prop{};
      if (!counts_only) cudaGetDeviceProperties(&prop, device);
      out << "# generated: " << ts << '\n';
      out << "# command: " << cmd.str() << '\n';
      out << "# machine: " << uts.sysname << " " << uts.release << " " << uts.machine
          << ", gpu: " << (counts_only ? "none" : prop.name) << ", library: libosmx_b200 v" << osmx_version() << '\n';
      out << "# config: algorithms=";
      for (size_t i = 0; i < algs.size(); ++i) out << (i ? "," : "") << kColumns[algs[i]];
      out << " batch=" << batch << " k=" << k << " repeats=" << repeats << " warmup=" << warmup << " seed=" << seed
          << " threads=" << threads << (counts_only ? " counts-only" : "") << " peak_gbs=" << peak << '\n';
      out << "# elements/second = batch*V / median(repeat seconds), one batched device launch per repeat, L2 "
             "flushed before each; loads/stores are the exact per-vector access model (counting.hpp:83-86); "
             "_GBps = 4 B x (loads + stores) x batch / median seconds\n";
    }
    out << 'V';
    if (!counts_only)
      for (int a : algs) out << d << kColumns[a];
    for (int a : algs) out << d << kColumns[a] << "_loads" << d << kColumns[a] << "_stores";
    for (auto r : ratios) out << d << kColumns[r.first] << "_over_" << kColumns[r.second];
    if (!counts_only)
      for (int a : algs) out << d << kColumns[a] << "_GBps" << d << kColumns[a] << "_frac";
    out << '\n';
    for (size_t si = 0; si < sizes.size(); ++si) {
      out << sizes[si];
      const auto& row = table[si];
      if (!counts_only)
        for (const auto& c : row) out << d << format_double(c.eps);
      for (const auto& c : row) {
        if (c.ok)
          out << d << c.loads << d << c.stores;
        else
          out << d << "nan" << d << "nan";
      }
      for (auto r : ratios) {
        const Cell& a = row[find(r.first)];
        const Cell& b = row[find(r.second)];
        out << d << format_double(a.ok && b.ok ? a.eps / b.eps : NAN);
      }
      if (!counts_only) {
        for (const auto& c : row) {
          const double gbps = c.ok ? c.eps / double(sizes[si]) * 4.0 * double(c.loads + c.stores) / 1e9 : NAN;
          out << d << format_double(gbps) << d << format_double(gbps / peak);
        }
      }
      out << '\n';
    }
    if (out_path == "-") {
      std::cout << out.str();
    } else {
      std::ofstream f(out_path);
      if (!f) throw std::runtime_error("cannot open for writing: " + out_path);
      f << out.str();
      std::cerr << "wrote " << out_path << " (" << sizes.size() << " rows)\n";
    }
    if (!plot_prefix.empty()) {  // bench.cpp:264-283
      auto series = [&](const std::string& name, auto&& value_of) {
        std::ofstream f(plot_prefix + "." + name + ".dat");
        if (!f) throw std::runtime_error("cannot open for writing: " + plot_prefix + "." + name + ".dat");
        f << "# series: " << name << "\nV " << name << '\n';
        for (size_t si = 0; si < sizes.size(); ++si) f << sizes[si] << ' ' << format_double(value_of(si)) << '\n';
      };
      for (size_t ai = 0; ai < algs.size(); ++ai)
        series(kColumns[algs[ai]], [&](size_t si) { return table[si][ai].eps; });
      for (auto r : ratios)
        series(std::string(kColumns[r.first]) + "_over_" + kColumns[r.second], [&](size_t si) {
          const Cell& a = table[si][find(r.first)];
          const Cell& b = table[si][find(r.second)];
          return a.ok && b.ok ? a.eps / b.eps : NAN;
        });
    }
    if (flush) cudaFree(flush);
    if (sink) cudaFree(sink);
    if (st) cudaStreamDestroy(st);
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 2;
  }
  return 0;
}
