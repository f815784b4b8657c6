// Analysis front end around the GPU batch path:
//   * read_dataset (io.cpp:48-120): the comma-delimited dataset, same
//     validation, messages and duplicate-label suffixing;
//   * filter_low_variance (analysis.cpp:92-113) with the variances computed on
//     the GPU (pearson.cu k_center_vars / k_variances);
//   * run_analysis + ResultWriter (analysis.cpp:133-191, io.cpp:122-154): the
//     pair sequence of an AnalysisTask scored on the GPU in blocks (per-variable
//     stages once per job: reuse_vars), every record formatted exactly like
//     format_record (io.cpp:17-47: "%.6g", "nan") -- on the GPU from the
//     HBM-resident statistics (format.cu; only the text crosses PCIe), or by
//     `workers` host threads with MINE_B200_HOST_FORMAT -- and written through
//     a temporary file renamed into place on success.
// Host C++; it drives the engine through the public C ABI.
#include <algorithm>
#include <charconv>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <memory>
#include <stdexcept>
#include <string>
#include <string_view>
#include <system_error>
#include <thread>
#include <unordered_map>
#include <vector>

#include <cuda_runtime.h>

#include "mine_b200.h"
#include "mine_kernels.h"

namespace mb200 {
void set_last_error(const std::string& msg);
int ctx_device(const mine_b200_ctx* ctx);
}

namespace {

template <typename F>
auto guarded(F&& f, decltype(f()) on_error) -> decltype(f()) {
  try {
    return f();
  } catch (const std::exception& e) {
    mb200::set_last_error(e.what());
    return on_error;
  }
}

std::string_view trim(std::string_view s) {
  while (!s.empty() && (s.front() == ' ' || s.front() == '\t')) s.remove_prefix(1);
  while (!s.empty() && (s.back() == ' ' || s.back() == '\t')) s.remove_suffix(1);
  return s;
}

[[noreturn]] void fail_line(const std::string& path, size_t line_no, const std::string& what) {
  throw std::runtime_error(path + ": line " + std::to_string(line_no) + ": " + what);
}

mine_b200_dataset* new_dataset(int p, int n, std::vector<double>&& values,
                               const std::vector<std::string>& names) {
  auto* ds = new mine_b200_dataset{};
  ds->p = p;
  ds->n = n;
  ds->values = new double[(size_t)p * n];
  std::copy(values.begin(), values.end(), ds->values);
  ds->names = new char*[(size_t)p];
  for (int j = 0; j < p; ++j) {
    ds->names[j] = new char[names[j].size() + 1];
    std::memcpy(ds->names[j], names[j].c_str(), names[j].size() + 1);
  }
  return ds;
}

// io.cpp:48-120
mine_b200_dataset* read_dataset(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error(path + ": cannot open for reading");
  std::vector<std::string> names;
  std::vector<double> values;  // row after row == variable-major
  long long n = -1;
  std::string line;
  size_t line_no = 0;
  while (std::getline(in, line)) {
    ++line_no;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (line.empty()) continue;
    std::vector<std::string_view> fields;
    std::string_view rest = line;
    while (true) {
      const size_t comma = rest.find(',');
      fields.push_back(rest.substr(0, comma));
      if (comma == std::string_view::npos) break;
      rest.remove_prefix(comma + 1);
    }
    if (fields.size() < 2) fail_line(path, line_no, "expected a label followed by at least one value");
    if (n == -1)
      n = (long long)fields.size() - 1;
    else if ((long long)fields.size() - 1 != n)
      fail_line(path, line_no,
                "expected " + std::to_string(n) + " values, got " + std::to_string(fields.size() - 1));
    const std::string_view label = trim(fields[0]);
    if (label.empty()) fail_line(path, line_no, "empty variable label");
    names.emplace_back(label);
    for (size_t f = 1; f < fields.size(); ++f) {
      const std::string_view tok = trim(fields[f]);
      double v = 0.0;
      const auto [ptr, ec] = std::from_chars(tok.data(), tok.data() + tok.size(), v);
      if (ec != std::errc{} || ptr != tok.data() + tok.size() || !std::isfinite(v))
        fail_line(path, line_no,
                  "field " + std::to_string(f + 1) + ": cannot parse '" + std::string(tok) +
                      "' as a finite number");
      values.push_back(v);
    }
  }
  if (names.empty()) throw std::runtime_error(path + ": no variables found");
  if (n < 2) throw std::runtime_error(path + ": need at least 2 samples per variable");
  // duplicate labels get an occurrence suffix (io.cpp:101-113)
  std::unordered_map<std::string, int> seen;
  for (auto& name : names) {
    int& count = seen[name];
    ++count;
    if (count > 1) {
      int suffix = count;
      std::string candidate = name + "_" + std::to_string(suffix);
      while (seen.count(candidate)) candidate = name + "_" + std::to_string(++suffix);
      seen[candidate] = 1;
      name = candidate;
    }
  }
  return new_dataset((int)names.size(), (int)n, std::move(values), names);
}

// analysis.cpp:92-113, variances on the GPU
mine_b200_dataset* filter_low_variance(mine_b200_ctx* ctx, const mine_b200_dataset* in,
                                       double threshold) {
  if (threshold < 0.0) throw std::invalid_argument("filter_low_variance: threshold must be >= 0");
  std::vector<double> var((size_t)in->p);
  if (mine_b200_variances(ctx, in->values, in->p, in->n, var.data()) != 0)
    throw std::runtime_error(mine_b200_last_error());
  std::vector<int> keep;
  for (int j = 0; j < in->p; ++j)
    if (!(var[(size_t)j] < threshold)) keep.push_back(j);
  if (keep.empty()) throw std::invalid_argument("filter_low_variance: no variables pass the threshold");
  std::vector<double> values;
  values.reserve(keep.size() * (size_t)in->n);
  std::vector<std::string> names;
  for (int j : keep) {
    values.insert(values.end(), in->values + (size_t)j * in->n, in->values + (size_t)(j + 1) * in->n);
    names.emplace_back(in->names[j]);
  }
  return new_dataset((int)keep.size(), in->n, std::move(values), names);
}

// "%.6g" of v without the C library, bit-for-bit the text glibc's printf
// writes (exact decimal rounding, ties to even, exponent chosen after
// rounding, trailing zeros stripped).  v = m 2^e is scaled EXACTLY by a power
// of ten in 128-bit integers: D = round(|v| 10^p) with 10^5 <= D < 10^6.
// Covers 1e-17 <= |v| < 1e15 (every MINE statistic); returns 0 outside, and
// the caller falls back to snprintf.  mine_b200_check_format compares it
// with snprintf on random and boundary values (tests/test_frontend.py).
int fmt6g_fast(double v, char* out) {
  const double a = std::fabs(v);
  if (!(a >= 1e-17) || !(a < 1e15)) return 0;
  int e2;
  const double fr = std::frexp(a, &e2);                  // a = fr 2^e2, fr in [0.5, 1)
  const unsigned long long m = (unsigned long long)std::ldexp(fr, 53);  // exact
  const int e = e2 - 53;                                 // a = m 2^e
  static const unsigned __int128 kPow10[] = {
      1ULL, 10ULL, 100ULL, 1000ULL, 10000ULL, 100000ULL, 1000000ULL, 10000000ULL, 100000000ULL,
      1000000000ULL, 10000000000ULL, 100000000000ULL, 1000000000000ULL, 10000000000000ULL,
      100000000000000ULL, 1000000000000000ULL, 10000000000000000ULL, 100000000000000000ULL,
      1000000000000000000ULL, (unsigned __int128)1000000000000000000ULL * 10,
      (unsigned __int128)1000000000000000000ULL * 100, (unsigned __int128)1000000000000000000ULL * 1000,
      (unsigned __int128)1000000000000000000ULL * 10000};
  // decimal exponent from the binary one: a in [2^(e2-1), 2^e2), so X is
  // this estimate or one more (the loop below settles it exactly)
  int X = (int)std::floor((e2 - 1) * 0.30102999566398120);
  unsigned long long D = 0;
  for (int iter = 0; iter < 4; ++iter) {
    const int p = 5 - X;  // -9 .. 22 for the covered range
    if (p < -9 || p > 22) return 0;
    unsigned __int128 q, r, den;
    if (p >= 0 && e < 0) {  // |v| < 1e6: the divisor is 2^-e, a shift
      const unsigned __int128 num = (unsigned __int128)m * kPow10[p];
      const int s = -e;
      if (s >= 127) return 0;
      q = num >> s;
      r = num - (q << s);
      den = (unsigned __int128)1 << s;
    } else {
      unsigned __int128 num = m;
      den = 1;
      if (p >= 0)
        num *= kPow10[p];
      else
        den = kPow10[-p];
      if (e >= 0)
        num <<= e;  // |v| < 1e15 < 2^53 keeps e < 0 in practice
      else
        den <<= -e;
      q = num / den;
      r = num - q * den;
    }
    if (q < 100000) {  // X was one too large
      --X;
      continue;
    }
    if (q >= 1000000) {  // X was one too small
      ++X;
      continue;
    }
    D = (unsigned long long)q;
    if (2 * r > den || (2 * r == den && (D & 1))) ++D;  // round half to even
    if (D == 1000000) {  // rounding carried into a new decade
      D = 100000;
      ++X;
    }
    break;
  }
  if (D == 0) return 0;
  char dig[6];
  for (int i = 5; i >= 0; --i, D /= 10) dig[i] = (char)('0' + D % 10);
  int nd = 6;
  while (nd > 1 && dig[nd - 1] == '0') --nd;  // %g strips trailing zeros
  char* o = out;
  if (std::signbit(v)) *o++ = '-';
  if (X >= -4 && X < 6) {  // %f style, precision 5 - X
    if (X >= 0) {
      for (int i = 0; i <= X; ++i) *o++ = i < nd ? dig[i] : '0';
      if (nd > X + 1) {
        *o++ = '.';
        for (int i = X + 1; i < nd; ++i) *o++ = dig[i];
      }
    } else {
      *o++ = '0';
      *o++ = '.';
      for (int i = 0; i < -X - 1; ++i) *o++ = '0';
      for (int i = 0; i < nd; ++i) *o++ = dig[i];
    }
  } else {  // %e style, precision 5
    *o++ = dig[0];
    if (nd > 1) {
      *o++ = '.';
      for (int i = 1; i < nd; ++i) *o++ = dig[i];
    }
    *o++ = 'e';
    *o++ = X < 0 ? '-' : '+';
    const int ax = X < 0 ? -X : X;
    if (ax >= 100) *o++ = (char)('0' + ax / 100);
    *o++ = (char)('0' + ax / 10 % 10);
    *o++ = (char)('0' + ax % 10);
  }
  *o = 0;
  return (int)(o - out);
}

// io.cpp:17-22
void append_value(std::string& out, double v) {
  if (std::isnan(v)) {
    out += "nan";
    return;
  }
  char buf[32];
  if (v == 0.0) {
    out += std::signbit(v) ? "-0" : "0";
    return;
  }
  if (fmt6g_fast(v, buf)) {
    out += buf;
    return;
  }
  std::snprintf(buf, sizeof buf, "%.6g", v);
  out += buf;
}

// The pair sequence of a task (analysis.cpp:43-90), each record oriented with
// the lower index first (score_pair, :117-129); 0-based (lo, hi).
struct Sequence {
  int mode = 0;
  long long p = 0, master = 0, first = 0, second = 0, size = 0;
  void at(long long w, int& lo, int& hi) const {
    long long i, j;
    if (mode == 0) {
      const long long total = p * (p - 1) / 2, r = total - w;
      long long m = (long long)((std::sqrt(8.0 * (double)r + 1.0) - 1.0) / 2.0);
      while (m * (m + 1) / 2 < r) ++m;
      while (m >= 1 && (m - 1) * m / 2 >= r) --m;
      i = p - m;
      j = i + 1 + (w - (total - m * (m + 1) / 2));
    } else if (mode == 1) {
      const long long jj = w + 1;
      i = master;
      j = jj < master ? jj : jj + 1;
    } else {
      i = first;
      j = second;
    }
    lo = (int)std::min(i, j) - 1;
    hi = (int)std::max(i, j) - 1;
  }
};

Sequence make_sequence(const mine_b200_task& t, long long p) {
  Sequence s;
  s.mode = t.mode;
  s.p = p;
  s.master = t.master;
  s.first = t.first;
  s.second = t.second;
  auto check = [&](long long idx, const char* what) {
    if (idx < 1 || idx > p) throw std::out_of_range(std::string("expand_pairs: ") + what + " index out of range");
  };
  if (t.mode == 0) {
    s.size = p * (p - 1) / 2;
  } else if (t.mode == 1) {
    check(t.master, "master");
    s.size = p - 1;
  } else if (t.mode == 2) {
    check(t.first, "first");
    check(t.second, "second");
    if (t.first == t.second) throw std::invalid_argument("expand_pairs: pair indices must differ");
    s.size = 1;
  } else {
    throw std::invalid_argument("run_analysis: unknown mode");
  }
  return s;
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// The device side of run_analysis: the dataset, the labels and each block's
// statistics stay in HBM; format.cu turns a block into its text, and only
// the text is copied back (pinned).
struct DeviceRecords {
  int dev = 0;
  cudaStream_t s = nullptr;
  double* vals = nullptr;
  char* names = nullptr;
  long long* noff = nullptr;
  double* st[6] = {};
  int *xi = nullptr, *yi = nullptr, *flag = nullptr, *h_fb = nullptr;
  void* scr = nullptr;
  char *text = nullptr, *h_text = nullptr;
  size_t cap = 0;

  DeviceRecords(mine_b200_ctx* ctx, const mine_b200_dataset* ds, long long block) {
    try {
      init(ctx, ds, block);
    } catch (...) {
      release();
      throw;
    }
  }
  void init(mine_b200_ctx* ctx, const mine_b200_dataset* ds, long long block) {
    dev = mb200::ctx_device(ctx);
    cuda_check(cudaSetDevice(dev), "cudaSetDevice");
    cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
    const size_t nv = (size_t)ds->p * ds->n;
    cuda_check(cudaMalloc(&vals, sizeof(double) * nv), "cudaMalloc");
    cuda_check(cudaMemcpy(vals, ds->values, sizeof(double) * nv, cudaMemcpyHostToDevice), "cudaMemcpy");
    std::vector<long long> off(1, 0);
    std::string all;
    size_t longest = 0;
    for (int j = 0; j < ds->p; ++j) {
      const size_t l = std::strlen(ds->names[j]);
      all.append(ds->names[j], l);
      off.push_back((long long)all.size());
      longest = std::max(longest, l);
    }
    cuda_check(cudaMalloc(&names, all.size() + 1), "cudaMalloc");
    cuda_check(cudaMemcpy(names, all.data(), all.size(), cudaMemcpyHostToDevice), "cudaMemcpy");
    cuda_check(cudaMalloc(&noff, sizeof(long long) * off.size()), "cudaMalloc");
    cuda_check(cudaMemcpy(noff, off.data(), sizeof(long long) * off.size(), cudaMemcpyHostToDevice),
               "cudaMemcpy");
    for (auto& p : st) cuda_check(cudaMalloc(&p, sizeof(double) * (size_t)block), "cudaMalloc");
    cuda_check(cudaMalloc(&xi, sizeof(int) * (size_t)block), "cudaMalloc");
    cuda_check(cudaMalloc(&yi, sizeof(int) * (size_t)block), "cudaMalloc");
    cuda_check(cudaMalloc(&flag, sizeof(int)), "cudaMalloc");
    cuda_check(cudaMallocHost(&h_fb, sizeof(int)), "cudaMallocHost");
    cuda_check(cudaMalloc(&scr, mb200::format_scratch_bytes(block)), "cudaMalloc");
    // a record is at most 2 labels + 6 values of <= 13 bytes + 8 separators
    grow((size_t)block * (2 * longest + 6 * 13 + 8));
  }
  void grow(size_t bytes) {
    if (bytes <= cap) return;
    if (text) cudaFree(text);
    if (h_text) cudaFreeHost(h_text);
    text = nullptr;
    h_text = nullptr;
    cuda_check(cudaMalloc(&text, bytes), "cudaMalloc");
    cuda_check(cudaMallocHost(&h_text, bytes), "cudaMallocHost");
    cap = bytes;
  }
  ~DeviceRecords() { release(); }
  void release() {
    cudaSetDevice(dev);
    for (auto& p : st) {
      cudaFree(p);
      p = nullptr;
    }
    cudaFree(vals);
    cudaFree(names);
    cudaFree(noff);
    cudaFree(xi);
    cudaFree(yi);
    cudaFree(flag);
    cudaFreeHost(h_fb);
    cudaFree(scr);
    cudaFree(text);
    cudaFreeHost(h_text);
    if (s) cudaStreamDestroy(s);
    vals = nullptr, names = nullptr, noff = nullptr, xi = yi = flag = h_fb = nullptr;
    scr = nullptr, text = h_text = nullptr, s = nullptr;
  }
};

long long run_analysis(mine_b200_ctx* ctx, const mine_b200_dataset* dataset,
                       const mine_b200_task& task, const std::string& out_path) {
  if (task.workers < 1) throw std::invalid_argument("run_analysis: workers must be positive");
  const mine_b200_dataset* ds = dataset;
  mine_b200_dataset* filtered = nullptr;
  struct Free {
    mine_b200_dataset*& d;
    ~Free() { mine_b200_free_dataset(d); }
  } free_filtered{filtered};
  if (task.has_min_variance) {
    filtered = filter_low_variance(ctx, dataset, task.min_variance);
    ds = filtered;
  }
  const Sequence seq = make_sequence(task, ds->p);

  // ResultWriter (io.cpp:122-154): temporary file, renamed into place on success
  const std::string tmp = out_path + ".tmp";
  std::FILE* f = std::fopen(tmp.c_str(), "wb");
  if (!f) throw std::runtime_error(tmp + ": cannot open for writing");
  struct Tmp {
    std::FILE*& f;
    const std::string& path;
    bool keep = false;
    ~Tmp() {
      if (f) std::fclose(f);
      if (!keep) {
        std::error_code ec;
        std::filesystem::remove(path, ec);
      }
    }
  } guard{f, tmp};
  static const char kHeader[] = "var1,var2,MIC,MAS,MEV,MCN,pearson,nonlinearity\n";
  std::fwrite(kHeader, 1, sizeof kHeader - 1, f);

  const mine_parameter par{task.alpha, task.c, MINE_EST_MIC_APPROX};
  const long long block = 1LL << 20;
  std::vector<double> st[6];
  std::vector<int> xi, yi;
  const unsigned nthreads = (unsigned)std::max(1, task.workers);
  std::vector<std::string> text(nthreads);
  const bool timing = std::getenv("MINE_B200_TIMING") != nullptr;
  double t_gpu = 0, t_fmt = 0, t_io = 0;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto secs = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
  // records are formatted on the GPU unless MINE_B200_HOST_FORMAT is set
  std::unique_ptr<DeviceRecords> dr;
  const auto s0 = now();
  if (!std::getenv("MINE_B200_HOST_FORMAT") && seq.size > 0) dr.reset(new DeviceRecords(ctx, ds, block));
  const double t_setup = secs(s0, now());
  for (long long base = 0; base < seq.size; base += block) {
    const long long count = std::min(block, seq.size - base);
    const auto c0 = now();
    if (dr) {  // statistics and text on the device
      mine_stats_out out{};
      out.mic = dr->st[0];
      out.mas = dr->st[1];
      out.mev = dr->st[2];
      out.mcn = dr->st[3];
      out.pearson_r = dr->st[4];
      out.nonlinearity = dr->st[5];
      mine_b200_opts opt{};
      opt.device_io = 1;
      opt.stream = dr->s;
      opt.reuse_vars = base > 0;
      mb200::PairSpace ps;
      int rc;
      if (seq.mode == 0) {
        opt.first = base;
        opt.count = count;
        rc = mine_b200_pairwise(ctx, dr->vals, ds->p, ds->n, &par, &opt, &out);
        ps.kind = mb200::kPairwise;
        ps.p = ds->p;
        ps.first = base;
      } else {
        xi.resize((size_t)count);
        yi.resize((size_t)count);
        for (long long w = 0; w < count; ++w) seq.at(base + w, xi[(size_t)w], yi[(size_t)w]);
        cuda_check(cudaMemcpyAsync(dr->xi, xi.data(), sizeof(int) * count, cudaMemcpyHostToDevice, dr->s),
                   "cudaMemcpyAsync");
        cuda_check(cudaMemcpyAsync(dr->yi, yi.data(), sizeof(int) * count, cudaMemcpyHostToDevice, dr->s),
                   "cudaMemcpyAsync");
        opt.count = count;
        rc = mine_b200_pairs(ctx, dr->vals, ds->p, ds->n, dr->xi, dr->yi, count, &par, &opt, &out);
        ps.kind = mb200::kList;
        ps.xi = dr->xi;
        ps.yi = dr->yi;
      }
      if (rc != 0) throw std::runtime_error(mine_b200_last_error());
      ps.count = count;
      const auto c1 = now();
      size_t bytes = 0;
      const double* const stp[6] = {dr->st[0], dr->st[1], dr->st[2], dr->st[3], dr->st[4], dr->st[5]};
      cuda_check(mb200::launch_format_records(ps, stp, dr->names, dr->noff, count, dr->scr, dr->text,
                                              dr->cap, &bytes, dr->flag, dr->h_fb, dr->s),
                 "format_records");
      if (!*dr->h_fb) {
        if (bytes > dr->cap) {  // cannot happen with the bound above; grow and redo
          dr->grow(bytes);
          cuda_check(mb200::launch_format_records(ps, stp, dr->names, dr->noff, count, dr->scr,
                                                  dr->text, dr->cap, &bytes, dr->flag, dr->h_fb, dr->s),
                     "format_records");
        }
        cuda_check(cudaMemcpyAsync(dr->h_text, dr->text, bytes, cudaMemcpyDeviceToHost, dr->s),
                   "cudaMemcpyAsync");
        cuda_check(cudaStreamSynchronize(dr->s), "cudaStreamSynchronize");
        const auto c2 = now();
        if (std::fwrite(dr->h_text, 1, bytes, f) != bytes) throw std::runtime_error(tmp + ": write failed");
        const auto c3 = now();
        t_gpu += secs(c0, c1);
        t_fmt += secs(c1, c2);
        t_io += secs(c2, c3);
        continue;
      }
      // a value outside the device formatter's range: this block on the host
      for (int k = 0; k < 6; ++k) {
        st[k].resize((size_t)count);
        cuda_check(cudaMemcpy(st[k].data(), dr->st[k], sizeof(double) * count, cudaMemcpyDeviceToHost),
                   "cudaMemcpy");
      }
    } else {  // statistics to host buffers, host formatting
      for (auto& v : st) v.resize((size_t)count);
      mine_stats_out out{};
      out.mic = st[0].data();
      out.mas = st[1].data();
      out.mev = st[2].data();
      out.mcn = st[3].data();
      out.pearson_r = st[4].data();
      out.nonlinearity = st[5].data();
      mine_b200_opts opt{};
      opt.reuse_vars = base > 0;  // the per-variable stages run once per job
      int rc;
      if (seq.mode == 0) {
        opt.first = base;
        opt.count = count;
        rc = mine_b200_pairwise(ctx, ds->values, ds->p, ds->n, &par, &opt, &out);
      } else {
        xi.resize((size_t)count);
        yi.resize((size_t)count);
        for (long long w = 0; w < count; ++w) seq.at(base + w, xi[(size_t)w], yi[(size_t)w]);
        opt.count = count;
        rc = mine_b200_pairs(ctx, ds->values, ds->p, ds->n, xi.data(), yi.data(), count, &par, &opt,
                             &out);
      }
      if (rc != 0) throw std::runtime_error(mine_b200_last_error());
    }
    const auto c1 = now();
    // format_record (io.cpp:37-47) for this block, `workers` threads
    auto format = [&](unsigned t) {
      const long long lo_w = count * t / nthreads, hi_w = count * (t + 1) / nthreads;
      std::string& s = text[t];
      s.clear();
      int lo = 0, hi = 0;
      if (lo_w < hi_w) seq.at(base + lo_w, lo, hi);
      for (long long w = lo_w; w < hi_w; ++w) {
        if (w > lo_w) {
          if (seq.mode == 0) {  // next (i, j) of the condensed order
            if (++hi == seq.p) {
              ++lo;
              hi = lo + 1;
            }
          } else {
            seq.at(base + w, lo, hi);
          }
        }
        s += ds->names[lo];
        s += ',';
        s += ds->names[hi];
        for (int k = 0; k < 6; ++k) {
          s += ',';
          append_value(s, st[k][(size_t)w]);
        }
        s += '\n';
      }
    };
    if (nthreads == 1) {
      format(0);
    } else {
      std::vector<std::thread> pool;
      for (unsigned t = 0; t < nthreads; ++t) pool.emplace_back(format, t);
      for (auto& th : pool) th.join();
    }
    const auto c2 = now();
    for (const auto& s : text)
      if (std::fwrite(s.data(), 1, s.size(), f) != s.size()) throw std::runtime_error(tmp + ": write failed");
    const auto c3 = now();
    t_gpu += secs(c0, c1);
    t_fmt += secs(c1, c2);
    t_io += secs(c2, c3);
  }
  const auto s1 = now();
  if (std::fflush(f) != 0 || std::ferror(f)) throw std::runtime_error(tmp + ": write failed");
  std::fclose(f);
  f = nullptr;
  std::error_code ec;
  std::filesystem::rename(tmp, out_path, ec);
  if (ec) throw std::runtime_error(out_path + ": cannot replace output: " + ec.message());
  guard.keep = true;
  dr.reset();
  if (timing)
    std::fprintf(stderr, "run_analysis: setup %.3f s, gpu %.3f s, format %.3f s, write %.3f s, close %.3f s\n",
                 t_setup, t_gpu, t_fmt, t_io, secs(s1, now()));
  return seq.size;
}

}  // namespace

extern "C" {

int mine_b200_read_dataset(const char* path, mine_b200_dataset** out) {
  return guarded(
      [&] {
        if (!path || !out) throw std::invalid_argument("read_dataset: null argument");
        *out = read_dataset(path);
        return 0;
      },
      -1);
}

void mine_b200_free_dataset(mine_b200_dataset* ds) {
  if (!ds) return;
  for (int j = 0; j < ds->p; ++j) delete[] ds->names[j];
  delete[] ds->names;
  delete[] ds->values;
  delete ds;
}

int mine_b200_filter_low_variance(mine_b200_ctx* ctx, const mine_b200_dataset* in, double threshold,
                                  mine_b200_dataset** out) {
  return guarded(
      [&] {
        if (!ctx || !in || !out) throw std::invalid_argument("filter_low_variance: null argument");
        *out = filter_low_variance(ctx, in, threshold);
        return 0;
      },
      -1);
}

long long mine_b200_run_analysis(mine_b200_ctx* ctx, const mine_b200_dataset* ds,
                                 const mine_b200_task* task, const char* out_path) {
  return guarded(
      [&] {
        if (!ctx || !ds || !task || !out_path) throw std::invalid_argument("run_analysis: null argument");
        return run_analysis(ctx, ds, *task, out_path);
      },
      -1LL);
}

// Self-test of the exact "%.6g" (records.cpp fmt6g_fast) against snprintf:
// `count` values (random magnitudes 1e-18 .. 1e16, values near rounding ties
// and decade boundaries, small rationals); returns the number of mismatches.
namespace {
// the self-test's value generator: random magnitudes 1e-18 .. 1e16, 6-digit
// decimals +- a few ulps (rounding ties), decade boundaries, small rationals
std::vector<double> format_test_values(long long count, unsigned long long seed) {
  unsigned long long st = seed * 6364136223846793005ULL + 1442695040888963407ULL;
  auto next = [&] {
    st = st * 6364136223846793005ULL + 1442695040888963407ULL;
    return st >> 11;  // 53 random bits
  };
  std::vector<double> out((size_t)count);
  for (long long i = 0; i < count; ++i) {
    double v;
    switch (i % 4) {
      case 0: {
        const double u = (double)next() / 9007199254740992.0;
        v = std::pow(10.0, -18.0 + 34.0 * u) * ((next() & 1) ? -1 : 1);
        break;
      }
      case 1: {
        const double d = 100000.0 + (double)(next() % 900000);
        const int x = (int)(next() % 30) - 17;
        v = (d + 0.5) * std::pow(10.0, x - 5);
        for (int k = (int)(next() % 7) - 3; k != 0; k += k > 0 ? -1 : 1)
          v = std::nextafter(v, k > 0 ? 1e300 : -1e300);
        break;
      }
      case 2: {
        const int x = (int)(next() % 30) - 17;
        v = std::pow(10.0, x) * (1.0 - 5e-7 * ((double)(next() % 2000) / 1000.0));
        break;
      }
      default: {
        const double num = (double)(next() % 100000), den = (double)(1 + next() % 100000);
        v = (next() & 1) ? num / den : std::log2(1.0 + (double)(next() % 100000));
        break;
      }
    }
    out[(size_t)i] = v;
  }
  return out;
}
}  // namespace

// Self-test of the exact "%.6g" record formatter (host: records.cpp
// fmt6g_fast; device >= 0: format.cu on that GPU) against snprintf on
// `count` generated values; returns the mismatch count (0 expected), -1 on a
// CUDA error.  Values the device formatter leaves to the host are skipped.
long long mine_b200_check_format(long long count, unsigned long long seed, int device) {
  const std::vector<double> vals = format_test_values(count, seed);
  std::vector<char> dev_text;
  std::vector<int> dev_len;
  if (device >= 0) {
    double* dv = nullptr;
    char* dt = nullptr;
    int* dl = nullptr;
    if (cudaSetDevice(device) != cudaSuccess || cudaMalloc(&dv, sizeof(double) * count) != cudaSuccess ||
        cudaMalloc(&dt, 24 * (size_t)count) != cudaSuccess || cudaMalloc(&dl, sizeof(int) * count) != cudaSuccess)
      return -1;
    cudaMemcpy(dv, vals.data(), sizeof(double) * count, cudaMemcpyHostToDevice);
    mb200::format_values_device(dv, count, dt, dl, nullptr);
    dev_text.resize(24 * (size_t)count);
    dev_len.resize((size_t)count);
    cudaMemcpy(dev_text.data(), dt, dev_text.size(), cudaMemcpyDeviceToHost);
    cudaMemcpy(dev_len.data(), dl, sizeof(int) * count, cudaMemcpyDeviceToHost);
    const bool ok = cudaGetLastError() == cudaSuccess;
    cudaFree(dv);
    cudaFree(dt);
    cudaFree(dl);
    if (!ok) return -1;
  }
  long long bad = 0;
  for (long long i = 0; i < count; ++i) {
    const double v = vals[(size_t)i];
    char want[40];
    std::snprintf(want, sizeof want, "%.6g", v);
    std::string got;
    if (device >= 0) {
      const int l = dev_len[(size_t)i];
      if (l == 0) continue;  // outside the device range: the host formats it
      got.assign(&dev_text[(size_t)i * 24], (size_t)l);
    } else {
      append_value(got, v);
    }
    if (got != want) ++bad;
  }
  return bad;
}

}  // extern "C"
