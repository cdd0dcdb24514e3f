// hygt_apply.cpp -- `hygt_gpu_apply`: the GPU drop-in for the reference CLI's `hygt apply`
// (tools/hygt_main.cpp:130-172, option surface :247-256, exit codes :275-284).
//
//   hygt_gpu_apply --model M.hygt --data D.rblk [--direction forward|inverse]
//                  [--arithmetic float|fixed] --out O.rblk [--timing]
//
// Reads the HYGT model bundle (bundle.hpp:105-191) and the RBLK dataset (dataset.hpp:72-119),
// transforms every block on the GPU through the C ABI (include/hygt_gpu.h) and writes the RBLK
// result. The whole dataset is parsed into pinned structure-of-arrays buffers (class ids u16,
// samples fp32 or int64) by several host threads, then streamed through the device in chunks on
// two CUDA streams so the copies overlap the kernels.
//
// Semantics kept from the reference:
//   * float arithmetic uses the bundle's float models, or the dequantized angles 2*pi*code/2^b
//     of a quantized bundle (bundle.hpp:83-86, fixedpoint.hpp:132-135); output is fp32;
//   * fixed arithmetic needs a quantized bundle, rounds inputs with llround (hygt_main.cpp:157)
//     and writes the int64 results as float(double(y)) exactly as write_rblk does;
//   * errors print "error: <message>" and exit 1 (ArgumentError), 2 (IoError), 3 (numerical).
// Classes with fewer rounds than the longest are padded with zero-angle rounds, which are the
// identity bit for bit in both arithmetics (cos 0 = 1, sin 0 = 0; (2^p a + 2^(p-1)) >> p = a).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <chrono>
#include <cstdio>
#include <memory>
#include <cstring>
#include <fstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "hygt_gpu.h"

namespace {

struct Fail : std::runtime_error {
  int code;
  Fail(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void arg_error(const std::string& m) { throw Fail(1, m); }
[[noreturn]] void io_error(const std::string& m) { throw Fail(2, m); }

void check(int status) {
  if (status == HYGT_OK) return;
  char msg[512] = {0};
  hygt_last_error(msg, sizeof msg);
  const int code = status == HYGT_ERR_ARGUMENT ? 1 : status == HYGT_ERR_IO ? 2
                 : (status == HYGT_ERR_NUMERICAL || status == HYGT_ERR_OVERFLOW) ? 3 : 4;
  throw Fail(code, msg);
}
void cu(cudaError_t e) {
  if (e != cudaSuccess) throw Fail(4, std::string("CUDA: ") + cudaGetErrorString(e));
}

// ---- little-endian readers over an in-memory file -------------------------------------------
struct Reader {
  const unsigned char* p;
  size_t n, off = 0;
  const char* what;
  void need(size_t k) {
    if (off + k > n) io_error("unexpected end of file");
  }
  uint8_t u8() { need(1); return p[off++]; }
  uint16_t u16() { need(2); uint16_t v = (uint16_t)(p[off] | (p[off + 1] << 8)); off += 2; return v; }
  uint32_t u32() { need(4); uint32_t v; std::memcpy(&v, p + off, 4); off += 4; return v; }
  double f64() { need(8); double v; std::memcpy(&v, p + off, 8); off += 8; return v; }
  void magic(const char* m) {
    if (off + 4 > n || std::memcmp(p + off, m, 4) != 0) io_error(std::string("bad magic: not a ") + what + " file");
    off += 4;
  }
};

std::vector<unsigned char> slurp(const std::string& path) {
  std::ifstream is(path, std::ios::binary | std::ios::ate);
  if (!is) io_error("cannot open for reading: " + path);
  const std::streamsize size = is.tellg();
  std::vector<unsigned char> buf((size_t)std::max<std::streamsize>(size, 0));
  is.seekg(0);
  if (size > 0 && !is.read(reinterpret_cast<char*>(buf.data()), size)) io_error("cannot read: " + path);
  return buf;
}

size_t num_parameters(int log2n, int rounds) { return (size_t)rounds * log2n * ((size_t)1 << (log2n - 1)); }

struct Bundle {
  int log2n = 0, classes = 0, angle_bits = 0, precision_bits = 10, max_rounds = 0;
  std::vector<int> rounds;
  std::vector<std::vector<double>> angles;     // float bundle
  std::vector<std::vector<uint16_t>> codes;    // quantized bundle
  std::vector<std::vector<uint16_t>> perm;     // empty = none
};

Bundle read_bundle(const std::string& path) {
  const auto buf = slurp(path);
  Reader r{buf.data(), buf.size(), 0, "HYGT model bundle"};
  r.magic("HYGT");
  if (r.u8() != 1) io_error("read_bundle: unsupported version");
  Bundle b;
  b.log2n = r.u8();
  b.classes = r.u16();
  b.angle_bits = r.u8();
  b.precision_bits = r.u8();
  if (b.log2n < 1 || b.log2n > 16) io_error("read_bundle: bad log2_n");
  if (b.classes == 0) io_error("read_bundle: no classes");
  if (b.angle_bits > 8) io_error("read_bundle: bad angle_bits");
  const size_t n = (size_t)1 << b.log2n;
  for (int c = 0; c < b.classes; ++c) {
    const int rounds = r.u8();
    const bool has_perm = r.u8() != 0;
    if (rounds < 1) io_error("read_bundle: num_parameters: log2_n and rounds must be >= 1");
    b.rounds.push_back(rounds);
    b.max_rounds = std::max(b.max_rounds, rounds);
    const size_t a = num_parameters(b.log2n, rounds);
    if (b.angle_bits == 0) {
      std::vector<double> v(a);
      for (double& x : v) {
        x = r.f64();
        if (!std::isfinite(x)) io_error("read_bundle: HyGTModel: non-finite angle");
      }
      b.angles.push_back(std::move(v));
    } else {
      std::vector<uint16_t> v(a);
      for (uint16_t& q : v) q = r.u8();
      b.codes.push_back(std::move(v));
    }
    std::vector<uint16_t> p;
    if (has_perm) {
      p.resize(n);
      std::vector<char> seen(n, 0);
      for (uint16_t& q : p) {
        q = r.u16();
        if (q >= n || seen[q]) io_error("read_bundle: HyGTModel: permutation is not a bijection");
        seen[q] = 1;
      }
    }
    b.perm.push_back(std::move(p));
  }
  return b;
}

// Final permutations as the plan's [C][R][N] gather table (bit R-1 of the mask), identity rows
// for classes without one.
uint32_t perm_table(const Bundle& b, std::vector<uint16_t>& out) {
  const size_t n = (size_t)1 << b.log2n, R = (size_t)b.max_rounds;
  bool any = false;
  for (const auto& p : b.perm) any |= !p.empty();
  if (!any) return 0;
  out.assign((size_t)b.classes * R * n, 0);
  for (int c = 0; c < b.classes; ++c)
    for (size_t k = 0; k < R; ++k)
      for (size_t i = 0; i < n; ++i)
        out[((size_t)c * R + k) * n + i] =
            (k == R - 1 && !b.perm[c].empty()) ? b.perm[c][i] : (uint16_t)i;
  return 1u << (R - 1);
}

struct Dataset {
  int log2n = 0, classes = 0;
  uint64_t count = 0;
  uint16_t* cls = nullptr;  // host, pageable
  void* x = nullptr;        // host fp32 or int64, pageable (outputs are written back into it)
};

// Parses RBLK records (u16 class + N fp32, dataset.hpp:68-70) into SoA buffers.
bool g_timing = false;  // --timing: per-phase wall times on stderr

Dataset read_rblk(const std::string& path, bool fixed, int bundle_classes, std::thread& cuda_init) {
  const bool timing = g_timing;
  auto t0 = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    const auto t = std::chrono::steady_clock::now();
    if (timing) std::fprintf(stderr, "[apply]   %-8s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(t - t0).count());
    t0 = t;
  };
  const auto buf = slurp(path);
  mark("slurp");
  Reader r{buf.data(), buf.size(), 0, "RBLK dataset"};
  r.magic("RBLK");
  if (r.u8() != 1) io_error("read_rblk: unsupported version");
  Dataset d;
  d.log2n = r.u8();
  d.classes = r.u16();
  d.count = r.u32();
  if (d.log2n < 1 || d.log2n > 16) io_error("read_rblk: bad log2_n");
  if (d.classes == 0) io_error("read_rblk: ResidualDataset: need at least one class");
  const size_t n = (size_t)1 << d.log2n, rec = 2 + 4 * n;
  if (r.off + d.count * rec > buf.size()) io_error("unexpected end of file");
  // pageable SoA buffers, filled while the CUDA context is still being created: pinning ~0.3-0.6 GB
  // costs more than the driver's staged copies of it (DESIGN, apply timing)
  d.cls = new uint16_t[std::max<size_t>(d.count, 1)];
  d.x = fixed ? static_cast<void*>(new int64_t[std::max<size_t>(d.count, 1) * n])
              : static_cast<void*>(new float[std::max<size_t>(d.count, 1) * n]);
  mark("alloc");
  const unsigned char* base = buf.data() + r.off;
  const unsigned threads = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  std::vector<std::thread> pool;
  std::vector<int> bad(threads, 0);
  for (unsigned t = 0; t < threads; ++t)
    pool.emplace_back([&, t] {
      const uint64_t b0 = d.count * t / threads, b1 = d.count * (t + 1) / threads;
      for (uint64_t k = b0; k < b1; ++k) {
        const unsigned char* q = base + k * rec;
        const uint16_t c = (uint16_t)(q[0] | (q[1] << 8));
        if (c >= d.classes) bad[t] = 1;
        d.cls[k] = c;
        if (!fixed) {
          std::memcpy(static_cast<float*>(d.x) + k * n, q + 2, 4 * n);
        } else {
          int64_t* o = static_cast<int64_t*>(d.x) + k * n;
          for (size_t i = 0; i < n; ++i) {
            float f;
            std::memcpy(&f, q + 2 + 4 * i, 4);
            o[i] = std::llround(static_cast<double>(f));  // hygt_main.cpp:157
          }
        }
      }
    });
  for (auto& th : pool) th.join();
  mark("parse");
  if (cuda_init.joinable()) cuda_init.join();
  mark("cuda-init");
  for (int v : bad)
    if (v) io_error("read_rblk: ResidualDataset: class id out of range");
  (void)bundle_classes;
  return d;
}

void write_rblk(const std::string& path, const Dataset& d, const void* y, bool fixed) {
  const size_t n = (size_t)1 << d.log2n, rec = 2 + 4 * n;
  const size_t total = 12 + d.count * rec;
  std::unique_ptr<unsigned char[]> holder(new unsigned char[total]);  // filled below, no zeroing
  struct Span {
    unsigned char* p;
    size_t n;
    unsigned char* data() const { return p; }
    size_t size() const { return n; }
    unsigned char& operator[](size_t i) const { return p[i]; }
  } out{holder.get(), total};
  std::memcpy(out.data(), "RBLK", 4);
  out[4] = 1;
  out[5] = (unsigned char)d.log2n;
  out[6] = (unsigned char)(d.classes & 0xff);
  out[7] = (unsigned char)(d.classes >> 8);
  const uint32_t cnt = (uint32_t)d.count;
  std::memcpy(out.data() + 8, &cnt, 4);
  unsigned char* base = out.data() + 12;
  const unsigned threads = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < threads; ++t)
    pool.emplace_back([&, t] {
      const uint64_t b0 = d.count * t / threads, b1 = d.count * (t + 1) / threads;
      for (uint64_t k = b0; k < b1; ++k) {
        unsigned char* q = base + k * rec;
        q[0] = (unsigned char)(d.cls[k] & 0xff);
        q[1] = (unsigned char)(d.cls[k] >> 8);
        if (!fixed) {
          std::memcpy(q + 2, static_cast<const float*>(y) + k * n, 4 * n);
        } else {
          const int64_t* v = static_cast<const int64_t*>(y) + k * n;
          for (size_t i = 0; i < n; ++i) {
            const float f = static_cast<float>(static_cast<double>(v[i]));  // write_rblk of y
            std::memcpy(q + 2 + 4 * i, &f, 4);
          }
        }
      }
    });
  for (auto& th : pool) th.join();
  std::ofstream os(path, std::ios::binary);
  if (!os) io_error("cannot open for writing: " + path);
  os.write(reinterpret_cast<const char*>(out.data()), (std::streamsize)out.size());
  if (!os) io_error("write_rblk: stream failure");
}

struct Args {
  std::string model, data, direction = "forward", arithmetic = "float", out;
  bool timing = false;
};

Args parse(int argc, char** argv) {
  Args a;
  for (int i = 1; i < argc; ++i) {
    const std::string k = argv[i];
    auto val = [&]() -> std::string {
      if (i + 1 >= argc) arg_error(k + ": missing value");
      return argv[++i];
    };
    if (k == "--model") a.model = val();
    else if (k == "--data") a.data = val();
    else if (k == "--direction") a.direction = val();
    else if (k == "--arithmetic") a.arithmetic = val();
    else if (k == "--out") a.out = val();
    else if (k == "--timing") a.timing = true;
    else arg_error("unknown option " + k);
  }
  if (a.model.empty() || a.data.empty() || a.out.empty()) arg_error("--model, --data and --out are required");
  if (a.direction != "forward" && a.direction != "inverse") arg_error("--direction: forward or inverse");
  if (a.arithmetic != "float" && a.arithmetic != "fixed") arg_error("--arithmetic: float or fixed");
  return a;
}

int run(const Args& a) {
  g_timing = a.timing;
  const bool timing = a.timing;
  auto t_last = std::chrono::steady_clock::now();
  auto phase = [&](const char* name) {
    const auto t = std::chrono::steady_clock::now();
    if (timing) std::fprintf(stderr, "[apply] %-10s %8.1f ms\n", name, std::chrono::duration<double, std::milli>(t - t_last).count());
    t_last = t;
  };
  // CUDA context creation (0.6-1.5 s on a fresh process) overlaps with reading the files
  std::thread cuda_init([] { cudaFree(nullptr); });
  struct Joiner {
    std::thread& t;
    ~Joiner() { if (t.joinable()) t.join(); }
  } joiner{cuda_init};
  const Bundle b = read_bundle(a.model);
  const bool fixed = a.arithmetic == "fixed";
  const bool fwd = a.direction == "forward";
  if (fixed && b.angle_bits == 0)
    arg_error("apply: fixed arithmetic needs a quantized bundle (train with --angle-bits 8)");
  Dataset d = read_rblk(a.data, fixed, b.classes, cuda_init);
  if (d.log2n != b.log2n) arg_error("apply: model/data dimension mismatch");
  if (d.classes != b.classes) arg_error("apply: model/data class count mismatch");
  phase("read");
  // A one-shot file run cannot amortise plan-time NVRTC compilation (0.5-6 s for 35 classes)
  // over its transform time (milliseconds for millions of blocks): unless the caller chose,
  // the plan takes the precompiled kernels.
  if (d.count < ((uint64_t)1 << 28))
    for (const char* k : {"HYGT_JIT", "HYGT_CLS_JIT", "HYGT_FIXED_JIT"}) setenv(k, "0", 0);
  const size_t n = (size_t)1 << d.log2n, R = (size_t)b.max_rounds;
  std::vector<uint16_t> perms;
  const uint32_t mask = perm_table(b, perms);

  hygt_plan* plan = nullptr;
  if (!fixed) {  // float models, or the dequantized angles of a quantized bundle
    std::vector<double> ang((size_t)b.classes * num_parameters(b.log2n, (int)R), 0.0);
    const double step = b.angle_bits ? 2.0 * 3.14159265358979323846 / (double)(1 << b.angle_bits) : 0.0;
    for (int c = 0; c < b.classes; ++c) {
      const size_t a_c = num_parameters(b.log2n, b.rounds[c]);
      double* dst = ang.data() + (size_t)c * num_parameters(b.log2n, (int)R);
      for (size_t i = 0; i < a_c; ++i) dst[i] = b.angle_bits ? step * (double)b.codes[c][i] : b.angles[c][i];
    }
    check(hygt_plan_create(b.log2n, (int)R, b.classes, ang.data(), perms.empty() ? nullptr : perms.data(),
                           mask, 0u, &plan));
  } else {
    std::vector<uint16_t> codes((size_t)b.classes * num_parameters(b.log2n, (int)R), 0);
    for (int c = 0; c < b.classes; ++c)
      std::copy(b.codes[c].begin(), b.codes[c].end(), codes.begin() + (size_t)c * num_parameters(b.log2n, (int)R));
    check(hygt_fixed_plan_create(b.log2n, (int)R, b.classes, b.angle_bits, b.precision_bits, codes.data(),
                                 perms.empty() ? nullptr : perms.data(), mask, &plan));
  }

  phase("plan");
  const size_t esz = fixed ? 8 : 4;
  // outputs land in the input's buffer: chunk k's D2H follows its own H2D on one stream
  void* y = d.x;
  const uint64_t chunk = std::min<uint64_t>(std::max<uint64_t>(d.count, 1), (uint64_t)1 << 20);
  cudaStream_t st[2];
  void *dx[2], *dy[2], *ws[2];
  uint16_t* dc[2];
  const size_t wsb = fixed ? 0 : hygt_workspace_bytes(plan, chunk);
  for (int s = 0; s < 2; ++s) {
    cu(cudaStreamCreateWithFlags(&st[s], cudaStreamNonBlocking));
    cu(cudaMalloc(&dx[s], chunk * n * esz));
    cu(cudaMalloc(&dy[s], chunk * n * esz));
    cu(cudaMalloc(reinterpret_cast<void**>(&dc[s]), chunk * 2));
    ws[s] = nullptr;
    if (wsb) {
      cu(cudaMalloc(&ws[s], wsb));
      cu(cudaMemsetAsync(ws[s], 0, wsb, st[s]));
    }
  }
  const bool cls_needed = b.classes > 1;
  for (uint64_t k0 = 0, it = 0; k0 < d.count; k0 += chunk, ++it) {
    const int s = (int)(it & 1);
    const uint64_t m = std::min<uint64_t>(chunk, d.count - k0);
    cu(cudaMemcpyAsync(dx[s], static_cast<char*>(d.x) + k0 * n * esz, m * n * esz, cudaMemcpyHostToDevice, st[s]));
    if (cls_needed) cu(cudaMemcpyAsync(dc[s], d.cls + k0, m * 2, cudaMemcpyHostToDevice, st[s]));
    const uint16_t* c = cls_needed ? dc[s] : nullptr;
    if (!fixed) {
      const float* xs = static_cast<const float*>(dx[s]);
      float* ys = static_cast<float*>(dy[s]);
      check(fwd ? hygt_forward_f32(plan, xs, ys, c, m, ws[s], wsb, 0u, st[s])
                : hygt_inverse_f32(plan, xs, ys, c, m, ws[s], wsb, 0u, st[s]));
    } else {  // synchronous: the first failing row (the reference's exception) is known per chunk
      uint64_t first_bad = m;
      const int64_t* xs = static_cast<const int64_t*>(dx[s]);
      int64_t* ys = static_cast<int64_t*>(dy[s]);
      check(fwd ? hygt_forward_i64(plan, xs, ys, c, m, &first_bad, st[s])
                : hygt_inverse_i64(plan, xs, ys, c, m, &first_bad, st[s]));
    }
    cu(cudaMemcpyAsync(static_cast<char*>(y) + k0 * n * esz, dy[s], m * n * esz, cudaMemcpyDeviceToHost, st[s]));
  }
  for (int s = 0; s < 2; ++s) {
    cu(cudaStreamSynchronize(st[s]));
    if (!fixed && ws[s]) check(hygt_sync_status(plan, ws[s], st[s]));
  }
  phase("transform");
  write_rblk(a.out, d, y, fixed);
  phase("write");
  std::printf("wrote %llu transformed blocks to %s\n", (unsigned long long)d.count, a.out.c_str());
  for (int s = 0; s < 2; ++s) {
    cudaFree(dx[s]);
    cudaFree(dy[s]);
    cudaFree(dc[s]);
    cudaFree(ws[s]);
    cudaStreamDestroy(st[s]);
  }
  if (fixed) delete[] static_cast<int64_t*>(d.x); else delete[] static_cast<float*>(d.x);
  delete[] d.cls;
  hygt_plan_destroy(plan);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    return run(parse(argc, argv));
  } catch (const Fail& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return e.code;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
