// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY. Exposes the UNMODIFIED reference
// (header-only C++20 library under /root/reference/proj/include, included at
// build time, never copied) through a flat C interface so that tests/ and
// bench.py's reference / cpu_baseline legs can drive it with ctypes.
//
// Built by oracle/Makefile into oracle/_ref/libaura_ref.so (git-ignored, but
// it travels to the GPU box with the gpurun snapshot).
//
// Entry points map 1:1 to the reference API:
//   ref_conv_*  aura::Convolver         convolver.hpp:65-220
//   ref_aur_*   aura::Auralizer         auralizer.hpp:25-123
//   ref_direct_convolve                 oracle.hpp:15-27
//   ref_verify                          verify.hpp:110-210
//   ref_backend_workers                 backend.hpp:157-181 (descriptor detail)
#include <aura/aura.hpp>

#include <cstring>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

namespace {

thread_local std::string g_last_error;
thread_local int g_last_code = 0;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const aura::Error& e) {
    g_last_error = e.what();
    g_last_code = 1 + static_cast<int>(e.code());
    return g_last_code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    g_last_code = 1000;
    return g_last_code;
  }
}

std::vector<std::vector<float>> rows(const float* data, std::size_t n_rows,
                                     std::size_t n_cols) {
  std::vector<std::vector<float>> out(n_rows);
  for (std::size_t r = 0; r < n_rows; ++r)
    out[r].assign(data + r * n_cols, data + (r + 1) * n_cols);
  return out;
}

struct RefConv {
  std::unique_ptr<aura::Convolver> conv;
  aura::AudioBlock in, out;
};

struct RefAur {
  std::unique_ptr<aura::Auralizer> aur;
  aura::AudioBlock mic, spk;
};

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_last_error.c_str(); }

int ref_conv_new(std::size_t block, std::size_t inputs, std::size_t outputs,
                 int mode, const float* filters, std::size_t n_rows,
                 std::size_t n_h, const char* backend, void** out) {
  return guarded([&] {
    auto r = std::make_unique<RefConv>();
    const auto cfg = aura::make_config(48000, block, inputs, outputs);
    const auto f = rows(filters, n_rows, n_h);
    r->conv = std::make_unique<aura::Convolver>(
        f, cfg, mode == 0 ? aura::ChannelMode::broadcast
                          : aura::ChannelMode::elementwise,
        aura::make_backend(backend));
    r->in = aura::AudioBlock(inputs, block);
    r->out = aura::AudioBlock(outputs, block);
    *out = r.release();
  });
}

int ref_conv_process(void* h, const float* in, float* out) {
  auto* r = static_cast<RefConv*>(h);
  return guarded([&] {
    std::memcpy(r->in.data().data(), in, r->in.data().size_bytes());
    r->conv->process(r->in, r->out);
    std::memcpy(out, r->out.data().data(), r->out.data().size_bytes());
  });
}

void ref_conv_reset(void* h) { static_cast<RefConv*>(h)->conv->reset(); }
std::size_t ref_conv_partitions(void* h) {
  return static_cast<RefConv*>(h)->conv->partition_count();
}
void ref_conv_spectrum(void* h, std::size_t c, std::size_t k, float* out) {
  const auto s = static_cast<RefConv*>(h)->conv->filters().spectrum(c, k);
  std::memcpy(out, s.data(), s.size_bytes());
}
void ref_conv_free(void* h) { delete static_cast<RefConv*>(h); }

int ref_aur_new(std::size_t block, std::size_t outputs, const float* synth,
                std::size_t n_h, const float* fc, std::size_t n_hf, float gain,
                const char* backend, void** out) {
  return guarded([&] {
    auto r = std::make_unique<RefAur>();
    const auto cfg = aura::make_config(48000, block, 1, outputs);
    r->aur = std::make_unique<aura::Auralizer>(
        rows(synth, outputs, n_h), rows(fc, outputs, n_hf), cfg,
        aura::make_backend(backend), gain);
    r->mic = aura::AudioBlock(1, block);
    r->spk = aura::AudioBlock(outputs, block);
    *out = r.release();
  });
}

int ref_aur_process(void* h, const float* mic, float* spk) {
  auto* r = static_cast<RefAur*>(h);
  return guarded([&] {
    std::memcpy(r->mic.data().data(), mic, r->mic.data().size_bytes());
    r->aur->process(r->mic, r->spk);
    std::memcpy(spk, r->spk.data().data(), r->spk.data().size_bytes());
  });
}

void ref_aur_estimate(void* h, float* out) {
  const auto e = static_cast<RefAur*>(h)->aur->feedback_estimate();
  std::memcpy(out, e.data(), e.size_bytes());
}
void ref_aur_reset(void* h) { static_cast<RefAur*>(h)->aur->reset(); }
void ref_aur_free(void* h) { delete static_cast<RefAur*>(h); }

int ref_forward(std::size_t n_f, const float* buf, float* spec) {
  return guarded([&] {
    aura::DftPlan plan(n_f);
    aura::DftWorkspace ws(plan);
    plan.forward(std::span<const float>(buf, n_f),
                 std::span<std::complex<float>>(
                     reinterpret_cast<std::complex<float>*>(spec), n_f / 2 + 1),
                 ws);
  });
}

int ref_inverse(std::size_t n_f, const float* spec, float* buf) {
  return guarded([&] {
    aura::DftPlan plan(n_f);
    aura::DftWorkspace ws(plan);
    plan.inverse_unchecked(
        std::span<const std::complex<float>>(
            reinterpret_cast<const std::complex<float>*>(spec), n_f / 2 + 1),
        std::span<float>(buf, n_f), ws);
  });
}

void ref_direct_convolve(const double* x, std::size_t nx, const double* h,
                         std::size_t nh, double* y) {
  const auto r = aura::oracle::direct_convolve(std::span<const double>(x, nx),
                                               std::span<const double>(h, nh));
  std::memcpy(y, r.data(), r.size() * sizeof(double));
}

std::size_t ref_partition_count(std::size_t n_h, std::size_t n_x) {
  return aura::partition_count(n_h, n_x);
}

unsigned ref_backend_workers(const char* backend) {
  auto b = aura::make_backend(backend);
  return static_cast<unsigned>(std::stoul(b->descriptor().detail == "single-threaded"
                                              ? std::string("1")
                                              : b->descriptor().detail));
}

// verify::run on the small or full grid; log text copied into buf.
int ref_verify(int full, char* buf, std::size_t cap) {
  std::ostringstream log;
  aura::verify::Options opts;
  opts.grid = full ? aura::verify::Grid::full : aura::verify::Grid::small;
  const bool ok = aura::verify::run(opts, log);
  const std::string s = log.str();
  const std::size_t n = s.size() < cap - 1 ? s.size() : cap - 1;
  std::memcpy(buf, s.data(), n);
  buf[n] = 0;
  return ok ? 0 : 1;
}

}  // extern "C"
