// diag.cu -- the measurement and diagnostics C-ABI of libaura_b200.so
// (include/aura_b200_diag.h): device- and host-timed block runs, per-phase
// timing and the roofline denominator, %globaltimer timelines, launch-mode
// and block-numbering controls. Not part of the reference-replacing
// boundary; bench.py and tools/ use it.
#include "engine.hpp"

extern "C" {

int aura_b200_seek_block(aura_b200_engine* e, uint64_t n) {
  return guarded([&] {
    if (e->blocks) fail(AURA_B200_E_INVALID_ARGUMENT, "seek only before the first block (or after reset)");
    if (e->G > 1) fail(AURA_B200_E_INVALID_ARGUMENT, "seek does not apply to sharded engines");
    CK(cudaSetDevice(e->device));
    CK(cudaStreamSynchronize(e->stream));
    // every delay line is zero here, so starting the ring slots (block mod
    // K) at n instead of 0 changes no value
    DevState st{};
    st.block = n;
    CK(cudaMemcpy(e->args.st, &st, sizeof(st), cudaMemcpyHostToDevice));
    e->block_base = n;
  });
}

int aura_b200_set_launch_mode(aura_b200_engine* e, int mode) {
  return guarded([&] {
    if (mode < 0 || mode > 1)
      fail(AURA_B200_E_INVALID_ARGUMENT, "launch mode is 0 (one CUDA graph per block) or 1 (kernels on the stream)");
    CK(cudaSetDevice(e->device));
    CK(cudaStreamSynchronize(e->stream));
    e->launch_mode = mode;
  });
}

int aura_b200_launch_mode(const aura_b200_engine* e) { return e->launch_mode; }


// Device-resident timing. block_us[b]: back-to-back block time, CUDA events
// recorded on the engine stream between consecutive block graphs (so a
// block's interval spans all of its kernels and the launch of the next).
// latency_us[b] (optional, separate pass): block start -> output written,
// from the graph's external event node after k_front.
int aura_b200_time_device_blocks(aura_b200_engine* e, const float* host_in,
                                 size_t n_in_blocks, size_t blocks, float* latency_us,
                                 float* block_us) {
  return guarded([&] {
    CK(cudaSetDevice(e->device));
    CK(cudaStreamSynchronize(e->stream));
    const size_t per = (size_t)e->Qx * e->N;
    if (host_in && n_in_blocks) {
      const size_t nb = std::min(n_in_blocks, e->pool_blocks);
      CK(cudaMemcpy(e->d_in_pool, host_in, nb * per * sizeof(float), cudaMemcpyHostToDevice));
    }
    // one block graph per pool slot (the input pointer is baked per slot);
    // graph mode: block b's own graph records ev[b + 1] after its last
    // kernel (an event node re-pointed per launch), so nothing is inserted
    // between two block graphs; stream mode: events between the blocks
    const size_t slots = std::max<size_t>(1, std::min(n_in_blocks, e->pool_blocks));
    const bool in_graph = e->launch_mode == 0;
    std::vector<cudaEvent_t> ev(blocks + 1);
    for (auto& x : ev) CK(cudaEventCreate(&x));
    std::vector<aura_b200_engine::BlockGraph> gs;
    for (size_t s = 0; s < slots; ++s) {
      BlockArgs a = e->dev_args;
      a.in = e->d_in_pool + s * per;
      gs.push_back(e->capture_block(a, nullptr, in_graph ? ev[0] : nullptr));
    }
    std::vector<BlockArgs> sa(slots, e->dev_args);
    for (size_t s = 0; s < slots; ++s) sa[s].in = e->d_in_pool + s * per;
    CK(cudaEventRecord(ev[0], e->stream));
    for (size_t b = 0; b < blocks; ++b) {
      auto& g = gs[b % slots];
      if (in_graph) {
        CK(cudaGraphExecEventRecordNodeSetEvent(g.ex, g.end_node, ev[b + 1]));
        CK(cudaGraphLaunch(g.ex, e->stream));
      } else {
        if (b) CK(cudaEventRecord(ev[b], e->stream));
        e->enqueue_block(g, sa[b % slots], nullptr);
      }
    }
    if (!in_graph) CK(cudaEventRecord(ev[blocks], e->stream));
    CK(cudaStreamSynchronize(e->stream));
    for (size_t b = 0; b < blocks; ++b) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, ev[b], ev[b + 1]));
      block_us[b] = ms * 1000.0f;
    }
    for (auto& g : gs) g.destroy();
    e->blocks += blocks;
    if (latency_us) {
      // separate pass: the output-ready event node is re-pointed per block
      cudaEvent_t proto;
      CK(cudaEventCreate(&proto));
      std::vector<aura_b200_engine::BlockGraph> gl;
      for (size_t s = 0; s < slots; ++s) {
        BlockArgs a = e->dev_args;
        a.in = e->d_in_pool + s * per;
        gl.push_back(e->capture_block(a, proto));
      }
      std::vector<cudaEvent_t> ev2(2 * blocks);
      for (auto& x : ev2) CK(cudaEventCreate(&x));
      for (size_t b = 0; b < blocks; ++b) {
        auto& g = gl[b % slots];
        CK(cudaGraphExecEventRecordNodeSetEvent(g.ex, g.out_node, ev2[2 * b + 1]));
        CK(cudaEventRecord(ev2[2 * b], e->stream));
        CK(cudaGraphLaunch(g.ex, e->stream));
      }
      CK(cudaStreamSynchronize(e->stream));
      for (size_t b = 0; b < blocks; ++b) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, ev2[2 * b], ev2[2 * b + 1]));
        latency_us[b] = ms * 1000.0f;
      }
      for (auto& x : ev2) cudaEventDestroy(x);
      for (auto& g : gl) g.destroy();
      cudaEventDestroy(proto);
      e->blocks += blocks;
    }
    for (auto& x : ev) cudaEventDestroy(x);
  });
}

// Device-resident blocks back to back with ONE event pair around all of
// them: the mean block time without per-block event records in the stream.
int aura_b200_time_device_span(aura_b200_engine* e, const float* host_in, size_t n_in_blocks,
                               size_t blocks, float* total_us) {
  return guarded([&] {
    CK(cudaSetDevice(e->device));
    CK(cudaStreamSynchronize(e->stream));
    const size_t per = (size_t)e->Qx * e->N;
    const size_t slots = std::max<size_t>(1, std::min(n_in_blocks, e->pool_blocks));
    if (host_in && n_in_blocks)
      CK(cudaMemcpy(e->d_in_pool, host_in, slots * per * sizeof(float), cudaMemcpyHostToDevice));
    std::vector<aura_b200_engine::BlockGraph> gs;
    std::vector<BlockArgs> sa(slots, e->dev_args);
    for (size_t s = 0; s < slots; ++s) {
      sa[s].in = e->d_in_pool + s * per;
      gs.push_back(e->capture_block(sa[s], nullptr));
    }
    cudaEvent_t t0, t1;
    CK(cudaEventCreate(&t0));
    CK(cudaEventCreate(&t1));
    CK(cudaEventRecord(t0, e->stream));
    for (size_t b = 0; b < blocks; ++b) e->enqueue_block(gs[b % slots], sa[b % slots], nullptr);
    CK(cudaEventRecord(t1, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, t0, t1));
    *total_us = ms * 1000.0f;
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
    for (auto& g : gs) g.destroy();
    e->blocks += blocks;
  });
}

int aura_b200_time_host_blocks(aura_b200_engine* e, const float* host_in,
                               size_t n_in_blocks, size_t blocks, double pace_us,
                               float* block_us) {
  if (!e || !host_in || !n_in_blocks || !block_us) {
    g_err = "null argument";
    return AURA_B200_E_INVALID_ARGUMENT;
  }
  const size_t per = (size_t)e->Qx * e->N;
  std::vector<float> out(e->L * e->N);
  using clk = std::chrono::steady_clock;
  auto next = clk::now();
  for (size_t b = 0; b < blocks; ++b) {
    if (pace_us > 0) {
      while (clk::now() < next) {
#if defined(__x86_64__)
        _mm_pause();
#endif
      }
      next += std::chrono::nanoseconds((long long)(pace_us * 1000.0));
    }
    const auto t0 = clk::now();
    const int rc = aura_b200_process(e, host_in + (b % n_in_blocks) * per, out.data());
    const auto t1 = clk::now();
    if (rc) return rc;
    block_us[b] = (float)std::chrono::duration<double, std::micro>(t1 - t0).count();
  }
  return AURA_B200_OK;
}

// Diagnostics: where the host-visible latency of process() goes (graph
// mode). Per block (optionally paced), steady_clock offsets in us from the
// call's start: {input staged, graph launched, background event recorded,
// output flag seen, output copied}.
int aura_b200_time_host_breakdown(aura_b200_engine* e, const float* host_in, size_t n_in_blocks,
                                  size_t blocks, double pace_us, double* out) {
  return guarded([&] {
    if (e->launch_mode != 0) fail(AURA_B200_E_INVALID_ARGUMENT, "graph mode only");
    CK(cudaSetDevice(e->device));
    const size_t per = (size_t)e->Qx * e->N;
    std::vector<float> y(e->L * e->N);
    using clk = std::chrono::steady_clock;
    auto next = clk::now();
    for (size_t b = 0; b < blocks; ++b) {
      if (pace_us > 0) {
        while (clk::now() < next) {
#if defined(__x86_64__)
          _mm_pause();
#endif
        }
        next += std::chrono::nanoseconds((long long)(pace_us * 1000.0));
      }
      const auto t0 = clk::now();
      auto us = [&](clk::time_point t) { return std::chrono::duration<double, std::micro>(t - t0).count(); };
      std::memcpy(e->h_in, host_in + (b % n_in_blocks) * per, per * sizeof(float));
      std::atomic_thread_fence(std::memory_order_release);
      const auto t1 = clk::now();
      const uint64_t nblk = device_block_hint(e);
      CK(cudaGraphLaunch(e->g_block.ex, e->stream));
      const auto t2 = clk::now();
      const auto t3 = t2;  // (no background event any more)
      wait_flag(e, nblk + 1, "block output");
      const auto t4 = clk::now();
      std::memcpy(y.data(), e->h_out, y.size() * sizeof(float));
      const auto t5 = clk::now();
      ++e->blocks;
      double* o = out + 5 * b;
      o[0] = us(t1);
      o[1] = us(t2);
      o[2] = us(t3);
      o[3] = us(t4);
      o[4] = us(t5);
    }
    CK(cudaStreamSynchronize(e->stream));
  });
}

int aura_b200_profile_phases(aura_b200_engine* e, size_t blocks, float* phase_us,
                             int* n_phases) {
  return guarded([&] {
    CK(cudaSetDevice(e->device));
    CK(cudaStreamSynchronize(e->stream));
    const int np = PH_COUNT;
    std::vector<cudaEvent_t> ev((size_t)(np + 1) * blocks);
    for (auto& x : ev) CK(cudaEventCreate(&x));
    for (size_t b = 0; b < blocks; ++b) {
      BlockArgs a = e->dev_args;
      a.in = e->d_in_pool + (b % e->pool_blocks) * (size_t)e->Qx * e->N;
      for (int ph = 0; ph < np; ++ph) {
        CK(cudaEventRecord(ev[b * (np + 1) + ph], e->stream));
        e->launch_phase(ph, a, e->stream);
      }
      CK(cudaEventRecord(ev[b * (np + 1) + np], e->stream));
    }
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(e->stream));
    for (int ph = 0; ph < np; ++ph) {
      double s = 0;
      for (size_t b = 0; b < blocks; ++b) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, ev[b * (np + 1) + ph], ev[b * (np + 1) + ph + 1]));
        s += ms;
      }
      phase_us[ph] = (float)(1000.0 * s / (double)blocks);
    }
    for (auto& x : ev) cudaEventDestroy(x);
    *n_phases = np;
    e->blocks += blocks;
  });
}

int aura_b200_time_phase(aura_b200_engine* e, int phase, size_t reps, float* avg_us) {
  return guarded([&] {
    if (phase != PH_BACK && phase != PH_FRONT && phase != PH_REDUCE)
      fail(AURA_B200_E_INVALID_ARGUMENT, "only the front, k_back and k_reduce can be re-launched");
    if (phase == PH_BACK && !e->has_back())
      fail(AURA_B200_E_INVALID_ARGUMENT, "this engine has no streaming work");
    CK(cudaSetDevice(e->device));
    CK(cudaStreamSynchronize(e->stream));
    // The relaunches are not idempotent (k_reduce advances the block
    // counter, k_back updates W in place, the fused canceller head shifts
    // the loudspeaker history): snapshot every mutable device buffer and put
    // it back afterwards, so the engine continues as if this never ran.
    const auto state = e->mutable_state();
    size_t total = 0;
    for (auto& b : state) total += (b.second + 255) & ~size_t(255);
    char* snap = nullptr;
    CK(cudaMalloc(&snap, std::max<size_t>(total, 1)));
    auto copy_all = [&](bool save) {
      size_t off = 0;
      for (auto& b : state) {
        char* s0 = snap + off;
        CK(cudaMemcpyAsync(save ? s0 : b.first, save ? b.first : s0, b.second, cudaMemcpyDeviceToDevice,
                           e->stream));
        off += (b.second + 255) & ~size_t(255);
      }
    };
    copy_all(true);
    // single launches, back to back without programmatic overlap, so the
    // mean is one launch's duration (ramp-up and tail included)
    BlockArgs a = e->dev_args;
    // k_reduce alone: its canceller CTA cannot wait for k_back's published
    // partials (k_back does not run), so it takes the griddepcontrol path
    if (phase == PH_REDUCE) a.afc_seq = nullptr;
    e->pdl_off = true;
    e->launch_phase(phase, a, e->stream);  // warm
    cudaEvent_t t0, t1;
    CK(cudaEventCreate(&t0));
    CK(cudaEventCreate(&t1));
    CK(cudaEventRecord(t0, e->stream));
    for (size_t r = 0; r < reps; ++r) e->launch_phase(phase, a, e->stream);
    CK(cudaEventRecord(t1, e->stream));
    e->pdl_off = false;
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(e->stream));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, t0, t1));
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
    *avg_us = 1000.0f * ms / (float)reps;
    copy_all(false);
    CK(cudaStreamSynchronize(e->stream));
    CK(cudaFree(snap));
  });
}

namespace {
// Timeline of `blocks` traced blocks (see aura_b200_trace_blocks). host_in:
// run them through process()'s own handshake (mapped input and output,
// output words, back to back) instead of device-resident I/O.
void trace_run(aura_b200_engine* e, size_t blocks, double* out, const float* host_in, size_t n_in) {
  CK(cudaSetDevice(e->device));
  CK(cudaStreamSynchronize(e->stream));
  blocks = std::min<size_t>(blocks, kTraceBlocks);
  const size_t words = (size_t)kTraceBlocks * kTraceKernels * 2;
  std::vector<unsigned long long> init(words);
  for (size_t i = 0; i < words; i += 2) {
    init[i] = ~0ull;
    init[i + 1] = 0ull;
  }
  unsigned long long* dtr = nullptr;
  CK(cudaMalloc(&dtr, words * sizeof(unsigned long long)));
  CK(cudaMemcpy(dtr, init.data(), words * sizeof(unsigned long long), cudaMemcpyHostToDevice));
  BlockArgs a = host_in ? e->args : e->dev_args;
  a.trace = dtr;
  unsigned long long* dflag = nullptr;  // device-side output words, so the front stamps TR_OUTPUT
  if (!host_in) {
    CK(cudaMalloc(&dflag, std::max<size_t>(1, e->n_outflags) * sizeof(unsigned long long)));
    a.out_flag = dflag;
  }
  auto g = e->capture_block(a, nullptr);
  if (host_in) {
    const size_t per = (size_t)e->Qx * e->N;
    std::vector<float> y(e->L * e->N);
    for (size_t i = 0; i < blocks; ++i) {
      std::memcpy(e->h_in, host_in + (i % n_in) * per, per * sizeof(float));
      std::atomic_thread_fence(std::memory_order_release);
      const uint64_t nblk = device_block_hint(e);
      CK(cudaGraphLaunch(g.ex, e->stream));
      wait_flag(e, nblk + 1, "traced block output");
      std::memcpy(y.data(), e->h_out, y.size() * sizeof(float));
      ++e->blocks;
    }
  } else {
    for (size_t i = 0; i < blocks; ++i) CK(cudaGraphLaunch(g.ex, e->stream));
    e->blocks += blocks;
  }
  CK(cudaStreamSynchronize(e->stream));
  std::vector<unsigned long long> tr(words);
  CK(cudaMemcpy(tr.data(), dtr, words * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  cudaFree(dtr);
  if (dflag) cudaFree(dflag);
  g.destroy();
  // out[i][k][2]: start/end in microseconds relative to block i's front
  // start; slot kTraceKernels-1 holds {next block's front start, 0}: the
  // back-to-back cycle time. The device block counter names the trace slots.
  DevState dst{};
  CK(cudaMemcpy(&dst, e->args.st, sizeof(dst), cudaMemcpyDeviceToHost));
  const uint64_t dev_first = (uint64_t)dst.block - blocks;
  for (size_t i = 0; i < blocks; ++i) {
    const size_t slot = (dev_first + i) % kTraceBlocks;
    const unsigned long long t0 = tr[(slot * kTraceKernels + TR_FRONT) * 2];
    for (int k = 0; k < kTraceKernels - 1; ++k) {
      const unsigned long long s0 = tr[(slot * kTraceKernels + k) * 2];
      const unsigned long long s1 = tr[(slot * kTraceKernels + k) * 2 + 1];
      const bool ran = s0 != ~0ull;
      out[(i * kTraceKernels + k) * 2] = ran ? (double)(long long)(s0 - t0) * 1e-3 : -1.0;
      out[(i * kTraceKernels + k) * 2 + 1] = ran ? (double)(long long)(s1 - t0) * 1e-3 : -1.0;
    }
    const size_t nslot = (dev_first + i + 1) % kTraceBlocks;
    const unsigned long long t1 = tr[(nslot * kTraceKernels + TR_FRONT) * 2];
    const bool nxt = i + 1 < blocks && t1 != ~0ull;
    out[(i * kTraceKernels + kTraceKernels - 1) * 2] = nxt ? (double)(long long)(t1 - t0) * 1e-3 : -1.0;
    out[(i * kTraceKernels + kTraceKernels - 1) * 2 + 1] = 0.0;
  }
}
}  // namespace

int aura_b200_trace_blocks(aura_b200_engine* e, size_t blocks, double* out) {
  return guarded([&] { trace_run(e, blocks, out, nullptr, 0); });
}

int aura_b200_trace_host_blocks(aura_b200_engine* e, const float* host_in, size_t n_in_blocks, size_t blocks,
                                double* out) {
  return guarded([&] {
    if (!host_in || !n_in_blocks) fail(AURA_B200_E_INVALID_ARGUMENT, "null argument");
    if (e->launch_mode != 0) fail(AURA_B200_E_INVALID_ARGUMENT, "graph mode only");
    trace_run(e, blocks, out, host_in, n_in_blocks);
  });
}

// Diagnostics: run `blocks` blocks with k_back's per-chunk / per-CTA
// %globaltimer stamps on; report the last block's, in us from k_back's
// earliest CTA start. out_segs[i] = {kind, tile, b, e, cta, start_us,
// partial_written_us, end_us} per item; out_ctas[c] = {start_us,
// first_data_us, exit_us}. Sizes via
// *n_segs / *n_ctas (call with null outputs first).
int aura_b200_trace_back(aura_b200_engine* e, size_t blocks, double* out_segs, size_t* n_segs,
                         double* out_ctas, size_t* n_ctas) {
  return guarded([&] {
    const size_t ns = e->h_chunks.size(), nc = (size_t)e->back_ctas;
    if (!out_segs || !out_ctas) {
      *n_segs = ns;
      *n_ctas = nc;
      return;
    }
    if (!e->has_back()) fail(AURA_B200_E_INVALID_ARGUMENT, "this engine has no streaming work");
    CK(cudaSetDevice(e->device));
    CK(cudaStreamSynchronize(e->stream));
    const size_t words = 4 * ns + 3 * nc;
    unsigned long long* d = nullptr;
    CK(cudaMalloc(&d, words * sizeof(unsigned long long)));
    BlockArgs a = e->dev_args;
    a.seg_trace = d;
    auto g = e->capture_block(a, nullptr);
    blocks = std::max<size_t>(1, blocks);
    for (size_t i = 0; i < blocks; ++i) CK(cudaGraphLaunch(g.ex, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    std::vector<unsigned long long> h(words);
    CK(cudaMemcpy(h.data(), d, words * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    cudaFree(d);
    g.destroy();
    unsigned long long t0 = ~0ull;
    for (size_t c = 0; c < nc; ++c) t0 = std::min(t0, h[4 * ns + 3 * c]);
    auto us = [&](unsigned long long t) { return (double)(long long)(t - t0) * 1e-3; };
    for (size_t i = 0; i < ns; ++i) {
      const int4 s = e->h_chunks[i];
      double* o = out_segs + 8 * i;
      o[0] = s.x & 1;
      o[1] = s.x >> 1;
      o[2] = s.y;
      o[3] = s.z;
      o[4] = (double)h[4 * i + 3];
      o[5] = us(h[4 * i]);
      o[6] = us(h[4 * i + 1]);
      o[7] = us(h[4 * i + 2]);
    }
    for (size_t c = 0; c < nc; ++c)
      for (int k = 0; k < 3; ++k) out_ctas[3 * c + k] = us(h[4 * ns + 3 * c + k]);
    e->blocks += blocks;
  });
}

const char* aura_b200_phase_name(const aura_b200_engine*, int phase) {
  return (phase >= 0 && phase < PH_COUNT) ? kPhaseNames[phase] : "";
}

double aura_b200_phase_bytes(const aura_b200_engine* e, int phase) { return e->phase_bytes(phase); }
int aura_b200_launches_per_block(const aura_b200_engine* e) { return e->launches_per_block(); }

int aura_b200_describe(const aura_b200_engine* e, char* buf, size_t cap) {
  return guarded([&] {
    const BlockArgs& a = e->args;
    std::snprintf(buf, cap,
                  "N=%zu Q=%zu L=%zu P=%zu K=%zu KF=%zu mode=%d LT=%d PT=%d | front: grid=%zu cpb=%d "
                  "warps=%d smem=%zu | back: ctas=%d x %d thr, CT=%d CTn=%d sp=%d spa=%d stages=%d slot=%d B "
                  "smem=%zu partials=%zu+%zu items=%d (static %d) w_l2=%d | reduce: %d+%d ctas l2keep=%d "
                  "nlms=%d cons=%d delta=%g knobs=%s",
                  e->N, e->Q, e->L, e->P, e->K, e->KF, e->mode, e->LT, e->PT,
                  (e->L + a.cpb - 1) / a.cpb, a.cpb, a.front_warps, e->smem_front, e->back_ctas, kBackThreads, a.CT,
                  a.CTn, a.sp, a.spa, a.stages, a.slot_f4 * 16, e->smem_back, e->n_syn_segs,
                  e->n_afc_segs, a.n_chunks, a.n_static, a.w_in_l2, a.red_syn_ctas, a.red_afc_ctas, a.h_in_l2,
                  a.nlms, a.afc_cons, (double)a.delta, e->knobs.empty() ? "none" : e->knobs.c_str());
  });
}

}  // extern "C"
