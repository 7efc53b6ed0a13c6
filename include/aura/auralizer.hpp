// Drop-in for the reference's aura/auralizer.hpp (auralizer.hpp:1-125):
// same aura::Auralizer API (m~ = g m - f^, l = synth(m~), f^ for the next
// block), with synthesis and the feedback canceller fused into one B200
// engine (include/aura_b200.h). Extensions: an AFC parameter overload that
// switches on the NLMS update of F^; mu = 0 (the default)
// is the reference's fixed canceller.
#pragma once

#include <memory>
#include <span>
#include <vector>

#include "aura/convolver.hpp"
#include "aura/engine.hpp"

namespace aura {

struct AfcParams {
  float mu = 0.0f;
  float lambda = 0.9f;
  float delta = 0.0f;  // 0 -> 1e-6 * block_size
  bool constrained = false;  // Appendix A step 2: constrained gradient
};

class Auralizer {
 public:
  Auralizer(std::span<const std::vector<float>> synth_filters,
            std::span<const std::vector<float>> fc_filters, const EngineConfig& cfg,
            std::shared_ptr<ExecutionBackend> backend = nullptr, float input_gain = 1.0f)
      : Auralizer(synth_filters, fc_filters, cfg, std::move(backend), input_gain, AfcParams{}) {}

  Auralizer(std::span<const std::vector<float>> synth_filters,
            std::span<const std::vector<float>> fc_filters, const EngineConfig& cfg,
            std::shared_ptr<ExecutionBackend> backend, float input_gain, const AfcParams& afc)
      : cfg_(validate_config(cfg)), backend_(b200_detail::resolve(backend)) {
    // auralizer.hpp:102-115, then both convolvers' checks
    if (cfg_.input_channels != 1)
      raise(ErrorCode::mode_channel_mismatch, "auralizer supports a single input channel");
    if (synth_filters.size() != fc_filters.size())
      raise(ErrorCode::channel_count_mismatch,
            "synthesis and feedback-cancellation filter sets must have the same channel count");
    for (auto set : {synth_filters, fc_filters}) {
      if (set.empty()) raise(ErrorCode::empty_filter, "need at least one filter");
      if (set.front().empty()) raise(ErrorCode::empty_filter, "filters must have at least one tap");
      for (const auto& f : set)
        if (f.size() != set.front().size())
          raise(ErrorCode::filter_length_mismatch, "all filters must share one length");
    }
    if (synth_filters.size() != cfg_.output_channels)
      raise(ErrorCode::mode_channel_mismatch,
            "filter count must equal the configured output channels");
    const int device = b200_detail::device_of(backend_);
    const auto s = b200_detail::row_pointers(synth_filters);
    const auto f = b200_detail::row_pointers(fc_filters);
    const auto c = b200_detail::to_c(cfg_);
    const aura_b200_afc p{afc.mu, afc.lambda,
                          afc.delta > 0.0f ? afc.delta : 1e-6f * static_cast<float>(cfg_.block_size),
                          afc.constrained ? 1 : 0};
    aura_b200_engine* e = nullptr;
    b200_detail::check(aura_b200_auralizer_create(&c, s.data(), s.size(),
                                                  synth_filters.front().size(), f.data(),
                                                  f.size(), fc_filters.front().size(), input_gain,
                                                  &p, device, &e));
    engine_.reset(e);
    estimate_.assign(cfg_.block_size, 0.0f);
    synth_view_.emplace(Convolver(Convolver::ViewTag{}, cfg_, ChannelMode::broadcast,
                                  aura_b200_partition_count(e), synth_filters.front().size(),
                                  backend_));
    fc_view_.emplace(Convolver(
        Convolver::ViewTag{},
        make_config(cfg_.sample_rate_hz, cfg_.block_size, cfg_.output_channels, cfg_.output_channels),
        ChannelMode::elementwise, aura_b200_fc_partition_count(e), fc_filters.front().size(),
        backend_));
  }

  const EngineConfig& config() const noexcept { return cfg_; }
  const Convolver& synthesis() const noexcept { return *synth_view_; }
  const Convolver& feedback_canceller() const noexcept { return *fc_view_; }
  std::size_t synth_partitions() const noexcept { return synth_view_->partition_count(); }
  std::size_t fc_partitions() const noexcept { return fc_view_->partition_count(); }

  float input_gain() const noexcept { return aura_b200_input_gain(engine_.get()); }
  void set_input_gain(float gain) { b200_detail::check(aura_b200_set_input_gain(engine_.get(), gain)); }

  /// auralizer.hpp:56-58: the estimate subtracted from the next input block.
  /// Waits for the last block's background work (which computes it) and
  /// copies it into this object's own buffer, so the span stays complete
  /// until the next process()/reset(), as the reference's does. Unlike the
  /// reference it is not noexcept: a CUDA failure or a shard-exchange
  /// timeout surfaces here as aura::Error instead of a stale estimate.
  std::span<const float> feedback_estimate() const {
    b200_detail::check(aura_b200_feedback_estimate(engine_.get(), estimate_.data()));
    return estimate_;
  }

  /// auralizer.hpp:61-87
  void process(const AudioBlock& mic, AudioBlock& speakers) {
    if (mic.channels() != 1 || mic.samples_per_channel() != cfg_.block_size)
      raise(ErrorCode::shape_mismatch, "microphone block must be 1 x block_size");
    if (!all_finite(mic)) raise(ErrorCode::non_finite_input, "microphone block contains NaN or Inf");
    if (speakers.channels() != cfg_.output_channels ||
        speakers.samples_per_channel() != cfg_.block_size)
      raise(ErrorCode::shape_mismatch, "speaker block must be output_channels x block_size");
    b200_detail::check(aura_b200_process(engine_.get(), mic.data().data(), speakers.data().data()));
  }

  AudioBlock auralize(const AudioBlock& mic) {
    AudioBlock speakers(cfg_.output_channels, cfg_.block_size);
    process(mic, speakers);
    return speakers;
  }

  void reset() { b200_detail::check(aura_b200_reset(engine_.get())); }

  aura_b200_engine* native_handle() const noexcept { return engine_.get(); }

 private:
  EngineConfig cfg_;
  std::shared_ptr<ExecutionBackend> backend_;
  b200_detail::EnginePtr engine_;
  mutable std::vector<float> estimate_;
  std::optional<Convolver> synth_view_, fc_view_;
};

}  // namespace aura
