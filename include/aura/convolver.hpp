// Drop-in for the reference's aura/convolver.hpp (convolver.hpp:1-222):
// same aura::Convolver API, argument meaning, error codes and streaming
// guarantee, with the whole block loop (r2c, FDL, partitioned MAC, c2r +
// overlap-save) on the B200 through the C-ABI (include/aura_b200.h).
// engine.hpp / dft.hpp still come from the reference.
#pragma once

#include <complex>
#include <memory>
#include <optional>
#include <span>
#include <vector>

#include "aura/backend.hpp"
#include "aura/dft.hpp"
#include "aura/engine.hpp"

namespace aura {

/// convolver.hpp:19-46 on the host (kept for API completeness; the engine
/// itself partitions on the GPU and mirrors the spectra lazily).
inline PartitionedFilterSet make_partitioned_filters(std::span<const std::vector<float>> filters,
                                                     std::size_t block_size,
                                                     const DftPlan& plan) {
  if (filters.empty()) raise(ErrorCode::empty_filter, "need at least one filter");
  const std::size_t n_h = filters.front().size();
  if (n_h == 0) raise(ErrorCode::empty_filter, "filters must have at least one tap");
  for (const auto& f : filters)
    if (f.size() != n_h)
      raise(ErrorCode::filter_length_mismatch, "all filters must share one length");
  PartitionedFilterSet set(filters.size(), n_h, block_size);
  std::vector<float> window(plan.size());
  DftWorkspace ws(plan);
  for (std::size_t c = 0; c < filters.size(); ++c)
    for (std::size_t k = 0; k < set.partition_count(); ++k) {
      std::fill(window.begin(), window.end(), 0.0f);
      const std::size_t first = k * block_size;
      const std::size_t count = std::min(block_size, n_h - first);
      for (std::size_t t = 0; t < count; ++t) window[t] = filters[c][first + t];
      plan.forward(window, set.spectrum(c, k), ws);
    }
  return set;
}

class Auralizer;

class Convolver {
 public:
  Convolver(std::span<const std::vector<float>> filters, const EngineConfig& cfg,
            ChannelMode mode, std::shared_ptr<ExecutionBackend> backend = nullptr)
      : cfg_(validate_config(cfg)), mode_(mode), backend_(b200_detail::resolve(backend)) {
    // convolver.hpp:22-30 then :84-93, same precedence
    if (filters.empty()) raise(ErrorCode::empty_filter, "need at least one filter");
    n_h_ = filters.front().size();
    if (n_h_ == 0) raise(ErrorCode::empty_filter, "filters must have at least one tap");
    for (const auto& f : filters)
      if (f.size() != n_h_)
        raise(ErrorCode::filter_length_mismatch, "all filters must share one length");
    if (mode == ChannelMode::broadcast && cfg_.input_channels != 1)
      raise(ErrorCode::mode_channel_mismatch, "broadcast mode requires one input channel");
    if (mode == ChannelMode::elementwise && cfg_.input_channels != cfg_.output_channels)
      raise(ErrorCode::mode_channel_mismatch,
            "elementwise mode requires input channels == output channels");
    if (filters.size() != cfg_.output_channels)
      raise(ErrorCode::mode_channel_mismatch,
            "filter count must equal the configured output channels");
    const int device = b200_detail::device_of(backend_);
    const auto rows = b200_detail::row_pointers(filters);
    const auto c = b200_detail::to_c(cfg_);
    aura_b200_engine* e = nullptr;
    b200_detail::check(aura_b200_convolver_create(
        &c, mode == ChannelMode::broadcast ? AURA_B200_BROADCAST : AURA_B200_ELEMENTWISE,
        rows.data(), rows.size(), n_h_, device, &e));
    engine_.reset(e);
    partitions_ = aura_b200_partition_count(e);
  }

  const EngineConfig& config() const noexcept { return cfg_; }
  ChannelMode mode() const noexcept { return mode_; }
  std::size_t partition_count() const noexcept { return partitions_; }
  std::size_t filter_length() const noexcept { return n_h_; }
  std::uint64_t blocks_processed() const noexcept {
    return engine_ ? aura_b200_blocks_processed(engine_.get()) : 0;
  }
  /// Host mirror of the device spectra, copied back on first use.
  const PartitionedFilterSet& filters() const {
    if (!filters_) {
      filters_.emplace(cfg_.output_channels, n_h_, cfg_.block_size);
      for (std::size_t c = 0; c < cfg_.output_channels; ++c)
        for (std::size_t k = 0; k < partitions_; ++k)
          b200_detail::check(aura_b200_filter_spectrum(
              engine_.get(), c, k, reinterpret_cast<float*>(filters_->spectrum(c, k).data())));
    }
    return *filters_;
  }
  /// Host mirror of the device FDL at the time of the call.
  const FrequencyDelayLine& delay_line() const {
    const std::size_t ch = mode_ == ChannelMode::broadcast ? 1 : cfg_.output_channels;
    fdl_.emplace(ch, partitions_, cfg_.bins());
    std::vector<std::complex<float>> s(cfg_.bins());
    for (std::size_t c = 0; c < ch; ++c)
      for (std::size_t age = partitions_; age-- > 0;) {
        b200_detail::check(aura_b200_fdl_slot(engine_.get(), 0, c, age,
                                              reinterpret_cast<float*>(s.data())));
        fdl_->push(c, s);
      }
    return *fdl_;
  }
  const ExecutionBackend& backend() const noexcept { return *backend_; }

  /// convolver.hpp:111-123
  void process(const AudioBlock& input, AudioBlock& output) {
    if (input.channels() != cfg_.input_channels ||
        input.samples_per_channel() != cfg_.block_size)
      raise(ErrorCode::shape_mismatch, "input block must be input_channels x block_size");
    if (output.channels() != cfg_.output_channels ||
        output.samples_per_channel() != cfg_.block_size)
      raise(ErrorCode::shape_mismatch, "output block must be output_channels x block_size");
    if (!all_finite(input)) raise(ErrorCode::non_finite_input, "input contains NaN or Inf");
    b200_detail::check(aura_b200_process(engine_.get(), input.data().data(), output.data().data()));
  }

  AudioBlock convolve(const AudioBlock& input) {
    AudioBlock output(cfg_.output_channels, cfg_.block_size);
    process(input, output);
    return output;
  }

  /// convolver.hpp:133-142
  void reset() { b200_detail::check(aura_b200_reset(engine_.get())); }

  /// The C-ABI handle (measurement / integration code).
  aura_b200_engine* native_handle() const noexcept { return engine_.get(); }

 private:
  friend class Auralizer;
  struct ViewTag {};
  // Metadata-only view of one stage of a fused Auralizer engine
  // (Auralizer::synthesis() / feedback_canceller()).
  Convolver(ViewTag, const EngineConfig& cfg, ChannelMode mode, std::size_t K, std::size_t n_h,
            std::shared_ptr<ExecutionBackend> backend)
      : cfg_(cfg), mode_(mode), backend_(std::move(backend)), n_h_(n_h), partitions_(K) {}

  EngineConfig cfg_;
  ChannelMode mode_;
  std::shared_ptr<ExecutionBackend> backend_;
  std::size_t n_h_ = 0;
  std::size_t partitions_ = 0;
  b200_detail::EnginePtr engine_;
  mutable std::optional<PartitionedFilterSet> filters_;
  mutable std::optional<FrequencyDelayLine> fdl_;
};

}  // namespace aura
