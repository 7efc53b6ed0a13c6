/*
 * aura_b200.h -- C-ABI of the B200-native UPOLS + feedback-canceller engine
 * (libaura_b200.so, built from paper_2509_04390_b200/csrc/).
 *
 * This is the drop-in boundary for the reference's C++ aura::Convolver /
 * aura::Auralizer hot path (/root/reference/proj/include/aura/). The C++
 * drop-in headers include/aura/{convolver,auralizer,backend}.hpp re-expose
 * these entry points with the reference's class names, argument meaning and
 * exceptions; a Python mirror lives in paper_2509_04390_b200/__init__.py.
 *
 * Conventions
 *  - Every int-returning call returns AURA_B200_OK (0) or 1 + the value of
 *    the reference's aura::ErrorCode (engine.hpp:15-37), so the C++ wrapper
 *    rethrows aura::Error(code - 1, aura_b200_last_error()). GPU-specific
 *    failures use the codes appended after invalid_argument.
 *  - Audio is planar float32, channel-major (AudioBlock, engine.hpp:133-176).
 *  - Spectra handed out are in the reference layout: N + 1 complex64 bins
 *    (PartitionedFilterSet, engine.hpp:192-227). On the device they are
 *    stored packed (N complex, DC real in bin 0 .re, Nyquist real in .im).
 *  - Calls on one engine are externally serialised; engines
 *    may move between threads. process() never allocates.
 *  - There is no CPU fallback: without a usable sm_100 device create()
 *    fails with AURA_B200_E_BACKEND_UNAVAILABLE.
 */
#ifndef AURA_B200_H
#define AURA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AURA_B200_ABI_VERSION 2

/* 1 + aura::ErrorCode (engine.hpp:15-37), then GPU codes */
enum aura_b200_status {
  AURA_B200_OK = 0,
  AURA_B200_E_NON_POWER_OF_TWO_BLOCK = 1,
  AURA_B200_E_FFT_SIZE_MISMATCH = 2,
  AURA_B200_E_BAD_CHANNEL_COMBINATION = 3,
  AURA_B200_E_ZERO_SAMPLE_RATE = 4,
  AURA_B200_E_ZERO_LENGTH = 5,
  AURA_B200_E_LENGTH_MISMATCH = 6,
  AURA_B200_E_NON_REAL_EDGE_BINS = 7,
  AURA_B200_E_FILTER_LENGTH_MISMATCH = 8,
  AURA_B200_E_EMPTY_FILTER = 9,
  AURA_B200_E_MODE_CHANNEL_MISMATCH = 10,
  AURA_B200_E_CHANNEL_COUNT_MISMATCH = 11,
  AURA_B200_E_SHAPE_MISMATCH = 12,
  AURA_B200_E_NON_FINITE_INPUT = 13,
  AURA_B200_E_EMPTY_INPUT = 14,
  AURA_B200_E_UNSUPPORTED_FORMAT = 15,
  AURA_B200_E_CORRUPT_HEADER = 16,
  AURA_B200_E_SAMPLE_RATE_MISMATCH = 17,
  AURA_B200_E_BACKEND_UNAVAILABLE = 18,
  AURA_B200_E_OUT_OF_MEMORY = 19,
  AURA_B200_E_IO_ERROR = 20,
  AURA_B200_E_INVALID_ARGUMENT = 21,
  /* appended GPU codes */
  AURA_B200_E_CUDA = 22,
  AURA_B200_E_TIMEOUT = 23,
};

/* channel modes: ChannelMode (engine.hpp:283) plus the MIMO composition */
enum aura_b200_mode {
  AURA_B200_BROADCAST = 0,   /* 1 input  -> L outputs, filters[l]        */
  AURA_B200_ELEMENTWISE = 1, /* L inputs -> L outputs, filters[l]        */
  AURA_B200_MIMO = 2,        /* Q inputs -> L outputs, filters[q*L + l]  */
};

typedef struct aura_b200_engine aura_b200_engine;

/* = aura::EngineConfig (engine.hpp:64-72); fft_size must be 2*block_size */
typedef struct {
  uint32_t sample_rate_hz;
  size_t block_size;
  size_t fft_size;
  size_t inputs;
  size_t outputs;
} aura_b200_config;

/* feedback-canceller adaptation. mu = 0 -> the
 * reference's fixed-F^ canceller (auralizer.hpp:34-37). */
typedef struct {
  float mu;        /* NLMS step */
  float lambda;    /* power forgetting factor */
  float delta;     /* regulariser */
  int constrained; /* != 0: constrained gradient (Appendix A step 2: c2r, keep
                      the first N samples, r2c) -- the partitions stay linear
                      convolutions; costs a pair of transforms per unit */
} aura_b200_afc;

/* ---- library ------------------------------------------------------- */
int aura_b200_abi_version(void);
/* thread-local message of the last failing call on this thread */
const char* aura_b200_last_error(void);
/* number of usable sm_100 devices (list_backends, backend.hpp:186-193) */
int aura_b200_device_count(int* n);
/* device name into buf (BackendDescriptor::detail, backend.hpp:22) */
int aura_b200_device_name(int device, char* buf, size_t cap);

/* ---- construction -------------------------------------------------- */
/* Replaces Convolver::Convolver (convolver.hpp:67-94) incl.
 * make_partitioned_filters (convolver.hpp:19-46), done on the GPU.
 * filters: row pointers, n_h taps each (broadcast/elementwise: outputs
 * rows; mimo: inputs*outputs rows). Errors as the reference: empty_filter,
 * filter_length_mismatch is impossible here (one n_h), mode_channel_mismatch,
 * plus validate_config's codes. */
int aura_b200_convolver_create(const aura_b200_config* cfg, int mode,
                               const float* const* filters, size_t n_rows,
                               size_t n_h, int device,
                               aura_b200_engine** out);

/* Replaces Auralizer::Auralizer (auralizer.hpp:27-41). cfg.inputs = Q
 * microphones/inputs (Q > 1 is the Appendix-B MIMO generalisation),
 * cfg.outputs = L loudspeakers. synth: Q*L rows (row q*L + l) of n_h taps;
 * fc: Q*L rows (row p*L + l) of n_hf taps. afc may be NULL (mu = 0). */
int aura_b200_auralizer_create(const aura_b200_config* cfg,
                               const float* const* synth, size_t n_synth_rows,
                               size_t n_h, const float* const* fc,
                               size_t n_fc_rows, size_t n_hf, float input_gain,
                               const aura_b200_afc* afc, int device,
                               aura_b200_engine** out);

void aura_b200_destroy(aura_b200_engine* e);

/* ---- streaming ----------------------------------------------------- */
/* One block: Convolver::process (convolver.hpp:111-123) /
 * Auralizer::process (auralizer.hpp:61-87). in: inputs x N planar host
 * floats, out: outputs x N. Blocking; no allocation; rejects non-finite
 * input with AURA_B200_E_NON_FINITE_INPUT (engine state untouched). */
int aura_b200_process(aura_b200_engine* e, const float* in, float* out);

/* Zero-copy variant for latency-critical hosts (SURVEY 8(b)'s io_buffers):
 * the engine's own pinned, device-mapped input (inputs x N) and output
 * (outputs x N) blocks, which k_front reads and writes over PCIe directly.
 * Write the next block into *in, call aura_b200_process_io, read the result
 * from *out before the next call -- no host copies on either side. Valid
 * between process_io calls only: during a call the device owns both. */
int aura_b200_io_buffers(aura_b200_engine* e, float** in, float** out);
int aura_b200_process_io(aura_b200_engine* e);

/* Failure detection (no reference counterpart): calls of
 * process / process_io whose host-visible latency exceeded the real-time
 * budget N / f_s since creation or the last reset, the largest and the last
 * latency (us), and the budget (us). */
int aura_b200_deadline_stats(const aura_b200_engine* e, uint64_t* misses, double* max_us, double* last_us,
                             double* budget_us);

/* Convolver::reset (convolver.hpp:133-142) / Auralizer::reset
 * (auralizer.hpp:95-99); an NLMS canceller is restored to its initial F^. */
int aura_b200_reset(aura_b200_engine* e);

/* Auralizer::feedback_estimate (auralizer.hpp:56-58): inputs x N floats,
 * copied out once the last processed block's background work (canceller,
 * f^ for the next block) is complete. */
int aura_b200_feedback_estimate(aura_b200_engine* e, float* out);
/* Auralizer::input_gain / set_input_gain (auralizer.hpp:51-52) */
int aura_b200_set_input_gain(aura_b200_engine* e, float gain);
float aura_b200_input_gain(const aura_b200_engine* e);

/* ---- accessors (convolver.hpp:96-107, auralizer.hpp:44-49) ----------- */
uint64_t aura_b200_blocks_processed(const aura_b200_engine* e);
size_t aura_b200_partition_count(const aura_b200_engine* e);    /* K (synth) */
size_t aura_b200_fc_partition_count(const aura_b200_engine* e); /* K_f, 0 for a convolver */
size_t aura_b200_filter_length(const aura_b200_engine* e);
int aura_b200_mode(const aura_b200_engine* e);
/* filters().spectrum(row, k) (engine.hpp:210-219): (N+1) complex as 2N+2
 * floats, copied back from the device. */
int aura_b200_filter_spectrum(aura_b200_engine* e, size_t row, size_t k,
                              float* out);
/* FrequencyDelayLine::slot(channel, age) (engine.hpp:261-266) of the input
 * FDL (which = 0) or the canceller FDL (which = 1): the spectrum pushed
 * `age` blocks ago, (N+1) complex in the reference layout. */
int aura_b200_fdl_slot(aura_b200_engine* e, int which, size_t channel,
                       size_t age, float* out);
/* Current canceller spectra W[p][l][k][j], P x L x K_f x (N+1) complex. */
int aura_b200_afc_coeffs(aura_b200_engine* e, float* out);
/* Load canceller spectra in the same layout (checkpoint / warm start of the
 * NLMS canceller, e.g. from a measured feedback path or a previous run's
 * aura_b200_afc_coeffs). DC and Nyquist bins must be real
 * (AURA_B200_E_NON_REAL_EDGE_BINS otherwise, as DftPlan::inverse,
 * dft.hpp:115-117). as_initial != 0: reset() returns to these spectra too
 * (NLMS engines; a mu = 0 canceller keeps whatever was loaded). */
int aura_b200_afc_load_coeffs(aura_b200_engine* e, const float* in, int as_initial);

/* Wait until every processed block has fully finished, including the
 * background work (next-block precompute, canceller update, f^). process()
 * returns as soon as the block's OUTPUT is ready. */
int aura_b200_synchronize(aura_b200_engine* e);

/* ---- multi-GPU loudspeaker sharding ---------------- */
/* An auralizer whose L loudspeakers are split over G engines (one per GPU,
 * one process per GPU): each engine is created with its contiguous slice of
 * loudspeaker rows (synth q*L_g + l, fc p*L_g + l) and the SAME mic input.
 * The canceller output and the NLMS power sum over all loudspeakers, so the
 * shards exchange P*N + 2N floats per block over NVLink (k_afc_finish: P2P
 * stores + system-scope flags, fixed rank-order sum, identical on every
 * shard). Convolvers need no exchange: their shards are independent.
 * Protocol: every rank calls shard_export, the G handles are all-gathered
 * by the host (torch.distributed is the plumbing), every rank calls
 * shard_connect; then all ranks process the same block sequence. reset()
 * must be called on every shard between two host barriers. */
#define AURA_B200_SHARD_HANDLE_BYTES 64
/* Allocate the exchange buffer; writes its CUDA IPC handle (64 bytes). */
int aura_b200_shard_export(aura_b200_engine* e, int world, int rank, void* handle);
/* handles: world x 64 bytes in rank order (own entry ignored). */
int aura_b200_shard_connect(aura_b200_engine* e, const void* handles);
/* Same wiring for G engines living in ONE process (virtual shards on one
 * GPU, or several GPUs of one process through P2P); engine g is rank g. */
int aura_b200_shard_connect_local(aura_b200_engine* const* engines, int world);
int aura_b200_shard_info(const aura_b200_engine* e, int* world, int* rank);
/* The same exchange through NCCL instead of our P2P kernel (SURVEY 8(e)'s
 * north-star transport, kept as the ablation): one ncclAllReduce(sum) of
 * the P*N + 2N partials per block, captured in the block's CUDA graph, then
 * k_afc_apply. NCCL is loaded at first use (libnccl.so.2); the summation
 * order is NCCL's (pin NCCL_ALGO / NCCL_PROTO for run-to-run determinism).
 * Protocol: rank 0 calls nccl_unique_id, the 128 bytes reach every rank by
 * the host's plumbing, every rank calls shard_connect_nccl. world = 1 is
 * allowed (a local all-reduce; bit-identical to the unsharded engine). */
#define AURA_B200_NCCL_ID_BYTES 128
int aura_b200_nccl_unique_id(void* id);
int aura_b200_shard_connect_nccl(aura_b200_engine* e, int world, int rank, const void* id);

/* Measurement and diagnostics entry points (bench.py, tools/): see
 * aura_b200_diag.h -- not part of the reference-replacing API. */

#ifdef __cplusplus
}
#endif
#endif /* AURA_B200_H */
