/*
 * aura_b200_diag.h -- measurement and diagnostics entry points of
 * libaura_b200.so (used by bench.py and tools/). Not part of the drop-in
 * boundary: nothing in the reference corresponds to them, and the C++
 * drop-in headers do not include this file. All of them run real blocks
 * (advancing the engine's block counter) unless stated otherwise.
 */
#ifndef AURA_B200_DIAG_H
#define AURA_B200_DIAG_H

#include "aura_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* How blocks run: 0 = one CUDA graph per block (default), 1 = the same
 * kernels launched on the engine stream (bit-identical; an A/B for launch
 * overhead). */
int aura_b200_set_launch_mode(aura_b200_engine* e, int mode);
int aura_b200_launch_mode(const aura_b200_engine* e);
/* Testing: number the device blocks from n instead of 0 (only before the
 * first block or right after reset; not for sharded engines). Outputs are
 * unchanged -- every delay line is zero, so the ring slots (block mod K)
 * may start anywhere -- which lets a test stream across 2^32 blocks. */
int aura_b200_seek_block(aura_b200_engine* e, uint64_t n);
/* Diagnostics: host-side breakdown of process() in graph mode, per block
 * (optionally paced): us from the call's start to {input staged, graph
 * launched, background event recorded, output flag seen, output copied}. */
int aura_b200_time_host_breakdown(aura_b200_engine* e, const float* host_in, size_t n_in_blocks,
                                  size_t blocks, double pace_us, double* out);
/* Run `blocks` blocks back to back with device-resident I/O (inputs already
 * in HBM, uploaded from host_in: n_in_blocks x inputs x N floats, cycled),
 * front and background graphs per block, timed with CUDA events on the
 * engine stream. latency_us[i] (may be NULL) = device time from block start
 * to its output written; block_us[i] = device time of ALL of block i's work
 * (front + background). */
int aura_b200_time_device_blocks(aura_b200_engine* e, const float* host_in,
                                 size_t n_in_blocks, size_t blocks,
                                 float* latency_us, float* block_us);
/* The same back-to-back blocks with ONE event pair around all of them
 * (no per-block event records in the stream): *total_us for `blocks`. */
int aura_b200_time_device_span(aura_b200_engine* e, const float* host_in, size_t n_in_blocks,
                               size_t blocks, float* total_us);
/* End-to-end latency through aura_b200_process() itself: `blocks` calls
 * with HOST input (cycling over host_in: n_in_blocks x inputs x N) and host
 * output, each timed with steady_clock from call to return (host->device
 * input transfer, all kernels, device->host output, completion wait).
 * pace_us > 0 spaces the calls on a real-time grid (one block every
 * pace_us, as an audio callback would) instead of back to back. */
int aura_b200_time_host_blocks(aura_b200_engine* e, const float* host_in,
                               size_t n_in_blocks, size_t blocks,
                               double pace_us, float* block_us);
/* Same blocks launched kernel by kernel with an event pair around each
 * phase; phase_us[p] = mean device time of phase p over `blocks`, names
 * via aura_b200_phase_name. Returns the phase count in *n_phases. */
int aura_b200_profile_phases(aura_b200_engine* e, size_t blocks,
                             float* phase_us, int* n_phases);
const char* aura_b200_phase_name(const aura_b200_engine* e, int phase);
/* Average device time of `reps` back-to-back single launches (no
 * programmatic overlap) of one phase kernel -- k_front = 0, k_back = 2,
 * k_reduce = 3 -- between two CUDA events on the engine stream: the
 * roofline denominator. The block counter, the canceller's smoothed power
 * and (k_back with NLMS) the canceller spectra W are restored afterwards. */
int aura_b200_time_phase(aura_b200_engine* e, int phase, size_t reps, float* avg_us);
/* Timeline of `blocks` (<= 64) back-to-back device-resident blocks from
 * %globaltimer stamps taken inside the kernels: out[(i*11 + k)*2 + {0,1}] =
 * first / last stamp (us, relative to block i's front start) of event k in
 * order k_front, k_back_head, k_back, k_reduce, canceller done, k_afc_finish,
 * output published, canceller sums in, f^ written, input spectra pushed;
 * slot 10 = {the next block's front start, 0}. -1 when the event did not
 * occur. Shows launch gaps and overlap. */
int aura_b200_trace_blocks(aura_b200_engine* e, size_t blocks, double* out);
/* The same timeline with the blocks run through process()'s own handshake
 * (mapped input and output, output words; host_in: n_in_blocks x inputs x N,
 * cycled), back to back: where the end-to-end path differs on the device. */
int aura_b200_trace_host_blocks(aura_b200_engine* e, const float* host_in, size_t n_in_blocks, size_t blocks,
                                double* out);
/* Diagnostics (not in the reference): per-segment / per-CTA timeline of the
 * streaming kernel k_back for the last of `blocks` blocks, us from the
 * kernel's first CTA start. out_segs: n_segs x {kind, tile, begin, end,
 * cta, start_us, partial_us, end_us} (one row per work item); out_ctas:
 * n_ctas x {start_us, first_data_us, exit_us}. Call with null outputs to get
 * the sizes. */
int aura_b200_trace_back(aura_b200_engine* e, size_t blocks, double* out_segs, size_t* n_segs,
                         double* out_ctas, size_t* n_ctas);
/* Kernels launched per block (front + background graphs). */
int aura_b200_launches_per_block(const aura_b200_engine* e);
/* Algorithmic bytes per block of each phase (SURVEY.md 8(d) formula). */
double aura_b200_phase_bytes(const aura_b200_engine* e, int phase);
/* Launch geometry summary as text ("grid=... block=... chunks=..."). */
int aura_b200_describe(const aura_b200_engine* e, char* buf, size_t cap);

#ifdef __cplusplus
}
#endif
#endif /* AURA_B200_DIAG_H */
