/*
 * aura_oracle.h -- TEST INFRASTRUCTURE ONLY (the parity checker, never the
 * product). Plain-C restatement of the reference's UPOLS + feedback-canceller
 * hot path, used by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg only.
 *
 * Reference anchors (under /root/reference/proj/include/aura/):
 *   ao_plan_*     dft.hpp:34-183   (DftPlan: n_f/2 complex radix-2 DIT + split)
 *   ao_conv_*     convolver.hpp:19-46, :65-220 (make_partitioned_filters,
 *                 Convolver process/reset) + engine.hpp:233-279 (FDL ring)
 *                 + backend.hpp:212-235 (spectral_mac_channel)
 *   ao_aur_*      auralizer.hpp:25-123 (Auralizer), extended by SURVEY.md
 *                 Appendix A (NLMS, mu > 0) and Appendix B (MIMO, Q = P > 1).
 *   ao_direct_convolve  oracle.hpp:15-27 (64-bit direct convolution)
 *
 * Parity pinning: with mu == 0 and Q == 1 every function here is checked
 * bit-for-bit against the real reference compiled from /root/reference
 * (oracle/_ref, see oracle/Makefile) and against tests/golden fixtures.
 * The NLMS update (mu > 0) has NO reference implementation: "parity
 * unpinned" for coefficient tracking -- see DESIGN.md section 3.
 *
 * Spectra use the reference layout: bins = N + 1 complex64 values stored
 * as interleaved float pairs.
 */
#ifndef AURA_ORACLE_H
#define AURA_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* arithmetic type: float (liboracle.so) or double (liboracle64.so, built
 * with -DAO_F64: the float64 ground truth); every array argument below is
 * of this type */
#ifdef AO_F64
typedef double ao_real;
#else
typedef float ao_real;
#endif

typedef struct ao_plan ao_plan;
typedef struct ao_conv ao_conv;
typedef struct ao_aur ao_aur;

/* mode values shared with the product C-ABI (include/aura_b200.h) */
enum { AO_BROADCAST = 0, AO_ELEMENTWISE = 1, AO_MIMO = 2 };

ao_plan* ao_plan_new(size_t fft_size);
void ao_plan_free(ao_plan* p);
/* spectrum: (fft_size/2 + 1) complex as 2 floats each */
void ao_forward(const ao_plan* p, const ao_real* buffer, ao_real* spectrum);
void ao_inverse(const ao_plan* p, const ao_real* spectrum, ao_real* buffer);

/* filters: rows x n_h contiguous. broadcast: rows = outputs, inputs = 1;
 * elementwise: rows = outputs = inputs; mimo: rows = inputs * outputs,
 * row q * outputs + l = H_{l,q}. Returns NULL on bad arguments. */
ao_conv* ao_conv_new(size_t block, size_t inputs, size_t outputs, int mode,
                     const ao_real* filters, size_t n_h);
void ao_conv_free(ao_conv* c);
void ao_conv_process(ao_conv* c, const ao_real* in, ao_real* out);
void ao_conv_reset(ao_conv* c);
size_t ao_conv_partitions(const ao_conv* c);
/* copy spectrum of filter row r, partition k: (N+1) complex */
void ao_conv_spectrum(const ao_conv* c, size_t row, size_t k, ao_real* out);

/* Auralizer. inputs Q = mics P. synth: Q*L rows x n_h (row q*L + l);
 * fc: P*L rows x n_hf (row p*L + l). mu == 0 -> fixed F^ (reference). */
ao_aur* ao_aur_new(size_t block, size_t inputs, size_t outputs,
                   const ao_real* synth, size_t n_h, const ao_real* fc,
                   size_t n_hf, ao_real gain, ao_real mu, ao_real lambda,
                   ao_real delta);
void ao_aur_free(ao_aur* a);
void ao_aur_process(ao_aur* a, const ao_real* mic, ao_real* speakers);
void ao_aur_reset(ao_aur* a);
void ao_aur_set_gain(ao_aur* a, ao_real gain);
/* SURVEY Appendix A step 2, optional constrained variant: per (p, l, k) the
 * gradient mu/(P + delta) conj(X) E is taken to the time domain (c2r),
 * its last N samples are zeroed (a partition's taps live in the first N),
 * and it is transformed back (r2c) before it is added to W. Returns 0, or
 * -1 when the scratch cannot be allocated. */
int ao_aur_set_constrained(ao_aur* a, int constrained);
void ao_aur_feedback_estimate(const ao_aur* a, ao_real* out /* P x N */);
size_t ao_aur_fc_partitions(const ao_aur* a);
size_t ao_aur_synth_partitions(const ao_aur* a);
/* W as P x L x K_f x (N+1) complex */
void ao_aur_coeffs(const ao_aur* a, ao_real* out);
/* NLMS power vector, N+1 floats */
void ao_aur_power(const ao_aur* a, ao_real* out);

/* y[0 .. nx+nh-2] = x * h in float64 (oracle.hpp:15-27) */
void ao_direct_convolve(const double* x, size_t nx, const double* h,
                        size_t nh, double* y);

#ifdef __cplusplus
}
#endif
#endif
