// stream.cuh -- k_back: the block's streaming work in ONE persistent,
// warp-specialised kernel (sm_100a).
//
// Per block n it computes
//   synthesis   S_l(n+1) = sum_q sum_{j=0}^{K-2} X_q(age j) (.) H_{l,q}[j+1]
//               (backend.hpp:212-235 over every partition but the first;
//               the first is k_front's, so block n+1's output is one small
//               kernel away from its input)
//   canceller   Yhat_p = sum_{l,k} W_{p,l}[k] (.) X_l(age k) with the fused
//               NLMS update W += mu/(P+delta) conj(X_l(pre-push age k)) E_p,
//               the loudspeaker power sum_l |X_l(age 0)|^2, and (last CTA)
//               one c2r per mic -> f^ for block n+1 (auralizer.hpp:73-86,
//               SURVEY Appendix A).
//
// Every byte of H and W is read exactly once per block, so the kernel is
// bound by HBM bandwidth (8 flop per 8 B; no tensor cores). It is built for
// that bound:
//  * one CTA per SM (grid <= 148); warp 8 lane 0 is the PRODUCER: it streams
//    the CTA's work through a ring of `stages` shared-memory slots with
//    cp.async.bulk (TMA bulk copies, SASS UBLKCP) completing on mbarriers --
//    100+ KB in flight per SM without holding anything in registers;
//  * warps 0-7 are CONSUMERS: per stage they wait on the slot's full
//    barrier, do the complex MACs out of shared memory into per-thread
//    register accumulators, and release the slot (one arrive per warp);
//  * the spectra are stored TILED so that every stage is one contiguous bulk
//    copy: H as [L/LT][NF/CT][tap][LT][CT] float4, W as [NF/CT][unit][P][CT],
//    and the delay lines as [ch][NF/CT][slot][CT] so a run of partitions is
//    one (or, at the ring wrap, two) copies;
//  * work is planned on the host (plan_back): every CTA streams a static
//    slice of the first 30% of every synthesis tile, then claims items from
//    one queue -- the middle of the synthesis with the canceller items spread
//    through it, small items for the tail, the age-0 stages last -- so the
//    canceller (whose inputs come from the front, overlapped with this
//    kernel via programmatic dependent launch) ends well before the stream;
//  * split-K partials are deterministic: warp shuffles over the tap phases
//    of a warp, a fixed-order shared-memory sum over the warps, one partial
//    per work item in a fixed slot; k_reduce sums each tile's partials in
//    slot order (fixed association => bit-reproducible). A tenth warp (the
//    signal warp) publishes each canceller partial for k_reduce's early
//    canceller CTA.
#pragma once
#include "kernels.cuh"

namespace aura_b200 {


// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy completing on an mbarrier, with an L2 policy
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// 128-bit store with an L2 eviction-priority hint (the canceller's W; never
// read back by this kernel, so no compiler memory barrier)
__device__ __forceinline__ void st_hint(float4* p, float4 v, uint64_t policy) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w), "l"(policy));
}
// programmatic dependent launch: wait for the preceding kernel (k_back_head)
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void consumers_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory");
}

// Work item (host-planned, kernels.cuh): kind (0 synthesis, 1 canceller) |
// tile << 1, item range [b, e) (synthesis: taps t = q (K-1) + j; canceller:
// units u = l KF + k), index of its split-K partial in the partials array.
// Everything the consumers need travels with the stage, so they never wait
// on a global load: the producer prefetches the next item's record while it
// streams the current one.
struct StageMeta {
  int item;       // < 0: no more work
  int t, t1;      // item range of this stage
  int flags;      // bit 0: last stage of the item; bit 1: canceller
  int tile;       // synthesis tile, or canceller column tile
  int slot;       // partial index (synthesis or canceller partials array)
};
// The consumers hand each published canceller partial to the signal warp
// through a small ring (afc_seq mode): {full, empty} mbarriers + the slot.
struct SigRing {
  uint64_t full[kSigSlots], empty[kSigSlots];
  int slot[kSigSlots];
};
static_assert(2 * kMaxStages * 8 + kMaxStages * sizeof(StageMeta) + sizeof(SigRing) <= kBackBarrierBytes,
              "barrier + metadata region");

// Rows v = vlo..vhi (vlo may be < 0: ring wrap) of a ring of `cap` rows of
// `row_bytes` at base -> dst, in increasing v.
__device__ __forceinline__ void copy_ring(float4* dst, const float4* base, int vlo, int vhi, int cap,
                                          int row_f4, uint64_t* bar, uint64_t pol) {
  const uint32_t rb = (uint32_t)row_f4 * 16u;
  if (vlo >= 0) {
    bulk_g2s(dst, base + (size_t)vlo * row_f4, (uint32_t)(vhi - vlo + 1) * rb, bar, pol);
  } else if (vhi < 0) {
    bulk_g2s(dst, base + (size_t)(vlo + cap) * row_f4, (uint32_t)(vhi - vlo + 1) * rb, bar, pol);
  } else {
    const int n1 = -vlo;
    bulk_g2s(dst, base + (size_t)(cap + vlo) * row_f4, (uint32_t)n1 * rb, bar, pol);
    bulk_g2s(dst + (size_t)n1 * row_f4, base, (uint32_t)(vhi + 1) * rb, bar, pol);
  }
}

// ----------------------------------------------------------------- producer
// Lane 0 of the producer warp: streams this CTA's static items, then claims
// queue items (one atomic each, issued an item ahead) until the queue is
// empty, then posts a sentinel stage. A stage never crosses an input
// (synthesis, MIMO) or a loudspeaker (canceller), so its delay-line rows are
// one ring run. Canceller stages also carry the column tile's NLMS error
// spectra and smoothed power.
// What the producer waits for before streaming rows produced by the
// current block's front half: with a separate k_back_head, k_front finished
// before k_back launched (stream order) and k_back_head is the PDL primary;
// in fused-head mode (front_head) k_front itself is the PDL primary, so rows
// it produces (X age 0) wait for it too (griddepcontrol.wait).
template <int LT, bool ELEM, int PT>
__device__ __forceinline__ void back_produce(const BlockArgs& a, blk_t n, uint64_t* full,
                                             uint64_t* empty, float4* slots, StageMeta* meta,
                                             uint32_t& q) {
  constexpr int XL = ELEM ? LT : 1;
  const int S = a.stages, CT = a.CT, CTn = a.CTn, K = a.K, KF = a.KF;
  const int Kt = K - 1, cap = KF + 1;
  const int T = (a.mode == 2 ? a.Q : 1) * Kt;
  const int nk = (int)(n % (blk_t)K);
  const int nka = PT > 0 ? (int)(n % (blk_t)cap) : 0;
  const uint64_t pol_stream = a.h_in_l2 ? policy_evict_normal() : policy_evict_first();
  const uint64_t pol_keep = policy_evict_last();
  unsigned* queue = a.tick + a.tick_queue;
  const bool planned = (int)blockIdx.x < a.plan_ctas;
  // this CTA's static range and its first record in ONE round of loads (the
  // ramp to the first bulk copy is on every launch's critical path)
  int4 r0 = make_int4(0, 0, 0, 0), first = make_int4(0, 0, 0, 0);
  if (planned) {
    r0 = a.cta_first[2 * blockIdx.x];
    first = a.cta_first[2 * blockIdx.x + 1];
  }
  const int s0 = r0.x, s1 = r0.y;
  // item sequence: static s0..s1-1, then queue claims
  auto claim = [&](int k) -> int {
    if (s0 + k < s1) return s0 + k;
    const int d = a.n_static + (int)atomicAdd(queue, 1u);
    return d < a.n_chunks ? d : -1;
  };
  bool waited = false, front_ok = !a.front_head;
  // ring cursor, advanced incrementally (no divisions on the per-stage path)
  int s = (int)(q % (uint32_t)S);
  uint32_t par = ((q / (uint32_t)S) & 1u) ^ 1u;
  int idx = claim(0);
  int4 rec = idx < 0 ? make_int4(0, 0, 0, 0) : (s0 < s1 ? first : a.chunks[idx]);
  for (int k = 0; idx >= 0; ++k) {
    // the next item: its claim (an atomic once past the static items) is
    // issued now, its record is loaded after this item's first stage is
    // issued -- neither round trip delays this item's first copy
    const int nidx = claim(k + 1);
    int4 nrec = make_int4(0, 0, 0, 0);
    bool have_next = false;
    const int kind = rec.x & 1, tile = rec.x >> 1;
    if (PT > 0 && kind == 1 && !waited) {
      griddep_wait();  // canceller inputs come from the head
      waited = true;
    }
    // per item: the input (synthesis) or loudspeaker (canceller) block b of
    // the first stage; stages never cross a block boundary
    const int B = kind ? KF : Kt;
    const int SP = kind ? a.spa : a.sp;
    int b = rec.y / B, b0 = b * B;
    const int g = tile / CTn, c = tile - g * CTn;
    const float4* hsrc = a.Ht + (size_t)tile * T * LT * CT;
    const uint32_t syn_tx = (uint32_t)((LT + XL) * CT) * 16u;
    for (int t = rec.y; t < rec.z;) {
      if (t == b0 + B) {
        ++b;
        b0 += B;
      }
      const int t1 = min(min(t + SP, rec.z), b0 + B);
      if (!front_ok && kind == 0 && t == b0) {
        griddep_wait();  // this stage reads X(age 0), pushed by the front
        front_ok = true;
      }
      mbar_wait(empty + s, par);
      meta[s] = StageMeta{idx, t, t1, (t1 == rec.z ? 1 : 0) | (kind << 1), tile, rec.w};
      float4* dst = slots + (size_t)s * a.slot_f4;
      const int nt = t1 - t;
      if (PT == 0 || kind == 0) {
        const int j0 = t - b0, j1 = t1 - b0;
        mbar_expect_tx(full + s, (uint32_t)nt * syn_tx);
        bulk_g2s(dst, hsrc + (size_t)t * LT * CT, (uint32_t)(nt * LT * CT) * 16u, full + s, pol_stream);
        float4* xd = dst + (size_t)a.sp * LT * CT;
#pragma unroll
        for (int i = 0; i < XL; ++i) {
          const int xc = ELEM ? g * LT + i : b;
          copy_ring(xd + (size_t)i * a.sp * CT, a.X + (size_t)(xc * CTn + c) * K * CT, nk - (j1 - 1),
                    nk - j0, K, CT, full + s, pol_keep);
        }
      } else {
        const int P = a.P, U = a.L * KF;
        const int l = b, k0 = t - b0;
        const int amax = k0 + nt - 1 + a.nlms;
        const int rows = amax - k0 + 1;
        const uint32_t cb = (uint32_t)CT * 16u;
        // E_p and the power: the consumers read them from the item's first stage only
        const bool ep = a.nlms && t == rec.y;
        mbar_expect_tx(full + s, (uint32_t)(nt * P * CT + rows * CT) * 16u + (ep ? (P + 1) * cb : 0u));
        bulk_g2s(dst, a.W + ((size_t)tile * U + t) * P * CT, (uint32_t)(nt * P * CT) * 16u, full + s,
                 a.w_in_l2 ? pol_keep : pol_stream);
        float4* xd = dst + (size_t)a.spa * P * CT;
        copy_ring(xd, a.XA + (size_t)(l * CTn + tile) * cap * CT, nka - amax, nka - k0, cap, CT, full + s,
                  pol_keep);
        if (ep) {  // E_p and the power of this column tile
          float4* ed = xd + (size_t)(a.spa + 1) * CT;
          for (int p = 0; p < P; ++p)
            bulk_g2s(ed + (size_t)p * CT, a.E + (size_t)p * a.NF + tile * CT, cb, full + s, pol_keep);
          bulk_g2s(ed + (size_t)P * CT, a.pw + (size_t)2 * tile * CT, cb, full + s, pol_keep);
        }
      }
      ++q;
      if (++s == S) {
        s = 0;
        par ^= 1u;
      }
      t = t1;
      if (!have_next) {
        if (nidx >= 0) nrec = a.chunks[nidx];
        have_next = true;
      }
    }
    if (!have_next && nidx >= 0) nrec = a.chunks[nidx];
    idx = nidx;
    rec = nrec;
  }
  mbar_wait(empty + s, par);
  meta[s].item = -1;
  mbar_arrive(full + s);
  ++q;
}

// Fixed-order split-K partial of R rows x CT columns from the consumers'
// register accumulators: warp shuffles over the 4 tap phases of a warp
// (lane bits 3-4), then the PG phase groups in order through `red`
// (PG * R * CT float4). Accumulator r goes to row row_of(r) (< 0: unused).
// Stores to dst[row * CT + f] (L2).
template <int RM, typename RowOf>
__device__ __forceinline__ void team_partial(float4 (&acc)[RM], int R, int CT, int PG, int pg, int f,
                                             int pl, float4* red, float4* dst, RowOf row_of) {
#pragma unroll
  for (int ra = 0; ra < RM; ++ra) {
    const int r = row_of(ra);
    if (r < 0) continue;
    float4 v = acc[ra];
#pragma unroll
    for (int m = 8; m <= 16; m <<= 1) {
      v.x += __shfl_xor_sync(0xffffffffu, v.x, m);
      v.y += __shfl_xor_sync(0xffffffffu, v.y, m);
      v.z += __shfl_xor_sync(0xffffffffu, v.z, m);
      v.w += __shfl_xor_sync(0xffffffffu, v.w, m);
    }
    if (pl == 0) red[((size_t)pg * R + r) * CT + f] = v;
  }
  consumers_sync();
  const int E = R * CT;
  for (int e = threadIdx.x; e < E; e += kConsumers) {
    float4 s = red[e];
    for (int g = 1; g < PG; ++g) s = f4add(s, red[(size_t)g * E + e]);
    __stcg(dst + e, s);
  }
  consumers_sync();
}

// --------------------------------------------------------------- consumers
// Warps 0-7: consume this CTA's stages of block n until the producer's
// sentinel (q is the CTA's running stage count, shared with the producer's
// by construction), leaving one split-K partial per work item.
// Consumer thread 0 -> signal warp: the canceller partial `slot` is stored
// (every consumer's stores precede the barrier that ended team_partial, and
// the arrive releases them at CTA scope). The signal warp makes them visible
// GPU-wide and publishes afc_seq[slot], so no consumer waits for that fence
// (a fence in a consumer warp waits for its in-flight W stores: ~1 us of
// k_back per canceller item). slot < 0: no more items.
__device__ __forceinline__ void sig_post(SigRing* r, uint32_t& k, int slot) {
  const int i = (int)(k % kSigSlots);
  mbar_wait(&r->empty[i], ((k / kSigSlots) & 1u) ^ 1u);
  r->slot[i] = slot;
  mbar_arrive(&r->full[i]);
  ++k;
}

template <int LT, bool ELEM, int PT>
__device__ __forceinline__ void back_consume(const BlockArgs& a, blk_t n, uint64_t* full,
                                             uint64_t* empty, StageMeta* meta, float4* red,
                                             float4* slots, uint32_t& q, unsigned long long* ctr,
                                             SigRing* sig) {
  uint32_t sq = 0;  // hand-offs posted (thread 0)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = a.stages;
  // consumer geometry: lane = pl * 8 + cl ; warp = pg * CG + cg
  const int CT = a.CT, CTn = a.CTn, KF = a.KF;
  const int CG = CT >> 3, PG = 8 / CG, PH = PG * 4;
  const int cl = lane & 7, pl = lane >> 3;
  const int cg = warp % CG, pg = warp / CG;
  const int f = cg * 8 + cl;     // column within the tile
  const int ph = pg * 4 + pl;    // tap phase
  const int P = PT > 0 ? a.P : 0;
  const int nl = PT > 0 ? a.nlms : 0;
  const int R = P + nl;  // canceller partial rows; row P: loudspeaker power
  // the canceller's W store: kept in L2 when it fits, else streamed out
  const uint64_t wpol = a.w_in_l2 ? policy_evict_last() : policy_evict_first();
  constexpr int PA = PT > 0 ? PT : 1;

  // ring cursor, advanced incrementally (no divisions on the per-stage path)
  int sl = (int)(q % (uint32_t)S);
  uint32_t par = (q / (uint32_t)S) & 1u;
  auto advance = [&]() {
    ++q;
    if (++sl == S) {
      sl = 0;
      par ^= 1u;
    }
  };
  for (;;) {
    mbar_wait(full + sl, par);
    StageMeta m = meta[sl];
    if (m.item < 0) {  // sentinel: release its slot too
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + sl);
      if (sig && threadIdx.x == 0) sig_post(sig, sq, -1);
      break;
    }
    if (ctr && q == 0 && threadIdx.x == 0) ctr[1] = globaltimer();
    const int item = m.item, tile = m.tile, slot = m.slot;
    if (a.seg_trace && threadIdx.x == 0) a.seg_trace[4 * (size_t)item] = globaltimer();
    if (PT == 0 || !(m.flags & 2)) {
      // ------------------------------------------------ synthesis item
      const int g = tile / CTn, c = tile - g * CTn;
      const bool dc = (c == 0 && f == 0);
      float4 acc[LT];
#pragma unroll
      for (int i = 0; i < LT; ++i) acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      for (;;) {
        const int nt = m.t1 - m.t;
        const float4* hs = slots + (size_t)sl * a.slot_f4;
        const float4* xs = hs + (size_t)a.sp * LT * CT;
        for (int i = ph; i < nt; i += PH) {
          const int r = nt - 1 - i;  // X rows are stored oldest-first
          if (ELEM) {
#pragma unroll
            for (int chn = 0; chn < LT; ++chn) {
              const XPack x = xpack(xs[((size_t)chn * a.sp + r) * CT + f], dc);
              cmac(acc[chn], x, hs[((size_t)i * LT + chn) * CT + f], dc);
            }
          } else {
            const XPack x = xpack(xs[(size_t)r * CT + f], dc);
            float4 h[LT];
#pragma unroll
            for (int chn = 0; chn < LT; ++chn) h[chn] = hs[((size_t)i * LT + chn) * CT + f];
#pragma unroll
            for (int chn = 0; chn < LT; ++chn) cmac(acc[chn], x, h[chn], dc);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + sl);
        advance();
        if (m.flags & 1) break;
        mbar_wait(full + sl, par);
        m = meta[sl];
      }
      const int E = LT * CT;
      team_partial<LT>(acc, LT, CT, PG, pg, f, pl, red, a.part_syn + (size_t)slot * E,
                       [](int r) { return r; });
      if (a.seg_trace && threadIdx.x == 0) a.seg_trace[4 * (size_t)item + 1] = globaltimer();
    } else if constexpr (PT > 0) {
      // ------------------------------------------------- canceller item
      const int c = tile;
      const int fg = c * CT + f;
      const bool dc = fg == 0;
      const int U = a.L * KF;
      float4 aac[PA + 1];  // P mics + the loudspeaker power
#pragma unroll
      for (int p = 0; p < PA + 1; ++p) aac[p] = make_float4(0.f, 0.f, 0.f, 0.f);
      // Each tap phase owns G consecutive units of a stage, so the row of age
      // k + 1 it needs for unit k's update is the age row of unit k + 1:
      // G + 1 delay-line rows per G units, all loads independent of the math.
      const int G = a.spa / PH;
      // NLMS error spectra and step mu / (power + delta) of this column: the
      // same for every stage of the item (staged in each; read from the first)
      float4 e4[PA];
      float4 st = make_float4(0.f, 0.f, 0.f, 0.f);
      if (nl) {
        const float4* es = slots + (size_t)sl * a.slot_f4 + (size_t)a.spa * P * CT + (size_t)(a.spa + 1) * CT;
#pragma unroll
        for (int p = 0; p < PA; ++p) e4[p] = p < P ? es[(size_t)p * CT + f] : st;
        const float4 pw = es[(size_t)P * CT + f];  // packed power of bins 2fg, 2fg+1
        st = make_float4(__fdiv_rn(a.mu, __fadd_rn(pw.x, a.delta)), __fdiv_rn(a.mu, __fadd_rn(pw.y, a.delta)),
                         __fdiv_rn(a.mu, __fadd_rn(pw.z, a.delta)), __fdiv_rn(a.mu, __fadd_rn(pw.w, a.delta)));
      }
      for (;;) {
        const int nt = m.t1 - m.t;
        const int l = m.t / KF, k0 = m.t - l * KF;
        const int amax = k0 + nt - 1 + nl;
        const float4* ws = slots + (size_t)sl * a.slot_f4;
        const float4* xs = ws + (size_t)a.spa * P * CT;
        const int i0 = ph * G, i1 = min(i0 + G, nt);
        // rows are oldest-first: unit i (age k0 + i) reads row amax - k0 - i
        const float4* xr = xs + (size_t)(amax - k0 - i0) * CT + f;
        const float4* wr = ws + (size_t)i0 * P * CT + f;
        if (nl && k0 == 0 && i0 == 0 && i1 > 0) {  // packed |X_l(age 0)|^2, rounded as the oracle
          const float4 xv = xr[0];
          float4& pa = aac[PA];
          if (dc) {
            pa.x = __fadd_rn(pa.x, __fmul_rn(xv.x, xv.x));
            pa.y = __fadd_rn(pa.y, __fmul_rn(xv.y, xv.y));
          } else {
            const float mm = __fadd_rn(__fmul_rn(xv.x, xv.x), __fmul_rn(xv.y, xv.y));
            pa.x = __fadd_rn(pa.x, mm);
            pa.y = __fadd_rn(pa.y, mm);
          }
          const float m2 = __fadd_rn(__fmul_rn(xv.z, xv.z), __fmul_rn(xv.w, xv.w));
          pa.z = __fadd_rn(pa.z, m2);
          pa.w = __fadd_rn(pa.w, m2);
        }
        // constrained variant: k_afc_constrain has already updated W
        if (nl && !a.afc_cons) {
          float4* wg = a.W + ((size_t)c * U + m.t + i0) * P * CT + f;
          float4 xa = xr[0];
#pragma unroll 4
          for (int i = i0; i < i1; ++i) {
            const float4 x1 = xr[-(int)CT];  // pre-push age k = post-push age k + 1
            xr -= CT;
            const XPack x0 = xpack(xa, dc);
#pragma unroll
            for (int p = 0; p < PA; ++p) {
              if (p >= P) break;
              float4 w = wr[(size_t)p * CT];
              // g = conj(x1) E_p (packed bin 0: DC and Nyquist real products),
              // rounded exactly as the oracle (aura_oracle.c nlms_update)
              const float4 ep = e4[p];
              const float px = __fmul_rn(x1.x, ep.x), py = __fmul_rn(x1.y, ep.y);
              float4 gr;
              gr.x = dc ? px : __fadd_rn(px, py);
              gr.y = dc ? py : __fsub_rn(__fmul_rn(x1.x, ep.y), __fmul_rn(x1.y, ep.x));
              gr.z = __fadd_rn(__fmul_rn(x1.z, ep.z), __fmul_rn(x1.w, ep.w));
              gr.w = __fsub_rn(__fmul_rn(x1.z, ep.w), __fmul_rn(x1.w, ep.z));
              w.x = __fadd_rn(w.x, __fmul_rn(st.x, gr.x));
              w.y = __fadd_rn(w.y, __fmul_rn(st.y, gr.y));
              w.z = __fadd_rn(w.z, __fmul_rn(st.z, gr.z));
              w.w = __fadd_rn(w.w, __fmul_rn(st.w, gr.w));
              st_hint(wg + (size_t)p * CT, w, wpol);
              cmac(aac[p], x0, w, dc);
            }
            xa = x1;
            wr += P * CT;
            wg += P * CT;
          }
        } else {
#pragma unroll 4
          for (int i = i0; i < i1; ++i) {
            const XPack x0 = xpack(xr[0], dc);
            xr -= CT;
#pragma unroll
            for (int p = 0; p < PA; ++p) {
              if (p >= P) break;
              cmac(aac[p], x0, wr[(size_t)p * CT], dc);
            }
            wr += P * CT;
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + sl);
        advance();
        if (m.flags & 1) break;
        mbar_wait(full + sl, par);
        m = meta[sl];
      }
      const int E = R * CT;
      // rows 0..P-1: the mics; row P: the loudspeaker power (accumulator PA)
      team_partial<PA + 1>(aac, R, CT, PG, pg, f, pl, red, a.part_afc + (size_t)slot * E,
                           [&](int r) { return r < P ? r : (r == PA && nl) ? P : -1; });
      if (sig && threadIdx.x == 0) sig_post(sig, sq, slot);
      if (a.seg_trace && threadIdx.x == 0) a.seg_trace[4 * (size_t)item + 1] = globaltimer();
    }
    if (a.seg_trace && threadIdx.x == 0) {
      a.seg_trace[4 * (size_t)item + 2] = globaltimer();
      a.seg_trace[4 * (size_t)item + 3] = blockIdx.x;
    }
  }
  ++q;  // the sentinel stage
}

// ------------------------------------------------------------------- k_back
// grid = back_ctas (<= 148, one per SM), kBackThreads threads, dynamic smem:
// [mbarriers + stage metadata | red (red_f4 float4; also the c2r scratch) |
// stages x slot].
template <int LT, bool ELEM, int PT>  // PT = 0: no canceller
__global__ void __launch_bounds__(kBackThreads, 1) k_back(const __grid_constant__ BlockArgs a) {
  extern __shared__ __align__(128) unsigned char bsm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(bsm);
  uint64_t* empty = full + kMaxStages;
  StageMeta* meta = reinterpret_cast<StageMeta*>(empty + kMaxStages);
  SigRing* ring = reinterpret_cast<SigRing*>(meta + kMaxStages);
  SigRing* sig = PT > 0 && a.afc_seq ? ring : nullptr;
  float4* red = reinterpret_cast<float4*>(bsm + kBackBarrierBytes);
  float4* slots = red + a.red_f4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = a.stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, kConsumers / 32);
    }
    for (int i = 0; i < kSigSlots; ++i) {
      mbar_init(&ring->full[i], 1);
      mbar_init(&ring->empty[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  griddep_launch();  // k_reduce may take the SMs this kernel's CTAs leave
  __syncthreads();
  const blk_t n = a.st->block;
  if (warp == kConsumers / 32) {
    uint32_t qp = 0;
    if (lane == 0) {
      if (a.front_head && a.front_hold) {
        // launched early (PDL) so this CTA is resident; hold the stream until
        // the front's outputs are out -- its loads are the latency path and
        // slow down badly under a saturated memory system (bounded: 2 s)
        const unsigned long long t0 = globaltimer();
        while (*reinterpret_cast<volatile unsigned long long*>(a.front_seq + (n & 1u)) <
                   (unsigned long long)a.front_ctas &&
               globaltimer() - t0 < 2000000000ull) {
          __nanosleep(100);
        }
      }
      back_produce<LT, ELEM, PT>(a, n, full, empty, slots, meta, qp);
    }
    return;
  }
  if (warp == kConsumers / 32 + 1) {
    // signal warp: publish each canceller partial the consumers hand over
    // (k_reduce's early canceller CTA waits for these words)
    if (sig && lane == 0) {
      for (uint32_t k = 0;; ++k) {
        const int i = (int)(k % kSigSlots);
        mbar_wait(&sig->full[i], (k / kSigSlots) & 1u);
        const int slot = sig->slot[i];
        mbar_arrive(&sig->empty[i]);
        if (slot < 0) break;
        __threadfence();
        *reinterpret_cast<volatile blk_t*>(a.afc_seq + slot) = n + 1;
      }
    }
    return;
  }
  if (a.trace && threadIdx.x == 0)
    atomicMin(&a.trace[((n % kTraceBlocks) * kTraceKernels + TR_BACK) * 2], globaltimer());
  unsigned long long* ctr = a.seg_trace ? a.seg_trace + 4 * (size_t)a.n_chunks + 3 * blockIdx.x : nullptr;
  if (ctr && threadIdx.x == 0) ctr[0] = globaltimer();

  uint32_t q = 0;
  back_consume<LT, ELEM, PT>(a, n, full, empty, meta, red, slots, q, ctr, sig);
  if (ctr && threadIdx.x == 0) ctr[2] = globaltimer();
  if (threadIdx.x == 0) {
    if (a.trace) atomicMax(&a.trace[((n % kTraceBlocks) * kTraceKernels + TR_BACK) * 2 + 1], globaltimer());
    // k_reduce (our dependent) must also find the front complete
    if (a.front_head) griddep_wait();
    // the last CTA out resets the work queue: every producer has stopped
    // claiming (its consumers saw the sentinel before getting here)
    unsigned* ex = a.tick + a.tick_queue + 1;
    if (atomicAdd(ex, 1u) == gridDim.x - 1u) {
      *ex = 0u;
      a.tick[a.tick_queue] = 0u;
    }
  }
}

// ----------------------------------------------------------------- k_reduce
// Helpers of k_reduce (the kernel and its description are below).

// Canceller reduce CTAs: stage the DftPlan tables and the smoothed power --
// they do not depend on the streaming kernel -- for whichever of them
// finishes f^. Call before the partials are ready; the caller syncs.
template <typename Team>
__device__ __forceinline__ void reduce_prefetch(const BlockArgs& a, int b, float4* rsm, Team tm) {
  if (b < a.red_syn_ctas) return;
  float2* z = reinterpret_cast<float2*>(rsm + kReduceThreads + afc_ys_f4(a.N, a.P));
  float2* tw = z + (a.N <= 1024 ? (size_t)a.P : 1) * a.N;
  float2* split = tw + a.N / 2;
  float2* pws = split + a.N / 2 + 1;
  stage_tables(tw, split, a.tw, a.split, a.N, tm);
  if (a.nlms)
    for (int jj = tm.tid(); jj < a.N; jj += tm.size()) pws[jj] = a.pw[jj];
}

// The plan record (first partial, count) of the tile reduce CTA b sums: a
// static table, so k_reduce loads it before waiting for k_back.
__device__ __forceinline__ int4 reduce_tile_info(const BlockArgs& a, int b) {
  const bool afc = b >= a.red_syn_ctas;
  const int cpt = afc ? a.red_afc_cpt : a.red_syn_cpt;
  const int tile = (afc ? b - a.red_syn_ctas : b) / cpt;
  return a.tinfo[afc ? a.n_syn_tiles + tile : tile];
}

// Reduce CTA b of block n (see k_reduce) with a team of kReduceThreads
// threads; ti = reduce_tile_info(a, b); s_last: shared int. The partials
// must be complete and visible.
template <typename Team>
__device__ void reduce_part(const BlockArgs& a, int b, blk_t n, float4* rsm, int* s_last, Team tm,
                            const int4 ti) {
  const int CT = a.CT, NF = a.NF;
  const int tid = tm.tid();
  const bool afc = b >= a.red_syn_ctas;
  const int E = afc ? a.red_afc_rows * CT : a.LTr * CT;
  const int cpt = afc ? a.red_afc_cpt : a.red_syn_cpt;  // CTAs per tile
  const int bb = afc ? b - a.red_syn_ctas : b;
  const int tile = bb / cpt, part = bb - tile * cpt;
  const int epc = (E + cpt - 1) / cpt;
  const int e0 = part * epc, e1 = min(E, e0 + epc);
  const float4* src = (afc ? a.part_afc : a.part_syn) + (size_t)ti.x * E;
  const int ne = e1 - e0;
  const int sub = max(1, kReduceThreads / max(ne, 1));
  const int per = (ti.y + sub - 1) / sub;
  const int el = tid % max(ne, 1), j = tid / max(ne, 1);
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  if (ne > 0 && j < sub) {
    const float4* p = src + e0 + el;
    const int i0 = j * per, i1 = min(ti.y, i0 + per);
    for (int i = i0; i < i1; i += 16) {  // 16 loads in flight, summed in slot order
      float4 t[16];
#pragma unroll
      for (int u = 0; u < 16; ++u)
        if (i + u < i1) t[u] = __ldcg(p + (size_t)(i + u) * E);
#pragma unroll
      for (int u = 0; u < 16; ++u)
        if (i + u < i1) v = (i + u == i0) ? t[u] : f4add(v, t[u]);
    }
  }
  // single: the whole canceller sum in this CTA (one column tile, few
  // partials): Yhat stays in shared memory, no ticket, no global round trips
  const bool single = afc && a.red_afc_ctas == 1 && afc_ys_f4(a.N, a.P) > 0;
  float4* ys = rsm + kReduceThreads;
  rsm[tid] = v;
  tm.sync();
  if (tid < ne) {
    float4 w = rsm[tid];
    for (int jj = 1; jj < sub; ++jj) w = f4add(w, rsm[jj * ne + tid]);
    const int e = e0 + tid;
    const int r = e / CT, col = e - r * CT;
    if (single) {
      ys[(size_t)r * NF + col] = w;
    } else if (afc) {
      __stcg(a.yhat + (size_t)r * NF + tile * CT + col, w);
    } else {
      const int CTn = a.CTn, g = tile / CTn, c = tile - g * CTn;
      __stcg(a.S + (size_t)(g * a.LTr + r) * NF + c * CT + col, w);
    }
  }
  if (!single) __threadfence();
  tm.sync();
  if (!afc) return;
  if (!single) {
    if (tid == 0) {
      unsigned* t = a.tick + 0;
      *s_last = atomicAdd(t, 1u) == (unsigned)a.red_afc_ctas - 1u;
      if (*s_last) *t = 0u;
    }
    tm.sync();
    if (!*s_last) return;
    __threadfence();
  }
  const float4* yh = single ? ys : a.yhat;
  auto stamp = [&](int id) {
    if (a.trace && tid == 0) {
      const unsigned long long now = globaltimer();
      atomicMin(&a.trace[((n % kTraceBlocks) * kTraceKernels + id) * 2], now);
      atomicMax(&a.trace[((n % kTraceBlocks) * kTraceKernels + id) * 2 + 1], now);
    }
  };
  stamp(TR_AFC_SUMMED);
  // the canceller of block n is complete: f^ for block n+1
  const int N = a.N, P = a.P;
  const bool sharded = a.xchg != 0;
  float2* z = reinterpret_cast<float2*>(rsm + kReduceThreads + afc_ys_f4(N, P));
  float2* tw = z + (N <= 1024 ? (size_t)P : 1) * N;
  float2* split = tw + N / 2;
  float2* pws = split + N / 2 + 1;
  // one c2r per mic: on one warp each (P <= 8 warps) for small transforms --
  // no CTA barrier per butterfly stage -- else on the whole team
  const bool warps = N <= 1024 && P * 32 <= tm.size();
  for (int p = 0; p < P; ++p) {
    // sharded: this shard's partial f^_p (c2r is linear), summed by k_afc_finish
    float* fh = sharded ? a.xmine + (size_t)p * N : a.fhat + (size_t)p * N;
    auto st = [&](int i, float x) { fh[i] = x; };
    const float2* yp = reinterpret_cast<const float2*>(yh + (size_t)p * NF);
    if (!warps) {
      irfft_packed_tail(yp, z, N, a.logN, tw, split, st, tm);
    } else if (tid / 32 == p) {
      irfft_warp_any(yp, z + (size_t)p * N, N, a.logN, tw, split, st);
    }
  }
  if (warps) tm.sync();
  stamp(TR_AFC_C2R);
  if (a.nlms) {
    const float2* sum = reinterpret_cast<const float2*>(yh + (size_t)P * NF);
    const float oml = __fsub_rn(1.0f, a.lambda);
    for (int jj = tid; jj < N; jj += tm.size()) {
      const float2 x = single ? sum[jj] : __ldcg(sum + jj);
      if (sharded) {  // partial power of this shard's loudspeakers
        reinterpret_cast<float2*>(a.xmine + (size_t)P * N)[jj] = x;
        continue;
      }
      float2 w = pws[jj];
      w.x = __fadd_rn(__fmul_rn(a.lambda, w.x), __fmul_rn(oml, x.x));
      w.y = __fadd_rn(__fmul_rn(a.lambda, w.y), __fmul_rn(oml, x.y));
      a.pw[jj] = w;
    }
  }
  if (a.trace && tid == 0) {
    const unsigned long long now = globaltimer();
    atomicMin(&a.trace[((n % kTraceBlocks) * kTraceKernels + TR_AFC_DONE) * 2], now);
    atomicMax(&a.trace[((n % kTraceBlocks) * kTraceKernels + TR_AFC_DONE) * 2 + 1], now);
  }
  __threadfence();
  tm.sync();
}

// ----------------------------------------------------------------- k_reduce
// The split-K reduction of block n, after k_back (programmatic dependent
// launch: its CTAs take the SMs k_back's CTAs leave and wait for k_back with
// griddepcontrol.wait -- except the single canceller CTA with afc_seq, which
// waits for the canceller partials k_back publishes). CTA b sums, for `epc` elements of one tile, the
// tile's partials in slot order -- `sub` threads per element over contiguous
// slot ranges, combined in order through shared memory -- so the association
// is fixed and results are bit-reproducible. Synthesis tiles -> S (block
// n+1's partitions >= 1); canceller column tiles -> Yhat, after which the
// last canceller CTA does one c2r per mic (f^ for block n+1; the sum over
// loudspeakers is done in the frequency domain -- one c2r per mic instead of
// the reference's L, auralizer.hpp:81-86) and smooths the power (Appendix A
// step 5). The last CTA advances the block (sharded: k_afc_finish does).
// grid = red_syn_ctas + red_afc_ctas, kReduceThreads threads.
__global__ void __launch_bounds__(kReduceThreads) k_reduce(const __grid_constant__ BlockArgs a) {
  extern __shared__ float4 rsm[];  // reduce_smem_f4(N, aur) float4
  __shared__ int s_last;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // early canceller (afc_seq): the single canceller CTA is index 0, so it is
  // the first to take an SM that k_back leaves, and it waits for the
  // canceller partials themselves -- which are done well before the
  // synthesis stream ends -- instead of for the whole of k_back
  const bool early = a.afc_seq != nullptr;
  const int b = !early ? (int)blockIdx.x : blockIdx.x == 0 ? a.red_syn_ctas : (int)blockIdx.x - 1;
  reduce_prefetch(a, b, rsm, Cta());
  // neither is written by k_back: load them before waiting for it
  const blk_t n = a.st->block;
  const int4 ti = reduce_tile_info(a, b);
  const bool afc_early = early && b == a.red_syn_ctas;
  if (afc_early) {
    const unsigned long long t0 = globaltimer();
    if (a.trace && threadIdx.x == 0) a.trace[((n % kTraceBlocks) * kTraceKernels + TR_AFC_WAIT) * 2] = t0;
    bool late = false;
    for (int i = threadIdx.x; i < ti.y; i += kReduceThreads) {
      const volatile blk_t* w = a.afc_seq + ti.x + i;
      while (*w != n + 1) {
        if (globaltimer() - t0 > 2000000000ull) {  // bounded: a lost partial fails the next call
          late = true;
          break;
        }
        __nanosleep(64);
      }
    }
    if (late) *reinterpret_cast<volatile unsigned*>(a.status_host) = 2u;
    __threadfence();
    __syncthreads();
    if (a.trace && threadIdx.x == 0)
      a.trace[((n % kTraceBlocks) * kTraceKernels + TR_AFC_WAIT) * 2 + 1] = globaltimer();
  } else {
    griddep_wait();  // k_back's partials
  }
  trace_begin(a, TR_REDUCE, n);
  reduce_part(a, b, n, rsm, &s_last, Cta(), ti);
  trace_end(a, TR_REDUCE, n);
  // this grid completes only after k_back (whose epilogue resets the queue)
  if (afc_early) griddep_wait();
  // retire: advance the block (sharded: k_afc_finish does)
  if (threadIdx.x == 0) {
    unsigned* t = a.tick + 1;
    if (atomicAdd(t, 1u) == gridDim.x - 1u) {
      *t = 0u;
      if (a.front_seq) a.front_seq[n & 1u] = 0ull;  // every producer of block n is past its hold
      if (a.xchg == 0) a.st->block = n + 1;
    }
  }
}

}  // namespace aura_b200
