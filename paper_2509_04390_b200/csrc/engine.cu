// engine.cu -- host side of libaura_b200.so: the reference-replacing C-ABI
// of include/aura_b200.h, the device memory layout, filter preparation on
// the GPU, the k_back work planner and the per-block CUDA graphs. The only
// translation unit that contains (and launches) the kernels; sharding is in
// shard.cu, the measurement entry points in diag.cu.
//
// Reference interfaces replaced (under /root/reference/proj/include/aura):
//   aura_b200_convolver_create  Convolver::Convolver      convolver.hpp:67-94
//   aura_b200_auralizer_create  Auralizer::Auralizer      auralizer.hpp:27-41
//   aura_b200_process           Convolver::process        convolver.hpp:111-123
//                               Auralizer::process        auralizer.hpp:61-87
//   aura_b200_reset             Convolver/Auralizer::reset convolver.hpp:133-142,
//                                                          auralizer.hpp:95-99
//   aura_b200_feedback_estimate Auralizer::feedback_estimate auralizer.hpp:56-58
//   aura_b200_filter_spectrum   PartitionedFilterSet::spectrum engine.hpp:210-219
//   aura_b200_device_count      list_backends             backend.hpp:186-193
#include "engine.hpp"
#include "kernels.cuh"
#include "stream.cuh"

thread_local std::string g_err;

// ---------------------------------------------------------------- launches

void aura_b200_engine::launch_phase(int ph, const BlockArgs& a, cudaStream_t s) {
  switch (ph) {
    case PH_FRONT:
      k_front<<<front_grid(a), kFrontThreads, smem_front, s>>>(a);
      break;
    case PH_BACK_HEAD:
      if (has_head())
        k_back_head<<<(unsigned)(aur ? L + (a.nlms ? P : 0) : 1), kFrontThreads, smem_head, s>>>(a);
      if (a.afc_cons && cons8)  // after the front (or head): E_p
        launch_pdl(k_afc_constrain8, (unsigned)cons_ctas, kCons8Threads, smem_cons, !pdl_off, a, s);
      else if (a.afc_cons)
        launch_pdl(k_afc_constrain, (unsigned)cons_ctas, 32u * cons_warps, smem_cons, !pdl_off, a, s);
      break;
    case PH_BACK:
      if (has_back())
        launch_pdl(back_fn, (unsigned)back_ctas, kBackThreads, smem_back,
                   (has_head() || front_head || a.afc_cons) && !pdl_off, a, s);
      break;
    case PH_REDUCE:
      if (has_back())
        launch_pdl(k_reduce, (unsigned)(a.red_syn_ctas + a.red_afc_ctas), kReduceThreads, smem_reduce,
                   !pdl_off, a, s);
      break;
    case PH_AFC_FINISH:
      if (sharded() && a.xchg == 1) k_afc_finish<<<1, kTailThreads, 0, s>>>(a);
      if (sharded() && a.xchg == 2) {
        nccl_check(nccl_api().allreduce(a.xmine, a.xsum, (size_t)(P * N + 2 * N), ncclFloat, ncclSum, nccl, s),
                   "ncclAllReduce");
        k_afc_apply<<<1, kTailThreads, 0, s>>>(a);
      }
      break;
    case PH_ADVANCE:
      if (!has_back()) k_advance<<<1, 1, 0, s>>>(a.st);
      break;
  }
}


namespace {

// Tuning knobs: AURA_B200_<name> environment overrides of measured defaults
// (experiments only). Every knob that is set is recorded in e->knobs, which
// describe() -- and so every bench line -- reports.
const char* knob_raw(aura_b200_engine* e, const char* name) {
  const std::string var = std::string("AURA_B200_") + name;
  const char* v = std::getenv(var.c_str());
  if (v) e->knobs += (e->knobs.empty() ? "" : ",") + std::string(name) + "=" + v;
  return v;
}
int knob_i(aura_b200_engine* e, const char* name, int def) {
  const char* v = knob_raw(e, name);
  return v ? std::atoi(v) : def;
}
double knob_f(aura_b200_engine* e, const char* name, double def) {
  const char* v = knob_raw(e, name);
  return v ? std::atof(v) : def;
}

void setup_tables(aura_b200_engine* e, BlockArgs& a) {
  // DftPlan ctor (dft.hpp:36-52), bit for bit: angle step computed once in
  // double, multiplied by the index, cos/sin in double, rounded to float.
  const size_t N = e->N;  // = half of n_f
  std::vector<float2> tw(N / 2), split(N / 2 + 1);
  const double step = -2.0 * M_PI / (double)N;
  for (size_t j = 0; j < N / 2; ++j)
    tw[j] = make_float2((float)std::cos(step * (double)j), (float)std::sin(step * (double)j));
  const double sstep = -2.0 * M_PI / (double)(2 * N);
  for (size_t j = 0; j <= N / 2; ++j)
    split[j] = make_float2((float)std::cos(sstep * (double)j), (float)std::sin(sstep * (double)j));
  float2* dtw = dalloc<float2>(tw.size(), e->dmem);
  float2* dsp = dalloc<float2>(split.size(), e->dmem);
  CK(cudaMemcpy(dtw, tw.data(), sizeof(float2) * tw.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dsp, split.data(), sizeof(float2) * split.size(), cudaMemcpyHostToDevice));
  a.tw = dtw;
  a.split = dsp;
}

// GPU make_partitioned_filters (convolver.hpp:19-46): rows of n_h taps are
// uploaded in bounded batches, transformed and scattered into the device
// layout described by `o`, base[r] and base0[r] (k_partition).
void partition_rows(aura_b200_engine* e, const BlockArgs& a, const float* const* rows, size_t n_rows,
                    size_t n_h, size_t K, PartOut o, const std::vector<long long>& base,
                    const std::vector<long long>& base0) {
  const size_t N = e->N;
  const size_t budget = size_t(256) << 20;  // bytes of staged taps per batch
  size_t batch = std::max<size_t>(1, budget / (n_h * sizeof(float)));
  batch = std::min<size_t>(batch, 65535);
  float* d_taps = nullptr;
  long long* d_off = nullptr;
  const size_t nb = std::min(batch, n_rows);
  CK(cudaMalloc(&d_taps, nb * n_h * sizeof(float)));
  CK(cudaMalloc(&d_off, 2 * nb * sizeof(long long)));
  const size_t smem = 16 * N + 8 * (size_t)table_f2((int)N);
  raise_smem_limit(k_partition, smem);
  std::vector<long long> offs(2 * nb);
  for (size_t r0 = 0; r0 < n_rows; r0 += batch) {
    const size_t nr = std::min(batch, n_rows - r0);
    for (size_t r = 0; r < nr; ++r)
      CK(cudaMemcpyAsync(d_taps + r * n_h, rows[r0 + r], n_h * sizeof(float), cudaMemcpyHostToDevice,
                         e->stream));
    for (size_t r = 0; r < nr; ++r) {
      offs[r] = base[r0 + r];
      offs[nb + r] = base0.empty() ? 0 : base0[r0 + r];
    }
    CK(cudaMemcpyAsync(d_off, offs.data(), 2 * nb * sizeof(long long), cudaMemcpyHostToDevice,
                       e->stream));
    dim3 grid((unsigned)K, (unsigned)nr);
    k_partition<<<grid, 256, smem, e->stream>>>(d_taps, n_h, (int)K, (int)N, ilog2(N), a.tw, a.split, o,
                                                 d_off, d_off + nb);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(e->stream));
  }
  cudaFree(d_taps);
  cudaFree(d_off);
}

int pick_tile(size_t L) {
  for (int t : {8, 4, 2})
    if (L % t == 0) return t;
  return 1;
}

template <int LT>
BackFn back_for(bool elem, int PT) {
  if (elem) return k_back<LT, true, 0>;
  switch (PT) {
    case 0: return k_back<LT, false, 0>;
    case 1: return k_back<LT, false, 1>;
    case 2: return k_back<LT, false, 2>;
    case 4: return k_back<LT, false, 4>;
    default: return k_back<LT, false, 8>;
  }
}

// Canceller partials per column tile that one k_reduce CTA sums in two load
// rounds per thread (kReduceThreads threads over E elements, 16 loads in
// flight per round: reduce_part; 32 in flight measured slower at c2 and c3).
long long afc_single_cap(int rows, int CT) {
  const int E = rows * CT;
  return E > kReduceThreads ? 0 : 2LL * 16LL * (kReduceThreads / E);
}

// Plan k_back (stream.cuh): tiling, stage sizes, pipeline depth, and the
// static work split. Three phases -- synthesis taps [0, TA) of every tile,
// the canceller units, synthesis taps [TA, T) -- are each cut into
// back_ctas equal contiguous pieces; CTA c runs piece c of each phase in
// that order. Every (CTA, tile) piece is one split-K partial; a tile's
// partials are numbered by tap position, which fixes the summation order.
void plan_back(aura_b200_engine* e, BlockArgs& a) {
  const int N = (int)e->N, NF = N / 2;
  const int CT = std::min(NF, 32), CTn = NF / CT, PH = kConsumers / CT;
  a.CT = CT;
  a.CTn = CTn;
  const bool elem = e->mode == AURA_B200_ELEMENTWISE;
  const int LT = e->LT, XL = elem ? LT : 1;
  const long long Kt = (long long)e->K - 1;
  const long long Qh = e->mode == AURA_B200_MIMO ? (long long)e->Q : 1;
  const long long T = Qh * Kt;
  const int tiles = (int)(e->L / LT) * CTn;
  a.n_syn_tiles = tiles;
  const int P = e->aur ? (int)e->P : 0;
  const long long U = e->aur ? (long long)e->L * e->KF : 0;
  if (T > INT32_MAX / 2 || U > INT32_MAX / 2) fail(AURA_B200_E_INVALID_ARGUMENT, "filters too long");
  // ~54 KB synthesis stages (three in the ring at c3): the single producer
  // lane's per-stage cost is what bounds an SM's stream
  // (profiles/r1s5_stream.md), so fewer, larger stages (sp need not be a
  // multiple of the 8 tap phases). Measured against 46 KB x 4 (round 2,
  // gpurun_out/r3ab, r3ac): mean block period c3 52.4 vs 53.2 us, c4 224.0
  // vs 224.9, c2 20.1 vs 20.5, c5 and c1 unchanged; 64 KB (two stages) and
  // 38 KB are slower.
  const int target_kb = std::max(4, knob_i(e, "STAGE_KB", 54));
  const int target_f4 = target_kb * 1024 / 16;
  const int syn_row = (LT + XL) * CT;
  a.sp = std::max(PH, target_f4 / syn_row);
  const int afc_row = (P + 1) * CT;
  a.spa = PH * std::max(1, target_f4 / (PH * std::max(afc_row, 1)));
  long long slot = 0;
  if (T > 0) slot = std::max<long long>(slot, (long long)a.sp * syn_row);
  if (U > 0)  // W rows, canceller FDL rows, then E_p and the power of the column tile
    slot = std::max<long long>(slot, (long long)a.spa * P * CT + (long long)(a.spa + 1) * CT +
                                         (long long)(P + 1) * CT);
  a.slot_f4 = (int)slot;
  const int rmax = std::max(LT, P + 1);
  a.red_f4 = std::max({kConsumers, 64 * rmax, NF});
  const size_t budget = (size_t)std::max(64, std::min(224, knob_i(e, "BACK_SMEM_KB", 200))) * 1024;
  const size_t fixed = kBackBarrierBytes + (size_t)a.red_f4 * 16;
  const size_t per = (size_t)a.slot_f4 * 16;
  a.stages = per ? (int)std::min<size_t>(kMaxStages, (budget - fixed) / per) : 0;
  if (const int st = knob_i(e, "STAGES", 0)) a.stages = std::max(2, std::min(a.stages, st));
  if (e->has_back() && a.stages < 2)
    fail(AURA_B200_E_INVALID_ARGUMENT, "block size / channel tile too large for the streaming kernel");
  e->smem_back = fixed + (size_t)a.stages * per;
  // footprint: keep the spectra in L2 across blocks when they fit
  const double foot = 8.0 * N * ((double)e->L * Qh * e->K + (double)e->Qx * e->K +
                                 (double)P * U + (double)(e->aur ? e->L * (e->KF + 1) : 0));
  a.h_in_l2 = foot < 80e6 ? 1 : 0;
  // Optionally pin the canceller's W (read-modify-write every block) in L2
  // with evict-last hints when its working set (W, its delay line, the input
  // FDL) is under AURA_B200_W_L2_MB. Off by default: measured at c3 it moves
  // ~25 MB per block off HBM but k_back gets ~1 us SLOWER (45.3 vs 46.2 us,
  // three A/B runs; profiles/r1s5_stream.md) -- the canceller units are not
  // HBM-bound once they run interleaved with the synthesis stream.
  const double afc_foot = 8.0 * N * ((double)P * U + (double)(e->aur ? e->L * (e->KF + 1) : 0) +
                                     (double)e->Qx * e->K);
  const double w_l2_mb = knob_f(e, "W_L2_MB", 0.0);
  a.w_in_l2 = (P > 0 && afc_foot < w_l2_mb * 1e6) ? 1 : 0;
  // grid: one CTA per SM, fewer for small work (>= ~96 KB per CTA). Sized
  // and planned from the synthesis alone when there is one, so the
  // synthesis association -- and the output bits -- are the same with or
  // without a canceller (test_auralizer.cpp:47-65 pins EXPECT_EQ).
  const double syn_b = (double)tiles * T * syn_row * 16.0;
  const double afc_b = (double)CTn * U * (P * (e->args.nlms ? 2 : 1) + 1) * CT * 16.0;
  const double drive = T > 0 ? syn_b : afc_b;
  const double cta_kb = std::max(1.0, knob_f(e, "CTA_KB", 96.0));  // bytes per CTA at least
  int ctas = (int)std::min<double>(e->sms, std::max(1.0, std::ceil(drive / (cta_kb * 1024))));
  if (const int c = knob_i(e, "BACK_CTAS", 0)) ctas = std::max(1, std::min(ctas, c));
  e->back_ctas = ctas;
  // Work: every CTA first runs a static piece of the first 30% of every
  // synthesis tile's taps (they start at t = 0, before anything can be
  // claimed, and cover the front half, which the canceller waits for), then
  // claims queue items until the queue is empty. The queue holds the rest of
  // the synthesis as tile-interleaved items -- larger ones for the middle
  // (to 85%), small ones for the last 15% so the CTAs finish together
  // whatever their start time -- with the canceller's items spread evenly
  // through the middle part: at any time about the canceller's share of the
  // SMs runs canceller units (mostly L2 hits) while the rest keep HBM busy
  // with the synthesis stream. Every item is one split-K partial with a fixed
  // slot, so which CTA claims it does not change the bits.
  const double fa = knob_f(e, "PHASE_A", 0.30);
  const long long TA = T > 0 ? std::max<long long>(1, (long long)std::ceil(fa * T)) : 0;
  // measured: 0.75 -> 0.85 gives c3 -2 us, c5 -2 us, c4 and c2 unchanged
  const double fb = knob_f(e, "PHASE_B", 0.85);
  const long long TB = T > 0 ? std::max<long long>(TA, (long long)std::ceil(fb * T)) : 0;
  // queue items: ~12 per CTA in the last 15%, at least two stages (keeps
  // the tail short and the partial count -- k_reduce's input -- small at c5
  // sizes); ~3 per CTA in the middle part
  // queue items per CTA: last part, middle part
  const long long nq_per = std::max(1, knob_i(e, "QITEMS", 12)), nb_per = std::max(1, knob_i(e, "BITEMS", 3));
  const long long qtaps = (T - TB) * tiles;
  const long long CQ = std::max<long long>(2LL * a.sp, (qtaps / (nq_per * ctas) + a.sp - 1) / a.sp * a.sp);
  const long long btaps = (TB - TA) * tiles;
  const long long CB = std::max<long long>(CQ, (btaps / (nb_per * ctas) + a.sp - 1) / a.sp * a.sp);
  std::vector<int4> chunks;
  std::vector<int> item_off(ctas + 1, 0);
  std::vector<std::vector<std::pair<int, int>>> at(tiles + CTn);  // per tile: (b, item)
  auto push = [&](int kind, int tile, long long b, long long e_) {
    at[kind ? tiles + tile : tile].push_back({(int)b, (int)chunks.size()});
    chunks.push_back(make_int4(kind | (tile << 1), (int)b, (int)e_, 0));
  };
  // The first stage of every input (taps [q (K-1), q (K-1) + sp)) reads
  // the input spectrum the front pushes this block; those stages are left out
  // of the static pieces and claimed last from the queue, so no CTA's static
  // work waits for the front half.
  const long long late = std::min<long long>(a.sp, Kt);
  auto lateset = [&](long long t) { return Kt > 0 && (t % Kt) < late; };
  // intervals of [lo, hi) without the late taps
  auto pieces = [&](long long lo, long long hi, std::vector<std::pair<long long, long long>>& out) {
    out.clear();
    long long t = lo;
    while (t < hi) {
      if (lateset(t)) {
        t = std::min<long long>(hi, (t / Kt) * Kt + late);
        continue;
      }
      const long long next_q = Kt > 0 ? (t / Kt + 1) * Kt : hi;
      const long long e_ = std::min<long long>(hi, next_q);
      out.push_back({t, e_});
      t = e_;
    }
  };
  std::vector<std::pair<long long, long long>> tmp;
  {  // static: piece c of phase A's intervals (tile-major, one linear item space)
    std::vector<std::tuple<int, long long, long long>> iv;
    for (int tile = 0; tile < tiles; ++tile) {
      pieces(0, TA, tmp);
      for (auto& pr : tmp) iv.emplace_back(tile, pr.first, pr.second);
    }
    long long n_items = 0;
    for (auto& x : iv) n_items += std::get<2>(x) - std::get<1>(x);
    for (int c = 0; c < ctas; ++c) {
      item_off[c] = (int)chunks.size();
      if (n_items <= 0) continue;
      long long i0 = n_items * c / ctas, i1 = n_items * (c + 1) / ctas;
      long long base = 0;
      for (auto& x : iv) {
        const long long len = std::get<2>(x) - std::get<1>(x);
        const long long s0 = std::max(i0, base), s1 = std::min(i1, base + len);
        if (s0 < s1) push(0, std::get<0>(x), std::get<1>(x) + (s0 - base), std::get<1>(x) + (s1 - base));
        base += len;
      }
    }
  }
  item_off[ctas] = (int)chunks.size();
  a.n_static = (int)chunks.size();
  {  // queue
    // synthesis [lo, hi) of every tile in items of `cs` taps, tile-interleaved
    // so every tile's partials spread over the whole range
    auto syn_items = [&](long long lo, long long hi, long long cs) {
      std::vector<std::vector<std::pair<long long, long long>>> qv(tiles);
      size_t nq = 0;
      for (int t = 0; t < tiles; ++t) {
        pieces(lo, hi, tmp);
        for (auto& pr : tmp)
          for (long long b = pr.first; b < pr.second; b += cs)
            qv[t].push_back({b, std::min<long long>(pr.second, b + cs)});
        nq = std::max(nq, qv[t].size());
      }
      std::vector<std::tuple<int, long long, long long>> out;
      for (size_t j = 0; j < nq; ++j)
        for (int t = 0; t < tiles; ++t)
          if (j < qv[t].size()) out.emplace_back(t, qv[t][j].first, qv[t][j].second);
      return out;
    };
    const auto mid = syn_items(TA, TB, CB);
    // canceller: ~2 items per CTA, each a contiguous run of units of one
    // column tile (units of several loudspeakers are fine: a stage never
    // crosses one)
    std::vector<std::tuple<int, long long, long long>> afc;
    if (U > 0) {
      long long per = std::max<long long>(a.spa, (U * CTn / (2LL * ctas) + a.spa - 1) / a.spa * a.spa);
      if (CTn == 1) {
        // one column tile: few enough partials that one k_reduce CTA sums
        // them in one round of loads and runs the c2r from shared memory
        // (reduce_part's single-CTA path; cpt_for below gives 1)
        // (only while the items stay short enough to balance: <= ~1.5 MB)
        // (halving the cap -- twice as long canceller items -- made c3's
        // k_back 11 us slower: the long items unbalance the queue)
        const long long cap = afc_single_cap(P + (e->args.nlms ? 1 : 0), CT);
        const double unit_b = (double)(P * (e->args.nlms ? 2 : 1) + 1) * CT * 16.0;
        const long long per1 = cap > 0 ? ((U + cap - 1) / cap + a.spa - 1) / a.spa * a.spa : 0;
        if (cap > 0 && (double)per1 * unit_b <= 1.5e6) per = std::max(per, per1);
      }
      for (int c = 0; c < CTn; ++c)
        for (long long b = 0; b < U; b += per) afc.emplace_back(c, b, std::min<long long>(U, b + per));
    }
    // merge: canceller items evenly through the middle synthesis items (the
    // first middle items go first: the canceller waits for the head)
    const size_t nm = mid.size(), na = afc.size();
    // over the first two thirds: the long items end well before the tail
    const double span_f = std::min(1.0, std::max(0.05, knob_f(e, "AFC_SPAN", 2.0 / 3.0)));
    // share of the middle items before the first canceller item: the CTAs
    // that reach the queue first (at the end of the static slice, ~11 us into
    // a c3 block) would otherwise wait for the front half's canceller head
    // (c3: k_back -0.6 us; c4 unchanged)
    const double start_f = std::min(0.9, std::max(0.0, knob_f(e, "AFC_START", 0.3)));
    const size_t first = (size_t)((double)nm * start_f);
    const size_t span = (size_t)((double)(nm - first) * span_f);
    size_t im = 0;
    for (size_t j = 0; j < na; ++j) {
      const size_t upto = first + span * (2 * j + 1) / (2 * na);  // middle items before canceller item j
      for (; im < upto; ++im) push(0, std::get<0>(mid[im]), std::get<1>(mid[im]), std::get<2>(mid[im]));
      push(1, std::get<0>(afc[j]), std::get<1>(afc[j]), std::get<2>(afc[j]));
    }
    for (; im < nm; ++im) push(0, std::get<0>(mid[im]), std::get<1>(mid[im]), std::get<2>(mid[im]));
    for (auto& x : syn_items(TB, T, CQ)) push(0, std::get<0>(x), std::get<1>(x), std::get<2>(x));
    // the late (age-0) stages last of all
    for (long long q = 0; Kt > 0 && q < Qh; ++q)
      for (int t = 0; t < tiles; ++t) push(0, t, q * Kt, q * Kt + late);
  }
  std::vector<int> cnt(tiles + CTn);
  for (int t = 0; t < tiles + CTn; ++t) {
    std::sort(at[t].begin(), at[t].end());
    cnt[t] = (int)at[t].size();
    for (int i = 0; i < cnt[t]; ++i) chunks[at[t][i].second].w = i;
  }
  std::vector<int4> tinfo(tiles + CTn);
  int slot_syn = 0, slot_afc = 0, max_syn = 1, max_afc = 1;
  for (int t = 0; t < tiles + CTn; ++t) {
    int& sl = t < tiles ? slot_syn : slot_afc;
    tinfo[t] = make_int4(sl, cnt[t], 0, 0);
    sl += cnt[t];
    (t < tiles ? max_syn : max_afc) = std::max(t < tiles ? max_syn : max_afc, cnt[t]);
  }
  // items carry their partial's index in the partials array (tile's first
  // partial + the item's rank in the tile), so k_back never reads tinfo
  for (auto& ch : chunks) {
    const int kind = ch.x & 1, tile = ch.x >> 1;
    ch.w += tinfo[kind ? tiles + tile : tile].x;
  }
  a.n_chunks = (int)chunks.size();
  a.plan_ctas = ctas;
  std::vector<int4> first(2 * (size_t)ctas);
  for (int c = 0; c < ctas; ++c) {
    first[2 * c] = make_int4(item_off[c], item_off[c + 1], 0, 0);
    first[2 * c + 1] = item_off[c] < item_off[c + 1] ? chunks[item_off[c]] : make_int4(0, 0, 0, 0);
  }
  int4* dfirst = dalloc<int4>(first.size(), e->dmem);
  CK(cudaMemcpy(dfirst, first.data(), first.size() * sizeof(int4), cudaMemcpyHostToDevice));
  a.cta_first = dfirst;
  e->n_syn_segs = slot_syn;
  e->n_afc_segs = slot_afc;
  e->h_chunks = chunks;
  int4* dch = dalloc<int4>(std::max<size_t>(1, chunks.size()), e->dmem);
  int4* dti = dalloc<int4>(std::max<size_t>(1, tinfo.size()), e->dmem);
  if (!chunks.empty())
    CK(cudaMemcpy(dch, chunks.data(), chunks.size() * sizeof(int4), cudaMemcpyHostToDevice));
  if (!tinfo.empty()) CK(cudaMemcpy(dti, tinfo.data(), tinfo.size() * sizeof(int4), cudaMemcpyHostToDevice));
  a.chunks = dch;
  a.tinfo = dti;
  // k_reduce geometry: ~16 partials per thread, elements split over CTAs
  a.LTr = LT;
  const int red_loads = std::max(1, std::min(32, knob_i(e, "RED_LOADS", 16)));  // partial loads per thread
  auto cpt_for = [&](int E, int maxcnt) {
    const int sub = std::min(16, std::max(1, (maxcnt + red_loads - 1) / red_loads));
    const int ne = std::max(1, kReduceThreads / sub);
    return (E + ne - 1) / ne;
  };
  a.red_syn_cpt = tiles ? cpt_for(LT * CT, max_syn) : 1;
  a.red_syn_ctas = T > 0 ? tiles * a.red_syn_cpt : 0;
  a.red_afc_rows = P + (e->args.nlms ? 1 : 0);
  a.red_afc_cpt = U > 0 ? cpt_for(a.red_afc_rows * CT, max_afc) : 1;
  if (U > 0 && CTn == 1 && max_afc <= afc_single_cap(a.red_afc_rows, CT)) a.red_afc_cpt = 1;
  a.red_afc_ctas = U > 0 ? CTn * a.red_afc_cpt : 0;
  // the single canceller CTA (reduce_part) starts as soon as k_back has
  // published the canceller partials, off the end-of-block critical path
  a.afc_seq = nullptr;
  e->n_afc_seq = 0;
  if (U > 0 && a.red_afc_ctas == 1 && afc_ys_f4((int)N, P) > 0 && knob_i(e, "AFC_EARLY", 1)) {
    e->n_afc_seq = (size_t)std::max(slot_afc, 1);
    a.afc_seq = dalloc<blk_t>(e->n_afc_seq, e->dmem);
    CK(cudaMemset(a.afc_seq, 0, e->n_afc_seq * sizeof(blk_t)));
  }
  e->smem_reduce = 16 * reduce_smem_f4(N, e->aur, P);
  raise_smem_limit(k_reduce, e->smem_reduce);
  // tickets: [0] canceller CTAs of k_reduce, [1] all k_reduce CTAs, [2] work
  // queue, [3] k_back exits, [4] canceller items done (fused tail)
  a.tick_queue = 2;
  a.tick = dalloc<unsigned>(6, e->dmem);
  CK(cudaMemset(a.tick, 0, 6 * sizeof(unsigned)));
  a.part_syn = dalloc<float4>(std::max<size_t>(1, (size_t)slot_syn * LT * CT), e->dmem);
  if (e->aur) {
    const size_t R = (size_t)P + 1;
    a.part_afc = dalloc<float4>(std::max<size_t>(1, (size_t)slot_afc * R * CT), e->dmem);
    a.yhat = dalloc<float4>(R * NF, e->dmem);
    CK(cudaMemset(a.yhat, 0, sizeof(float4) * R * NF));
  }
  switch (LT) {
    case 1: e->back_fn = back_for<1>(elem, e->PT); break;
    case 2: e->back_fn = back_for<2>(elem, e->PT); break;
    case 4: e->back_fn = back_for<4>(elem, e->PT); break;
    default: e->back_fn = back_for<8>(elem, e->PT); break;
  }
  if (e->has_back())
    raise_smem_limit(e->back_fn, e->smem_back);
}

void common_init(aura_b200_engine* e, int device) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    fail(AURA_B200_E_BACKEND_UNAVAILABLE, "accelerator backend is not available: no CUDA device");
  }
  if (device < 0 || device >= n) fail(AURA_B200_E_INVALID_ARGUMENT, "device index out of range");
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    fail(AURA_B200_E_BACKEND_UNAVAILABLE,
         std::string("accelerator backend needs an sm_100 (B200) device, found ") + prop.name);
  e->device = device;
  e->sms = prop.multiProcessorCount;
  CK(cudaSetDevice(device));
  CK(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&e->ev_front, cudaEventDisableTiming));
}


void finish_init(aura_b200_engine* e) {
  BlockArgs& a = e->args;
  const size_t N = e->N, NF = N / 2;
  // state + I/O
  a.st = dalloc<DevState>(1, e->dmem);
  CK(cudaMemset(a.st, 0, sizeof(DevState)));
  a.S = dalloc<float4>(e->L * NF, e->dmem);
  CK(cudaMemset(a.S, 0, sizeof(float4) * e->L * NF));
  const size_t in_ch = (size_t)e->Qx;
  CK(cudaHostAlloc(&e->h_in, in_ch * N * sizeof(float), cudaHostAllocMapped | cudaHostAllocPortable));
  CK(cudaHostAlloc(&e->h_out, e->L * N * sizeof(float), cudaHostAllocMapped | cudaHostAllocPortable));
  std::memset(e->h_in, 0, in_ch * N * sizeof(float));
  std::memset(e->h_out, 0, e->L * N * sizeof(float));
  CK(cudaHostAlloc(&e->h_status, sizeof(unsigned), cudaHostAllocMapped | cudaHostAllocPortable));
  *e->h_status = 0;
  CK(cudaHostGetDevicePointer((void**)&a.status_host, e->h_status, 0));
  a.G = 1;
  a.grank = 0;
  a.xchg = 0;
  a.xsum = nullptr;
  float* din;
  float* dout;
  CK(cudaHostGetDevicePointer((void**)&din, e->h_in, 0));
  CK(cudaHostGetDevicePointer((void**)&dout, e->h_out, 0));
  a.in = din;
  a.out = dout;
  a.cur_mt = dalloc<float>(std::max<size_t>(1, e->Q) * N, e->dmem);
  CK(cudaMemset(a.cur_mt, 0, sizeof(float) * std::max<size_t>(1, e->Q) * N));
  set_advance_total(e);
  // front: one CTA per cpb output channels
  a.cpb = (int)std::max<size_t>(1, (e->L + 4 * e->sms - 1) / (4 * e->sms));
  const size_t Qs = e->mode == AURA_B200_ELEMENTWISE ? 1 : e->Q;
  // shared memory: the FFT work areas, then (when they fit) the DftPlan
  // tables and the first channel's S and partition-0 spectra
  e->smem_front = 8 * N * (Qs + 2);
  e->smem_head = 24 * N;
  const size_t tables = 8 * (size_t)table_f2((int)N);
  a.smem_tables = std::max(e->smem_front, e->smem_head) + tables <= 200 * 1024 ? 1 : 0;
  if (a.smem_tables) {
    e->smem_front += tables;
    e->smem_head += tables;
  }
  {
    const size_t pre = 8 * N * (1 + Qs);
    a.front_pre = e->smem_front + pre <= 160 * 1024 ? 1 : 0;
    if (a.front_pre) e->smem_front += pre;
  }
  // one output channel per warp (8 per CTA) where the per-warp areas fit:
  // small transforms synchronise with __syncwarp instead of CTA barriers
  a.front_warps = 0;
  {
    const char* fw = knob_raw(e, "FRONT_WARPS");
    const int W = kFrontThreads / 32;
    const size_t sw = 8 * front_warps_f2((int)N, (int)Qs, W);
    // measured (profiles/r1s4_front.md, r1s5_stream.md): a clear win at
    // N <= 64; at N = 128 a warp's transform alone is slower than the CTA
    // version, but 8x fewer front CTAs let k_back's CTAs start at once (c5:
    // -13 us per block, c2 -2 us); at N = 256 the output comes later
    const bool want = fw ? std::atoi(fw) != 0 : N <= 128;
    if (e->mode != AURA_B200_ELEMENTWISE && sw <= 160 * 1024 && want) {
      a.front_warps = W;
      a.cpb = W;
      e->smem_front = std::max(e->smem_front, sw);
    }
  }
  if (e->smem_front > 227 * 1024)
    fail(AURA_B200_E_INVALID_ARGUMENT, "block size too large for this many inputs (shared memory)");
  raise_smem_limit(k_front, e->smem_front);
  raise_smem_limit(k_back_head, e->smem_head);
  // device-resident I/O variant for measurement
  e->pool_blocks = 64;
  e->d_in_pool = dalloc<float>(e->pool_blocks * in_ch * N, e->dmem);
  CK(cudaMemset(e->d_in_pool, 0, e->pool_blocks * in_ch * N * sizeof(float)));
  e->d_out = dalloc<float>(e->L * N, e->dmem);
  // second window-history buffer (fused head: prev_in / hist1 by block parity)
  a.hist1 = dalloc<float>(in_ch * N, e->dmem);
  CK(cudaMemset(a.hist1, 0, sizeof(float) * in_ch * N));
  // fused head (profiles/r1s4_front.md): k_back launches as k_front's
  // programmatic dependent -- measured better for the auralizer (no separate
  // canceller head kernel) and for convolvers (the stream starts early)
  e->front_head = true;
  e->front_head = knob_i(e, "FRONT_HEAD", 1) != 0;
  a.front_head = e->front_head ? 1 : 0;
  a.front_hold = 0;  // measured: holding the stream does not speed the front up (profiles/r1s4_front.md)
  a.front_hold = knob_i(e, "FRONT_HOLD", 0);
  a.front_seq = dalloc<unsigned long long>(2, e->dmem);
  CK(cudaMemset(a.front_seq, 0, 2 * sizeof(unsigned long long)));
  // output-ready words for process(): mapped host memory, one per k_front
  // CTA -- the output CTAs and the NLMS error-spectrum CTAs, which read the
  // mapped input too (the host refills it only once all of them are done)
  a.front_ctas = (int)((e->L + a.cpb - 1) / a.cpb);
  e->n_outflags = (size_t)e->front_grid(a);
  CK(cudaHostAlloc(&e->h_outflag, e->n_outflags * sizeof(unsigned long long),
                   cudaHostAllocMapped | cudaHostAllocPortable));
  std::memset(e->h_outflag, 0, e->n_outflags * sizeof(unsigned long long));
  CK(cudaHostGetDevicePointer((void**)&a.out_flag, e->h_outflag, 0));
  e->use_outflag = knob_i(e, "OUTFLAG", 1) != 0;
  e->rebuild_graphs();
  e->dev_args = a;
  e->dev_args.out = e->d_out;
  e->dev_args.in = e->d_in_pool;
  e->dev_args.out_flag = nullptr;  // device-resident measurement: no host handshake
  CK(cudaStreamSynchronize(e->stream));
}

void reset_state(aura_b200_engine* e) {
  BlockArgs& a = e->args;
  const size_t N = e->N, NF = N / 2;
  cudaStream_t s = e->stream;
  CK(cudaStreamSynchronize(s));
  CK(cudaMemsetAsync(a.st, 0, sizeof(DevState), s));
  if (a.afc_seq) CK(cudaMemsetAsync(a.afc_seq, 0, e->n_afc_seq * sizeof(blk_t), s));
  CK(cudaMemsetAsync(a.prev_in, 0, sizeof(float) * e->Qx * N, s));
  if (a.hist1) CK(cudaMemsetAsync(a.hist1, 0, sizeof(float) * e->Qx * N, s));
  if (a.front_seq) CK(cudaMemsetAsync(a.front_seq, 0, 2 * sizeof(unsigned long long), s));
  CK(cudaMemsetAsync(a.X, 0, sizeof(float4) * (size_t)e->Qx * e->K * NF, s));
  CK(cudaMemsetAsync(a.S, 0, sizeof(float4) * e->L * NF, s));
  if (e->aur) {
    CK(cudaMemsetAsync(a.prev_spk, 0, sizeof(float) * e->L * N, s));
    CK(cudaMemsetAsync(a.XA, 0, sizeof(float4) * e->L * (e->KF + 1) * NF, s));
    CK(cudaMemsetAsync(a.fhat, 0, sizeof(float) * e->P * N, s));
    CK(cudaMemsetAsync(a.pw, 0, sizeof(float2) * N, s));
    if (a.nlms)
      CK(cudaMemcpyAsync(a.W, e->W0, sizeof(float4) * e->w_elems, cudaMemcpyDeviceToDevice, s));
    // sharded: the caller resets every shard between two barriers (no block
    // in flight anywhere), so zeroing the own flags restarts the sequence
    if (e->xbuf) CK(cudaMemsetAsync(e->xbuf, 0, e->xbuf_bytes, s));
  }
  CK(cudaStreamSynchronize(s));
  e->blocks = 0;
  e->block_base = 0;
  for (size_t i = 0; i < e->n_outflags; ++i) reinterpret_cast<volatile unsigned long long*>(e->h_outflag)[i] = 0;
  // a shard-exchange timeout is cleared by a coordinated reset of every shard
  *reinterpret_cast<volatile unsigned*>(e->h_status) = 0u;
}

void alloc_synth(aura_b200_engine* e, BlockArgs& a) {
  const size_t N = e->N, NF = N / 2;
  a.N = (int)N;
  a.logN = ilog2(N);
  a.NF = (int)NF;
  a.Q = (int)e->Q;
  a.L = (int)e->L;
  a.K = (int)e->K;
  a.mode = e->mode;
  a.CT = (int)std::min<size_t>(NF, 32);
  a.CTn = (int)(NF / a.CT);
  const size_t Qh = e->mode == AURA_B200_MIMO ? e->Q : 1;
  a.Ht = dalloc<float4>(std::max<size_t>(1, e->L * Qh * (e->K - 1) * NF), e->dmem);
  a.H0 = dalloc<float4>(e->L * Qh * NF, e->dmem);
  a.X = dalloc<float4>((size_t)e->Qx * e->K * NF, e->dmem);
  a.prev_in = dalloc<float>((size_t)e->Qx * N, e->dmem);
  CK(cudaMemset(a.X, 0, sizeof(float4) * (size_t)e->Qx * e->K * NF));
  CK(cudaMemset(a.prev_in, 0, sizeof(float) * e->Qx * N));
}

// Synthesis spectra: partition 0 -> H0 [L][Qh][NF]; partitions k >= 1 ->
// Ht [L/LT][CTn][T][LT][CT], tap t = q (K-1) + k - 1 (kernels.cuh).
void upload_synth(aura_b200_engine* e, BlockArgs& a, const float* const* rows, size_t n_rows,
                  size_t n_h) {
  const long long NF = (long long)e->N / 2, CT = a.CT, CTn = a.CTn, LT = e->LT;
  const long long Qh = e->mode == AURA_B200_MIMO ? (long long)e->Q : 1;
  const long long Kt = (long long)e->K - 1, T = Qh * Kt;
  std::vector<long long> base(n_rows), base0(n_rows);
  for (size_t r = 0; r < n_rows; ++r) {
    long long l = (long long)r, q = 0;
    if (e->mode == AURA_B200_MIMO) { q = (long long)(r / e->L); l = (long long)(r % e->L); }
    const long long g = l / LT, i = l % LT;
    base[r] = ((g * CTn) * T + q * Kt - 1) * LT * CT + i * CT;
    base0[r] = (l * Qh + q) * NF;
  }
  PartOut o{const_cast<float4*>(a.Ht), const_cast<float4*>(a.H0), LT * CT, T * LT * CT, (int)CT};
  partition_rows(e, a, rows, n_rows, n_h, e->K, o, base, base0);
}

void check_rows(const float* const* rows, size_t n_rows) {
  if (!rows) fail(AURA_B200_E_EMPTY_FILTER, "need at least one filter");
  for (size_t r = 0; r < n_rows; ++r)
    if (!rows[r]) fail(AURA_B200_E_INVALID_ARGUMENT, "null filter row");
}

}  // namespace

static void unpack_row(const float2* packed, size_t N, float* out) {
  // packed bin 0 = (DC, Nyquist) -> reference bins 0 and N, imag exactly 0
  out[0] = packed[0].x;
  out[1] = 0.0f;
  for (size_t j = 1; j < N; ++j) {
    out[2 * j] = packed[j].x;
    out[2 * j + 1] = packed[j].y;
  }
  out[2 * N] = packed[0].y;
  out[2 * N + 1] = 0.0f;
}

// ====================================================================== ABI

extern "C" {

int aura_b200_abi_version(void) { return AURA_B200_ABI_VERSION; }
const char* aura_b200_last_error(void) { return g_err.c_str(); }

int aura_b200_device_count(int* out) {
  return guarded([&] {
    int n = 0, usable = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    for (int d = 0; d < n; ++d) {
      cudaDeviceProp p;
      if (cudaGetDeviceProperties(&p, d) == cudaSuccess && p.major == 10) ++usable;
    }
    *out = usable;
  });
}

int aura_b200_device_name(int device, char* buf, size_t cap) {
  return guarded([&] {
    cudaDeviceProp p;
    CK(cudaGetDeviceProperties(&p, device));
    std::snprintf(buf, cap, "%s (sm_%d%d, %d SMs)", p.name, p.major, p.minor, p.multiProcessorCount);
  });
}

int aura_b200_convolver_create(const aura_b200_config* cfg, int mode,
                               const float* const* filters, size_t n_rows,
                               size_t n_h, int device, aura_b200_engine** out) {
  return guarded([&] {
    if (!out) fail(AURA_B200_E_INVALID_ARGUMENT, "out is null");
    *out = nullptr;
    if (mode < 0 || mode > 2) fail(AURA_B200_E_INVALID_ARGUMENT, "unknown channel mode");
    validate(cfg, mode == AURA_B200_MIMO);
    // convolver.hpp:22-30 (make_partitioned_filters runs before the mode checks)
    if (n_rows == 0 || !filters) fail(AURA_B200_E_EMPTY_FILTER, "need at least one filter");
    if (n_h == 0) fail(AURA_B200_E_EMPTY_FILTER, "filters must have at least one tap");
    check_rows(filters, n_rows);
    // convolver.hpp:84-93
    if (mode == AURA_B200_BROADCAST && cfg->inputs != 1)
      fail(AURA_B200_E_MODE_CHANNEL_MISMATCH, "broadcast mode requires one input channel");
    if (mode == AURA_B200_ELEMENTWISE && cfg->inputs != cfg->outputs)
      fail(AURA_B200_E_MODE_CHANNEL_MISMATCH,
           "elementwise mode requires input channels == output channels");
    const size_t want = mode == AURA_B200_MIMO ? cfg->inputs * cfg->outputs : cfg->outputs;
    if (n_rows != want)
      fail(AURA_B200_E_MODE_CHANNEL_MISMATCH, "filter count must equal the configured output channels");
    std::unique_ptr<aura_b200_engine> e(new aura_b200_engine());
    common_init(e.get(), device);
    e->mode = mode;
    e->N = cfg->block_size;
    e->budget_us = 1e6 * (double)cfg->block_size / (double)cfg->sample_rate_hz;
    e->Q = mode == AURA_B200_ELEMENTWISE ? 1 : cfg->inputs;
    e->L = cfg->outputs;
    e->Qx = mode == AURA_B200_ELEMENTWISE ? (int)cfg->outputs : (int)cfg->inputs;
    e->K = (n_h + e->N - 1) / e->N;
    e->n_h = n_h;
    e->LT = pick_tile(e->L);
    BlockArgs& a = e->args;
    setup_tables(e.get(), a);
    alloc_synth(e.get(), a);
    upload_synth(e.get(), a, filters, n_rows, n_h);
    a.is_aur = 0;
    a.nlms = 0;
    a.P = 0;
    e->PT = 0;
    plan_back(e.get(), a);
    finish_init(e.get());
    *out = e.release();
  });
}

int aura_b200_auralizer_create(const aura_b200_config* cfg,
                               const float* const* synth, size_t n_synth_rows,
                               size_t n_h, const float* const* fc,
                               size_t n_fc_rows, size_t n_hf, float input_gain,
                               const aura_b200_afc* afc, int device,
                               aura_b200_engine** out) {
  return guarded([&] {
    if (!out) fail(AURA_B200_E_INVALID_ARGUMENT, "out is null");
    *out = nullptr;
    validate(cfg, true);
    const size_t Q = cfg->inputs, L = cfg->outputs;
    // auralizer.hpp:102-115 (single input in the reference; Q > 1 is the
    // Appendix-B MIMO extension), then both convolvers' checks.
    if (n_synth_rows != n_fc_rows)
      fail(AURA_B200_E_CHANNEL_COUNT_MISMATCH,
           "synthesis and feedback-cancellation filter sets must have the same channel count");
    if (n_synth_rows == 0 || !synth || !fc) fail(AURA_B200_E_EMPTY_FILTER, "need at least one filter");
    if (n_h == 0 || n_hf == 0) fail(AURA_B200_E_EMPTY_FILTER, "filters must have at least one tap");
    check_rows(synth, n_synth_rows);
    check_rows(fc, n_fc_rows);
    if (n_synth_rows != Q * L)
      fail(AURA_B200_E_MODE_CHANNEL_MISMATCH, "filter count must equal inputs x output channels");
    if (Q > 8) fail(AURA_B200_E_INVALID_ARGUMENT, "at most 8 microphones/inputs are supported");
    const float mu = afc ? afc->mu : 0.0f;
    if (afc && (!(mu >= 0.0f) || !(afc->lambda >= 0.0f && afc->lambda <= 1.0f) ||
                !(afc->delta > 0.0f) || !std::isfinite(mu)))
      fail(AURA_B200_E_INVALID_ARGUMENT, "afc needs mu >= 0, 0 <= lambda <= 1, delta > 0");
    std::unique_ptr<aura_b200_engine> e(new aura_b200_engine());
    common_init(e.get(), device);
    e->aur = true;
    e->mode = Q == 1 ? AURA_B200_BROADCAST : AURA_B200_MIMO;
    e->N = cfg->block_size;
    e->budget_us = 1e6 * (double)cfg->block_size / (double)cfg->sample_rate_hz;
    e->Q = Q;
    e->L = L;
    e->P = Q;
    e->Qx = (int)Q;
    e->K = (n_h + e->N - 1) / e->N;
    e->KF = (n_hf + e->N - 1) / e->N;
    e->n_h = n_h;
    e->n_hf = n_hf;
    e->LT = pick_tile(L);
    e->PT = Q == 1 ? 1 : Q == 2 ? 2 : Q <= 4 ? 4 : 8;
    BlockArgs& a = e->args;
    setup_tables(e.get(), a);
    alloc_synth(e.get(), a);
    upload_synth(e.get(), a, synth, n_synth_rows, n_h);
    const size_t N = e->N, NF = N / 2;
    a.is_aur = 1;
    a.P = (int)Q;
    a.KF = (int)e->KF;
    a.gain = input_gain;
    a.mu = mu;
    a.lambda = afc ? afc->lambda : 0.9f;
    a.delta = afc ? afc->delta : kDefaultDeltaPerN * (float)N;
    a.nlms = mu > 0.0f;
    a.afc_cons = a.nlms && afc->constrained != 0;
    if (a.afc_cons) {
      // one warp per canceller unit, two per CTA (one when a warp's transform
      // scratch is large), 64 registers; 12 CTAs per SM (measured: 8 / 12 /
      // 16 give a c3 block of 120.8 / 116.8 / 116.8 us)
      const size_t per_warp = cons_smem_per_warp((int)N);
      a.cons_tables = cons_smem_tables((int)N) + per_warp <= 227 * 1024;
      const size_t tables = a.cons_tables ? cons_smem_tables((int)N) : 0;
      e->cons_warps = (int)std::max<size_t>(1, std::min<size_t>(kConsThreads / 32, (227 * 1024 - tables) / per_warp));
      e->smem_cons = tables + (size_t)e->cons_warps * per_warp;
      if (e->smem_cons > 227 * 1024)
        fail(AURA_B200_E_INVALID_ARGUMENT, "block size too large for the constrained canceller update");
      raise_smem_limit(k_afc_constrain, e->smem_cons);
      const long long units = (long long)Q * L * (long long)e->KF;
      if (units >= (1LL << 30)) fail(AURA_B200_E_INVALID_ARGUMENT, "too many canceller partitions for the constrained update");
      a.cons_prefetch = knob_i(e.get(), "CONS_PREFETCH", 1);
      const long long per_sm = std::max(1, knob_i(e.get(), "CONS_CTAS_PER_SM", 12));
      e->cons_ctas = (int)std::min<long long>(per_sm * e->sms, (units + e->cons_warps - 1) / e->cons_warps);
      // N = 64: eight threads per unit, every butterfly computed once
      // (k_afc_constrain8)
      if (N == 64 && knob_i(e.get(), "CONS_OCT", 1)) {
        e->cons8 = true;
        e->smem_cons = cons8_smem((int)Q);
        raise_smem_limit(k_afc_constrain8, e->smem_cons);
        const long long per8 = std::max(1, knob_i(e.get(), "CONS8_CTAS_PER_SM", 4));
        e->cons_ctas = (int)std::min<long long>(per8 * e->sms, (units + 15) / 16);
      }
    }
    e->w_elems = Q * L * e->KF * NF;
    a.W = dalloc<float4>(e->w_elems, e->dmem);
    {  // W [CTn][L*KF][P][CT], row p*L + l
      const long long CT = a.CT, KF = (long long)e->KF, P = (long long)Q;
      const long long U = (long long)L * KF;
      std::vector<long long> base(n_fc_rows);
      for (size_t r = 0; r < n_fc_rows; ++r) {
        const long long p = (long long)(r / L), l = (long long)(r % L);
        base[r] = (l * KF * P + p) * CT;
      }
      PartOut o{a.W, nullptr, P * CT, U * P * CT, (int)CT};
      partition_rows(e.get(), a, fc, n_fc_rows, n_hf, e->KF, o, base, {});
    }
    if (a.nlms) {
      e->W0 = dalloc<float4>(e->w_elems, e->dmem);
      CK(cudaMemcpy(e->W0, a.W, sizeof(float4) * e->w_elems, cudaMemcpyDeviceToDevice));
    }
    a.XA = dalloc<float4>(L * (e->KF + 1) * NF, e->dmem);
    a.prev_spk = dalloc<float>(L * N, e->dmem);
    a.spk = dalloc<float>(L * N, e->dmem);
    a.fhat = dalloc<float>(Q * N, e->dmem);
    a.pw = dalloc<float2>(N, e->dmem);
    a.E = dalloc<float4>(Q * NF, e->dmem);
    CK(cudaMemset(a.XA, 0, sizeof(float4) * L * (e->KF + 1) * NF));
    CK(cudaMemset(a.prev_spk, 0, sizeof(float) * L * N));
    CK(cudaMemset(a.fhat, 0, sizeof(float) * Q * N));
    CK(cudaMemset(a.pw, 0, sizeof(float2) * N));
    CK(cudaMemset(a.E, 0, sizeof(float4) * Q * NF));
    plan_back(e.get(), a);
    finish_init(e.get());
    *out = e.release();
  });
}

void aura_b200_destroy(aura_b200_engine* e) { delete e; }


// One block: launch FRONT then BACK; return as soon as the front has
// written the output. The background keeps running; the next call's front
// is stream-ordered after it, and feedback_estimate()/synchronize() wait
// for it explicitly.
namespace {
// One block whose input is already in the mapped staging buffer h_in: launch
// the block graph and wait until every k_front CTA has published its output
// word (h_out holds the block's output, and no CTA reads h_in any more).
void run_staged_block(aura_b200_engine* e) {
  const size_t n_in = (size_t)e->Qx * e->N;
  for (size_t i = 0; i < n_in; ++i)
    if (!std::isfinite(e->h_in[i])) fail(AURA_B200_E_NON_FINITE_INPUT, "input contains NaN or Inf");
  std::atomic_thread_fence(std::memory_order_release);
  const uint64_t nblk = device_block_hint(e);
  // (nothing else goes on the stream per block: an extra stream operation
  // between two block graphs costs device time at every block boundary)
  e->enqueue_block(e->g_block, e->args, e->use_outflag ? nullptr : e->ev_front);
  if (e->use_outflag) {
    // k_front's last CTA publishes block + 1 once every output is written
    wait_flag(e, nblk + 1, "block output");
  } else {
    wait_event(e, e->ev_front, "block output");
  }
  ++e->blocks;
}
}  // namespace

// Failure detection: every call's host-visible latency against
// the real-time budget N / f_s.
static void note_latency(aura_b200_engine* e, std::chrono::steady_clock::time_point t0) {
  const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
  e->last_us = us;
  if (us > e->max_us) e->max_us = us;
  if (us > e->budget_us) ++e->deadline_misses;
}

int aura_b200_process(aura_b200_engine* e, const float* in, float* out) {
  return guarded([&] {
    if (!e || !in || !out) fail(AURA_B200_E_INVALID_ARGUMENT, "null argument");
    const auto t0 = std::chrono::steady_clock::now();
    const size_t n_in = (size_t)e->Qx * e->N;
    for (size_t i = 0; i < n_in; ++i)
      if (!std::isfinite(in[i])) fail(AURA_B200_E_NON_FINITE_INPUT, "input contains NaN or Inf");
    CK(cudaSetDevice(e->device));
    check_shard_status(e);
    // every k_front CTA of the previous block (output and error-spectrum
    // CTAs) has published its word, so none still reads the staging buffer
    std::memcpy(e->h_in, in, n_in * sizeof(float));
    run_staged_block(e);
    std::memcpy(out, e->h_out, e->L * e->N * sizeof(float));
    note_latency(e, t0);
  });
}

int aura_b200_io_buffers(aura_b200_engine* e, float** in, float** out) {
  return guarded([&] {
    if (!e || !in || !out) fail(AURA_B200_E_INVALID_ARGUMENT, "null argument");
    *in = e->h_in;
    *out = e->h_out;
  });
}

int aura_b200_process_io(aura_b200_engine* e) {
  return guarded([&] {
    if (!e) fail(AURA_B200_E_INVALID_ARGUMENT, "null argument");
    const auto t0 = std::chrono::steady_clock::now();
    CK(cudaSetDevice(e->device));
    check_shard_status(e);
    run_staged_block(e);
    note_latency(e, t0);
  });
}

int aura_b200_deadline_stats(const aura_b200_engine* e, uint64_t* misses, double* max_us, double* last_us,
                             double* budget_us) {
  return guarded([&] {
    if (!e || !misses || !max_us || !last_us || !budget_us) fail(AURA_B200_E_INVALID_ARGUMENT, "null argument");
    *misses = e->deadline_misses;
    *max_us = e->max_us;
    *last_us = e->last_us;
    *budget_us = e->budget_us;
  });
}

int aura_b200_synchronize(aura_b200_engine* e) {
  return guarded([&] {
    CK(cudaSetDevice(e->device));
    wait_event(e, nullptr, "block background");
    check_shard_status(e);
  });
}

int aura_b200_reset(aura_b200_engine* e) {
  return guarded([&] {
    CK(cudaSetDevice(e->device));
    reset_state(e);
    e->deadline_misses = 0;
    e->max_us = e->last_us = 0.0;
  });
}

int aura_b200_feedback_estimate(aura_b200_engine* e, float* out) {
  return guarded([&] {
    if (!e->aur) fail(AURA_B200_E_INVALID_ARGUMENT, "not an auralizer");
    CK(cudaSetDevice(e->device));
    wait_event(e, nullptr, "block background");
    check_shard_status(e);
    // f^ stays in device memory (the background kernels never write mapped
    // host memory: a system-scope write over PCIe at the end of k_reduce
    // would stretch every block's kernel boundary); copy it out on demand
    CK(cudaMemcpy(out, e->args.fhat, sizeof(float) * e->P * e->N, cudaMemcpyDeviceToHost));
  });
}

int aura_b200_fdl_slot(aura_b200_engine* e, int which, size_t channel, size_t age,
                       float* out) {
  return guarded([&] {
    CK(cudaSetDevice(e->device));
    CK(cudaStreamSynchronize(e->stream));
    size_t cap, chans;
    const float4* base;
    if (which == 0) {
      cap = e->K;
      chans = (size_t)e->Qx;
      base = e->args.X;
    } else {
      if (!e->aur) fail(AURA_B200_E_INVALID_ARGUMENT, "not an auralizer");
      cap = e->KF + 1;
      chans = e->L;
      base = e->args.XA;
    }
    if (channel >= chans || age >= (which == 0 ? e->K : e->KF))
      fail(AURA_B200_E_INVALID_ARGUMENT, "delay-line index out of range");
    // device block b's spectrum lives at slot b % cap; age a is host block
    // (blocks-1-a), device block (blocks-1-a) + block_base
    std::vector<float2> buf(e->N, make_float2(0.f, 0.f));
    if (age < e->blocks) {  // tiled [ch][CTn][cap][CT]
      const uint64_t blk = e->blocks - 1 - age + e->block_base;
      const size_t slot = (size_t)(blk % (uint64_t)cap);
      const size_t CT = e->args.CT, CTn = e->args.CTn;
      for (size_t c = 0; c < CTn; ++c)
        CK(cudaMemcpy(buf.data() + 2 * c * CT, base + ((channel * CTn + c) * cap + slot) * CT,
                      sizeof(float4) * CT, cudaMemcpyDeviceToHost));
    }
    unpack_row(buf.data(), e->N, out);
  });
}

int aura_b200_set_input_gain(aura_b200_engine* e, float gain) {
  return guarded([&] {
    if (!e->aur) fail(AURA_B200_E_INVALID_ARGUMENT, "not an auralizer");
    CK(cudaSetDevice(e->device));
    CK(cudaStreamSynchronize(e->stream));
    e->args.gain = gain;
    e->dev_args.gain = gain;
    e->rebuild_graphs();
  });
}

float aura_b200_input_gain(const aura_b200_engine* e) { return e->args.gain; }
uint64_t aura_b200_blocks_processed(const aura_b200_engine* e) { return e->blocks; }
size_t aura_b200_partition_count(const aura_b200_engine* e) { return e->K; }
size_t aura_b200_fc_partition_count(const aura_b200_engine* e) { return e->aur ? e->KF : 0; }
size_t aura_b200_filter_length(const aura_b200_engine* e) { return e->n_h; }
int aura_b200_mode(const aura_b200_engine* e) { return e->mode; }


int aura_b200_filter_spectrum(aura_b200_engine* e, size_t row, size_t k, float* out) {
  return guarded([&] {
    const size_t rows = e->mode == AURA_B200_MIMO ? e->Q * e->L : e->L;
    if (row >= rows || k >= e->K) fail(AURA_B200_E_INVALID_ARGUMENT, "spectrum index out of range");
    CK(cudaSetDevice(e->device));
    size_t l = row, q = 0;
    if (e->mode == AURA_B200_MIMO) { q = row / e->L; l = row % e->L; }
    const size_t NF = e->N / 2;
    const size_t Qh = e->mode == AURA_B200_MIMO ? e->Q : 1;
    std::vector<float2> buf(e->N);
    if (k == 0) {
      CK(cudaMemcpy(buf.data(), e->args.H0 + (l * Qh + q) * NF, sizeof(float2) * e->N,
                    cudaMemcpyDeviceToHost));
    } else {  // Ht [L/LT][CTn][T][LT][CT]
      const size_t CT = e->args.CT, CTn = e->args.CTn, LT = e->LT;
      const size_t Kt = e->K - 1, T = Qh * Kt, t = q * Kt + k - 1, g = l / LT, i = l % LT;
      for (size_t c = 0; c < CTn; ++c)
        CK(cudaMemcpy(buf.data() + 2 * c * CT, e->args.Ht + (((g * CTn + c) * T + t) * LT + i) * CT,
                      sizeof(float4) * CT, cudaMemcpyDeviceToHost));
    }
    unpack_row(buf.data(), e->N, out);
  });
}

int aura_b200_afc_coeffs(aura_b200_engine* e, float* out) {
  return guarded([&] {
    if (!e->aur) fail(AURA_B200_E_INVALID_ARGUMENT, "not an auralizer");
    CK(cudaSetDevice(e->device));
    CK(cudaStreamSynchronize(e->stream));
    std::vector<float4> buf(e->w_elems);
    CK(cudaMemcpy(buf.data(), e->args.W, sizeof(float4) * e->w_elems, cudaMemcpyDeviceToHost));
    // tiled [CTn][U][P][CT] -> reference rows [p][l][k], N + 1 bins each
    const size_t CT = e->args.CT, CTn = e->args.CTn, P = e->P, U = e->L * e->KF;
    std::vector<float4> row(e->N / 2);
    for (size_t p = 0; p < P; ++p)
      for (size_t u = 0; u < U; ++u) {
        for (size_t c = 0; c < CTn; ++c)
          std::memcpy(&row[c * CT], &buf[((c * U + u) * P + p) * CT], sizeof(float4) * CT);
        unpack_row(reinterpret_cast<const float2*>(row.data()), e->N,
                   out + (p * U + u) * 2 * (e->N + 1));
      }
  });
}

int aura_b200_afc_load_coeffs(aura_b200_engine* e, const float* in, int as_initial) {
  return guarded([&] {
    if (!e || !in) fail(AURA_B200_E_INVALID_ARGUMENT, "null argument");
    if (!e->aur) fail(AURA_B200_E_INVALID_ARGUMENT, "not an auralizer");
    const size_t N = e->N, CT = e->args.CT, CTn = e->args.CTn, P = e->P, U = e->L * e->KF;
    // reference rows [p][l][k] of N + 1 bins -> tiled [CTn][U][P][CT]; the
    // DC and Nyquist bins must be real (dft.hpp:115-117's inverse() check)
    std::vector<float4> buf(e->w_elems);
    for (size_t p = 0; p < P; ++p)
      for (size_t u = 0; u < U; ++u) {
        const float* r = in + (p * U + u) * 2 * (N + 1);
        if (r[1] != 0.0f || r[2 * N + 1] != 0.0f)
          fail(AURA_B200_E_NON_REAL_EDGE_BINS, "DC and Nyquist bins must have zero imaginary part");
        std::vector<float2> packed(N);
        packed[0] = make_float2(r[0], r[2 * N]);
        for (size_t j = 1; j < N; ++j) packed[j] = make_float2(r[2 * j], r[2 * j + 1]);
        const float4* pk = reinterpret_cast<const float4*>(packed.data());
        for (size_t c = 0; c < CTn; ++c)
          std::memcpy(&buf[((c * U + u) * P + p) * CT], pk + c * CT, sizeof(float4) * CT);
      }
    CK(cudaSetDevice(e->device));
    CK(cudaStreamSynchronize(e->stream));
    CK(cudaMemcpy(e->args.W, buf.data(), sizeof(float4) * e->w_elems, cudaMemcpyHostToDevice));
    if (as_initial && e->W0) CK(cudaMemcpy(e->W0, buf.data(), sizeof(float4) * e->w_elems, cudaMemcpyHostToDevice));
  });
}

}  // extern "C"
