// loop.cuh -- k_loop: the whole block loop as ONE persistent cooperative
// kernel driven by a doorbell in pinned mapped host memory (launch mode 2).
//
// The graph mode (kernels.cuh / stream.cuh) pays a kernel launch and drain
// at every phase boundary and a graph launch per block. Here one CTA per SM
// stays resident across blocks and runs, for block n:
//
//   wait     CTA 0 polls the host doorbell (system scope), releases the grid
//   front    consumer warps of the first CTAs: k_front's work for their
//            loudspeakers (the leader publishes "input spectra pushed");
//            the last one publishes "output written" to the host mailbox;
//            then the canceller head for the same loudspeakers, and the
//            NLMS error spectra on P further CTAs ("head done" count)
//   stream   meanwhile, from the moment the block is released, every
//            CTA's producer lane streams its work items (stream.cuh); it
//            waits only before rows produced by this block's front half
//   reduce   grid barrier, k_reduce's work spread over the CTAs, grid
//            barrier, block done (mailbox bg_done)
//
// So the streaming starts while the output is still being computed, no
// phase boundary drains the machine, and the host sees the output through
// the mapped mailbox as soon as the last front CTA has written it.
//
// Every internal wait is bounded (kLoopTimeoutNs): a broken protocol sets
// the error word in the mailbox and ends the kernel instead of hanging the
// GPU. An idle engine (no doorbell for loop_idle_ns, 20 ms) parks: the
// kernel exits, so it never holds the SMs -- or a device-wide sync elsewhere
// in the process -- for long, and the host relaunches it on the next block.
#pragma once
#include "stream.cuh"

namespace aura_b200 {

constexpr unsigned long long kLoopTimeoutNs = 2ull * 1000 * 1000 * 1000;
constexpr unsigned long long kLoopStop = ~0ull;
constexpr int kLoopStampCap = 4096;
constexpr int kLoopStamps = 7;  // per block: released, output, X pushed, heads done, streamed, done, CTA 0 reduced

__device__ __forceinline__ unsigned long long ld_acquire_gpu_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_gpu_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// generic-proxy global writes (fronts, heads, the previous block) before
// this thread's later cp.async.bulk reads of them
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ void loop_fail(const BlockArgs& a) {
  atomicExch(&a.ctl->err, 1u);
  *reinterpret_cast<volatile unsigned*>(&a.mbox->err) = 1u;
  __threadfence_system();
}

// Spin (one thread) until *p >= target; false on timeout or a peer's error.
__device__ __forceinline__ bool spin_ge(const BlockArgs& a, const unsigned long long* p,
                                        unsigned long long target) {
  const unsigned long long t0 = globaltimer();
  while (ld_acquire_gpu_u64(p) < target) {
    if (*reinterpret_cast<volatile unsigned*>(&a.ctl->err)) return false;
    if (globaltimer() - t0 > kLoopTimeoutNs) {
      loop_fail(a);
      return false;
    }
  }
  return true;
}

// Grid-wide barrier of the cooperative grid (all threads of every CTA).
// Returns false in every thread if it timed out or a peer failed.
__device__ bool grid_sync(const BlockArgs& a, int* s_ok) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned* gen = &a.ctl->bar_gen;
    const unsigned g = ld_acquire_gpu_u32(gen);
    bool ok = true;
    __threadfence();
    if (atomicAdd(&a.ctl->bar_count, 1u) == gridDim.x - 1u) {
      a.ctl->bar_count = 0u;
      __threadfence();
      atomicAdd(gen, 1u);
    } else {
      const unsigned long long t0 = globaltimer();
      while (ld_acquire_gpu_u32(gen) == g) {
        if (*reinterpret_cast<volatile unsigned*>(&a.ctl->err) || globaltimer() - t0 > kLoopTimeoutNs) {
          ok = false;
          break;
        }
      }
    }
    if (!ok || *reinterpret_cast<volatile unsigned*>(&a.ctl->err)) {
      if (ok) ok = false;
      else loop_fail(a);
    }
    *s_ok = ok;
  }
  __syncthreads();
  return *s_ok != 0;
}

// The producer's dependencies in the loop: input spectra pushed by the
// leader (x_seq), canceller heads and error spectra done (head_seq).
struct LoopDeps {
  const BlockArgs* a;
  unsigned long long x_target, head_target;
  __device__ __forceinline__ const unsigned* abort() const { return &a->ctl->err; }
  __device__ __forceinline__ bool wait_front(uint32_t) const {
    const bool ok = spin_ge(*a, &a->ctl->x_seq, x_target);
    fence_proxy_async_global();
    return ok;
  }
  __device__ __forceinline__ bool wait_head(uint32_t) const {
    const bool ok = spin_ge(*a, &a->ctl->head_seq, head_target);
    fence_proxy_async_global();
    return ok;
  }
};

// grid = back_ctas (cooperative, one CTA per SM), kBackThreads threads.
// smem: [barriers + metadata | red | ring | front/head scratch]; the ring
// doubles as the reduction scratch (it is drained by then).
template <int LT, bool ELEM, int PT>
__global__ void __launch_bounds__(kBackThreads, 1) k_loop(const __grid_constant__ BlockArgs a) {
  extern __shared__ __align__(128) unsigned char bsm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(bsm);
  uint64_t* empty = full + kMaxStages;
  StageMeta* meta = reinterpret_cast<StageMeta*>(empty + kMaxStages);
  float4* red = reinterpret_cast<float4*>(bsm + kBackBarrierBytes);
  float4* slots = red + a.red_f4;
  float2* fsm = reinterpret_cast<float2*>(slots + (size_t)a.stages * a.slot_f4);  // front scratch
  __shared__ int s_ok;
  __shared__ unsigned long long s_go;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = a.stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, kConsumers / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  const uint32_t n0 = a.st->block;
  const int N = a.N;
  const int nfront = a.loop_front_ctas;
  const int P = PT > 0 ? a.P : 0;
  const int nerr = (PT > 0 && a.nlms) ? P : 0;  // error-spectrum CTAs
  const unsigned long long heads = PT > 0 ? (unsigned long long)(a.L + nerr) : 0ull;
  const int nred = a.red_syn_ctas + a.red_afc_ctas;
  const size_t in_stride = (size_t)(a.mode == 1 ? a.L : a.Q) * N;
  uint32_t qp = 0, qc = 0;  // producer / consumer stage counts (persist across blocks)
  const Consumers<kConsumers> team;

  for (uint32_t n = n0;; ++n) {
    // ------------------------------------------------------- wait for block n
    if (threadIdx.x == 0) {
      unsigned long long go;
      if (blockIdx.x == 0) {
        const unsigned long long t_idle = globaltimer();
        for (;;) {
          const unsigned long long d = ld_acquire_sys_u64(&a.mbox->doorbell);
          if (*reinterpret_cast<volatile unsigned*>(&a.mbox->stop)) {
            go = kLoopStop;
            break;
          }
          if (d > n) {
            go = (unsigned long long)n + 1;
            break;
          }
          if (globaltimer() - t_idle > a.loop_idle_ns) {
            // idle: park, so that an idle engine never holds every SM (and
            // device-wide syncs such as cudaFree elsewhere in the process
            // cannot wait on it); the host relaunches on the next block
            *reinterpret_cast<volatile unsigned*>(&a.mbox->parked) = 1u;
            __threadfence_system();
            go = kLoopStop;
            break;
          }
        }
        if (a.loop_stamps) a.loop_stamps[((n - n0) % kLoopStampCap) * kLoopStamps] = globaltimer();
        st_release_gpu_u64(&a.ctl->go, go);
      } else {
        for (;;) {  // idle is legitimate: no timeout while the leader waits for the host
          go = ld_acquire_gpu_u64(&a.ctl->go);
          if (go == kLoopStop || go >= (unsigned long long)n + 1) break;
          if (*reinterpret_cast<volatile unsigned*>(&a.ctl->err)) {
            go = kLoopStop;
            break;
          }
        }
      }
      s_go = go;
    }
    __syncthreads();
    if (s_go == kLoopStop) break;
    const float* in = a.in + (size_t)(n % (uint32_t)a.in_slots) * in_stride;
    const float* prev = (n & 1u) ? a.hist1 : a.prev_in;    // this block's window history
    float* cur = (n & 1u) ? a.prev_in : a.hist1;           // ... and the next block's
    const unsigned long long blk = (unsigned long long)(n - n0) + 1;

    if (warp == kConsumers / 32) {
      // ------------------------------------------------------------ stream
      if (lane == 0) {
        // hold the stream until the fronts have their inputs in (their loads
        // are the latency-critical path; under a saturated stream each L2
        // round trip costs microseconds)
        const LoopDeps deps{&a, blk * (unsigned long long)nfront, blk * heads};
        if (a.loop_hold && !deps.wait_front(n)) {
          // timed out: fall through, the producer posts its sentinel at once
        }
        fence_proxy_async_global();  // the previous block's generic writes (W, pw, ...)
        back_produce<LT, ELEM, PT, LoopDeps>(a, n, full, empty, slots, meta, qp, deps);
      }
    } else {
      // --------------------------------------------------------- front half
      const int b = blockIdx.x;
      if (b < nfront) {
        const int c0 = b * a.cpb, c1 = min(c0 + a.cpb, a.L);
        front_body(a, n, c0, c1, fsm, in, prev, cur, b == 0, team, [&] {
          // this CTA's input spectra pushed (the leader's, or elementwise its
          // own channels'): once every front CTA says so, X(age 0) is complete
          __threadfence();
          team.sync();
          if (threadIdx.x == 0 && atomicAdd(&a.ctl->x_seq, 1ull) + 1 == blk * (unsigned long long)nfront &&
              a.loop_stamps)
            a.loop_stamps[((n - n0) % kLoopStampCap) * kLoopStamps + 2] = globaltimer();
        });
        // outputs written: the last front CTA tells the host
        __threadfence_system();
        team.sync();
        if (threadIdx.x == 0) {
          const unsigned long long done = atomicAdd(&a.ctl->front_seq, 1ull) + 1;
          if (done == blk * (unsigned long long)nfront) {
            if (a.loop_stamps) a.loop_stamps[((n - n0) % kLoopStampCap) * kLoopStamps + 1] = globaltimer();
            st_release_sys_u64(&a.mbox->out_done, (unsigned long long)n + 1);
          }
        }
        if (PT > 0) {  // the canceller's stage 1 on the loudspeakers just produced
          const float2* tw = a.smem_tables ? fsm + front_work_f2(N, a.mode == 1 ? 1 : a.Q) : a.tw;  // staged by the front
          const float2* split = a.smem_tables ? tw + N / 2 : a.split;
          head_channels(a, n, c0, c1, fsm, tw, split, team);
          __threadfence();
          team.sync();
          if (threadIdx.x == 0 && atomicAdd(&a.ctl->head_seq, (unsigned long long)(c1 - c0)) + (c1 - c0) ==
                                      blk * heads && a.loop_stamps)
            a.loop_stamps[((n - n0) % kLoopStampCap) * kLoopStamps + 3] = globaltimer();
        }
      } else if (PT > 0 && b < nfront + nerr) {
        const float2* tw = a.tw;
        const float2* split = a.split;
        error_spectrum(a, b - nfront, in, fsm, tw, split, team);
        __threadfence();
        team.sync();
        if (threadIdx.x == 0 && atomicAdd(&a.ctl->head_seq, 1ull) + 1 == blk * heads && a.loop_stamps)
          a.loop_stamps[((n - n0) % kLoopStampCap) * kLoopStamps + 3] = globaltimer();
      }
      // ------------------------------------------------------------ stream
      back_consume<LT, ELEM, PT>(a, n, full, empty, meta, red, slots, qc, nullptr, &a.ctl->err);
    }

    // --------------------------------------------------------------- reduce
    if (!grid_sync(a, &s_ok)) break;
    if (blockIdx.x == 0 && threadIdx.x == 0 && a.loop_stamps)
      a.loop_stamps[((n - n0) % kLoopStampCap) * kLoopStamps + 4] = globaltimer();
    if (warp < kConsumers / 32) {
      float4* rsm = slots;  // the ring is drained
      for (int r = blockIdx.x; r < nred; r += gridDim.x) {
        reduce_prefetch(a, r, rsm, team);
        team.sync();
        reduce_part(a, r, n, rsm, &s_ok, team, reduce_tile_info(a, r));
        team.sync();
      }
      if (blockIdx.x == 0 && threadIdx.x == 0 && a.loop_stamps)
        a.loop_stamps[((n - n0) % kLoopStampCap) * kLoopStamps + 6] = globaltimer();
    }
    if (!grid_sync(a, &s_ok)) break;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      a.st->block = n + 1;
      a.tick[a.tick_queue] = 0u;  // the work queue, for block n + 1
      __threadfence();
      if (a.loop_stamps) a.loop_stamps[((n - n0) % kLoopStampCap) * kLoopStamps + 5] = globaltimer();
      st_release_sys_u64(&a.mbox->bg_done, (unsigned long long)n + 1);
    }
    // the queue reset must be visible before any producer claims for n + 1:
    // the claims happen after the next go, which CTA 0 publishes after this
  }
}

}  // namespace aura_b200
