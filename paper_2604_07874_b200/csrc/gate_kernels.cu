// gate_kernels.cu -- the device-resident preemption gate and the gated offline workload.
//
// Reference mechanism: ChannelController disables the offline compute channel and the
// in-flight offline kernel is suspended with its remaining work saved
// (channel.cpp:13-20,64-79; sim.cpp:860-873 suspend_all_offline; resume sim.cpp:759-782).
// B200 equivalent without a driver change: a u32 `closed` word in HBM written by a
// stream memory operation (no SM needed), polled by lane 0 of every warp at each tile
// boundary with ld.acquire.gpu and broadcast with a shuffle.  A warp that sees the gate
// closed stops claiming tiles; the last warp of a CTA retires the CTA and decrements
// `live_ctas`; the online stream waits for live_ctas == 0 (cuStreamWaitValue32).  The
// context save is the HBM tile cursor: every claimed tile completes, unclaimed tiles are
// resumed by the next launch, so each tile runs exactly once across preemptions
// (work conservation, SPEC.md:207 / test_sim.cpp:105-131).
#include <cuda_bf16.h>

#include "valve_kernels.h"

namespace valve {

namespace {

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned ld_relaxed_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ float dot8(const uint4& kv, const float* q) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&kv);
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(h[i]);
    s = fmaf(f.x, q[2 * i], s);
    s = fmaf(f.y, q[2 * i + 1], s);
  }
  return s;
}

}  // namespace

// One tile = one chunk of one (request, page).  The page is read through the block table
// as bf16 and reduced against a fixed query vector (fp32 accumulate): the memory-bound
// shape of a decode-attention score pass.  A block-table entry equal to the quarantine page
// (the reclaim remap) is never dereferenced; it is counted as a canary hit instead.
__global__ void __launch_bounds__(256) k_offline_decode(OfflineArgs A) {
  __shared__ int s_exited;
  const int lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  if (threadIdx.x == 0) s_exited = 0;
  __syncthreads();
  float q[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) q[i] = 0.0625f * (float)((lane * 8 + i) % 16 - 8);
  unsigned long long done = 0;
  const unsigned long long total = (unsigned long long)A.tile_prefix[A.n_requests];
  const unsigned long long per = (total + kStripes - 1) / kStripes;
  int stripe = (blockIdx.x * 7 + (threadIdx.x >> 5) * 13) % kStripes, visited = 0;  // lane 0 state
  // The gate read for the next claim is issued at the start of the current tile (relaxed: the
  // gate publishes no data) and consumed at its end, so its latency hides under the tile's
  // loads; a gate raised mid-tile is therefore seen one tile late at most (quiesce <= 2 tiles).
  unsigned gate_seen = A.poll ? ld_acquire_gpu(&A.g->closed) : 0u;
  for (;;) {
    long long tile = -1;
    if (lane == 0) {
      bool stop = false;
      if (gate_seen) {
        stop = true;
        atomicCAS(&A.g->t_first_seen, 0ull, globaltimer_ns());
      }
      while (!stop && visited < kStripes) {  // claim from this warp's stripe, then move on
        const unsigned long long local = atomicAdd(&A.g->cursor[stripe], 1ull);
        const unsigned long long t = (unsigned long long)stripe * per + local;
        if (local < per && t < total) {
          tile = (long long)t;
          break;
        }
        stripe = (stripe + 1) % kStripes;
        ++visited;
      }
    }
    tile = __shfl_sync(kFull, tile, 0);
    if (tile < 0) break;
    if (A.poll && lane == 0) gate_seen = ld_relaxed_gpu(&A.g->closed);  // consumed next round
    // locate (request, page, chunk): binary search over the tile prefix
    int lo = 0, hi = A.n_requests - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (A.tile_prefix[mid] <= tile) lo = mid;
      else hi = mid - 1;
    }
    const int64_t local = tile - A.tile_prefix[lo];
    const int page = (int)(local / A.chunks_per_page);
    const int64_t off = (local % A.chunks_per_page) * A.chunk_bytes;
    const int row = A.rows ? A.rows[lo] : lo;  // rows == nullptr: every request row
    const int phys = A.bt[(int64_t)row * A.P + page];
    float acc = 0.f;
    if (phys == A.quarantine || phys < 0) {
      if (lane == 0) atomicAdd(&A.g->canary, 1ull);
    } else {
      const int64_t len = min(A.chunk_bytes, A.page_bytes - off);
      const uint4* src = reinterpret_cast<const uint4*>(A.pages + (int64_t)phys * A.slot_bytes + off);
      const int nvec = (int)(len >> 4);
      for (int base = 0; base < nvec; base += 32 * 8) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = base + u * 32 + lane;
          v[u] = i < nvec ? ld_stream(src + i) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += dot8(v[u], q);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
    if (lane == 0) {
      if (A.out) A.out[tile] = acc;
      else if (acc == 1.2345e-30f) atomicAdd(&A.g->canary, 0ull);  // keeps the loads live
    }
    ++done;
  }
  // warp done: publish its tiles, then the CTA's last warp retires the CTA (the quiesce ack)
  if (lane == 0 && done) atomicAdd(&A.g->tiles_done, done);
  if (lane == 0 && atomicAdd(&s_exited, 1) == nw - 1) {
    __threadfence();
    if (atomicSub(&A.g->live_ctas, 1u) == 1u) {
      A.g->t_quiesced = globaltimer_ns();
      __threadfence_system();
    }
  }
}

// Diagnostic raise from a one-thread kernel: stamps %globaltimer next to the gate store so the
// device-side preempt-to-quiesce (t_quiesced - t_raise) can be split from the stream-memop and
// event overheads.  Needs a free SM slot (the memop raise does not).
__global__ void k_gate_raise_stamp(GateDev* g, unsigned gen) {
  g->t_first_seen = 0;
  g->gen = gen;
  g->t_raise = globaltimer_ns();
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&g->closed), "r"(1u) : "memory");
}

}  // namespace valve
