// gemm_kernels.cu -- the gated offline GEMM: a persistent tcgen05/TMA bf16 GEMM whose tile loop
// honours the preemption gate ("persistent tile-looped kernels, GEMM via tcgen05
// tiles ... every tile executes exactly once across preemptions").
//
// C[m, n] = sum_k A[m, k] * B[n, k]   (A activations, B an nn.Linear weight, both K-major bf16,
// fp32 accumulation in TMEM, bf16 output).
//
// Per CTA (one per SM, 256 threads):
//   warp 0 lane 0 : TMA producer  -- 128x64 A box + 256x64 B box per k-block, SWIZZLE_128B,
//                                    into a kStages-deep smem ring (full/empty mbarriers)
//   warp 1 lane 0 : MMA issuer    -- 4 x tcgen05.mma.cta_group::1.kind::f16 (M=128, N=256,
//                                    K=16) per k-block, tcgen05.commit frees the smem stage
//   warp 2        : TMEM owner    -- tcgen05.alloc / dealloc of 2 x 256 fp32 columns (two
//                                    accumulators: the epilogue of tile j overlaps the
//                                    mainloop of tile j+1)
//   warps 4..7    : epilogue      -- tcgen05.ld 32x32b.x32, bf16 pack, 16-byte global stores
// Tiles (128 x 256 of C) are claimed from the gate's striped HBM cursors by thread 0 after reading the
// gate word; a closed gate ends the loop, so the in-flight tile always completes (quiesce <= one
// tile) and unclaimed tiles resume on the next launch.  The CTA's retirement is the same
// live_ctas ack the decode kernel gives (gate_kernels.cu).
#include <cuda.h>
#include <cuda_bf16.h>

#include "valve_kernels.h"

namespace valve {

namespace {

constexpr int kBM = 128, kBN = 256, kBK = 64, kUK = 16;
constexpr int kABytes = kBM * kBK * 2;  // 16 KiB
constexpr int kBBytes = kBN * kBK * 2;  // 32 KiB
constexpr int kStageBytes = kABytes + kBBytes;
constexpr uint32_t kTmemCols = 256;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
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
      "W_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
          "r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}
// K-major operand tile written by TMA with SWIZZLE_128B: 128-byte rows, 8-row (1024 B) atoms
// stacked along M/N -> stride byte offset 1024, layout type 2 (SWIZZLE_128B), descriptor
// version 1 (sm_100).  Advancing K by 16 bf16 inside the 128-byte atom moves the start by 32 B.
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// kind::f16 instruction descriptor: D f32, A/B bf16, both K-major, N = 256, M = 128
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kBN >> 3) << 17) |
                            ((uint32_t)(kBM >> 4) << 24);

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accum) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(kIdesc), "r"(accum));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}


// ---- cluster helpers (pair mode: two CTAs of a cluster share each B tile via TMA multicast)
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void st_cluster_s64(uint32_t caddr, long long v) {
  asm volatile("st.shared::cluster.s64 [%0], %1;" ::"r"(caddr), "l"(v) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t caddr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(caddr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WC_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

// ---- cta_group::2 (CTA pair on one TPC): the leader issues M=256 MMAs that read A rows and
// B columns from both CTAs' shared memory and write each CTA's TMEM
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;  // shared::cluster address bit 24 = CTA rank in the pair
// kind::f16, D f32, A/B bf16 K-major, M = 256, N = 256
constexpr uint32_t kIdesc2 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(256 >> 3) << 17) |
                             ((uint32_t)(256 >> 4) << 24);
__device__ __forceinline__ void mma_bf16_2sm(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accum) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(kIdesc2), "r"(accum));
}
__device__ __forceinline__ void mma_commit_2sm(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
// both CTAs load their half; completion bytes land on the LEADER's barrier (same offset)
__device__ __forceinline__ void tma_load_2d_2sm(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar) & kPeerMask), "r"(x), "r"(y)
      : "memory");
}

}  // namespace

// kPair = false: one CTA per 128x256 tile of C (tcgen05.mma.cta_group::1, M=128).
// kPair = true : a CTA pair (2-CTA cluster on one TPC) per 256x256 tile with
//   tcgen05.mma.cta_group::2 (M=256): CTA r holds rows 128r.. of A and columns 128r.. of B for
//   each k-block (32 KiB per SM per stage instead of 48, so 6 stages fit), the leader (rank 0)
//   issues the MMAs, which read both CTAs' shared memory and accumulate each CTA's 128 rows in its
//   own TMEM.  Both CTAs' TMA loads complete on the leader's full barrier; the leader's commits
//   multicast to both CTAs' empty / tmem_full barriers; both epilogues must drain before the
//   leader reuses an accumulator.  Rank 0 also owns the tile schedule and the gate check and
//   publishes each tile id to both CTAs (st.shared::cluster + remote mbarrier arrive).
template <bool kPair>
__device__ __forceinline__ void offline_gemm_body(const CUtensorMap& map_a, const CUtensorMap& map_b,
                                                  const GemmArgs& G) {
  constexpr int kStages = kPair ? kGemmStagesPair : kGemmStages;
  constexpr int kBRows = kPair ? kBN / 2 : kBN;           // B rows this CTA loads per k-block
  constexpr int kStage = kABytes + kBRows * kBK * 2;       // bytes per stage in this CTA
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[kStages], empty_bar[kStages];
  __shared__ __align__(8) uint64_t tile_full[2], tile_empty[2], tmem_full[2], tmem_empty[2];
  __shared__ long long s_tile[2];
  __shared__ uint32_t s_tmem;
  // 1024-byte alignment for the swizzled operand tiles
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = kPair ? cluster_rank() : 0u;
  constexpr uint16_t kBoth = 0x3;
  // tile-id readers: per CTA 128 epilogue threads + the MMA thread (leader) / producer (rank 1)
  constexpr uint32_t kReaders = kPair ? 2 * 129 : 129;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tile_full[s], 1);                     // scheduler published the slot's tile id
      mbar_init(&tile_empty[s], kReaders);             // every reader took it (rank 0's counts)
      mbar_init(&tmem_full[s], 1);                     // tcgen05.commit: accumulator complete
      mbar_init(&tmem_empty[s], kPair ? 256 : 128);    // epilogue(s) drained the accumulator
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_b) : "memory");
  }
  if (kPair) cluster_sync();  // the peer's barriers exist before anyone arrives on them
  if (warp == 2) {
    if (kPair) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                   "r"(2 * kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                   "r"(2 * kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  fence_before();
  if (kPair) cluster_sync();
  else __syncthreads();
  fence_after();
  const uint32_t tmem = s_tmem;
  constexpr int kTM = kPair ? 2 * kBM : kBM;  // rows of C per scheduled tile
  const int tiles_m = G.m / kTM;
  const int kblocks = G.k / kBK;
  unsigned long long done = 0;
  // "slot consumed" / "accumulator drained" go to rank 0's barriers (remote for rank 1)
  auto consumed = [&](uint32_t slot) {
    if (kPair) mbar_arrive_cluster(mapa(smem_u32(&tile_empty[slot]), 0));
    else mbar_arrive(&tile_empty[slot]);
  };
  auto wait_tile = [&](uint32_t slot, uint32_t parity) {
    if (kPair) mbar_wait_cluster(&tile_full[slot], parity);
    else mbar_wait(&tile_full[slot], parity);
  };
  if (warp == 0 && lane == 0) {
    // ---------------- scheduler (rank 0) + TMA producer (both ranks).  Tile j goes through smem
    // slot j & 1; the producer runs at most one tile ahead of the epilogue (two accumulators).
    // one HBM cursor (148 claimers at one claim per ~15 us do not contend), so the tiles in
    // flight are consecutive claims; claims are rasterised M-fastest, so the clusters running
    // together share each B (weight) tile through L2 and A stays L2-resident
    const unsigned long long total = (unsigned long long)G.total_tiles;
    uint32_t it = 0;
    for (uint32_t j = 0;; ++j) {
      const uint32_t slot = j & 1, use = j >> 1;
      long long t = -1;
      if (rank == 0) {
        if (G.poll && ld_acquire(&G.g->closed)) {
          atomicCAS(&G.g->t_first_seen, 0ull, globaltimer_ns());
        } else {
          const unsigned long long c = atomicAdd(&G.g->cursor[0], 1ull);
          if (c < total) t = (long long)c;
        }
        if (kPair) mbar_wait_cluster(&tile_empty[slot], (use & 1) ^ 1);
        else mbar_wait(&tile_empty[slot], (use & 1) ^ 1);
        s_tile[slot] = t;
        if (kPair) {
          st_cluster_s64(mapa(smem_u32(&s_tile[slot]), 1), t);
          mbar_arrive_cluster(mapa(smem_u32(&tile_full[slot]), 1));
        }
        mbar_arrive(&tile_full[slot]);
      } else {  // pair rank 1: follow rank 0's schedule
        wait_tile(slot, use & 1);
        t = s_tile[slot];
        consumed(slot);
      }
      if (t < 0) break;
      const int m0 = (int)(t % tiles_m) * kTM + (int)rank * kBM;
      const int n0 = (int)(t / tiles_m) * kBN + (int)rank * (kBN - kBRows);
      for (int kb = 0; kb < kblocks; ++kb, ++it) {
        const uint32_t st = it % kStages, ph = (it / kStages) & 1u;
        mbar_wait(&empty_bar[st], ph ^ 1);
        uint8_t* sa = smem + st * kStage;
        uint8_t* sb = sa + kABytes;
        if (kPair) {
          // the leader's full barrier collects both CTAs' A and B halves
          if (rank == 0) mbar_expect_tx(&full_bar[st], 2 * kStage);
          tma_load_2d_2sm(sa, &map_a, &full_bar[st], kb * kBK, m0);
          tma_load_2d_2sm(sb, &map_b, &full_bar[st], kb * kBK, n0);
        } else {
          mbar_expect_tx(&full_bar[st], kStage);
          tma_load_2d(sa, &map_a, &full_bar[st], kb * kBK, m0);
          tma_load_2d(sb, &map_b, &full_bar[st], kb * kBK, n0);
        }
      }
    }
  } else if (warp == 1 && lane == 0 && rank == 0) {
    // ---------------- MMA issuer (leader): accumulator j & 1 (TMEM columns 0 / 256)
    uint32_t it = 0;
    for (uint32_t j = 0;; ++j) {
      const uint32_t slot = j & 1, use = j >> 1;
      wait_tile(slot, use & 1);
      const long long t = s_tile[slot];
      consumed(slot);
      if (t < 0) break;
      if (kPair) mbar_wait_cluster(&tmem_empty[slot], (use & 1) ^ 1);
      else mbar_wait(&tmem_empty[slot], (use & 1) ^ 1);
      fence_after();
      const uint32_t acc = tmem + slot * kTmemCols;
      for (int kb = 0; kb < kblocks; ++kb, ++it) {
        const uint32_t st = it % kStages, ph = (it / kStages) & 1u;
        mbar_wait(&full_bar[st], ph);
        fence_after();
        const uint32_t sa = smem_u32(smem + st * kStage);
        const uint32_t sb = sa + kABytes;
#pragma unroll
        for (int k = 0; k < kBK / kUK; ++k) {
          if (kPair) mma_bf16_2sm(acc, smem_desc(sa + k * kUK * 2), smem_desc(sb + k * kUK * 2), (kb | k) != 0);
          else mma_bf16(acc, smem_desc(sa + k * kUK * 2), smem_desc(sb + k * kUK * 2), (kb | k) != 0);
        }
        // the stage is free once these MMAs have read it -- in both CTAs of a pair
        if (kPair) mma_commit_2sm(&empty_bar[st], kBoth);
        else mma_commit(&empty_bar[st]);
      }
      if (kPair) mma_commit_2sm(&tmem_full[slot], kBoth);
      else mma_commit(&tmem_full[slot]);
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: TMEM lanes 32*(warp-4).. -> rows of C, overlapped with the
    // next tile's mainloop in the other accumulator
    const int q = warp - 4;
    for (uint32_t j = 0;; ++j) {
      const uint32_t slot = j & 1, use = j >> 1;
      wait_tile(slot, use & 1);
      const long long t = s_tile[slot];
      consumed(slot);
      if (t < 0) break;
      const int m0 = (int)(t % tiles_m) * kTM + (int)rank * kBM, n0 = (int)(t / tiles_m) * kBN;
      mbar_wait(&tmem_full[slot], use & 1);
      fence_after();
      const int row = m0 + q * 32 + lane;
      __nv_bfloat16* crow = reinterpret_cast<__nv_bfloat16*>(G.c) + (int64_t)row * G.n + n0;
#pragma unroll 1
      for (int c0 = 0; c0 < kBN; c0 += 32) {
        uint32_t v[32];
        const uint32_t taddr = tmem + slot * kTmemCols + ((uint32_t)(q * 32) << 16) + (uint32_t)c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
              "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
              "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
              "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        uint4* dst = reinterpret_cast<uint4*>(crow + c0);
#pragma unroll
        for (int jj = 0; jj < 4; ++jj)
          dst[jj] = make_uint4(pack_bf16(__uint_as_float(v[8 * jj + 0]), __uint_as_float(v[8 * jj + 1])),
                               pack_bf16(__uint_as_float(v[8 * jj + 2]), __uint_as_float(v[8 * jj + 3])),
                               pack_bf16(__uint_as_float(v[8 * jj + 4]), __uint_as_float(v[8 * jj + 5])),
                               pack_bf16(__uint_as_float(v[8 * jj + 6]), __uint_as_float(v[8 * jj + 7])));
      }
      fence_before();
      if (kPair) mbar_arrive_cluster(mapa(smem_u32(&tmem_empty[slot]), 0));
      else mbar_arrive(&tmem_empty[slot]);
      ++done;
    }
  }
  __syncthreads();
  // one count per scheduled tile (a pair's tile is counted by rank 0)
  if (threadIdx.x == 128 && done && rank == 0) atomicAdd(&G.g->tiles_done, done);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicSub(&G.g->live_ctas, 1u) == 1u) {
      G.g->t_quiesced = globaltimer_ns();
      __threadfence_system();
    }
  }
  fence_before();
  if (kPair) cluster_sync();  // no CTA leaves while its peer may still load / arrive into it
  else __syncthreads();
  fence_after();
  if (warp == 2) {
    if (kPair)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * kTmemCols));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * kTmemCols));
  }
}

__global__ void __launch_bounds__(256, 1)
    k_offline_gemm(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                   GemmArgs G) {
  offline_gemm_body<false>(map_a, map_b, G);
}

__global__ void __launch_bounds__(256, 1)
    k_offline_gemm_pair(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                        GemmArgs G) {
  offline_gemm_body<true>(map_a, map_b, G);
}

}  // namespace valve
