// copy_kernels.cu -- reclaim gather-copy: the pages invalidated by apply_reclaim, in the
// reference's report order (request ascending, page id ascending; memory.cpp:176-179),
// from their physical HBM slots into pinned host memory over PCIe.
//
// Work unit = one chunk (default 64 KiB) of one page, claimed from an HBM cursor so a few
// CTAs stream the whole list while the rest of the GPU stays with online work.  Each thread
// keeps kVec 16-byte loads in flight (ld.global.nc.L1::no_allocate -- the pool is read once),
// then issues 16-byte stores to the host-mapped destination (posted PCIe writes).  The rate
// bound is a GCRA token bucket on %globaltimer whose state (the theoretical arrival time) lives
// in the pool, so it holds across copy launches: in any window of length w the copies issue at
// most rate * w + burst + one chunk bytes.
// No UVM: the destination is cudaHostAlloc'd / registered memory, never managed memory.
#include "valve_kernels.h"

namespace valve {

namespace {

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void st_host(uint4* p, const uint4& v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

__device__ __forceinline__ void start_time(unsigned long long* t_first) {
  atomicCAS(t_first, 0ull, globaltimer_ns());
}

// GCRA pacing of one chunk of `bytes`: reserve [s, s + bytes * ns_per_byte) on the pool's
// virtual timeline, s = max(tat, now - burst_ns), and start at s.  Consecutive reservations
// never overlap, and s >= now - burst_ns, so chunks starting inside any window [a, b] have
// s in [a - burst_ns, b]: at most (b - a) * rate + burst + one chunk bytes.
__device__ __forceinline__ void pace(const CopyArgs& A, int64_t bytes, long long c) {
  if (A.ns_per_byte > 0.0) {
    const unsigned long long cost = (unsigned long long)((double)bytes * A.ns_per_byte);
    const unsigned long long now = globaltimer_ns();
    const unsigned long long burst = (unsigned long long)A.burst_ns;
    const unsigned long long floor = now > burst ? now - burst : 0ull;
    unsigned long long old = *(volatile unsigned long long*)A.tat, s;
    for (;;) {
      s = old > floor ? old : floor;
      const unsigned long long prev = atomicCAS(A.tat, old, s + cost);
      if (prev == old) break;
      old = prev;
    }
    while (globaltimer_ns() < s) __nanosleep(1000);
  }
  if (A.trace) A.trace[c] = globaltimer_ns();
}

// Publishes every completed wave in order (any thread may call; CAS hands each wave to one).
__device__ __forceinline__ void publish_waves(const CopyArgs& A, unsigned per_wave) {
  __threadfence();  // this chunk's count before the read of wave_next (store-buffer pattern)
  for (;;) {
    const unsigned w = *(volatile unsigned*)A.wave_next;
    if (w >= (unsigned)A.n_waves) break;
    if (*(volatile unsigned*)&A.wave_done[w] < per_wave) break;
    if (atomicCAS(A.wave_next, w, w + 1) == w) atomicMax(A.landed, A.wave_base + w + 1);
    __threadfence();
  }
}

// Last CTA out publishes the whole copy (paths without per-wave publication, and a backstop).
__device__ __forceinline__ void publish_all(const CopyArgs& A) {
  __threadfence();
  if (atomicAdd(A.ctas_done, 1u) == gridDim.x - 1 && A.n_waves > 0)
    atomicMax(A.landed, A.wave_base + (unsigned long long)A.n_waves);
}

// Source offset in the page store, destination offset and length of chunk c of the report:
// page-major (page = c / cpp) or wave-major (wave = c / n_pages: bytes [wave * chunk, ...) of
// every page, so the landed counter can publish a wave once all pages' wave bytes are read), or
// located by the chunk prefix when evicted requests have their own page sizes.
__device__ __forceinline__ void locate(const CopyArgs& A, long long c, int64_t cpp, int64_t& src, int64_t& dst,
                                       int64_t& len) {
  if (A.ev_cbase) {  // variable page sizes: locate the evicted request by its chunk prefix
    int lo = 0, hi = A.n_ev - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (A.ev_cbase[mid] <= c) lo = mid;
      else hi = mid - 1;
    }
    const int64_t pb = A.ev_pbytes[lo];
    const int64_t cp = (pb + A.chunk_bytes - 1) / A.chunk_bytes;
    const int64_t local = c - A.ev_cbase[lo];
    const int64_t pg = local / cp, off = (local % cp) * A.chunk_bytes;
    src = (int64_t)A.phys[A.inv_off[lo] + pg] * A.slot_bytes + off;
    dst = A.ev_base[lo] + pg * pb + off;
    len = min(A.chunk_bytes, pb - off);
    return;
  }
  int64_t page, off;
  if (A.wave_major) {
    page = c % A.n_pages;
    off = (c / A.n_pages) * A.chunk_bytes;
  } else {
    page = c / cpp;
    off = (c % cpp) * A.chunk_bytes;
  }
  src = (int64_t)A.phys[page] * A.slot_bytes + off;
  dst = page * A.page_bytes + off;
  len = min(A.chunk_bytes, A.page_bytes - off);
}

}  // namespace

constexpr int kVec = 8;

// Chunk prefix of a report with per-request page sizes: cbase[e] = sum over earlier evicted
// requests of pages * ceil(page_bytes / chunk).
__global__ void k_copy_plan(const int64_t* ev_pbytes, const int* inv_off, int n_ev, int64_t chunk,
                            int64_t* cbase) {
  int64_t carry = 0;
  for (int base = 0; base < n_ev; base += blockDim.x) {
    const int e = base + threadIdx.x;
    const int64_t v = e < n_ev ? (int64_t)(inv_off[e + 1] - inv_off[e]) * ((ev_pbytes[e] + chunk - 1) / chunk) : 0;
    int64_t tot;
    const int64_t ex = block_excl_scan64(v, tot);
    if (e < n_ev) cbase[e] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) cbase[n_ev] = carry;
}

__global__ void __launch_bounds__(512) k_reclaim_copy(CopyArgs A) {
  __shared__ long long s_chunk;
  __shared__ int64_t s_src, s_dst, s_len;
  if (threadIdx.x == 0) start_time(A.t_first);
  const int64_t cpp = (A.page_bytes + A.chunk_bytes - 1) / A.chunk_bytes;
  const long long n_chunks = A.ev_cbase ? A.ev_cbase[A.n_ev] : A.n_chunks;
  long long prev = -1;  // thread 0: the chunk this CTA finished last (its wave is counted next)
  for (;;) {
    if (A.wave_major) __syncthreads();  // every thread's loads of chunk `prev` have returned
    if (threadIdx.x == 0) {
      if (prev >= 0 && A.wave_major) {
        const unsigned w = (unsigned)(prev / A.n_pages);
        if (atomicAdd(&A.wave_done[w], 1u) + 1u == (unsigned)A.n_pages) publish_waves(A, (unsigned)A.n_pages);
      }
      const long long c = (long long)atomicAdd(A.cursor, 1ull);
      s_chunk = c;
      prev = c;
      if (c < n_chunks) {
        int64_t so, d, l;
        locate(A, c, cpp, so, d, l);
        s_src = so, s_dst = d, s_len = l;
        pace(A, s_len, c);
      }
    }
    __syncthreads();
    const long long c = s_chunk;
    const int64_t src_off = s_src, dst_off = s_dst, len = s_len;
    __syncthreads();
    if (c >= n_chunks) break;
    const uint4* src = reinterpret_cast<const uint4*>(A.pages + src_off);
    uint4* dst = reinterpret_cast<uint4*>(A.dst + dst_off);
    const int nvec = (int)(len >> 4);
    const int step = blockDim.x * kVec;
    for (int base = 0; base < nvec; base += step) {
      uint4 v[kVec];
#pragma unroll
      for (int u = 0; u < kVec; ++u) {
        const int i = base + u * blockDim.x + threadIdx.x;
        if (i < nvec) v[u] = ld_stream(src + i);
      }
#pragma unroll
      for (int u = 0; u < kVec; ++u) {
        const int i = base + u * blockDim.x + threadIdx.x;
        if (i < nvec) st_host(dst + i, v[u]);
      }
    }
  }
  // stores retired system-wide before the completion stamp
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicMax(A.t_last, globaltimer_ns());
    publish_all(A);
  }
}

// Variant staging each chunk through shared memory with the bulk-copy engine:
// cp.async.bulk global->shared (mbarrier complete_tx), then cp.async.bulk shared->global
// into the host-mapped destination.  Double-buffered: the load of chunk i+1 overlaps the
// store of chunk i.
constexpr int kTmaChunk = 32768;

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* g, unsigned bytes, uint64_t* bar) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(s),
      "l"(g), "r"(bytes), "r"(b)
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* g, const void* smem, unsigned bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(s),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_le1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// One elected thread per CTA drives the bulk engine; each claimed chunk (any layout: page-major,
// wave-major or per-request page sizes) moves in kTmaChunk pieces, and its wave is counted as
// soon as its last piece has landed in shared memory (its HBM bytes are read), so the landed
// tickets advance exactly as with the register-staged kernel.
__global__ void __launch_bounds__(32) k_reclaim_copy_tma(CopyArgs A) {
  extern __shared__ __align__(128) unsigned char sbuf[];  // 2 x kTmaChunk
  __shared__ __align__(8) uint64_t bar[2];
  if (threadIdx.x != 0) return;
  start_time(A.t_first);
  mbar_init(&bar[0], 1);
  mbar_init(&bar[1], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int64_t cpp = (A.page_bytes + A.chunk_bytes - 1) / A.chunk_bytes;
  const long long n_chunks = A.ev_cbase ? A.ev_cbase[A.n_ev] : A.n_chunks;
  unsigned phase[2] = {0, 0};
  int buf = 0;
  for (;;) {
    const long long c = (long long)atomicAdd(A.cursor, 1ull);
    if (c >= n_chunks) break;
    int64_t so, d, len;
    locate(A, c, cpp, so, d, len);
    pace(A, len, c);
    const uint8_t* src = A.pages + so;
    uint8_t* dst = A.dst + d;
    for (int64_t o = 0; o < len; o += kTmaChunk) {
      const unsigned bytes = (unsigned)min((int64_t)kTmaChunk, len - o);
      unsigned char* sm = sbuf + buf * kTmaChunk;
      bulk_wait_read_le1();  // the store that last read this buffer has drained
      mbar_expect_tx(&bar[buf], bytes);
      bulk_g2s(sm, src + o, bytes, &bar[buf]);
      mbar_wait(&bar[buf], phase[buf]);
      phase[buf] ^= 1;
      bulk_s2g(dst + o, sm, bytes);
      buf ^= 1;
    }
    if (A.wave_major) {  // every byte of this chunk has been read out of HBM
      const unsigned w = (unsigned)(c / A.n_pages);
      if (atomicAdd(&A.wave_done[w], 1u) + 1u == (unsigned)A.n_pages) publish_waves(A, (unsigned)A.n_pages);
    }
  }
  bulk_wait_all();
  __threadfence_system();
  atomicMax(A.t_last, globaltimer_ns());
  publish_all(A);
}

// Scatter of host-resident pages back into HBM (the restore side of a reclaim that copied,
// e.g. evicted offline weight pages): host page i goes to block blk_of_page[i] of the
// request, i.e. to physical slot bt_row[blk]; 16-byte loads from the host-mapped source
// (PCIe reads), 16-byte stores to HBM.  Chunks are claimed from an HBM cursor.
__global__ void __launch_bounds__(512) k_restore_scatter(ScatterArgs A) {
  __shared__ long long s_chunk;
  const int64_t cpp = (A.page_bytes + A.chunk_bytes - 1) / A.chunk_bytes;
  for (;;) {
    if (threadIdx.x == 0) s_chunk = (long long)atomicAdd(A.cursor, 1ull);
    __syncthreads();
    const long long c = s_chunk;
    __syncthreads();
    if (c >= A.n_chunks) break;
    const int64_t page = c / cpp;
    const int64_t off = (c % cpp) * A.chunk_bytes;
    const int64_t len = min(A.chunk_bytes, A.page_bytes - off);
    const int blk = A.blk_of_page[page];
    const int phys = blk < *A.nblk ? A.bt_row[blk] : -1;
    if (phys < 0 || phys >= A.quarantine) {
      if (threadIdx.x == 0 && off == 0) atomicAdd(A.bad, 1ull);
      continue;
    }
    const uint4* src = reinterpret_cast<const uint4*>(A.src + page * A.page_bytes + off);
    uint4* dst = reinterpret_cast<uint4*>(A.pages + (int64_t)phys * A.slot_bytes + off);
    const int nvec = (int)(len >> 4);
    const int step = blockDim.x * kVec;
    for (int base = 0; base < nvec; base += step) {
      uint4 v[kVec];
#pragma unroll
      for (int u = 0; u < kVec; ++u) {
        const int i = base + u * blockDim.x + threadIdx.x;
        if (i < nvec) v[u] = src[i];
      }
#pragma unroll
      for (int u = 0; u < kVec; ++u) {
        const int i = base + u * blockDim.x + threadIdx.x;
        if (i < nvec) dst[i] = v[u];
      }
    }
  }
}

}  // namespace valve
