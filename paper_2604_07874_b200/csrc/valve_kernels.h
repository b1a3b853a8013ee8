// valve_kernels.h -- kernel entry points shared between the .cu translation units.
#pragma once
#include <cuda.h>

#include "valve_common.cuh"

namespace valve {

// Device-side arguments of the selection kernels over a host-provided instance.
struct SelectArgs {
  int n, m, k, mode, nnz;
  const int* hid;
  const int64_t* mapped;
  const int* roff;
  const int* rref;     // dense cost index per ref, -1 = no cost entry
  const int64_t* cost;
  int64_t* marg;
  int* taken;
  int* ev;
  int* qoff;
  int* qcnt;
  int* qh;
  int* out;
  int* status;
  int64_t* result;
};

__global__ void k_online_grow(PoolDev P, int k, int64_t t);
__global__ void k_online_release(PoolDev P, int k, int64_t online_used);
__global__ void k_offline_reserve(PoolDev P, int64_t req, int pages, int64_t t, int max_off);
__global__ void k_offline_release(PoolDev P, int64_t req);
__global__ void k_ht_rehash(PoolDev P, const int* old_row, int old_hc);
__global__ void k_requests_on_handle(PoolDev P, int h, int64_t* out);
__global__ void k_handles_of_request(PoolDev P, int64_t req, int* out);
__global__ void k_offline_pages_of(PoolDev P, int64_t req);
__global__ void k_block_table(PoolDev P, int64_t req, int* out);
__global__ void k_snapshot_handles(PoolDev P);
__global__ void k_snapshot(PoolDev P);
__global__ void k_apply(PoolDev P, const int* ids, int k, int64_t t);
__global__ void k_reclaim_rows(PoolDev P);
__global__ void k_reclaim(PoolDev P, int k, int mode, int64_t t);
__global__ void k_reclaim_fused(PoolDev P, int k, int mode, int64_t t, int64_t seq);
__global__ void k_check_invariants(PoolDev P, int64_t online_used);
__global__ void k_fill_pages(PoolDev P);
__global__ void k_set_costs(PoolDev P, int n, const int64_t* reqs, const int64_t* costs, int which);
__global__ void k_select_instance(SelectArgs A);
__global__ void k_map_refs(const int64_t* reqs, int nnz, const int64_t* keys, int m, int* rref);
__global__ void k_tile_prefix(const int* npages, int n, int cpp, int64_t* prefix,
                              unsigned long long* total_out, unsigned* frozen);
__global__ void k_evicted_cost(SelectArgs A, const int* pick, int n_pick);
extern __device__ long long g_greedy_cycles[2];
extern __device__ long long g_select_ns[5];
extern __device__ long long g_apply_ns[10];

// reclaim copy (copy_kernels.cu)
struct CopyArgs {
  const uint8_t* pages;
  int64_t slot_bytes, page_bytes, chunk_bytes;
  const int* phys;
  int n_pages;
  int64_t n_chunks;
  uint8_t* dst;  // device alias of pinned host memory
  double ns_per_byte;  // 0 = unbounded
  int64_t burst_bytes;
  unsigned long long* cursor;
  unsigned long long* t_first;
  unsigned long long* t_last;
  // variable page sizes (some request has set_page_bytes): ev_cbase != nullptr
  const int64_t* ev_pbytes;  // page size per evicted request
  const int64_t* ev_base;    // destination byte offset per evicted request
  const int64_t* ev_cbase;   // chunk prefix per evicted request [n_ev + 1]
  const int* inv_off;        // first report page of each evicted request
  int n_ev;
  // Wave-major order (uniform page size): chunk c covers byte range wave*chunk of page
  // c % n_pages, wave = c / n_pages, so wave w holds the same slot bytes of every page.  Once
  // every chunk of wave w has been read from HBM the kernel publishes wave_base + w + 1 to the
  // pool-global, monotone `landed` word, in wave order: an online write into a reclaimed slot
  // may proceed (cuStreamWaitValue64 >= ticket) once the waves covering its bytes are out.
  int wave_major;
  int n_waves;                   // waves this copy publishes (0: no chunks)
  unsigned* wave_done;           // [n_waves] chunks read per wave
  unsigned* wave_next;           // next wave to publish
  unsigned* ctas_done;           // CTAs finished (the last one publishes everything)
  unsigned long long* landed;    // pool-global published-wave counter
  unsigned long long wave_base;  // global index of this copy's wave 0
  // Rate bound across launches: a GCRA token bucket whose theoretical arrival time (ns) lives
  // in the pool, so back-to-back copies share one budget of rate * window + burst bytes.
  unsigned long long* tat;
  double burst_ns;
  unsigned long long* trace;     // optional [n_chunks]: issue time of each chunk (tests)
};
__global__ void k_reclaim_copy(CopyArgs A);
__global__ void k_copy_plan(const int64_t* ev_pbytes, const int* inv_off, int n_ev, int64_t chunk,
                            int64_t* cbase);
__global__ void k_reclaim_copy_tma(CopyArgs A);

// restore scatter (copy_kernels.cu): host pages back into a request's (re-reserved) slots
struct ScatterArgs {
  uint8_t* pages;
  int64_t slot_bytes, page_bytes, chunk_bytes;
  const int* bt_row;       // the request's block table row
  const int* blk_of_page;  // block index of host page i
  const int* nblk;         // the request's mapped block count
  int n_pages;
  int64_t n_chunks;
  const uint8_t* src;      // device alias of pinned host memory (n_pages * page_bytes)
  int quarantine;
  unsigned long long* cursor;
  unsigned long long* bad;  // pages whose block is not mapped (skipped)
};
__global__ void k_restore_scatter(ScatterArgs A);

// gate (gate_kernels.cu)
// The tile space of a work list is split into kStripes contiguous stripes, each with its own
// claim cursor (a single cursor saturates one L2 atomic unit at ~9k claiming warps).
constexpr int kStripes = 64;
struct GateDev {
  unsigned int closed;        // polled word
  unsigned int gen;
  unsigned int live_ctas;     // gated CTAs resident or pending
  unsigned int quiesced_gen;
  unsigned long long t_first_seen;
  unsigned long long t_quiesced;
  unsigned long long tiles_done;
  unsigned long long canary;
  unsigned long long total;               // tiles of the current work list
  unsigned long long cursor[kStripes];    // per-stripe claims (the context save)
  unsigned long long t_raise;             // %globaltimer of a kernel-issued raise (diagnostic)
  unsigned long long stripes;             // cursors the current work list uses (0 = kStripes)
  unsigned int frozen;                    // decode work list (tile prefix) fixed since the reset
  unsigned int pad_;
};
__global__ void k_gate_raise_stamp(GateDev* g, unsigned gen);
struct OfflineArgs {
  GateDev* g;
  const uint8_t* pages;
  int64_t slot_bytes, page_bytes, chunk_bytes;
  int chunks_per_page;
  const int* bt;
  int P, quarantine;
  const int* rows;
  const int64_t* tile_prefix;  // [n_requests+1] tiles before request i
  int n_requests;
  int64_t total_tiles;
  float* out;
  int poll;
};
__global__ void k_offline_decode(OfflineArgs A);

// gated offline GEMM (gemm_kernels.cu): 128x256 tiles claimed from the gate's striped cursors
constexpr int kGemmStages = 4;      // 48 KiB per stage (A 128x64 + B 256x64)
constexpr int kGemmStagesPair = 6;  // 32 KiB per stage per CTA (A 128x64 + B 128x64)
constexpr int kGemmSmemBytes = kGemmStages * (128 * 64 + 256 * 64) * 2 + 1024;
struct GemmArgs {
  GateDev* g;
  void* c;  // bf16 [m, n]
  int m, n, k;
  long long total_tiles;
  int poll;
};
__global__ void k_offline_gemm(const __grid_constant__ CUtensorMap map_a,
                               const __grid_constant__ CUtensorMap map_b, GemmArgs G);
// CTA-pair variant (tcgen05.mma.cta_group::2, M=256): 256x256 tiles
__global__ void k_offline_gemm_pair(const __grid_constant__ CUtensorMap map_a,
                                    const __grid_constant__ CUtensorMap map_b, GemmArgs G);

}  // namespace valve
