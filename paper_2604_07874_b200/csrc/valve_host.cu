// valve_host.cu -- host side of the C-ABI (include/valve_cuda.h): device allocation,
// kernel launches on the pool's stream, error translation, and the two host control
// planes the north star keeps on the CPU (ReservationController, ChannelController state
// machine).  No exception or CUDA error crosses extern "C".
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/valve_cuda.h"
#include "valve_kernels.h"

using namespace valve;

namespace {

thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};

struct Err {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw Err{code, msg}; }

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(VALVE_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return VALVE_OK;
  } catch (const Err& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return VALVE_RUNTIME_ERROR;
  } catch (const std::exception& e) {
    g_err = e.what();
    return VALVE_RUNTIME_ERROR;
  }
}

void counted() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// Driver stream memory operations, fetched through the runtime (no -lcuda link dependency).
using PFN_write32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using PFN_wait32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using PFN_write64 = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
using PFN_wait64 = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
using PFN_batch = CUresult (*)(CUstream, unsigned int, CUstreamBatchMemOpParams*, unsigned int);
struct MemOps {
  PFN_write32 write32 = nullptr;
  PFN_wait32 wait32 = nullptr;
  PFN_write64 write64 = nullptr;
  PFN_wait64 wait64 = nullptr;
  PFN_batch batch = nullptr;
};
const MemOps& memops() {
  static MemOps ops;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuStreamWriteValue32", (void**)&ops.write32, cudaEnableDefault, &q);
    cudaGetDriverEntryPoint("cuStreamWaitValue32", (void**)&ops.wait32, cudaEnableDefault, &q);
    cudaGetDriverEntryPoint("cuStreamWriteValue64", (void**)&ops.write64, cudaEnableDefault, &q);
    cudaGetDriverEntryPoint("cuStreamWaitValue64", (void**)&ops.wait64, cudaEnableDefault, &q);
    cudaGetDriverEntryPoint("cuStreamBatchMemOp", (void**)&ops.batch, cudaEnableDefault, &q);
  });
  if (!ops.write32 || !ops.wait32 || !ops.write64 || !ops.wait64 || !ops.batch)
    fail(VALVE_CUDA_ERROR, "stream memory operations unavailable in this driver");
  return ops;
}
void cu_ck(CUresult r, const char* what) {
  if (r != CUDA_SUCCESS) fail(VALVE_CUDA_ERROR, std::string(what) + " failed (CUresult " + std::to_string((int)r) + ")");
}

CUdeviceptr dptr(const void* p) { return reinterpret_cast<CUdeviceptr>(p); }

int64_t next_pow2(int64_t n) {
  int64_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

const char* detail_msg(int det) {
  switch (det) {
    case kDetGrowExceeds: return "online_grow: k exceeds free handles";
    case kDetRowsFull: return "offline_reserve: device request table full (raise max_requests)";
    case kDetBlocksFull: return "offline_reserve: request exceeds max_pages_per_request";
    case kDetNoCost: return "reclaim: request without cost entry";
    case kDetInvPartition: return "MemoryPool: handle sets do not partition the pool";
    case kDetInvOnline: return "MemoryPool: online page accounting out of bounds";
    case kDetInvSlots: return "MemoryPool: slot accounting mismatch";
    case kDetInvNonOffline: return "MemoryPool: non-offline handle holds offline pages";
    case kDetInvRow: return "MemoryPool: request page count does not match its slots";
    case kDetInvBlock: return "MemoryPool: block table does not point back at its slot";
    default: return "device error";
  }
}

}  // namespace

// ===================================================================================== pool

struct valve_pool {
  valve_pool_config cfg{};
  int H = 0, S = 0, R = 0, Pblk = 0;
  cudaStream_t stream = nullptr;
  PoolDev d{};
  Mirror* mirror = nullptr;  // pinned host
  uint8_t* hst = nullptr;    // pinned staging for snapshot / apply results (read by the host)
  size_t hst_bytes = 0;
  int64_t online_used = 0;   // memory.hpp:97 aggregate (host scalar)
  int* d_ids = nullptr;      // apply ids upload
  int64_t* d_in64 = nullptr; // cost upload
  int64_t* d_in64b = nullptr;
  size_t smem_snapshot = 0, smem_reclaim = 0;
  std::vector<void*> dev_allocs;
  // block tables replaced by growth: a gated offline launch already enqueued (possibly parked
  // behind a closed gate) holds the old pointer, so the old table lives until the pool does
  std::vector<void*> retired_bt;
  int last_n_handles = 0, last_n_evicted = 0, last_n_pages = 0;
  int64_t last_copy_bytes = 0;  // destination bytes of the last report (per-request page sizes)
  int last_custom = 0;          // some evicted request has its own page size
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaStream_t copy_stream = nullptr;  // reclaim copies overlap pool bookkeeping
  cudaStream_t plan_stream = nullptr;  // report snapshots for queued copies (not behind a running copy)
  cudaEvent_t ev_report = nullptr;
  unsigned long long* d_copyctr = nullptr;  // restore / copy-engine counters (pool stream)
  // Reclaim copies in flight (FIFO ring).  Each copy first snapshots the report it needs (the
  // physical page list, plus the byte layout for per-request page sizes) into its own slot on
  // the plan stream, so the next decision may rewrite the report while the bytes are still
  // crossing the link: back-to-back reclaim ops keep the host link busy.
  struct CopySlot {
    int* phys = nullptr;
    int* inv_off = nullptr;
    int64_t* ev_pbytes = nullptr;
    int64_t* ev_base = nullptr;
    int64_t* ev_cbase = nullptr;
    unsigned long long* ctr = nullptr;  // cursor, t_first, t_last
    unsigned* waves = nullptr;          // [kMaxWaves] per-wave done counts, then next, ctas_done
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev_plan = nullptr;
    int64_t bytes = 0, pages = 0;
    uint64_t wave_base = 0;
    int n_waves = 0;
    int64_t wave_bytes = 0;
  };
  static constexpr int kMaxWaves = 1024;
  unsigned long long* d_landed = nullptr;  // published copy waves (monotone, all copies)
  unsigned long long* d_tat = nullptr;     // rate bound: GCRA theoretical arrival time (ns)
  uint64_t waves_issued = 0;               // sum of n_waves over started copies
  static constexpr int kCopySlots = VALVE_COPY_RING;
  CopySlot cs[kCopySlots];
  int cs_head = 0, cs_n = 0, cs_last = -1;

  // Kernels that rewrite the report (apply/reclaim) must not overtake the report snapshot of
  // the latest copy; kernels that rewrite page bytes (fill, restore) must not overtake the copy
  // itself.  Copies run in order on the copy stream, so the latest one covers the earlier ones.
  void order_after_copy_plan() {
    if (cs_last >= 0) ck(cudaStreamWaitEvent(stream, cs[cs_last].ev_plan, 0), "event wait");
  }
  void order_after_copy() {
    if (cs_last >= 0) ck(cudaStreamWaitEvent(stream, cs[cs_last].ev1, 0), "event wait");
  }

  template <class T>
  T* dalloc(int64_t n) {
    void* p = nullptr;
    ck(cudaMalloc(&p, std::max<int64_t>(n, 1) * sizeof(T)), "cudaMalloc");
    dev_allocs.push_back(p);
    return static_cast<T*>(p);
  }

  int64_t op_seq = 0;
  // Completion by polling the pinned mirror (the kernel stores done_seq after its results and a
  // system-scope fence): no stream-synchronize wake-up on the decision path.  Falls back to a
  // stream synchronize (which surfaces faults) when the word does not appear within 200 ms.
  void wait_seq(int64_t seq, const char* op) {
    const auto t0 = std::chrono::steady_clock::now();
    for (int spin = 0; mirror->done_seq != seq; ++spin) {
      if ((spin & 1023) == 1023 && std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(200)) {
        ck(cudaStreamSynchronize(stream), op);
        if (mirror->done_seq != seq) fail(VALVE_RUNTIME_ERROR, std::string(op) + ": completion word not written");
        break;
      }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    check_err();
  }

  void sync_and_check(const char* op) {
    ck(cudaGetLastError(), op);
    ck(cudaStreamSynchronize(stream), op);
    check_err();
  }

  void check_err() {
    if (mirror->err) {
      const int code = mirror->err;
      const int det = mirror->err_detail;
      std::string msg;
      if (det == kDetNotOffline)
        msg = "apply_reclaim: handle " + std::to_string(mirror->err_arg) + " is not offline-mapped";
      else if (det == kDetApplyRange)
        msg = "apply_reclaim: handle " + std::to_string(mirror->err_arg) + " out of range";
      else
        msg = detail_msg(det);
      fail(code, msg);
    }
  }

  // Single-CTA bookkeeping op: the kernel ends in publish(), which stores this launch's
  // sequence number into the pinned mirror; the host polls it (wait_seq) instead of a stream
  // synchronize.  `d` (passed by value) carries the sequence.
  template <class K, class... Args>
  void launch1(const char* op, K kernel, size_t smem, Args... args) {
    ck(cudaSetDevice(cfg.device), "cudaSetDevice");
    kernel<<<1, kNT, smem, stream>>>(args...);
    counted();
    ck(cudaGetLastError(), op);
    wait_seq(d.seq, op);
  }
  // next launch's sequence (call before building the kernel arguments from `d`)
  void next_seq() { d.seq = ++op_seq; }

  // pinned staging of `bytes` (grown on demand; the pool stream is idle when this is called)
  uint8_t* stage(size_t bytes) {
    if (bytes > hst_bytes) {
      if (hst) cudaFreeHost(hst);
      hst = nullptr;
      hst_bytes = std::max(bytes, 2 * hst_bytes);
      ck(cudaHostAlloc((void**)&hst, hst_bytes, cudaHostAllocDefault), "cudaHostAlloc staging");
    }
    return hst;
  }

  void counts(int64_t out[5]) const {
    out[0] = mirror->n_free;
    out[1] = mirror->n_online;
    out[2] = mirror->n_offline;
    out[3] = online_used;
    out[4] = (int64_t)mirror->n_online * S;
  }

  void d2h(void* dst, const void* src, size_t bytes) {
    if (!bytes || !dst) return;
    ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, stream), "cudaMemcpyAsync");
  }

  ~valve_pool() {
    // drain in-flight copies (and their report snapshots) before their buffers go away
    for (cudaStream_t s : {plan_stream, copy_stream, stream})
      if (s) cudaStreamSynchronize(s);
    for (void* p : dev_allocs) cudaFree(p);
    for (void* p : retired_bt) cudaFree(p);
    if (d.pages) cudaFree(d.pages);
    if (mirror) cudaFreeHost(mirror);
    if (hst) cudaFreeHost(hst);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (ev_report) cudaEventDestroy(ev_report);
    for (CopySlot& c : cs)
      for (cudaEvent_t e : {c.ev0, c.ev1, c.ev_plan})
        if (e) cudaEventDestroy(e);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (plan_stream) cudaStreamDestroy(plan_stream);
    if (stream) cudaStreamDestroy(stream);
  }
};

// see reclaim_kernels.cu.  Kept at 160 KiB: the rest of the SM's 256 KiB stays L1, which the
// instance and slot-collection passes' global reads use (200 KiB measured 3x slower collection)
constexpr size_t kReclaimSmemBytes = 160 * 1024;

// With CUDA's lazy module loading, a kernel's code is loaded at its first launch -- and that load
// waits for the kernels already running on the device.  Under colocation the first
// offline_release of a run can then sit behind a ~100 ms gated decode pass (measured: one 90 ms
// pool op per process, gone under CUDA_MODULE_LOADING=EAGER).  Load every kernel of this library
// up front instead (querying its attributes loads it), once per device, when the first pool /
// gate / selection is created -- nothing is running yet at that point.
static void preload_kernels(int device) {
  static std::mutex mu;
  static uint64_t done = 0;
  std::lock_guard<std::mutex> lk(mu);
  if (device < 0 || device >= 64 || (done >> device) & 1ull) return;
  const void* ks[] = {
      (const void*)k_online_grow, (const void*)k_online_release, (const void*)k_offline_reserve,
      (const void*)k_offline_release, (const void*)k_ht_rehash, (const void*)k_requests_on_handle,
      (const void*)k_handles_of_request, (const void*)k_offline_pages_of, (const void*)k_block_table,
      (const void*)k_snapshot_handles, (const void*)k_snapshot, (const void*)k_apply, (const void*)k_reclaim_rows,
      (const void*)k_reclaim, (const void*)k_reclaim_fused, (const void*)k_check_invariants,
      (const void*)k_fill_pages, (const void*)k_set_costs, (const void*)k_select_instance, (const void*)k_map_refs,
      (const void*)k_tile_prefix, (const void*)k_evicted_cost, (const void*)k_reclaim_copy,
      (const void*)k_copy_plan, (const void*)k_reclaim_copy_tma, (const void*)k_restore_scatter,
      (const void*)k_gate_raise_stamp, (const void*)k_offline_decode, (const void*)k_offline_gemm,
      (const void*)k_offline_gemm_pair};
  for (const void* k : ks) {
    cudaFuncAttributes a{};
    ck(cudaFuncGetAttributes(&a, k), "load kernel");
  }
  done |= 1ull << device;
}

static void set_reclaim_smem_attrs() {
  // per device, per process (cheap to repeat)
  int dev = 0;
  ck(cudaGetDevice(&dev), "cudaGetDevice");
  preload_kernels(dev);
  ck(cudaFuncSetAttribute(k_reclaim_copy_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 32768),
     "cudaFuncSetAttribute");
  ck(cudaFuncSetAttribute(k_reclaim_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kReclaimSmemBytes),
     "smem attribute");
  ck(cudaFuncSetAttribute(k_reclaim, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kReclaimSmemBytes),
     "cudaFuncSetAttribute");
  ck(cudaFuncSetAttribute(k_apply, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kReclaimSmemBytes),
     "cudaFuncSetAttribute");
  ck(cudaFuncSetAttribute(k_select_instance, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)kReclaimSmemBytes),
     "cudaFuncSetAttribute");
}

static void pool_reset_state(valve_pool* p);

static void pool_init(valve_pool* p, const valve_pool_config& c) {
  if (c.total_handles <= 0 || c.handle_size_pages <= 0 || c.page_size_tokens <= 0)
    fail(VALVE_INVALID_ARGUMENT, "MemoryPool: sizes must be > 0");  // memory.cpp:15
  if (c.handle_size_pages > 256)
    fail(VALVE_INVALID_ARGUMENT, "MemoryPool: handle_size_pages > 256 is not supported on device");
  if ((int64_t)c.total_handles * c.handle_size_pages >= (1 << 24))
    fail(VALVE_INVALID_ARGUMENT, "MemoryPool: total pages must be < 2^24");
  if (c.max_requests <= 0 || c.max_requests >= (1 << 24) || c.max_pages_per_request <= 0)
    fail(VALVE_INVALID_ARGUMENT, "MemoryPool: bad request-table geometry");
  if (c.slot_bytes < 0 || c.page_bytes < 0 || c.page_bytes > c.slot_bytes || c.page_bytes % 16 ||
      c.slot_bytes % 16)
    fail(VALVE_INVALID_ARGUMENT, "MemoryPool: page/slot bytes must be 16-byte multiples, page <= slot");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= 0)
    fail(VALVE_CUDA_ERROR, "no CUDA device: the valve pool runs only on the GPU");
  if (c.device < 0 || c.device >= ndev) fail(VALVE_INVALID_ARGUMENT, "MemoryPool: bad device ordinal");
  p->cfg = c;
  p->H = c.total_handles;
  p->S = c.handle_size_pages;
  p->R = c.max_requests;
  p->Pblk = c.max_pages_per_request;
  ck(cudaSetDevice(c.device), "cudaSetDevice");
  ck(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking), "cudaStreamCreate");
  ck(cudaEventCreate(&p->ev0), "cudaEventCreate");
  ck(cudaEventCreate(&p->ev1), "cudaEventCreate");
  ck(cudaEventCreateWithFlags(&p->ev_report, cudaEventDisableTiming), "cudaEventCreate");
  ck(cudaStreamCreateWithFlags(&p->copy_stream, cudaStreamNonBlocking), "cudaStreamCreate");
  ck(cudaStreamCreateWithFlags(&p->plan_stream, cudaStreamNonBlocking), "cudaStreamCreate");
  const int H = p->H, S = p->S, R = p->R;
  const int64_t HS = (int64_t)H * S;
  PoolDev& d = p->d;
  d.H = H;
  d.S = S;
  d.R = R;
  d.P = p->Pblk;
  d.HC = (int)next_pow2(2 * (int64_t)R);
  d.quarantine = (int)HS;
  d.hstate = p->dalloc<uint8_t>(H);
  d.hmapped = p->dalloc<int64_t>(H);
  d.hused = p->dalloc<int>(H);
  d.slot_row = p->dalloc<int>(HS);
  d.slot_lid = p->dalloc<int>(HS);
  d.slot_blk = p->dalloc<int>(HS);
  d.row_req = p->dalloc<int64_t>(R);
  d.row_cost = p->dalloc<int64_t>(R);
  d.row_pbytes = p->dalloc<int64_t>(R);
  d.row_npages = p->dalloc<int>(R);
  d.row_nblk = p->dalloc<int>(R);
  d.bt = p->dalloc<int>((int64_t)R * p->Pblk);
  d.ht_key = p->dalloc<int64_t>(d.HC);
  d.ht_row = p->dalloc<int>(d.HC);
  d.ring = p->dalloc<int>(R);
  d.hdr = p->dalloc<PoolHdr>(1);
  const int64_t HSR = std::max<int64_t>(HS, R);
  d.s_hid = p->dalloc<int>(H);
  d.s_hmap = p->dalloc<int64_t>(H);
  d.s_roff = p->dalloc<int>(H + 1);
  d.s_rref = p->dalloc<int>(HS);
  d.s_qoff = p->dalloc<int>(R + 1);
  d.s_qcnt = p->dalloc<int>(HSR);
  d.s_dense = p->dalloc<int>(R);
  ck(cudaMemset(d.s_dense, 0xff, (size_t)R * 4), "memset");
  d.s_qh = p->dalloc<int>(HS);
  d.s_marg = p->dalloc<int64_t>(H);
  d.s_taken = p->dalloc<int>(H);
  d.s_ev = p->dalloc<int>(R);
  d.s_pick = p->dalloc<int>(H);
  d.s_evrows = p->dalloc<int>(R);
  d.s_rank = p->dalloc<int>(R);
  d.s_key = p->dalloc<uint64_t>(next_pow2(HS));
  d.s_pay = p->dalloc<int>(next_pow2(HS));
  d.s_cnt = p->dalloc<int>(H);
  d.ticket = p->dalloc<unsigned>(1);
  ck(cudaMemset(d.ticket, 0, sizeof(unsigned)), "memset");
  d.s_tphys = p->dalloc<int>(HS);
  d.s_tblk = p->dalloc<int>(HS);
  d.res_handles = p->dalloc<int>(H);
  d.res_evicted = p->dalloc<int64_t>(R);
  d.res_inv_off = p->dalloc<int>(R + 1);
  d.res_pages = p->dalloc<int64_t>(HS);
  d.res_phys = p->dalloc<int>(HS);
  d.res_blk = p->dalloc<int>(HS);
  d.res_counts = p->dalloc<int>(4);
  d.res_ev_pbytes = p->dalloc<int64_t>(R);
  d.res_ev_base = p->dalloc<int64_t>(R + 1);
  d.res_ev_cbase = p->dalloc<int64_t>(R + 1);
  p->d_ids = p->dalloc<int>(std::max(std::max(H, 1) * 2, p->Pblk));
  p->d_in64 = p->dalloc<int64_t>(R);
  p->d_in64b = p->dalloc<int64_t>(R);
  p->d_copyctr = p->dalloc<unsigned long long>(4);
  p->d_landed = p->dalloc<unsigned long long>(1);
  p->d_tat = p->dalloc<unsigned long long>(1);
  for (auto& cs : p->cs) {
    cs.phys = p->dalloc<int>(HS);
    cs.inv_off = p->dalloc<int>(R + 1);
    cs.ev_pbytes = p->dalloc<int64_t>(R);
    cs.ev_base = p->dalloc<int64_t>(R + 1);
    cs.ev_cbase = p->dalloc<int64_t>(R + 1);
    cs.ctr = p->dalloc<unsigned long long>(4);
    cs.waves = p->dalloc<unsigned>(valve_pool::kMaxWaves + 2);
    ck(cudaEventCreate(&cs.ev0), "cudaEventCreate");
    ck(cudaEventCreate(&cs.ev1), "cudaEventCreate");
    ck(cudaEventCreateWithFlags(&cs.ev_plan, cudaEventDisableTiming), "cudaEventCreate");
  }
  d.slot_bytes = c.slot_bytes;
  d.page_bytes = c.page_bytes;
  if (c.slot_bytes > 0) {
    void* pg = nullptr;
    ck(cudaMalloc(&pg, (size_t)(HS * c.slot_bytes)), "cudaMalloc(page store)");
    d.pages = static_cast<uint8_t*>(pg);
  }
  ck(cudaHostAlloc((void**)&p->mirror, sizeof(Mirror), cudaHostAllocMapped), "cudaHostAlloc");
  // result staging sized for a whole-pool snapshot / report now: a first-use cudaHostAlloc inside
  // a reclaim on the online critical path took milliseconds
  p->stage((size_t)H * 16 + (size_t)H * S * 16 + (size_t)R * 16 + 64);
  ck(cudaHostGetDevicePointer((void**)&d.mirror, p->mirror, 0), "cudaHostGetDevicePointer");
  pool_reset_state(p);
  // dynamic shared memory: greedy marginals (2048 handles) aliased with the apply sort
  // buffers (8192 x {u64 key, i32 block})
  p->smem_snapshot = 0;
  p->smem_reclaim = kReclaimSmemBytes;
  set_reclaim_smem_attrs();
}

// Initial state: all handles free, no slots, empty request table, every row in the ring, no
// copies published, an idle rate bucket.  (The page store keeps its bytes.)
static void pool_reset_state(valve_pool* p) {
  PoolDev& d = p->d;
  const int H = p->H, S = p->S, R = p->R;
  const int64_t HS = (int64_t)H * S;
  std::memset(p->mirror, 0, sizeof(Mirror));
  ck(cudaMemsetAsync(d.hstate, 0, H, p->stream), "memset");
  ck(cudaMemsetAsync(d.hmapped, 0, H * 8, p->stream), "memset");
  ck(cudaMemsetAsync(d.hused, 0, H * 4, p->stream), "memset");
  ck(cudaMemsetAsync(d.slot_row, 0xff, HS * 4, p->stream), "memset");
  ck(cudaMemsetAsync(d.slot_lid, 0xff, HS * 4, p->stream), "memset");
  ck(cudaMemsetAsync(d.slot_blk, 0xff, HS * 4, p->stream), "memset");
  ck(cudaMemsetAsync(d.row_npages, 0, R * 4, p->stream), "memset");
  ck(cudaMemsetAsync(d.row_nblk, 0, R * 4, p->stream), "memset");
  ck(cudaMemsetAsync(d.row_cost, 0, R * 8, p->stream), "memset");
  ck(cudaMemsetAsync(d.row_pbytes, 0, R * 8, p->stream), "memset");
  ck(cudaMemsetAsync(d.bt, 0xff, (size_t)R * p->Pblk * 4, p->stream), "memset");
  ck(cudaMemsetAsync(d.ht_row, 0xff, (size_t)d.HC * 4, p->stream), "memset");
  ck(cudaMemsetAsync(d.s_ev, 0, R * 4, p->stream), "memset");
  std::vector<int> ring(R);
  for (int i = 0; i < R; ++i) ring[i] = i;
  ck(cudaMemcpyAsync(d.ring, ring.data(), R * 4, cudaMemcpyHostToDevice, p->stream), "upload");
  PoolHdr hdr{H, 0, 0, 0, R, 0};
  ck(cudaMemcpyAsync(d.hdr, &hdr, sizeof hdr, cudaMemcpyHostToDevice, p->stream), "upload");
  ck(cudaMemsetAsync(p->d_landed, 0, 8, p->stream), "memset");
  ck(cudaMemsetAsync(p->d_tat, 0, 8, p->stream), "memset");
  ck(cudaStreamSynchronize(p->stream), "init");
  p->mirror->n_free = H;
  p->online_used = 0;
  p->waves_issued = 0;
  p->last_n_handles = p->last_n_evicted = p->last_n_pages = 0;
  p->last_copy_bytes = 0;
  p->last_custom = 0;
  p->cs_head = p->cs_n = 0;
  p->cs_last = -1;
}

namespace {

// Replaces a pool array by a larger one; `keep` leading elements are copied, the rest is
// filled with `fill` bytes (or left uninitialised for scratch when fill < 0).
template <class T>
void regrow(valve_pool* p, T*& ptr, int64_t keep, int64_t n, int fill) {
  // stream-ordered allocation: cudaMalloc / cudaFree may synchronize the whole device, which
  // would wait for (and deadlock on) a gated tenant's stream parked behind a closed gate
  void* np = nullptr;
  ck(cudaMallocAsync(&np, std::max<int64_t>(n, 1) * sizeof(T), p->stream), "cudaMallocAsync(table growth)");
  if (fill >= 0) ck(cudaMemsetAsync(np, fill, n * sizeof(T), p->stream), "memset");
  if (keep > 0) ck(cudaMemcpyAsync(np, ptr, keep * sizeof(T), cudaMemcpyDeviceToDevice, p->stream), "copy");
  auto it = std::find(p->dev_allocs.begin(), p->dev_allocs.end(), static_cast<void*>(ptr));
  if (it != p->dev_allocs.end()) *it = np;
  if (ptr) ck(cudaFreeAsync(ptr, p->stream), "cudaFreeAsync(table growth)");
  ck(cudaStreamSynchronize(p->stream), "table growth");
  ptr = static_cast<T*>(np);
}

// Grows the device request table to R2 rows of P2 blocks.  The reference MemoryPool has no
// limit on live requests or pages per request (memory.hpp:81-97 std::map / std::vector); the
// device tables start small (apply and reserve scan them) and grow on demand, so a drop-in
// caller never sees a capacity error the reference would not raise.  Row ids, the free-row
// FIFO order, block tables and the last reclaim report are preserved; the request hash is
// rebuilt at its new capacity.
void grow_tables(valve_pool* p, int R2, int P2) {
  const int R = p->R, P = p->Pblk;
  R2 = std::max(R2, R);
  P2 = std::max(P2, P);
  if (R2 == R && P2 == P) return;
  if (R2 >= (1 << 24)) fail(VALVE_RUNTIME_ERROR, "MemoryPool: request table beyond 2^24 rows");
  for (cudaStream_t s : {p->plan_stream, p->copy_stream, p->stream})
    ck(cudaStreamSynchronize(s), "table growth");
  PoolDev& d = p->d;
  const int64_t HS = (int64_t)p->H * p->S;
  if (P2 != P || R2 != R) {  // block tables: new pitch and/or more rows
    int* nbt = nullptr;
    ck(cudaMallocAsync((void**)&nbt, (size_t)R2 * P2 * 4, p->stream), "cudaMallocAsync(block tables)");
    ck(cudaMemsetAsync(nbt, 0xff, (size_t)R2 * P2 * 4, p->stream), "memset");
    ck(cudaMemcpy2DAsync(nbt, (size_t)P2 * 4, d.bt, (size_t)P * 4, (size_t)P * 4, R, cudaMemcpyDeviceToDevice,
                         p->stream), "copy");
    auto it = std::find(p->dev_allocs.begin(), p->dev_allocs.end(), static_cast<void*>(d.bt));
    if (it != p->dev_allocs.end()) *it = nbt;
    ck(cudaStreamSynchronize(p->stream), "table growth");
    p->retired_bt.push_back(d.bt);  // not freed: see retired_bt
    d.bt = nbt;
  }
  if (P2 != P) regrow(p, p->d_ids, 0, std::max<int64_t>(std::max(p->H, 1) * 2, P2), -1);
  if (R2 != R) {
    // free-row FIFO: the live window [head, tail) in order, then the new rows
    PoolHdr hdr;
    ck(cudaMemcpy(&hdr, d.hdr, sizeof hdr, cudaMemcpyDeviceToHost), "read");
    std::vector<int> ring(R), nring;
    ck(cudaMemcpy(ring.data(), d.ring, (size_t)R * 4, cudaMemcpyDeviceToHost), "read");
    for (int i = hdr.ring_head; i < hdr.ring_tail; ++i) nring.push_back(ring[i % R]);
    for (int r = R; r < R2; ++r) nring.push_back(r);
    regrow(p, d.ring, 0, R2, -1);
    ck(cudaMemcpy(d.ring, nring.data(), nring.size() * 4, cudaMemcpyHostToDevice), "upload");
    hdr.ring_head = 0;
    hdr.ring_tail = (int)nring.size();
    hdr.tombstones = 0;
    // state rows (kept) and per-row scratch (fresh)
    regrow(p, d.row_req, R, R2, 0);
    regrow(p, d.row_cost, R, R2, 0);
    regrow(p, d.row_pbytes, R, R2, 0);
    regrow(p, d.row_npages, R, R2, 0);
    regrow(p, d.row_nblk, R, R2, 0);
    regrow(p, d.s_ev, 0, R2, 0);
    regrow(p, d.s_qoff, 0, R2 + 1, -1);
    regrow(p, d.s_qcnt, 0, std::max<int64_t>(HS, R2), -1);
    regrow(p, d.s_dense, 0, R2, 0xff);  // -1 everywhere between selections (greedy_select)
    regrow(p, d.s_evrows, 0, R2, -1);
    regrow(p, d.s_rank, 0, R2, -1);
    regrow(p, d.res_evicted, R, R2, 0);
    regrow(p, d.res_inv_off, R + 1, R2 + 1, 0);
    regrow(p, d.res_ev_pbytes, R, R2, 0);
    regrow(p, d.res_ev_base, R + 1, R2 + 1, 0);
    regrow(p, d.res_ev_cbase, R + 1, R2 + 1, 0);
    regrow(p, p->d_in64, 0, R2, -1);
    regrow(p, p->d_in64b, 0, R2, -1);
    for (auto& c : p->cs) {
      regrow(p, c.inv_off, 0, R2 + 1, -1);
      regrow(p, c.ev_pbytes, 0, R2, -1);
      regrow(p, c.ev_base, 0, R2 + 1, -1);
      regrow(p, c.ev_cbase, 0, R2 + 1, -1);
    }
    // request hash at its new capacity: re-insert every live row
    const int HC2 = (int)next_pow2(2 * (int64_t)R2);
    int* old_row = d.ht_row;
    int64_t* old_key = d.ht_key;
    const int HC = d.HC;
    int* nrow = nullptr;
    int64_t* nkey = nullptr;
    ck(cudaMallocAsync((void**)&nrow, (size_t)HC2 * 4, p->stream), "cudaMallocAsync(request hash)");
    ck(cudaMallocAsync((void**)&nkey, (size_t)HC2 * 8, p->stream), "cudaMallocAsync(request hash)");
    ck(cudaMemsetAsync(nrow, 0xff, (size_t)HC2 * 4, p->stream), "memset");
    d.ht_row = nrow;
    d.ht_key = nkey;
    d.HC = HC2;
    d.R = R2;
    p->R = R2;
    ck(cudaMemcpyAsync(d.hdr, &hdr, sizeof hdr, cudaMemcpyHostToDevice, p->stream), "upload");
    k_ht_rehash<<<(HC + 255) / 256, 256, 0, p->stream>>>(d, old_row, HC);
    counted();
    ck(cudaGetLastError(), "rehash launch");
    ck(cudaStreamSynchronize(p->stream), "rehash");
    for (void*& a : p->dev_allocs) {
      if (a == old_row) a = nrow;
      else if (a == old_key) a = nkey;
    }
    ck(cudaFreeAsync(old_row, p->stream), "cudaFreeAsync(request hash)");
    ck(cudaFreeAsync(old_key, p->stream), "cudaFreeAsync(request hash)");
    ck(cudaStreamSynchronize(p->stream), "rehash");
  }
  d.P = P2;
  p->Pblk = P2;
  p->cfg.max_requests = p->R;
  p->cfg.max_pages_per_request = P2;
}

// The last report, staged through the pool's pinned buffer (one synchronize, DMA into pinned
// memory), then copied into the caller's arrays.  Returns the staged arrays.
struct Staged {
  const int* handles;
  const int64_t* evicted;
  const int* inv_off;
  const int64_t* pages;
  const int* phys;
  const int* blk;
};

Staged stage_apply_results(valve_pool* p, bool phys_blk) {
  const int nh = p->last_n_handles, ne = p->last_n_evicted, np = p->last_n_pages;
  const size_t o_ev = 0, o_pg = o_ev + (size_t)ne * 8, o_h = o_pg + (size_t)np * 8,
               o_off = o_h + (size_t)nh * 4, o_ph = o_off + (size_t)(ne + 1) * 4,
               o_bl = o_ph + (phys_blk ? (size_t)np * 4 : 0), total = o_bl + (phys_blk ? (size_t)np * 4 : 0);
  uint8_t* h = p->stage(total + 16);
  const cudaMemcpyKind k = cudaMemcpyDeviceToHost;
  if (ne) ck(cudaMemcpyAsync(h + o_ev, p->d.res_evicted, (size_t)ne * 8, k, p->stream), "stage");
  if (np) ck(cudaMemcpyAsync(h + o_pg, p->d.res_pages, (size_t)np * 8, k, p->stream), "stage");
  if (nh) ck(cudaMemcpyAsync(h + o_h, p->d.res_handles, (size_t)nh * 4, k, p->stream), "stage");
  ck(cudaMemcpyAsync(h + o_off, p->d.res_inv_off, (size_t)(ne + 1) * 4, k, p->stream), "stage");
  if (phys_blk && np) {
    ck(cudaMemcpyAsync(h + o_ph, p->d.res_phys, (size_t)np * 4, k, p->stream), "stage");
    ck(cudaMemcpyAsync(h + o_bl, p->d.res_blk, (size_t)np * 4, k, p->stream), "stage");
  }
  ck(cudaStreamSynchronize(p->stream), "apply results");
  return Staged{reinterpret_cast<const int*>(h + o_h), reinterpret_cast<const int64_t*>(h + o_ev),
                reinterpret_cast<const int*>(h + o_off), reinterpret_cast<const int64_t*>(h + o_pg),
                phys_blk ? reinterpret_cast<const int*>(h + o_ph) : nullptr,
                phys_blk ? reinterpret_cast<const int*>(h + o_bl) : nullptr};
}

void read_apply_results(valve_pool* p, int* handles, int64_t* evicted, int* inv_off, int64_t* pages,
                        int* phys, int* blk, int cap_h, int cap_ev, int cap_pages) {
  const int nh = p->last_n_handles, ne = p->last_n_evicted, np = p->last_n_pages;
  if (!handles && !evicted && !inv_off && !pages && !phys && !blk) return;
  const Staged st = stage_apply_results(p, phys || blk);
  if (handles) std::memcpy(handles, st.handles, (size_t)std::min(nh, cap_h) * 4);
  if (evicted) std::memcpy(evicted, st.evicted, (size_t)std::min(ne, cap_ev) * 8);
  if (inv_off && cap_ev >= ne) std::memcpy(inv_off, st.inv_off, (size_t)(ne + 1) * 4);
  const size_t n = (size_t)std::min(np, cap_pages);
  if (pages) std::memcpy(pages, st.pages, n * 8);
  if (phys) std::memcpy(phys, st.phys, n * 4);
  if (blk) std::memcpy(blk, st.blk, n * 4);
}

}  // namespace

// The colocation runtime keeps many streams busy at once (online, offline tenant, gate, pool, copy,
// plan, observers) and some of them block on stream memory operations for long periods (a gated
// launch waits for the gate to open; a landed-ticket wait lasts until its copy wave is out).  With
// CUDA's default of 8 hardware work queues, streams share queues and a blocked wait stalls every
// stream behind it in the same queue (measured: a 1-CTA pool op delayed 90 ms behind a ticket
// wait).  Ask for the maximum number of queues before the process creates its CUDA context; a
// caller's own setting wins.
__attribute__((constructor)) static void valve_connections() { setenv("CUDA_DEVICE_MAX_CONNECTIONS", "32", 0); }

extern "C" {

const char* valve_last_error(void) { return g_err.c_str(); }
int64_t valve_kernel_launches(void) { return g_launches.load(); }

void valve_pool_config_default(valve_pool_config* c) {
  std::memset(c, 0, sizeof *c);
  c->device = 0;
  c->total_handles = 128;
  c->handle_size_pages = 64;
  c->page_size_tokens = 16;
  c->max_requests = 4096;
  c->max_pages_per_request = 4096;
}

int valve_pool_create_ex(const valve_pool_config* cfg, valve_pool** out) {
  return guard([&] {
    auto* p = new valve_pool;
    try {
      pool_init(p, *cfg);
    } catch (...) {
      delete p;
      throw;
    }
    *out = p;
  });
}

int valve_pool_create(int H, int S, int T, valve_pool** out) {
  valve_pool_config c;
  valve_pool_config_default(&c);
  c.total_handles = H;
  c.handle_size_pages = S;
  c.page_size_tokens = T;
  if (H > 0 && S > 0) c.max_pages_per_request = std::min<int64_t>((int64_t)H * S, 4096);
  return valve_pool_create_ex(&c, out);
}

void valve_pool_destroy(valve_pool* p) { delete p; }

int valve_pool_reset(valve_pool* p) {
  return guard([&] {
    ck(cudaSetDevice(p->cfg.device), "cudaSetDevice");
    for (cudaStream_t s : {p->plan_stream, p->copy_stream, p->stream}) ck(cudaStreamSynchronize(s), "reset");
    pool_reset_state(p);
  });
}

int valve_pool_online_handles(const valve_pool* cp, int* out, int cap, int* n) {
  auto* p = const_cast<valve_pool*>(cp);
  return guard([&] {
    ck(cudaSetDevice(p->cfg.device), "cudaSetDevice");
    std::vector<uint8_t> st(p->H);
    ck(cudaMemcpyAsync(st.data(), p->d.hstate, p->H, cudaMemcpyDeviceToHost, p->stream), "read");
    ck(cudaStreamSynchronize(p->stream), "read");
    int k = 0;
    for (int h = 0; h < p->H; ++h)
      if (st[h] == kOnline) {
        if (out && k < cap) out[k] = h;
        ++k;
      }
    *n = k;
  });
}

int valve_pool_counts(const valve_pool* p, int64_t out[5]) {
  p->counts(out);
  return VALVE_OK;
}

int valve_pool_geometry(const valve_pool* p, int out[4]) {
  out[0] = p->H;
  out[1] = p->S;
  out[2] = p->cfg.page_size_tokens;
  out[3] = p->d.quarantine;
  return VALVE_OK;
}

int64_t valve_pool_quarantine_page_id(const valve_pool* p) { return (int64_t)p->H * p->S; }

int valve_pool_online_grow(valve_pool* p, int k, int64_t t) {
  return guard([&] {
    if (k < 0) fail(VALVE_INVALID_ARGUMENT, "online_grow: k must be >= 0");  // memory.cpp:32
    p->next_seq(), p->launch1("online_grow", k_online_grow, 0, p->d, k, t);
  });
}

int valve_pool_online_release(valve_pool* p, int k, int* released) {
  return guard([&] {
    if (k < 0) fail(VALVE_INVALID_ARGUMENT, "online_release: k must be >= 0");  // memory.cpp:38
    p->next_seq(), p->launch1("online_release", k_online_release, 0, p->d, k, p->online_used);
    *released = (int)p->mirror->r[0];
  });
}

int valve_pool_online_use_pages(valve_pool* p, int64_t n) {
  return guard([&] {
    // memory.cpp:53-58: aggregate accounting against the device-resident capacity
    if (n < 0) fail(VALVE_INVALID_ARGUMENT, "online_use_pages: n must be >= 0");
    if (p->online_used + n > (int64_t)p->mirror->n_online * p->S)
      fail(VALVE_LOGIC_ERROR, "online_use_pages: overcommit beyond reserved capacity");
    p->online_used += n;
  });
}

int valve_pool_online_free_pages(valve_pool* p, int64_t n) {
  return guard([&] {
    if (n < 0 || n > p->online_used) fail(VALVE_LOGIC_ERROR, "online_free_pages: bad page count");
    p->online_used -= n;
  });
}

int valve_pool_offline_reserve(valve_pool* p, int64_t req, int pages, int64_t t, int max_off, int* ok) {
  return guard([&] {
    if (pages < 0) fail(VALVE_INVALID_ARGUMENT, "offline_reserve: pages must be >= 0");  // memory.cpp:67
    if (pages == 0) {  // memory.cpp:68
      *ok = 1;
      return;
    }
    // The kernel checks table capacity before it mutates anything: on a full table, grow it
    // and run the reservation again (the reference has no such limit).
    const int64_t HS = (int64_t)p->H * p->S;
    for (int attempt = 0;; ++attempt) {
      try {
        p->next_seq(), p->launch1("offline_reserve", k_offline_reserve, 0, p->d, req, pages, t, max_off);
        break;
      } catch (const Err&) {
        const int det = p->mirror->err_detail;
        if (attempt >= 4 || (det != kDetRowsFull && det != kDetBlocksFull)) throw;
        p->mirror->err = 0;
        if (det == kDetRowsFull)
          grow_tables(p, (int)std::min<int64_t>(2 * (int64_t)p->R, std::max<int64_t>(HS, p->R + 1)), p->Pblk);
        else
          grow_tables(p, p->R, (int)std::min<int64_t>(std::max<int64_t>(2 * (int64_t)p->Pblk, p->mirror->err_arg),
                                                       std::max<int64_t>(HS, p->mirror->err_arg)));
      }
    }
    *ok = (int)p->mirror->r[0];
  });
}

int valve_pool_offline_release(valve_pool* p, int64_t req) {
  return guard([&] { p->next_seq(), p->launch1("offline_release", k_offline_release, 0, p->d, req); });
}

int valve_pool_requests_on_handle(const valve_pool* cp, int h, int64_t* out, int cap, int* n) {
  auto* p = const_cast<valve_pool*>(cp);
  return guard([&] {
    if (h < 0 || h >= p->H) fail(VALVE_OUT_OF_RANGE, "requests_on_handle: handle out of range");
    p->next_seq(), p->launch1("requests_on_handle", k_requests_on_handle, 0, p->d, h, (int64_t*)p->d.res_pages);
    *n = (int)p->mirror->r[0];
    if (out) p->d2h(out, p->d.res_pages, (size_t)std::min(*n, cap) * 8);
    ck(cudaStreamSynchronize(p->stream), "requests_on_handle");
  });
}

int valve_pool_handles_of_request(const valve_pool* cp, int64_t req, int* out, int cap, int* n) {
  auto* p = const_cast<valve_pool*>(cp);
  return guard([&] {
    p->next_seq(), p->launch1("handles_of_request", k_handles_of_request, 0, p->d, req, p->d.res_handles);
    *n = (int)p->mirror->r[0];
    if (out) p->d2h(out, p->d.res_handles, (size_t)std::min(*n, cap) * 4);
    ck(cudaStreamSynchronize(p->stream), "handles_of_request");
  });
}

int valve_pool_offline_pages_of(const valve_pool* cp, int64_t req, int* out) {
  auto* p = const_cast<valve_pool*>(cp);
  return guard([&] {
    ck(cudaSetDevice(p->cfg.device), "cudaSetDevice");
    k_offline_pages_of<<<1, 32, 0, p->stream>>>(p->d, req);
    counted();
    p->sync_and_check("offline_pages_of");
    *out = (int)p->mirror->r[0];
  });
}

int valve_pool_request_row(const valve_pool* cp, int64_t req, int* row) {
  auto* p = const_cast<valve_pool*>(cp);
  return guard([&] {
    ck(cudaSetDevice(p->cfg.device), "cudaSetDevice");
    k_offline_pages_of<<<1, 32, 0, p->stream>>>(p->d, req);
    counted();
    p->sync_and_check("request_row");
    *row = (int)p->mirror->r[1];
  });
}

int valve_pool_block_table(const valve_pool* cp, int64_t req, int* out, int cap, int* n) {
  auto* p = const_cast<valve_pool*>(cp);
  return guard([&] {
    p->order_after_copy_plan();  // the page list is written into the report buffer
    p->next_seq(), p->launch1("block_table", k_block_table, 0, p->d, req, p->d.res_phys);
    *n = (int)p->mirror->r[0];
    if (out) p->d2h(out, p->d.res_phys, (size_t)std::min(*n, cap) * 4);
    ck(cudaStreamSynchronize(p->stream), "block_table");
  });
}

namespace {
void snapshot_staged(valve_pool* p, const int** ids, const int64_t** mapped, const int** off,
                     const int64_t** reqs, int* nh, int* nr) {
  ck(cudaSetDevice(p->cfg.device), "cudaSetDevice");
  k_snapshot_handles<<<(p->H + 7) / 8, 256, 0, p->stream>>>(p->d);
  counted();
  p->next_seq(), p->launch1("snapshot", k_snapshot, p->smem_snapshot, p->d);
  const int h = (int)p->mirror->r[0], r = (int)p->mirror->r[1];
  const size_t o_r = 0, o_m = o_r + (size_t)r * 8, o_i = o_m + (size_t)h * 8, o_o = o_i + (size_t)h * 4,
               total = o_o + (size_t)(h + 1) * 4;
  uint8_t* s = p->stage(total + 16);
  const cudaMemcpyKind k = cudaMemcpyDeviceToHost;
  if (r) ck(cudaMemcpyAsync(s + o_r, p->d.res_pages, (size_t)r * 8, k, p->stream), "stage");
  if (h) ck(cudaMemcpyAsync(s + o_m, p->d.s_hmap, (size_t)h * 8, k, p->stream), "stage");
  if (h) ck(cudaMemcpyAsync(s + o_i, p->d.s_hid, (size_t)h * 4, k, p->stream), "stage");
  ck(cudaMemcpyAsync(s + o_o, p->d.s_roff, (size_t)(h + 1) * 4, k, p->stream), "stage");
  ck(cudaStreamSynchronize(p->stream), "snapshot");
  *nh = h;
  *nr = r;
  *reqs = reinterpret_cast<const int64_t*>(s + o_r);
  *mapped = reinterpret_cast<const int64_t*>(s + o_m);
  *ids = reinterpret_cast<const int*>(s + o_i);
  *off = reinterpret_cast<const int*>(s + o_o);
}
}  // namespace

int valve_pool_snapshot(const valve_pool* cp, int* ids, int64_t* mapped, int* off, int64_t* reqs,
                        int cap_h, int cap_r, int* nh, int* nr) {
  auto* p = const_cast<valve_pool*>(cp);
  return guard([&] {
    const int *si, *so;
    const int64_t *sm, *sr;
    snapshot_staged(p, &si, &sm, &so, &sr, nh, nr);
    if (ids) std::memcpy(ids, si, (size_t)std::min(*nh, cap_h) * 4);
    if (mapped) std::memcpy(mapped, sm, (size_t)std::min(*nh, cap_h) * 8);
    if (off && cap_h >= *nh) std::memcpy(off, so, (size_t)(*nh + 1) * 4);
    if (reqs) std::memcpy(reqs, sr, (size_t)std::min(*nr, cap_r) * 8);
  });
}

int valve_pool_snapshot_view(valve_pool* p, const int** ids, const int64_t** mapped, const int** off,
                             const int64_t** reqs, int* nh, int* nr) {
  return guard([&] { snapshot_staged(p, ids, mapped, off, reqs, nh, nr); });
}

int valve_pool_apply_reclaim_view(valve_pool* p, const int* ids, int k, int64_t t, const int** handles,
                                  int* n_handles, const int64_t** evicted, int* n_evicted, const int** inv_off,
                                  const int64_t** inv_pages, int* n_pages) {
  const int code = valve_pool_apply_reclaim(p, ids, k, t, nullptr, n_handles, nullptr, n_evicted, nullptr,
                                            nullptr, nullptr, nullptr, 0, 0, n_pages);
  if (code != VALVE_OK && code != VALVE_LOGIC_ERROR && code != VALVE_OUT_OF_RANGE) return code;
  const std::string saved = g_err;
  const int rc = guard([&] {
    const Staged st = stage_apply_results(p, false);
    *handles = st.handles;
    *evicted = st.evicted;
    *inv_off = st.inv_off;
    *inv_pages = st.pages;
  });
  if (code != VALVE_OK) {
    g_err = saved;
    return code;
  }
  return rc;
}

int valve_pool_apply_reclaim(valve_pool* p, const int* ids, int k, int64_t t, int* handles,
                             int* n_handles, int64_t* evicted, int* n_evicted, int* inv_off,
                             int64_t* inv_pages, int* inv_phys, int* inv_blk, int cap_ev,
                             int cap_pages, int* n_pages) {
  int code = guard([&] {
    if (k < 0) fail(VALVE_INVALID_ARGUMENT, "apply_reclaim: negative handle count");
    // beyond H+1 entries the list must already contain a repeat or a bad id, at which the
    // reference stops (memory.cpp:160-161): only that prefix matters
    k = std::min(k, p->H + 1);
    ck(cudaSetDevice(p->cfg.device), "cudaSetDevice");
    if (k) ck(cudaMemcpyAsync(p->d_ids, ids, (size_t)k * 4, cudaMemcpyHostToDevice, p->stream), "upload ids");
    try {
      p->order_after_copy_plan();
      p->next_seq(), p->launch1("apply_reclaim", k_apply, p->smem_reclaim, p->d, (const int*)p->d_ids, k, t);
    } catch (const Err&) {
      p->last_n_handles = (int)p->mirror->r[0];
      p->last_n_evicted = (int)p->mirror->r[1];
      p->last_n_pages = (int)p->mirror->r[2];
    p->last_copy_bytes = p->mirror->copy_bytes;
    p->last_custom = p->mirror->copy_custom;
      throw;
    }
    p->last_n_handles = (int)p->mirror->r[0];
    p->last_n_evicted = (int)p->mirror->r[1];
    p->last_n_pages = (int)p->mirror->r[2];
    p->last_copy_bytes = p->mirror->copy_bytes;
    p->last_custom = p->mirror->copy_custom;
  });
  if (n_handles) *n_handles = p->last_n_handles;
  if (n_evicted) *n_evicted = p->last_n_evicted;
  if (n_pages) *n_pages = p->last_n_pages;
  if (code != VALVE_OK && code != VALVE_LOGIC_ERROR && code != VALVE_OUT_OF_RANGE) return code;
  const std::string saved = g_err;
  const int rc = guard([&] {
    read_apply_results(p, handles, evicted, inv_off, inv_pages, inv_phys, inv_blk, p->H, cap_ev,
                       cap_pages);
  });
  if (code != VALVE_OK) {
    g_err = saved;
    return code;
  }
  return rc;
}

int valve_pool_handle_state(const valve_pool* cp, int h, int* st) {
  auto* p = const_cast<valve_pool*>(cp);
  return guard([&] {
    if (h < 0 || h >= p->H) fail(VALVE_OUT_OF_RANGE, "handle_state: handle out of range");
    uint8_t v = 0;
    ck(cudaMemcpyAsync(&v, p->d.hstate + h, 1, cudaMemcpyDeviceToHost, p->stream), "read");
    ck(cudaStreamSynchronize(p->stream), "read");
    *st = v;
  });
}

int valve_pool_handle_mapped_at(const valve_pool* cp, int h, int64_t* t) {
  auto* p = const_cast<valve_pool*>(cp);
  return guard([&] {
    if (h < 0 || h >= p->H) fail(VALVE_OUT_OF_RANGE, "handle_mapped_at: handle out of range");
    ck(cudaMemcpyAsync(t, p->d.hmapped + h, 8, cudaMemcpyDeviceToHost, p->stream), "read");
    ck(cudaStreamSynchronize(p->stream), "read");
  });
}

int valve_pool_check_invariants(const valve_pool* cp) {
  auto* p = const_cast<valve_pool*>(cp);
  return guard([&] { p->next_seq(), p->launch1("check_invariants", k_check_invariants, 0, p->d, p->online_used); });
}

int valve_pool_set_costs(valve_pool* p, int n, const int64_t* reqs, const int64_t* costs) {
  return guard([&] {
    if (n < 0 || n > p->R) fail(VALVE_INVALID_ARGUMENT, "set_costs: bad count");
    if (!n) return;
    ck(cudaSetDevice(p->cfg.device), "cudaSetDevice");
    ck(cudaMemcpyAsync(p->d_in64, reqs, (size_t)n * 8, cudaMemcpyHostToDevice, p->stream), "upload");
    ck(cudaMemcpyAsync(p->d_in64b, costs, (size_t)n * 8, cudaMemcpyHostToDevice, p->stream), "upload");
    p->next_seq(), p->launch1("set_costs", k_set_costs, 0, p->d, n, (const int64_t*)p->d_in64,
               (const int64_t*)p->d_in64b, 0);
    if (p->mirror->r[0]) fail(VALVE_INVALID_ARGUMENT, "set_costs: request has no live pages in the pool");
  });
}

int valve_pool_set_page_bytes(valve_pool* p, int n, const int64_t* reqs, const int64_t* bytes) {
  return guard([&] {
    if (n < 0 || n > p->R) fail(VALVE_INVALID_ARGUMENT, "set_page_bytes: bad count");
    for (int i = 0; i < n; ++i)
      if (bytes[i] < 0 || bytes[i] > p->d.slot_bytes || bytes[i] % 16 || (bytes[i] && !p->d.pages))
        fail(VALVE_INVALID_ARGUMENT, "set_page_bytes: need 0 or a 16-byte multiple <= slot_bytes");
    if (!n) return;
    ck(cudaSetDevice(p->cfg.device), "cudaSetDevice");
    ck(cudaMemcpyAsync(p->d_in64, reqs, (size_t)n * 8, cudaMemcpyHostToDevice, p->stream), "upload");
    ck(cudaMemcpyAsync(p->d_in64b, bytes, (size_t)n * 8, cudaMemcpyHostToDevice, p->stream), "upload");
    p->next_seq(), p->launch1("set_page_bytes", k_set_costs, 0, p->d, n, (const int64_t*)p->d_in64,
               (const int64_t*)p->d_in64b, 1);
    if (p->mirror->r[0]) fail(VALVE_INVALID_ARGUMENT, "set_page_bytes: request has no live pages in the pool");
  });
}

int valve_pool_last_copy_layout(const valve_pool* cp, int64_t* page_bytes, int cap, int64_t* total) {
  auto* p = const_cast<valve_pool*>(cp);
  return guard([&] {
    if (total) *total = p->last_copy_bytes;
    if (page_bytes && p->last_n_evicted) {
      ck(cudaMemcpyAsync(page_bytes, p->d.res_ev_pbytes, (size_t)std::min(cap, p->last_n_evicted) * 8,
                         cudaMemcpyDeviceToHost, p->stream), "read");
      ck(cudaStreamSynchronize(p->stream), "read");
    }
  });
}

int valve_pool_reclaim(valve_pool* p, int k, int mode, int64_t t, int* n_handles, int* n_evicted,
                       int* n_pages) {
  return guard([&] {
    if (k < 0) fail(VALVE_INVALID_ARGUMENT, "selective_reclaim: k must be >= 0");
    if (mode != VALVE_SELECT_SELECTIVE && mode != VALVE_SELECT_FIFO)
      fail(VALVE_INVALID_ARGUMENT, "reclaim: device-fused mode must be selective or fifo");
    p->order_after_copy_plan();
    ck(cudaSetDevice(p->cfg.device), "cudaSetDevice");
    // one launch: ceil(H / 32) CTAs build the instance rows (warp per handle), the last CTA to
    // finish runs selection + apply; the host spins on the completion sequence the kernel writes
    // into the pinned mirror instead of a stream synchronize
    p->next_seq();
    const int64_t seq = p->d.seq;
    k_reclaim_fused<<<(p->H + 31) / 32, kNT, p->smem_reclaim, p->stream>>>(p->d, k, mode, t, seq);
    counted();
    ck(cudaGetLastError(), "reclaim");
    p->wait_seq(seq, "reclaim");
    p->last_n_handles = (int)p->mirror->r[0];
    p->last_n_evicted = (int)p->mirror->r[1];
    p->last_n_pages = (int)p->mirror->r[2];
    p->last_copy_bytes = p->mirror->copy_bytes;
    p->last_custom = p->mirror->copy_custom;
    if (n_handles) *n_handles = p->last_n_handles;
    if (n_evicted) *n_evicted = p->last_n_evicted;
    if (n_pages) *n_pages = p->last_n_pages;
  });
}

int valve_pool_reclaim_phases(const valve_pool* p, int64_t out[16]) {
  const int64_t* r = p->mirror->r;
  out[0] = r[4] - r[3];
  out[1] = r[5] - r[4];
  out[2] = r[6] - r[5];
  long long cyc[2] = {0, 0};
  cudaMemcpyFromSymbol(cyc, valve::g_greedy_cycles, sizeof cyc);
  out[3] = cyc[0];
  out[4] = cyc[1];
  long long an[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  cudaMemcpyFromSymbol(an, valve::g_apply_ns, sizeof an);
  out[5] = an[1] - an[0];  // evicted-row compaction + ranks
  out[6] = an[2] - an[1];  // report order + outputs
  out[7] = an[3] - an[2];  // residual page release
  out[8] = an[4] - an[3];  // request-table erase
  out[9] = an[6] - an[5];  // validation of the pick
  out[10] = an[7] > an[6] ? an[7] - an[6] : 0;  // slot collection + clear (fast path)
  out[11] = an[8] > an[7] ? an[8] - an[7] : 0;  // per-handle ranks + pairs (fast path)
  long long sn[5] = {0, 0, 0, 0, 0};
  cudaMemcpyFromSymbol(sn, valve::g_select_ns, sizeof sn);
  out[12] = sn[1] > sn[0] ? sn[1] - sn[0] : 0;  // selection: dense request ids
  out[13] = sn[2] > sn[1] ? sn[2] - sn[1] : 0;  //   CSR listings + reverse index + marginals
  out[14] = sn[3] > sn[2] ? sn[3] - sn[2] : 0;  //   packed-key / duplicate checks
  out[15] = sn[4] > sn[3] ? sn[4] - sn[3] : 0;  //   the k rounds
  return VALVE_OK;
}

int valve_pool_last_reclaim(const valve_pool* cp, int* handles, int64_t* evicted, int* inv_off,
                            int64_t* inv_pages, int* inv_phys, int* inv_blk, int cap_h, int cap_ev,
                            int cap_pages) {
  auto* p = const_cast<valve_pool*>(cp);
  return guard([&] {
    read_apply_results(p, handles, evicted, inv_off, inv_pages, inv_phys, inv_blk, cap_h, cap_ev,
                       cap_pages);
  });
}

int valve_pool_fill_pages(valve_pool* p) {
  return guard([&] {
    if (!p->d.pages) fail(VALVE_LOGIC_ERROR, "fill_pages: pool has no page store (slot_bytes = 0)");
    ck(cudaSetDevice(p->cfg.device), "cudaSetDevice");
    p->order_after_copy();
    k_fill_pages<<<148 * 8, 256, 0, p->stream>>>(p->d);
    counted();
    p->sync_and_check("fill_pages");
  });
}

int valve_pool_view_get(const valve_pool* p, valve_pool_view* v) {
  v->pages = p->d.pages;
  v->block_tables = p->d.bt;
  v->slot_bytes = p->d.slot_bytes;
  v->page_bytes = p->d.page_bytes;
  v->max_pages_per_request = p->Pblk;
  v->quarantine_page = p->d.quarantine;
  v->stream = p->stream;
  return VALVE_OK;
}

// -------------------------------------------------------------------------- reclaim copy

void valve_copy_params_default(valve_copy_params* c) {
  c->ctas = 16;
  c->threads = 512;
  c->chunk_bytes = 65536;
  c->rate_bytes_per_s = 0;
  c->burst_bytes = 0;
  c->use_tma = 1;  // shared-memory staged bulk copies (same link rate as the register-staged kernel)
  c->trace = nullptr;
}

int valve_pool_reclaim_copy_start(valve_pool* p, void* host_dst, int64_t dst_bytes,
                                  const valve_copy_params* prm) {
  return guard([&] {
    valve_copy_params c;
    valve_copy_params_default(&c);
    if (prm) c = *prm;
    if (c.ctas <= 0) c.ctas = 16;
    if (c.threads <= 0) c.threads = 512;
    if (c.chunk_bytes <= 0) c.chunk_bytes = 65536;
    if (!p->d.pages) fail(VALVE_LOGIC_ERROR, "reclaim_copy: pool has no page store");
    if (c.chunk_bytes % 16 || c.threads % 32 || c.threads > 512)
      fail(VALVE_INVALID_ARGUMENT, "reclaim_copy: chunk must be a 16-byte multiple, threads <= 512");
    if (p->cs_n == valve_pool::kCopySlots)
      fail(VALVE_LOGIC_ERROR, "reclaim_copy: the copy ring is full (call reclaim_copy_wait)");
    const int64_t need = p->last_copy_bytes;
    if (dst_bytes < need) fail(VALVE_INVALID_ARGUMENT, "reclaim_copy: destination too small");
    if (reinterpret_cast<uintptr_t>(host_dst) % 16)
      fail(VALVE_INVALID_ARGUMENT, "reclaim_copy: destination must be 16-byte aligned");
    const bool custom = p->last_custom != 0;
    ck(cudaSetDevice(p->cfg.device), "cudaSetDevice");
    void* ddst = nullptr;
    ck(cudaHostGetDevicePointer(&ddst, host_dst, 0),
       "reclaim_copy: destination is not pinned/mapped host memory");
    const int si = (p->cs_head + p->cs_n) % valve_pool::kCopySlots;
    valve_pool::CopySlot& S = p->cs[si];
    const int n_pages = p->last_n_pages, n_ev = p->last_n_evicted;
    CopyArgs A{};
    A.pages = p->d.pages;
    A.slot_bytes = p->d.slot_bytes;
    A.page_bytes = p->d.page_bytes;
    A.chunk_bytes = c.chunk_bytes;
    A.phys = S.phys;
    A.n_pages = n_pages;
    const int64_t cpp = (A.page_bytes + c.chunk_bytes - 1) / c.chunk_bytes;
    A.n_chunks = (int64_t)A.n_pages * cpp;
    A.dst = static_cast<uint8_t*>(ddst);
    A.ns_per_byte = c.rate_bytes_per_s > 0 ? 1e9 / c.rate_bytes_per_s : 0.0;
    A.burst_bytes = c.burst_bytes;
    A.burst_ns = (double)std::max<int64_t>(c.burst_bytes, 0) * A.ns_per_byte;
    A.tat = p->d_tat;
    A.trace = static_cast<unsigned long long*>(c.trace);
    A.cursor = S.ctr;
    A.t_first = S.ctr + 1;
    A.t_last = S.ctr + 2;
    // landed tickets: wave-major order (one wave = the same chunk_bytes of every page) when the
    // page size is uniform; otherwise the whole copy is one wave
    A.wave_major = (!custom && cpp <= valve_pool::kMaxWaves && n_pages > 0) ? 1 : 0;
    A.n_waves = n_pages == 0 ? 0 : (A.wave_major ? (int)cpp : 1);
    A.wave_done = S.waves;
    A.wave_next = S.waves + valve_pool::kMaxWaves;
    A.ctas_done = S.waves + valve_pool::kMaxWaves + 1;
    A.landed = p->d_landed;
    A.wave_base = p->waves_issued;
    // the copy runs on its own stream after the report exists and works from its own snapshot
    // of it; bookkeeping and the next decision proceed on the pool stream meanwhile
    // the snapshot runs on the plan stream, so a copy queued behind a running one does not hold
    // the next decision back; the slot is free (its previous copy completed: ring FIFO + wait)
    ck(cudaEventRecord(p->ev_report, p->stream), "event");
    ck(cudaStreamWaitEvent(p->plan_stream, p->ev_report, 0), "event wait");
    const cudaMemcpyKind d2d = cudaMemcpyDeviceToDevice;
    if (n_pages) ck(cudaMemcpyAsync(S.phys, p->d.res_phys, (size_t)n_pages * 4, d2d, p->plan_stream), "snapshot");
    if (custom && n_ev) {
      ck(cudaMemcpyAsync(S.inv_off, p->d.res_inv_off, (size_t)(n_ev + 1) * 4, d2d, p->plan_stream), "snapshot");
      ck(cudaMemcpyAsync(S.ev_pbytes, p->d.res_ev_pbytes, (size_t)n_ev * 8, d2d, p->plan_stream), "snapshot");
      ck(cudaMemcpyAsync(S.ev_base, p->d.res_ev_base, (size_t)(n_ev + 1) * 8, d2d, p->plan_stream), "snapshot");
    }
    ck(cudaEventRecord(S.ev_plan, p->plan_stream), "event");
    ck(cudaStreamWaitEvent(p->copy_stream, S.ev_plan, 0), "event wait");
    ck(cudaMemsetAsync(S.ctr, 0, 24, p->copy_stream), "memset");
    ck(cudaMemsetAsync(S.waves, 0, (valve_pool::kMaxWaves + 2) * sizeof(unsigned), p->copy_stream), "memset");
    if (custom) {  // per-request page sizes: chunk prefix over the evicted requests first
      A.ev_pbytes = S.ev_pbytes;
      A.ev_base = S.ev_base;
      A.ev_cbase = S.ev_cbase;
      A.inv_off = S.inv_off;
      A.n_ev = n_ev;
      A.n_chunks = n_ev > 0 ? 1 : 0;  // the kernel reads the total from ev_cbase
      if (A.n_chunks) {
        k_copy_plan<<<1, 1024, 0, p->copy_stream>>>(A.ev_pbytes, A.inv_off, A.n_ev, A.chunk_bytes, S.ev_cbase);
        counted();
      }
    }
    ck(cudaEventRecord(S.ev0, p->copy_stream), "event");
    if (A.n_chunks > 0) {
      if (c.use_tma) {
        k_reclaim_copy_tma<<<c.ctas, 32, 2 * 32768, p->copy_stream>>>(A);
      } else {
        k_reclaim_copy<<<c.ctas, c.threads, 0, p->copy_stream>>>(A);
      }
      counted();
    }
    ck(cudaEventRecord(S.ev1, p->copy_stream), "event");
    ck(cudaGetLastError(), "reclaim_copy launch");
    S.bytes = need;
    S.pages = n_pages;
    S.wave_base = A.wave_base;
    S.n_waves = A.n_waves;
    S.wave_bytes = A.wave_major ? c.chunk_bytes : p->d.slot_bytes;
    p->waves_issued += (uint64_t)A.n_waves;
    p->cs_n++;
    p->cs_last = si;
  });
}

int valve_pool_reclaim_copy_wait(valve_pool* p, valve_copy_stats* st) {
  return guard([&] {
    if (!p->cs_n) fail(VALVE_LOGIC_ERROR, "reclaim_copy_wait: no copy in flight");
    ck(cudaSetDevice(p->cfg.device), "cudaSetDevice");
    valve_pool::CopySlot& S = p->cs[p->cs_head];
    ck(cudaEventSynchronize(S.ev1), "reclaim_copy");
    p->cs_head = (p->cs_head + 1) % valve_pool::kCopySlots;
    p->cs_n--;
    if (st) {
      float ms = 0;
      ck(cudaEventElapsedTime(&ms, S.ev0, S.ev1), "event");
      unsigned long long t[3];
      ck(cudaMemcpy(t, S.ctr, 24, cudaMemcpyDeviceToHost), "read");
      st->bytes = S.bytes;
      st->pages = S.pages;
      st->kernel_ms = ms;
      st->t_first_ns = t[1];
      st->t_last_ns = t[2];
    }
  });
}

int valve_pool_copy_ticket(const valve_pool* p, uint64_t* wave_base, int* n_waves, int64_t* wave_bytes) {
  return guard([&] {
    if (p->cs_last < 0) fail(VALVE_LOGIC_ERROR, "copy_ticket: no reclaim copy was started");
    const valve_pool::CopySlot& S = p->cs[p->cs_last];
    if (wave_base) *wave_base = S.wave_base;
    if (n_waves) *n_waves = S.n_waves;
    if (wave_bytes) *wave_bytes = S.wave_bytes;
  });
}

int valve_pool_wait_landed(valve_pool* p, uint64_t target, void* stream) {
  return guard([&] {
    const MemOps& op = memops();
    if (target > p->waves_issued)
      fail(VALVE_INVALID_ARGUMENT, "wait_landed: ticket beyond the waves of the copies started");
    if (target == 0) return;
    ck(cudaSetDevice(p->cfg.device), "cudaSetDevice");
    cu_ck(op.wait64((CUstream)(stream ? static_cast<cudaStream_t>(stream) : p->stream), dptr(p->d_landed),
                    (cuuint64_t)target, CU_STREAM_WAIT_VALUE_GEQ),
          "cuStreamWaitValue64");
  });
}

int valve_pool_landed(const valve_pool* p, uint64_t* landed, uint64_t* issued) {
  return guard([&] {
    ck(cudaSetDevice(p->cfg.device), "cudaSetDevice");
    unsigned long long v = 0;
    ck(cudaMemcpy(&v, p->d_landed, 8, cudaMemcpyDeviceToHost), "read");
    if (landed) *landed = v;
    if (issued) *issued = p->waves_issued;
  });
}

int valve_pool_reclaim_copy(valve_pool* p, void* host_dst, int64_t dst_bytes,
                            const valve_copy_params* prm, valve_copy_stats* st) {
  if (p->cs_n) {
    g_err = "reclaim_copy: a copy started with reclaim_copy_start is still in flight";
    return VALVE_LOGIC_ERROR;
  }
  const int rc = valve_pool_reclaim_copy_start(p, host_dst, dst_bytes, prm);
  if (rc != VALVE_OK) return rc;
  return valve_pool_reclaim_copy_wait(p, st);
}

int valve_pool_restore(valve_pool* p, int64_t req, const void* host_src, int n_pages,
                       const int* blk_of_page, const valve_copy_params* prm, valve_copy_stats* st) {
  return guard([&] {
    valve_copy_params c;
    valve_copy_params_default(&c);
    if (prm) c = *prm;
    if (c.ctas <= 0) c.ctas = 16;
    if (c.threads <= 0 || c.threads > 512 || c.threads % 32) c.threads = 512;
    if (c.chunk_bytes <= 0 || c.chunk_bytes % 16) c.chunk_bytes = 65536;
    if (!p->d.pages) fail(VALVE_LOGIC_ERROR, "restore: pool has no page store");
    if (n_pages < 0 || n_pages > p->Pblk) fail(VALVE_INVALID_ARGUMENT, "restore: bad page count");
    if (n_pages && !blk_of_page) fail(VALVE_INVALID_ARGUMENT, "restore: null block list");
    for (int i = 0; i < n_pages; ++i)
      if (blk_of_page[i] < 0 || blk_of_page[i] >= p->Pblk)
        fail(VALVE_OUT_OF_RANGE, "restore: block index out of range");
    if (reinterpret_cast<uintptr_t>(host_src) % 16)
      fail(VALVE_INVALID_ARGUMENT, "restore: source must be 16-byte aligned");
    ck(cudaSetDevice(p->cfg.device), "cudaSetDevice");
    p->order_after_copy();
    // the request's row (device lookup) -> block table row pointer
    k_offline_pages_of<<<1, 32, 0, p->stream>>>(p->d, req);
    counted();
    p->sync_and_check("restore");
    const int row = (int)p->mirror->r[1];
    const int64_t pb = p->mirror->r[2];  // the request's page size (set_page_bytes or the pool's)
    if (row < 0) fail(VALVE_LOGIC_ERROR, "restore: request holds no pages (reserve it first)");
    if (n_pages == 0) return;
    const void* dsrc = nullptr;
    ck(cudaHostGetDevicePointer(const_cast<void**>(&dsrc), const_cast<void*>(host_src), 0),
       "restore: source is not pinned/mapped host memory");
    ck(cudaMemcpyAsync(p->d_ids, blk_of_page, (size_t)n_pages * 4, cudaMemcpyHostToDevice, p->stream),
       "upload");
    ScatterArgs A{};
    A.pages = p->d.pages;
    A.slot_bytes = p->d.slot_bytes;
    A.page_bytes = pb;
    A.chunk_bytes = c.chunk_bytes;
    A.bt_row = p->d.bt + (int64_t)row * p->Pblk;
    A.nblk = p->d.row_nblk + row;
    A.blk_of_page = p->d_ids;
    A.n_pages = n_pages;
    A.n_chunks = (int64_t)n_pages * ((A.page_bytes + c.chunk_bytes - 1) / c.chunk_bytes);
    A.src = static_cast<const uint8_t*>(dsrc);
    A.quarantine = p->d.quarantine;
    ck(cudaMemsetAsync(p->d_copyctr, 0, 32, p->stream), "memset");
    A.cursor = p->d_copyctr;
    A.bad = p->d_copyctr + 3;
    ck(cudaEventRecord(p->ev0, p->stream), "event");
    k_restore_scatter<<<c.ctas, c.threads, 0, p->stream>>>(A);
    counted();
    ck(cudaEventRecord(p->ev1, p->stream), "event");
    ck(cudaGetLastError(), "restore launch");
    ck(cudaStreamSynchronize(p->stream), "restore");
    unsigned long long bad = 0;
    ck(cudaMemcpy(&bad, p->d_copyctr + 3, 8, cudaMemcpyDeviceToHost), "read");
    if (bad) fail(VALVE_LOGIC_ERROR, "restore: a block of the request is not mapped");
    if (st) {
      float ms = 0;
      ck(cudaEventElapsedTime(&ms, p->ev0, p->ev1), "event");
      st->bytes = (int64_t)n_pages * pb;
      st->pages = n_pages;
      st->kernel_ms = ms;
      st->t_first_ns = st->t_last_ns = 0;
    }
  });
}

int valve_stream_create(int device, int high_priority, void** out) {
  return guard([&] {
    ck(cudaSetDevice(device), "cudaSetDevice");
    int lo = 0, hi = 0;
    ck(cudaDeviceGetStreamPriorityRange(&lo, &hi), "priority range");
    cudaStream_t s = nullptr;
    ck(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, high_priority ? hi : lo), "stream");
    *out = s;
  });
}

void valve_stream_destroy(void* s) {
  if (s) cudaStreamDestroy(static_cast<cudaStream_t>(s));
}

int valve_stream_synchronize(void* s) {
  return guard([&] { ck(cudaStreamSynchronize(static_cast<cudaStream_t>(s)), "cudaStreamSynchronize"); });
}

int valve_host_alloc(int64_t bytes, void** out) {
  return guard([&] {
    if (bytes <= 0) fail(VALVE_INVALID_ARGUMENT, "host_alloc: bytes must be > 0");
    ck(cudaHostAlloc(out, (size_t)bytes, cudaHostAllocMapped | cudaHostAllocPortable), "cudaHostAlloc");
  });
}

void valve_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int valve_pool_reclaim_copy_ce(valve_pool* p, void* host_dst, int64_t dst_bytes, valve_copy_stats* st) {
  return guard([&] {
    if (!p->d.pages) fail(VALVE_LOGIC_ERROR, "reclaim_copy: pool has no page store");
    const int64_t need = p->last_copy_bytes;
    if (dst_bytes < need) fail(VALVE_INVALID_ARGUMENT, "reclaim_copy: destination too small");
    ck(cudaSetDevice(p->cfg.device), "cudaSetDevice");
    p->order_after_copy();
    std::vector<int> phys(p->last_n_pages);
    std::vector<size_t> sizes(phys.size(), (size_t)p->d.page_bytes);
    std::vector<size_t> offs(phys.size());
    if (!phys.empty()) {
      ck(cudaMemcpyAsync(phys.data(), p->d.res_phys, phys.size() * 4, cudaMemcpyDeviceToHost, p->stream), "read");
      std::vector<int64_t> pb(p->last_n_evicted), base(p->last_n_evicted + 1);
      std::vector<int> io(p->last_n_evicted + 1);
      if (p->last_custom) {
        ck(cudaMemcpyAsync(pb.data(), p->d.res_ev_pbytes, pb.size() * 8, cudaMemcpyDeviceToHost, p->stream), "read");
        ck(cudaMemcpyAsync(base.data(), p->d.res_ev_base, base.size() * 8, cudaMemcpyDeviceToHost, p->stream), "read");
        ck(cudaMemcpyAsync(io.data(), p->d.res_inv_off, io.size() * 4, cudaMemcpyDeviceToHost, p->stream), "read");
      }
      ck(cudaStreamSynchronize(p->stream), "read");
      for (size_t i = 0; i < phys.size(); ++i) offs[i] = i * (size_t)p->d.page_bytes;
      if (p->last_custom)
        for (int e = 0; e < p->last_n_evicted; ++e)
          for (int j = io[e]; j < io[e + 1]; ++j) {
            sizes[j] = (size_t)pb[e];
            offs[j] = (size_t)(base[e] + (int64_t)(j - io[e]) * pb[e]);
          }
    }
    // Pages that sit in consecutive physical slots and land back to back in the destination form
    // a run: one 2D copy-engine transfer (source pitch = slot, destination pitch = page) instead
    // of one transfer per page, so the per-copy setup no longer shows against the link rate.
    struct Run { size_t first, n; };
    std::vector<Run> runs;
    for (size_t i = 0; i < phys.size(); ++i) {
      if (!runs.empty()) {
        Run& r = runs.back();
        const size_t j = r.first + r.n - 1;
        if (phys[i] == phys[j] + 1 && sizes[i] == sizes[j] && offs[i] == offs[j] + sizes[j]) {
          ++r.n;
          continue;
        }
      }
      runs.push_back({i, 1});
    }
    ck(cudaEventRecord(p->ev0, p->stream), "event");
    for (const Run& r : runs) {
      uint8_t* dst = static_cast<uint8_t*>(host_dst) + offs[r.first];
      const uint8_t* src = p->d.pages + (int64_t)phys[r.first] * p->d.slot_bytes;
      const size_t w = sizes[r.first];
      if (r.n == 1 || w == (size_t)p->d.slot_bytes)
        ck(cudaMemcpyAsync(dst, src, w * r.n, cudaMemcpyDeviceToHost, p->stream), "cudaMemcpyAsync");
      else
        ck(cudaMemcpy2DAsync(dst, w, src, (size_t)p->d.slot_bytes, w, r.n, cudaMemcpyDeviceToHost, p->stream),
           "cudaMemcpy2DAsync");
    }
    ck(cudaEventRecord(p->ev1, p->stream), "event");
    ck(cudaStreamSynchronize(p->stream), "reclaim_copy_ce");
    if (st) {
      float ms = 0;
      ck(cudaEventElapsedTime(&ms, p->ev0, p->ev1), "event");
      st->bytes = need;
      st->pages = p->last_n_pages;
      st->kernel_ms = ms;
      st->t_first_ns = st->t_last_ns = 0;
    }
  });
}

}  // extern "C"

// =================================================================== selection (host instance)

namespace {

struct SelectCtx {
  int device = -1;
  cudaStream_t stream = nullptr;
  int64_t cap_n = 0, cap_nnz = 0, cap_m = 0;
  int* hid = nullptr;
  int64_t* mapped = nullptr;
  int* roff = nullptr;
  int64_t* reqs = nullptr;
  int* rref = nullptr;
  int64_t* keys = nullptr;
  int64_t* cost = nullptr;
  int64_t* marg = nullptr;
  int* taken = nullptr;
  int* ev = nullptr;
  int* qoff = nullptr;
  int* qcnt = nullptr;
  int* qh = nullptr;
  int* out = nullptr;
  int* pick = nullptr;
  int* status = nullptr;
  int64_t* result = nullptr;
  std::mutex mu;

  // stream-ordered (see regrow): a device-synchronizing cudaFree here would wait for a gated
  // tenant's stream parked behind a closed gate -- the host that would reopen it is in here
  template <class T>
  void grow(T*& ptr, int64_t n) {
    if (ptr) ck(cudaFreeAsync(ptr, stream), "cudaFreeAsync");
    ck(cudaMallocAsync((void**)&ptr, std::max<int64_t>(n, 1) * sizeof(T), stream), "cudaMallocAsync");
  }
  void reserve(int64_t n, int64_t nnz, int64_t m) {
    if (!stream) ck(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "stream");
    if (!status) {
      grow(status, 4);
      grow(result, 2);
    }
    if (n > cap_n) {
      cap_n = std::max<int64_t>(n, 2 * cap_n);
      grow(hid, cap_n);
      grow(mapped, cap_n);
      grow(roff, cap_n + 1);
      grow(marg, cap_n);
      grow(taken, cap_n);
      grow(out, cap_n);
      grow(pick, cap_n);
    }
    if (nnz > cap_nnz) {
      cap_nnz = std::max<int64_t>(nnz, 2 * cap_nnz);
      grow(reqs, cap_nnz);
      grow(rref, cap_nnz);
      grow(qh, cap_nnz);
    }
    const int64_t mm = std::max(m, n);
    if (mm > cap_m) {
      cap_m = std::max<int64_t>(mm, 2 * cap_m);
      grow(keys, cap_m);
      grow(cost, cap_m);
      grow(ev, cap_m);
      grow(qoff, cap_m + 1);
      grow(qcnt, std::max(cap_m, cap_n));
    }
  }
};

SelectCtx& select_ctx(int device) {
  static SelectCtx ctx[16];
  if (device < 0 || device >= 16) fail(VALVE_INVALID_ARGUMENT, "select: bad device ordinal");
  ctx[device].device = device;
  return ctx[device];
}

SelectArgs upload_instance(SelectCtx& C, int n, const int* ids, const int64_t* mapped, const int* off,
                           const int64_t* reqs, int m, const int64_t* keys, const int64_t* vals, int k,
                           int mode) {
  const int nnz = n ? off[n] : 0;
  C.reserve(n, nnz, m);
  auto up = [&](void* d, const void* h, size_t b) {
    if (b) ck(cudaMemcpyAsync(d, h, b, cudaMemcpyHostToDevice, C.stream), "upload");
  };
  up(C.hid, ids, (size_t)n * 4);
  if (mapped) up(C.mapped, mapped, (size_t)n * 8);
  up(C.roff, off, (size_t)(n + 1) * 4);
  up(C.reqs, reqs, (size_t)nnz * 8);
  up(C.keys, keys, (size_t)m * 8);
  up(C.cost, vals, (size_t)m * 8);
  if (nnz) {
    k_map_refs<<<(nnz + 255) / 256, 256, 0, C.stream>>>(C.reqs, nnz, C.keys, m, C.rref);
    counted();
  }
  SelectArgs A{};
  A.n = n;
  A.m = m;
  A.k = k;
  A.mode = mode;
  A.nnz = nnz;
  A.hid = C.hid;
  A.mapped = C.mapped;
  A.roff = C.roff;
  A.rref = C.rref;
  A.cost = C.cost;
  A.marg = C.marg;
  A.taken = C.taken;
  A.ev = C.ev;
  A.qoff = C.qoff;
  A.qcnt = C.qcnt;
  A.qh = C.qh;
  A.out = C.out;
  A.status = C.status;
  A.result = C.result;
  return A;
}

}  // namespace

extern "C" {

int valve_select(int device, int n, const int* ids, const int64_t* mapped, const int* off,
                 const int64_t* reqs, int m, const int64_t* keys, const int64_t* vals, int k, int mode,
                 int* out, int* n_out) {
  return guard([&] {
    const char* who = mode == 0 ? "selective_reclaim" : mode == 1 ? "fifo_reclaim" : "oracle_reclaim";
    if (mode < 0 || mode > 2) fail(VALVE_INVALID_ARGUMENT, "select: unknown mode");
    if (k < 0) fail(VALVE_INVALID_ARGUMENT, std::string(who) + ": k must be >= 0");  // reclaim.cpp:34,70,86
    if (mode == 2 && n > 20)
      fail(VALVE_INVALID_ARGUMENT, "oracle_reclaim: instance too large (> 20 handles)");  // reclaim.cpp:88
    if (n < 0 || m < 0) fail(VALVE_INVALID_ARGUMENT, "select: negative sizes");
    k = std::min(k, n);
    *n_out = k;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= 0)
      fail(VALVE_CUDA_ERROR, "no CUDA device: selection runs only on the GPU");
    SelectCtx& C = select_ctx(device);
    std::lock_guard<std::mutex> lk(C.mu);
    ck(cudaSetDevice(device), "cudaSetDevice");
    SelectArgs A = upload_instance(C, n, ids, mapped, off, reqs, m, keys, vals, k, mode);
    set_reclaim_smem_attrs();
    k_select_instance<<<1, kNT, kReclaimSmemBytes, C.stream>>>(A);
    counted();
    ck(cudaGetLastError(), "select launch");
    int status = 0;
    ck(cudaMemcpyAsync(&status, C.status, 4, cudaMemcpyDeviceToHost, C.stream), "read");
    if (k) ck(cudaMemcpyAsync(out, C.out, (size_t)k * 4, cudaMemcpyDeviceToHost, C.stream), "read");
    ck(cudaStreamSynchronize(C.stream), "select");
    if (status == kDetNoCost) fail(VALVE_INVALID_ARGUMENT, "reclaim: request without cost entry");
  });
}

int valve_evicted_cost(int device, int n, const int* ids, const int* off, const int64_t* reqs, int m,
                       const int64_t* keys, const int64_t* vals, const int* pick, int n_pick,
                       int64_t* cost) {
  return guard([&] {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= 0)
      fail(VALVE_CUDA_ERROR, "no CUDA device: evicted_cost runs only on the GPU");
    SelectCtx& C = select_ctx(device);
    std::lock_guard<std::mutex> lk(C.mu);
    ck(cudaSetDevice(device), "cudaSetDevice");
    if (n < 0 || m < 0 || n_pick < 0) fail(VALVE_INVALID_ARGUMENT, "evicted_cost: negative sizes");
    // size every buffer (the pick list may be longer than the instance: duplicates and unknown
    // ids are legal input, reclaim.cpp:19-31) BEFORE the upload -- growing afterwards would free
    // buffers the uploaded SelectArgs still point at
    C.reserve(std::max(n, n_pick), n ? off[n] : 0, m);
    SelectArgs A = upload_instance(C, n, ids, nullptr, off, reqs, m, keys, vals, 0, 0);
    if (n_pick)
      ck(cudaMemcpyAsync(C.pick, pick, (size_t)n_pick * 4, cudaMemcpyHostToDevice, C.stream), "upload");
    A.ev = C.ev;
    k_evicted_cost<<<1, 32, 0, C.stream>>>(A, C.pick, n_pick);
    counted();
    ck(cudaGetLastError(), "evicted_cost launch");
    int status = 0;
    ck(cudaMemcpyAsync(&status, C.status, 4, cudaMemcpyDeviceToHost, C.stream), "read");
    ck(cudaMemcpyAsync(cost, C.result, 8, cudaMemcpyDeviceToHost, C.stream), "read");
    ck(cudaStreamSynchronize(C.stream), "evicted_cost");
    if (status == kDetApplyRange) fail(VALVE_INVALID_ARGUMENT, "evicted_cost: unknown handle id");
    if (status == kDetNoCost) fail(VALVE_INVALID_ARGUMENT, "reclaim: request without cost entry");
  });
}

// =============================================================== reservation controller

}  // extern "C"

struct valve_resctl {
  valve_resparams p;
  int64_t t = 0, last_tick = 0;
  std::vector<int64_t> pressure;  // event times, ascending (record order)
};

extern "C" {

void valve_resparams_default(valve_resparams* p) {
  // memory.hpp:103-114
  p->alpha = 1.5;
  p->beta = 2.0;
  p->t_init_us = 1000000;
  p->delta_us = 100000;
  p->t_min_us = 100000;
  p->t_max_us = 60000000;
  p->window_us = 60000000;
  p->target_per_window = 1.0;
  p->h_min = 1;
  p->pressure_threshold = 0.9;
}

int valve_resctl_create(const valve_resparams* p, valve_resctl** out) {
  return guard([&] {
    // memory.cpp:213-218
    if (p->alpha <= 1.0 || p->beta <= 1.0)
      fail(VALVE_INVALID_ARGUMENT, "ReservationParams: alpha/beta must be > 1");
    if (p->t_init_us <= 0 || p->t_min_us <= 0 || p->t_max_us < p->t_min_us || p->window_us <= 0)
      fail(VALVE_INVALID_ARGUMENT, "ReservationParams: bad interval bounds");
    if (p->h_min < 0) fail(VALVE_INVALID_ARGUMENT, "ReservationParams: h_min must be >= 0");
    auto* c = new valve_resctl;
    c->p = *p;
    c->t = p->t_init_us;
    *out = c;
  });
}
void valve_resctl_destroy(valve_resctl* c) { delete c; }
int64_t valve_resctl_interval(const valve_resctl* c) { return c->t; }
int64_t valve_resctl_pressure_events(const valve_resctl* c) { return (int64_t)c->pressure.size(); }
int valve_resctl_grow_target(const valve_resctl* c, int h, int cap) {
  // memory.cpp:220-223 -- IEEE-double ceil, then clamps
  const int target = (int)std::ceil(c->p.alpha * (double)h);
  return std::min(std::max({target, h, 1}), cap);
}
void valve_resctl_record_pressure(valve_resctl* c, int64_t t) { c->pressure.push_back(t); }
int valve_resctl_release_due(const valve_resctl* c, int64_t t, int h) {
  // memory.cpp:227-234: quiet since the previous tick?
  if (h <= c->p.h_min) return 0;
  for (auto it = c->pressure.rbegin(); it != c->pressure.rend() && *it > c->last_tick; ++it)
    if (*it <= t) return 0;
  return 1;
}
void valve_resctl_note_tick(valve_resctl* c, int64_t t) { c->last_tick = t; }
int64_t valve_resctl_pressure_in_window(const valve_resctl* c, int64_t t) {
  // memory.cpp:248-255: events in (t - window, t]
  int64_t n = 0;
  for (auto it = c->pressure.rbegin(); it != c->pressure.rend() && *it > t - c->p.window_us; ++it)
    n += *it <= t;
  return n;
}
int64_t valve_resctl_window_tick(valve_resctl* c, int64_t t) {
  // memory.cpp:238-246: x beta (truncated double) on a hot window, - delta otherwise
  const double rate = (double)valve_resctl_pressure_in_window(c, t);
  if (rate > c->p.target_per_window)
    c->t = std::min((int64_t)((double)c->t * c->p.beta), c->p.t_max_us);
  else
    c->t = std::max(c->t - c->p.delta_us, c->p.t_min_us);
  return c->t;
}

}  // extern "C"

// ================================================================================= gate

struct valve_gate {
  int device = 0;
  GateDev* d = nullptr;
  cudaStream_t stream = nullptr;  // high priority
  std::vector<valve_gate*> peers;
  int64_t* d_prefix = nullptr;
  int64_t cap_prefix = 0;
  bool remote = false;  // words opened from another process (CUDA IPC): no stream, no kernels
  cudaStream_t work_stream = nullptr;  // default stream of gated work launched without one
  // leader of a TP group: one high-priority helper stream + event per member, so the waits
  // on the members' acks run concurrently (front-end waits are serial within a stream)
  std::vector<cudaStream_t> wait_streams;
  std::vector<cudaEvent_t> wait_events;
  int fanout_mode = VALVE_FANOUT_BATCHED;
  // The decode work list (tile prefix over the listed rows) is frozen by the first launch after
  // valve_offline_reset: resumed launches reuse it, so the striped cursors (the context save)
  // keep meaning the same tiles even when reclaims / re-admissions change the pool's rows.
  std::vector<void*> retired;  // replaced prefix buffers (freed with the gate)
  bool frozen = false;
  const int* frozen_rows = nullptr;
  int frozen_n = 0;
  int64_t frozen_chunk = 0;
  ~valve_gate() {
    if (stream) cudaStreamSynchronize(stream);
    if (work_stream) {
      cudaStreamSynchronize(work_stream);
      cudaStreamDestroy(work_stream);
    }
    for (cudaStream_t s : wait_streams) cudaStreamDestroy(s);
    for (cudaEvent_t e : wait_events) cudaEventDestroy(e);
    if (d && remote) cudaIpcCloseMemHandle(d);
    else if (d) cudaFree(d);
    if (d_prefix) cudaFree(d_prefix);
    for (void* r : retired) cudaFree(r);
    if (stream) cudaStreamDestroy(stream);
  }
};

namespace {
cudaStream_t as_stream(void* s, cudaStream_t dflt) { return s ? static_cast<cudaStream_t>(s) : dflt; }

// One submission of stream memory operations (executed in array order by the front end).
struct MemBatch {
  std::vector<CUstreamBatchMemOpParams> ops;
  void write32(const void* addr, uint32_t v) {
    CUstreamBatchMemOpParams p{};
    p.writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_32;
    p.writeValue.address = dptr(addr);
    p.writeValue.value = v;
    ops.push_back(p);
  }
  void write64(const void* addr, uint64_t v) {
    CUstreamBatchMemOpParams p{};
    p.writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_64;
    p.writeValue.address = dptr(addr);
    p.writeValue.value64 = v;
    ops.push_back(p);
  }
  void wait_eq32(const void* addr, uint32_t v) {
    CUstreamBatchMemOpParams p{};
    p.waitValue.operation = CU_STREAM_MEM_OP_WAIT_VALUE_32;
    p.waitValue.address = dptr(addr);
    p.waitValue.value = v;
    p.waitValue.flags = CU_STREAM_WAIT_VALUE_EQ;
    ops.push_back(p);
  }
  void submit(const MemOps& op, cudaStream_t st) {
    for (size_t i = 0; i < ops.size(); i += 256) {  // driver limit per call
      const unsigned n = (unsigned)std::min<size_t>(256, ops.size() - i);
      cu_ck(op.batch((CUstream)st, n, ops.data() + i, 0), "cuStreamBatchMemOp");
    }
  }
};
}  // namespace

extern "C" {

int valve_gate_create(int device, valve_gate** out) {
  return guard([&] {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= 0)
      fail(VALVE_CUDA_ERROR, "no CUDA device: the gate lives in HBM");
    memops();
    auto* g = new valve_gate;
    g->device = device;
    try {
      ck(cudaSetDevice(device), "cudaSetDevice");
      preload_kernels(device);
      int lo = 0, hi = 0;
      ck(cudaDeviceGetStreamPriorityRange(&lo, &hi), "priority range");
      ck(cudaStreamCreateWithPriority(&g->stream, cudaStreamNonBlocking, hi), "stream");
      ck(cudaMalloc((void**)&g->d, sizeof(GateDev)), "cudaMalloc");
      ck(cudaMemset(g->d, 0, sizeof(GateDev)), "memset");
    } catch (...) {
      delete g;
      throw;
    }
    *out = g;
  });
}

void valve_gate_destroy(valve_gate* g) { delete g; }

void* valve_gate_stream(const valve_gate* g) { return g->stream; }

int valve_gate_raise(valve_gate* g, uint32_t gen, void* s) {
  return guard([&] {
    const MemOps& op = memops();
    cudaStream_t st = as_stream(s, g->stream);
    ck(cudaSetDevice(g->device), "cudaSetDevice");
    // one submission: every member's `closed` word first (leader, then the TP members over peer
    // memory -- a flat fan-out), the diagnostic generation after (t_first_seen is cleared at
    // release, while nothing polls)
    MemBatch b;
    b.write32(&g->d->closed, 1);
    for (valve_gate* x : g->peers) b.write32(&x->d->closed, 1);
    b.write32(&g->d->gen, gen);  // diagnostic generation: the leader's word only (each memop ~1 us)
    b.submit(op, st);
  });
}

int valve_gate_raise_stamped(valve_gate* g, uint32_t gen, void* s) {
  return guard([&] {
    cudaStream_t st = as_stream(s, g->stream);
    ck(cudaSetDevice(g->device), "cudaSetDevice");
    k_gate_raise_stamp<<<1, 1, 0, st>>>(g->d, gen);
    counted();
    ck(cudaGetLastError(), "raise_stamped");
  });
}

int valve_gate_release(valve_gate* g, uint32_t gen, void* s) {
  return guard([&] {
    const MemOps& op = memops();
    cudaStream_t st = as_stream(s, g->stream);
    ck(cudaSetDevice(g->device), "cudaSetDevice");
    std::vector<valve_gate*> all{g};
    all.insert(all.end(), g->peers.begin(), g->peers.end());
    // clear the diagnostics first (nothing polls a closed gate, and a raise issued on another
    // stream after this release cannot have its first-seen stamp wiped), then reopen every
    // member and stamp the leader's gen
    MemBatch b;
    for (valve_gate* x : all) b.write64(&x->d->t_first_seen, 0);
    for (valve_gate* x : all) b.write32(&x->d->closed, 0);
    b.write32(&g->d->gen, gen);
    b.submit(op, st);
  });
}

int valve_gate_wait_quiesced(valve_gate* g, uint32_t gen, void* s) {
  return guard([&] {
    const MemOps& op = memops();
    cudaStream_t st = as_stream(s, g->stream);
    ck(cudaSetDevice(g->device), "cudaSetDevice");
    if (g->fanout_mode == VALVE_FANOUT_BATCHED || g->peers.empty()) {
      // one submission on `st`: the waits run in order, but every member started quiescing at
      // the raise, so each later wait finds its counter already at zero (cost ~ max, not sum)
      MemBatch b;
      b.wait_eq32(&g->d->live_ctas, 0);
      for (valve_gate* x : g->peers) b.wait_eq32(&x->d->live_ctas, 0);
      b.write32(&g->d->quiesced_gen, gen);  // the group's ack: on the leader's word
      b.submit(op, st);
      return;
    }
    // VALVE_FANOUT_STREAMS: members on their own helper streams (concurrent), joined by events
    for (size_t i = 0; i < g->peers.size(); ++i) {
      cudaStream_t ws = g->wait_streams[i];
      ck(cudaEventRecord(g->wait_events[2 * i], st), "event");  // order after the raise on st
      ck(cudaStreamWaitEvent(ws, g->wait_events[2 * i], 0), "event wait");
      cu_ck(op.wait32((CUstream)ws, dptr(&g->peers[i]->d->live_ctas), 0, CU_STREAM_WAIT_VALUE_EQ),
            "cuStreamWaitValue32");
      ck(cudaEventRecord(g->wait_events[2 * i + 1], ws), "event");
    }
    cu_ck(op.wait32((CUstream)st, dptr(&g->d->live_ctas), 0, CU_STREAM_WAIT_VALUE_EQ), "cuStreamWaitValue32");
    cu_ck(op.write32((CUstream)st, dptr(&g->d->quiesced_gen), gen, 0), "cuStreamWriteValue32");
    for (size_t i = 0; i < g->peers.size(); ++i)
      ck(cudaStreamWaitEvent(st, g->wait_events[2 * i + 1], 0), "event wait");
  });
}

int valve_gate_wait_closed_quiesced(valve_gate* g, void* s) {
  return guard([&] {
    if (g->remote) fail(VALVE_LOGIC_ERROR, "gate_wait_closed_quiesced: call it on the member's own gate");
    const MemOps& op = memops();
    cudaStream_t st = as_stream(s, g->stream);
    ck(cudaSetDevice(g->device), "cudaSetDevice");
    MemBatch b;
    b.wait_eq32(&g->d->closed, 1);
    b.wait_eq32(&g->d->live_ctas, 0);
    b.submit(op, st);
  });
}

int valve_gate_set_fanout(valve_gate* g, int mode) {
  return guard([&] {
    if (mode != VALVE_FANOUT_BATCHED && mode != VALVE_FANOUT_STREAMS)
      fail(VALVE_INVALID_ARGUMENT, "gate_set_fanout: mode must be VALVE_FANOUT_BATCHED or VALVE_FANOUT_STREAMS");
    g->fanout_mode = mode;
  });
}

int valve_gate_export(const valve_gate* g, void* handle_out) {
  return guard([&] {
    if (g->remote) fail(VALVE_LOGIC_ERROR, "gate_export: a remote gate cannot be re-exported");
    static_assert(sizeof(cudaIpcMemHandle_t) <= VALVE_GATE_HANDLE_BYTES, "handle size");
    ck(cudaSetDevice(g->device), "cudaSetDevice");
    cudaIpcMemHandle_t h;
    ck(cudaIpcGetMemHandle(&h, g->d), "cudaIpcGetMemHandle");
    std::memset(handle_out, 0, VALVE_GATE_HANDLE_BYTES);
    std::memcpy(handle_out, &h, sizeof h);
  });
}

int valve_gate_open_remote(int device, const void* handle, valve_gate** out) {
  return guard([&] {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= 0)
      fail(VALVE_CUDA_ERROR, "no CUDA device: the gate lives in HBM");
    memops();
    auto* g = new valve_gate;
    g->device = device;
    g->remote = true;
    try {
      ck(cudaSetDevice(device), "cudaSetDevice");
      cudaIpcMemHandle_t h;
      std::memcpy(&h, handle, sizeof h);
      void* p = nullptr;
      ck(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
      g->d = static_cast<GateDev*>(p);
    } catch (...) {
      delete g;
      throw;
    }
    *out = g;
  });
}

int valve_gate_attach_peers(valve_gate* leader, valve_gate** members, int n) {
  return guard([&] {
    ck(cudaSetDevice(leader->device), "cudaSetDevice");
    for (int i = 0; i < n; ++i) {
      valve_gate* m = members[i];
      if (m->device != leader->device) {
        int ok = 0;
        ck(cudaDeviceCanAccessPeer(&ok, leader->device, m->device), "cudaDeviceCanAccessPeer");
        if (!ok) fail(VALVE_RUNTIME_ERROR, "attach_peers: no peer access between the GPUs");
        const cudaError_t e = cudaDeviceEnablePeerAccess(m->device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) ck(e, "cudaDeviceEnablePeerAccess");
        cudaGetLastError();
      }
      leader->peers.push_back(m);
      int lo = 0, hi = 0;
      ck(cudaDeviceGetStreamPriorityRange(&lo, &hi), "priority range");
      cudaStream_t ws = nullptr;
      ck(cudaStreamCreateWithPriority(&ws, cudaStreamNonBlocking, hi), "stream");
      leader->wait_streams.push_back(ws);
      for (int e = 0; e < 2; ++e) {
        cudaEvent_t ev = nullptr;
        ck(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
        leader->wait_events.push_back(ev);
      }
    }
  });
}

int valve_gate_read(const valve_gate* g, valve_gate_state* o) {
  return guard([&] {
    GateDev h{};
    ck(cudaSetDevice(g->device), "cudaSetDevice");
    ck(cudaMemcpy(&h, g->d, sizeof h, cudaMemcpyDeviceToHost), "read gate");
    o->gen = h.gen;
    o->closed = h.closed;
    o->quiesced_gen = h.quiesced_gen;
    o->live_ctas = h.live_ctas;
    o->t_first_seen_ns = h.t_first_seen;
    o->t_quiesced_ns = h.t_quiesced;
    o->tiles_done = h.tiles_done;
    o->canary_hits = h.canary;
    const int ns = h.stripes ? (int)std::min<unsigned long long>(h.stripes, kStripes) : kStripes;
    const unsigned long long per = (h.total + ns - 1) / ns;
    unsigned long long claimed = 0;
    for (int i = 0; i < ns; ++i) {
      const unsigned long long len = h.total > i * per ? std::min(per, h.total - i * per) : 0;
      claimed += std::min(h.cursor[i], len);
    }
    o->tiles_claimed = claimed;
    o->t_raise_ns = h.t_raise;
    o->total_tiles = h.total;
  });
}

int valve_offline_reset(valve_gate* g) {
  return guard([&] {
    ck(cudaSetDevice(g->device), "cudaSetDevice");
    ck(cudaMemsetAsync(&g->d->t_first_seen, 0, 4 * sizeof(unsigned long long), g->stream), "memset");
    ck(cudaMemsetAsync(g->d->cursor, 0, sizeof(g->d->cursor), g->stream), "memset");
    ck(cudaMemsetAsync(&g->d->frozen, 0, sizeof(unsigned), g->stream), "memset");
    ck(cudaStreamSynchronize(g->stream), "reset");
    g->frozen = false;
  });
}

int valve_offline_cancel(valve_gate* g) {
  return guard([&] {
    if (g->remote) fail(VALVE_LOGIC_ERROR, "offline_cancel: remote gate");
    ck(cudaSetDevice(g->device), "cudaSetDevice");
    // saturated cursors: every stripe reads as exhausted (the kernels compare before claiming)
    ck(cudaMemsetAsync(g->d->cursor, 0x7f, sizeof(g->d->cursor), g->stream), "memset");
    ck(cudaStreamSynchronize(g->stream), "cancel");
  });
}

int valve_offline_launch(valve_gate* g, valve_pool* p, const valve_offline_work* w, void* s) {
  return guard([&] {
    const MemOps& op = memops();
    if (!p->d.pages) fail(VALVE_LOGIC_ERROR, "offline_launch: pool has no page store");
    // rows == NULL: decode every request row of the pool (blocks from the device table)
    const bool all_rows = w->rows == nullptr;
    const int n_req = all_rows ? p->R : w->n_requests;
    const int* npages = all_rows ? p->d.row_nblk : w->npages;
    if (n_req <= 0) return;
    cudaStream_t st = as_stream(s, p->stream);
    ck(cudaSetDevice(g->device), "cudaSetDevice");
    const int64_t chunk = w->tile_bytes > 0 ? w->tile_bytes : 16384;
    if (chunk % 16) fail(VALVE_INVALID_ARGUMENT, "offline_launch: tile_bytes must be a 16-byte multiple");
    const int cpp = (int)((p->d.page_bytes + chunk - 1) / chunk);
    if (!g->frozen) {
      if (n_req + 1 > g->cap_prefix) {
        // an earlier launch may still read the old prefix (possibly queued behind a closed
        // gate): retire it to the gate's lifetime instead of freeing it now
        if (g->d_prefix) g->retired.push_back(g->d_prefix);
        g->cap_prefix = std::max<int64_t>(n_req + 1, 2 * g->cap_prefix);
        ck(cudaMalloc((void**)&g->d_prefix, g->cap_prefix * 8), "cudaMalloc");
      }
      g->frozen = true;
      g->frozen_rows = w->rows;
      g->frozen_n = n_req;
      g->frozen_chunk = chunk;
    } else if (g->frozen_rows != w->rows || g->frozen_n != n_req || g->frozen_chunk != chunk) {
      fail(VALVE_LOGIC_ERROR,
           "offline_launch: resumed with another work list (call valve_offline_reset for new work)");
    }
    // always enqueued (a no-op on the device once the list is frozen), so a captured launch
    // sequence freezes its list on the first replay after a reset, like a direct launch
    k_tile_prefix<<<1, kNT, 0, st>>>(npages, n_req, cpp, g->d_prefix, &g->d->total, &g->d->frozen);
    counted();
    int threads = w->threads > 0 ? w->threads : 256;
    int ctas = w->ctas;
    if (ctas <= 0) {
      int per_sm = 0, sms = 0;
      ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_offline_decode, threads, 0), "occupancy");
      ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device), "attr");
      // 16 warps per SM with 8 x 16 B loads in flight per lane saturate HBM; more warps only
      // stretch each tile (quiesce = one tile) without adding bandwidth
      ctas = std::min(per_sm, std::max(1, 512 / threads)) * sms;
    }
    // never start tiles into a closed gate; count the CTAs before they can retire
    cu_ck(op.write64((CUstream)st, dptr(&g->d->stripes), (cuuint64_t)kStripes, 0), "cuStreamWriteValue64");
    cu_ck(op.wait32((CUstream)st, dptr(&g->d->closed), 0, CU_STREAM_WAIT_VALUE_EQ), "cuStreamWaitValue32");
    cu_ck(op.write32((CUstream)st, dptr(&g->d->live_ctas), (cuuint32_t)ctas, 0), "cuStreamWriteValue32");
    OfflineArgs A{};
    A.g = g->d;
    A.pages = p->d.pages;
    A.slot_bytes = p->d.slot_bytes;
    A.page_bytes = p->d.page_bytes;
    A.chunk_bytes = chunk;
    A.chunks_per_page = cpp;
    A.bt = p->d.bt;
    A.P = p->Pblk;
    A.quarantine = p->d.quarantine;
    A.rows = w->rows;
    A.tile_prefix = g->d_prefix;
    A.n_requests = n_req;
    A.total_tiles = w->total_tiles;
    A.out = w->out;
    A.poll = w->poll;
    k_offline_decode<<<ctas, threads, 0, st>>>(A);
    counted();
    ck(cudaGetLastError(), "offline launch");
  });
}

namespace {
using PFN_encodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
PFN_encodeTiled encode_tiled() {
  static PFN_encodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&fn, cudaEnableDefault, &q);
  });
  if (!fn) fail(VALVE_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable in this driver");
  return fn;
}
// K-major bf16 [rows, k] -> boxes of box_rows x 64 (128 B, the SWIZZLE_128B span)
CUtensorMap kmajor_map(const void* base, int rows, int k, int box_rows) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {(cuuint64_t)k, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)k * 2};
  const cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  cu_ck(encode_tiled()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE),
        "cuTensorMapEncodeTiled");
  return m;
}
}  // namespace

int valve_offline_gemm(valve_gate* g, const valve_offline_gemm_work* w, void* s) {
  return guard([&] {
    const MemOps& op = memops();
    if (g->remote) fail(VALVE_LOGIC_ERROR, "offline_gemm: remote gate (launch on the owning process)");
    if (!w || !w->a || !w->b || !w->c) fail(VALVE_INVALID_ARGUMENT, "offline_gemm: null operand");
    if (w->m <= 0 || w->n <= 0 || w->k <= 0 || w->m % 128 || w->n % 256 || w->k % 64)
      fail(VALVE_INVALID_ARGUMENT, "offline_gemm: need m % 128 == 0, n % 256 == 0, k % 64 == 0");
    if ((reinterpret_cast<uintptr_t>(w->a) | reinterpret_cast<uintptr_t>(w->b) |
         reinterpret_cast<uintptr_t>(w->c)) % 16)
      fail(VALVE_INVALID_ARGUMENT, "offline_gemm: operands must be 16-byte aligned");
    ck(cudaSetDevice(g->device), "cudaSetDevice");
    // never the gate's own stream: the raise must be able to overtake the running work
    if (!s && !g->work_stream)
      ck(cudaStreamCreateWithFlags(&g->work_stream, cudaStreamNonBlocking), "cudaStreamCreate");
    cudaStream_t st = as_stream(s, g->work_stream);
    if (w->mode < 0 || w->mode > 2) fail(VALVE_INVALID_ARGUMENT, "offline_gemm: mode must be 0, 1 or 2");
    if (w->mode == 2 && w->m % 256) fail(VALVE_INVALID_ARGUMENT, "offline_gemm: CTA pairs need m % 256 == 0");
    // auto = CTA pairs (tcgen05 cta_group::2) whenever m allows: 1,484 vs 1,368 TFLOP/s for
    // single-CTA tiles at 4096x37888x3584 on B200 (cuBLAS 1,624)
    const bool pair = w->mode == 2 || (w->mode == 0 && w->m % 256 == 0);
    // per device (cudaFuncSetAttribute applies to the current device); cheap to repeat
    ck(cudaFuncSetAttribute(k_offline_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, kGemmSmemBytes),
       "cudaFuncSetAttribute");
    ck(cudaFuncSetAttribute(k_offline_gemm_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, kGemmSmemBytes),
       "cudaFuncSetAttribute");
    const CUtensorMap ma = kmajor_map(w->a, w->m, w->k, 128);
    const CUtensorMap mb = kmajor_map(w->b, w->n, w->k, pair ? 128 : 256);  // pairs load half-B boxes
    int ctas = w->ctas;
    if (ctas <= 0) ck(cudaDeviceGetAttribute(&ctas, cudaDevAttrMultiProcessorCount, g->device), "attr");
    GemmArgs G{};
    G.g = g->d;
    G.c = w->c;
    G.m = w->m;
    G.n = w->n;
    G.k = w->k;
    G.total_tiles = (long long)(w->m / (pair ? 256 : 128)) * (w->n / 256);
    G.poll = w->poll;
    if (pair) ctas = 2 * (int)std::min<long long>(std::max(ctas / 2, 1), G.total_tiles);
    else ctas = (int)std::min<long long>(ctas, G.total_tiles);
    if (w->fresh) {
      ck(cudaMemsetAsync(&g->d->t_first_seen, 0, 4 * sizeof(unsigned long long), st), "memset");
      ck(cudaMemsetAsync(g->d->cursor, 0, sizeof(g->d->cursor), st), "memset");
    }
    cu_ck(op.write64((CUstream)st, dptr(&g->d->total), (cuuint64_t)G.total_tiles, 0), "cuStreamWriteValue64");
    cu_ck(op.write64((CUstream)st, dptr(&g->d->stripes), 1, 0), "cuStreamWriteValue64");
    cu_ck(op.wait32((CUstream)st, dptr(&g->d->closed), 0, CU_STREAM_WAIT_VALUE_EQ), "cuStreamWaitValue32");
    cu_ck(op.write32((CUstream)st, dptr(&g->d->live_ctas), (cuuint32_t)ctas, 0), "cuStreamWriteValue32");
    if (pair) {
      cudaLaunchConfig_t lc{};
      lc.gridDim = dim3(ctas);
      lc.blockDim = dim3(256);
      lc.dynamicSmemBytes = kGemmSmemBytes;
      lc.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      lc.attrs = at;
      lc.numAttrs = 1;
      ck(cudaLaunchKernelEx(&lc, k_offline_gemm_pair, ma, mb, G), "offline gemm (pair) launch");
    } else {
      k_offline_gemm<<<ctas, 256, kGemmSmemBytes, st>>>(ma, mb, G);
    }
    counted();
    ck(cudaGetLastError(), "offline gemm launch");
  });
}

}  // extern "C"

// ============================================================================= channel

struct valve_channel {
  // channel.hpp:69-79
  int64_t toggle = 0, cooldown = 0;
  valve_channel_hooks h{};
  int state = 0;  // 0 enabled, 1 disabling, 2 disabled, 3 enabling (channel.hpp:32)
  bool any_busy = false, enable_after_disable = false, cooldown_pending = false;
  int64_t gen = 0, cooldown_gen = 0, effective_at = 0, disables = 0;
  valve_gate* gate = nullptr;

  void log(int64_t t, int what, int64_t aux, int mem) {
    if (h.log) h.log(h.user, t, what, aux, mem);
  }
  // First failed device-gate store since the last valve_channel_gate_status() (the state
  // machine's entry points return void, like the reference's): sticky, so a failed raise is
  // never lost between two edges.
  int gate_status = VALVE_OK;
  std::string gate_err;
  void gate_store(int rc) {
    if (rc != VALVE_OK && gate_status == VALVE_OK) {
      gate_status = rc;
      gate_err = g_err;
    }
  }
  void gate_raise() {
    if (gate) gate_store(valve_gate_raise(gate, (uint32_t)gen, gate_stream));
  }
  void gate_release() {
    if (gate) gate_store(valve_gate_release(gate, (uint32_t)gen, gate_stream));
  }
  void* gate_stream = nullptr;  // stream the gate stores are issued on (NULL: the gate's own)
  void issue_disable(int64_t t, bool mem) {
    // channel.cpp:13-20; the device gate closes at issue (offline stops at its next tile)
    state = 1;
    effective_at = t + toggle;
    ++gen;
    ++disables;
    gate_raise();
    if (h.schedule) h.schedule(h.user, effective_at, gen, 0);
    log(t, 0, effective_at, mem ? 1 : 0);
  }
  void issue_enable(int64_t t) {
    // channel.cpp:22-28
    state = 3;
    effective_at = t + toggle;
    ++gen;
    if (h.schedule) h.schedule(h.user, effective_at, gen, 0);
    log(t, 2, effective_at, 0);
  }
};

extern "C" {

int valve_channel_create(int64_t toggle, int64_t cooldown, const valve_channel_hooks* hooks,
                         valve_channel** out) {
  return guard([&] {
    if (toggle < 0 || cooldown < 0)
      fail(VALVE_INVALID_ARGUMENT, "ChannelController: latencies must be >= 0");  // channel.cpp:9-10
    auto* c = new valve_channel;
    c->toggle = toggle;
    c->cooldown = cooldown;
    if (hooks) c->h = *hooks;
    *out = c;
  });
}
void valve_channel_destroy(valve_channel* c) { delete c; }
int valve_channel_bind_gate(valve_channel* c, valve_gate* g) {
  c->gate = g;
  return VALVE_OK;
}
int valve_channel_bind_gate_stream(valve_channel* c, valve_gate* g, void* stream) {
  c->gate = g;
  c->gate_stream = stream;
  return VALVE_OK;
}
int valve_channel_gate_status(valve_channel* c) {
  const int rc = c->gate_status;
  if (rc != VALVE_OK) g_err = "ChannelController: device gate store failed: " + c->gate_err;
  c->gate_status = VALVE_OK;
  c->gate_err.clear();
  return rc;
}
int valve_channel_state(const valve_channel* c) { return c->state; }
int valve_channel_offline_compute_allowed(const valve_channel* c) { return c->state == 0; }
int64_t valve_channel_disables_issued(const valve_channel* c) { return c->disables; }
int64_t valve_channel_pending_effective(const valve_channel* c) { return c->effective_at; }

void valve_channel_note_busy(valve_channel* c, int64_t t) {
  // channel.cpp:30-39
  c->any_busy = true;
  c->enable_after_disable = false;
  if (c->cooldown_pending) {
    c->cooldown_pending = false;
    ++c->cooldown_gen;
    c->log(t, 5, 0, 0);
  }
  if (c->state == 0 || c->state == 3) c->issue_disable(t, false);
}

void valve_channel_note_all_idle(valve_channel* c, int64_t t) {
  // channel.cpp:41-48
  c->any_busy = false;
  if (c->state == 0 || c->state == 3) return;
  c->cooldown_pending = true;
  ++c->cooldown_gen;
  if (c->h.schedule) c->h.schedule(c->h.user, t + c->cooldown, c->cooldown_gen, 1);
  c->log(t, 4, t + c->cooldown, 0);
}

int64_t valve_channel_ensure_disabled(valve_channel* c, int64_t t) {
  // channel.cpp:50-62
  if (c->state == 2) return t;
  if (c->state == 1) return c->effective_at;
  c->issue_disable(t, true);
  return c->effective_at;
}

void valve_channel_handle_toggle(valve_channel* c, int64_t t, int64_t gen) {
  // channel.cpp:64-79
  if (gen != c->gen) return;
  if (c->state == 1) {
    c->state = 2;
    c->log(t, 1, 0, 0);
    if (c->h.on_disabled) c->h.on_disabled(c->h.user, t);
    if (c->enable_after_disable && !c->any_busy) {
      c->enable_after_disable = false;
      c->issue_enable(t);
    }
  } else if (c->state == 3) {
    c->state = 0;
    c->gate_release();  // offline may claim tiles again
    c->log(t, 3, 0, 0);
    if (c->h.on_enabled) c->h.on_enabled(c->h.user, t);
  }
}

void valve_channel_handle_cooldown(valve_channel* c, int64_t t, int64_t gen) {
  // channel.cpp:81-90
  if (gen != c->cooldown_gen || !c->cooldown_pending) return;
  c->cooldown_pending = false;
  if (c->any_busy) return;
  if (c->state == 2) c->issue_enable(t);
  else if (c->state == 1) c->enable_after_disable = true;
}

}  // extern "C"
