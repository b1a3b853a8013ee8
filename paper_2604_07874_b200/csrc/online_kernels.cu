// online_kernels.cu -- the ONLINE tenant's paged decode attention (harness, not the valve hot
// path): the real-time loop's Llama-3-8B keeps its KV in the pool's 2 MiB slots (one 16-token
// page of all 32 layers per slot, SURVEY §8 geometry), so a decode step attends straight from
// the slots its block table names -- no gather copy.  libonline.so, sm_100a.
//
// Slot layout (bytes from the slot base): layer l at l * layer_bytes; K at +0, V at +v_off;
// kv head g at g * head_bytes; inside a head 16 tokens x 128 dims bf16 (4 KiB).
//
// Split-K flash decoding: CTA (b, g, s) handles query heads g*rep .. g*rep+rep-1 (one warp
// each, GQA) over pages [s*pps, (s+1)*pps) of request b with an online softmax; a second kernel
// merges the splits (log-sum-exp).  Memory-bound: each K/V page tile is read once per layer.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>

namespace {

constexpr int kD = 128, kTok = 16;

__device__ __forceinline__ float bf(const __nv_bfloat16 x) { return __bfloat162float(x); }

__global__ void __launch_bounds__(256) k_paged_decode(const __nv_bfloat16* __restrict__ q, const uint8_t* pages,
                                                      int64_t slot_bytes, int64_t layer_off, int64_t v_off,
                                                      int64_t head_bytes, const int* __restrict__ bt, int bt_stride,
                                                      const int* __restrict__ lens, int hq, int rep, float scale_log2,
                                                      int pps, float* __restrict__ part_acc,
                                                      float* __restrict__ part_ml, int splits) {
  __shared__ __align__(16) __nv_bfloat16 sk[kTok * kD];
  __shared__ __align__(16) __nv_bfloat16 sv[kTok * kD];
  const int b = blockIdx.x, g = blockIdx.y, s = blockIdx.z;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = g * rep + w;  // this warp's query head
  const int len = lens[b];
  const int npages = (len + kTok - 1) / kTok;
  const int p0 = s * pps, p1 = min(npages, p0 + pps);
  float qv[4], acc[4] = {0.f, 0.f, 0.f, 0.f};
  const __nv_bfloat16* qh = q + ((int64_t)b * hq + h) * kD + lane * 4;
#pragma unroll
  for (int i = 0; i < 4; ++i) qv[i] = bf(qh[i]) * scale_log2;
  float m = -INFINITY, l = 0.f;
  const int nthr = blockDim.x;
  for (int p = p0; p < p1; ++p) {
    const int phys = bt[(int64_t)b * bt_stride + p];
    const uint8_t* kb = pages + (int64_t)phys * slot_bytes + layer_off + (int64_t)g * head_bytes;
    const uint4* ks = reinterpret_cast<const uint4*>(kb);
    const uint4* vs = reinterpret_cast<const uint4*>(kb + v_off);
    __syncthreads();  // the previous page's tiles are consumed
    for (int i = threadIdx.x; i < kTok * kD / 8; i += nthr) {
      reinterpret_cast<uint4*>(sk)[i] = ks[i];
      reinterpret_cast<uint4*>(sv)[i] = vs[i];
    }
    __syncthreads();
    const int valid = min(kTok, len - p * kTok);
    float sc[kTok];
    float mp = -INFINITY;
#pragma unroll
    for (int t = 0; t < kTok; ++t) {
      const __nv_bfloat162* kr = reinterpret_cast<const __nv_bfloat162*>(sk + t * kD + lane * 4);
      const float2 a = __bfloat1622float2(kr[0]), c = __bfloat1622float2(kr[1]);
      float x = qv[0] * a.x + qv[1] * a.y + qv[2] * c.x + qv[3] * c.y;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      sc[t] = t < valid ? x : -INFINITY;
      mp = fmaxf(mp, sc[t]);
    }
    const float mn = fmaxf(m, mp);
    const float corr = exp2f(m - mn);
    l *= corr;
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i] *= corr;
#pragma unroll
    for (int t = 0; t < kTok; ++t) {
      const float pt = exp2f(sc[t] - mn);
      l += pt;
      const __nv_bfloat162* vr = reinterpret_cast<const __nv_bfloat162*>(sv + t * kD + lane * 4);
      const float2 a = __bfloat1622float2(vr[0]), c = __bfloat1622float2(vr[1]);
      acc[0] += pt * a.x;
      acc[1] += pt * a.y;
      acc[2] += pt * c.x;
      acc[3] += pt * c.y;
    }
    m = mn;
  }
  const int64_t idx = ((int64_t)b * hq + h) * splits + s;
  float4* pa = reinterpret_cast<float4*>(part_acc + idx * kD) + lane;
  *pa = make_float4(acc[0], acc[1], acc[2], acc[3]);
  if (lane == 0) {
    part_ml[idx * 2] = m;
    part_ml[idx * 2 + 1] = l;
  }
}

__global__ void k_paged_combine(const float* __restrict__ part_acc, const float* __restrict__ part_ml, int hq,
                                int splits, __nv_bfloat16* __restrict__ out) {
  const int b = blockIdx.x, h = blockIdx.y, d = threadIdx.x;
  const int64_t base = ((int64_t)b * hq + h) * splits;
  float M = -INFINITY;
  for (int s = 0; s < splits; ++s) M = fmaxf(M, part_ml[(base + s) * 2]);
  float num = 0.f, den = 0.f;
  if (M > -INFINITY) {
    for (int s = 0; s < splits; ++s) {
      const float ms = part_ml[(base + s) * 2];
      if (ms == -INFINITY) continue;
      const float f = exp2f(ms - M);
      num += f * part_acc[(base + s) * kD + d];
      den += f * part_ml[(base + s) * 2 + 1];
    }
  }
  out[((int64_t)b * hq + h) * kD + d] = __float2bfloat16(den > 0.f ? num / den : 0.f);
}

// SM clock probe (diagnostics of the real-time harness): one thread spins ~4 us of %globaltimer
// and stores the SM clock (clock64 ticks per ns * 1000 = MHz) into out[slot].
__global__ void k_clock_probe(float* out, int slot) {
  uint64_t g0, g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  const long long c0 = clock64();
  do {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  } while (g1 - g0 < 4000);
  const long long c1 = clock64();
  out[slot] = (float)(c1 - c0) * 1000.f / (float)(g1 - g0);
}

}  // namespace

extern "C" {

int online_clock_probe(float* out, int slot, void* stream) {
  k_clock_probe<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(out, slot);
  return (int)cudaGetLastError();
}


// q, out: bf16 [B, hq, 128] (device).  bt: int32 [B, bt_stride] physical slots, lens: int32 [B]
// tokens to attend (incl. the one just written).  part_acc: fp32 [B*hq*splits*128], part_ml:
// fp32 [B*hq*splits*2] scratch.  Returns a cudaError_t.
int online_paged_decode_attn(const void* q, const void* pages, int64_t slot_bytes, int64_t layer_off,
                             int64_t v_off, int64_t head_bytes, const int* bt, int bt_stride, const int* lens,
                             int B, int hq, int hkv, float scale, int splits, int pages_per_split,
                             float* part_acc, float* part_ml, void* out, void* stream) {
  if (B <= 0) return 0;
  const int rep = hq / hkv;
  if (rep * hkv != hq || rep < 1 || rep > 8 || splits < 1 || pages_per_split < 1) return (int)cudaErrorInvalidValue;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const float scale_log2 = scale * 1.4426950408889634f;
  k_paged_decode<<<dim3(B, hkv, splits), 32 * rep, 0, st>>>(
      static_cast<const __nv_bfloat16*>(q), static_cast<const uint8_t*>(pages), slot_bytes, layer_off, v_off,
      head_bytes, bt, bt_stride, lens, hq, rep, scale_log2, pages_per_split, part_acc, part_ml, splits);
  k_paged_combine<<<dim3(B, hq), kD, 0, st>>>(part_acc, part_ml, hq, splits, static_cast<__nv_bfloat16*>(out));
  return (int)cudaGetLastError();
}

}  // extern "C"
