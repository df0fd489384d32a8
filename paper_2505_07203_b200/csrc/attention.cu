// Causal GQA prefill attention on tcgen05 (FlashAttention-style, full sequence in one pass).
//
// Realises _attention (ps/numerics.py:132-146): softmax(Q K^T / sqrt(d)) V with the causal (triu) mask,
// generalised to multi-head GQA with head_dim 128 and a q_offset so that rows of cached prefix tokens
// (n_cached, ps/costs.py:275-277) serve only as keys.
//
// Layout: one bf16 buffer qkv[n_total, ld] per layer; columns [0,Hq*128) = Q (roped), then K, then V.
// Rows [0, q_offset) hold only K/V (cached prefix, gathered from the prefix pool); rows >= q_offset are
// the miss tokens. Output ctx[n_total - q_offset, Hq*128] bf16.
//
// CTA = one 128-row query block x one kv head x two query heads of that group (K/V tiles shared).
//   warps 0-3   softmax for query head slot 0 (thread = query row = TMEM lane)
//   warps 4-7   softmax for query head slot 1
//   warp  8     TMA loader (Q once, K/V 128-key tiles through a 2-stage ring)
//   warp  9     MMA issuer: S_i = Q_i K^T (SS), O_i += P_i V (TS: P read straight from TMEM)
//   warp 10     TMEM allocator (S0 | S1 | O0 | O1, 128 columns each)
// P is written back by the softmax warps as bf16 over the first 64 columns of S_i. The running max is
// kept stale until it grows by > 8 (log2 units), so O is rescaled in TMEM only rarely; the final
// normalisation divides by the matching running sum, so the result is exact softmax.
#include "sm100.cuh"
#include "attention.cuh"
#include "../../include/prefillonly.h"
#include <cmath>
#include <cstdlib>

namespace po {
int set_error(int code, const char* fmt, ...);
void keep_pool_memory();
int make_tmap_2d_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t row_stride_bytes,
                      uint32_t box_inner, uint32_t box_outer);
int make_tmap_3d_bf16(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t stride1_bytes,
                      uint64_t stride2_bytes, uint32_t b0, uint32_t b1, uint32_t b2);
int make_tmap_4d_bf16(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t d3,
                      uint64_t stride1_bytes, uint64_t stride2_bytes, uint64_t stride3_bytes, uint32_t b0, uint32_t b1,
                      uint32_t b2, uint32_t b3);

namespace {
constexpr int HD = 128;
constexpr int BQ = 128;
constexpr int BKV = 128;
constexpr int BOX_BYTES = 128 * 64 * 2;        // one 128-row x 64-col swizzled box (16 KB)
constexpr int TILE_BYTES = 2 * BOX_BYTES;      // 128 x 128 bf16
constexpr int NTHREADS = 384;
constexpr int SMEM_BYTES = 6 * TILE_BYTES + 1024 + 256;
constexpr float RESCALE_THRESHOLD = 8.0f;      // log2 units
#ifndef POLY_NUM
#define POLY_NUM 3  // POLY_NUM of every POLY_DEN exp2 pairs run as the FMA-pipe polynomial (MUFU offload)
#endif
#ifndef POLY_DEN
#define POLY_DEN 8
#endif
}  // namespace

struct AttnArgs {
  int n_total;     // keys (= rows of qkv)
  int q_offset;    // first query row (cached prefix length)
  int n_q;         // query rows
  int hq, hkv, pairs;
  int num_qb;
  __nv_bfloat16* out;
  long long ldo;
  float scale_log2;
  int splits;         // KV splits per (query block, head pair); 1 = write normalised bf16 output directly
  int tiles_per_split;
  __nv_bfloat16* part_o;  // [splits][n_q][hq*128] unnormalised partial outputs, bf16 (splits > 1)
  float2* part_ml;    // [splits][n_q][hq] (running max in log2 units, running sum)
  int mode;           // what the two 128-row TMEM slots of a CTA hold (see AttnLayout)
  int R;              // MODE_PACKED: query rows per head in a slot (128 / GQA group)
  int G;              // GQA group size (query heads per kv head)
  int num_units;      // CTAs per split: query blocks (HEADS x head pairs), block pairs x heads, or chunk pairs x kv
  // Pool-direct keys: rows [0, n_pool) of K/V are read straight from the prefix pool ([slot][layer][16][kv_dim],
  // block b of the request in slot pool_slots[b]) instead of a gathered copy in qkv; rows >= n_pool from qkv.
  int n_pool;         // 0 = every key row from qkv
  const int* pool_slots;
  int pool_layer, pool_layers;  // map_pool block index = slot * pool_layers + pool_layer
  int pool_kcol, pool_vcol;     // column of this launch's K / V head 0 within a pool row
  int kv_band;                  // MODE_HEADS CTA order: kv heads per band (0 = all heads interleaved)
  int pool_runs;                // map_run is valid: whole tiles in 8 consecutive slots load as two boxes
};

// Slot layouts. HEADS: two query heads of one GQA group over the same 128-row query block (K/V shared).
// QBLOCKS: two consecutive 128-row query blocks of one head (odd groups, e.g. Qwen 40/8). PACKED: short queries
// (prefix hits) - each slot stacks the G heads of one kv group over R = 128/G query rows, so a 160-token miss
// suffix fills 128-row MMA tiles instead of padding every head to 128 rows.
enum AttnMode : int { MODE_HEADS = 0, MODE_QBLOCKS = 1, MODE_PACKED = 2 };

// ---- packed f32x2 math (sm_100 FFMA2 / FADD2) and a polynomial exp2 on the FMA pipe (MUFU offload)
__device__ __forceinline__ uint64_t pk2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void up2(uint64_t v, float& a, float& b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); }
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t fsub2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// 2^x for a pair, x <= ~8: Cody-Waite split x = j + f (j = rint(x), |f| <= 1/2), cubic minimax for 2^f
// (max rel. error 7.5e-5, far below the bf16 rounding of P), exponent add for 2^j. x is clamped at -125.
__device__ __forceinline__ void exp2_poly2(float x0, float x1, float& y0, float& y1) {
  const float MAGIC = 12582912.0f;  // 1.5 * 2^23: adding it rounds to an integer held in the low bits
  x0 = fmaxf(x0, -125.f);
  x1 = fmaxf(x1, -125.f);
  const uint64_t x = pk2(x0, x1);
  const uint64_t t = fadd2(x, pk2(MAGIC, MAGIC));
  const uint64_t f = fsub2(x, fsub2(t, pk2(MAGIC, MAGIC)));
  uint64_t p = ffma2(pk2(0.05517098f, 0.05517098f), f, pk2(0.2426097f, 0.2426097f));
  p = ffma2(p, f, pk2(0.69326097f, 0.69326097f));
  p = ffma2(p, f, pk2(0.99992818f, 0.99992818f));
  float p0, p1, t0, t1;
  up2(p, p0, p1);
  up2(t, t0, t1);
  y0 = __int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23));
  y1 = __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23));
}

// One 128-key tile of online softmax for this thread's query row (TMEM lane). The whole row of S is read from TMEM
// once into registers (one wait), the max
// uses 3-input FMNMX chains, and P is written back in 32-key chunks. `on_half` runs after the first 64 keys
// of P are stored (the caller may let the MMA warp start the first half of P.V early).
template <bool MASKED, typename HalfFn>
__device__ __forceinline__ void softmax_tile1(uint32_t s_addr, uint32_t o_addr, int lim, float sl2, int j, float& m,
                                              float& l, HalfFn on_half) {
  uint32_t v[128];
#pragma unroll
  for (int c = 0; c < 4; ++c) tmem_ld32(s_addr + c * 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32 * c));
  tmem_ld_wait();
  if (MASKED) {
#pragma unroll
    for (int c = 0; c < 128; ++c)
      if (c >= lim) v[c] = __float_as_uint(-INFINITY);
  }
  float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
  for (int e = 0; e < 128; e += 8) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      mx[k] = fmaxf(mx[k], fmaxf(__uint_as_float(v[e + 2 * k]), __uint_as_float(v[e + 2 * k + 1])));
  }
  const float m_new = fmaxf(m, fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])) * sl2);
  const bool resc = m_new > m + RESCALE_THRESHOLD;
  const float alpha = resc ? ex2_approx(m - m_new) : 1.0f;
  if (j > 0 && __any_sync(0xffffffffu, resc)) {
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
      uint32_t o[32];
      tmem_ld32(o_addr + c * 32, o);
      tmem_ld_wait();
#pragma unroll
      for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
      tmem_st32(o_addr + c * 32, o);
    }
    tmem_st_wait();
  }
  if (resc) {
    l *= alpha;
    m = m_new;
  }
  const float nm = -m;
  const uint64_t sc2 = pk2(sl2, sl2), nm2 = pk2(nm, nm);
  uint64_t acc0 = pk2(0.f, 0.f), acc1 = pk2(0.f, 0.f);
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint32_t p[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int col = 32 * c + 2 * e;
      float x0, x1;
      up2(ffma2(pk2(__uint_as_float(v[col]), __uint_as_float(v[col + 1])), sc2, nm2), x0, x1);
      if (!MASKED && (e % POLY_DEN) >= POLY_DEN - POLY_NUM) {
        exp2_poly2(x0, x1, x0, x1);
      } else {
        x0 = ex2_approx(x0);
        x1 = ex2_approx(x1);
      }
      if (MASKED) {  // rows with no visible key yet (m = -inf) would otherwise produce NaN
        if (col >= lim) x0 = 0.f;
        if (col + 1 >= lim) x1 = 0.f;
      }
      if (e & 1)
        acc1 = fadd2(acc1, pk2(x0, x1));
      else
        acc0 = fadd2(acc0, pk2(x0, x1));
      p[e] = pack_bf16(x0, x1);
    }
    tmem_st16(s_addr + c * 16, p);  // P columns [16c, 16c+16): S already in registers
    if (c == 1) on_half();
  }
  float s0, s1, s2, s3;
  up2(acc0, s0, s1);
  up2(acc1, s2, s3);
  l += (s0 + s1) + (s2 + s3);
}


// ATTN_SPLIT_S=1 (build-time A/B): S in two N = 64 halves, the first half's softmax overlapping the second half's
// MMA. Bit-identical results, but measured slower (20k: 1279 vs 1394 TFLOP/s, 64k: 1180 vs 1278; two waits and TMEM
// load rounds per tile, 24 bytes of spills): off.
#ifndef ATTN_SPLIT_S
#define ATTN_SPLIT_S 0
#endif
// One P chunk c (keys 32c .. 32c+31) of this row: x = s*sl2 - m, exp2 (MUFU or the FMA-pipe polynomial), the row sum
// in acc0/acc1 (pairs alternate), bf16 P stored over S columns [16c, 16c+16). Same arithmetic as softmax_tile1.
template <bool MASKED>
__device__ __forceinline__ void p_chunk(const uint32_t (&v)[128], int c, uint32_t s_addr, int lim, uint64_t sc2,
                                        uint64_t nm2, uint64_t& acc0, uint64_t& acc1) {
  uint32_t p[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const int col = 32 * c + 2 * e;
    float x0, x1;
    up2(ffma2(pk2(__uint_as_float(v[col]), __uint_as_float(v[col + 1])), sc2, nm2), x0, x1);
    if (!MASKED && (e % POLY_DEN) >= POLY_DEN - POLY_NUM) {
      exp2_poly2(x0, x1, x0, x1);
    } else {
      x0 = ex2_approx(x0);
      x1 = ex2_approx(x1);
    }
    if (MASKED) {
      if (col >= lim) x0 = 0.f;
      if (col + 1 >= lim) x1 = 0.f;
    }
    if (e & 1)
      acc1 = fadd2(acc1, pk2(x0, x1));
    else
      acc0 = fadd2(acc0, pk2(x0, x1));
    p[e] = pack_bf16(x0, x1);
  }
  tmem_st16(s_addr + c * 16, p);
}

// softmax_tile1 with S arriving in two 64-key halves (ATTN_SPLIT_S): the first half is read as soon as its N = 64
// MMA commits (s_half) and its P chunks are computed with the running max while the tensor core computes the second
// half; the row max over all 128 keys then decides as before (rescale only when it grew by > RESCALE_THRESHOLD). If
// it did, O is rescaled and the first half's P recomputed with the new max, so the result is bit-identical to
// softmax_tile1. P of the first half is signalled (p_half) once the max is known to be final.
template <bool MASKED, typename HalfFn>
__device__ __forceinline__ void softmax_tile2(uint32_t s_addr, uint32_t o_addr, int lim, float sl2, int j, float& m,
                                              float& l, HalfFn on_half, uint64_t* s_half_bar, uint64_t* s_full_bar) {
  uint32_t v[128];
  mbar_wait(s_half_bar, j & 1);
  tc_fence_after();
  tmem_ld32(s_addr, *reinterpret_cast<uint32_t(*)[32]>(v));
  tmem_ld32(s_addr + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
  tmem_ld_wait();
  if (MASKED) {
#pragma unroll
    for (int c = 0; c < 64; ++c)
      if (c >= lim) v[c] = __float_as_uint(-INFINITY);
  }
  float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
  for (int e = 0; e < 64; e += 8) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      mx[k] = fmaxf(mx[k], fmaxf(__uint_as_float(v[e + 2 * k]), __uint_as_float(v[e + 2 * k + 1])));
  }
  // speculative first half with the running max (kept unless the whole row's max forces a rescale)
  const bool spec = m != -INFINITY;
  uint64_t acc0 = pk2(0.f, 0.f), acc1 = pk2(0.f, 0.f);
  {
    const uint64_t sc2 = pk2(sl2, sl2), nm2 = pk2(-m, -m);
    if (spec) {
      p_chunk<MASKED>(v, 0, s_addr, lim, sc2, nm2, acc0, acc1);
      p_chunk<MASKED>(v, 1, s_addr, lim, sc2, nm2, acc0, acc1);
    }
  }
  mbar_wait(s_full_bar, j & 1);
  tc_fence_after();
  tmem_ld32(s_addr + 64, *reinterpret_cast<uint32_t(*)[32]>(v + 64));
  tmem_ld32(s_addr + 96, *reinterpret_cast<uint32_t(*)[32]>(v + 96));
  tmem_ld_wait();
  if (MASKED) {
#pragma unroll
    for (int c = 64; c < 128; ++c)
      if (c >= lim) v[c] = __float_as_uint(-INFINITY);
  }
#pragma unroll
  for (int e = 64; e < 128; e += 8) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      mx[k] = fmaxf(mx[k], fmaxf(__uint_as_float(v[e + 2 * k]), __uint_as_float(v[e + 2 * k + 1])));
  }
  const float m_new = fmaxf(m, fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])) * sl2);
  const bool resc = m_new > m + RESCALE_THRESHOLD;
  const float alpha = resc ? ex2_approx(m - m_new) : 1.0f;
  const bool redo = __any_sync(0xffffffffu, resc) || !spec;  // warp-uniform
  if (j > 0 && __any_sync(0xffffffffu, resc)) {
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
      uint32_t o[32];
      tmem_ld32(o_addr + c * 32, o);
      tmem_ld_wait();
#pragma unroll
      for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
      tmem_st32(o_addr + c * 32, o);
    }
    tmem_st_wait();
  }
  if (resc) {
    l *= alpha;
    m = m_new;
  }
  const uint64_t sc2 = pk2(sl2, sl2), nm2 = pk2(-m, -m);
  if (redo) {  // the first half again with the final max (same order of the sums as softmax_tile1)
    acc0 = pk2(0.f, 0.f);
    acc1 = pk2(0.f, 0.f);
    p_chunk<MASKED>(v, 0, s_addr, lim, sc2, nm2, acc0, acc1);
    p_chunk<MASKED>(v, 1, s_addr, lim, sc2, nm2, acc0, acc1);
  }
  on_half();
  p_chunk<MASKED>(v, 2, s_addr, lim, sc2, nm2, acc0, acc1);
  p_chunk<MASKED>(v, 3, s_addr, lim, sc2, nm2, acc0, acc1);
  float s0, s1, s2, s3;
  up2(acc0, s0, s1);
  up2(acc1, s2, s3);
  l += (s0 + s1) + (s2 + s3);
}

// -DATTN_TRACE: clock64 stamps of the pipeline events of one CTA (blockIdx.x == ATTN_TRACE) for tools/attn_trace.py
#ifdef ATTN_TRACE
constexpr int TRACE_EVENTS = 24, TRACE_TILES = 512;
__device__ unsigned long long g_attn_trace[TRACE_EVENTS * TRACE_TILES];
#define TR(ev, j) \
  do { if (blockIdx.x == ATTN_TRACE && (j) < TRACE_TILES) g_attn_trace[(ev) * TRACE_TILES + (j)] = clock64(); } while (0)
#else
#define TR(ev, j) do { } while (0)
#endif
// -DATTN_SPAN: globaltimer at entry, after setup, and at exit of every CTA (tools/attn_span.py), plus its split / unit
#ifdef ATTN_SPAN
__device__ unsigned long long g_attn_span[8192 * 4];
__device__ __forceinline__ unsigned long long span_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define SPAN(i, v) do { if (threadIdx.x == 0 && blockIdx.x < 8192) g_attn_span[blockIdx.x * 4 + (i)] = (v); } while (0)
#else
#define SPAN(i, v) do { } while (0)
#endif

__global__ void __launch_bounds__(NTHREADS, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap map, const __grid_constant__ CUtensorMap map_q,
                    const __grid_constant__ CUtensorMap map_pool, const __grid_constant__ CUtensorMap map16,
                    const __grid_constant__ CUtensorMap map_run, const AttnArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint8_t* sQ = smem;                       // 2 tiles
  uint8_t* sK = smem + 2 * TILE_BYTES;      // 2 stages
  uint8_t* sV = smem + 4 * TILE_BYTES;      // 2 stages
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 6 * TILE_BYTES);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;    // [2]
  uint64_t* v_full = bars + 3;    // [2]
  uint64_t* k_empty = bars + 5;   // [2] K stage free: both slots' S MMAs of the tile are done
  uint64_t* s_full = bars + 7;    // [2] per head slot
  uint64_t* p_full = bars + 9;    // [2]
  uint64_t* o_final = bars + 11;  // [2]
  uint64_t* p_half = bars + 13;   // [2] first 64 keys of P stored
  uint64_t* v_empty = bars + 15;  // [2] V stage free: both slots' P.V MMAs of the tile are done
  uint64_t* s_half = bars + 17;   // [2] first 64 keys of S computed (ATTN_SPLIT_S)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 19);

  const int warp = warp_id();
  const int lane = lane_id();
  if (threadIdx.x == 0) TR(21, 0);
#ifdef ATTN_SPAN
  SPAN(0, span_now());
#endif

  // heaviest (longest causal extent) units first. Slot i of this CTA: head hs_i (first head of the kv group
  // when packed), first query position qs_i; rows_slot query rows per head in the slot.
  int unit = a.num_units - 1 - blockIdx.x / (a.splits * (a.mode == MODE_HEADS ? a.hkv * a.pairs
                                                          : a.mode == MODE_QBLOCKS ? a.hq : a.hkv));
  int split, g, hs0, hs1, qs0, qs1;
  int rows_slot = BQ;
  if (a.mode == MODE_HEADS) {
    // kv_band > 0 (long sequences): CTAs run in bands of kv_band kv heads (heaviest query block first within a
    // band), so the CTAs resident at any time share the K/V of a few heads and that working set stays in L2
    const int band = a.kv_band > 0 ? a.kv_band : a.hkv;
    const int per_qb = band * a.pairs * a.splits;
    const int band_ctas = a.num_units * per_qb;
    const int b = a.kv_band > 0 ? blockIdx.x / band_ctas : 0;
    const int r = a.kv_band > 0 ? blockIdx.x % band_ctas : blockIdx.x;
    unit = a.num_units - 1 - r / per_qb;
    int rem = r % per_qb;
    split = rem % a.splits;
    rem /= a.splits;
    g = b * band + rem / a.pairs;
    hs0 = g * (2 * a.pairs) + 2 * (rem % a.pairs);
    hs1 = hs0 + 1;
    qs0 = qs1 = a.q_offset + unit * BQ;
  } else if (a.mode == MODE_QBLOCKS) {
    const int rem = blockIdx.x % (a.hq * a.splits);
    split = rem % a.splits;
    hs0 = hs1 = rem / a.splits;
    g = hs0 / a.G;
    qs0 = a.q_offset + unit * 2 * BQ;
    qs1 = qs0 + BQ;
  } else {
    const int rem = blockIdx.x % (a.hkv * a.splits);
    split = rem % a.splits;
    g = rem / a.splits;
    hs0 = hs1 = g * a.G;
    rows_slot = a.R;
    qs0 = a.q_offset + unit * 2 * a.R;
    qs1 = qs0 + a.R;
  }
  const int q_lo = qs0;                                     // earliest query position of the CTA
  const int q_hi = min(qs1 + rows_slot - 1, a.n_total - 1); // last real query position of the CTA
  const int all_tiles = q_hi / BKV + 1;
  const int t0 = split * a.tiles_per_split;                 // this CTA's KV tile range [t0, t0 + n_tiles)
  const int n_tiles = max(0, min(all_tiles, t0 + a.tiles_per_split) - t0);

  if (n_tiles == 0) return;  // a KV split past this query block's causal extent (uniform across the CTA)
#ifdef ATTN_SPAN
  SPAN(3, ((unsigned long long)split << 32) | (unsigned)unit);
#endif

  if (warp == 8 && lane == 0) {
    tma_prefetch_desc(&map);
    for (int i = 0; i < 19; ++i) mbar_init(&bars[i], (i == 9 || i == 10 || i == 13 || i == 14) ? 128 : 1);
    fence_barrier_init();
  }
  if (warp == 10) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) TR(21, 1);
#ifdef ATTN_SPAN
  SPAN(1, span_now());
#endif
  pdl_wait();     // qkv of this layer (QKV GEMM, pool gather) complete
  pdl_trigger();
  // registers move from the loader/MMA warpgroup (warps 8-11) to the two softmax warpgroups, which hold a
  // whole 128-key row of S: 2 x 128 x 208 + 128 x 80 <= 384 x 168, the CTA's pool (asking for more blocks
  // setmaxnreg.inc forever). Issued inside each role branch so ptxas allocates each region to its own budget.
  if (warp >= 8) {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 80;\n" ::: "memory");
  if (warp == 8) {
    const uint64_t keep = l2_policy_evict_last();
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, 2 * TILE_BYTES);
      if (a.mode != MODE_PACKED) {
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int half = 0; half < 2; ++half)
            tma_load_2d(sQ + i * TILE_BYTES + half * BOX_BYTES, &map, q_full, (i ? hs1 : hs0) * HD + half * 64,
                        i ? qs1 : qs0);
      } else {
        // slot i = G stacked (R rows x 128) head tiles; each R-row box lands 1024-B aligned (R % 8 == 0)
        for (int i = 0; i < 2; ++i)
          for (int k = 0; k < a.G; ++k)
#pragma unroll
            for (int half = 0; half < 2; ++half)
              tma_load_2d(sQ + i * TILE_BYTES + half * BOX_BYTES + k * a.R * 128, &map_q, q_full,
                          (g * a.G + k) * HD + half * 64, i ? qs1 : qs0);
      }
    }
    const int kcol = a.hq * HD + g * HD;
    const int vcol = (a.hq + a.hkv) * HD + g * HD;
    // Pool-direct tiles: lanes 0-7 hold the pool slots of the tile's eight 16-key blocks, fetched one tile ahead
    auto tile_slots = [&](int jj) -> int {
      const int blk = (t0 + jj) * (BKV / 16) + (lane & 7);
      return (jj < n_tiles && blk * 16 < a.n_pool) ? __ldg(a.pool_slots + blk) : 0;
    };
    int nxt = a.n_pool > 0 ? tile_slots(0) : 0;
    // one 128-key K or V tile: a 128-row box from qkv, or per 16-key block a pool box (cached rows) or a 16-row box
    // from qkv (the miss rows of the tile straddling n_pool); 16-row boxes land at 2 KB steps (swizzle-consistent)
    auto load_kv = [&](uint8_t* dst, uint64_t* bar, int col, int pcol, int kr, int cur) {
      if (kr >= a.n_pool) {
        if (lane == 0) {
          tma_load_2d_hint(dst, &map, bar, col, kr, keep);
          tma_load_2d_hint(dst + BOX_BYTES, &map, bar, col + 64, kr, keep);
        }
        return;
      }
      // a whole cached tile whose eight blocks sit in consecutive slots (the usual case: a request's prefix is
      // admitted in order into free slots): two 128-row boxes over [slot][layer][16][kv_dim], as many TMA
      // operations as a tile from qkv instead of sixteen 16-row boxes
      const int s0 = __shfl_sync(0xffffffffu, cur, 0);
      if (a.pool_runs && kr + BKV <= a.n_pool && __all_sync(0xffffffffu, cur == s0 + (lane & 7))) {
        if (lane == 0) {
          tma_load_4d_hint(dst, &map_run, bar, pcol, 0, a.pool_layer, s0, keep);
          tma_load_4d_hint(dst + BOX_BYTES, &map_run, bar, pcol + 64, 0, a.pool_layer, s0, keep);
        }
        return;
      }
      // lane b < 8 issues block b's two boxes (the TMA issue work of a pool tile spreads over 8 lanes)
      if (lane < BKV / 16) {
        const int r = kr + 16 * lane;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          uint8_t* d = dst + half * BOX_BYTES + lane * 2048;
          if (r < a.n_pool)
            tma_load_3d_hint(d, &map_pool, bar, pcol + half * 64, 0, cur * a.pool_layers + a.pool_layer, keep);
          else
            tma_load_2d_hint(d, &map16, bar, col + half * 64, r, keep);
        }
      }
    };
    for (int j = 0; j < n_tiles; ++j) {
      const int st = j & 1;
      const uint32_t ph = (j >> 1) & 1;
      const int cur = nxt;
      if (a.n_pool > 0) nxt = tile_slots(j + 1);
      // K of tile j+2 streams in as soon as the S MMAs of tile j are done, well before its P.V
      mbar_wait(&k_empty[st], ph ^ 1);
      TR(14, j);
      const int kr = (t0 + j) * BKV;
      if (lane == 0) mbar_arrive_expect_tx(&k_full[st], TILE_BYTES);
      __syncwarp();  // expect_tx before any lane's copies complete on the barrier
      load_kv(sK + st * TILE_BYTES, &k_full[st], kcol, a.pool_kcol + g * HD, kr, cur);
      mbar_wait(&v_empty[st], ph ^ 1);
      TR(20, j);
      if (lane == 0) mbar_arrive_expect_tx(&v_full[st], TILE_BYTES);
      __syncwarp();
      load_kv(sV + st * TILE_BYTES, &v_full[st], vcol, a.pool_vcol + g * HD, kr, cur);
    }
    __syncwarp();
  } else if (warp == 9) {
    // the whole warp runs the issue loop (warp-uniform descriptors stay in uniform registers) and one elected lane
    // issues the MMAs and commits
    {
      const bool issuer = elect_one();
      constexpr uint32_t idesc_s = idesc_bf16_f32(128, ATTN_SPLIT_S ? 64 : 128, false, false);
      constexpr uint32_t idesc_o = idesc_bf16_f32(128, 128, false, true);
      auto issue_s = [&](int i, int st) {
#if ATTN_SPLIT_S
        // two N = 64 halves (keys 0..63, then 64..127 = +64 rows of the K tile), committed separately
#pragma unroll
        for (int h = 0; h < 2; ++h) {
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {
            const uint32_t off = (kk >> 2) * BOX_BYTES + (kk & 3) * 32;
            if (issuer) mma_bf16_ss(tmem + i * 128 + h * 64, sdesc_kmajor_sw128(smem_u32(sQ + i * TILE_BYTES + off)),
                        sdesc_kmajor_sw128(smem_u32(sK + st * TILE_BYTES + off + h * 64 * 128)), idesc_s, kk > 0);
          }
          if (issuer) mma_commit(h == 0 ? &s_half[i] : &s_full[i]);
        }
#else
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * BOX_BYTES + (kk & 3) * 32;
          if (issuer) mma_bf16_ss(tmem + i * 128, sdesc_kmajor_sw128(smem_u32(sQ + i * TILE_BYTES + off)),
                      sdesc_kmajor_sw128(smem_u32(sK + st * TILE_BYTES + off)), idesc_s, kk > 0);
        }
        if (issuer) mma_commit(&s_full[i]);
#endif
      };
      auto issue_pv_range = [&](int i, int st, bool acc, int k0, int k1) {
#pragma unroll
        for (int kk = k0; kk < k1; ++kk) {
          const uint64_t vdesc = sdesc_mnmajor_sw128(smem_u32(sV + st * TILE_BYTES + kk * 16 * 128), BOX_BYTES, 1024);
          if (issuer) mma_bf16_ts(tmem + 256 + i * 128, tmem + i * 128 + kk * 8, vdesc, idesc_o, (acc || kk > 0) ? 1u : 0u);
        }
      };
      // O_i += P_i V once P_i is in TMEM: the first 64 keys go as soon as their half of P is
      auto issue_pv = [&](int i, int st, bool acc, int j) {
        mbar_wait(&p_half[i], j & 1);
        TR(8 + 3 * i, j);
        tc_fence_after();
        issue_pv_range(i, st, acc, 0, BKV / 32);
        TR(15 + 3 * i, j);
        mbar_wait(&p_full[i], j & 1);
        TR(9 + 3 * i, j);
        tc_fence_after();
        issue_pv_range(i, st, acc, BKV / 32, BKV / 16);
        TR(16 + 3 * i, j);
      };
      mbar_wait(q_full, 0);
      mbar_wait(&k_full[0], 0);
      tc_fence_after();
      issue_s(0, 0);
      issue_s(1, 0);
      if (issuer) mma_commit(&k_empty[0]);
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        const bool more = j + 1 < n_tiles;
        const int st2 = (j + 1) & 1;
        const uint32_t ph2 = ((j + 1) >> 1) & 1;
        mbar_wait(&v_full[st], ph);
        issue_pv(0, st, j > 0, j);
        if (!more && issuer) mma_commit(&o_final[0]);
        if (more) {
          mbar_wait(&k_full[st2], ph2);
          TR(10, j);
          tc_fence_after();
          issue_s(0, st2);
          TR(17, j);
        }
        issue_pv(1, st, j > 0, j);
        if (issuer) mma_commit(&v_empty[st]);
        if (!more && issuer) mma_commit(&o_final[1]);
        if (more) {
          issue_s(1, st2);
          if (issuer) mma_commit(&k_empty[st2]);
        }
        TR(13, j);
      }
    }
    __syncwarp();
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 208;\n" ::: "memory");
    const int i = warp >> 2;
    const int r = (warp & 3) * 32 + lane;
    const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t s_addr = tmem + lane_base + i * 128;
    const uint32_t o_addr = tmem + lane_base + 256 + i * 128;
    const int my_qlo = i ? qs1 : qs0;  // smallest query position in the slot
    const bool packed = a.mode == MODE_PACKED;
    const int my_h = packed ? (i ? hs1 : hs0) + r / a.R : (i ? hs1 : hs0);
    const int qr = packed ? r % a.R : r;  // query row within the slot
    const int pos = my_qlo + qr;
    float m = -INFINITY;  // running max (scaled, log2 units), possibly stale
    float l = 0.f;
    const bool tr_lane = ((warp & 3) | lane) == 0;
    for (int j = 0; j < n_tiles; ++j) {
      if (tr_lane) TR(4 * i, j);
#if !ATTN_SPLIT_S
      mbar_wait(&s_full[i], j & 1);
      tc_fence_after();
#endif
      if (tr_lane) TR(4 * i + 1, j);
      const int kbase = (t0 + j) * BKV;
      // the first 64 keys of P are signalled as soon as they are stored (the MMA warp starts that half of P.V)
      auto half = [&]() {
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&p_half[i]);
        if (tr_lane) TR(4 * i + 2, j);
      };
      // warp-uniform: only tiles crossing the diagonal of this query block pay for the mask
#if ATTN_SPLIT_S
      if (kbase + BKV - 1 > my_qlo)
        softmax_tile2<true>(s_addr, o_addr, pos - kbase + 1, a.scale_log2, j, m, l, half, &s_half[i], &s_full[i]);
      else
        softmax_tile2<false>(s_addr, o_addr, BKV, a.scale_log2, j, m, l, half, &s_half[i], &s_full[i]);
#else
      if (kbase + BKV - 1 > my_qlo)
        softmax_tile1<true>(s_addr, o_addr, pos - kbase + 1, a.scale_log2, j, m, l, half);
      else
        softmax_tile1<false>(s_addr, o_addr, BKV, a.scale_log2, j, m, l, half);
#endif
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&p_full[i]);
      if (tr_lane) TR(4 * i + 3, j);
    }
    mbar_wait(&o_final[i], 0);
    tc_fence_after();
    const int row = (packed && qr >= rows_slot) ? a.n_q : my_qlo - a.q_offset + qr;
    if (a.splits == 1) {
      const float inv = 1.0f / l;
      __nv_bfloat16* dst = a.out + (long long)row * a.ldo + my_h * HD;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t v[32];
        tmem_ld32(o_addr + c * 32, v);
        tmem_ld_wait();
        if (row < a.n_q) {
          uint4* d4 = reinterpret_cast<uint4*>(dst + c * 32);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            d4[q] = make_uint4(pack_bf16(__uint_as_float(v[8 * q + 0]) * inv, __uint_as_float(v[8 * q + 1]) * inv),
                               pack_bf16(__uint_as_float(v[8 * q + 2]) * inv, __uint_as_float(v[8 * q + 3]) * inv),
                               pack_bf16(__uint_as_float(v[8 * q + 4]) * inv, __uint_as_float(v[8 * q + 5]) * inv),
                               pack_bf16(__uint_as_float(v[8 * q + 6]) * inv, __uint_as_float(v[8 * q + 7]) * inv));
          }
        }
      }
    } else {
      // split-KV partial: unnormalised O, running max m (log2 units) and sum l for the combine kernel
      const long long prow = (long long)split * a.n_q + row;
      uint4* dst = reinterpret_cast<uint4*>(a.part_o + prow * (a.hq * HD) + my_h * HD);
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t v[32];
        tmem_ld32(o_addr + c * 32, v);
        tmem_ld_wait();
        if (row < a.n_q) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            dst[c * 4 + q] = make_uint4(pack_bf16(__uint_as_float(v[8 * q + 0]), __uint_as_float(v[8 * q + 1])),
                                        pack_bf16(__uint_as_float(v[8 * q + 2]), __uint_as_float(v[8 * q + 3])),
                                        pack_bf16(__uint_as_float(v[8 * q + 4]), __uint_as_float(v[8 * q + 5])),
                                        pack_bf16(__uint_as_float(v[8 * q + 6]), __uint_as_float(v[8 * q + 7])));
        }
      }
      if (row < a.n_q) a.part_ml[prow * a.hq + my_h] = make_float2(m, l);
    }
    if (tr_lane) TR(22 + i, 0);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 10) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
#ifdef ATTN_SPAN
  SPAN(2, span_now());
#endif
}

// out[row, h, :] = sum_s 2^(m_s - M) O_s / sum_s 2^(m_s - M) l_s over the KV splits that exist for the row's block
__global__ void attn_combine_kernel(const __nv_bfloat16* __restrict__ part_o, const float2* __restrict__ part_ml, int n_q,
                                    int hq, int splits, int tiles_per_split, int q_offset, int n_total, int span,
                                    __nv_bfloat16* __restrict__ out, long long ldo) {
  pdl_wait();
  pdl_trigger();
  // 32-bit indices (n_q * hq * 32 < 2^31 for any split launch: n_q <= 148 * 128): 64-bit divisions by hq are a
  // ~70-instruction software sequence each
  const int total = n_q * hq * (HD / 4);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int q4 = i % (HD / 4);
    const int rh = i / (HD / 4);
    const int h = rh % hq;
    const int row = rh / hq;
    const int q_hi = min(q_offset + (row / span) * span + span - 1, n_total - 1);
    const int all_tiles = q_hi / BKV + 1;
    const int ns = min(splits, (all_tiles + tiles_per_split - 1) / tiles_per_split);
    // split s of (row, h) at ml + s * stride, its O quad at o + s * stride * HD / 4 (pointer increments)
    const int rh_idx = row * hq + h;
    const size_t stride = (size_t)n_q * hq;
    const float2* ml = part_ml + rh_idx;
    const uint2* o4 = reinterpret_cast<const uint2*>(part_o) + (size_t)rh_idx * (HD / 4) + q4;
    float M = -INFINITY;
    {
      const float2* mp = ml;
#pragma unroll 4
      for (int s = 0; s < ns; ++s, mp += stride) M = fmaxf(M, mp->x);
    }
    float L = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s0 = 0; s0 < ns; s0 += 4) {
      // a group's (m, l) and O loads issued together, then the in-order weighted sums
      float2 mls[4];
      uint2 obs[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        mls[k] = s0 + k < ns ? *ml : make_float2(-INFINITY, 0.f);
        obs[k] = s0 + k < ns ? *o4 : make_uint2(0u, 0u);
        ml += stride;
        o4 += stride * (HD / 4);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (s0 + k < ns) {
          const float w = mls[k].x == -INFINITY ? 0.f : exp2f(mls[k].x - M);
          L += w * mls[k].y;
          const float2 o01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&obs[k].x));
          const float2 o23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&obs[k].y));
          acc.x += w * o01.x;
          acc.y += w * o01.y;
          acc.z += w * o23.x;
          acc.w += w * o23.y;
        }
      }
    }
    const float inv = 1.0f / L;
    reinterpret_cast<uint2*>(out + (long long)row * ldo + h * HD)[q4] =
        make_uint2(pack_bf16(acc.x * inv, acc.y * inv), pack_bf16(acc.z * inv, acc.w * inv));
  }
}

struct AttnLayout {
  int mode, R, G, units, ctas, span;  // units = CTAs per KV split; span = query rows per CTA
};

AttnLayout attention_layout(int n_total, int q_offset, int hq, int hkv) {
  AttnLayout L{};
  const int n_q = n_total - q_offset;
  const int num_qb = (n_q + BQ - 1) / BQ;
  L.G = hq / hkv;
  if (L.G % 2) {
    L.mode = MODE_QBLOCKS;
    L.units = (num_qb + 1) / 2;
    L.ctas = L.units * hq;
    L.span = 2 * BQ;
  } else {
    L.mode = MODE_HEADS;
    L.units = num_qb;
    L.ctas = num_qb * hq / 2;
    L.span = BQ;
  }
  L.R = BQ;
  // short queries (prefix hits): stack the group's heads into the 128-row tiles when that shrinks the grid
  if (L.G > 1 && BQ % L.G == 0 && (BQ / L.G) % 8 == 0 && L.ctas < 148) {
    const int R = BQ / L.G;
    const int pairs = ((n_q + R - 1) / R + 1) / 2;
    if (pairs * hkv < L.ctas) {
      L.mode = MODE_PACKED;
      L.R = R;
      L.units = pairs;
      L.ctas = pairs * hkv;
      L.span = 2 * R;
    }
  }
  return L;
}

// KV splits for a launch: split only when the layout's grid cannot fill the SMs.
void attention_split_plan(int n_total, int q_offset, int hq, int hkv, int* splits, int* tiles_per_split) {
  const int base = attention_layout(n_total, q_offset, hq, hkv).ctas;
  const int max_tiles = (n_total - 1) / BKV + 1;
  int s = 1;
  if (base < 148 && max_tiles >= 8) {
    // equal-work CTAs, one per SM: fill exactly one wave (a second partial wave costs a whole extra wave)
    s = 148 / base;
    s = min(s, max_tiles / 4);
    s = min(s, 32);
    s = max(s, 1);
  }
  const int tps = (max_tiles + s - 1) / s;
  *tiles_per_split = tps;
  *splits = (max_tiles + tps - 1) / tps;
}

size_t attention_workspace_bytes(int n_total, int q_offset, int hq, int hkv) {
  int s, tps;
  attention_split_plan(n_total, q_offset, hq, hkv, &s, &tps);
  if (s == 1) return 0;
  const size_t n_q = n_total - q_offset;
  return (size_t)s * n_q * hq * (HD * sizeof(__nv_bfloat16) + sizeof(float2));
}

int attention_run(const void* qkv, long long ld, int n_total, int q_offset, int hq, int hkv, void* out, long long ldo,
                  cudaStream_t stream, void* workspace, size_t workspace_bytes, const AttnPool* pool) {
  if (hq % hkv) return -3;
  const AttnLayout lay = attention_layout(n_total, q_offset, hq, hkv);
  CUtensorMap map, map_q, map_pool, map16, map_run;
  if (make_tmap_2d_bf16(&map, qkv, ld, n_total, ld * 2, 64, 128)) return -2;
  if (make_tmap_2d_bf16(&map_q, qkv, ld, n_total, ld * 2, 64, lay.R)) return -2;
  const bool use_pool = pool && pool->n_rows > 0;
  if (use_pool) {
    if (pool->block_tokens != 16 || pool->n_rows % 16 || pool->n_rows > n_total) return -3;
    if (make_tmap_3d_bf16(&map_pool, pool->base, pool->kv_dim, 16, (uint64_t)pool->num_blocks * pool->num_layers,
                          (uint64_t)pool->kv_dim * 2, (uint64_t)pool->kv_dim * 2 * 16, 64, 16, 1))
      return -2;
    if (make_tmap_2d_bf16(&map16, qkv, ld, n_total, ld * 2, 64, 16)) return -2;
    map_run = map;
  } else {
    map_pool = map;
    map16 = map;
    map_run = map;
  }
  static int runs_env = -1;  // PO_POOL_RUNS=0: every pool tile as per-block boxes (A/B)
  if (runs_env < 0) runs_env = (getenv("PO_POOL_RUNS") && getenv("PO_POOL_RUNS")[0] == '0') ? 0 : 1;
  const bool pool_runs = use_pool && runs_env &&
      make_tmap_4d_bf16(&map_run, pool->base, pool->kv_dim, 16, pool->num_layers, pool->num_blocks,
                        (uint64_t)pool->kv_dim * 2, (uint64_t)pool->kv_dim * 2 * 16,
                        (uint64_t)pool->kv_dim * 2 * 16 * pool->num_layers, 64, 16, 1, BKV / 16) == 0;
  ensure_smem_attr<attn_fwd_kernel>(SMEM_BYTES);
  AttnArgs a{};
  a.n_total = n_total;
  a.q_offset = q_offset;
  a.n_q = n_total - q_offset;
  a.hq = hq;
  a.hkv = hkv;
  a.mode = lay.mode;
  a.R = lay.R;
  a.G = lay.G;
  a.num_units = lay.units;
  a.pairs = lay.G % 2 ? 1 : lay.G / 2;
  a.num_qb = (a.n_q + BQ - 1) / BQ;
  a.out = static_cast<__nv_bfloat16*>(out);
  a.ldo = ldo;
  a.scale_log2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(HD)));
  {
    // K + V bytes of all kv heads: when they overflow ~1/3 of L2, band the CTA order by kv head
    static int force = -2;
    if (force == -2) force = getenv("PO_ATTN_KVBAND") ? atoi(getenv("PO_ATTN_KVBAND")) : -1;
    const double kv_all = (double)n_total * hkv * HD * 2 * 2;
    int band = 0;
    if (force >= 0) {
      band = force;
    } else if (kv_all > 40e6) {
      band = hkv;
      while (band > 1 && (double)n_total * band * HD * 2 * 2 > 40e6) band /= 2;
      while (band > 1 && hkv % band) --band;
    }
    a.kv_band = (lay.mode == MODE_HEADS && band > 0 && hkv % band == 0) ? band : 0;
  }
  if (use_pool) {
    a.pool_runs = pool_runs ? 1 : 0;
    a.n_pool = pool->n_rows;
    a.pool_slots = pool->slots;
    a.pool_layer = pool->layer;
    a.pool_layers = pool->num_layers;
    a.pool_kcol = 0;
    a.pool_vcol = hkv * HD;
  }
  attention_split_plan(n_total, q_offset, hq, hkv, &a.splits, &a.tiles_per_split);
  const size_t need = attention_workspace_bytes(n_total, q_offset, hq, hkv);
  if (a.splits > 1 && (!workspace || workspace_bytes < need)) {
    a.splits = 1;  // no workspace: fall back to the unsplit kernel (same kernel, full KV range per CTA)
    a.tiles_per_split = (n_total - 1) / BKV + 1;
  }
  if (a.splits > 1) {
    a.part_o = static_cast<__nv_bfloat16*>(workspace);
    a.part_ml = reinterpret_cast<float2*>(static_cast<char*>(workspace) +
                                          (size_t)a.splits * a.n_q * hq * HD * sizeof(__nv_bfloat16));
  }
  const int grid = lay.ctas * a.splits;
  launch_pdl(attn_fwd_kernel, dim3(grid), dim3(NTHREADS), SMEM_BYTES, stream, map, map_q, map_pool, map16, map_run,
             a);
  if (a.splits > 1) {
    const long long total = (long long)a.n_q * hq * (HD / 4);
    const int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 16);
    launch_pdl(attn_combine_kernel, dim3(blocks), dim3(256), 0, stream, (const __nv_bfloat16*)a.part_o,
               (const float2*)a.part_ml, a.n_q, hq, a.splits, a.tiles_per_split, q_offset, n_total, lay.span, a.out,
               ldo);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : -4;
}

}  // namespace po

#ifdef ATTN_SPAN
extern "C" int po_debug_attn_span(unsigned long long* host, int n) {
  if (n > 8192 * 4) n = 8192 * 4;
  return cudaMemcpyFromSymbol(host, po::g_attn_span, n * sizeof(unsigned long long)) == cudaSuccess ? 0 : -1;
}
#endif

#ifdef ATTN_TRACE
extern "C" int po_debug_attn_trace(unsigned long long* host, int n) {
  if (n > po::TRACE_EVENTS * po::TRACE_TILES) n = po::TRACE_EVENTS * po::TRACE_TILES;
  return cudaMemcpyFromSymbol(host, po::g_attn_trace, n * sizeof(unsigned long long)) == cudaSuccess ? 0 : -1;
}
#endif

extern "C" int po_op_attention(const void* qkv, int64_t ld, int32_t n_total, int32_t q_offset, int32_t n_heads,
                               int32_t n_kv_heads, void* out, int64_t ldo, void* stream) {
  if (!qkv || !out) return po::set_error(PO_ERR_ARG, "po_op_attention: null pointer");
  if (n_total <= 0 || q_offset < 0 || q_offset >= n_total)
    return po::set_error(PO_ERR_ARG, "po_op_attention: need 0 <= q_offset < n_total (got %d, %d)", q_offset, n_total);
  if (n_heads <= 0 || n_kv_heads <= 0 || n_heads % n_kv_heads)
    return po::set_error(PO_ERR_ARG, "po_op_attention: heads %d/%d must give an integer GQA group", n_heads,
                         n_kv_heads);
  if (ld < (int64_t)(n_heads + 2 * n_kv_heads) * 128 || ld % 8)
    return po::set_error(PO_ERR_ARG, "po_op_attention: ld %lld too small or unaligned", (long long)ld);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  po::keep_pool_memory();
  const size_t ws_bytes = po::attention_workspace_bytes(n_total, q_offset, n_heads, n_kv_heads);
  void* ws = nullptr;
  if (ws_bytes && cudaMallocAsync(&ws, ws_bytes, st) != cudaSuccess)
    return po::set_error(PO_ERR_CUDA, "po_op_attention: workspace allocation failed");
  int rc = po::attention_run(qkv, ld, n_total, q_offset, n_heads, n_kv_heads, out, ldo, st, ws, ws_bytes, nullptr);
  if (ws) cudaFreeAsync(ws, st);
  if (rc) return po::set_error(PO_ERR_CUDA, "po_op_attention: failed (%d): %s", rc,
                               cudaGetErrorString(cudaGetLastError()));
  return PO_OK;
}
