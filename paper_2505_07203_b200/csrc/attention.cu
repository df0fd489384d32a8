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
#include "../../include/prefillonly.h"
#include <cmath>

namespace po {
int set_error(int code, const char* fmt, ...);
int make_tmap_2d_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t row_stride_bytes,
                      uint32_t box_inner, uint32_t box_outer);

namespace {
constexpr int HD = 128;
constexpr int BQ = 128;
constexpr int BKV = 128;
constexpr int BOX_BYTES = 128 * 64 * 2;        // one 128-row x 64-col swizzled box (16 KB)
constexpr int TILE_BYTES = 2 * BOX_BYTES;      // 128 x 128 bf16
constexpr int NTHREADS = 384;
constexpr int SMEM_BYTES = 6 * TILE_BYTES + 1024 + 256;
constexpr float RESCALE_THRESHOLD = 8.0f;      // log2 units
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
};

// One 128-key tile of online softmax for this thread's query row (TMEM lane): reads S, writes P (bf16,
// packed over the first 64 columns of S), keeps (m, l). `lim` = number of visible keys in the tile
// (keys kbase + c with c < lim); only the MASKED instantiation tests it.
template <bool MASKED>
__device__ __forceinline__ void softmax_tile(uint32_t s_addr, uint32_t o_addr, int lim, float sl2, int j, float& m,
                                             float& l) {
  float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
  for (int c = 0; c < 4; c += 2) {
    uint32_t v0[32], v1[32];
    tmem_ld32(s_addr + c * 32, v0);
    tmem_ld32(s_addr + (c + 1) * 32, v1);
    tmem_ld_wait();
#pragma unroll
    for (int e = 0; e < 32; e += 2) {
      float a0 = __uint_as_float(v0[e]), a1 = __uint_as_float(v0[e + 1]);
      float b0 = __uint_as_float(v1[e]), b1 = __uint_as_float(v1[e + 1]);
      if (MASKED) {
        if (c * 32 + e >= lim) a0 = -INFINITY;
        if (c * 32 + e + 1 >= lim) a1 = -INFINITY;
        if ((c + 1) * 32 + e >= lim) b0 = -INFINITY;
        if ((c + 1) * 32 + e + 1 >= lim) b1 = -INFINITY;
      }
      mx0 = fmaxf(mx0, fmaxf(a0, a1));
      mx1 = fmaxf(mx1, fmaxf(b0, b1));
    }
  }
  const float m_new = fmaxf(m, fmaxf(mx0, mx1) * sl2);
  const bool resc = m_new > m + RESCALE_THRESHOLD;
  const float alpha = resc ? ex2_approx(m - m_new) : 1.0f;
  if (j > 0 && __any_sync(0xffffffffu, resc)) {
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
      uint32_t v[32];
      tmem_ld32(o_addr + c * 32, v);
      tmem_ld_wait();
#pragma unroll
      for (int e = 0; e < 32; ++e) v[e] = __float_as_uint(__uint_as_float(v[e]) * alpha);
      tmem_st32(o_addr + c * 32, v);
    }
    tmem_st_wait();
  }
  if (resc) {
    l *= alpha;
    m = m_new;
  }
  const float nm = -m;
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
  for (int c = 0; c < 4; c += 2) {
    uint32_t v0[32], v1[32];
    tmem_ld32(s_addr + c * 32, v0);
    tmem_ld32(s_addr + (c + 1) * 32, v1);
    tmem_ld_wait();
    uint32_t p0[16], p1[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      float x0 = ex2_approx(fmaf(__uint_as_float(v0[2 * e]), sl2, nm));
      float x1 = ex2_approx(fmaf(__uint_as_float(v0[2 * e + 1]), sl2, nm));
      float y0 = ex2_approx(fmaf(__uint_as_float(v1[2 * e]), sl2, nm));
      float y1 = ex2_approx(fmaf(__uint_as_float(v1[2 * e + 1]), sl2, nm));
      if (MASKED) {
        if (c * 32 + 2 * e >= lim) x0 = 0.f;
        if (c * 32 + 2 * e + 1 >= lim) x1 = 0.f;
        if ((c + 1) * 32 + 2 * e >= lim) y0 = 0.f;
        if ((c + 1) * 32 + 2 * e + 1 >= lim) y1 = 0.f;
      }
      s0 += x0;
      s1 += x1;
      s2 += y0;
      s3 += y1;
      p0[e] = pack_bf16(x0, x1);
      p1[e] = pack_bf16(y0, y1);
    }
    // P columns [16c, 16c+32) lie inside S chunks already consumed (c/2 <= c)
    tmem_st16(s_addr + c * 16, p0);
    tmem_st16(s_addr + (c + 1) * 16, p1);
  }
  l += (s0 + s1) + (s2 + s3);
}

__global__ void __launch_bounds__(NTHREADS, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap map, const AttnArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                       // 2 tiles
  uint8_t* sK = smem + 2 * TILE_BYTES;      // 2 stages
  uint8_t* sV = smem + 4 * TILE_BYTES;      // 2 stages
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 6 * TILE_BYTES);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;    // [2]
  uint64_t* v_full = bars + 3;    // [2]
  uint64_t* kv_empty = bars + 5;  // [2]
  uint64_t* s_full = bars + 7;    // [2] per head slot
  uint64_t* p_full = bars + 9;    // [2]
  uint64_t* o_final = bars + 11;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 13);

  const int warp = warp_id();
  const int lane = lane_id();

  // heaviest (longest causal extent) query blocks first
  const int per_qb = a.hkv * a.pairs;
  const int qb = a.num_qb - 1 - blockIdx.x / per_qb;
  const int rem = blockIdx.x % per_qb;
  const int g = rem / a.pairs;
  const int h0 = g * (2 * a.pairs) + 2 * (rem % a.pairs);
  const int q_lo = a.q_offset + qb * BQ;                    // position of query row 0 of this block
  const int q_hi = min(q_lo + BQ - 1, a.n_total - 1);       // last real query position
  const int n_tiles = q_hi / BKV + 1;

  if (warp == 8 && lane == 0) {
    tma_prefetch_desc(&map);
    for (int i = 0; i < 13; ++i) mbar_init(&bars[i], (i == 9 || i == 10) ? 128 : 1);
    fence_barrier_init();
  }
  if (warp == 10) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 8) {
    if (lane == 0) {
      const uint64_t keep = l2_policy_evict_last();
      mbar_arrive_expect_tx(q_full, 2 * TILE_BYTES);
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int half = 0; half < 2; ++half)
          tma_load_2d(sQ + i * TILE_BYTES + half * BOX_BYTES, &map, q_full, (h0 + i) * HD + half * 64, q_lo);
      const int kcol = a.hq * HD + g * HD;
      const int vcol = (a.hq + a.hkv) * HD + g * HD;
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        mbar_wait(&kv_empty[st], ph ^ 1);
        mbar_arrive_expect_tx(&k_full[st], TILE_BYTES);
        tma_load_2d_hint(sK + st * TILE_BYTES, &map, &k_full[st], kcol, j * BKV, keep);
        tma_load_2d_hint(sK + st * TILE_BYTES + BOX_BYTES, &map, &k_full[st], kcol + 64, j * BKV, keep);
        mbar_arrive_expect_tx(&v_full[st], TILE_BYTES);
        tma_load_2d_hint(sV + st * TILE_BYTES, &map, &v_full[st], vcol, j * BKV, keep);
        tma_load_2d_hint(sV + st * TILE_BYTES + BOX_BYTES, &map, &v_full[st], vcol + 64, j * BKV, keep);
      }
    }
    __syncwarp();
  } else if (warp == 9) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = idesc_bf16_f32(128, 128, false, false);
      constexpr uint32_t idesc_o = idesc_bf16_f32(128, 128, false, true);
      auto issue_s = [&](int i, int st) {
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * BOX_BYTES + (kk & 3) * 32;
          mma_bf16_ss(tmem + i * 128, sdesc_kmajor_sw128(smem_u32(sQ + i * TILE_BYTES + off)),
                      sdesc_kmajor_sw128(smem_u32(sK + st * TILE_BYTES + off)), idesc_s, kk > 0);
        }
        mma_commit(&s_full[i]);
      };
      auto issue_pv = [&](int i, int st, bool acc) {
#pragma unroll
        for (int kk = 0; kk < BKV / 16; ++kk) {
          const uint64_t vdesc = sdesc_mnmajor_sw128(smem_u32(sV + st * TILE_BYTES + kk * 16 * 128), BOX_BYTES, 1024);
          mma_bf16_ts(tmem + 256 + i * 128, tmem + i * 128 + kk * 8, vdesc, idesc_o, (acc || kk > 0) ? 1u : 0u);
        }
      };
      mbar_wait(q_full, 0);
      mbar_wait(&k_full[0], 0);
      tc_fence_after();
      issue_s(0, 0);
      issue_s(1, 0);
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        const bool more = j + 1 < n_tiles;
        const int st2 = (j + 1) & 1;
        const uint32_t ph2 = ((j + 1) >> 1) & 1;
        mbar_wait(&v_full[st], ph);
        mbar_wait(&p_full[0], j & 1);
        tc_fence_after();
        issue_pv(0, st, j > 0);
        if (!more) mma_commit(&o_final[0]);
        if (more) {
          mbar_wait(&k_full[st2], ph2);
          tc_fence_after();
          issue_s(0, st2);
        }
        mbar_wait(&p_full[1], j & 1);
        tc_fence_after();
        issue_pv(1, st, j > 0);
        mma_commit(&kv_empty[st]);
        if (!more) mma_commit(&o_final[1]);
        if (more) issue_s(1, st2);
      }
    }
    __syncwarp();
  } else if (warp < 8) {
    const int i = warp >> 2;
    const int r = (warp & 3) * 32 + lane;
    const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t s_addr = tmem + lane_base + i * 128;
    const uint32_t o_addr = tmem + lane_base + 256 + i * 128;
    const int pos = q_lo + r;
    float m = -INFINITY;  // running max (scaled, log2 units), possibly stale
    float l = 0.f;
    for (int j = 0; j < n_tiles; ++j) {
      mbar_wait(&s_full[i], j & 1);
      tc_fence_after();
      const int kbase = j * BKV;
      // warp-uniform: only tiles crossing the diagonal of this query block pay for the mask
      if (kbase + BKV - 1 > q_lo) {
        softmax_tile<true>(s_addr, o_addr, pos - kbase + 1, a.scale_log2, j, m, l);
      } else {
        softmax_tile<false>(s_addr, o_addr, BKV, a.scale_log2, j, m, l);
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&p_full[i]);
    }
    mbar_wait(&o_final[i], 0);
    tc_fence_after();
    const float inv = 1.0f / l;
    const int row = qb * BQ + r;
    __nv_bfloat16* dst = a.out + (long long)row * a.ldo + (h0 + i) * HD;
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
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 10) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

struct AttnPlan {
  CUtensorMap map;
};

int attention_run(const void* qkv, long long ld, int n_total, int q_offset, int hq, int hkv, void* out, long long ldo,
                  cudaStream_t stream) {
  if (hq % hkv || (hq / hkv) % 2) return -3;
  AttnPlan plan;
  if (make_tmap_2d_bf16(&plan.map, qkv, ld, n_total, ld * 2, 64, 128)) return -2;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(attn_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    configured = true;
  }
  AttnArgs a;
  a.n_total = n_total;
  a.q_offset = q_offset;
  a.n_q = n_total - q_offset;
  a.hq = hq;
  a.hkv = hkv;
  a.pairs = hq / hkv / 2;
  a.num_qb = (a.n_q + BQ - 1) / BQ;
  a.out = static_cast<__nv_bfloat16*>(out);
  a.ldo = ldo;
  a.scale_log2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(HD)));
  const int grid = a.num_qb * hkv * a.pairs;
  attn_fwd_kernel<<<grid, NTHREADS, SMEM_BYTES, stream>>>(plan.map, a);
  return cudaGetLastError() == cudaSuccess ? 0 : -4;
}

}  // namespace po

extern "C" int po_op_attention(const void* qkv, int64_t ld, int32_t n_total, int32_t q_offset, int32_t n_heads,
                               int32_t n_kv_heads, void* out, int64_t ldo, void* stream) {
  if (!qkv || !out) return po::set_error(PO_ERR_ARG, "po_op_attention: null pointer");
  if (n_total <= 0 || q_offset < 0 || q_offset >= n_total)
    return po::set_error(PO_ERR_ARG, "po_op_attention: need 0 <= q_offset < n_total (got %d, %d)", q_offset, n_total);
  if (n_heads <= 0 || n_kv_heads <= 0 || n_heads % n_kv_heads || (n_heads / n_kv_heads) % 2)
    return po::set_error(PO_ERR_ARG, "po_op_attention: heads %d/%d must give an even GQA group", n_heads, n_kv_heads);
  if (ld < (int64_t)(n_heads + 2 * n_kv_heads) * 128 || ld % 8)
    return po::set_error(PO_ERR_ARG, "po_op_attention: ld %lld too small or unaligned", (long long)ld);
  int rc = po::attention_run(qkv, ld, n_total, q_offset, n_heads, n_kv_heads, out, ldo,
                             static_cast<cudaStream_t>(stream));
  if (rc) return po::set_error(PO_ERR_CUDA, "po_op_attention: failed (%d): %s", rc,
                               cudaGetErrorString(cudaGetLastError()));
  return PO_OK;
}
