// Fused GEMM epilogues shared by the per-GEMM kernels (gemm.cu) and the persistent weight-streaming layer kernel
// (stream.cu): one thread owns one accumulator row (TMEM lane) and walks its columns 32 at a time.
#pragma once
#include "gemm.cuh"

namespace po {

// Split-K partial tiles added to the TMEM accumulator before the fused epilogue (stream.cu fix-up): partial j of this
// tile is p + j * stride, row-major [row][ld] fp32, rows < M written. Summed in j order after the TMEM value.
struct PartSrc {
  const float* p;
  int n;
  long long stride;
  int ld;
};

template <bool PART>
__device__ __forceinline__ void add_parts(const PartSrc& ps, int row, int c, uint32_t (&r)[32]) {
  if constexpr (PART) {
    for (int j = 0; j < ps.n; ++j) {
      const float4* src = reinterpret_cast<const float4*>(ps.p + j * ps.stride + (long long)row * ps.ld + c);
      float4 v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = __ldcg(src + q);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        r[4 * q + 0] = __float_as_uint(__uint_as_float(r[4 * q + 0]) + v[q].x);
        r[4 * q + 1] = __float_as_uint(__uint_as_float(r[4 * q + 1]) + v[q].y);
        r[4 * q + 2] = __float_as_uint(__uint_as_float(r[4 * q + 2]) + v[q].z);
        r[4 * q + 3] = __float_as_uint(__uint_as_float(r[4 * q + 3]) + v[q].w);
      }
    }
  }
}

// silu(g) = g / (1 + e^-g) with the fast division (MUFU reciprocal, no IEEE slow-path branch per element, so the
// epilogues interleave elements); for g < -87 the denominator overflows and the result is the limit -0.
__device__ __forceinline__ float silu_f(float g) { return __fdividef(g, 1.0f + __expf(-g)); }

// 1/rms of output row `row` from the producer's per-segment sums of squares (fixed summation order; the loads go
// out 8 at a time so their latency is paid once per 8 segments, not once per segment)
__device__ __forceinline__ float row_inv_rms(const GemmArgs& a, int row) {
  const float* p = a.ss_in + (long long)row * a.ss_nseg;
  float s = 0.f;
  for (int i0 = 0; i0 < a.ss_nseg; i0 += 8) {
    float x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = i0 + i < a.ss_nseg ? __ldcg(p + i0 + i) : 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (i0 + i < a.ss_nseg) s += x[i];
  }
  return rsqrtf(s / a.norm_dim + a.norm_eps);
}

// Prefix-pool row (offset so that column index col addresses it) of output row `row` when its block is admitted
// and the column block [hcol, hcol + 128) holds K or V; null otherwise (see GemmArgs::kv_slot).
__device__ __forceinline__ __nv_bfloat16* pool_row(const GemmArgs& a, int row, int hcol) {
  if (!a.kv_pool || hcol < a.kv_col0) return nullptr;
  const int pos = a.pos_offset + row;
  const int slot = a.kv_slot[pos >> 4];
  if (slot < 0) return nullptr;
  return a.kv_pool + (((long long)slot * a.pool_layers + a.pool_layer) * 16 + (pos & 15)) * a.kv_dim - a.kv_col0;
}
__device__ __forceinline__ void store_bf16_32(__nv_bfloat16* dst, const uint32_t (&r)[32]) {
  uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int q = 0; q < 4; ++q)
    d[q] = make_uint4(pack_bf16(__uint_as_float(r[8 * q + 0]), __uint_as_float(r[8 * q + 1])),
                      pack_bf16(__uint_as_float(r[8 * q + 2]), __uint_as_float(r[8 * q + 3])),
                      pack_bf16(__uint_as_float(r[8 * q + 4]), __uint_as_float(r[8 * q + 5])),
                      pack_bf16(__uint_as_float(r[8 * q + 6]), __uint_as_float(r[8 * q + 7])));
}

template <int EPI>
__device__ __forceinline__ float epilogue_chunk(const GemmArgs& a, int row, int col0, const uint32_t (&r)[32],
                                                float sc = 1.0f) {
  float sq = 0.f;
  if constexpr (EPI == EPI_BF16) {
    uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(a.out) + (long long)row * a.ldo + col0);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 v;
      v.x = pack_bf16(__uint_as_float(r[8 * q + 0]), __uint_as_float(r[8 * q + 1]));
      v.y = pack_bf16(__uint_as_float(r[8 * q + 2]), __uint_as_float(r[8 * q + 3]));
      v.z = pack_bf16(__uint_as_float(r[8 * q + 4]), __uint_as_float(r[8 * q + 5]));
      v.w = pack_bf16(__uint_as_float(r[8 * q + 6]), __uint_as_float(r[8 * q + 7]));
      dst[q] = v;
    }
  } else if constexpr (EPI == EPI_F32) {
    float4* dst = reinterpret_cast<float4*>(static_cast<float*>(a.out) + (long long)row * a.ldo + col0);
#pragma unroll
    for (int q = 0; q < 8; ++q)
      dst[q] = make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]), __uint_as_float(r[4 * q + 2]),
                           __uint_as_float(r[4 * q + 3]));
  } else if constexpr (EPI == EPI_RESID_F32) {
    float4* dst = reinterpret_cast<float4*>(a.resid + (long long)row * a.ldr + col0);
    float4 v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = __ldcg(dst + q);  // all loads in flight first (L2: another CTA may own it)
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      v[q].x += __uint_as_float(r[4 * q + 0]);
      v[q].y += __uint_as_float(r[4 * q + 1]);
      v[q].z += __uint_as_float(r[4 * q + 2]);
      v[q].w += __uint_as_float(r[4 * q + 3]);
      dst[q] = v[q];
    }
    if (a.xg_out) {
      const float4* g4 = reinterpret_cast<const float4*>(a.g_next + col0);
      uint4* xo = reinterpret_cast<uint4*>(a.xg_out + (long long)row * a.ldxg + col0);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float4 ga = g4[2 * q], gb = g4[2 * q + 1];
        const float4 va = v[2 * q], vb = v[2 * q + 1];
        xo[q] = make_uint4(pack_bf16(va.x * ga.x, va.y * ga.y), pack_bf16(va.z * ga.z, va.w * ga.w),
                           pack_bf16(vb.x * gb.x, vb.y * gb.y), pack_bf16(vb.z * gb.z, vb.w * gb.w));
        sq += va.x * va.x + va.y * va.y + va.z * va.z + va.w * va.w + vb.x * vb.x + vb.y * vb.y + vb.z * vb.z +
              vb.w * vb.w;
      }
    }
  } else if constexpr (EPI == EPI_SILU_MUL) {
    // 32 accumulator columns = 16 gate columns followed by the matching 16 up columns; sc = this row's 1/rms
    uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(a.out) + (long long)row * a.ldo + col0 / 2);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      uint32_t w[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int j = 8 * q + 2 * e;
        const float x0 = silu_f(sc * __uint_as_float(r[j])) * (sc * __uint_as_float(r[16 + j]));
        const float x1 = silu_f(sc * __uint_as_float(r[j + 1])) * (sc * __uint_as_float(r[16 + j + 1]));
        w[e] = pack_bf16(x0, x1);
      }
      dst[q] = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
  return sq;
}

// FP8: dequantise 32 accumulator columns [col0, col0 + 32) of this row: acc * a_scale[row] * b_scale[col]
template <bool F8>
__device__ __forceinline__ void dequant32(const GemmArgs& a, float as, int col0, uint32_t (&r)[32]) {
  if constexpr (F8) {
    const float4* b4 = reinterpret_cast<const float4*>(a.b_scale + col0);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float4 b = __ldg(b4 + q);
      r[4 * q + 0] = __float_as_uint(__uint_as_float(r[4 * q + 0]) * as * b.x);
      r[4 * q + 1] = __float_as_uint(__uint_as_float(r[4 * q + 1]) * as * b.y);
      r[4 * q + 2] = __float_as_uint(__uint_as_float(r[4 * q + 2]) * as * b.z);
      r[4 * q + 3] = __float_as_uint(__uint_as_float(r[4 * q + 3]) * as * b.w);
    }
  }
}

// Epilogue of one 128-row x 256-column accumulator (this thread: TMEM lane = output row `row`).
// Columns [c_lo, c_hi) of the tile (a multiple of 128 wide and 128-aligned when the work is shared between several
// warps of one TMEM lane quadrant): the default is the whole tile.
template <int EPI, int BNT = 256, bool F8 = false, bool PART = false>
__device__ __forceinline__ void epilogue_tile(const GemmArgs& args, uint32_t taddr, int row, int nb, int ksp, int t,
                                              const PartSrc& ps = PartSrc{}, int c_lo = 0, int c_hi = BNT) {
  const bool prow = PART && row < args.M;  // partial tiles hold rows < M only
  const float as = (F8 && row < args.M) ? args.a_scale[row] : 0.f;
  if (ksp > 1) {
    // split-K partial: raw fp32 tile into the workspace slice of this split
    GemmArgs pa = args;
    pa.out = args.split_ws + (size_t)(t % ksp) * args.M * args.N;
    pa.ldo = args.N;
#pragma unroll 1
    for (int c = c_lo; c < c_hi; c += 32) {
      uint32_t r[32];
      tmem_ld32(taddr + c, r);
      tmem_ld_wait();
      if (row < args.M) epilogue_chunk<EPI_F32>(pa, row, nb * BNT + c, r);
    }
  } else if constexpr (EPI == EPI_QKV_ROPE) {
    // two 128-column heads per tile; rotate-half pairs (i, i+64)
    const float sc = (args.ss_in && row < args.M) ? row_inv_rms(args, row) : 1.0f;
#pragma unroll 1
    for (int h = c_lo / 128; h < c_hi / 128; ++h) {
      const int hcol = nb * BNT + h * 128;
      const bool rot = hcol < args.rope_cols;
      const float2* cs = args.rope + (long long)(args.pos_offset + row) * 64;
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {
        uint32_t x1[32], x2[32];
        tmem_ld32(taddr + h * 128 + half * 32, x1);
        tmem_ld32(taddr + h * 128 + 64 + half * 32, x2);
        tmem_ld_wait();
        dequant32<F8>(args, as, hcol + half * 32, x1);
        dequant32<F8>(args, as, hcol + 64 + half * 32, x2);
        if (prow) {
          add_parts<PART>(ps, row, h * 128 + half * 32, x1);
          add_parts<PART>(ps, row, h * 128 + 64 + half * 32, x2);
        }
        if (args.ss_in) {
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            x1[i] = __float_as_uint(sc * __uint_as_float(x1[i]));
            x2[i] = __float_as_uint(sc * __uint_as_float(x2[i]));
          }
        }
        if (args.bias) {
          const float* b1 = args.bias + hcol + half * 32;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            x1[i] = __float_as_uint(__uint_as_float(x1[i]) + b1[i]);
            x2[i] = __float_as_uint(__uint_as_float(x2[i]) + b1[64 + i]);
          }
        }
        if (row < args.M) {
          if (rot) {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const float2 c = cs[half * 32 + i];
              const float a0 = __uint_as_float(x1[i]);
              const float b0 = __uint_as_float(x2[i]);
              x1[i] = __float_as_uint(a0 * c.x - b0 * c.y);
              x2[i] = __float_as_uint(b0 * c.x + a0 * c.y);
            }
          }
          epilogue_chunk<EPI_BF16>(args, row, hcol + half * 32, x1);
          epilogue_chunk<EPI_BF16>(args, row, hcol + 64 + half * 32, x2);
          if (__nv_bfloat16* prow = pool_row(args, row, hcol)) {
            store_bf16_32(prow + hcol + half * 32, x1);
            store_bf16_32(prow + hcol + 64 + half * 32, x2);
          }
        }
      }
    }
  } else if constexpr (EPI == EPI_RESID_F32) {
    float sq[2] = {0.f, 0.f};
#pragma unroll 1
    for (int c = c_lo; c < c_hi; c += 32) {
      uint32_t r[32];
      tmem_ld32(taddr + c, r);
      tmem_ld_wait();
      dequant32<F8>(args, as, nb * BNT + c, r);
      if (prow) add_parts<PART>(ps, row, c, r);
      if (row < args.M) sq[c >> 7] += epilogue_chunk<EPI>(args, row, nb * BNT + c, r);
    }
    if (args.ss_out && row < args.M) {
      for (int k = c_lo / 128; k < c_hi / 128; ++k)
        args.ss_out[(long long)row * args.ss_nseg + nb * (BNT / 128) + k] = sq[k];
    }
  } else {
    const float sc = (EPI == EPI_SILU_MUL && args.ss_in && row < args.M) ? row_inv_rms(args, row) : 1.0f;
#pragma unroll 1
    for (int c = c_lo; c < c_hi; c += 32) {
      uint32_t r[32];
      tmem_ld32(taddr + c, r);
      tmem_ld_wait();
      dequant32<F8>(args, as, nb * BNT + c, r);
      if (prow) add_parts<PART>(ps, row, c, r);
      if (row < args.M) epilogue_chunk<EPI>(args, row, nb * BNT + c, r, sc);
    }
  }
}


// Sum of the k-split partials at p, p + slice, ... in split order; the loads of each group of four issued before its
// adds. Group width 4 and pointer increments (not 8 predicated slots with 64-bit index products): the reduce launches
// of short-M GEMMs are issue-bound, and 3-6 splits are the usual counts.
__device__ __forceinline__ float4 split_sum(const float* p, size_t slice, int splits) {
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  const float4* q = reinterpret_cast<const float4*>(p);
  const size_t step = slice / 4;  // slice is a multiple of 4 floats (N % 4 == 0)
  for (int s0 = 0; s0 < splits; s0 += 4) {
    float4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v[k] = s0 + k < splits ? __ldcg(q) : make_float4(0.f, 0.f, 0.f, 0.f);
      q += step;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (s0 + k < splits) {
        acc.x += v[k].x; acc.y += v[k].y; acc.z += v[k].z; acc.w += v[k].w;
      }
    }
  }
  return acc;
}

// FP8 split-K: dequantise a summed 4-column group (same order as dequant32: (acc * a_scale) * b_scale)
__device__ __forceinline__ void dq4(const GemmArgs& a, int row, int col, float4& v) {
  if (!a.b_scale) return;
  const float as = a.a_scale[row];
  const float4 b = *reinterpret_cast<const float4*>(a.b_scale + col);
  v.x = v.x * as * b.x;
  v.y = v.y * as * b.y;
  v.z = v.z * as * b.z;
  v.w = v.w * as * b.w;
}

// One split-K output quad: sum the k-split partials of (row, col..col+3) at p, p + slice, ... in split order, then
// apply the fused epilogue (gate/up pairs at col + 16, RoPE pairs at col + 64 in the same partial row). Used by
// splitk_reduce_kernel (gemm.cu) and the streaming kernel's cooperative fix-up (stream.cu).
template <int EPI>
__device__ __forceinline__ void splitk_reduce_quad(const GemmArgs& a, int row, int col, const float* p, size_t slice,
                                                   int splits, float sc_pre = -1.f) {
  float4 acc = split_sum(p, slice, splits);
  dq4(a, row, col, acc);
  float sc = 1.0f;
  if constexpr (EPI == EPI_SILU_MUL || EPI == EPI_QKV_ROPE) {
    if (a.ss_in) sc = sc_pre >= 0.f ? sc_pre : row_inv_rms(a, row);
    acc.x *= sc; acc.y *= sc; acc.z *= sc; acc.w *= sc;
  }
  if constexpr (EPI == EPI_BF16) {
    *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(a.out) + (long long)row * a.ldo + col) =
        make_uint2(pack_bf16(acc.x, acc.y), pack_bf16(acc.z, acc.w));
  } else if constexpr (EPI == EPI_F32) {
    *reinterpret_cast<float4*>(static_cast<float*>(a.out) + (long long)row * a.ldo + col) = acc;
  } else if constexpr (EPI == EPI_RESID_F32) {
    float4* d = reinterpret_cast<float4*>(a.resid + (long long)row * a.ldr + col);
    float4 v = __ldcg(d);
    v.x += acc.x; v.y += acc.y; v.z += acc.z; v.w += acc.w;
    *d = v;
    if (a.xg_out) {
      // N % 128 == 0: each warp covers one 128-column segment of one row (warps stay converged)
      const float4 g = *reinterpret_cast<const float4*>(a.g_next + col);
      *reinterpret_cast<uint2*>(a.xg_out + (long long)row * a.ldxg + col) =
          make_uint2(pack_bf16(v.x * g.x, v.y * g.y), pack_bf16(v.z * g.z, v.w * g.w));
      float sq = v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
#pragma unroll
      for (int o = 16; o; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
      if ((threadIdx.x & 31) == 0) a.ss_out[(long long)row * a.ss_nseg + col / 128] = sq;
    }
  } else if constexpr (EPI == EPI_SILU_MUL) {
    // 16-column groups: [gate 16 | up 16]; this thread's 4 columns are gate or up of output cols
    const int grp = col / 32, w = col % 32;
    if (w < 16) {
      float4 up = split_sum(p + 16, slice, splits);
      dq4(a, row, col + 16, up);
      up.x *= sc; up.y *= sc; up.z *= sc; up.w *= sc;
      const int oc = grp * 16 + w;
      *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(a.out) + (long long)row * a.ldo + oc) =
          make_uint2(pack_bf16(silu_f(acc.x) * up.x, silu_f(acc.y) * up.y),
                     pack_bf16(silu_f(acc.z) * up.z, silu_f(acc.w) * up.w));
    }
  } else if constexpr (EPI == EPI_QKV_ROPE) {
    const int head_col = col % 128;
    if (a.bias) {
      acc.x += a.bias[col]; acc.y += a.bias[col + 1]; acc.z += a.bias[col + 2]; acc.w += a.bias[col + 3];
    }
    if (col < a.rope_cols && head_col < 64) {
      float4 x2 = split_sum(p + 64, slice, splits);
      dq4(a, row, col + 64, x2);
      x2.x *= sc; x2.y *= sc; x2.z *= sc; x2.w *= sc;
      if (a.bias) {
        x2.x += a.bias[col + 64]; x2.y += a.bias[col + 65]; x2.z += a.bias[col + 66]; x2.w += a.bias[col + 67];
      }
      const float2* cs = a.rope + (long long)(a.pos_offset + row) * 64 + head_col;
      const float4 x1 = acc;
      const float2 c0 = cs[0], c1 = cs[1], c2 = cs[2], c3 = cs[3];
      __nv_bfloat16* o = static_cast<__nv_bfloat16*>(a.out) + (long long)row * a.ldo + col;
      const uint2 lo = make_uint2(pack_bf16(x1.x * c0.x - x2.x * c0.y, x1.y * c1.x - x2.y * c1.y),
                                  pack_bf16(x1.z * c2.x - x2.z * c2.y, x1.w * c3.x - x2.w * c3.y));
      const uint2 hi = make_uint2(pack_bf16(x2.x * c0.x + x1.x * c0.y, x2.y * c1.x + x1.y * c1.y),
                                  pack_bf16(x2.z * c2.x + x1.z * c2.y, x2.w * c3.x + x1.w * c3.y));
      *reinterpret_cast<uint2*>(o) = lo;
      *reinterpret_cast<uint2*>(o + 64) = hi;
      if (__nv_bfloat16* prow = pool_row(a, row, col - head_col)) {
        *reinterpret_cast<uint2*>(prow + col) = lo;
        *reinterpret_cast<uint2*>(prow + col + 64) = hi;
      }
    } else if (col >= a.rope_cols) {
      const uint2 v = make_uint2(pack_bf16(acc.x, acc.y), pack_bf16(acc.z, acc.w));
      *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(a.out) + (long long)row * a.ldo + col) = v;
      if (__nv_bfloat16* prow = pool_row(a, row, col - head_col)) *reinterpret_cast<uint2*>(prow + col) = v;
    }
  }
}

// ---- cross-CTA flags (stream-K fix-ups): relaxed poll, release store, generic <-> async proxy ordering
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// generic-proxy writes of other CTAs (epilogue stores) -> this CTA's async-proxy reads (TMA), and the reverse
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// Fused epilogue of one 4-column group of a fixed-up (summed) row: acc = columns col..col+3; part = the partner group
// (gate -> up at col + 16; RoPE x1 -> x2 at col + 64); sc = the row's 1/rms (folded RMSNorm consumers); rv = the
// residual row's values (EPI_RESID_F32). Same arithmetic order as epilogue_tile / splitk_reduce_quad.
template <int EPI>
__device__ __forceinline__ void quad_epi(const GemmArgs& a, int row, int col, float4 acc, float4 part, float sc,
                                         float4 rv) {
  if constexpr (EPI == EPI_BF16) {
    *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(a.out) + (long long)row * a.ldo + col) =
        make_uint2(pack_bf16(acc.x, acc.y), pack_bf16(acc.z, acc.w));
  } else if constexpr (EPI == EPI_RESID_F32) {
    rv.x += acc.x; rv.y += acc.y; rv.z += acc.z; rv.w += acc.w;
    *reinterpret_cast<float4*>(a.resid + (long long)row * a.ldr + col) = rv;
    if (a.xg_out) {
      const float4 gm = *reinterpret_cast<const float4*>(a.g_next + col);
      *reinterpret_cast<uint2*>(a.xg_out + (long long)row * a.ldxg + col) =
          make_uint2(pack_bf16(rv.x * gm.x, rv.y * gm.y), pack_bf16(rv.z * gm.z, rv.w * gm.w));
      float sq = rv.x * rv.x + rv.y * rv.y + rv.z * rv.z + rv.w * rv.w;
#pragma unroll
      for (int o = 16; o; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
      if ((threadIdx.x & 31) == 0) a.ss_out[(long long)row * a.ss_nseg + col / 128] = sq;
    }
  } else if constexpr (EPI == EPI_SILU_MUL) {
    const int oc = (col / 32) * 16 + (col % 32);
    *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(a.out) + (long long)row * a.ldo + oc) =
        make_uint2(pack_bf16(silu_f(sc * acc.x) * (sc * part.x), silu_f(sc * acc.y) * (sc * part.y)),
                   pack_bf16(silu_f(sc * acc.z) * (sc * part.z), silu_f(sc * acc.w) * (sc * part.w)));
  } else if constexpr (EPI == EPI_QKV_ROPE) {
    const int head_col = col % 128;
    acc.x *= sc; acc.y *= sc; acc.z *= sc; acc.w *= sc;
    if (a.bias) {
      acc.x += a.bias[col]; acc.y += a.bias[col + 1]; acc.z += a.bias[col + 2]; acc.w += a.bias[col + 3];
    }
    __nv_bfloat16* o = static_cast<__nv_bfloat16*>(a.out) + (long long)row * a.ldo + col;
    if (col < a.rope_cols) {
      float4 x2 = part;
      x2.x *= sc; x2.y *= sc; x2.z *= sc; x2.w *= sc;
      if (a.bias) {
        x2.x += a.bias[col + 64]; x2.y += a.bias[col + 65]; x2.z += a.bias[col + 66]; x2.w += a.bias[col + 67];
      }
      const float2* cs = a.rope + (long long)(a.pos_offset + row) * 64 + head_col;
      const float2 c0 = cs[0], c1 = cs[1], c2 = cs[2], c3 = cs[3];
      const uint2 lo = make_uint2(pack_bf16(acc.x * c0.x - x2.x * c0.y, acc.y * c1.x - x2.y * c1.y),
                                  pack_bf16(acc.z * c2.x - x2.z * c2.y, acc.w * c3.x - x2.w * c3.y));
      const uint2 hi = make_uint2(pack_bf16(x2.x * c0.x + acc.x * c0.y, x2.y * c1.x + acc.y * c1.y),
                                  pack_bf16(x2.z * c2.x + acc.z * c2.y, x2.w * c3.x + acc.w * c3.y));
      *reinterpret_cast<uint2*>(o) = lo;
      *reinterpret_cast<uint2*>(o + 64) = hi;
      if (__nv_bfloat16* prow = pool_row(a, row, col - head_col)) {
        *reinterpret_cast<uint2*>(prow + col) = lo;
        *reinterpret_cast<uint2*>(prow + col + 64) = hi;
      }
    } else {
      const uint2 v = make_uint2(pack_bf16(acc.x, acc.y), pack_bf16(acc.z, acc.w));
      *reinterpret_cast<uint2*>(o) = v;
      if (__nv_bfloat16* prow = pool_row(a, row, col - head_col)) *reinterpret_cast<uint2*>(prow + col) = v;
    }
  }
}

}  // namespace po
