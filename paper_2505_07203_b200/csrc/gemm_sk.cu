// Stream-K swap-AB pair GEMM for short launches (M <= 256 rows: prefix-hit suffixes, short requests, the last
// layer's final row). D[M,N] = X[M,K] . W[N,K]^T with the weight as the MMA's M operand (256 weight rows per pair
// tile, 128 per CTA) and the M activation rows as its N operand (NP = M rounded up to 16), as in gemm_swap.cu.
//
// Such a launch is a weight stream: its time is the weight bytes over the HBM rate the busy SMs can pull
// (tools/probe/stream_bw.cu: ~96 KB in flight per SM needs >= 128 SMs for 6 TB/s). The per-GEMM swap kernel hands
// whole (tile, k split) units to the pairs, so at M = 160 a Llama-3.1-8B gate/up (112 tiles) runs two rounds on 74
// pairs with the second one half empty, and the split GEMMs pay a reduce launch each (8-13 us). Here the T x nk
// (tile, k-block) work items are cut into one equal contiguous range per pair, so every SM streams the same weight
// bytes in one round, and a tile cut between pairs is fixed up inside the kernel, cooperatively:
//   * a segment covering a whole tile (gate/up) runs the fused epilogue straight from TMEM;
//   * a CUT segment (a tile shared by pairs q0..q1) dumps its fp32 accumulator to the CTA's slot of sk_ws
//     ([M][128] fp32, bulk stores; one slot for the pair's first segment, one for its last) and raises the slot's
//     flag to the launch epoch. A pair's cut segments are its first and/or its last, so the dumps of a tile's
//     contributors are all written by the time the contributors finish their ranges, which balanced ranges make
//     simultaneous;
//   * then each contributor j of a cut tile finalises rows [j M / c, (j + 1) M / c) of it (c contributors): one
//     bulk copy per contributor of those rows into the freed stage ring, the sum in k order (contributor order),
//     and the fused epilogue. The fix-up is parallel over the tile's SMs and costs one L2 round trip.
// Flag waits go to CTAs that are resident (all CTAs are resident before any dependent launch, PDL), so they cannot
// deadlock.
//
// Epilogue: the accumulator (TMEM lane = output column, TMEM column = activation row) is staged 32 rows at a time in
// shared memory as [row][128 columns] fp32, and quad_epi (gemm_epi.cuh, the reduce kernel's arithmetic) writes every
// mode from there: RoPE + prefix-pool admission, residual + folded-norm outputs, SiLU.mul, bf16, fp32.
//
// CTA pair layout (cluster of 2, 256 threads per CTA, one CTA per SM):
//   warp 0      TMA producer (one lane): per k-block its 128 weight rows (16 KB) + NP/2 activation rows
//   warp 1      MMA issuer (leader CTA): M256 x NP x K16 x 4 per k-block into a TMEM accumulator (double buffered)
//   warp 2      TMEM allocator
//   warps 4..7  epilogue (thread = one of the CTA's 128 output columns while draining TMEM)
#include "gemm.cuh"
#include "gemm_epi.cuh"
#include "stream.cuh"
#include <algorithm>
#include <cstdlib>

namespace po {

#ifdef SK_TRACE
// globaltimer stamps per CTA of the last launch with N == SK_TRACE_N (tools/dbg_sk_trace.py): 0 start, 1 setup done,
// 2 first full barrier (MMA), 3 last MMA commit, 4 first tfull (epilogue), 5 a dump published, 6 fix-up flags seen,
// 7 fix-up rows landed, 8 epilogue done, 9 exit
__device__ unsigned long long g_sk_trace[296 * 16];
__device__ __forceinline__ unsigned long long sk_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define SKT(i, cond) \
  do {               \
    if ((cond) && args.N == SK_TRACE_N && args.M > 1) g_sk_trace[blockIdx.x * 16 + (i)] = sk_gtime(); \
  } while (0)
#else
#define SKT(i, cond) \
  do {               \
  } while (0)
#endif

namespace {
constexpr int BK = 64;
constexpr int W_BYTES = 128 * BK * 2;  // 16 KB: this CTA's 128 weight rows of a k-block
constexpr int X_MAX = 128 * BK * 2;    // up to 128 activation rows (NP <= 256, half per CTA)
constexpr int STAGE = W_BYTES + X_MAX;
constexpr int STAGES = 6;
constexpr int CH = 32;                   // activation rows per epilogue chunk
constexpr int CH_BYTES = CH * 128 * 4;   // one chunk of the CTA's 128 columns in fp32 (= W_BYTES: a fix-up piece)
constexpr int SMEM = STAGES * STAGE + 2 * CH_BYTES + 1024 + 256 + 1024;
constexpr int NT = 256;
constexpr int ACC_STRIDE = 256;          // TMEM columns between the two accumulators
}  // namespace

// Segment of a pair's range [f, hi) that starts at work item f: tile t, k-blocks [a, b).
struct SkSeg {
  int t, a, b;
};
__device__ __forceinline__ SkSeg sk_seg(int f, int hi, int nk) {
  SkSeg s;
  s.t = f / nk;
  s.a = f - s.t * nk;
  s.b = min(nk, hi - s.t * nk);
  return s;
}

// Per-column constants of the row-major epilogue for this thread's 4 columns [col, col + 4) of a 128-column half tile
struct SkCols {
  float4 g4, b1, b2;
};
template <int EPI>
__device__ __forceinline__ SkCols sk_cols(const GemmArgs& a, int col, int lc) {
  SkCols k{};
  if (EPI == EPI_RESID_F32 && a.xg_out) k.g4 = *reinterpret_cast<const float4*>(a.g_next + col);
  if (EPI == EPI_QKV_ROPE && a.bias) {
    k.b1 = *reinterpret_cast<const float4*>(a.bias + col);
    if (col < a.rope_cols && lc < 64) k.b2 = *reinterpret_cast<const float4*>(a.bias + col + 64);
  }
  return k;
}

// Fused epilogue of rows row0 + i (i < nrows; warp wq takes i = wq, wq + 4, ...) of a CTA's 128-column half tile,
// row-major: lane = 4 columns [col, col + 4) (lc = col - col0). src(i, off) returns the summed fp32 values of local
// row i at columns lc + off .. + 3. aux: per local row, the residual values of the half tile (EPI_RESID_F32, 128
// floats) or the RoPE (cos, sin) pairs of the row's position (EPI_QKV_ROPE, 64 float2), aux_ld floats apart; shared
// memory (fix-up: bulk-copied next to the partials, so the loop issues no global load) or global memory. slots:
// the prefix-pool slot of each local row's block (admission; shared memory) or null (read kv_slot). One warp per
// SM sub-partition runs this, so a row's dependent chain (shared loads, MUFU, store) is exposed unless independent
// rows overlap: unrolled by 4 (a single-row loop measured ~675 cycles per row). Arithmetic as quad_epi's.
template <int EPI, typename Src>
__device__ __forceinline__ void sk_rows(const GemmArgs& a, int row0, int nrows, int wq, int lane, int col0,
                                        const float* s_inv, const SkCols& kc, const float* aux, int aux_ld,
                                        const int* slots, Src src) {
  const int lc = lane * 4;
  const int col = col0 + lc;
#pragma unroll 4
  for (int i = wq; i < nrows; i += 4) {
    const int row = row0 + i;
    if constexpr (EPI == EPI_RESID_F32) {
      const float4 a4 = src(i, 0);
      float4 v = *reinterpret_cast<const float4*>(aux + (long long)i * aux_ld + lc);
      v.x += a4.x; v.y += a4.y; v.z += a4.z; v.w += a4.w;
      *reinterpret_cast<float4*>(a.resid + (long long)row * a.ldr + col) = v;
      if (a.xg_out) {
        *reinterpret_cast<uint2*>(a.xg_out + (long long)row * a.ldxg + col) =
            make_uint2(pack_bf16(v.x * kc.g4.x, v.y * kc.g4.y), pack_bf16(v.z * kc.g4.z, v.w * kc.g4.w));
        float sq = v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
#pragma unroll
        for (int o = 16; o; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
        if (lane == 0) a.ss_out[(long long)row * a.ss_nseg + col / 128] = sq;
      }
    } else if constexpr (EPI == EPI_QKV_ROPE) {
      const bool rot = col < a.rope_cols;
      if (rot && lc >= 64) continue;  // the partner lane (lc - 64) writes the rotated pair
      const int pos = a.pos_offset + row;
      int pslot = -1;
      if (a.kv_pool && col0 >= a.kv_col0) pslot = slots ? slots[i] : a.kv_slot[pos >> 4];
      __nv_bfloat16* prow = pslot >= 0
          ? a.kv_pool + (((long long)pslot * a.pool_layers + a.pool_layer) * 16 + (pos & 15)) * a.kv_dim - a.kv_col0
          : nullptr;
      const float sc = s_inv[row];
      float4 acc = src(i, 0);
      acc.x *= sc; acc.y *= sc; acc.z *= sc; acc.w *= sc;
      acc.x += kc.b1.x; acc.y += kc.b1.y; acc.z += kc.b1.z; acc.w += kc.b1.w;
      __nv_bfloat16* o = static_cast<__nv_bfloat16*>(a.out) + (long long)row * a.ldo + col;
      if (rot) {
        float4 x2 = src(i, 64);
        x2.x *= sc; x2.y *= sc; x2.z *= sc; x2.w *= sc;
        x2.x += kc.b2.x; x2.y += kc.b2.y; x2.z += kc.b2.z; x2.w += kc.b2.w;
        const float4 ca = *reinterpret_cast<const float4*>(aux + (long long)i * aux_ld + 2 * lc);
        const float4 cb = *reinterpret_cast<const float4*>(aux + (long long)i * aux_ld + 2 * lc + 4);
        const uint2 lo = make_uint2(pack_bf16(acc.x * ca.x - x2.x * ca.y, acc.y * ca.z - x2.y * ca.w),
                                    pack_bf16(acc.z * cb.x - x2.z * cb.y, acc.w * cb.z - x2.w * cb.w));
        const uint2 hi = make_uint2(pack_bf16(x2.x * ca.x + acc.x * ca.y, x2.y * ca.z + acc.y * ca.w),
                                    pack_bf16(x2.z * cb.x + acc.z * cb.y, x2.w * cb.z + acc.w * cb.w));
        *reinterpret_cast<uint2*>(o) = lo;
        *reinterpret_cast<uint2*>(o + 64) = hi;
        if (prow) {
          *reinterpret_cast<uint2*>(prow + col) = lo;
          *reinterpret_cast<uint2*>(prow + col + 64) = hi;
        }
      } else {
        const uint2 v = make_uint2(pack_bf16(acc.x, acc.y), pack_bf16(acc.z, acc.w));
        *reinterpret_cast<uint2*>(o) = v;
        if (prow) *reinterpret_cast<uint2*>(prow + col) = v;
      }
    } else if constexpr (EPI == EPI_SILU_MUL) {
      if ((lc & 31) < 16) quad_epi<EPI>(a, row, col, src(i, 0), src(i, 16), s_inv[row], float4{});
    } else if constexpr (EPI == EPI_F32) {
      *reinterpret_cast<float4*>(static_cast<float*>(a.out) + (long long)row * a.ldo + col) = src(i, 0);
    } else {
      quad_epi<EPI>(a, row, col, src(i, 0), float4{}, 1.f, float4{});
    }
  }
}

template <int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NT, 1)
    gemm_sk_kernel(const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_x,
                   const __grid_constant__ CUtensorMap map_st, const __grid_constant__ CUtensorMap map_r,
                   const __grid_constant__ CUtensorMap map_xo, const GemmArgs args, int np) {
  // HEADFIX (epilogues with a transposed TMA-store form: SiLU.mul, bf16, fp32): the pair holding a cut tile's
  // k-block 0 finalises the whole tile - the other contributors' partials (their first segments, dumped early) are
  // bulk-copied into the freed stage ring, added to the TMEM values per 32-row chunk, and the chunk leaves through
  // the same staged TMA stores as the per-GEMM swap kernel. Other epilogues use the cooperative fix-up below.
  // EPI_RESID_F32 joins it with a transposed residual epilogue: per warp and chunk a [32 rows x 32 fp32] residual box
  // by TMA (128-byte swizzle: thread = column reads a row's 128 bytes conflict-free), updated in place, stored back
  // with the bf16 folded-norm input box; the per-row sums of squares over the CTA's 128 columns by a butterfly
  // transpose-reduction inside each warp and a 4-warp sum in shared memory.
  constexpr bool HEADFIX = EPI == EPI_SILU_MUL || EPI == EPI_BF16 || EPI == EPI_F32 || EPI == EPI_RESID_F32;
  constexpr bool RESID = EPI == EPI_RESID_F32;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint8_t* sW = smem;
  uint8_t* sX = smem + STAGES * W_BYTES;
  uint8_t* stg = smem + STAGES * STAGE;
  float* s_inv = reinterpret_cast<float*>(stg + 2 * CH_BYTES);  // 1/rms per activation row (<= 256)
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(stg + 2 * CH_BYTES + 1024);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* fx_bar = tempty_bar + 2;  // fix-up copies, one phase per cut tile
  uint64_t* ss_bar = fx_bar + 1;      // the rows' RMS segment sums (folded-norm consumers)
  uint64_t* fx2 = ss_bar + 1;         // [2] HEADFIX: the contributors' rows of chunk k in ring buffer k & 1
  uint64_t* rb_bar = fx2 + 2;         // [4] RESID: each epilogue warp's residual box
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rb_bar + 4);

  const int warp = warp_id();
  const int lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1;
  const int P = gridDim.x >> 1;
  const int nk = args.K / BK;
  const long long W = (long long)(args.N / 256) * nk;
  const int lo = stream_pair_start(W, P, pair);
  const int hi = stream_pair_start(W, P, pair + 1);
  const int M = args.M;
  const int xh = np / 2;
  const uint32_t x_bytes = (uint32_t)xh * BK * 2;
  SKT(0, threadIdx.x == 0);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_w);
    tma_prefetch_desc(&map_x);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 2);
    }
    mbar_init(fx_bar, 1);
    mbar_init(ss_bar, 1);
    for (int b = 0; b < 2; ++b) mbar_init(&fx2[b], 1);
    for (int b = 0; b < 4; ++b) mbar_init(&rb_bar[b], 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_pair(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  SKT(1, threadIdx.x == 0);
  // weights are constant: the producer streams its first STAGES weight k-blocks before waiting for the kernel that
  // writes the activations
  if (warp != 0) pdl_wait();
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t full0 = mapa_shared(smem_u32(full_bar), 0);
      int s = 0;
      uint32_t ph = 0;
      int pend_s[STAGES], pend_kb[STAGES];
      int npend = 0;
      bool open = false;
      const int xrow = args.a_row0 + (int)rank * xh;
      auto flush = [&]() {
        pdl_wait();
        open = true;
        for (int i = 0; i < npend; ++i)
          tma_load_2d_pair(sX + pend_s[i] * X_MAX, &map_x, full0 + pend_s[i] * 8, pend_kb[i] * BK, xrow);
        npend = 0;
      };
      for (int f = lo; f < hi;) {
        const SkSeg sg = sk_seg(f, hi, nk);
        for (int kb = sg.a; kb < sg.b; ++kb) {
          mbar_wait(&empty_bar[s], ph ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&full_bar[s], 2 * (W_BYTES + x_bytes));
          const uint32_t fb = full0 + s * 8;
          tma_load_2d_pair(sW + s * W_BYTES, &map_w, fb, kb * BK, sg.t * 256 + (int)rank * 128);
          if (open) {
            tma_load_2d_pair(sX + s * X_MAX, &map_x, fb, kb * BK, xrow);
          } else {
            pend_s[npend] = s;
            pend_kb[npend] = kb;
            if (++npend == STAGES) flush();
          }
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
        f = sg.t * nk + sg.b;
      }
      if (!open) flush();
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      const uint32_t idesc = idesc_bf16_f32(256, (uint32_t)np);
      int s = 0;
      uint32_t ph = 0;
      int it = 0;
      for (int f = lo; f < hi; ++it) {
        const SkSeg sg = sk_seg(f, hi, nk);
        const int acc = it & 1;
        mbar_wait(&tempty_bar[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * ACC_STRIDE;
        for (int kb = sg.a; kb < sg.b; ++kb) {
          mbar_wait(&full_bar[s], ph);
          tc_fence_after();
          SKT(2, it == 0 && kb == sg.a);
          const uint64_t adesc = sdesc_kmajor_sw128(smem_u32(sW + s * W_BYTES));
          const uint64_t bdesc = sdesc_kmajor_sw128(smem_u32(sX + s * X_MAX));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            mma_bf16_ss_pair(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb != sg.a || k != 0) ? 1u : 0u);
          mma_commit_pair(&empty_bar[s], 0x3);
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
        mma_commit_pair(&tfull_bar[acc], 0x3);
        f = sg.t * nk + sg.b;
      }
      SKT(3, true);
    }
    __syncwarp();
  } else if (warp >= 4) {
    const int wq = warp & 3;
    const int et = threadIdx.x - 128;  // this thread's column of the CTA's 128 while draining TMEM
    const int lc = lane * 4;           // ... and its 4 columns in the row-major epilogue
    const uint32_t tempty0 = mapa_shared(smem_u32(tempty_bar), 0);
    if ((EPI == EPI_SILU_MUL || EPI == EPI_QKV_ROPE) && !args.sk_red) {
      // 1/rms of every activation row, once per launch: the rows' segment sums arrive by bulk copy (one L2 round
      // trip instead of a dependent chain per row), then each thread sums its rows in segment order (row_inv_rms)
      const int nseg = args.ss_nseg;
      if (!args.ss_in || (reinterpret_cast<uintptr_t>(args.ss_in) & 15) || ((nseg * 4) & 15)) {
        // (bulk copies need 16-byte aligned rows: small models / odd row offsets load per row)
        for (int r = et; r < M; r += 128) s_inv[r] = args.ss_in ? row_inv_rms(args, r) : 1.0f;
      } else {
        const int rpp = min(M, (2 * CH_BYTES) / (nseg * 4));  // rows per staged piece
        const float* ss = reinterpret_cast<const float*>(stg);
        uint32_t ph = 0;
        for (int p0 = 0; p0 < M; p0 += rpp, ph ^= 1) {
          const int nr = min(rpp, M - p0);
          if (et == 0) {
            mbar_arrive_expect_tx(ss_bar, (uint32_t)nr * nseg * 4);
            bulk_g2s(stg, args.ss_in + (size_t)p0 * nseg, (uint32_t)nr * nseg * 4, ss_bar);
          }
          mbar_wait(ss_bar, ph);
          for (int r = et; r < nr; r += 128) {
            float sum = 0.f;
            for (int i = 0; i < nseg; ++i) sum += ss[r * nseg + i];
            s_inv[p0 + r] = rsqrtf(sum / args.norm_dim + args.norm_eps);
          }
          named_bar_sync(1, 128);  // the next piece overwrites the staging buffer
        }
      }
    }
    const int first_t = lo / nk;
    int it = 0, nch = 0;
    uint32_t rb_ph = 0;  // RESID: parity of this warp's residual box barrier
    for (int f = lo; f < hi; ++it) {
      const SkSeg sg = sk_seg(f, hi, nk);
      f = sg.t * nk + sg.b;
      const bool cut = args.sk_red || sg.a > 0 || sg.b < nk;  // reduce mode: every segment is a partial
      const int acc = it & 1;
      mbar_wait(&tfull_bar[acc], (it >> 1) & 1);
      tc_fence_after();
      SKT(4, et == 0 && it == 0);
      const uint32_t taddr = tmem_base + ((uint32_t)(wq * 32) << 16) + acc * ACC_STRIDE;
      const int col0 = sg.t * 256 + (int)rank * 128;  // the CTA's first output column of this tile
      const int slot = (int)blockIdx.x * 2 + (sg.t == first_t ? 0 : 1);  // dump slot of a cut segment
      const SkCols kc = cut ? SkCols{} : sk_cols<EPI>(args, col0 + lc, lc);
      const bool head = HEADFIX && !args.sk_red && sg.a == 0 && sg.b < nk;  // HEADFIX: this pair finalises the cut tile
      const bool dump = cut && !head;
      int nq = 0;
      // HEADFIX: chunk k of the contributors' partials (their rows c0 .. c0+31, 16 KB each) into ring buffer k & 1
      auto issue_piece = [&](int k) {
        if (warp == 4 && lane == 0 && k * CH < M) {
          const uint32_t bytes = (uint32_t)min(CH, M - k * CH) * 512;
          mbar_arrive_expect_tx(&fx2[k & 1], bytes * nq);
          for (int q = 0; q < nq; ++q)
            bulk_g2s(smem + (size_t)((k & 1) * nq + q) * CH_BYTES,
                     args.sk_ws + ((size_t)((2 * (pair + 1 + q) + (int)rank) * 2) * 256 + k * CH) * 128, bytes,
                     &fx2[k & 1]);
        }
      };
      if (head) {
        // contributors pair+1 .. q1 hold the rest of the tile, each as its first segment (dump slot 0)
        const int q1 = stream_owner(W, P, sg.t * nk + nk - 1);
        nq = q1 - pair;
        if (warp == 4) {
          bool ok;
          uint32_t ns = 32;
          do {
            ok = true;
            for (int q = pair + 1 + lane; q <= q1; q += 32)
              ok &= (int)(ld_relaxed_u32(args.sk_flags + (size_t)((2 * q + (int)rank) * 2) * SK_FLAG_STRIDE) -
                          args.sk_epoch) >= 0;
            ok = __all_sync(0xffffffffu, ok);
            if (!ok) {
              __nanosleep(ns);
              ns = ns < 256 ? ns * 2 : 256;
            }
          } while (!ok);
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
          fence_proxy_async_global();
          SKT(6, lane == 0);
        }
        issue_piece(0);
        issue_piece(1);
        SKT(7, et == 0);
      }
#pragma unroll 1
      for (int c0 = 0; c0 < M; c0 += CH, ++nch) {
        uint32_t r[32];
        tmem_ld32(taddr + c0, r);
        tmem_ld_wait();
        const int rows = min(CH, M - c0);
        if constexpr (HEADFIX) {
          if (!dump) {
            const int k = c0 / CH;
            float4* rbox = reinterpret_cast<float4*>(stg + wq * 8192);  // RESID: this warp's residual box
            if constexpr (RESID) {
              if (lane == 0) {
                bulk_wait_read<0>();  // the previous chunk's store has read the box
                mbar_arrive_expect_tx(&rb_bar[wq], 4096);
                tma_load_2d(rbox, &map_r, &rb_bar[wq], col0 + wq * 32, c0);
              }
            }
            if (nq > 0) {
              // partials of the other contributors, in k order (this chunk's rows in ring buffer k & 1)
              mbar_wait(&fx2[k & 1], (k >> 1) & 1);
              for (int q = 0; q < nq; ++q) {
                const float* pp = reinterpret_cast<const float*>(smem + (size_t)((k & 1) * nq + q) * CH_BYTES) + et;
#pragma unroll
                for (int i = 0; i < 32; ++i)
                  if (i < rows) r[i] = __float_as_uint(__uint_as_float(r[i]) + pp[i * 128]);
              }
              named_bar_sync(1, 128);  // every thread is done with buffer k & 1: refill it with chunk k + 2
              issue_piece(k + 2);
            }
            if constexpr (RESID) {
              mbar_wait(&rb_bar[wq], rb_ph);
              rb_ph ^= 1;
              const float gcol = args.xg_out ? args.g_next[col0 + wq * 32 + lane] : 0.f;
              __nv_bfloat16* xbox = reinterpret_cast<__nv_bfloat16*>(stg + wq * 8192 + 4096);
              float a2[32];
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                // element (row i, column lane) of the 128B-swizzled box: 16-byte chunk (lane / 4) ^ (i & 7)
                float* e = reinterpret_cast<float*>(rbox + i * 8 + ((lane >> 2) ^ (i & 7))) + (lane & 3);
                const float v = *e + __uint_as_float(r[i]);
                *e = v;
                xbox[i * 32 + lane] = __float2bfloat16_rn(v * gcol);
                a2[i] = v * v;
              }
              fence_proxy_async_smem();
              __syncwarp();
              if (lane == 0) {
                tma_store_2d(&map_r, rbox, col0 + wq * 32, c0);
                if (args.xg_out) tma_store_2d(&map_xo, xbox, col0 + wq * 32, c0);
                bulk_commit();
              }
              if (args.ss_out) {
                // butterfly transpose-reduction: lane l ends with this warp's sum of squares of row l
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1) {
                  const bool up = (lane & off) != 0;
#pragma unroll
                  for (int i = 0; i < off; ++i) {
                    const float send = up ? a2[i] : a2[i + off];
                    const float keep = up ? a2[i + off] : a2[i];
                    a2[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
                  }
                }
                float* s_sq = s_inv;  // [4 warps][32 rows]
                s_sq[wq * 32 + lane] = a2[0];
                named_bar_sync(1, 128);
                if (wq == 0 && lane < rows)
                  args.ss_out[(long long)(c0 + lane) * args.ss_nseg + col0 / 128] =
                      ((s_sq[lane] + s_sq[32 + lane]) + s_sq[64 + lane]) + s_sq[96 + lane];
                named_bar_sync(1, 128);  // s_sq is rewritten by the next chunk
              }
              continue;
            }
            // transposed TMA-store epilogue (as gemm_swap.cu): this warp's 32 rows x 32 columns staged, one store
            uint8_t* wb = stg + (wq * 2 + (nch & 1)) * 4096;
            if (lane == 0) bulk_wait_read<1>();  // the store that last read this buffer (two chunks ago) is done
            __syncwarp();
            int sc0 = col0 + wq * 32;
            if constexpr (EPI == EPI_F32) {
              float* tt = reinterpret_cast<float*>(wb);
#pragma unroll
              for (int j = 0; j < 32; ++j) tt[j * 32 + lane] = __uint_as_float(r[j]);
            } else if constexpr (EPI == EPI_BF16) {
              __nv_bfloat16* tt = reinterpret_cast<__nv_bfloat16*>(wb);
#pragma unroll
              for (int j = 0; j < 32; ++j) tt[j * 32 + lane] = __float2bfloat16_rn(__uint_as_float(r[j]));
            } else {
              // weight rows in 16-row groups [gate 16 | up 16]: lanes 0..15 hold gate columns, 16..31 the matching up
              // columns; two activation rows per step, every lane busy (see gemm_swap.cu)
              __nv_bfloat16* tt = reinterpret_cast<__nv_bfloat16*>(wb);
              const bool hi = lane >= 16;
#pragma unroll
              for (int j = 0; j < 32; j += 2) {
                const float mine = __uint_as_float(hi ? r[j] : r[j + 1]);
                const float other = __shfl_xor_sync(0xffffffffu, mine, 16);
                const float g = hi ? other : __uint_as_float(r[j]);
                const float up = hi ? __uint_as_float(r[j + 1]) : other;
                const int row = j + (hi ? 1 : 0);
                const float sc = s_inv[min(c0 + row, 255)];
                tt[row * 16 + (lane & 15)] = __float2bfloat16_rn(silu_f(sc * g) * (sc * up));
              }
              sc0 /= 2;
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_3d(&map_st, wb, sc0, c0, 0);
              bulk_commit();
            }
            continue;
          }
        }
        if (args.sk_red) {
          // contributor j of tile sg.t (k order) -> split_ws slice j ([maxc][M][N] fp32): this warp's 32 rows x 32
          // columns staged transposed in shared memory, one TMA store (as the swap kernel's split-K partials)
          const int j = pair - stream_owner(W, P, sg.t * nk);
          uint8_t* wb = stg + (wq * 2 + (nch & 1)) * 4096;
          if (lane == 0) bulk_wait_read<1>();  // the store that last read this buffer (two chunks ago) is done
          __syncwarp();
          float* tt = reinterpret_cast<float*>(wb);
#pragma unroll
          for (int i = 0; i < 32; ++i) tt[i * 32 + lane] = __uint_as_float(r[i]);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_3d(&map_st, wb, col0 + wq * 32, c0, j);
            bulk_commit();
          }
          continue;
        }
        if (cut) {  // the fp32 partial, straight from registers: one 128-byte line per warp and row
          float* dst = args.sk_ws + ((size_t)slot * 256 + c0) * 128 + et;
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (i < rows) dst[i * 128] = __uint_as_float(r[i]);
          continue;
        }
        float* buf = reinterpret_cast<float*>(stg + (nch & 1) * CH_BYTES);
        named_bar_sync(1, 128);  // every thread's epilogue reads of this buffer (two chunks ago) are done
#pragma unroll
        for (int i = 0; i < 32; ++i) buf[i * 128 + et] = __uint_as_float(r[i]);
        named_bar_sync(1, 128);
        const float* brow = buf + lc;
        const float* aux = EPI == EPI_RESID_F32 ? args.resid + (long long)c0 * args.ldr + col0
                           : EPI == EPI_QKV_ROPE ? reinterpret_cast<const float*>(args.rope + (long long)(args.pos_offset + c0) * 64)
                                                 : nullptr;
        sk_rows<EPI>(args, c0, rows, wq, lane, col0, s_inv, kc, aux,
                     EPI == EPI_RESID_F32 ? (int)args.ldr : 128, nullptr, [=](int i, int off) {
                       return *reinterpret_cast<const float4*>(brow + i * 128 + off);
                     });
      }
      if (dump) __threadfence();  // this thread's partial stores, before the flag below
      tc_fence_before();
      named_bar_sync(1, 128);
      if (et == 0) {
        mbar_arrive_cluster(tempty0 + acc * 8);
        if (dump && !args.sk_red) {  // publish the partial (the reduce launch needs no flag)
          st_release_u32(args.sk_flags + (size_t)slot * SK_FLAG_STRIDE, args.sk_epoch);
          SKT(5, true);
        }
      }
    }
    // Cooperative fix-up of the cut tiles this pair holds a segment of: its first and/or last segment. The stage
    // ring is free (every MMA of this CTA has completed), so each contributor's rows of this CTA's share land there.
    const SkSeg first = sk_seg(lo, hi, nk);
    const SkSeg last = sk_seg(max(lo, (hi - 1) / nk * nk), hi, nk);
    uint32_t fx_phase = 0;
#pragma unroll 1
    for (int w = 0; w < ((HEADFIX || args.sk_red) ? 0 : 2); ++w) {
      const SkSeg sg = w == 0 ? first : last;
      if (w == 1 && last.t == first.t) break;
      if (sg.a == 0 && sg.b == nk) continue;  // a whole tile: done above
      const int t = sg.t;
      const int q0 = stream_owner(W, P, t * nk), q1 = stream_owner(W, P, t * nk + nk - 1);
      const int c = q1 - q0 + 1, j = pair - q0;
      const int r0 = (int)((long long)j * M / c), r1 = (int)((long long)(j + 1) * M / c);
      if (r0 == r1) continue;
      const int nr = r1 - r0;
      const uint32_t bytes = (uint32_t)nr * 512;
      float* aux = reinterpret_cast<float*>(smem + (size_t)c * bytes);  // residual or RoPE rows of the share
      int* s_slot = reinterpret_cast<int*>(stg);                       // pool slot per row of the share (<= 128)
      if (EPI == EPI_QKV_ROPE && args.kv_pool)
        for (int i = et; i < nr; i += 128) s_slot[i] = args.kv_slot[(args.pos_offset + r0 + i) >> 4];
      const int col0 = t * 256 + (int)rank * 128;
      if (warp == 4) {
        // poll every contributor's dump flag for this tile (slot 0 if the tile is its first segment's), one lane each
        bool ok;
        uint32_t ns = 32;
        do {
          ok = true;
          for (int q = q0 + lane; q <= q1; q += 32) {
            const int qs = (2 * q + (int)rank) * 2 + (stream_pair_start(W, P, q) / nk == t ? 0 : 1);
            ok &= (int)(ld_relaxed_u32(args.sk_flags + (size_t)qs * SK_FLAG_STRIDE) - args.sk_epoch) >= 0;
          }
          ok = __all_sync(0xffffffffu, ok);
#ifdef PO_DEBUG_HANG
          if (!ok && ns == 256 && lane == 0) {
            static_assert(true, "");
            if (clock64() % 100000 < 50)
              printf("SK POLL block %d tile %d q0 %d q1 %d epoch %u M %d N %d K %d\n", blockIdx.x, t, q0, q1,
                     args.sk_epoch, M, args.N, args.K);
          }
#endif
          if (!ok) {
            __nanosleep(ns);
            ns = ns < 256 ? ns * 2 : 256;
          }
        } while (!ok);
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        fence_proxy_async_global();
        SKT(6, lane == 0);
        const uint32_t aux_bytes = (EPI == EPI_RESID_F32 || EPI == EPI_QKV_ROPE) ? bytes : 0;
        if (lane == 0) mbar_arrive_expect_tx(fx_bar, bytes * c + aux_bytes);
        __syncwarp();
        for (int q = q0 + lane; q <= q1; q += 32) {
          const int qs = (2 * q + (int)rank) * 2 + (stream_pair_start(W, P, q) / nk == t ? 0 : 1);
          bulk_g2s(smem + (size_t)(q - q0) * bytes, args.sk_ws + ((size_t)qs * 256 + r0) * 128, bytes, fx_bar);
        }
        if constexpr (EPI == EPI_RESID_F32) {  // the share's residual rows (512 B each at row stride ldr)
          for (int i = lane; i < nr; i += 32)
            bulk_g2s(aux + i * 128, args.resid + (long long)(r0 + i) * args.ldr + col0, 512, fx_bar);
        } else if constexpr (EPI == EPI_QKV_ROPE) {  // the positions' (cos, sin) rows: one contiguous block
          if (lane == 0) bulk_g2s(aux, args.rope + (long long)(args.pos_offset + r0) * 64, bytes, fx_bar);
        }
      }
      mbar_wait(fx_bar, fx_phase);
      fx_phase ^= 1;
      if (EPI == EPI_QKV_ROPE && args.kv_pool) named_bar_sync(1, 128);  // s_slot
      SKT(7, et == 0);
      SKT(10 + 3 * w, et == 0);
      const SkCols kc = sk_cols<EPI>(args, col0 + lc, lc);
      const float* part = reinterpret_cast<const float*>(smem) + lc;
      const int pstride = (int)(bytes / 4);
      sk_rows<EPI>(args, r0, nr, wq, lane, col0, s_inv, kc, aux, 128, s_slot, [=](int i, int off) {
        const float* p = part + i * 128 + off;
        float4 v = *reinterpret_cast<const float4*>(p);
        for (int q = 1; q < c; ++q) {
          const float4 u = *reinterpret_cast<const float4*>(p + q * pstride);
          v.x += u.x; v.y += u.y; v.z += u.z; v.w += u.w;
        }
        return v;
      });
      SKT(12 + 3 * w, et == 0);
      named_bar_sync(1, 128);  // the copies of the next cut tile overwrite these rows
    }
    SKT(8, et == 0);
    // every warp's TMA stores (outputs, residual boxes, partials) complete before the CTA exits: bulk groups are
    // per issuing thread, so each warp's lane 0 waits for its own
    if ((HEADFIX || args.sk_red) && lane == 0) bulk_wait_all();

  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, 512);
  }
  SKT(9, threadIdx.x == 0);
}

// Which short launches run through this kernel: PO_SK=0 none, PO_SK=1 every epilogue, default (unset) SiLU.mul /
// bf16 / fp32 (the prefix hit's gate/up), whose head fix-up streams the contributors' rows and leaves through staged
// TMA stores. The cooperative fix-up of the residual / RoPE epilogues measured slower than the split-K reduce launches
// (DESIGN.md "Short-M GEMMs").
static int sk_mode() {  // 0: off, 1: every epilogue, 2 (default): SiLU.mul / bf16 / fp32
  static int mode = -1;
  if (mode < 0) {
    const char* v = getenv("PO_SK");
    mode = !v ? 2 : (v[0] == '1' ? 1 : 0);
  }
  return mode;
}
// PO_SK_RED=1 (opt-in, measured slower: DESIGN.md "Short-M GEMMs"): the residual / RoPE epilogues run stream-K with
// every partial written to the split-K workspace and the split-K reduce kernel as the epilogue
static bool sk_red_enabled() {
  static int on = -1;
  if (on < 0) on = (getenv("PO_SK_RED") && getenv("PO_SK_RED")[0] == '1') ? 1 : 0;
  return on == 1;
}
static bool sk_red_epi(int epi) { return sk_mode() == 2 && sk_red_enabled() && (epi == EPI_RESID_F32 || epi == EPI_QKV_ROPE); }
bool gemm_sk_enabled(int epi) {
  const int mode = sk_mode();
  if (mode == 1) return true;
  if (sk_red_epi(epi)) return true;
  // (the residual epilogue's head fix-up - 3-5 contributors streamed per chunk, transposed residual boxes - measured
  // slower than swap + reduce on the hit's O / down: 1.12 vs 0.81 ms and 1.58 vs 1.29 ms per forward)
  return mode == 2 && (epi == EPI_SILU_MUL || epi == EPI_BF16 || epi == EPI_F32);
}
bool gemm_sk_enabled() { return sk_mode() != 0; }
int splitk_reduce_launch(int epi, const GemmArgs& args, cudaStream_t stream);

size_t gemm_sk_ws_bytes() { return (size_t)num_sms() * 2 * 256 * 128 * sizeof(float); }
size_t gemm_sk_flag_bytes() { return (size_t)num_sms() * 2 * SK_FLAG_STRIDE * sizeof(uint32_t); }

int gemm_launch_sk(const CUtensorMap& map_w, const void* x, long long ldx, int epi, const GemmArgs& in,
                   cudaStream_t stream) {
  if (!in.sk_ws || !in.sk_flags || in.M < 1 || in.M > 256 || in.N % 256 || in.K % BK || in.K <= 0) return 1;
  GemmArgs args = in;
  args.k_splits = 1;
  const int np = (args.M + 15) / 16 * 16;
  const long long W = (long long)(args.N / 256) * (args.K / BK);
  const int P = (int)(W < num_sms() / 2 ? W : num_sms() / 2);
  CUtensorMap map_x, map_st, map_r, map_xo;
  if (make_tmap_2d_bf16(&map_x, x, args.K, (uint64_t)args.a_row0 + args.M, ldx * 2, BK, np / 2)) return -2;
  map_st = map_r = map_xo = map_x;  // unused unless HEADFIX / RESID
  if (sk_red_epi(epi)) {
    // stream-K + reduce: each tile's contributors write slices 0 .. c-1 of split_ws, then the split-K reduce kernel
    // sums them in k order and runs the epilogue
    const int nk = args.K / BK;
    int maxc = 1;
    for (int t = 0; t < args.N / 256; ++t)
      maxc = std::max(maxc, stream_owner(W, P, t * nk + nk - 1) - stream_owner(W, P, t * nk) + 1);
    if (!args.split_ws || (size_t)maxc * args.M * args.N * sizeof(float) > args.split_ws_bytes) return 1;
    if (make_tmap_store_3d(&map_st, args.split_ws, true, args.N, args.M, maxc, (uint64_t)args.N * 4,
                           (uint64_t)args.N * args.M * 4, 32, 32))
      return 1;
    args.sk_red = 1;
    args.sk_w = W;
    args.sk_p = P;
    args.sk_nk = nk;
    switch (epi) {
      case EPI_RESID_F32:
        ensure_smem_attr<gemm_sk_kernel<EPI_RESID_F32>>(SMEM);
        launch_pdl(gemm_sk_kernel<EPI_RESID_F32>, dim3(2 * P), dim3(NT), SMEM, stream, map_w, map_x, map_st, map_r,
                   map_xo, args, np);
        break;
      case EPI_QKV_ROPE:
        ensure_smem_attr<gemm_sk_kernel<EPI_QKV_ROPE>>(SMEM);
        launch_pdl(gemm_sk_kernel<EPI_QKV_ROPE>, dim3(2 * P), dim3(NT), SMEM, stream, map_w, map_x, map_st, map_r,
                   map_xo, args, np);
        break;
      default: return 1;
    }
    if (cudaGetLastError() != cudaSuccess) return -4;
    return splitk_reduce_launch(epi, args, stream);
  }
  args.sk_red = 0;
  if (epi == EPI_SILU_MUL || epi == EPI_BF16 || epi == EPI_F32 || epi == EPI_RESID_F32) {
    // HEADFIX: the head pair streams the other contributors' rows through two halves of its stage ring, 32 rows
    // (16 KB) per contributor per chunk
    const int nk = args.K / BK;
    int maxc = 1;
    for (int t = 0; t < args.N / 256; ++t)
      maxc = std::max(maxc, stream_owner(W, P, t * nk + nk - 1) - stream_owner(W, P, t * nk) + 1);
    if ((size_t)(maxc - 1) * 2 * CH_BYTES > (size_t)STAGES * STAGE) return 1;
  }
  if (epi == EPI_RESID_F32) {
    if (make_tmap_2d_epi(&map_r, args.resid, true, args.N, args.M, (uint64_t)args.ldr * 4, true) ||
        (args.xg_out && make_tmap_2d_epi(&map_xo, args.xg_out, false, args.N, args.M, (uint64_t)args.ldxg * 2, false)))
      return 1;
  }
  if (epi == EPI_SILU_MUL || epi == EPI_BF16 || epi == EPI_F32) {
    int mrc;
    if (epi == EPI_F32)
      mrc = make_tmap_store_3d(&map_st, args.out, true, args.N, args.M, 1, (uint64_t)args.ldo * 4,
                               (uint64_t)args.ldo * 4 * args.M, 32, 32);
    else if (epi == EPI_BF16)
      mrc = make_tmap_store_3d(&map_st, args.out, false, args.N, args.M, 1, (uint64_t)args.ldo * 2,
                               (uint64_t)args.ldo * 2 * args.M, 32, 32);
    else
      mrc = make_tmap_store_3d(&map_st, args.out, false, args.N / 2, args.M, 1, (uint64_t)args.ldo * 2,
                               (uint64_t)args.ldo * 2 * args.M, 16, 32);
    if (mrc) return 1;
  }
  switch (epi) {
#define PO_SK_CASE(E)                                                                                  \
  case E:                                                                                              \
    ensure_smem_attr<gemm_sk_kernel<E>>(SMEM);                                                         \
    launch_pdl(gemm_sk_kernel<E>, dim3(2 * P), dim3(NT), SMEM, stream, map_w, map_x, map_st, map_r, map_xo, args, np); \
    break;
    PO_SK_CASE(EPI_BF16)
    PO_SK_CASE(EPI_F32)
    PO_SK_CASE(EPI_SILU_MUL)
    PO_SK_CASE(EPI_RESID_F32)
    PO_SK_CASE(EPI_QKV_ROPE)
#undef PO_SK_CASE
    default: return 1;
  }
  return cudaGetLastError() == cudaSuccess ? 0 : -4;
}

}  // namespace po

#ifdef SK_TRACE
extern "C" int po_debug_swap_trace(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, po::g_sk_trace, sizeof(unsigned long long) * 296 * 16) == cudaSuccess ? 0 : -1;
}
#endif
