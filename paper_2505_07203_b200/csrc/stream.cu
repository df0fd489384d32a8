// Persistent weight-streaming layer kernel (see stream.cuh for the design).
//
// CTA pair layout (cluster of 2, 256 threads per CTA, one CTA per SM, grid = all SMs):
//   warp 0      TMA producer (one lane): per k-block its CTA's 128 activation rows + 128 of the 256 weight rows
//   warp 1      MMA issuer (leader CTA, one lane): tcgen05.mma.cta_group::2 M256 N256 K16 into a TMEM accumulator
//   warp 2      TMEM allocator (2 x 256 columns, double buffered across units and phases)
//   warps 4..7  epilogue: fused epilogue from TMEM, or fp32 partial dump + flag and the cooperative fix-up of the
//               split tiles; grid-barrier arrival after each phase
#include "stream.cuh"
#include "gemm_epi.cuh"
#include <algorithm>

namespace po {

#ifdef STREAM_DBG_TRACE
__device__ unsigned long long g_stream_trace[148 * 16];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TRACE(i, cond) \
  do {                 \
    if (cond) g_stream_trace[blockIdx.x * 16 + (i)] = gtime(); \
  } while (0)
#else
#define TRACE(i, cond) \
  do {                 \
  } while (0)
#endif

namespace {
constexpr int BM = 128;                        // rows per CTA (pair tile: 256)
constexpr int BN = 256;                        // weight rows (output columns) per pair tile
constexpr int BK = 64;
constexpr int HALF = 128 * BK * 2;             // 16 KB: 128 rows x 64 bf16 (A half or B half per CTA)
constexpr int STAGE = 2 * HALF;
constexpr int STAGES = 5;
constexpr int STG = 64 * 1024;                 // epilogue staging: partial dumps (4 warps x 2 x 4 KB), fix-up loads
constexpr int RBUF = STG / 2;                  // one fix-up batch buffer (two, double buffered)
constexpr int SMEM = STAGES * STAGE + STG + 1024 + 256 + 1024;
constexpr int NT = 256;
constexpr int FLAG_STRIDE = 32;                // one flag per 128-byte line: pollers of different flags never share one

struct Geo {
  int nk, ntiles, spt, M, P;  // P: pairs with work (min(pairs, W): every one of them owns >= 1 k-block)
  long long W;
};
__device__ __forceinline__ Geo geo_of(const StreamPhase& p, int pairs) {
  Geo g;
  g.nk = p.g.K / BK;
  g.ntiles = p.g.N / BN;
  g.W = (long long)g.nk * g.ntiles;
  g.P = g.W < pairs ? (int)g.W : pairs;
  g.spt = p.slots_per_tile;
  g.M = p.g.M;
  return g;
}
__device__ __forceinline__ int range_lo(const Geo& g, int pair) {
  return pair < g.P ? stream_pair_start(g.W, g.P, pair) : (int)g.W;
}
__device__ __forceinline__ int range_hi(const Geo& g, int pair) {
  return pair < g.P ? stream_pair_start(g.W, g.P, pair + 1) : (int)g.W;
}
struct Unit {
  int tile, kb0, kb1, seg, nseg;
};
// The unit of pair `pair` that starts at global k-block kb (ends at its range end or the tile end).
__device__ __forceinline__ Unit unit_at(const Geo& g, int pair, int kb) {
  Unit u;
  u.tile = kb / g.nk;
  const int t0 = u.tile * g.nk;
  const int end = min(range_hi(g, pair), t0 + g.nk);
  u.kb0 = kb - t0;
  u.kb1 = end - t0;
  const int first = stream_owner(g.W, g.P, t0);
  u.seg = pair - first;
  u.nseg = stream_owner(g.W, g.P, t0 + g.nk - 1) - first + 1;
  return u;
}

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// spin until *p >= target, then an acquire fence. One thread per CTA polls the single counter line with growing
// sleeps: 148 tight pollers saturate that line's L2 slice and stall every other access that hashes to it.
__device__ __forceinline__ void wait_counter(const unsigned long long* p, unsigned long long target) {
  uint32_t ns = 64;
  while (ld_relaxed_u64(p) < target) {
    __nanosleep(ns);
    ns = ns < 512 ? ns * 2 : 512;
  }
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

}  // namespace

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NT, 1) stream_kernel(const __grid_constant__ StreamArgs A) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * HALF;
  uint8_t* stg = smem + STAGES * STAGE;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(stg + STG);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* rbar = tempty_bar + 2;  // fix-up batch loads, one per buffer
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rbar + 2);
  float* s_inv = reinterpret_cast<float*>(stg + STG + 256);  // 1/rms of the rows a fix-up reduces (<= 256)

  const int warp = warp_id();
  const int lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1;
  const int P = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    for (int f = 0; f < A.nph; ++f) {
      tma_prefetch_desc(&A.ph[f].a);
      tma_prefetch_desc(&A.ph[f].b);
    }
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 2);
      mbar_init(&rbar[s], 1);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_pair(tmem_slot, 2 * BN);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // the producer streams phase 0's first weight k-blocks before waiting for the previous kernel (weights are
  // constant); everyone else waits now
  if (warp != 0) pdl_wait();
  pdl_trigger();
  TRACE(0, threadIdx.x == 0);

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t full0 = mapa_shared(smem_u32(full_bar), 0);
      int s = 0;
      uint32_t ph = 0;
      for (int f = 0; f < A.nph; ++f) {
        const StreamPhase& F = A.ph[f];
        const Geo g = geo_of(F, P);
        const int lo = range_lo(g, pair), hi = range_hi(g, pair);
        int pend_s[STAGES], pend_k[STAGES];
        int npend = 0;
        bool open = false;
        for (int kb = lo; kb < hi; ++kb) {
          const int tile = kb / g.nk, kk = kb - tile * g.nk;
          mbar_wait(&empty_bar[s], ph ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&full_bar[s], 2 * STAGE);
          const uint32_t fb = full0 + s * 8;
          tma_load_2d_pair(sB + s * HALF, &F.b, fb, kk * BK, tile * BN + rank * (BN / 2));
          if (open) {
            tma_load_2d_pair(sA + s * HALF, &F.a, fb, kk * BK, F.g.a_row0 + rank * BM);
          } else {
            pend_s[npend] = s;
            pend_k[npend] = kk;
            ++npend;
            if (npend == STAGES || kb + 1 == hi) {
              // the activations of this phase are the previous phase's output: wait for every CTA's epilogue
              if (f == 0) {
                pdl_wait();
              } else {
                wait_counter(A.bar, A.bar_base + (unsigned long long)f * gridDim.x);
              }
              fence_proxy_async_global();
              open = true;
              for (int i = 0; i < npend; ++i)
                tma_load_2d_pair(sA + pend_s[i] * HALF, &F.a, full0 + pend_s[i] * 8, pend_k[i] * BK,
                                 F.g.a_row0 + rank * BM);
              npend = 0;
            }
          }
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
        TRACE(1, f == 0);
        if (f == 0 && !open) pdl_wait();
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(2 * BM, BN);
      int s = 0;
      uint32_t ph = 0;
      int it = 0;
      for (int f = 0; f < A.nph; ++f) {
        const Geo g = geo_of(A.ph[f], P);
        const int hi = range_hi(g, pair);
        for (int kb = range_lo(g, pair); kb < hi; ++it) {
          const Unit u = unit_at(g, pair, kb);
          const int acc = it & 1;
          const uint32_t acc_ph = (it >> 1) & 1;
          mbar_wait(&tempty_bar[acc], acc_ph ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + acc * BN;
          for (int k = u.kb0; k < u.kb1; ++k) {
            mbar_wait(&full_bar[s], ph);
            tc_fence_after();
            const uint64_t adesc = sdesc_kmajor_sw128(smem_u32(sA + s * HALF));
            const uint64_t bdesc = sdesc_kmajor_sw128(smem_u32(sB + s * HALF));
#pragma unroll
            for (int j = 0; j < BK / 16; ++j)
              mma_bf16_ss_pair(d_tmem, adesc + 2 * j, bdesc + 2 * j, idesc, (k != u.kb0 || j) ? 1u : 0u);
            mma_commit_pair(&empty_bar[s], 0x3);
            if (++s == STAGES) { s = 0; ph ^= 1; }
          }
          mma_commit_pair(&tfull_bar[acc], 0x3);
          kb += u.kb1 - u.kb0;
        }
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    const int wq = warp & 3;
    const int et = threadIdx.x - 128;  // 0..127 within the epilogue warps
    const uint32_t tempty0 = mapa_shared(smem_u32(tempty_bar), 0);
    const int row = rank * BM + wq * 32 + lane;  // accumulator row of this thread (single 256-row m tile)
    int it = 0;
    uint32_t rb = 0;  // fix-up batches so far: buffer rb & 1, mbarrier parity (rb >> 1) & 1
    for (int f = 0; f < A.nph; ++f) {
      const StreamPhase& F = A.ph[f];
      const Geo g = geo_of(F, P);
      const uint32_t tag = A.tag * 8u + (uint32_t)f;
      const long long slot_elems = (long long)g.M * BN;
      int split_tiles[2], nsplit = 0;
      const int hi = range_hi(g, pair);
      for (int kb = range_lo(g, pair); kb < hi; ++it) {
        const Unit u = unit_at(g, pair, kb);
        kb += u.kb1 - u.kb0;
        const int acc = it & 1;
        const uint32_t acc_ph = (it >> 1) & 1;
        mbar_wait(&tfull_bar[acc], acc_ph);
        tc_fence_after();
        TRACE(2, f == 0 && et == 0 && kb == u.kb1 - u.kb0 + range_lo(g, pair));
        TRACE(3, f == 0 && et == 0);
        const uint32_t taddr = tmem_base + ((uint32_t)(wq * 32) << 16) + acc * BN;
        if (u.nseg > 1) {
          // a tile cut across pairs: dump this segment's fp32 partial and raise its flag; the segments' owners
          // reduce the tile together once all are in (below)
          // Layout of a partial slot: [8 column chunks][M rows][32 fp32], 128-byte rows with float4 q stored at
          // q ^ (row & 7). Each warp stages its 32 rows x 32 columns in shared memory and one lane writes the 4 KB
          // block with a bulk copy (full-line writes instead of 1 KB-strided per-thread stores).
          const long long slot = (long long)u.tile * g.spt + u.seg;
          const int rowbase = rank * BM + wq * 32;
          const int valid = min(max(g.M - rowbase, 0), 32);
          float* dst0 = A.ws + slot * slot_elems + (long long)rowbase * 32;
#pragma unroll 1
          for (int c = 0; c < 8; ++c) {
            uint32_t r[32];
            tmem_ld32(taddr + c * 32, r);
            uint8_t* wb = stg + (wq * 2 + (c & 1)) * 4096;
            if (lane == 0) bulk_wait_read<1>();  // the copy that last read this buffer (chunk c - 2) is done
            __syncwarp();
            tmem_ld_wait();
#pragma unroll
            for (int q = 0; q < 8; ++q)
              *reinterpret_cast<float4*>(wb + lane * 128 + ((q ^ (lane & 7)) << 4)) =
                  make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]), __uint_as_float(r[4 * q + 2]),
                              __uint_as_float(r[4 * q + 3]));
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0 && valid > 0) {
              bulk_s2g(dst0 + (long long)c * g.M * 32, wb, valid * 128);
              bulk_commit();
            }
          }
          if (lane == 0) {
            bulk_wait_all();
            fence_proxy_async_global();
          }
          tc_fence_before();
          named_bar_sync(1, 128);
          if (et == 0) {
            mbar_arrive_cluster(tempty0 + acc * 8);
            __threadfence();
            st_release_u32(A.flags + (slot * 2 + rank) * FLAG_STRIDE, tag);
          }
          split_tiles[nsplit++] = u.tile;
        } else {
          // a whole tile in one unit: fused epilogue straight from TMEM
          switch (F.epi) {
            case EPI_RESID_F32: epilogue_tile<EPI_RESID_F32, BN>(F.g, taddr, row, u.tile, 1, 0); break;
            case EPI_SILU_MUL: epilogue_tile<EPI_SILU_MUL, BN>(F.g, taddr, row, u.tile, 1, 0); break;
            case EPI_QKV_ROPE: epilogue_tile<EPI_QKV_ROPE, BN>(F.g, taddr, row, u.tile, 1, 0); break;
            default: epilogue_tile<EPI_BF16, BN>(F.g, taddr, row, u.tile, 1, 0); break;
          }
          tc_fence_before();
          named_bar_sync(1, 128);
          if (et == 0) mbar_arrive_cluster(tempty0 + acc * 8);
        }
      }
      TRACE(4, f == 0 && et == 0);
      // cooperative fix-up of the split tiles this pair holds a segment of (at most two: its first and last unit):
      // the tile's 2 x nseg CTAs each sum every segment for an interleaved share of its rows, in segment order
      for (int i = 0; i < nsplit; ++i) {
        const int t = split_tiles[i];
        const int q0 = stream_owner(g.W, g.P, t * g.nk);
        const int nseg = stream_owner(g.W, g.P, t * g.nk + g.nk - 1) - q0 + 1;
        const long long slot0 = (long long)t * g.spt;
        // this CTA's contiguous share of the tile's rows, reduced in batches of B rows (all segments of a batch
        // fit one RBUF buffer and are fetched by bulk copies, double buffered)
        const int workers = 2 * nseg, worker = 2 * (pair - q0) + rank;
        const int r0 = (int)((long long)worker * g.M / workers), r1 = (int)((long long)(worker + 1) * g.M / workers);
        const int B = min(16, RBUF / (nseg * 1024));
        if (et < 32) {
          // every segment's flag (both CTA halves when rows reach the second), polled in parallel by one warp, then
          // one acquire fence
          const int nfl = nseg * (g.M > BM ? 2 : 1);
          const int stride = g.M > BM ? 1 : 2;
          uint32_t ns = 64;
          for (;;) {
            bool ok = true;
            for (int k = lane; k < nfl; k += 32)
              ok &= ld_relaxed_u32(A.flags + (slot0 * 2 + k * stride) * FLAG_STRIDE) == tag;
            if (__all_sync(0xffffffffu, ok)) break;
            __nanosleep(ns);
            ns = ns < 256 ? ns * 2 : 256;
          }
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
        // the folded-norm consumers scale rows by 1/rms: one load chain per row, up front
        if (F.epi == EPI_SILU_MUL || F.epi == EPI_QKV_ROPE)
          for (int rr = r0 + et; rr < r1; rr += 128) s_inv[rr - r0] = F.g.ss_in ? row_inv_rms(F.g, rr) : 1.0f;
        named_bar_sync(2, 128);
        TRACE(5, f == 0 && et == 0 && i == 0);
        TRACE(14, f == 0 && et == 0 && i == 1);
        const float* seg0 = A.ws + slot0 * slot_elems;
        // one batch = nseg x 8 bulk copies (segment j, column chunk c), spread over the lanes of the first warp
        auto issue = [&](int b0, int buf) {
          const int nb = min(B, r1 - b0);
          if (lane == 0) mbar_arrive_expect_tx(&rbar[buf], nseg * 8 * nb * 128);
          __syncwarp();
          uint8_t* dstb = stg + buf * RBUF;
          for (int k = lane; k < nseg * 8; k += 32) {
            const int j = k >> 3, c = k & 7;
            bulk_g2s(dstb + k * B * 128, seg0 + j * slot_elems + ((long long)c * g.M + b0) * 32, nb * 128, &rbar[buf]);
          }
        };
        if (r0 < r1 && et < 32) issue(r0, rb & 1);
        for (int b0 = r0; b0 < r1; b0 += B, ++rb) {
          const int buf = rb & 1;
          if (b0 + B < r1 && et < 32) issue(b0 + B, buf ^ 1);
          const int nb = min(B, r1 - b0);
          // items: (row, quad) with each warp on one 128-column half of a row (RESID's sum of squares)
          const int q = (et & 63);
          const int c4 = q * 4;
          float4 rv[8];
          if (F.epi == EPI_RESID_F32) {  // residual rows in flight before the partials land
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const int rl = (et >> 6) + 2 * k;
              if (rl < nb)
                rv[k] = __ldcg(reinterpret_cast<const float4*>(F.g.resid + (long long)(b0 + rl) * F.g.ldr + t * BN + c4));
            }
          }
          mbar_wait(&rbar[buf], (rb >> 1) & 1);
          TRACE(8 + (b0 - r0) / B, f == 0 && et == 0 && i == 0 && (b0 - r0) / B < 5);
          const uint8_t* rbuf = stg + buf * RBUF;
          auto sum_quad = [&](int rl, int qd) {
            const int row_g = b0 + rl;
            const uint8_t* pq = rbuf + ((qd >> 3) * B + rl) * 128 + (((qd & 7) ^ (row_g & 7)) << 4);
            float4 acc = *reinterpret_cast<const float4*>(pq);
            for (int j = 1; j < nseg; ++j) {
              const float4 v = *reinterpret_cast<const float4*>(pq + j * 8 * B * 128);
              acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
            }
            return acc;
          };
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int rl = (et >> 6) + 2 * k;
            if (rl >= nb) break;  // warp-uniform
            const int row_g = b0 + rl;
            const int col = t * BN + c4;
            switch (F.epi) {
              case EPI_RESID_F32: quad_epi<EPI_RESID_F32>(F.g, row_g, col, sum_quad(rl, q), float4{}, 1.f, rv[k]); break;
              case EPI_SILU_MUL:
                if ((q & 7) < 4)
                  quad_epi<EPI_SILU_MUL>(F.g, row_g, col, sum_quad(rl, q), sum_quad(rl, q + 4), s_inv[row_g - r0], rv[k]);
                break;
              case EPI_QKV_ROPE: {
                const bool lo_half = (q & 31) < 16;
                const bool rot = col < F.g.rope_cols;
                if (!rot || lo_half)
                  quad_epi<EPI_QKV_ROPE>(F.g, row_g, col, sum_quad(rl, q), rot ? sum_quad(rl, q + 16) : float4{},
                                         s_inv[row_g - r0], rv[k]);
                break;
              }
              default: quad_epi<EPI_BF16>(F.g, row_g, col, sum_quad(rl, q), float4{}, 1.f, rv[k]); break;
            }
          }
          named_bar_sync(2, 128);  // every thread is done with this buffer before it is refilled
        }
        TRACE(13 + 2 * i, f == 0 && et == 0 && i < 2);
      }
      TRACE(6, f == 0 && et == 0);
      // this CTA's outputs of phase f are stored: arrive on the grid barrier
      named_bar_sync(1, 128);
      if (et == 0) {
        // one counter serves every phase: a CTA with no work in phase f must not arrive for it before the barrier of
        // phase f - 1 is complete, or its arrival would be counted toward f - 1
        if (f > 0) {
          wait_counter(A.bar, A.bar_base + (unsigned long long)f * gridDim.x);
        }
        fence_proxy_async_global();
        __threadfence();
        TRACE(7, f == 0);
        atomicAdd(A.bar, 1ull);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, 2 * BN);
  }
}

// ------------------------------------------------------------------ host side
int stream_pairs() { return num_sms() / 2; }

// partial slots per tile: every segment of a split tile dumps (0 when no tile is split)
static int slots_per_tile(int N, int K) {
  const int nk = K / BK, ntiles = N / BN;
  const long long W = (long long)nk * ntiles;
  const int P = W < stream_pairs() ? (int)W : stream_pairs();
  int most = 1;
  for (int t = 0; t < ntiles; ++t) {
    const int nseg = stream_owner(W, P, (t + 1) * nk - 1) - stream_owner(W, P, t * nk) + 1;
    most = nseg > most ? nseg : most;
  }
  return most > 1 ? most : 0;
}

size_t stream_ws_bytes(int M, int N, int K) { return (size_t)(N / BN) * slots_per_tile(N, K) * M * BN * sizeof(float); }
size_t stream_flag_count(int N, int K) { return (size_t)(N / BN) * slots_per_tile(N, K) * 2 * FLAG_STRIDE; }

int stream_launch(StreamArgs& a, cudaStream_t stream) {
  if (a.nph <= 0 || a.nph > STREAM_MAX_PHASES) return -3;
  for (int f = 0; f < a.nph; ++f) {
    StreamPhase& p = a.ph[f];
    const GemmArgs& g = p.g;
    if (g.M <= 0 || g.M > 2 * BM || g.N % BN || g.K % BK) return -3;
    p.slots_per_tile = slots_per_tile(g.N, g.K);
    if (p.slots_per_tile * 1024 > RBUF) return -3;  // one row of every segment must fit a fix-up buffer
    if (stream_ws_bytes(g.M, g.N, g.K) > a.ws_bytes || stream_flag_count(g.N, g.K) > a.n_flags) return -3;
  }
  ensure_smem_attr<stream_kernel>(SMEM);
  launch_pdl(stream_kernel, dim3(2 * stream_pairs()), dim3(NT), SMEM, stream, a);
  return cudaGetLastError() == cudaSuccess ? 0 : -4;
}

}  // namespace po

// ------------------------------------------------------------------ C-ABI op (kernel-level parity tests, A/B timing)
#include "../../include/prefillonly.h"
namespace po {
int set_error(int code, const char* fmt, ...);
void keep_pool_memory();
}  // namespace po

extern "C" int po_op_stream_gemm(const void* A, int64_t lda, const void* B1, int64_t ldb1, void* out1, int64_t ldo1,
                                 int32_t M, int32_t N1, int32_t K, const void* B2, int64_t ldb2, void* out2,
                                 int64_t ldo2, int32_t N2, void* stream) {
  using namespace po;
  if (!A || !B1 || !out1 || (B2 && !out2)) return set_error(PO_ERR_ARG, "po_op_stream_gemm: null pointer");
  if (M < 1 || M > 256 || N1 <= 0 || N1 % 256 || K <= 0 || K % 64 || (B2 && (N2 <= 0 || N2 % 256)))
    return set_error(PO_ERR_ARG, "po_op_stream_gemm: need 1 <= M <= 256, N %% 256 == 0, K %% 64 == 0");
  StreamArgs a{};
  a.nph = B2 ? 2 : 1;
  auto phase = [&](StreamPhase& p, const void* x, long long ldx, int k, const void* w, long long ldw, int n, void* o,
                   long long ldo) {
    p.g.M = M; p.g.N = n; p.g.K = k; p.g.out = o; p.g.ldo = ldo;
    p.epi = EPI_BF16;
    return make_tmap_a(&p.a, x, ldx, M, k) || make_tmap_a(&p.b, w, ldw, n, k);
  };
  if (phase(a.ph[0], A, lda, K, B1, ldb1, N1, out1, ldo1) ||
      (B2 && phase(a.ph[1], out1, ldo1, N1, B2, ldb2, N2, out2, ldo2)))
    return set_error(PO_ERR_ARG, "po_op_stream_gemm: tensor-map encode failed (alignment?)");
  // the op keeps one workspace per device, a monotonic barrier counter and a fresh tag per call, like an engine
  struct Ws {
    void* buf = nullptr;
    size_t ws = 0, nf = 0;
    unsigned long long base = 0;
    uint32_t tag = 0;
  };
  static Ws per_dev[64];
  int dev = 0;
  cudaGetDevice(&dev);
  Ws& w = per_dev[dev & 63];
  const size_t need_ws = std::max(stream_ws_bytes(M, N1, K), B2 ? stream_ws_bytes(M, N2, N1) : 0);
  const size_t need_nf = std::max(stream_flag_count(N1, K), B2 ? stream_flag_count(N2, N1) : 0);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (!w.buf || need_ws > w.ws || need_nf > w.nf) {
    if (w.buf) {
      cudaDeviceSynchronize();
      cudaFree(w.buf);
    }
    w.ws = std::max(need_ws, w.ws);
    w.nf = std::max(need_nf, w.nf);
    const size_t fl_off = (w.ws + 255) / 256 * 256, bar_off = fl_off + (w.nf * 4 + 255) / 256 * 256;
    if (cudaMalloc(&w.buf, bar_off + 8) != cudaSuccess || cudaMemset(w.buf, 0, bar_off + 8) != cudaSuccess) {
      w.buf = nullptr;
      return set_error(PO_ERR_CUDA, "po_op_stream_gemm: workspace allocation failed");
    }
    w.base = 0;
    w.tag = 0;
  }
  const size_t fl_off = (w.ws + 255) / 256 * 256, bar_off = fl_off + (w.nf * 4 + 255) / 256 * 256;
  a.ws = static_cast<float*>(w.buf);
  a.ws_bytes = w.ws;
  a.flags = reinterpret_cast<uint32_t*>(static_cast<char*>(w.buf) + fl_off);
  a.n_flags = w.nf;
  a.bar = reinterpret_cast<unsigned long long*>(static_cast<char*>(w.buf) + bar_off);
  a.bar_base = w.base;
  a.tag = ++w.tag;
  const int rc = stream_launch(a, st);
  if (!rc) w.base += (unsigned long long)a.nph * 2 * stream_pairs();
  if (rc) return set_error(PO_ERR_CUDA, "po_op_stream_gemm: launch failed (%d): %s", rc,
                           cudaGetErrorString(cudaGetLastError()));
  return PO_OK;
}

#ifdef STREAM_DBG_TRACE
extern "C" int po_debug_stream_trace(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, po::g_stream_trace, sizeof(unsigned long long) * 148 * 16) == cudaSuccess ? 0 : -1;
}
#endif
