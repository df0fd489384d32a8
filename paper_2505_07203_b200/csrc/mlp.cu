// Fused hybrid-prefill MLP of one layer in one persistent launch (ps/numerics.py:259-274):
//   for each piece p of rows:  act[p % 2] = silu(xg Wg^T) * (xg Wu^T)     (gate/up tiles, SiLU.mul epilogue)
//                              resid[p] += act[p % 2] Wd^T                 (down tiles, residual + next-norm epilogue)
// The [piece, d_ff] intermediate lives in a two-buffer ring that the engine pins in L2 (persisting access-policy
// window, po_init), and the down tiles of piece p run interleaved with the gate/up tiles of piece p + 1 inside the
// same grid, so the intermediate is consumed while it is L2-resident and no launch boundary (tail wave + ramp) sits
// between the two GEMMs of a piece.
//
// Schedule: one tile sequence,  GU(0) | GU(1) + D(0) | GU(2) + D(1) | ... | D(P-1)  with the D tiles spread evenly
// among the GU tiles of a segment, fetched in order by the persistent CTA pairs from an atomic counter (a D tile costs
// 3.5 GU tiles, so a static deal leaves pairs unevenly loaded; measured 17% slower). The leader CTA's producer
// fetches and publishes each tile index through a small shared-memory queue to its MMA thread, its epilogue and the
// peer CTA (distributed shared memory + cluster mbarriers). GU tiles sweep the weight columns outermost (row blocks of the piece fastest, so a weight tile is read once
// per piece); D tiles likewise. Dependencies, all on tiles earlier in the sequence (the earliest unfinished tile never
// waits, so the grid cannot deadlock):
//   * D(p, rb, *) reads act rows of row block rb: the producer waits until all gate/up tiles of (p, rb) have stored
//     (counter gu_done[p][rb], raised by both CTAs of each tile after their stores);
//   * GU(p, *, *) overwrites buffer p % 2: its epilogue waits until every D tile of piece p - 2 has finished
//     (counter d_done[p - 2]).
// Writers: stores, __threadfence, CTA barrier, one relaxed atomicAdd. Readers: acquire load, then
// fence.proxy.async.global before the TMA loads (async proxy) of the act rows. The last CTA to exit zeroes the
// counters for the next launch.
//
// CTA pair layout: as gemm2_kernel (gemm.cu) with 256 x 256 tiles: warp 0 TMA producer, warp 1 MMA issuer (leader,
// tcgen05.mma.cta_group::2 M256 N256 K16), warp 2 TMEM allocator, warps 4..7 epilogue (TMEM lane = row).
#include "gemm.cuh"
#include "gemm_epi.cuh"
#include "mlp.cuh"
#include <algorithm>
#include <cstdlib>

namespace po {

namespace {
constexpr int BK = 64;
constexpr int HALF = 128 * BK * 2;       // 16 KB: 128 rows x 64 bf16
constexpr int STAGE = 2 * HALF;          // A half + B half per CTA
constexpr int STAGES = 6;
constexpr int QD = 8;                    // tile-queue depth (the producer runs up to ~3 tiles ahead of the epilogue)
constexpr int SMEM = STAGES * STAGE + 1024 + 512;
constexpr int NT = 256;

struct Tile {
  bool d;   // down tile (else gate/up)
  int p;    // piece
  int rb;   // 256-row block inside the piece
  int n;    // 256-column weight tile
};

__device__ __forceinline__ int piece_rows(const MlpArgs& a, int p) { return min(a.piece, a.rows - p * a.piece); }
__device__ __forceinline__ int piece_rbs(const MlpArgs& a, int p) { return (piece_rows(a, p) + 255) / 256; }

// Sequence position t -> tile (see the schedule above). Inside segment s (G gate/up tiles of piece s, D down tiles of
// piece s - 1): the first `lead` positions (two rounds of the grid) are gate/up tiles, so piece s - 1's last gate/up
// tiles, fetched just before, have finished when its down tiles come up; the D tiles are then spread evenly over the
// next (G - lead) / 2 gate/up tiles, so they are done well before piece s + 1's gate/up tiles overwrite their buffer;
// the remaining gate/up tiles close the segment.
__device__ __forceinline__ Tile decode(const MlpArgs& a, int t) {
  // segments: 0 = GU(0); s in [1, P) = GU(s) + D(s - 1); P = D(P - 1)
  int s = 0, base = 0;
  for (;;) {
    const int g = s < a.npieces ? piece_rbs(a, s) * a.n_gu : 0;
    const int dd = s > 0 ? piece_rbs(a, s - 1) * a.n_d : 0;
    if (t < base + g + dd) {
      const int j = t - base;
      const int lead = min(g, 2 * a.npairs);
      const int mid = (g - lead) / 2;
      int gi = -1, di = -1;
      if (j < lead) {
        gi = j;
      } else if (j < lead + mid + dd) {
        const int k = j - lead;
        const long long tot = mid + dd;
        const int nd_before = (int)((long long)k * dd / tot);
        if ((int)((long long)(k + 1) * dd / tot) > nd_before)
          di = nd_before;
        else
          gi = lead + k - nd_before;
      } else {
        gi = j - dd;
      }
      Tile tl;
      tl.d = di >= 0;
      tl.p = tl.d ? s - 1 : s;
      const int rbs = piece_rbs(a, tl.p);
      const int idx = tl.d ? di : gi;
      tl.n = idx / rbs;
      tl.rb = idx % rbs;
      return tl;
    }
    base += g + dd;
    ++s;
  }
}

__device__ __forceinline__ int ld_acquire_i32(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// wait on this CTA's mbarrier with cluster-scope acquire: the data it guards was stored by the peer CTA
// (st.shared::cluster before its mbarrier.arrive.release.cluster)
__device__ __forceinline__ void mbar_wait_acq_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void st_cluster_u32(uint32_t cluster_addr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(cluster_addr), "r"(v) : "memory");
}
__device__ __forceinline__ void wait_at_least(const int* p, int target) {
  uint32_t ns = 32;
  while (ld_acquire_i32(p) < target) {
    __nanosleep(ns);
    ns = ns < 512 ? ns * 2 : 512;
  }
}
}  // namespace

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NT, 1)
    mlp2_kernel(const __grid_constant__ CUtensorMap map_xg, const __grid_constant__ CUtensorMap map_wgu,
                const __grid_constant__ CUtensorMap map_act, const __grid_constant__ CUtensorMap map_wd,
                const MlpArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * HALF;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* q_full = tempty_bar + 2;     // [QD] tile index published (leader's producer -> every consumer)
  uint64_t* q_empty = q_full + QD;       // [QD] leader: the slot was read by its 4 consumers
  int* q_tile = reinterpret_cast<int*>(q_empty + QD);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_tile + QD);

  const int warp = warp_id();
  const int lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1;
  const int npairs = gridDim.x >> 1;
  const int nk_gu = a.gu.K / BK, nk_d = a.dn.K / BK;
  int* gu_done = a.cnt;                              // [npieces][max_rbs]
  int* d_done = a.cnt + a.npieces * a.max_rbs;       // [npieces]

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_xg);
    tma_prefetch_desc(&map_wgu);
    tma_prefetch_desc(&map_act);
    tma_prefetch_desc(&map_wd);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 2);
    }
    for (int s = 0; s < QD; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&q_empty[s], 4);  // leader's MMA thread + leader's epilogue + peer's producer + peer's epilogue
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_pair(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();  // xg, the norm sums and the residual rows come from the O-projection launch
  pdl_trigger();
  const uint32_t q_empty0 = mapa_shared(smem_u32(q_empty), 0);
  // tile i of this pair (every role walks the same queue; the consumer releases the slot to the leader)
  auto next_tile = [&](int i, bool release) -> int {
    const int slot = i % QD;
    mbar_wait_acq_cluster(&q_full[slot], (i / QD) & 1);
    const int t = q_tile[slot];
    if (release) mbar_arrive_cluster(q_empty0 + slot * 8);
    return t;
  };

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t full0 = mapa_shared(smem_u32(full_bar), 0);
      int s = 0;
      uint32_t ph = 0;
      const uint32_t q_full_peer = mapa_shared(smem_u32(q_full), 1);
      const uint32_t q_tile_peer = mapa_shared(smem_u32(q_tile), 1);
      for (int i = 0;; ++i) {
        int t;
        if (rank == 0) {
          // fetch the next tile of the sequence and publish it to this CTA's consumers and to the peer
          const int slot = i % QD;
          if (i >= QD) mbar_wait(&q_empty[slot], ((i / QD) - 1) & 1);
          t = atomicAdd(a.next, 1);
          q_tile[slot] = t;
          st_cluster_u32(q_tile_peer + slot * 4, (uint32_t)t);
          mbar_arrive(&q_full[slot]);
          mbar_arrive_cluster(q_full_peer + slot * 8);
        } else {
          t = next_tile(i, true);
        }
        if (t >= a.total) break;
        const Tile tl = decode(a, t);
        const int nk = tl.d ? nk_d : nk_gu;
        int arow;
        if (tl.d) {
          // the act rows of (p, rb) are complete once both CTAs of every gate/up tile of that row block stored them
          wait_at_least(gu_done + tl.p * a.max_rbs + tl.rb, 2 * a.n_gu);
          fence_proxy_async_global();
          arow = (tl.p & 1) * a.piece + tl.rb * 256 + (int)rank * 128;
        } else {
          arow = a.gu.a_row0 + tl.p * a.piece + tl.rb * 256 + (int)rank * 128;
        }
        const CUtensorMap* ma = tl.d ? &map_act : &map_xg;
        const CUtensorMap* mb = tl.d ? &map_wd : &map_wgu;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&empty_bar[s], ph ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&full_bar[s], 2 * STAGE);
          const uint32_t fb = full0 + s * 8;
          tma_load_2d_pair(sB + s * HALF, mb, fb, kb * BK, tl.n * 256 + (int)rank * 128);
          tma_load_2d_pair(sA + s * HALF, ma, fb, kb * BK, arow);
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(256, 256);
      int s = 0;
      uint32_t ph = 0;
      for (int it = 0;; ++it) {
        const int t = next_tile(it, true);
        if (t >= a.total) break;
        const Tile tl = decode(a, t);
        const int nk = tl.d ? nk_d : nk_gu;
        const int acc = it & 1;
        mbar_wait(&tempty_bar[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * 256;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full_bar[s], ph);
          tc_fence_after();
          const uint64_t adesc = sdesc_kmajor_sw128(smem_u32(sA + s * HALF));
          const uint64_t bdesc = sdesc_kmajor_sw128(smem_u32(sB + s * HALF));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) mma_bf16_ss_pair(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0);
          mma_commit_pair(&empty_bar[s], 0x3);
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
        mma_commit_pair(&tfull_bar[acc], 0x3);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    const int wq = warp & 3;
    const int et = threadIdx.x - 128;
    const uint32_t tempty0 = mapa_shared(smem_u32(tempty_bar), 0);
    for (int it = 0;; ++it) {
      const int t = next_tile(it, false);
      named_bar_sync(1, 128);  // every epilogue thread has read the slot
      if (et == 0) mbar_arrive_cluster(q_empty0 + (it % QD) * 8);
      if (t >= a.total) break;
      const Tile tl = decode(a, t);
      const int acc = it & 1;
      const int p0 = tl.p * a.piece;  // first MLP row of the piece
      GemmArgs g = tl.d ? a.dn : a.gu;
      g.M = piece_rows(a, tl.p);
      if (tl.d) {
        g.resid = a.dn.resid + (long long)p0 * a.dn.ldr;
        if (g.xg_out) {
          g.xg_out = a.dn.xg_out + (long long)p0 * a.dn.ldxg;
          g.ss_out = a.dn.ss_out + (long long)p0 * a.dn.ss_nseg;
        }
      } else {
        g.out = static_cast<__nv_bfloat16*>(a.gu.out) + (long long)(tl.p & 1) * a.piece * a.gu.ldo;
        if (g.ss_in) g.ss_in = a.gu.ss_in + (long long)p0 * a.gu.ss_nseg;
        // WAR: buffer p % 2 was last read by the down tiles of piece p - 2
        if (tl.p >= 2) {
          if (et == 0) wait_at_least(d_done + tl.p - 2, 2 * a.n_d * piece_rbs(a, tl.p - 2));
          named_bar_sync(1, 128);
        }
      }
      mbar_wait(&tfull_bar[acc], (it >> 1) & 1);
      tc_fence_after();
      const int row = tl.rb * 256 + (int)rank * 128 + wq * 32 + lane;  // row inside the piece
      const uint32_t taddr = tmem_base + ((uint32_t)(wq * 32) << 16) + acc * 256;
      if (tl.d)
        epilogue_tile<EPI_RESID_F32, 256>(g, taddr, row, tl.n, 1, t);
      else
        epilogue_tile<EPI_SILU_MUL, 256>(g, taddr, row, tl.n, 1, t);
      __threadfence();  // this thread's stores, before the tile's completion count below
      tc_fence_before();
      named_bar_sync(1, 128);
      if (et == 0) {
        mbar_arrive_cluster(tempty0 + acc * 8);
        atomicAdd(tl.d ? d_done + tl.p : gu_done + tl.p * a.max_rbs + tl.rb, 1);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, 512);
  }
  // the last CTA out zeroes the counters (every tile of the launch has completed by then)
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(a.ticket, 1u) == gridDim.x - 1) {
      for (int i = 0; i < a.npieces * (a.max_rbs + 1); ++i) a.cnt[i] = 0;
      *a.next = 0;
      __threadfence();
      *a.ticket = 0;
    }
  }
}

// PO_FUSED_MLP=1 runs each layer's MLP through this kernel. Off by default: on the 20k-token Llama-3.1-8B step it
// measured 61.5k tok/s with the intermediate L2-pinned (chunk 2560: pieces of 1,250 rows) and 62.1k at chunk 8192,
// against 65.7k for the per-chunk launches at chunk 8192, at SM clocks 40-60 MHz lower under the power cap: small
// pieces re-stream the gate/up and down weights once per piece (5.6 GB per layer at 20k tokens, against ~2.4 GB plus
// the 1.15 GB intermediate round trip for 8192-row chunks), and the extra DRAM and L2 traffic costs clock
// (DESIGN.md "MLP intermediate").
bool mlp_fused_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* v = getenv("PO_FUSED_MLP");
    on = (v && v[0] == '1') ? 1 : 0;
  }
  return on == 1;
}

size_t mlp_counter_ints(long long max_rows, int piece) {
  const long long np = (max_rows + piece - 1) / piece;
  const long long rbs = (piece + 255) / 256;
  return (size_t)(np * (rbs + 1));
}

int mlp_launch(const CUtensorMap& map_xg, const CUtensorMap& map_wgu, const CUtensorMap& map_act,
               const CUtensorMap& map_wd, const MlpArgs& in, cudaStream_t stream) {
  if (in.rows <= 0) return 0;
  if (in.gu.N % 256 || in.dn.N % 256 || in.gu.K % BK || in.dn.K % BK || in.piece <= 0 || !in.cnt || !in.ticket ||
      !in.next)
    return -3;
  MlpArgs a = in;
  a.n_gu = a.gu.N / 256;
  a.n_d = a.dn.N / 256;
  a.npieces = (a.rows + a.piece - 1) / a.piece;
  a.max_rbs = (a.piece + 255) / 256;
  a.total = 0;
  for (int p = 0; p < a.npieces; ++p) {
    const int rbs = (std::min(a.piece, a.rows - p * a.piece) + 255) / 256;
    a.total += rbs * (a.n_gu + a.n_d);
  }
  const int npairs = std::min(num_sms() / 2, a.total);
  a.npairs = npairs;
  ensure_smem_attr<mlp2_kernel>(SMEM);
  launch_pdl(mlp2_kernel, dim3(2 * npairs), dim3(NT), SMEM, stream, map_xg, map_wgu, map_act, map_wd, a);
  return cudaGetLastError() == cudaSuccess ? 0 : -4;
}

}  // namespace po
