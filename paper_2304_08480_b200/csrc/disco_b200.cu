// B200-native DisCo contrastive loss: kernels + C ABI (include/disco_b200.h).
//
// Hot path replaced: reference pkg/src/disco/shard.py:98-208 (local_loss_and_grads,
// disco_step).  Per rank n (b = B/N rows), two directions d in {i2t, t2i}:
//   S_d   = t * A_d . C_d^T           A_0 = I_n, C_0 = T_g ; A_1 = T_n, C_1 = I_g
//   ce_d  = lse(S_d rows) - S_d[r, n*b + r]
//   G_d   = softmax(S_d) - onehot     (unscaled, f16)
//   intra : Y_g = G_d . C_d           (own rows; g = image for d = 0, text for d = 1)
//   cross : X_g = G_d'^T . A_d'       (all B rows, sent to the owning rank)
//   d_g   = t * 0.5 / B * (Y_g + sum_over_ranks X_g)
//
// Kernels
//   logits_kernel<FWDE> : tcgen05 bf16 GEMM tiles of S with a fused online (max, sum-exp) +
//                         target epilogue that also stores E = exp2(y - group max) in f16
//                         (canonical shapes); S never hits HBM.  Variants: one launch, H2D
//                         wavefronts, flag-gated persistent (streamed) over waves.
//   logits_kernel<FWD>  : statistics only; logits_kernel<GRAD>: tiles recomputed -> f16 G
//                         (non-canonical shapes).
//   gemm_kernel         : grouped f16 GEMM (K-major or MN-major operands via the UMMA
//                         descriptor major bits; no transposes), E -> G rescaled in shared memory
//                         by transform warps, fp32 tiles into partial / slab buffers or, with the
//                         peer transport, straight into the owning rank's window; static LPT
//                         schedule over CTA pairs.
//   small kernels       : pack, unpack / peer gather-unpack, stats combine, E -> G factors,
//                         presum, owner combine, contribution, loss, peer signal / wait, towers.
// All tensor-core kernels run on CTA pairs (cluster of 2, cta_group::2):
//   TMA (SWIZZLE_128B; each CTA loads its 128 A rows and its 128-column half of
//   B, completion counted on the leader's barrier) -> 6-stage smem ring ->
//   single-thread tcgen05.mma M=256 N=256 K=16 issued by the leader ->
//   double-buffered TMEM accumulators (each CTA holds its 128 rows x 256 cols)
//   -> 8 epilogue warps per CTA (tcgen05.ld 32x32b).  Persistent grid of
//   <= #SM CTAs; a unit of work is owned by a CTA pair.
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <mutex>
#include <string>
#include <unordered_map>
#include <algorithm>
#include <vector>
#include <type_traits>

#include "disco_b200.h"
#include "ptx.cuh"

namespace disco {

// Profiling experiments and ablations (DISCO_DEBUG_FLAGS bits, the symmetric single-rank forward,
// the A-resident forward ring) exist only in builds with -DDISCO_EXPERIMENTS=1
// (python -m paper_2304_08480_b200.build --out ... -D DISCO_EXPERIMENTS=1; tools/ab_kernels.py).
// The default library compiles none of their checks into the kernels.
#ifndef DISCO_EXPERIMENTS
#define DISCO_EXPERIMENTS 0
#endif
constexpr bool XP = DISCO_EXPERIMENTS != 0;

// ------------------------------------------------------------------ tiling
constexpr int BM = 128;      // rows per CTA (the pair covers 256)
constexpr int BN = 256;      // accumulator columns (each CTA loads 128 of the B operand rows)
constexpr int BK = 64;
constexpr int PAIR_M = 2 * BM;
constexpr int A_STAGE_BYTES = BM * BK * 2;        // 16 KiB
constexpr int B_STAGE_BYTES = (BN / 2) * BK * 2;  // 16 KiB (this CTA's half of one 256-column N tile)
constexpr int TILE_RING_BYTES = 192 * 1024;      // operand ring: 6 x 32 KiB (NB=1) or 4 x 48 KiB (NB=2)
// NB = number of 256-column N tiles per unit (2 = "wide": all 512 columns of D, two accumulators);
// NA = A tiles per stage (2: the fused single-rank backward stages both directions' E tiles)
template <int NB, int NA = 1> struct Ring {
  static constexpr int STAGE_BYTES = NA * A_STAGE_BYTES + NB * B_STAGE_BYTES;
  static constexpr int STAGES = TILE_RING_BYTES / STAGE_BYTES;
};
constexpr int STAGES = Ring<1>::STAGES;  // max stage count (barrier arrays)
constexpr int STAGE_BYTES = Ring<1>::STAGE_BYTES;
static_assert(Ring<1>::STAGES == 6 && Ring<2>::STAGES == 4 && Ring<2, 2>::STAGES == 3, "ring geometry");
constexpr int NUM_THREADS = 320;  // warp0 TMA, warp1 MMA, warps2-9 epilogue
constexpr int NUM_EPI_WARPS = 8;
// E-operand GEMMs add 4 transform warps (10-13) that rescale each A stage in smem (E -> G).
constexpr int NUM_XF_WARPS = 4;   // transform warps per group: one 128-row A stage
// Transform groups: group g takes the ring stages s with s % groups == g (build switches; one group
// each by default: a second group measured +1.7% cycles on the wide dual backward, -6% on the
// exchange backward and -2% on the narrow units of D = 768, where it costs 20 bytes of spills).
#ifndef DISCO_XF_GROUPS
#define DISCO_XF_GROUPS 1
#endif
#ifndef DISCO_XF_GROUPS_NARROW
#define DISCO_XF_GROUPS_NARROW 1
#endif
template <int NB>
__host__ __device__ constexpr int xf_groups() { return NB == 1 ? DISCO_XF_GROUPS_NARROW : DISCO_XF_GROUPS; }
constexpr int XF_GROUPS_MAX = DISCO_XF_GROUPS > DISCO_XF_GROUPS_NARROW ? DISCO_XF_GROUPS : DISCO_XF_GROUPS_NARROW;
template <int NB, bool XF>
__host__ __device__ constexpr int gemm_threads() { return XF ? NUM_THREADS + 32 * NUM_XF_WARPS * xf_groups<NB>() : NUM_THREADS; }
constexpr int GROUP_COLS = 64;    // E offset granularity: one exp2 offset per (row, 64-column group)
// The forward stores E = exp2(y - m_g + E_HEADROOM) (m_g: the row's group max without the label),
// values in (0, 2^15].  E-operand GEMMs therefore see scaled operands: the two-GEMM (exchange)
// backward forms 2^15 G, the dual backward 2^14 H (H <= 2); the combines undo the power of two.
constexpr float E_HEADROOM = 15.f;
constexpr float G_EXCHANGE_SCALE = 32768.f;  // 2^E_HEADROOM
constexpr float H_DUAL_LOG2 = 14.f;
constexpr int TMEM_COLS = 512;    // 2 accumulators of 128 lanes x 256 fp32 columns
constexpr float LOG2E = 1.4426950408889634f;
constexpr float LN2 = 0.6931471805599453f;

struct SmemCtl {
  uint64_t full[STAGES];   // leader: TMA bytes of both CTAs landed
  uint64_t empty[STAGES];  // both: MMA done reading the stage (multicast commit)
  uint64_t tfull[2];       // both: accumulator ready (multicast commit)
  uint64_t tempty[2];      // leader: both CTAs' epilogues drained the accumulator
  uint64_t xfull[STAGES];  // leader: both CTAs' transform warps rescaled the stage (E-operand GEMMs)
  uint64_t afull[8];       // leader: resident A slice k of the unit landed (logits kernel, Dp <= 512)
  uint64_t aempty[8];      // both: the unit's last MMA on A slice k retired
  uint32_t tmem_base;
};
// Epilogue staging: 8 warps x STAGING_BUFS x (32 rows x 128 B), swizzled like TMA SWIZZLE_128B.
constexpr int STAGING_TILE = 32 * 128;
constexpr int STAGING_BUFS = 1;
constexpr int STAGING_BYTES = NUM_EPI_WARPS * STAGING_BUFS * STAGING_TILE;
constexpr size_t SMEM_BYTES = 1024 /*align slack*/ + size_t(TILE_RING_BYTES) + STAGING_BYTES + 512;
// Logits kernel with a resident A block (Dp <= 512): A = 8 slices x 16 KiB, then a 4-stage B ring.
constexpr int ARES_SLICES = 8;
#ifndef DISCO_ARES_B_STAGES
#define DISCO_ARES_B_STAGES 4
#endif
constexpr int ARES_B_STAGES = DISCO_ARES_B_STAGES;
static_assert(ARES_SLICES * A_STAGE_BYTES + ARES_B_STAGES * B_STAGE_BYTES <= TILE_RING_BYTES + STAGING_BYTES / 2,
              "A-resident layout");
static_assert(SMEM_BYTES <= 232448, "exceeds the 227 KB per-CTA shared memory limit");
// Dual backward (E-operand GEMMs, xform = 2): per ring stage, the q factors of the stage's 64 K
// columns (256 B) land by bulk copy beside the tiles, after the control block.
constexpr int DUAL_Q_BYTES = 64 * 4;
constexpr size_t SMEM_BYTES_XF = SMEM_BYTES + size_t(STAGES) * DUAL_Q_BYTES;
static_assert(SMEM_BYTES_XF <= 232448, "E-operand GEMM smem");
// A row is fixed up (recomputed exactly, dual_fixup_kernel) when one of its groups' maxima exceeds
// the smallest column LSE of the group by more than this (log2 units): only then can an E entry
// below the f16 normal range (29 binades under m_g) carry >= 2^-13 of a column's softmax mass,
// and only then can the f16 factor a_r + p_r q_c exceed 2^15.
constexpr float DUAL_SAFE_SPAN = 16.f;
static_assert(sizeof(uint64_t) * 46 + 4 <= 512, "control block");

// -------------------------------------------------------- status flag bits
constexpr int FLAG_INPUT_NONFINITE = 1;
constexpr int FLAG_LOSS_NONFINITE = 2;
constexpr int FLAG_GRAD_NONFINITE = 4;
constexpr int FLAG_PEER_TIMEOUT = 8;  // peer transport: a peer's slabs never arrived (wait kernel gave up)
constexpr int FLAG_H2D_TIMEOUT = 16;  // streamed forward: an H2D chunk never landed

struct Status {
  double loss;
  int flags;
  int fix_count;             // dual backward: rows queued for the exact recompute (DISCO_R_FIX)
  double dlogit;             // dL/d(logit scale), disco_b200_logit_scale_grad
  double loss_partial[128];  // loss_partial_kernel scratch (LOSS_BLOCKS)
  // clock probe (CTA 0 of the tensor-core kernels): {SM clock64, globaltimer ns} at entry and exit,
  // [0..3] logits kernel, [4..7] backward GEMM -> the SM clock the kernel actually ran at
  unsigned long long probe[8];
  // drain probe (backward GEMM, epilogue warp 2 of every leader CTA): sum over units of the
  // cycles from "accumulators full" to "accumulators released", and the unit count
  unsigned long long drain[2];
  // streamed forward (host inputs): wave k's rows landed in FEAT once wave_flags[k] >= the step's
  // epoch; written by the copy stream (cuStreamWriteValue32), polled by the logits producers
  unsigned int wave_flags[32];
};

// ----------------------------------------------------------- kernel params
// One direction of the logits GEMM: A rows are the rank's local rows of the
// gathered matrix (row offset rank*b), B rows are all B gathered rows.
struct LogitsParams {
  CUtensorMap a_map[2];  // dir 0: I_g, dir 1: T_g   box {64, 128}
  CUtensorMap b_map[2];  // dir 0: T_g, dir 1: I_g   box {64, 128} (each CTA loads its half of N)
  CUtensorMap g_map[2];  // blocked-G store maps (4-D), box {64, 32, 1, 1}
  CUtensorMap e_map[2];  // FWDE: blocked-E store maps, half slices: box {32, 32, 1, 1}, 64-byte swizzle
  int B, b, Dp, rank;
  int nchunk, chunk_cols, tiles_per_chunk, row_tiles;  // row_tiles counts 256-row pair tiles
  float tl2e;  // t * log2(e)
  // FWD outputs
  float2* stats;   // [2][nchunk][2 column halves][b]
  float* target;   // [2][b]  (log2-domain target logit)
  // GRAD inputs / outputs
  const float* lse2;    // [2][b]
  const float* glabel;  // [2][b]
  __half* G;            // [2][b][ldG] row-major, or blocked (see g_blocked)
  int64_t ldG;
  int g_blocked;        // 1: G stored as [2][b/128][B/128][128][128] (contiguous 32 KiB blocks)
  int debug_flags;      // DISCO_DEBUG_FLAGS (profiling experiments only): bit0 skip G stores
  // FWDE outputs: E = exp2(y - m_g) into the blocked G region, m_g per (dir, 64-column group, row)
  float* mg;            // [2][groups][b]
  int groups;           // B / 64 (GROUP_COLS)
  // wave >= 0 (single rank, H2D-pipelined forward): only the units whose row chunk or column
  // chunk is `wave` and the other index <= wave, i.e. the units that became computable when
  // (stats sub-)chunk `wave` of I and T landed.  rt_per_chunk = 256-row tiles per (sub-)chunk.
  int wave, rt_per_chunk;
  // streamed (wave == -2): one persistent launch over all waves in order; the producers wait for
  // wave_flags[k] >= epoch before loading wave k's tiles
  const unsigned int* wave_flags;
  unsigned int epoch;
  int nwaves;
  unsigned long long timeout_ns;
  int* status_flags;
  unsigned long long* probe;  // Status::probe (may be null)
};

struct GemmProblem {
  CUtensorMap a_map;
  CUtensorMap b_map;
  CUtensorMap out_map;    // 3-D fp32 store map {N, row_div, z}, box {32, 32, 1}
  int tma_store;          // 1: TMA stores through staging smem; 0: direct st.global
  int skip_store;         // profiling experiment (DISCO_DEBUG_FLAGS bit4): drain TMEM, store nothing
  int ablate;             // profiling experiments: bit10 transform warps skip the rescale, bit11 no drain
  // peer transport (N > 1): output rows of destination rank r = row / peer_b are TMA-stored straight
  // into rank r's peer-mapped slab window through peer_map[r] (z = local partial index)
  int peer, peer_b;
  CUtensorMap peer_map[8];
  int paired;             // 1: unit = chunks (2kc, 2kc+1), summed in the epilogue
  int a_blocked;          // 1: A is a blocked G ([rows/128][cols/128][128][128], 4-D map)
  int a_mn_major, b_mn_major;
  int M, N;               // valid output extents
  int m_tiles, n_tiles, k_chunks;  // m tiles of 256 rows (CTA pair), n tiles of 256 columns
  int m_off;              // first m tile (row-block launches cover tiles [m_off, m_off + m_tiles))
  int n_off;              // first output column (split-width launches: [0, 512k) wide, the rest narrow)
  int k_chunk_len;        // elements of K per chunk (multiple of 64 unless k_chunks == 1)
  int k_total;            // total K extent
  int a_k_off, b_k_off;   // added to the K coordinate of MN-major operands
  int a_row_off;          // added to the row coordinate of a K-major A
  float* out;
  int64_t ld_out;         // floats between rows
  int64_t row_div;        // output row r -> (r / row_div) * stride_hi + (r % row_div) * ld_out
  int64_t stride_hi;
  int64_t chunk_stride;   // floats between k-chunk partial outputs
  // E operand (xform = 1): A holds blocked E; the transform warps rescale every A stage to G
  int xform;
  const __half* xscale;   // [groups][xb] exp2(m_g - lse2) of this problem's direction (f16)
  const float* xlabel;    // [xb] label-column value P_label - 1
  int xb;                 // local rows b (pitch of xscale)
  int lab_off;            // rank * b: global column of local row 0's positive pair
  // dual backward (xform = 2, K-major E rows of direction d): the transform warps write
  // H' = 2^14 (G_d + G_d'^T) = E (a_r + p_r q_c) over the rank's own E block, with
  // a_r = exp2(m_g - 1 - lse2_d[r]), p_r = exp2(m_g - 1 - Q_g), q_c = exp2(Q_g - lse2_d'[c]) (< 2^100)
  const float* xmg;       // [groups][xb] group maxima m_g of direction d (f32)
  const float* xlse;      // [xb] lse2 of direction d (this rank's rows)
  const float* xq;        // [B] q_c (bulk-copied per stage; sign -1 under the flip hook)
  const float2* xgm;      // [groups] (Q_g, smallest column lse2 of the group or -inf)
  int* fix_list;          // rows needing the exact recompute: fix_tag + row
  int* fix_count;
  int fix_tag, fix_cap;
};
constexpr int MAX_PROBLEMS = 4;
constexpr int MAX_SCHED_PAIRS = 80;
constexpr int MAX_SCHED_UNITS = 4096;
struct GemmParams {
  GemmProblem prob[MAX_PROBLEMS];
  int nprob;
  int units[MAX_PROBLEMS + 1];  // prefix sums of per-problem unit counts
  // split > 0: problems [0, split) (list A) and [split, nprob) (list B) are interleaved in
  // proportion to their unit counts (Bresenham), so pairs walking the unit sequence with a
  // stride of #pairs see A and B units in different phases (spreads the accumulator drains).
  int split;
  unsigned long long* probe;  // Status::probe + 4 (may be null)
  // Static longest-processing-time schedule (host-computed): pair i runs the unit sequence
  // indices sched[sched_off[i] .. sched_off[i + 1]) in order; sched_n == 0: round-robin.
  int sched_n;
  uint16_t sched_off[MAX_SCHED_PAIRS + 1];
  uint16_t sched[MAX_SCHED_UNITS];
};

// --------------------------------------------------------- shared helpers
// TMA load of one operand stage into this CTA's smem; completion on the leader's barrier.
// Blocked operands (G in [r/128][c/128][128][128] layout) are addressed through a 4-D map:
// K-major: rows = G rows, K = G columns; MN-major: MN = G columns, K = G rows.
__device__ __forceinline__ void load_blocked(const CUtensorMap* map, int mn_major, uint8_t* dst, uint32_t bar,
                                             int mn0, int k0, int rows, uint64_t policy) {
  if (!mn_major) {
    ptx::tma_load_4d_pair(dst, map, bar, k0 & 127, mn0 & 127, k0 >> 7, mn0 >> 7, policy);  // box {64, rows, 1, 1}
  } else {
    for (int j = 0; j < rows / 64; ++j) {
      const int c = mn0 + j * 64;
      ptx::tma_load_4d_pair(dst + j * 8192, map, bar, c & 127, k0 & 127, c >> 7, k0 >> 7, policy);  // {64, 64, 1, 1}
    }
  }
}

__device__ __forceinline__ void load_operand(const CUtensorMap* map, int mn_major, uint8_t* dst, uint32_t bar,
                                             int mn0, int k0, int rows, uint64_t policy) {
  if (!mn_major) {
    ptx::tma_load_2d_pair(dst, map, bar, k0, mn0, policy);  // box {64 (K), rows}
  } else {
    for (int j = 0; j < rows / 64; ++j)  // box {64 (MN), 64 (K)} per 8 KiB atom column
      ptx::tma_load_2d_pair(dst + j * 8192, map, bar, mn0 + j * 64, k0, policy);
  }
}

__device__ __forceinline__ uint64_t operand_desc(uint32_t base, int mn_major, int kk) {
  return mn_major ? ptx::smem_desc_sw128(base + kk * 2048, 8192, 1024)  // 16 K-rows of 128 B per MMA
                  : ptx::smem_desc_sw128(base + kk * 32, 16, 1024);     // 16 K-elements = 32 B per MMA
}

#ifndef DISCO_WAITPROBE
#define DISCO_WAITPROBE 0
#endif
#if DISCO_WAITPROBE
// profiling build only: logits kernel barrier-wait cycles {MMA full, MMA tempty, MMA total, MMA
// threads, epilogue tfull by warp quadrant x4}; backward GEMM {8: MMA operand wait (full/xfull),
// 9: MMA tempty wait, 10: MMA total, 11: MMA threads, 12: transform TMA wait, 13: transform total,
// 14: transform threads}; read by disco_b200_waitprobe
__device__ unsigned long long g_waitprobe[16];
#endif
template <int NSTAGES = STAGES>
struct Pipe {
  uint32_t stage = 0, phase = 0;
  __device__ __forceinline__ void advance() {
    if (++stage == NSTAGES) {
      stage = 0;
      phase ^= 1;
    }
  }
};

__device__ __forceinline__ uint8_t* smem_base(uint8_t* raw) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
}

// Leader-side MMA issue for one unit: nk k-blocks of BK, 4 UMMAs per N tile each.
// NB = 2: the same A stage feeds two N tiles into accumulators d_tmem and d_tmem + BN.
// Called by the whole (leader) MMA warp: barrier waits and descriptor arithmetic are
// warp-uniform (uniform registers), one elected lane issues the UMMAs and the commits.
// Successive K=16 steps advance the descriptor start address by 32 B (K-major) or 2 KiB
// (MN-major), i.e. by 2 or 128 in the descriptor's 16-byte units.
template <int NB, bool XF = false, int RS = Ring<NB>::STAGES, int NA = 1>
__device__ __forceinline__ void mma_blocks(SmemCtl* ctl, uint8_t* tiles, Pipe<RS>& pipe, int nk, int kb0,
                                           uint32_t d_tmem, uint32_t idesc, int a_mn, int b_mn, int j_lo, int j_hi,
                                           bool wait, bool release) {
  const uint64_t a_step = a_mn ? 128 : 2, b_step = b_mn ? 128 : 2;
  for (int kb = 0; kb < nk; ++kb) {
#if DISCO_WAITPROBE
    const long long w0 = clock64();
#endif
    if (wait) ptx::mbar_wait(XF ? &ctl->xfull[pipe.stage] : &ctl->full[pipe.stage], pipe.phase);
#if DISCO_WAITPROBE
    if (wait && (threadIdx.x & 31) == 0) atomicAdd(&g_waitprobe[8], (unsigned long long)(clock64() - w0));
#endif
    ptx::tc_fence_after();
    const uint32_t a_base = ptx::smem_u32(tiles + pipe.stage * Ring<NB, NA>::STAGE_BYTES);
    const uint32_t b_base = a_base + NA * A_STAGE_BYTES;
    const uint64_t ad0 = operand_desc(a_base, a_mn, 0);
    uint64_t bd0[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) bd0[j] = operand_desc(b_base + j * B_STAGE_BYTES, b_mn, 0);
    if (ptx::elect_one()) {
#pragma unroll
      for (int kk = 0; kk < BK / 16; ++kk) {
#pragma unroll
        for (int j = 0; j < NB; ++j)
          if (j >= j_lo && j < j_hi)
            ptx::umma_f16_pair(d_tmem + j * BN, ad0 + kk * a_step, bd0[j] + kk * b_step, idesc, ((kb0 + kb) | kk) != 0);
      }
      if (release) ptx::umma_commit_pair(&ctl->empty[pipe.stage], 0x3);  // both CTAs' smem slots free
    }
    __syncwarp();
    pipe.advance();
  }
}

template <int NB, bool XF = false, int RS = Ring<NB>::STAGES, int NA = 1>
__device__ __forceinline__ void mma_tile(SmemCtl* ctl, uint8_t* tiles, Pipe<RS>& pipe, int nk,
                                         uint32_t d_tmem, uint32_t idesc, int a_mn, int b_mn) {
  mma_blocks<NB, XF, RS, NA>(ctl, tiles, pipe, nk, 0, d_tmem, idesc, a_mn, b_mn, 0, NB, true, true);
}

// Producer side of one k-block: wait for the slot, arm the leader's barrier, load.
// LOCAL (E-operand GEMMs): each CTA counts its own bytes on its own barrier, which its
// transform warps wait on; otherwise the leader's barrier counts both CTAs' bytes.
template <int NB, bool LOCAL = false, int RS = Ring<NB>::STAGES, int NA = 1>
__device__ __forceinline__ uint8_t* producer_acquire(SmemCtl* ctl, uint8_t* tiles, Pipe<RS>& pipe,
                                                     bool leader, uint32_t& bar, uint32_t crank = 0,
                                                     uint32_t extra_bytes = 0) {
  ptx::mbar_wait(&ctl->empty[pipe.stage], pipe.phase ^ 1);
  if (LOCAL) {
    ptx::mbar_arrive_expect_tx(&ctl->full[pipe.stage], Ring<NB, NA>::STAGE_BYTES + extra_bytes);
    bar = ptx::map_to_rank(&ctl->full[pipe.stage], crank);
  } else {
    if (leader) ptx::mbar_arrive_expect_tx(&ctl->full[pipe.stage], 2 * Ring<NB, NA>::STAGE_BYTES);
    bar = ptx::map_to_rank(&ctl->full[pipe.stage], 0);
  }
  return tiles + pipe.stage * Ring<NB, NA>::STAGE_BYTES;
}

// E -> 2^15 G on one 128-byte smem row (64 f16 of one G row i, G columns [j0, j0 + 64)) of a
// SWIZZLE_128B operand stage: multiply by the f16 factor sc = exp2(m_g - lse2) (HMUL2; E carries
// the 2^15 headroom); the label column (j == lab) gets 2^15 (P_label - 1).  Logical 16-byte chunk c sits at physical c ^ (row & 7);
// walking physical chunks in lane order keeps the 8 rows of a quarter-warp on distinct banks.
__device__ __forceinline__ void xform_row(uint32_t rowp, int sw, __half sc, int lab_rel, float glab) {
  const __half2 s2 = __half2half2(sc);  // packed f16 multiply: 4 HMUL2 per 16-byte chunk
  uint4 x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = ptx::lds128(rowp + ((c ^ sw) << 4));
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    __half2* h = reinterpret_cast<__half2*>(&x[c]);
#pragma unroll
    for (int k = 0; k < 4; ++k) h[k] = __hmul2(h[k], s2);
    ptx::sts128(rowp + ((c ^ sw) << 4), x[c]);
  }
  if (unsigned(lab_rel) < 64u)
    ptx::sts16(rowp + (((lab_rel >> 3) ^ sw) << 4) + (lab_rel & 7) * 2,
               __half_as_ushort(__float2half_rn(glab * G_EXCHANGE_SCALE)));
}

// Clock probe: CTA 0, thread 0 records {clock64, globaltimer} at slot [at, at + 1].
__device__ __forceinline__ void probe_mark(unsigned long long* probe, int at) {
  // ctaid / tid re-read (volatile) so the entry and exit marks share no live predicate (it spilled)
  unsigned bid, tid;
  asm volatile("mov.u32 %0, %%ctaid.x;" : "=r"(bid));
  asm volatile("mov.u32 %0, %%tid.x;" : "=r"(tid));
  if (probe && bid == 0 && tid == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    probe[at] = clock64();
    probe[at + 1] = t;
  }
}

__device__ __forceinline__ void kernel_prologue(SmemCtl* ctl, int warp, int lane, int epi_warps = NUM_EPI_WARPS) {
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {  // the NB=2 ring uses the first Ring<2>::STAGES
      ptx::mbar_init(&ctl->full[s], 1);
      ptx::mbar_init(&ctl->empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&ctl->tfull[i], 1);
      ptx::mbar_init(&ctl->tempty[i], 2 * epi_warps);  // every epilogue warp of both CTAs
    }
    for (int s = 0; s < STAGES; ++s) ptx::mbar_init(&ctl->xfull[s], 2 * NUM_XF_WARPS);
    for (int s = 0; s < ARES_SLICES; ++s) {
      ptx::mbar_init(&ctl->afull[s], 1);
      ptx::mbar_init(&ctl->aempty[s], 1);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 1) {
    ptx::tmem_alloc_pair(&ctl->tmem_base, TMEM_COLS);
    ptx::tmem_relinquish_pair();
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
}

__device__ __forceinline__ void kernel_epilogue(SmemCtl* ctl, int warp) {
  ptx::tc_fence_before();
  ptx::cluster_sync();  // neither CTA leaves while the pair's MMAs / arrivals may touch it
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_pair(ctl->tmem_base, TMEM_COLS);
  }
}

// Epilogue warp releases an accumulator buffer on the leader's barrier.
__device__ __forceinline__ void release_accumulator(SmemCtl* ctl, int buf, int lane) {
  ptx::tc_fence_before();
  __syncwarp();
  if (lane == 0) ptx::mbar_arrive_cluster(ptx::map_to_rank(&ctl->tempty[buf], 0));
}

// =====================================================================
// logits kernel: S tiles for both directions, CTA pair = 256 local rows.
//   FWD : unit = (dir, row pair tile, column chunk); tiles = column tiles of
//         the chunk; each epilogue thread keeps an online (max, sum-exp) for
//         its row over its column half of every tile of the unit.
//   GRAD: unit = (dir, row pair tile, column chunk, column tile); writes G.
// Both kinds walk identical tiles (same column origin and K order), so the
// recomputed S in GRAD is bit-identical to the forward S.
// Epilogue: 8 warps; warp w reads TMEM lane quadrant (w % 4) and column half
// (w - 2) / 4 of this CTA's 128 x 256 accumulator.
// =====================================================================
// FWDE (canonical shapes): the forward epilogue also stores E = exp2(y - m_g), f16, where
// m_g is the max of the row over its 64-column group, plus m_g itself.  The backward
// GEMMs turn E into G = E * exp2(m_g - lse2) (label column: P_label - 1) in shared memory,
// so the logits are never recomputed.
enum { KIND_FWD = 0, KIND_GRAD = 1, KIND_FWDE = 2 };

// ARES: the unit's A block (its 256 local rows x Dp, Dp <= 512) stays resident in smem for all
// column tiles of the unit and only B streams through a 4-stage ring; A slice k of the next unit
// is reloaded as soon as the unit's last tile has consumed it.  Halves the TMA fill traffic and
// cuts smem traffic per MMA from ~128 to ~96 B/clk/SM (the narrow 256-column tile is smem-bound).
#ifndef DISCO_FWD_STAGES
#define DISCO_FWD_STAGES 5  // 5 x 32 KiB: same-process A/B 2-3% fewer cycles than 6, 4 and 3 much slower
#endif
#ifndef DISCO_ESTORE_POLICY
#define DISCO_ESTORE_POLICY ptx::kEvictFirst  // L2 policy of the forward's E stores
#endif
#ifndef DISCO_FWD_NOESTORE
#define DISCO_FWD_NOESTORE 0
#endif
#ifndef DISCO_FWDE_WARPS
#define DISCO_FWDE_WARPS 8
#endif
#ifndef DISCO_FWD_EBUFS
#define DISCO_FWD_EBUFS 2
#endif
constexpr int FWD_STAGES = DISCO_FWD_STAGES;  // forward operand ring stages (32 KiB each)
constexpr int FWD_EBUFS = DISCO_FWD_EBUFS;    // forward E staging half-buffers per epilogue warp (2 KiB each)
static_assert(FWD_STAGES * STAGE_BYTES + NUM_EPI_WARPS * FWD_EBUFS * (STAGING_TILE / 2) <= TILE_RING_BYTES + STAGING_BYTES,
              "forward smem layout");
// FWDE epilogue width: 16 warps (4 per SM sub-partition, each draining a 64-column quarter of the
// 256-column accumulator) instead of 8 (128-column halves).  The E epilogue is latency-bound
// (dependent FFMA -> MUFU -> FADD chains, TMEM loads, staging), so twice the warps per scheduler
// keep the MUFU and FMA pipes fed while the MMA of the next tile runs.  Costs one operand stage
// (5 x 32 KiB ring, measured neutral) for the 16 warps' staging buffers.
#ifndef DISCO_FWDE_PACKED
#define DISCO_FWDE_PACKED 0
#endif
constexpr int FWDE_EPI = DISCO_FWDE_WARPS;
// y = S t log2(e) - m_g and the running sums as packed FP32 pairs (FFMA2 / FADD2) or scalar
__device__ __forceinline__ float2 fwde_y(float a, float b, float2 tl2, float2 nmg) {
#if DISCO_FWDE_PACKED
  return ptx::ffma2(make_float2(a, b), tl2, nmg);
#else
  return make_float2(fmaf(a, tl2.x, nmg.x), fmaf(b, tl2.y, nmg.y));
#endif
}
__device__ __forceinline__ float2 fwde_acc(float2 s, float e0, float e1) {
#if DISCO_FWDE_PACKED
  return ptx::fadd2(s, make_float2(e0, e1));
#else
  return make_float2(s.x + e0, s.y + e1);
#endif
}
constexpr int FWDE_STAGES = FWDE_EPI == 16 ? 5 : FWD_STAGES;
static_assert(FWDE_EPI == 8 || FWDE_EPI == 16, "FWDE epilogue warps");
static_assert(FWDE_STAGES * STAGE_BYTES + FWDE_EPI * FWD_EBUFS * (STAGING_TILE / 2) <= TILE_RING_BYTES + STAGING_BYTES,
              "FWDE smem layout");
static_assert(!XP || ARES_SLICES * A_STAGE_BYTES + ARES_B_STAGES * B_STAGE_BYTES +
                             NUM_EPI_WARPS * FWD_EBUFS * (STAGING_TILE / 2) <= TILE_RING_BYTES + STAGING_BYTES,
              "A-resident smem layout");
template <int KIND, bool ARES>
__host__ __device__ constexpr int logits_epi() { return (KIND == KIND_FWDE && !ARES) ? FWDE_EPI : NUM_EPI_WARPS; }
template <int KIND, bool ARES>
__host__ __device__ constexpr int logits_threads() { return 64 + 32 * logits_epi<KIND, ARES>(); }
// statistics parts per (row, sub-chunk) the FWDE / FWD kernels write: one per epilogue column part
constexpr int FWDE_PARTS = FWDE_EPI / 4;

template <int KIND, bool ARES>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(logits_threads<KIND, ARES>(), 1)
    logits_kernel(const __grid_constant__ LogitsParams p) {
  constexpr int EPI = logits_epi<KIND, ARES>();          // epilogue warps
  constexpr int NPARTS = EPI / 4;                        // column parts of a 256-column tile
  constexpr int PART_COLS = BN / NPARTS;                 // columns per epilogue warp and tile
  constexpr int LRS = EPI == 16 ? FWDE_STAGES : FWD_STAGES;  // operand ring stages
  constexpr int EBUFS = FWD_EBUFS;                           // E staging half-buffers per warp
  constexpr int NDIR = 2;                                    // directions walked by the units
  extern __shared__ uint8_t smem_raw[];
  uint8_t* tiles = smem_base(smem_raw);
  uint8_t* staging = tiles + (ARES ? ARES_SLICES * A_STAGE_BYTES + ARES_B_STAGES * B_STAGE_BYTES : LRS * STAGE_BYTES);
  SmemCtl* ctl = reinterpret_cast<SmemCtl*>(tiles + TILE_RING_BYTES + STAGING_BYTES);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int crank = int(ptx::cluster_ctarank());
  const bool leader = crank == 0;
  const int pair = blockIdx.x / 2, npairs = gridDim.x / 2;

  if (warp == 0 && lane == 0) {
    for (int d = 0; d < 2; ++d) {
      ptx::prefetch_tmap(&p.a_map[d]);
      ptx::prefetch_tmap(&p.b_map[d]);
    }
  }
  probe_mark(p.probe, 0);
  kernel_prologue(ctl, warp, lane, EPI);

  constexpr bool CHUNK_UNITS = KIND != KIND_GRAD;  // unit = all tiles of one column chunk
  const int wave = CHUNK_UNITS ? p.wave : -1;
  // streamed modes: -2 = H2D row/column wavefront (single rank), -3 = peer column waves (N > 1:
  // wave k = the columns of source rank (rank + k) % N, all local row tiles)
  const bool streamed = wave == -2 || wave == -3;
  const bool colwaves = wave == -3;
  const int spr = colwaves ? p.nchunk / p.nwaves : 1;          // sub-chunks per source rank
  const int per_cwave = 2 * p.row_tiles * spr;                  // units per column wave
  const int per_dir = wave >= 0 ? p.rt_per_chunk * (2 * wave + 1)
                                : p.row_tiles * p.nchunk * (CHUNK_UNITS ? 1 : p.tiles_per_chunk);
  const int num_units = colwaves ? per_cwave * p.nwaves
                                 : streamed ? NDIR * p.rt_per_chunk * p.nwaves * p.nwaves : NDIR * per_dir;
  // -2: unit u belongs to wave k with 2 R k^2 <= u < 2 R (k+1)^2 (wave k holds 2 R (2k+1));
  auto wave_of = [&](int u) {
    if (colwaves) return u / per_cwave;
    int k = int(sqrtf(float(u) / float(NDIR * p.rt_per_chunk)));
    while (k > 0 && NDIR * p.rt_per_chunk * k * k > u) --k;
    while (NDIR * p.rt_per_chunk * (k + 1) * (k + 1) <= u) ++k;
    return k;
  };
  const int tiles_per_unit = CHUNK_UNITS ? p.tiles_per_chunk : 1;
  const int nk = p.Dp / BK;

  auto decode = [&](int u, int& dir, int& rt, int& ch, int& t0) {
    if (colwaves) {
      const int k = u / per_cwave;
      int rem = u - k * per_cwave;
      dir = rem / (p.row_tiles * spr);
      rem -= dir * p.row_tiles * spr;
      rt = rem / spr;
      ch = ((p.rank + k) % p.nwaves) * spr + rem % spr;
      t0 = 0;
      return;
    }
    int wv = wave, pd = per_dir;
    if (streamed) {
      wv = wave_of(u);
      u -= NDIR * p.rt_per_chunk * wv * wv;
      pd = p.rt_per_chunk * (2 * wv + 1);
    }
    dir = u / pd;
    int rem = u - dir * pd;
    if (wv >= 0) {  // new row tiles x chunks [0, wave], then old row tiles x chunk `wave`
      const int fresh = p.rt_per_chunk * (wv + 1);
      if (rem < fresh) {
        rt = wv * p.rt_per_chunk + rem / (wv + 1);
        ch = rem % (wv + 1);
      } else {
        rt = rem - fresh;
        ch = wv;
      }
      t0 = 0;
    } else if (CHUNK_UNITS) {
      rt = rem / p.nchunk;
      ch = rem - rt * p.nchunk;
      t0 = 0;
    } else {
      const int per_rt = p.nchunk * p.tiles_per_chunk;
      rt = rem / per_rt;
      rem -= rt * per_rt;
      ch = rem / p.tiles_per_chunk;
      t0 = rem - ch * p.tiles_per_chunk;
    }
  };

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer (both CTAs)
      Pipe<LRS> pipe;
      if constexpr (ARES) {
        Pipe<ARES_B_STAGES> bp;
        uint8_t* bring = tiles + ARES_SLICES * A_STAGE_BYTES;
        uint32_t uphase = 0;
        for (int u = pair; u < num_units; u += npairs, uphase ^= 1) {
          int dir, rt, ch, t0;
          decode(u, dir, rt, ch, t0);
          const int a_row = p.rank * p.b + rt * PAIR_M + crank * BM;
          for (int ti = 0; ti < tiles_per_unit; ++ti) {
            const int col0 = ch * p.chunk_cols + (t0 + ti) * BN + crank * (BN / 2);
            for (int kb = 0; kb < nk; ++kb) {
              if (ti == 0) {  // this unit's A slice kb, once the previous unit released it
                ptx::mbar_wait(&ctl->aempty[kb], uphase ^ 1);
                if (leader) ptx::mbar_arrive_expect_tx(&ctl->afull[kb], 2 * A_STAGE_BYTES);
                ptx::tma_load_2d_pair(tiles + kb * A_STAGE_BYTES, &p.a_map[dir], ptx::map_to_rank(&ctl->afull[kb], 0),
                                      kb * BK, a_row, ptx::kEvictLast);
              }
              ptx::mbar_wait(&ctl->empty[bp.stage], bp.phase ^ 1);
              if (leader) ptx::mbar_arrive_expect_tx(&ctl->full[bp.stage], 2 * B_STAGE_BYTES);
              ptx::tma_load_2d_pair(bring + bp.stage * B_STAGE_BYTES, &p.b_map[dir],
                                    ptx::map_to_rank(&ctl->full[bp.stage], 0), kb * BK, col0, ptx::kEvictLast);
              bp.advance();
            }
          }
        }
      } else {
        unsigned int landed = 0;  // streamed: waves known to have landed
        for (int u = pair; u < num_units; u += npairs) {
          int dir, rt, ch, t0;
          decode(u, dir, rt, ch, t0);
          if (streamed) {
            const int k = wave_of(u);
            if (k >= int(landed)) {
              unsigned long long t_start;
              asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
              while (true) {
                unsigned int v;
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p.wave_flags + k) : "memory");
                if (int(v - p.epoch) >= 0) break;  // epoch-relative: wraps safely
                unsigned long long t_now;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_now));
                if (t_now - t_start > p.timeout_ns) {  // never hang: flag it, compute garbage, host raises
                  atomicOr(p.status_flags, FLAG_H2D_TIMEOUT);
                  break;
                }
                __nanosleep(128);
              }
              asm volatile("fence.proxy.async.global;" ::: "memory");  // the TMA loads below see the rows
              landed = unsigned(k) + 1;
            }
          }
          const int a_row = p.rank * p.b + rt * PAIR_M + crank * BM;
          for (int ti = 0; ti < tiles_per_unit; ++ti) {
            const int col0 = ch * p.chunk_cols + (t0 + ti) * BN + crank * (BN / 2);
            for (int kb = 0; kb < nk; ++kb) {
              uint32_t bar;
              uint8_t* st = producer_acquire<1, false, LRS>(ctl, tiles, pipe, leader, bar);
              ptx::tma_load_2d_pair(st, &p.a_map[dir], bar, kb * BK, a_row, ptx::kEvictLast);
              ptx::tma_load_2d_pair(st + A_STAGE_BYTES, &p.b_map[dir], bar, kb * BK, col0, ptx::kEvictLast);
              pipe.advance();
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {  // ---------------- MMA issuer (leader CTA, whole warp; one elected lane issues)
      constexpr uint32_t idesc = ptx::instr_desc_f16(PAIR_M, BN, 1, 1, 0, 0);  // bf16 x bf16, both K-major
      Pipe<LRS> pipe;
      Pipe<ARES_B_STAGES> bp;
      uint8_t* bring = tiles + ARES_SLICES * A_STAGE_BYTES;
      uint32_t it = 0, uphase = 0;
#if DISCO_WAITPROBE
      long long wp_full = 0, wp_tempty = 0;
      const long long wp_t0 = clock64();
#endif
      for (int u = pair; u < num_units; u += npairs, uphase ^= 1) {
        for (int ti = 0; ti < tiles_per_unit; ++ti, ++it) {
          const uint32_t buf = it & 1, use = it >> 1;
#if DISCO_WAITPROBE
          const long long w1 = clock64();
#endif
          ptx::mbar_wait(&ctl->tempty[buf], (use & 1) ^ 1);
#if DISCO_WAITPROBE
          wp_tempty += clock64() - w1;
#endif
          ptx::tc_fence_after();
          const uint32_t d_tmem = ctl->tmem_base + buf * BN;
          if constexpr (ARES) {
            for (int kb = 0; kb < nk; ++kb) {
              if (ti == 0) ptx::mbar_wait(&ctl->afull[kb], uphase);
              ptx::mbar_wait(&ctl->full[bp.stage], bp.phase);
              ptx::tc_fence_after();
              const uint64_t ad0 = operand_desc(ptx::smem_u32(tiles + kb * A_STAGE_BYTES), 0, 0);
              const uint64_t bd0 = operand_desc(ptx::smem_u32(bring + bp.stage * B_STAGE_BYTES), 0, 0);
              if (ptx::elect_one()) {
#pragma unroll
                for (int kk = 0; kk < BK / 16; ++kk)
                  ptx::umma_f16_pair(d_tmem, ad0 + 2 * kk, bd0 + 2 * kk, idesc, (kb | kk) != 0);
                ptx::umma_commit_pair(&ctl->empty[bp.stage], 0x3);
                if (ti == tiles_per_unit - 1) ptx::umma_commit_pair(&ctl->aempty[kb], 0x3);
              }
              __syncwarp();
              bp.advance();
            }
          } else {
#if DISCO_WAITPROBE
            for (int kb = 0; kb < nk; ++kb) {
              const long long w0 = clock64();
              ptx::mbar_wait(&ctl->full[pipe.stage], pipe.phase);
              wp_full += clock64() - w0;
              mma_blocks<1, false, LRS>(ctl, tiles, pipe, 1, kb, d_tmem, idesc, 0, 0, 0, 1, false, true);
            }
#else
            mma_tile<1, false, LRS>(ctl, tiles, pipe, nk, d_tmem, idesc, 0, 0);
#endif
          }
          if (ptx::elect_one()) ptx::umma_commit_pair(&ctl->tfull[buf], 0x3);
          __syncwarp();
        }
      }
#if DISCO_WAITPROBE
      if (lane == 0) {
        atomicAdd(&g_waitprobe[0], (unsigned long long)wp_full);
        atomicAdd(&g_waitprobe[1], (unsigned long long)wp_tempty);
        atomicAdd(&g_waitprobe[2], (unsigned long long)(clock64() - wp_t0));
        atomicAdd(&g_waitprobe[3], 1ull);
      }
#endif
    }
  } else {  // ---------------------------- epilogue warps 2..(EPI + 1)
    const int ew = warp - 2;
    const int quad = warp & 3;   // TMEM lane quadrant (fixed by the warp's position in its warpgroup)
    const int cpart = ew >> 2;   // column part of the 256-wide tile (PART_COLS columns)
    const int r_in_tile = crank * BM + quad * 32 + lane;
    uint8_t* tile = staging + ew * EBUFS * (STAGING_TILE / 2);
    uint32_t it = 0, gslice = 0;
    // FWDE E-store pipeline state: one pending (written, not yet stored) 32 x 32 half slice
    bool epend = false;
    int ebuf = 0, epend_buf = 0, epend_cb = 0, epend_rb = 0, epend_dir = 0;
    auto e_flush = [&]() {
      if (!epend) return;
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        if (epend_rb < p.b && !DISCO_FWD_NOESTORE)  // (profiling build: E stores off)
          ptx::tma_store_4d(&p.e_map[epend_dir], tile + epend_buf * (STAGING_TILE / 2), epend_cb & 127,
                            epend_rb & 127, epend_cb >> 7, epend_rb >> 7, DISCO_ESTORE_POLICY);
        ptx::bulk_commit();
      }
      epend = false;
    };
    // Stage one 32 x 32 half slice (written by `write` into a free staging half-buffer) as the new
    // pending store at (column cb, row rb) of direction d's E; the previous pending one is issued.
    auto e_push = [&](auto&& write, int cb, int rb, int d) {
      e_flush();  // fence + store the pending half (its STS completed during this half's math)
      uint8_t* hb = tile + ebuf * (STAGING_TILE / 2);
      if (lane == 0) ptx::bulk_wait_read<EBUFS - 1>();  // this buffer's previous store has read smem
      __syncwarp();
      write(hb);
      epend = true;
      epend_buf = ebuf;
      epend_cb = cb;
      epend_rb = rb;
      epend_dir = d;
      ebuf = ebuf + 1 == EBUFS ? 0 : ebuf + 1;
    };
    for (int u = pair; u < num_units; u += npairs) {
      int dir, rt, ch, t0;
      decode(u, dir, rt, ch, t0);
      const int row = rt * PAIR_M + r_in_tile;    // local row
      const bool row_ok = row < p.b;
      const int label = p.rank * p.b + row;        // global column of the positive pair
      const int chunk_lo = ch * p.chunk_cols;
      const int chunk_hi = min(chunk_lo + p.chunk_cols, p.B);
      float m2 = -INFINITY, l = 0.f, yt = 0.f;
      bool has_t = false;
      float lse2 = 0.f, gl = 0.f;
      __half* grow = nullptr;
      if (KIND == KIND_GRAD && row_ok) {
        lse2 = p.lse2[dir * p.b + row];
        gl = p.glabel[dir * p.b + row];
        grow = p.G + (int64_t(dir) * p.b + row) * p.ldG;
      }
      for (int ti = 0; ti < tiles_per_unit; ++ti, ++it) {
        const uint32_t buf = it & 1, use = it >> 1;
#if DISCO_WAITPROBE
        const long long w2 = clock64();
#endif
        ptx::mbar_wait(&ctl->tfull[buf], use & 1);
#if DISCO_WAITPROBE
        if (lane == 0) atomicAdd(&g_waitprobe[4 + (ew & 3)], (unsigned long long)(clock64() - w2));
#endif
        ptx::tc_fence_after();
        const int col0 = chunk_lo + (t0 + ti) * BN + cpart * PART_COLS;
        const uint32_t taddr = ctl->tmem_base + (uint32_t(quad * 32) << 16) + buf * BN + cpart * PART_COLS;
        if (KIND == KIND_FWD) {
#pragma unroll 1
          for (int j = 0; j < PART_COLS / 32; ++j) {
            const int cb = col0 + j * 32;
            if (cb >= chunk_hi) break;  // warp-uniform
            float v[32];
            ptx::tmem_ld32(taddr + j * 32, v);
            const int li = label - cb;
            const bool has_label = unsigned(li) < 32u && label < chunk_hi;
            if (cb + 32 <= chunk_hi && !has_label) {
              // fast path (all but one group per row): no masking, no label handling.
              float cm = v[0];
#pragma unroll
              for (int i = 1; i < 32; ++i) cm = fmaxf(cm, v[i]);
              const float mnew = fmaxf(m2, cm * p.tl2e);
              float s0 = 0.f, s1 = 0.f;
#pragma unroll
              for (int i = 0; i < 32; i += 2) {
                s0 += ptx::ex2(fmaf(v[i], p.tl2e, -mnew));
                s1 += ptx::ex2(fmaf(v[i + 1], p.tl2e, -mnew));
              }
              l = l * ptx::ex2(m2 - mnew) + (s0 + s1);
              m2 = mnew;
            } else {
              // edge / label group: mask columns past the chunk, keep the label term out of l.
              float cm = -INFINITY;
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                const bool ok = cb + i < chunk_hi;
                cm = ok ? fmaxf(cm, v[i]) : cm;
                if (i == li && has_label) {
                  yt = v[i] * p.tl2e;
                  has_t = true;
                }
              }
              const float mnew = fmaxf(m2, cm * p.tl2e);
              float s = 0.f;
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                const float e = ptx::ex2(fmaf(v[i], p.tl2e, -mnew));
                s += (cb + i < chunk_hi && i != li) ? e : 0.f;
              }
              l = l * ptx::ex2(m2 - mnew) + s;
              m2 = mnew;
            }
          }
        } else if (KIND == KIND_FWDE) {
          // canonical chunks: this warp's PART_COLS columns are entirely inside or past the chunk.
          // One TMEM pass (a second pass would pace the tile at the TMEM read rate): each
          // 64-column group is loaded once (both 32-column halves under one tcgen05.wait::ld), its
          // max taken in registers, then E = exp2(y - m_g) packed to f16 and stored as two 32 x 32
          // half slices.  y = S t log2(e) - m_g and the two running sums use packed FP32 pairs
          // (FFMA2 / FADD2: bit-identical to the scalar fmaf / add, half the issue slots).
          constexpr int NJ = PART_COLS / 64;
          if (col0 < chunk_hi) {  // warp-uniform
            const int li = label - col0;  // label column relative to this warp's columns
            const float2 tl2 = make_float2(p.tl2e, p.tl2e);
            uint32_t ra[32], rb[32];  // both halves of a slice under one tcgen05.wait::ld
            ptx::tmem_ld32_async(taddr, ra);
            ptx::tmem_ld32_async(taddr + 32, rb);
            ptx::tmem_wait_ld_dep(ra, rb);
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
              float va[32], vb[32];
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                va[i] = __uint_as_float(ra[i]);
                vb[i] = __uint_as_float(rb[i]);
              }
              if (j + 1 < NJ) {  // the next slice's TMEM loads fly while this one is computed
                ptx::tmem_ld32_async(taddr + 64 * (j + 1), ra);
                ptx::tmem_ld32_async(taddr + 64 * (j + 1) + 32, rb);
              }
              // The label column leaves the group max, the sum and E: its logit goes to yt and the
              // element becomes -inf (so E = 0 there).  li - 64 j = lane + 32 m (labels and columns
              // are 32-aligned), so "this group holds the warp's labels" is warp-uniform and lane
              // L's label is element L of half m.
              const int lj = li - j * 64;
              if (unsigned(lj) < 32u) {
#pragma unroll
                for (int i = 0; i < 32; ++i)
                  if (i == lane) {
                    yt = va[i] * p.tl2e;
                    va[i] = -INFINITY;
                  }
                has_t = true;
              } else if (unsigned(lj - 32) < 32u) {
#pragma unroll
                for (int i = 0; i < 32; ++i)
                  if (i == lane) {
                    yt = vb[i] * p.tl2e;
                    vb[i] = -INFINITY;
                  }
                has_t = true;
              }
              float mx[32];  // max over the 64 columns as a depth-6 tree
#pragma unroll
              for (int i = 0; i < 32; ++i) mx[i] = fmaxf(va[i], vb[i]);
#pragma unroll
              for (int w = 16; w >= 1; w >>= 1)
#pragma unroll
                for (int i = 0; i < w; ++i) mx[i] = fmaxf(mx[i], mx[i + w]);
              const float cm = mx[0];
              const float mg = cm * p.tl2e;  // group max of y, label excluded
              // E = exp2(y - mg + E_HEADROOM) in (0, 2^15]: the headroom keeps entries down to 29
              // binades below the group max normal in f16, which the dual backward's column term
              // needs (it rescales the row-offset E by the column statistics)
              const float2 nmg = make_float2(E_HEADROOM - mg, E_HEADROOM - mg);
              float2 s2 = make_float2(0.f, 0.f);  // (even-column sum, odd-column sum), label excluded
              uint32_t h[32];
#pragma unroll
              for (int half = 0; half < 2; ++half) {
                const float* v = half ? vb : va;
#pragma unroll
                for (int i = 0; i < 32; i += 2) {  // the label element is -inf: E = 0, out of the sum
                  const float2 y = fwde_y(v[i], v[i + 1], tl2, nmg);
                  const float e0 = ptx::ex2(y.x), e1 = ptx::ex2(y.y);
                  s2 = fwde_acc(s2, e0, e1);
                  __half2 hh = __floats2half2_rn(e0, e1);
                  h[half * 16 + i / 2] = *reinterpret_cast<uint32_t*>(&hh);
                }
                // Half-slice store pipeline: this half goes into staging half-buffer `ebuf`; the
                // previous half, written one compute phase ago, is fenced and TMA-stored first, so
                // neither the STS -> fence.proxy.async latency nor the TMA read is exposed.
                const int rbase = rt * PAIR_M + crank * BM + quad * 32;
                const int hcb = col0 + j * 64 + half * 32;
                e_push([&](uint8_t* hb) { ptx::st_swizzled_row64(hb, lane, h + half * 16); }, hcb, rbase, dir);
              }
              const int cb = col0 + j * 64;
              const float mnew = fmaxf(m2, mg);
              l = l * ptx::ex2(m2 - mnew) + (s2.x + s2.y) * ptx::ex2(mg - E_HEADROOM - mnew);
              m2 = mnew;
              if (row_ok) p.mg[(int64_t(dir) * p.groups + cb / GROUP_COLS) * p.b + row] = mg;
              if (j + 1 < NJ) ptx::tmem_wait_ld_dep(ra, rb);
            }
          }
        } else {
          // G = exp2(y - lse2) (label column: P_label - 1), f16, 64-column slices
          // transposed through swizzled smem and written as full 128-byte rows.
#pragma unroll 1
          for (int j = 0; j < PART_COLS / 64; ++j) {
            const int cb = col0 + j * 64;
            if (cb >= chunk_hi) break;  // warp-uniform
            uint32_t h[32];
            const int li = label - cb;
#pragma unroll
            for (int half = 0; half < 2; ++half) {
              float v[32];
              ptx::tmem_ld32(taddr + j * 64 + half * 32, v);
#pragma unroll
              for (int i = 0; i < 32; i += 2) {
                float g0 = ptx::ex2(fmaf(v[i], p.tl2e, -lse2));
                float g1 = ptx::ex2(fmaf(v[i + 1], p.tl2e, -lse2));
                __half2 hh = __floats2half2_rn(g0, g1);
                h[half * 16 + i / 2] = *reinterpret_cast<uint32_t*>(&hh);
              }
            }
            if (unsigned(li) < 64u) {  // label column: P_label - 1 (warp-uniform for canonical layouts)
#pragma unroll
              for (int k = 0; k < 32; ++k) {
                if (li >> 1 == k) {
                  __half2 hh = *reinterpret_cast<__half2*>(&h[k]);
                  if (li & 1) hh.y = __float2half_rn(gl); else hh.x = __float2half_rn(gl);
                  h[k] = *reinterpret_cast<uint32_t*>(&hh);
                }
              }
            }
            if (p.g_blocked) {
              // asynchronous TMA bulk store of the 32 x 64 slice into its 128 x 128 block;
              // the warp only waits when it reuses a staging buffer.
              const int rbase = rt * PAIR_M + crank * BM + quad * 32;
              uint8_t* stile = staging + (ew * STAGING_BUFS + (gslice % STAGING_BUFS)) * STAGING_TILE;
              if (lane == 0) ptx::bulk_wait_read<STAGING_BUFS - 1>();
              __syncwarp();
              ptx::st_swizzled_row(stile, lane, h);
              ptx::fence_proxy_async_smem();
              __syncwarp();
              if (lane == 0) {
                if (rbase < p.b) ptx::tma_store_4d(&p.g_map[dir], stile, cb & 127, rbase & 127, cb >> 7, rbase >> 7);
                ptx::bulk_commit();
              }
              ++gslice;
            } else if ((chunk_lo & 63) == 0 && (cb + 64 <= chunk_hi || (chunk_hi == p.B && (p.B & 63) == 0))) {
              // row-major G: transpose through swizzled smem, 4 full 128-byte rows per store
              ptx::st_swizzled_row(tile, lane, h);
              __syncwarp();
              const int rbase = rt * PAIR_M + crank * BM + quad * 32;
              __half* gbase = p.G + int64_t(dir) * p.b * p.ldG + cb;
              ptx::store_tile_rows(tile, lane, [&](int r) -> uint8_t* {
                return rbase + r < p.b ? reinterpret_cast<uint8_t*>(gbase + int64_t(rbase + r) * p.ldG) : nullptr;
              }, ptx::kEvictFirst);
              __syncwarp();
            } else if (row_ok) {  // non-canonical chunk edges (b not a multiple of 64): scalar path
#pragma unroll
              for (int i = 0; i < 64; i += 2) {
                const uint32_t w = h[i / 2];
                if (cb + i < chunk_hi) grow[cb + i] = __ushort_as_half((unsigned short)(w & 0xFFFF));
                if (cb + i + 1 < chunk_hi) grow[cb + i + 1] = __ushort_as_half((unsigned short)(w >> 16));
              }
            }
          }
        }
        release_accumulator(ctl, buf, lane);
      }
      if (KIND != KIND_GRAD && row_ok) {
        p.stats[((int64_t(dir) * p.nchunk + ch) * NPARTS + cpart) * p.b + row] = make_float2(m2, l);
        if (has_t) {
          p.target[dir * p.b + row] = yt;
        }
      }
    }
    if (KIND == KIND_FWDE) e_flush();
    if (KIND != KIND_FWD && lane == 0) ptx::bulk_wait_all();  // drain any bulk stores
  }
  kernel_epilogue(ctl, warp);
  probe_mark(p.probe, 2);
}

// =====================================================================
// Grouped f16 GEMM with fp32 tile outputs, CTA pair = 256 x 256 tile.
//   unit = (problem, m tile, n tile, k chunk); one accumulator tile per unit,
//   or, for `paired` problems, two consecutive canonical K chunks accumulated
//   into the two TMEM buffers and summed in the epilogue ((c0 + c1): the first
//   level of the fixed reduction tree).
// =====================================================================
template <int NB, bool XF>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(gemm_threads<NB, XF>(), 1)
    gemm_kernel(const __grid_constant__ GemmParams p) {
  constexpr int NA = 1;  // A tiles per stage
  constexpr int RS = Ring<NB, NA>::STAGES;
  static_assert(NB == 1 || NB == 2, "one or two N tiles per unit");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* tiles = smem_base(smem_raw);
  uint8_t* staging = tiles + TILE_RING_BYTES;
  SmemCtl* ctl = reinterpret_cast<SmemCtl*>(tiles + TILE_RING_BYTES + STAGING_BYTES);
  uint8_t* qrec = reinterpret_cast<uint8_t*>(ctl) + 512;  // dual: [RS][DUAL_Q_BYTES] (SMEM_BYTES_XF)
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int crank = int(ptx::cluster_ctarank());
  const bool leader = crank == 0;
  const int pair = blockIdx.x / 2, npairs = gridDim.x / 2;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < p.nprob; ++i) {
      ptx::prefetch_tmap(&p.prob[i].a_map);
      ptx::prefetch_tmap(&p.prob[i].b_map);
      if (p.prob[i].tma_store && !p.prob[i].peer) ptx::prefetch_tmap(&p.prob[i].out_map);
      for (int r = 0; r < (p.prob[i].peer ? p.prob[i].M / p.prob[i].peer_b : 0); ++r)
        ptx::prefetch_tmap(&p.prob[i].peer_map[r]);
    }
  }
  probe_mark(p.probe, 0);
  kernel_prologue(ctl, warp, lane);

  const int num_units = p.units[p.nprob];
  // this pair's sequence of unit indices: the static schedule, or round-robin over pairs
  const int my_units = p.sched_n ? int(p.sched_off[pair + 1]) - int(p.sched_off[pair])
                                 : (num_units - pair + npairs - 1) / npairs;
  auto unit_at = [&](int k) -> int { return p.sched_n ? int(p.sched[p.sched_off[pair] + k]) : pair + k * npairs; };
  // unit -> (problem, mt, nt, kc); nt fastest so pairs sharing an A tile run together.
  auto decode = [&](int u, int& pi, int& mt, int& nt, int& kc) {
    if (p.split > 0) {
      const int64_t nA = p.units[p.split];
      const int64_t cA = int64_t(u) * nA / num_units, cA1 = int64_t(u + 1) * nA / num_units;
      u = cA1 > cA ? int(cA) : int(nA + u - cA1);
    }
    pi = 0;
    while (pi + 1 < p.nprob && u >= p.units[pi + 1]) ++pi;
    int rem = u - p.units[pi];
    const GemmProblem& q = p.prob[pi];
    nt = rem % q.n_tiles;
    rem /= q.n_tiles;
    kc = rem % q.k_chunks;
    mt = rem / q.k_chunks + q.m_off;
  };
  // canonical chunk index `c` -> [k0, k0 + nk*BK)
  auto k_range = [&](const GemmProblem& q, int c, int& k0, int& nk) {
    k0 = c * q.k_chunk_len;
    const int k1 = min(k0 + q.k_chunk_len, q.k_total);
    nk = (k1 - k0 + BK - 1) / BK;
  };

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer (both CTAs)
      Pipe<RS> pipe;
      for (int uk = 0; uk < my_units; ++uk) {
        const int u = unit_at(uk);
        int pi, mt, nt, kc;
        decode(u, pi, mt, nt, kc);
        const GemmProblem& q = p.prob[pi];
        const int m0 = mt * PAIR_M + crank * BM;
        const int n0 = nt * NB * BN + crank * (BN / 2) + q.n_off;
        for (int sub = 0; sub <= q.paired; ++sub) {
          int k0, nk;
          k_range(q, kc * (1 + q.paired) + sub, k0, nk);
          for (int kb = 0; kb < nk; ++kb) {
            uint32_t bar;
            const bool dual = XF && q.xform == 2;
            uint8_t* st = producer_acquire<NB, XF, RS, NA>(ctl, tiles, pipe, leader, bar, crank,
                                                           dual ? DUAL_Q_BYTES : 0);
            const int k = k0 + kb * BK;
            if (q.a_blocked)
              load_blocked(&q.a_map, q.a_mn_major, st, bar, m0, k, BM, ptx::kEvictFirst);
            else if (q.a_mn_major)
              load_operand(&q.a_map, 1, st, bar, m0, k + q.a_k_off, BM, ptx::kEvictFirst);
            else
              load_operand(&q.a_map, 0, st, bar, m0 + q.a_row_off, k, BM, ptx::kEvictFirst);
            if (dual)  // the stage's 64 column factors q_c
              ptx::bulk_g2s(ptx::smem_u32(qrec + pipe.stage * DUAL_Q_BYTES), q.xq + k, DUAL_Q_BYTES, bar);
#pragma unroll
            for (int j = 0; j < NB; ++j)
              load_operand(&q.b_map, q.b_mn_major, st + NA * A_STAGE_BYTES + j * B_STAGE_BYTES, bar, n0 + j * BN,
                           k + q.b_k_off, BN / 2, ptx::kEvictLast);
            pipe.advance();
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {  // ---------------- MMA issuer (leader CTA, whole warp; one elected lane issues)
      Pipe<RS> pipe;
      uint32_t it = 0;
#if DISCO_WAITPROBE
      const long long wt0 = clock64();
#endif
      for (int uk = 0; uk < my_units; ++uk) {
        const int u = unit_at(uk);
        int pi, mt, nt, kc;
        decode(u, pi, mt, nt, kc);
        const GemmProblem& q = p.prob[pi];
        const uint32_t idesc = ptx::instr_desc_f16(PAIR_M, BN, 0, 0, q.a_mn_major, q.b_mn_major);  // f16 x f16
        if constexpr (NB == 2) {  // wide unit: both accumulators, one pass over K
          int k0, nk;
          k_range(q, kc, k0, nk);
          const uint32_t ph = ((it >> 1) & 1) ^ 1;
          {
            // The epilogue releases accumulator 0 half-way through its drain: issue the unit's first
            // ring-full of k-blocks into accumulator 0 alone (the stages stay resident), then, once
            // accumulator 1 is free, the same stages into accumulator 1, releasing them, then the rest
            // of K into both.  Each accumulator still sums its k-blocks in the same order.
            const int pre = nk < RS ? nk : RS;
#if DISCO_WAITPROBE
            const long long w1 = clock64();
#endif
            ptx::mbar_wait(&ctl->tempty[0], ph);
#if DISCO_WAITPROBE
            if (lane == 0) atomicAdd(&g_waitprobe[9], (unsigned long long)(clock64() - w1));
#endif
            Pipe<RS> first = pipe;
            mma_blocks<NB, XF, RS, NA>(ctl, tiles, first, pre, 0, ctl->tmem_base, idesc, q.a_mn_major, q.b_mn_major,
                                       0, 1, true, false);
#if DISCO_WAITPROBE
            const long long w2 = clock64();
#endif
            ptx::mbar_wait(&ctl->tempty[1], ph);
#if DISCO_WAITPROBE
            if (lane == 0) atomicAdd(&g_waitprobe[9], (unsigned long long)(clock64() - w2));
#endif
            mma_blocks<NB, XF, RS, NA>(ctl, tiles, pipe, pre, 0, ctl->tmem_base, idesc, q.a_mn_major, q.b_mn_major,
                                       1, 2, false, true);
            mma_blocks<NB, XF, RS, NA>(ctl, tiles, pipe, nk - pre, pre, ctl->tmem_base, idesc, q.a_mn_major,
                                       q.b_mn_major, 0, 2, true, true);
          }
          if (ptx::elect_one()) {
            ptx::umma_commit_pair(&ctl->tfull[0], 0x3);
            ptx::umma_commit_pair(&ctl->tfull[1], 0x3);
          }
          __syncwarp();
          it += 2;
        }
        if constexpr (NB == 1) {
          for (int sub = 0; sub <= q.paired; ++sub, ++it) {
            int k0, nk;
            k_range(q, kc * (1 + q.paired) + sub, k0, nk);
            const uint32_t buf = it & 1, use = it >> 1;
            ptx::mbar_wait(&ctl->tempty[buf], (use & 1) ^ 1);
            ptx::tc_fence_after();
            mma_tile<1, XF, RS>(ctl, tiles, pipe, nk, ctl->tmem_base + buf * BN, idesc, q.a_mn_major, q.b_mn_major);
            if (ptx::elect_one()) ptx::umma_commit_pair(&ctl->tfull[buf], 0x3);
            __syncwarp();
          }
        }
      }
#if DISCO_WAITPROBE
      if (lane == 0) {
        atomicAdd(&g_waitprobe[10], (unsigned long long)(clock64() - wt0));
        atomicAdd(&g_waitprobe[11], 1ull);
      }
#endif
    }
  } else if (XF && warp >= 2 + NUM_EPI_WARPS) {  // ---------------- transform warps 10..13
    // Thread xt owns one 128-byte row of this CTA's A stage:
    //   K-major A (intra, G rows = M): row xt = G row m0 + xt, G columns [k, k + 64);
    //   MN-major A (cross, G^T): atom xt / 64, K-row xt % 64 = G row k + xt % 64,
    //   G columns [m0 + 64 * (xt / 64), +64).
    // The scale of the next stage is loaded one stage ahead (it only depends on K within a unit).
    const int xgroup = (warp - (2 + NUM_EPI_WARPS)) / NUM_XF_WARPS;
    const int xt = threadIdx.x - 32 * (2 + NUM_EPI_WARPS) - 32 * NUM_XF_WARPS * xgroup;
    const uint32_t xbar = 0;  // transform completion is counted on the leader's xfull barriers
    Pipe<RS> pipe;
#if DISCO_WAITPROBE
    const long long xt0 = clock64();
#endif
    for (int uk = 0; uk < my_units; ++uk) {
        const int u = unit_at(uk);
      int pi, mt, nt, kc;
      decode(u, pi, mt, nt, kc);
      const GemmProblem& q = p.prob[pi];
      const int m0 = mt * PAIR_M + crank * BM;
      if (q.xform == 2) {
        // Dual backward: thread xt owns row r = m0 + xt of this direction's E block (K-major) and
        // rewrites each 64-column stage to H' = E f with f = a_r + p_r q_c formed in fp32 (FFMA2)
        // and rounded once to f16 (saturating: only rows the fixup recomputes can exceed the
        // range), the product by HMUL2 -- the exchange backward's roundings.  The label column is
        // zeroed (the combine adds its fp32 value).  All 8 E chunks are loaded before any math and
        // the column factors one chunk ahead; the row's group maxima and the group metadata run
        // XPF stages ahead.
        const int r = m0 + xt;
        const bool act = r < q.xb;  // rows past b were zero-filled by TMA: nothing to transform
        const float lse_r = act ? q.xlse[r] : 0.f;
        const float* xmg_r = q.xmg + r;
        const float2* xgm = q.xgm;
        const int64_t xb = q.xb;
        const int lab_base = q.lab_off + r;
        const int sw = xt & 7;
        int k0, nk;
        k_range(q, kc, k0, nk);
        constexpr int XPF = 6;
        auto ld_mg = [&](int kb) { return (act && kb < nk) ? xmg_r[int64_t((k0 + kb * BK) >> 6) * xb] : 0.f; };
        auto ld_gm = [&](int kb) { return kb < nk ? xgm[(k0 + kb * BK) >> 6] : make_float2(0.f, 0.f); };
        float mq[XPF];
        float2 gq[XPF];
#pragma unroll
        for (int i = 0; i < XPF; ++i) {
          mq[i] = ld_mg(i);
          gq[i] = ld_gm(i);
        }
        bool unsafe = false;
        for (int kb0 = 0; kb0 < nk; kb0 += XPF) {
#pragma unroll
          for (int i = 0; i < XPF; ++i) {
            const int kb = kb0 + i;
            if (kb >= nk) break;
            const int k = k0 + kb * BK;
            const float mg = mq[i];
            const float2 gm = gq[i];
            mq[i] = ld_mg(kb + XPF);
            gq[i] = ld_gm(kb + XPF);
            if (xf_groups<NB>() > 1 && int(pipe.stage % xf_groups<NB>()) != xgroup) {  // the other group's stage
              pipe.advance();
              continue;
            }
#if DISCO_WAITPROBE
            const long long w3 = clock64();
#endif
            ptx::mbar_wait(&ctl->full[pipe.stage], pipe.phase);
#if DISCO_WAITPROBE
            if ((threadIdx.x & 31) == 0) atomicAdd(&g_waitprobe[12], (unsigned long long)(clock64() - w3));
#endif
            if (act) {
              unsafe |= mg - gm.y > DUAL_SAFE_SPAN;
              const float a = ptx::ex2(mg + (H_DUAL_LOG2 - E_HEADROOM) - lse_r);
              const float pr = ptx::ex2(mg + (H_DUAL_LOG2 - E_HEADROOM) - gm.x);
              const float2 a2 = make_float2(a, a), p2 = make_float2(pr, pr);
              const uint32_t rowp = ptx::smem_u32(tiles + pipe.stage * Ring<NB, NA>::STAGE_BYTES + xt * 128);
              const uint32_t qs = ptx::smem_u32(qrec + pipe.stage * DUAL_Q_BYTES);
              uint4 x[8];
#pragma unroll
              for (int c = 0; c < 8; ++c) x[c] = ptx::lds128(rowp + ((c ^ sw) << 4));
              float4 q0 = ptx::lds128f(qs), q1 = ptx::lds128f(qs + 16);
#pragma unroll
              for (int c = 0; c < 8; ++c) {
                float4 n0, n1;
                if (c < 7) {
                  n0 = ptx::lds128f(qs + 32 * (c + 1));
                  n1 = ptx::lds128f(qs + 32 * (c + 1) + 16);
                }
                const float2 qv[4] = {make_float2(q0.x, q0.y), make_float2(q0.z, q0.w), make_float2(q1.x, q1.y),
                                      make_float2(q1.z, q1.w)};
                __half2* h = reinterpret_cast<__half2*>(&x[c]);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const uint32_t f = ptx::f2_to_h2_satfinite(ptx::ffma2(p2, qv[e], a2));
                  h[e] = __hmul2(h[e], *reinterpret_cast<const __half2*>(&f));
                }
                ptx::sts128(rowp + ((c ^ sw) << 4), x[c]);
                if (c < 7) {
                  q0 = n0;
                  q1 = n1;
                }
              }
              const int lab_rel = lab_base - k;
              if (unsigned(lab_rel) < 64u) ptx::sts16(rowp + (((lab_rel >> 3) ^ sw) << 4) + (lab_rel & 7) * 2, 0);
              ptx::fence_proxy_async_smem();
            }
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_cluster(ptx::map_to_rank(&ctl->xfull[pipe.stage], 0));
            pipe.advance();
          }
        }
        if (unsafe) {
          const int slot = atomicAdd(q.fix_count, 1);
          if (slot < q.fix_cap) q.fix_list[slot] = q.fix_tag + r;
        }
        continue;
      }
      const int rowoff = q.a_mn_major ? (xt >> 6) * 8192 + (xt & 63) * 128 : xt * 128;
      const int sw = (rowoff >> 7) & 7;
      // per-stage scale index (64-column groups): K-major: (k / 64) * xb + (m0 + xt);
      // MN-major: ((m0 + 64 * (xt / 64)) / 64) * xb + k + xt % 64
      auto sidx = [&](int k) -> int64_t {
        return q.a_mn_major ? int64_t((m0 >> 6) + (xt >> 6)) * q.xb + k + (xt & 63) : int64_t(k >> 6) * q.xb + m0 + xt;
      };
      // rows past b (last pair tile when b / 128 is odd) were zero-filled by TMA: nothing to scale
      const bool active = q.xform && (q.a_mn_major || m0 + xt < q.xb);
      const float glab_row = (active && !q.a_mn_major) ? q.xlabel[m0 + xt] : 0.f;
      for (int sub = 0; sub <= q.paired; ++sub) {
        int k0, nk;
        k_range(q, kc * (1 + q.paired) + sub, k0, nk);
        // scales run XPF stages ahead of the stage being transformed (the scale array is
        // L2-cold: one stage of lead time does not cover an HBM round trip); the loop is
        // unrolled by XPF so every prefetch register keeps a fixed role (no moves that would
        // wait on an in-flight load).
        constexpr int XPF = 4;
        auto ld_scale = [&](int kb) { return (active && kb < nk) ? q.xscale[sidx(k0 + kb * BK)] : __float2half(0.f); };
        __half sq[XPF];
#pragma unroll
        for (int r = 0; r < XPF; ++r) sq[r] = ld_scale(r);
        for (int kb0 = 0; kb0 < nk; kb0 += XPF) {
#pragma unroll
          for (int r = 0; r < XPF; ++r) {
            const int kb = kb0 + r;
            if (kb >= nk) break;
            const int k = k0 + kb * BK;
            const __half sc = sq[r];
            sq[r] = ld_scale(kb + XPF);
            if (xf_groups<NB>() > 1 && int(pipe.stage % xf_groups<NB>()) != xgroup) {  // the other group's stage
              pipe.advance();
              continue;
            }
            ptx::mbar_wait(&ctl->full[pipe.stage], pipe.phase);
            if (active && !(XP && (q.ablate & 1024))) {
              const uint32_t rowp = ptx::smem_u32(tiles + pipe.stage * Ring<NB, NA>::STAGE_BYTES + rowoff);
              int lab_rel;
              float glab;
              if (q.a_mn_major) {  // row = G row i = k + xt % 64; label column lab_off + i
                const int i = k + (xt & 63);
                lab_rel = q.lab_off + i - (m0 + (xt >> 6) * 64);
                glab = unsigned(lab_rel) < 64u ? q.xlabel[i] : 0.f;
              } else {  // row = G row m0 + xt
                lab_rel = q.lab_off + m0 + xt - k;
                glab = glab_row;
              }
              xform_row(rowp, sw, sc, lab_rel, glab);
              ptx::fence_proxy_async_smem();
            }
            __syncwarp();
            // CTA-scope release is enough: the pair MMA reads each CTA's stage with that CTA's own
            // tensor core, and fence.proxy.async above already published the writes to it.  A
            // cluster-scope release would emit MEMBAR.GPU, which also drains the scale prefetches.
            if (lane == 0) ptx::mbar_arrive_cluster(ptx::map_to_rank(&ctl->xfull[pipe.stage], xbar));
            pipe.advance();
          }
        }
      }
    }
#if DISCO_WAITPROBE
    if (lane == 0) {
      atomicAdd(&g_waitprobe[13], (unsigned long long)(clock64() - xt0));
      atomicAdd(&g_waitprobe[14], 1ull);
    }
#endif
  } else if (warp >= 2) {  // ---------------------------- epilogue warps 2..9
    const int ew = warp - 2;
    const int quad = warp & 3;
    const int chalf = ew >> 2;
    uint8_t* tile = staging + ew * STAGING_BUFS * STAGING_TILE;
    uint32_t it = 0, gslice = 0;
    for (int uk = 0; uk < my_units; ++uk) {
        const int u = unit_at(uk);
      int pi, mt, nt, kc;
      decode(u, pi, mt, nt, kc);
      const GemmProblem& q = p.prob[pi];
      const bool two = q.paired || NB == 2;  // unit occupies both accumulators
      const uint32_t buf0 = it & 1, buf1 = (it + 1) & 1;
      ptx::mbar_wait(&ctl->tfull[buf0], (it >> 1) & 1);
      if (two) ptx::mbar_wait(&ctl->tfull[buf1], ((it + 1) >> 1) & 1);
      ptx::tc_fence_after();
      const long long drain_t0 = clock64();
      const int row0 = mt * PAIR_M + crank * BM + quad * 32;  // first row of this warp's 32-row slab
      const int row = row0 + lane;
      const uint32_t lane_base = ctl->tmem_base + (uint32_t(quad * 32) << 16) + chalf * (BN / 2);
      const uint32_t ta0 = lane_base + buf0 * BN, ta1 = lane_base + buf1 * BN;
      const int cbase = nt * NB * BN + chalf * (BN / 2) + q.n_off;
      float* orow = nullptr;
      if (!q.tma_store && row < q.M)
        orow = q.out + kc * q.chunk_stride + (row / q.row_div) * q.stride_hi + (row % q.row_div) * q.ld_out;
      const int z = int(row0 / q.row_div) + kc;
      const int rlo = int(row0 % q.row_div);
      if (NB == 2 && q.tma_store == 1 && !(XP && (q.skip_store || q.ablate))) {
        // Wide drain, software-pipelined: slice jj + 1's TMEM load is in flight while slice jj is
        // staged and TMA-stored, and accumulator 0 is released as soon as its last slice sits in
        // registers, so the MMA starts the next unit (accumulator 0 half) during this drain.
        uint32_t ra[32], rb[32];
        auto taddr_of = [&](int jj) { return (jj < 4 ? ta0 : ta1) + (jj & 3) * 32; };
        auto stage_store = [&](const uint32_t (&w)[32], int jj) {
          const int c0 = cbase + (jj >> 2) * BN + (jj & 3) * 32;
          if (c0 >= q.N) return;  // warp-uniform
          if (lane == 0) ptx::bulk_wait_read<STAGING_BUFS - 1>();
          __syncwarp();
          ptx::st_swizzled_row(tile, lane, w);
          ptx::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            if (q.peer) {  // NVLink push: this slice belongs to rank row0 / b
              const int dest = row0 / q.peer_b;
              if (row0 < q.M) ptx::tma_store_3d(&q.peer_map[dest], tile, c0, row0 - dest * q.peer_b, kc);
            } else if (row0 < q.M) {
              ptx::tma_store_3d(&q.out_map, tile, c0, rlo, z);
            }
            ptx::bulk_commit();
          }
        };
        ptx::tmem_ld32_async(taddr_of(0), ra);
        ptx::tmem_wait_ld_dep1(ra);
#pragma unroll
        for (int jj = 0; jj < 8; jj += 2) {
          ptx::tmem_ld32_async(taddr_of(jj + 1), rb);
          stage_store(ra, jj);
          ptx::tmem_wait_ld_dep1(rb);
          if (jj + 1 == 3) release_accumulator(ctl, buf0, lane);  // slices 0..3 (accumulator 0) are out
          if (jj + 2 < 8) ptx::tmem_ld32_async(taddr_of(jj + 2), ra);
          stage_store(rb, jj + 1);
          if (jj + 2 < 8) ptx::tmem_wait_ld_dep1(ra);
        }
        release_accumulator(ctl, buf1, lane);
        if (p.probe && ew == 0 && lane == 0 && leader) {
          atomicAdd(p.probe + 4, (unsigned long long)(clock64() - drain_t0));
          atomicAdd(p.probe + 5, 1ull);
        }
        it += 2;
        continue;
      }
#pragma unroll 1
      for (int jj = 0; jj < ((XP && (q.ablate & 2048)) ? 0 : NB * (BN / 64)); ++jj) {
        // NB = 2: slices 0..3 from accumulator 0 (columns [0,256)), 4..7 from accumulator 1
        const int j = jj % (BN / 64), acc = jj / (BN / 64);
        const int c0 = cbase + acc * BN + j * 32;
        if (c0 >= q.N) continue;  // warp-uniform
        float v[32];
        ptx::tmem_ld32((acc ? ta1 : ta0) + j * 32, v);
        if (NB == 1 && q.paired) {
          float v1[32];
          ptx::tmem_ld32(ta1 + j * 32, v1);
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] += v1[i];
        }
        if (XP && q.skip_store) {
          if (v[0] == 12345.678f) asm volatile("trap;");  // keep the TMEM load live
        } else if (XP && q.tma_store == 2) {
          // 32 x 32 fp32 slice transposed through swizzled smem, then written by the warp as
          // 128-byte row segments (4 rows per instruction); no async-proxy round trip.
          uint32_t w[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) w[i] = __float_as_uint(v[i]);
          ptx::st_swizzled_row(tile, lane, w);
          __syncwarp();
          ptx::store_tile_rows(tile, lane, [&](int r) -> uint8_t* {
            const int rr = row0 + r;
            if (rr >= q.M || c0 + 32 > q.N) return nullptr;
            return reinterpret_cast<uint8_t*>(q.out + kc * q.chunk_stride + (rr / q.row_div) * q.stride_hi +
                                              (rr % q.row_div) * q.ld_out + c0);
          }, ptx::kEvictFirst);
          __syncwarp();
        } else if (q.tma_store) {
          // 32 x 32 fp32 slice through swizzled staging -> 3-D TMA store (clipped at M / N).
          uint32_t w[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) w[i] = __float_as_uint(v[i]);
          uint8_t* stile = tile + (gslice % STAGING_BUFS) * STAGING_TILE;
          if (lane == 0) ptx::bulk_wait_read<STAGING_BUFS - 1>();
          __syncwarp();
          ptx::st_swizzled_row(stile, lane, w);
          ptx::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0 && !(XP && (q.ablate & 32768))) {  // bit15 ablation: stage but never store
            if (q.peer) {  // NVLink push: this slice belongs to rank row0 / b
              const int dest = row0 / q.peer_b;
              if (row0 < q.M) ptx::tma_store_3d(&q.peer_map[dest], stile, c0, row0 - dest * q.peer_b, kc);
            } else if (row0 < q.M) {
              ptx::tma_store_3d(&q.out_map, stile, c0, rlo, z);
            }
            ptx::bulk_commit();
          }
          ++gslice;
        } else if (orow) {
          if (c0 + 32 <= q.N) {
            float4* dst = reinterpret_cast<float4*>(orow + c0);
#pragma unroll
            for (int i = 0; i < 8; ++i) dst[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
          } else {
            for (int i = 0; i < 32 && c0 + i < q.N; ++i) orow[c0 + i] = v[i];
          }
        }
      }
      release_accumulator(ctl, buf0, lane);
      if (two) release_accumulator(ctl, buf1, lane);
      if (p.probe && ew == 0 && lane == 0 && leader) {
        atomicAdd(p.probe + 4, (unsigned long long)(clock64() - drain_t0));  // Status::drain follows probe
        atomicAdd(p.probe + 5, 1ull);
      }
      it += two ? 2 : 1;
    }
    if (lane == 0) {
      ptx::bulk_wait_all();
      bool any_peer = false;
      for (int i = 0; i < p.nprob; ++i) any_peer |= p.prob[i].peer != 0;
      if (any_peer) {  // pushed tiles are complete; order them before the arrival flags (next kernel)
        asm volatile("fence.proxy.async.global;" ::: "memory");
        __threadfence_system();
      }
    }
  }
  kernel_epilogue(ctl, warp);
  probe_mark(p.probe, 2);
}


// =====================================================================
// Small HBM-bound kernels
// =====================================================================
template <typename T>
__device__ __forceinline__ float load_as_float(const void* p, int64_t i) {
  return static_cast<float>(static_cast<const T*>(p)[i]);
}
template <>
__device__ __forceinline__ float load_as_float<__nv_bfloat16>(const void* p, int64_t i) {
  return __bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]);
}
template <>
__device__ __forceinline__ float load_as_float<__half>(const void* p, int64_t i) {
  return __half2float(static_cast<const __half*>(p)[i]);
}

// Round local features to bf16, pad D..Dp with zeros: out [2][b][Dp].
// One thread per 8 output elements (one 16-byte store); f64 inputs are rounded
// directly f64 -> bf16 (a single rounding).
// out16 (optional): also write the f16 copy (single rank: packed == gathered layout).
// Rows [row0, row0 + nrows) of both matrices (the H2D-pipelined single-rank path packs one
// canonical chunk at a time as it lands).
// vec: both inputs 16-byte aligned with D and the row strides multiples of 8 (host-checked):
// bf16 / f32 groups of 8 are read with 16-byte loads (same values as the scalar path).
template <typename T>
__global__ void pack_kernel(const void* I, const void* Tm, int64_t ldI, int64_t ldT, int b, int D, int Dp,
                            __nv_bfloat16* out, __half* out16, Status* status, int row0, int nrows, int vec) {
  const int v8 = Dp / 8;
  const int64_t total = int64_t(2) * nrows * v8;
  bool bad = false;
  const unsigned uv8 = unsigned(v8), unr = unsigned(nrows);  // total < 2^31: 32-bit index math
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < total; j += int64_t(gridDim.x) * blockDim.x) {
    const unsigned ju = unsigned(j), rr = ju / uv8;
    const int c0 = int(ju - rr * uv8) * 8;
    const int dir = int(rr / unr), r = row0 + int(rr - unsigned(dir) * unr);
    const int64_t i = (int64_t(dir) * b + r) * v8 + c0 / 8;
    const void* src = dir ? Tm : I;
    const int64_t base = r * (dir ? ldT : ldI);
    __align__(16) __nv_bfloat16 o[8];
    constexpr bool VEC_T = std::is_same<T, __nv_bfloat16>::value || std::is_same<T, float>::value;
    if (VEC_T && vec && c0 + 8 <= D) {
      if constexpr (std::is_same<T, __nv_bfloat16>::value) {
        const uint4 v = *reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(src) + base + c0);
        const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 f = __bfloat1622float2(h2[k]);
          bad |= !(isfinite(f.x) && isfinite(f.y));
        }
        *reinterpret_cast<uint4*>(o) = v;
      } else if constexpr (std::is_same<T, float>::value) {
        const float4* p4 = reinterpret_cast<const float4*>(static_cast<const float*>(src) + base + c0);
        const float4 a = p4[0], z = p4[1];
        const float f[8] = {a.x, a.y, a.z, a.w, z.x, z.y, z.z, z.w};
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          bad |= !isfinite(f[k]);
          o[k] = __float2bfloat16_rn(f[k]);
        }
      }
    } else {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int c = c0 + k;
      __nv_bfloat16 x = __float2bfloat16_rn(0.f);
      if (c < D) {
        if constexpr (sizeof(T) == 8) {
          const double xv = static_cast<const double*>(src)[base + c];
          bad |= !isfinite(xv);
          x = __double2bfloat16(xv);
        } else {
          const float xv = load_as_float<T>(src, base + c);
          bad |= !isfinite(xv);
          x = __float2bfloat16_rn(xv);
        }
      }
      o[k] = x;
    }
    }
    reinterpret_cast<uint4*>(out)[i] = *reinterpret_cast<const uint4*>(o);
    if (out16) {
      __align__(16) __half h[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) h[k] = __float2half_rn(__bfloat162float(o[k]));
      reinterpret_cast<uint4*>(out16)[i] = *reinterpret_cast<const uint4*>(h);
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(&status->flags, FLAG_INPUT_NONFINITE);
}

__global__ void clear_status_kernel(Status* s) {
  s->loss = 0.0;
  s->flags = 0;
  s->fix_count = 0;
}

// gathered [N][2][b][Dp] bf16 -> feat [2][B][Dp] bf16 and feat16 [2][B][Dp] f16. 8 elements per thread.
__global__ void unpack_kernel(const uint4* gathered, int N, int b, int Dp, uint4* feat, uint4* feat16) {
  const int vec_per_row = Dp / 8;
  const int64_t total = int64_t(N) * 2 * b * vec_per_row;
  const int64_t B = int64_t(N) * b;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int vc = int(i % vec_per_row);
    int64_t rr = i / vec_per_row;
    const int r = int(rr % b);
    rr /= b;
    const int dir = int(rr % 2);
    const int n = int(rr / 2);
    const uint4 x = gathered[i];
    const int64_t o = (dir * B + int64_t(n) * b + r) * vec_per_row + vc;
    feat[o] = x;
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&x);
    uint4 y;
    __half2* hy = reinterpret_cast<__half2*>(&y);
#pragma unroll
    for (int k = 0; k < 4; ++k) hy[k] = __float22half2_rn(__bfloat1622float2(h[k]));
    feat16[o] = y;
  }
}

// Streamed forward: the H2D copies wrote the bf16 operands (FEAT) directly; derive the f16
// backward operands and raise the non-finite input flag (the pack's other two jobs).
__global__ void feat16_kernel(const uint4* feat, uint4* feat16, int64_t n, Status* status) {
  bool bad = false;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const uint4 x = feat[i];
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&x);
    uint4 y;
    __half2* hy = reinterpret_cast<__half2*>(&y);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 f = __bfloat1622float2(h[k]);
      bad |= !(isfinite(f.x) && isfinite(f.y));
      hy[k] = __float22half2_rn(f);
    }
    feat16[i] = y;
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(&status->flags, FLAG_INPUT_NONFINITE);
}

// Per (dir,row): fixed-order combine of the (column chunk, column half)
// (max, sum-exp) partials.  Within a chunk: half 0 + half 1; across the 8
// canonical chunks: balanced tree ((0+1)+(2+3))+((4+5)+(6+7)); non-canonical
// chunkings: ascending order.
//   lse2 (log2 domain), ce = -log softmax[label], glabel = P_label - 1 = -(sum_{j!=label} P_j).
// ssub: stats sub-chunks per canonical chunk (the forward's units cover one sub-chunk); a chunk's
// sum is the fixed tree over its (sub-chunk, column half) partials.
// Shared tail: (m, lo = sum of non-label terms relative to m, target yt) -> lse2, glabel, ce of row i.
// m is the max over the non-label columns (the E offsets exclude the label), so the target may
// exceed it: the row total is taken relative to M = max(m, yt).
__device__ __forceinline__ void finish_row(int i, float m, float lo, float yt, float* lse2_out, float* glabel_out,
                                           float* ce_out, Status* status) {
  const float M = fmaxf(m, yt);
  const float lom = lo * ptx::ex2(m - M);  // non-label mass relative to M
  const float lall = lom + ptx::ex2(yt - M);
  const float lse2 = M + log2f(lall);
  const float dlt = m - yt;  // ce = ln(1 + lo 2^(m - yt))
  const float ce = dlt < 64.f ? log1pf(lo * exp2f(dlt)) : dlt * LN2 + logf(lo + exp2f(-dlt));
  lse2_out[i] = lse2;
  glabel_out[i] = -lom / lall;
  ce_out[i] = ce;
  if (!isfinite(ce) || !isfinite(lse2)) atomicOr(&status->flags, FLAG_LOSS_NONFINITE);
}

// ndir = 1: direction 0 only (the symmetric single-rank forward combines direction 1 separately).
// Per (dir, row): the forward left one online (max, sum) per (sub-chunk, column part); combine
// them in a fixed tree -- parts ((0 + 1) + (2 + 3)), sub-chunks, then the 8 canonical chunks
// ((0 + 1) + (2 + 3)) + ((4 + 5) + (6 + 7)) -- a function of B only, never of N.
__global__ void stats_combine_kernel(const float2* stats, const float* target, int nchunk, int ssub, int nparts,
                                     int b, int ndir, float* lse2_out, float* glabel_out, float* ce_out,
                                     Status* status) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ndir * b) return;
  const int dir = i / b, r = i % b;
  const int nsc = nchunk * ssub;
  auto at = [&](int sc, int h) { return stats[((int64_t(dir) * nsc + sc) * nparts + h) * b + r]; };
  float m = -INFINITY;
  for (int sc = 0; sc < nsc; ++sc)
    for (int h = 0; h < nparts; ++h) m = fmaxf(m, at(sc, h).x);
  auto part = [&](int sc, int h) {
    const float2 s = at(sc, h);
    return s.y * ptx::ex2(s.x - m);
  };
  auto sub_sum = [&](int sc) {
    return nparts == 4 ? (part(sc, 0) + part(sc, 1)) + (part(sc, 2) + part(sc, 3)) : part(sc, 0) + part(sc, 1);
  };
  auto chunk_sum = [&](int c) {
    return ssub == 2 ? sub_sum(2 * c) + sub_sum(2 * c + 1) : sub_sum(c);
  };
  float lo;
  if (nchunk == 8) {
    float t[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) t[c] = chunk_sum(c);
    lo = ((t[0] + t[1]) + (t[2] + t[3])) + ((t[4] + t[5]) + (t[6] + t[7]));
  } else {
    lo = 0.f;
    for (int c = 0; c < nchunk; ++c) lo += chunk_sum(c);
  }
  finish_row(i, m, lo, target[i], lse2_out, glabel_out, ce_out, status);
}

// E path: m_g [2][groups][b] (f32, log2 domain) -> sc [2][groups][b] = exp2(m_g - lse2[dir][r]) as f16,
// the E -> G factor of every (row, 64-column group).  8 elements per thread (b % 8 == 0).
__global__ void scale_kernel(const float4* mg, const float* lse2, int groups, int b, uint4* sc) {
  const int64_t per_dir = int64_t(groups) * b / 8;
  const int64_t total = 2 * per_dir;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int dir = int(i / per_dir);
    const int r = int((i * 8) % b);
    const float4 m0 = mg[2 * i], m1 = mg[2 * i + 1];
    const float4 l0 = *reinterpret_cast<const float4*>(lse2 + int64_t(dir) * b + r);
    const float4 l1 = *reinterpret_cast<const float4*>(lse2 + int64_t(dir) * b + r + 4);
    uint4 o;
    __half2* h = reinterpret_cast<__half2*>(&o);
    h[0] = __floats2half2_rn(ptx::ex2(m0.x - l0.x), ptx::ex2(m0.y - l0.y));
    h[1] = __floats2half2_rn(ptx::ex2(m0.z - l0.z), ptx::ex2(m0.w - l0.w));
    h[2] = __floats2half2_rn(ptx::ex2(m1.x - l1.x), ptx::ex2(m1.y - l1.y));
    h[3] = __floats2half2_rn(ptx::ex2(m1.z - l1.z), ptx::ex2(m1.w - l1.w));
    sc[i] = o;
  }
}

__device__ __forceinline__ float4 f4add(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
__device__ __forceinline__ float4 f4neg(float4 a) { return make_float4(-a.x, -a.y, -a.z, -a.w); }

// Fixed-order sum of n float4 terms: balanced binary tree over ascending index
// when n is a power of two <= 8 (a subtree of the canonical 8-chunk tree),
// ascending sequential otherwise.  Fixed-size cases are fully unrolled so the
// terms stay in registers (all loads issued before the adds).
template <int N, typename Get>
__device__ __forceinline__ float4 tree_fixed(Get get) {
  float4 acc[N];
#pragma unroll
  for (int k = 0; k < N; ++k) acc[k] = get(k);
#pragma unroll
  for (int w = 1; w < N; w <<= 1)
#pragma unroll
    for (int k = 0; k + w < N; k += 2 * w) acc[k] = f4add(acc[k], acc[k + w]);
  return acc[0];
}
template <typename Get>
__device__ __forceinline__ float4 tree_sum(int n, Get get) {
  switch (n) {
    case 1: return get(0);
    case 2: return tree_fixed<2>(get);
    case 4: return tree_fixed<4>(get);
    case 8: return tree_fixed<8>(get);
    default: {
      float4 acc = get(0);
      for (int k = 1; k < n; ++k) acc = f4add(acc, get(k));
      return acc;
    }
  }
}

// Sender-side tree over this rank's np paired-chunk partials:
//   xpart [2][B][np][Dp] (leaf-interleaved) -> send [N][2][b][Dp] (destination-major).
__global__ void presum_kernel(const float4* xpart, int np, int N, int b, int Dp, float4* send) {
  const int v4 = Dp / 4;
  const int64_t B = int64_t(N) * b;
  const int64_t per_g = B * v4;
  const int64_t total = 2 * per_g;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int g = int(i / per_g);
    const int64_t rem = i - g * per_g;
    const int64_t c = rem / v4;
    const int vc = int(rem % v4);
    const float4* src = xpart + ((int64_t(g) * B + c) * np) * v4 + vc;
    const float4 acc = tree_sum(np, [&](int k) { return __ldcs(src + k * v4); });
    const int64_t dest = c / b, r = c % b;
    send[((dest * 2 + g) * b + r) * v4 + vc] = acc;
  }
}

// Owner combine: d_g[r] = s * (intra_g[r] + cross_g[r]) written b x D (ld_out), where
//   cross = tree over the N received slabs recv[src][g][r] (negated for src != rank if flip), or,
//   single rank with canonical chunks (xpart != null), tree over the np local paired partials.
// Rows [row0, row0 + nrows) only (row-block pipelining); outputs are indexed by the absolute row.
// Peer transport: xpart = this rank's slab window [2][np leaves][b][Dp] (every source rank's chunk
// partials, pushed by their cross GEMMs); leaves outside [own_lo, own_hi) came from other ranks.
__global__ void combine_kernel(const float4* intra, int ksplit, const float4* recv, const float4* xpart, int np,
                               int N, int rank, int b, int Dp, int D, float s, int flip, float* d_image,
                               float* d_text, int64_t ld_out, int row0, int nrows, Status* status, int own_lo = 0,
                               int own_hi = 1 << 30, int interleaved = 0) {
  const int v4 = Dp / 4;
  const bool vec_out = (ld_out % 4 == 0) && ((reinterpret_cast<uintptr_t>(d_image) | reinterpret_cast<uintptr_t>(d_text)) % 16 == 0);
  const int64_t per_g = int64_t(b) * v4;
  const int64_t per_blk = int64_t(nrows) * v4;
  const int64_t total = 2 * per_blk;
  bool bad = false;
  // 32-bit index math (total < 2^31 for every supported shape); partials are read once: __ldcs
  const unsigned pb = unsigned(per_blk), uv4 = unsigned(v4);
  for (int64_t ii = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; ii < total; ii += int64_t(gridDim.x) * blockDim.x) {
    const unsigned iu = unsigned(ii);
    const int g = int(iu / pb);
    const int64_t rem = int64_t(iu - unsigned(g) * pb) + int64_t(row0) * v4;
    const int r = int(unsigned(rem) / uv4), vc = int(unsigned(rem) % uv4);
    float4 cross;
    if (xpart) {  // leaves [2][np][b][Dp] (peer windows) or leaf-interleaved [2][b][np][Dp] (local partials)
      const int64_t ls = interleaved ? v4 : per_g;
      const float4* src = xpart + (int64_t(g) * np) * per_g + (interleaved ? int64_t(r) * np * v4 + vc : rem);
      cross = tree_sum(np, [&](int k) {
        const float4 x = __ldcs(src + k * ls);
        return (flip && (k < own_lo || k >= own_hi)) ? f4neg(x) : x;
      });
    } else if (N > 0) {
      cross = tree_sum(N, [&](int src) {
        const float4 x = recv[((int64_t(src) * 2 + g) * b) * v4 + rem];
        return (flip && src != rank) ? f4neg(x) : x;
      });
    } else {  // N == 0: fused single-rank backward, the intra partials already hold the cross terms
      cross = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const float4* ib = intra + (int64_t(g) * ksplit) * per_g + rem;  // intra K-split partials, fixed order
    const float4 yi = ksplit == 2 ? f4add(__ldcs(ib), __ldcs(ib + per_g)) : __ldcs(ib);
    const float4 t = f4add(yi, cross);
    const float4 o = make_float4(t.x * s, t.y * s, t.z * s, t.w * s);
    float* out = (g == 0 ? d_image : d_text) + int64_t(r) * ld_out;
    const int c = vc * 4;
    bad |= !(isfinite(o.x) && isfinite(o.y) && isfinite(o.z) && isfinite(o.w));
    if (c + 4 <= D && vec_out) {
      __stcs(reinterpret_cast<float4*>(out + c), o);  // streaming store: outputs are not re-read here
    } else {
      const float ov[4] = {o.x, o.y, o.z, o.w};
      for (int k = 0; k < 4 && c + k < D; ++k) out[c + k] = ov[k];
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(&status->flags, FLAG_GRAD_NONFINITE);
}

// Full-size contribution of this rank (reference LocalGradContribution):
//   d_full_g[c] = s * (cross_g[c] + [c in own rows] intra_g[c - rank*b]), rows outside negated if flip.
//   cross_g[c] comes from the destination-major send slabs, or (single rank, canonical chunks) the
//   tree over the paired partials.
__global__ void contribution_kernel(const float4* intra, int ksplit, const float4* send, const float4* xpart,
                                    int np, int N, int rank, int b, int Dp, int D, float s, int flip,
                                    float* d_image, float* d_text, int64_t ld_out, Status* status) {
  const int v4 = Dp / 4;
  const int64_t B = int64_t(N) * b;
  const int64_t per_g = B * v4;
  const int64_t total = 2 * per_g;
  bool bad = false;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int g = int(i / per_g);
    const int64_t rem = i - g * per_g;
    const int64_t c = rem / v4;
    const int vc = int(rem % v4);
    const int64_t dest = c / b, r = c % b;
    float4 x;
    if (xpart) {
      const float4* src = xpart + ((int64_t(g) * B + c) * np) * v4 + vc;
      x = tree_sum(np, [&](int k) { return src[k * v4]; });
    } else if (send) {
      x = send[((dest * 2 + g) * b + r) * v4 + vc];
    } else {  // fused single-rank backward: no separate cross terms
      x = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const bool own = dest == rank;
    if (own) {
      const int64_t per_b = int64_t(b) * v4;
      const float4* ib = intra + (int64_t(g) * ksplit) * per_b + r * v4 + vc;
      x = f4add(ksplit == 2 ? f4add(ib[0], ib[per_b]) : ib[0], x);
    }
    float sg = (flip && !own) ? -s : s;
    float o[4] = {x.x * sg, x.y * sg, x.z * sg, x.w * sg};
    float* out = (g == 0 ? d_image : d_text) + c * ld_out;
    for (int k = 0; k < 4; ++k) {
      const int cc = vc * 4 + k;
      if (cc < D) {
        out[cc] = o[k];
        bad |= !isfinite(o[k]);
      }
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(&status->flags, FLAG_GRAD_NONFINITE);
}

// ---------------------------------------------------------------- peer transport
// Peer window of a rank (one cudaMalloc, IPC-exported): PEER_FLAG_BYTES of u32 arrival flags
// (slot src = the epoch of the last step whose slabs source rank src pushed here), then two
// parity windows of [2][L][b][Dp] f32 slabs (L = N * chunk partials per rank).  Step s writes
// parity s & 1: a rank's push for step s + 1 can only start after its own combine of step s,
// which waited for every peer's step-s arrival, so no window is overwritten while being read.
constexpr int64_t PEER_FLAG_BYTES = 1024;
struct PeerPtrs {
  uint32_t* flag[8];  // &flags[rank] inside each destination's window
};

// =====================================================================
// Dual backward (DISCO_PATH_DUAL).  Rank n's rows r need, besides their own softmax G_d[r, :],
// the other direction's softmax at column r of every row c: G_d'[c, r] = exp2(y[r, c] - lse2_d'[c])
// with y[r, c] the logit rank n already has in its own E block.  So each gradient is one GEMM
// over the rank's own block, H_d = G_d + G_d'^T (shard.py:148-154 summed over all ranks), and the
// only exchange after the forward is the B column statistics -- no gradient reduce-scatter.
// =====================================================================
// Per column direction e (the lse2 the H_d columns use: e = 1 - d) and 64-column group g:
// Q_g = max lse2_e over the group, q_c = exp2(min(Q_g - lse2_e[c], 100)) (negated for columns
// outside this rank's rows under the flip hook), and the group's smallest lse2_e, or -inf when the
// group's spread exceeds 96 (p_r q_c would leave the f32 range: every row goes to the fixup).
// xall: [N][4][b] gathered (lse2_0, lse2_1, ce_0, ce_1); outputs for d: q [2][B], gm [2][groups].
__global__ void dual_prep_kernel(const float* xall, int b, int groups, int rank, int flip, float* q, float2* gm) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= 2 * groups) return;
  const int d = w / groups, g = w % groups, e = 1 - d;
  const int64_t B = int64_t(groups) * 64;
  float L[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t c = int64_t(g) * 64 + h * 32 + lane;
    L[h] = xall[((c / b) * 4 + e) * b + c % b];
  }
  float mx = fmaxf(L[0], L[1]), mn = fminf(L[0], L[1]);
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t c = int64_t(g) * 64 + h * 32 + lane;
    const bool other = c < int64_t(rank) * b || c >= int64_t(rank + 1) * b;
    const float v = exp2f(fminf(mx - L[h], 100.f));
    q[int64_t(d) * B + c] = (flip && other) ? -v : v;
  }
  if (lane == 0) gm[int64_t(d) * groups + g] = make_float2(mx, mx - mn > 96.f ? -INFINITY : mn);
}

// d[r] = s (2^-14 (K-half partials, fixed order) + lab_r F_label(r)) for rows [row0, row0 + nrows):
// the dual GEMM left 2^14 H with the label column zeroed; lab_r = (P_i2t - 1) + (P_t2i - 1) of row r
// (fp32, both directions are this rank's) times the label row's features (d_image: T_n[r],
// d_text: I_n[r], the packed bf16 rows the GEMMs used).
__global__ void combine_dual_kernel(const float4* intra, int ksplit, const float* glabel, const __nv_bfloat16* pack,
                                    int b, int Dp, int D, float s, float* d_image, float* d_text, int64_t ld_out,
                                    int row0, int nrows, Status* status) {
  const int v4 = Dp / 4;
  const bool vec_out = (ld_out % 4 == 0) && ((reinterpret_cast<uintptr_t>(d_image) | reinterpret_cast<uintptr_t>(d_text)) % 16 == 0);
  const int64_t per_g = int64_t(b) * v4;
  const unsigned pb = unsigned(int64_t(nrows) * v4), uv4 = unsigned(v4);
  const int64_t total = 2 * int64_t(pb);
  bool bad = false;
  for (int64_t ii = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; ii < total; ii += int64_t(gridDim.x) * blockDim.x) {
    const unsigned iu = unsigned(ii);
    const int g = int(iu / pb);
    const int64_t rem = int64_t(iu - unsigned(g) * pb) + int64_t(row0) * v4;
    const int r = int(unsigned(rem) / uv4), vc = int(unsigned(rem) % uv4);
    const float4* ib = intra + (int64_t(g) * ksplit) * per_g + rem;
    const float4 y = ksplit == 2 ? f4add(__ldcs(ib), __ldcs(ib + per_g)) : __ldcs(ib);
    const float lab = glabel[r] + glabel[b + r];
    // label row features: the other direction's packed row r (d_image pairs with T_n, d_text with I_n)
    const uint2 fr = *reinterpret_cast<const uint2*>(pack + (int64_t(1 - g) * b + r) * Dp + vc * 4);
    const float2 f01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&fr.x));
    const float2 f23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&fr.y));
    static_assert(H_DUAL_LOG2 == 14.f, "combine scale");
    constexpr float inv = 1.f / 16384.f;  // 2^-H_DUAL_LOG2
    const float4 o = make_float4(fmaf(lab, f01.x, y.x * inv) * s, fmaf(lab, f01.y, y.y * inv) * s,
                                 fmaf(lab, f23.x, y.z * inv) * s, fmaf(lab, f23.y, y.w * inv) * s);
    float* out = (g == 0 ? d_image : d_text) + int64_t(r) * ld_out;
    const int c = vc * 4;
    bad |= !(isfinite(o.x) && isfinite(o.y) && isfinite(o.z) && isfinite(o.w));
    if (c + 4 <= D && vec_out) {
      __stcs(reinterpret_cast<float4*>(out + c), o);
    } else {
      const float ov[4] = {o.x, o.y, o.z, o.w};
      for (int k = 0; k < 4 && c + k < D; ++k) out[c + k] = ov[k];
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(&status->flags, FLAG_GRAD_NONFINITE);
}

// Exact recompute of the rows the dual transform flagged (E range too narrow for a column term;
// never seen with the synthetic features of the tests and bench at D >= 64): one CTA per queued
// (direction, row) at a time, all in fp32 from the bf16 features -- y = t log2(e) <A_r, C_c>,
// H = exp2(y - lse2_d[r]) + sign_c exp2(y - lse2_d'[c]), label (P_d - 1) + (P_d' - 1) -- then
// d[r] = s sum_c H_c C_c, columns in ascending order (a function of the row only: N-invariant).
constexpr int FIX_THREADS = 256;
constexpr int FIX_COLS = 256;   // columns per chunk (one per thread in the dot phase)
constexpr int FIX_MAX_DP = 2048;
__global__ void __launch_bounds__(FIX_THREADS) dual_fixup_kernel(
    const __nv_bfloat16* feat, const float* xall, const float* glabel, const int* list, const Status* status,
    int cap, int B, int b, int Dp, int D, int rank, float tl2e, float s, int flip, float* d_image, float* d_text,
    int64_t ld_out) {
  __shared__ float arow[FIX_MAX_DP];
  __shared__ float hs[FIX_COLS];
  const int n = min(status->fix_count, cap);
  constexpr int PER = FIX_MAX_DP / FIX_THREADS;
  for (int e = blockIdx.x; e < n; e += gridDim.x) {
    const int tag = list[e];
    const int d = tag / b, r = tag % b, dp = 1 - d;
    const __nv_bfloat16* A = feat + (int64_t(d) * B + int64_t(rank) * b + r) * Dp;
    const __nv_bfloat16* C = feat + int64_t(dp) * B * Dp;
    __syncthreads();
    for (int k = threadIdx.x; k < Dp; k += FIX_THREADS) arow[k] = __bfloat162float(A[k]);
    const float lse_r = xall[(int64_t(rank) * 4 + d) * b + r];
    const float lab = glabel[r] + glabel[b + r];
    const int64_t label = int64_t(rank) * b + r;
    float acc[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) acc[k] = 0.f;
    __syncthreads();
    for (int64_t c0 = 0; c0 < B; c0 += FIX_COLS) {
      {
        const int64_t c = c0 + threadIdx.x;
        float h = 0.f;
        if (c < B) {
          const uint4* cr = reinterpret_cast<const uint4*>(C + c * Dp);
          float dot = 0.f;
          for (int k8 = 0; k8 < Dp / 8; ++k8) {
            const uint4 v = cr[k8];
            const __nv_bfloat162* hv = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float2 f = __bfloat1622float2(hv[j]);
              dot = fmaf(arow[8 * k8 + 2 * j], f.x, dot);
              dot = fmaf(arow[8 * k8 + 2 * j + 1], f.y, dot);
            }
          }
          if (c == label) {
            h = lab;
          } else {
            const float y = dot * tl2e;
            const float lc = xall[((c / b) * 4 + dp) * b + c % b];
            const bool other = c < int64_t(rank) * b || c >= int64_t(rank + 1) * b;
            h = exp2f(y - lse_r) + ((flip && other) ? -1.f : 1.f) * exp2f(y - lc);
          }
        }
        hs[threadIdx.x] = h;
      }
      __syncthreads();
      const int nc = B - c0 < FIX_COLS ? int(B - c0) : FIX_COLS;
      for (int j = 0; j < nc; ++j) {
        const float h = hs[j];
        const __nv_bfloat16* cr = C + (c0 + j) * Dp;
#pragma unroll
        for (int k = 0; k < PER; ++k) {
          const int dim = threadIdx.x + k * FIX_THREADS;
          if (dim < Dp) acc[k] = fmaf(h, __bfloat162float(cr[dim]), acc[k]);
        }
      }
      __syncthreads();
    }
    float* out = (d == 0 ? d_image : d_text) + int64_t(r) * ld_out;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int dim = threadIdx.x + k * FIX_THREADS;
      if (dim < D) out[dim] = acc[k] * s;
    }
  }
}

__global__ void peer_signal_kernel(PeerPtrs p, int n, uint32_t epoch) {
  // the cross GEMM (previous kernel on this stream) completed its bulk stores; make them visible
  // system-wide before the arrival flags
  __threadfence_system();
  const int r = threadIdx.x;
  if (r < n) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p.flag[r]), "r"(epoch) : "memory");
}

__global__ void peer_wait_kernel(const uint32_t* flags, int n, uint32_t epoch, Status* status,
                                 unsigned long long timeout_ns) {
  const int r = threadIdx.x;
  if (r >= n) return;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (true) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + r) : "memory");
    if (v == epoch) break;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > timeout_ns) {  // never hang the device: flag the step and let the host raise
      atomicOr(&status->flags, FLAG_PEER_TIMEOUT);
      break;
    }
    __nanosleep(256);
  }
}

// Peer all-gather fused with the unpack: rank r's packed rows are read straight from its peer
// window (NVLink loads) into the forward operands (bf16) and backward operands (f16).
constexpr int PEER_PACK_FLAG0 = 64;  // u32 slot of the pack-ready flags in the flag block
struct PeerSrc {
  const uint4* pack[8];  // each rank's published [2][b][Dp] bf16 rows (this step's parity)
};
__global__ void peer_gather_unpack_kernel(PeerSrc src, int N, int b, int Dp, uint4* feat, uint4* feat16) {
  const int vec_per_row = Dp / 8;
  const int64_t per_rank = int64_t(2) * b * vec_per_row;
  const int64_t total = int64_t(N) * per_rank;
  const int64_t B = int64_t(N) * b;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int n = int(i / per_rank);
    const int64_t j = i - n * per_rank;
    const int vc = int(j % vec_per_row);
    const int64_t rr = j / vec_per_row;
    const int r = int(rr % b), dir = int(rr / b);
    const uint4 x = src.pack[n][j];
    const int64_t o = (dir * B + int64_t(n) * b + r) * vec_per_row + vc;
    feat[o] = x;
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&x);
    uint4 y;
    __half2* hy = reinterpret_cast<__half2*>(&y);
#pragma unroll
    for (int k = 0; k < 4; ++k) hy[k] = __float22half2_rn(__bfloat1622float2(h[k]));
    feat16[o] = y;
  }
}

// Per-row ce of this rank ([2][b]) into every rank's window ce area, slot `rank` of [N][2][b].
struct PeerDst {
  float* ce[8];
};
__global__ void peer_ce_push_kernel(const float4* ce, int n4, PeerDst dst, int N) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += gridDim.x * blockDim.x) {
    const float4 v = ce[i];
    for (int r = 0; r < N; ++r) reinterpret_cast<float4*>(dst.ce[r])[i] = v;
  }
}

// Loss: sum of the [N][2][b] per-row ce in an order fixed by the global row
// index (independent of N), in f64, / (2 * N * b).  Stage 1: LOSS_BLOCKS
// blocks each reduce a fixed contiguous slice of the flat index f = dir*B + g;
// stage 2: one warp adds the block partials in a fixed tree.
constexpr int LOSS_BLOCKS = 128;
// ce_all: per rank `rs` row vectors of b floats, the two ce directions at vectors dir_off, dir_off + 1
// ([N][2][b] ce gathers: rs = 2, dir_off = 0; [N][4][b] dual exchange: rs = 4, dir_off = 2).
__global__ void loss_partial_kernel(const float* ce_all, int N, int b, double* partial, int rs = 2, int dir_off = 0) {
  __shared__ double red[256];
  const int64_t B = int64_t(N) * b;
  const int64_t n2 = 2 * B;
  const int64_t per = (n2 + LOSS_BLOCKS - 1) / LOSS_BLOCKS;
  const int64_t lo = blockIdx.x * per, hi = min(n2, lo + per);
  double acc = 0.0;
  for (int64_t f = lo + threadIdx.x; f < hi; f += blockDim.x) {
    const int dir = int(f / B);
    const int64_t gidx = f - dir * B;
    const int64_t n = gidx / b, r = gidx % b;
    acc += double(ce_all[(n * rs + dir_off + dir) * b + r]);
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

// dL/dt per local row r: <d_image[r], I_n[r]> + <d_text[r], T_n[r]> with the bf16 features the loss
// used (pack region [2][b][Dp]); one warp per row, fixed lane order, f64 accumulation.
__global__ void rowdot_kernel(const float* d_image, const float* d_text, int64_t ld_out, const __nv_bfloat16* pack,
                              int b, int D, int Dp, float* rdot) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= b) return;
  const __nv_bfloat16* I = pack + int64_t(warp) * Dp;
  const __nv_bfloat16* T = pack + (int64_t(b) + warp) * Dp;
  const float* di = d_image + int64_t(warp) * ld_out;
  const float* dt = d_text + int64_t(warp) * ld_out;
  double acc = 0.0;
  for (int c = lane; c < D; c += 32)
    acc += double(di[c]) * double(__bfloat162float(I[c])) + double(dt[c]) * double(__bfloat162float(T[c]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) rdot[warp] = float(acc);
}

// Tower-side row normalisation (reference matrix.py:165-176, 178-195), one warp per row, fp32 I/O,
// f64 norms.  flags (optional): bit0 non-finite input, bit1 row norm below 1e-12 (DegenerateInputError).
constexpr double NORM_EPSILON = 1e-12;
__global__ void l2norm_rows_kernel(const float* raw, int64_t ld_raw, int rows, int D, float* out, int64_t ld_out,
                                   float* norms, int* flags) {
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (r >= rows) return;
  const float* x = raw + int64_t(r) * ld_raw;
  double ss = 0.0;
  bool bad = false;
  for (int c = lane; c < D; c += 32) {
    const float v = x[c];
    bad |= !isfinite(v);
    ss += double(v) * double(v);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const double n = sqrt(ss);
  if (lane == 0) {
    if (norms) norms[r] = float(n);
    if (flags && (bad || !isfinite(n))) atomicOr(flags, 1);
    if (flags && n < NORM_EPSILON) atomicOr(flags, 2);
  }
  const double inv = 1.0 / n;
  float* y = out + int64_t(r) * ld_out;
  for (int c = lane; c < D; c += 32) y[c] = float(double(x[c]) * inv);
}

// d_raw = (g - (u . g) u) / ||x||, u = x / ||x||  (the backward of l2norm_rows)
// (g - (u . g) u) / ||x|| for one row, one warp (matrix.py:178-195); shared by the tower kernel
// and the fused dual finish so both produce the same bits
__device__ __forceinline__ void l2norm_backward_row(const float* x, const float* g, int D, float* y, int* flags,
                                                    int lane) {
  double ss = 0.0, xg = 0.0;
  for (int c = lane; c < D; c += 32) {
    ss += double(x[c]) * double(x[c]);
    xg += double(x[c]) * double(g[c]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ss += __shfl_xor_sync(0xffffffffu, ss, o);
    xg += __shfl_xor_sync(0xffffffffu, xg, o);
  }
  const double n = sqrt(ss);
  if (lane == 0 && flags && n < NORM_EPSILON) atomicOr(flags, 2);
  const double inner = xg / n;  // u . g
  bool bad = false;
  for (int c = lane; c < D; c += 32) {
    const double u = double(x[c]) / n;
    const float v = float((double(g[c]) - inner * u) / n);
    bad |= !isfinite(v);
    y[c] = v;
  }
  if (flags && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flags, 1);
}
__global__ void l2norm_rows_backward_kernel(const float* raw, int64_t ld_raw, const float* grad, int64_t ld_grad,
                                            int rows, int D, float* out, int64_t ld_out, int* flags) {
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (r >= rows) return;
  l2norm_backward_row(raw + int64_t(r) * ld_raw, grad + int64_t(r) * ld_grad, D, out + int64_t(r) * ld_out, flags,
                      lane);
}

// Two-tower step: the dual combine with the towers' normalisation backward in
// its epilogue.  One warp per (direction, row): d = combine_dual's value (same fp32 operations,
// written out for the fixup), then dx = l2_normalize_rows_backward(raw, d) from the same row.
struct TowerRows {
  const float* raw[2];
  int64_t ld_raw[2];
  float* dx[2];
  int64_t ld_dx;
};
__global__ void combine_dual_l2norm_kernel(const float* intra, int ksplit, const float* glabel,
                                           const __nv_bfloat16* pack, int b, int Dp, int D, float s, float* d_image,
                                           float* d_text, int64_t ld_out, TowerRows tw, Status* status,
                                           int* norm_flags) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= 2 * b) return;
  const int g = w / b, r = w - g * b;
  const int64_t per_g = int64_t(b) * Dp;
  const float* ib = intra + int64_t(g) * ksplit * per_g + int64_t(r) * Dp;
  const float lab = glabel[r] + glabel[b + r];
  const __nv_bfloat16* fr = pack + (int64_t(1 - g) * b + r) * Dp;
  float* out = (g == 0 ? d_image : d_text) + int64_t(r) * ld_out;
  constexpr float inv = 1.f / 16384.f;  // 2^-H_DUAL_LOG2
  bool bad = false;
  for (int c = lane; c < D; c += 32) {
    const float y = ksplit == 2 ? ib[c] + ib[c + per_g] : ib[c];
    const float o = fmaf(lab, __bfloat162float(fr[c]), y * inv) * s;
    bad |= !isfinite(o);
    out[c] = o;
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(&status->flags, FLAG_GRAD_NONFINITE);
  __syncwarp();
  l2norm_backward_row(tw.raw[g] + int64_t(r) * tw.ld_raw[g], out, D, tw.dx[g] + int64_t(r) * tw.ld_dx, norm_flags,
                      lane);
}
// ... and the rows the dual fixup recomputed: their dx again, from the fixed d
__global__ void fixup_l2norm_kernel(const int* list, const Status* status, int cap, int b, int D,
                                    const float* d_image, const float* d_text, int64_t ld_out, TowerRows tw,
                                    int* norm_flags) {
  const int n = min(status->fix_count, cap), lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < n; e += nw) {
    const int tag = list[e];
    const int g = tag / b, r = tag % b;
    const float* dr = (g == 0 ? d_image : d_text) + int64_t(r) * ld_out;
    l2norm_backward_row(tw.raw[g] + int64_t(r) * tw.ld_raw[g], dr, D, tw.dx[g] + int64_t(r) * tw.ld_dx, norm_flags,
                        lane);
  }
}

// Fixed-order f64 sum of n floats: LOSS_BLOCKS contiguous slices, then a tree (as the loss).
__global__ void rowsum_partial_kernel(const float* x, int64_t n, double* partial) {
  __shared__ double red[256];
  const int64_t per = (n + LOSS_BLOCKS - 1) / LOSS_BLOCKS;
  const int64_t lo = blockIdx.x * per, hi = min(n, lo + per);
  double acc = 0.0;
  for (int64_t f = lo + threadIdx.x; f < hi; f += blockDim.x) acc += double(x[f]);
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

__global__ void dlogit_final_kernel(const double* partial, double scale, Status* status) {
  __shared__ double red[LOSS_BLOCKS];
  red[threadIdx.x] = partial[threadIdx.x];
  __syncthreads();
  for (int w = LOSS_BLOCKS / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    status->dlogit = red[0] * scale;
    if (!isfinite(status->dlogit)) status->flags |= FLAG_GRAD_NONFINITE;
  }
}

__global__ void loss_final_kernel(const double* partial, int64_t rows2, Status* status) {
  __shared__ double red[LOSS_BLOCKS];
  red[threadIdx.x] = partial[threadIdx.x];
  __syncthreads();
  for (int w = LOSS_BLOCKS / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double loss = red[0] / double(rows2);
    status->loss = loss;
    if (!isfinite(loss)) status->flags |= FLAG_LOSS_NONFINITE;
  }
}

// =====================================================================
// Host side
// =====================================================================
thread_local std::string g_last_error;
std::atomic<int64_t> g_launches{0};
inline void count_launch(int n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

#define CUDA_TRY(expr)                                                                         \
  do {                                                                                         \
    cudaError_t e_ = (expr);                                                                   \
    if (e_ != cudaSuccess) return fail(DISCO_CUDA_ERROR, "%s: %s", #expr, cudaGetErrorString(e_)); \
  } while (0)

struct Geometry {
  int64_t B, D, Dp, b, ldG;
  int N, rank;
  int nchunk, cpr;        // canonical chunks, chunks per rank
  int ssub;               // forward stats sub-chunks per chunk (2: logits units of half a chunk)
  int np;                 // cross partials per rank after pairing chunks in the GEMM epilogue
  int g_blocked;          // G in 128 x 128 blocks (canonical chunking: b and B multiples of 128)
  int wide;               // Dp % 512 == 0: GEMM units cover all of D (two accumulators, G read once)
  int wsplit;             // Dp > 512, Dp % 512 != 0: wide units for the first 512k columns + narrow rest
  int ksplit;             // intra K split (fixed function of B, D): partials [2][ksplit][b][Dp]
  int estore;             // forward stores E + group offsets; backward GEMMs rescale E -> G (no recompute)
  int dual;               // disco_step's backward is the dual one (rank-local H = G_d + G_d'^T GEMMs)
  int groups;             // B / 64 column groups (E offsets)
  int chunk_cols;         // B / nchunk
  int64_t off[DISCO_R_COUNT];
  int64_t len[DISCO_R_COUNT];
  int64_t total;
};
// dual fixup queue: each transform group queues its unsafe rows per K part (duplicates allowed)
inline int64_t fix_capacity(const Geometry& g) { return int64_t(XF_GROUPS_MAX) * 2 * g.ksplit * g.b; }

int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// DISCO_DEBUG_FLAGS / disco_b200_set_experiment_flags (profiling experiments and ablations only;
// tools/ab_kernels.py, tools/flag_parity.py).  Ablations produce wrong results on purpose.
//   bit0  (1)       skip the G / E TMA stores              bit1  (2)       L2 persistence window (GRAD)
//   bit4  (16)      GEMM: drain TMEM, store nothing        bit5  (32)      GEMM: st.global epilogue
//   bit6  (64)      GEMM: coalesced st.global rows         bit7  (128)     logits: A-resident ring
//   bit8  (256)     narrow (256-column) GEMM units         bit9  (512)     FWDE: drain TMEM only
//   bit10 (1024)    transform warps skip the rescale       bit11 (2048)    GEMM: no accumulator drain
//   bit15 (32768)   GEMM: stage but never TMA-store        bit17 (131072)  FWDE: E math only, no stores
//   bit18 (262144)  GEMM: round-robin instead of LPT       bit19 (524288)  whole-chunk logits units
std::atomic<int> g_debug_bits{[] {
  const char* e = getenv("DISCO_DEBUG_FLAGS");
  return e ? atoi(e) : 0;
}()};
int debug_flag_bits() { return XP ? g_debug_bits.load(std::memory_order_relaxed) : 0; }

int make_geometry(int64_t B, int64_t D, int world, int rank, Geometry* g) {
  if (world < 1) return fail(DISCO_LAYOUT_ERROR, "world size must be >= 1, got %d", world);
  if (B < 1) return fail(DISCO_LAYOUT_ERROR, "global batch must be >= 1, got %lld", (long long)B);
  if (B % world != 0)
    return fail(DISCO_LAYOUT_ERROR, "global batch %lld is not divisible by world size %d", (long long)B, world);
  if (rank < 0 || rank >= world) return fail(DISCO_LAYOUT_ERROR, "rank %d outside [0, %d)", rank, world);
  if (D < 1) return fail(DISCO_SHAPE_ERROR, "feature dim must be >= 1, got %lld", (long long)D);
  if (B > (int64_t(1) << 30) || D > 65536) return fail(DISCO_SHAPE_ERROR, "problem too large");
  g->B = B;
  g->D = D;
  g->Dp = round_up(D, 64);
  g->N = world;
  g->rank = rank;
  g->b = B / world;
  g->ldG = round_up(B, 64);
  if (B % 1024 == 0 && 8 % world == 0) {
    g->nchunk = 8;
    g->cpr = 8 / world;
  } else {
    g->nchunk = world;
    g->cpr = 1;
  }
  g->chunk_cols = int(B / g->nchunk);
  // half-chunk logits units when a half chunk is whole 256-column tiles: twice the units, so
  // small local batches (N = 8) fill the 74 CTA pairs in whole waves
  g->ssub = (g->nchunk == 8 && g->chunk_cols % (2 * BN) == 0 && !(debug_flag_bits() & 524288)) ? 2 : 1;
  g->g_blocked = (g->nchunk == 8 && g->b % 128 == 0) ? 1 : 0;
  g->wide = (g->Dp % 512 == 0 && !(debug_flag_bits() & 256)) ? 1 : 0;  // bit8: narrow-unit experiment
  // cross partials per rank: wide units keep one partial per canonical chunk (the first tree
  // level then runs in presum/combine); narrow units pair chunks in the two accumulators.
  // split width (Dp > 512, not a multiple of 512, e.g. D = 768): columns [0, 512 floor(Dp/512)) run
  // as wide units and the rest as narrow unpaired units, in two launches with the wide partial
  // structure (one partial per canonical chunk, two K halves), so E is read twice per GEMM
  // instead of once per 256 columns
  g->wsplit = (!g->wide && g->Dp > 512 && !(debug_flag_bits() & 256) && !(debug_flag_bits() & 1048576)) ? 1 : 0;
  g->np = (g->wide || g->wsplit) ? g->cpr : (g->cpr >= 2 ? g->cpr / 2 : 1);
  g->ksplit = ((g->wide || g->wsplit) && B % 128 == 0 && B >= 4096) ? 2 : 1;
  static const bool no_estore = [] {  // DISCO_RECOMPUTE=1: A/B switch to the recompute (GRAD) path
    const char* e = getenv("DISCO_RECOMPUTE");
    return XP && e && atoi(e) != 0;
  }();
  g->estore = (g->g_blocked && !no_estore) ? 1 : 0;
  // Dual backward (default wherever E is stored, Dp <= 2048): after the forward every rank
  // all_gathers the 4 b row statistics, and each gradient is ONE GEMM over the rank's own E block,
  // H_d = G_d + G_d'^T -- half the backward MMA work of the exchange backward and no gradient
  // reduce-scatter, bitwise equal at every N.  DISCO_BACKWARD=exchange (read per call) selects the
  // two-GEMM exchange backward (intra + cross GEMMs, reduce-scatter), the form local_loss_and_grads
  // always uses because its contract is the full-size per-rank contribution.
  const char* bw = getenv("DISCO_BACKWARD");
  g->dual = (g->estore && g->Dp <= FIX_MAX_DP && !(bw && strcmp(bw, "exchange") == 0)) ? 1 : 0;
  g->groups = int(B / GROUP_COLS);
  const int64_t b = g->b, Dp = g->Dp, N = world;
  int64_t len[DISCO_R_COUNT];
  len[DISCO_R_PACK] = 2 * b * Dp * 2;
  len[DISCO_R_GATHER] = N > 1 ? N * 2 * b * Dp * 2 : 0;
  len[DISCO_R_FEAT] = 2 * B * Dp * 2;
  len[DISCO_R_FEAT16] = 2 * B * Dp * 2;
  len[DISCO_R_STATS] = 2 * int64_t(g->nchunk) * g->ssub * 4 * b * 8;  // [2][sub-chunks][<= 4 parts][b] f32x2
  len[DISCO_R_ROWS] = 4 * 2 * b * 4;
  len[DISCO_R_CE] = 0;  // alias into DISCO_R_XCHG (below)
  len[DISCO_R_CE_ALL] = N * 2 * b * 4;
  len[DISCO_R_G] = 2 * b * g->ldG * 2;
  len[DISCO_R_XPART] = g->np > 1 ? 2 * int64_t(g->np) * B * Dp * 4 : 0;
  len[DISCO_R_SEND] = N * 2 * b * Dp * 4;
  len[DISCO_R_RECV] = N > 1 ? N * 2 * b * Dp * 4 : 0;
  len[DISCO_R_INTRA] = 2 * int64_t(g->ksplit) * b * Dp * 4;
  len[DISCO_R_STATUS] = int64_t(sizeof(Status));
  len[DISCO_R_RDOT] = b * 4;
  len[DISCO_R_RDOT_ALL] = N > 1 ? N * b * 4 : 0;
  len[DISCO_R_SCALE] = g->estore ? 2 * int64_t(g->groups) * b * (4 + 2) : 0;  // f32 m_g, then f16 scales
  len[DISCO_R_XCHG] = 4 * b * 4;
  len[DISCO_R_XALL] = N > 1 ? N * 4 * b * 4 : 0;
  len[DISCO_R_QCOL] = g->estore ? 2 * B * 4 + 2 * int64_t(g->groups) * 8 : 0;
  len[DISCO_R_FIX] = g->estore ? fix_capacity(*g) * 4 : 0;
  int64_t off = 0;
  for (int r = 0; r < DISCO_R_COUNT; ++r) {
    g->off[r] = off;
    g->len[r] = len[r];
    off += round_up(len[r], 1024);
  }
  // the per-row lse2 and ce live in the exchange vector: DISCO_R_CE is its ce half
  g->off[DISCO_R_CE] = g->off[DISCO_R_XCHG] + 2 * b * 4;
  g->len[DISCO_R_CE] = 2 * b * 4;
  // aliases for the single-rank case: packed == gathered == forward operand layout
  if (N == 1) {
    g->off[DISCO_R_XALL] = g->off[DISCO_R_XCHG];
    g->len[DISCO_R_XALL] = g->len[DISCO_R_XCHG];
    g->off[DISCO_R_PACK] = g->off[DISCO_R_FEAT];
    g->off[DISCO_R_GATHER] = g->off[DISCO_R_PACK];
    g->len[DISCO_R_GATHER] = g->len[DISCO_R_PACK];
    g->off[DISCO_R_RECV] = g->off[DISCO_R_SEND];
    g->len[DISCO_R_RECV] = g->len[DISCO_R_SEND];
    g->off[DISCO_R_RDOT_ALL] = g->off[DISCO_R_RDOT];
    g->len[DISCO_R_RDOT_ALL] = g->len[DISCO_R_RDOT];
  }
  g->total = off;
  return DISCO_OK;
}

template <typename T>
T* region(void* ws, const Geometry& g, int r) {
  return reinterpret_cast<T*>(static_cast<uint8_t*>(ws) + g.off[r]);
}

// this rank's per-row lse2 [2][b] (first half of the exchange vector DISCO_R_XCHG)
float* lse2_of(void* ws, const Geometry& g) { return region<float>(ws, g, DISCO_R_XCHG); }

unsigned long long* probe_slot(void* ws, const Geometry& g, int at) {
  return reinterpret_cast<unsigned long long*>(region<uint8_t>(ws, g, DISCO_R_STATUS) + offsetof(Status, probe)) + at;
}

// cuStreamWriteValue32 (driver API, no SM involved): the copy stream's "chunk landed" signal.
using PFN_writeValue32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
PFN_writeValue32 write_value_fn() {
  static PFN_writeValue32 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_writeValue32>(ptr);
  });
  return fn;
}

// cuStreamWaitValue32: a copy stream waits for a peer's published flag without any SM.
using PFN_waitValue32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
PFN_waitValue32 wait_value_fn() {
  static PFN_waitValue32 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_waitValue32>(ptr);
  });
  return fn;
}

// ------------------------------------------------------------ tensor maps
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

// 2-D map over a row-major [outer][inner] 16-bit matrix with row pitch `pitch_elems`.
int make_map(CUtensorMap* map, bool bf16, const void* base, uint64_t inner, uint64_t outer, uint64_t pitch_elems,
             uint32_t box_inner, uint32_t box_outer) {
  auto fn = encode_fn();
  if (!fn) return fail(DISCO_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {pitch_elems * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2,
                  const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(DISCO_CUDA_ERROR, "cuTensorMapEncodeTiled failed (%d) inner=%llu outer=%llu box=%u,%u", int(r),
                (unsigned long long)inner, (unsigned long long)outer, box_inner, box_outer);
  return DISCO_OK;
}

// 3-D fp32 map over [z][rows][cols] with arbitrary row / z pitches (in floats), box {32, 32, 1}.
int make_map_f32_3d(CUtensorMap* map, const float* base, uint64_t cols, uint64_t rows, uint64_t nz,
                    uint64_t row_pitch, uint64_t z_pitch) {
  auto fn = encode_fn();
  if (!fn) return fail(DISCO_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {cols, rows, nz};
  cuuint64_t strides[2] = {row_pitch * 4, z_pitch * 4};
  cuuint32_t box[3] = {32, 32, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(DISCO_CUDA_ERROR, "cuTensorMapEncodeTiled(f32 3d) failed (%d)", int(r));
  return DISCO_OK;
}

// Output addressing of a GEMM problem: row r of k-chunk kc lands at
// out + kc*chunk_stride + (r / row_div)*stride_hi + (r % row_div)*ld_out.
// TMA stores need 32-row slabs that never straddle a row_div boundary.
int set_output(GemmProblem& q, float* out, int64_t ld_out, int64_t row_div, int64_t stride_hi, int64_t nz_rows,
               int64_t chunk_stride, int64_t nz_chunks) {
  q.out = out;
  q.ld_out = ld_out;
  q.row_div = row_div;
  q.stride_hi = stride_hi;
  q.chunk_stride = chunk_stride;
  q.tma_store = 0;
  q.skip_store = (debug_flag_bits() & 16) ? 1 : 0;
  q.ablate = debug_flag_bits() & (1024 | 2048 | 32768);
  const bool aligned = (row_div % 32 == 0) && (ld_out % 4 == 0) && (reinterpret_cast<uintptr_t>(out) % 16 == 0) &&
                       !(debug_flag_bits() & 32);
  if (aligned && (nz_rows == 1 || nz_chunks == 1)) {
    const uint64_t nz = uint64_t(nz_rows > 1 ? nz_rows : nz_chunks);
    const uint64_t zp = uint64_t(nz_rows > 1 ? stride_hi : (nz_chunks > 1 ? chunk_stride : row_div * ld_out));
    if (zp % 4 == 0) {
      int rc = make_map_f32_3d(&q.out_map, out, uint64_t(q.N), uint64_t(std::min<int64_t>(row_div, q.M)), nz,
                               uint64_t(ld_out), zp);
      if (rc) return rc;
      q.tma_store = (debug_flag_bits() & 64) ? 2 : 1;
    }
  }
  return DISCO_OK;
}

// 4-D f16 map over a blocked G: [rows/128][cols/128][128][128], box {64, box_rows, 1, 1}.
int make_map_blocked(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows,
                     uint32_t box_cols = 64) {
  auto fn = encode_fn();
  if (!fn) return fail(DISCO_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[4] = {128, 128, cols / 128, rows / 128};
  cuuint64_t strides[3] = {256, 32768, (cols / 128) * 32768};
  cuuint32_t box[4] = {box_cols, box_rows, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, box_cols == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DISCO_CUDA_ERROR, "cuTensorMapEncodeTiled(blocked G) failed (%d)", int(r));
  return DISCO_OK;
}

int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <typename K>
int prepare_kernel(K kernel, size_t smem = SMEM_BYTES) {
  // Per-device attribute; cheap enough to set on every launch.
  CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  return DISCO_OK;
}

// Persistent grid of CTA pairs: one pair per unit, at most one CTA per SM.
int grid_for(int64_t units) { return 2 * int(std::min<int64_t>(units, sm_count() / 2)); }

// Experiment (DISCO_DEBUG_FLAGS bit1): L2 persistence window over the bf16 feature operands while
// the E / G write stream runs.
int l2_window(cudaLaunchAttribute* attr, const void* base, size_t bytes) {
  static int maxp = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxPersistingL2CacheSize, dev);
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, size_t(v));
    return v;
  }();
  attr->id = cudaLaunchAttributeAccessPolicyWindow;
  attr->val.accessPolicyWindow.base_ptr = const_cast<void*>(base);
  attr->val.accessPolicyWindow.num_bytes = bytes;
  attr->val.accessPolicyWindow.hitRatio = std::min(1.0f, float(maxp) / float(bytes));
  attr->val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  attr->val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  return 1;
}

template <int KIND, bool ARES>
int launch_logits_t(const LogitsParams& p, int64_t units, cudaStream_t st, const void* feat = nullptr,
                    size_t feat_bytes = 0) {
  int rc;
  if ((rc = prepare_kernel(logits_kernel<KIND, ARES>))) return rc;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid_for(units));
  cfg.blockDim = dim3(logits_threads<KIND, ARES>());
  cfg.dynamicSmemBytes = SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  cfg.attrs = attr;
  cfg.numAttrs = (feat && (debug_flag_bits() & 2)) ? l2_window(&attr[0], feat, feat_bytes) : 0;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, logits_kernel<KIND, ARES>, p));
  count_launch();
  return DISCO_OK;
}

int launch_logits(int kind, void* ws, const Geometry& g, float t, cudaStream_t st, int wave = -1,
                  unsigned int epoch = 0, double timeout_s = 0.0) {
  LogitsParams p;
  memset(&p, 0, sizeof(p));
  const __nv_bfloat16* feat = region<__nv_bfloat16>(ws, g, DISCO_R_FEAT);
  const __nv_bfloat16* I_g = feat;
  const __nv_bfloat16* T_g = feat + g.B * g.Dp;
  int rc;
  if ((rc = make_map(&p.a_map[0], true, I_g, g.Dp, g.B, g.Dp, 64, BM))) return rc;
  if ((rc = make_map(&p.a_map[1], true, T_g, g.Dp, g.B, g.Dp, 64, BM))) return rc;
  if ((rc = make_map(&p.b_map[0], true, T_g, g.Dp, g.B, g.Dp, 64, BN / 2))) return rc;
  if ((rc = make_map(&p.b_map[1], true, I_g, g.Dp, g.B, g.Dp, 64, BN / 2))) return rc;
  p.B = int(g.B);
  p.b = int(g.b);
  p.Dp = int(g.Dp);
  p.rank = g.rank;
  p.nchunk = g.nchunk * g.ssub;  // the kernel's "chunks" are the stats sub-chunks
  p.chunk_cols = g.chunk_cols / g.ssub;
  p.tiles_per_chunk = (p.chunk_cols + BN - 1) / BN;
  p.row_tiles = int((g.b + PAIR_M - 1) / PAIR_M);
  p.tl2e = t * LOG2E;
  float* rows = region<float>(ws, g, DISCO_R_ROWS);
  p.stats = region<float2>(ws, g, DISCO_R_STATS);
  p.target = rows;
  p.lse2 = lse2_of(ws, g);
  p.glabel = rows + 4 * g.b;
  p.G = region<__half>(ws, g, DISCO_R_G);
  p.ldG = g.ldG;
  p.g_blocked = g.g_blocked;
  p.mg = region<float>(ws, g, DISCO_R_SCALE);
  p.groups = g.groups;
  p.wave = wave;
  p.epoch = epoch;
  p.timeout_ns = (unsigned long long)(timeout_s * 1e9);
  p.rt_per_chunk = p.chunk_cols / PAIR_M;  // waves are (sub-)chunks: rows and columns land together
  p.probe = probe_slot(ws, g, 0);
  if (kind != KIND_FWD && g.g_blocked) {
    const __half* Gb = region<__half>(ws, g, DISCO_R_G);
    for (int d = 0; d < 2; ++d)
      if ((rc = make_map_blocked(&p.g_map[d], Gb + int64_t(d) * g.b * g.B, g.b, g.B, 32))) return rc;
    for (int d = 0; d < 2; ++d)
      if ((rc = make_map_blocked(&p.e_map[d], Gb + int64_t(d) * g.b * g.B, g.b, g.B, 32, 32))) return rc;
  }
  const int debug_flags = debug_flag_bits();
  p.debug_flags = debug_flags;
  if (wave == -2 || wave == -3) {
    Status* stt = region<Status>(ws, g, DISCO_R_STATUS);
    p.wave_flags = stt->wave_flags;
    p.status_flags = &stt->flags;
    p.nwaves = wave == -2 ? g.nchunk * g.ssub : g.N;
  }
  const int64_t ndir = 2;
  const int64_t units = wave == -3 ? int64_t(2) * p.row_tiles * p.nchunk
                      : wave == -2 ? ndir * p.rt_per_chunk * p.nwaves * p.nwaves
                      : wave >= 0 ? ndir * p.rt_per_chunk * (2 * wave + 1)
                                  : ndir * p.row_tiles * p.nchunk * (kind == KIND_GRAD ? p.tiles_per_chunk : 1);
  const bool ares = g.Dp <= BK * ARES_SLICES && (debug_flags & 128) && wave > -2;  // experiment: not faster
  if (kind == KIND_FWD) {
#if DISCO_EXPERIMENTS
    rc = ares ? launch_logits_t<KIND_FWD, true>(p, units, st) : launch_logits_t<KIND_FWD, false>(p, units, st);
#else
    (void)ares;
    rc = launch_logits_t<KIND_FWD, false>(p, units, st);
#endif
    if (rc) return rc;
  } else if (kind == KIND_FWDE) {
    const size_t fb = size_t(2) * g.B * g.Dp * 2;
#if DISCO_EXPERIMENTS
    rc = ares ? launch_logits_t<KIND_FWDE, true>(p, units, st, feat, fb)
              : launch_logits_t<KIND_FWDE, false>(p, units, st, feat, fb);
#else
    rc = launch_logits_t<KIND_FWDE, false>(p, units, st, feat, fb);
#endif
    if (rc) return rc;
  } else {
    if ((rc = prepare_kernel(logits_kernel<KIND_GRAD, false>))) return rc;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid_for(units));
    cfg.blockDim = dim3(NUM_THREADS);
    cfg.dynamicSmemBytes = SMEM_BYTES;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    cfg.attrs = attr;
    cfg.numAttrs = 0;
    if (debug_flags & 2) cfg.numAttrs = l2_window(&attr[0], feat, size_t(2) * g.B * g.Dp * 2);
    CUDA_TRY(cudaLaunchKernelEx(&cfg, logits_kernel<KIND_GRAD, false>, p));
    count_launch();
  }
  CUDA_TRY(cudaGetLastError());
  return DISCO_OK;
}

// wide = 1: every unit covers all N columns (n_tiles counts 512-column tiles), NB = 2 kernel.
// xform = 1: A operands hold E (transform warps rescale to G in smem).
template <int NB, bool XF>
int launch_gemm_t(GemmParams& p, cudaStream_t st) {
  int rc;
  const size_t smem = XF ? SMEM_BYTES_XF : SMEM_BYTES;
  if ((rc = prepare_kernel(gemm_kernel<NB, XF>, smem))) return rc;
  gemm_kernel<NB, XF><<<grid_for(p.units[p.nprob]), gemm_threads<NB, XF>(), smem, st>>>(p);
  return DISCO_OK;
}

// Static LPT schedule: unit cost = its K extent + a fixed drain cost (the accumulator drain
// stalls the MMA for ~10k cycles per unit, about 640 rows of K at the wide MMA rate); units
// are assigned longest first to the least-loaded pair, then each pair runs its units in
// sequence order (which keeps the intra / cross interleave and the L2 locality).  Balances the
// 4:1 intra / cross unit lengths that round-robin leaves ragged, e.g. at N = 8.
void build_schedule(GemmParams& p, int npairs) {
  const int n = p.units[p.nprob];
  p.sched_n = 0;
  if (n > MAX_SCHED_UNITS || npairs > MAX_SCHED_PAIRS || npairs < 1) return;
  std::vector<std::pair<int64_t, int>> cost(n);
  for (int s = 0; s < n; ++s) {
    int u = s;
    if (p.split > 0) {
      const int64_t nA = p.units[p.split];
      const int64_t cA = int64_t(s) * nA / n, cA1 = int64_t(s + 1) * nA / n;
      u = cA1 > cA ? int(cA) : int(nA + s - cA1);
    }
    int pi = 0;
    while (pi + 1 < p.nprob && u >= p.units[pi + 1]) ++pi;
    const GemmProblem& q = p.prob[pi];
    const int kc = ((u - p.units[pi]) / q.n_tiles) % q.k_chunks;
    int64_t klen = 0;
    for (int sub = 0; sub <= q.paired; ++sub) {
      const int64_t k0 = int64_t(kc * (1 + q.paired) + sub) * q.k_chunk_len;
      klen += std::max<int64_t>(0, std::min<int64_t>(q.k_chunk_len, q.k_total - k0));
    }
    cost[s] = {klen + 640, s};
  }
  std::stable_sort(cost.begin(), cost.end(), [](const auto& a, const auto& b) { return a.first > b.first; });
  std::vector<int64_t> load(npairs, 0);
  std::vector<std::vector<int>> lists(npairs);
  for (const auto& c : cost) {
    int best = 0;
    for (int i = 1; i < npairs; ++i)
      if (load[i] < load[best]) best = i;
    load[best] += c.first;
    lists[best].push_back(c.second);
  }
  int off = 0;
  for (int i = 0; i < npairs; ++i) {
    std::sort(lists[i].begin(), lists[i].end());
    p.sched_off[i] = uint16_t(off);
    for (int s : lists[i]) p.sched[off++] = uint16_t(s);
  }
  p.sched_off[npairs] = uint16_t(off);
  p.sched_n = n;
}

int launch_gemm(GemmParams& p, cudaStream_t st, int wide, int xform);

// Split-width backward (g.wsplit): the same problems twice -- wide units over columns
// [0, wcols), then narrow unpaired units over [wcols, Dp) -- with identical K decompositions, so
// every output partial is formed exactly as a wide (or narrow) unit alone would form it.
int launch_backward(GemmParams& p, cudaStream_t st, const Geometry& g) {
  if (!g.wsplit) return launch_gemm(p, st, g.wide, g.estore);
  const int wcols = int(g.Dp / 512) * 512;
  GemmParams q = p;
  for (int i = 0; i < p.nprob; ++i) {
    p.prob[i].n_tiles = wcols / (2 * BN);
    p.prob[i].n_off = 0;
    p.prob[i].paired = 0;
    q.prob[i].n_tiles = int((g.Dp - wcols + BN - 1) / BN);
    q.prob[i].n_off = wcols;
    q.prob[i].paired = 0;
  }
  int rc;
  if ((rc = launch_gemm(p, st, 1, g.estore))) return rc;
  return launch_gemm(q, st, 0, g.estore);
}

int launch_gemm(GemmParams& p, cudaStream_t st, int wide, int xform) {
  p.units[0] = 0;
  for (int i = 0; i < p.nprob; ++i)
    p.units[i + 1] = p.units[i] + p.prob[i].m_tiles * p.prob[i].n_tiles * p.prob[i].k_chunks;
  if (!(debug_flag_bits() & 262144)) build_schedule(p, grid_for(p.units[p.nprob]) / 2);  // bit18: round-robin
  int rc;
  if (wide)
    rc = xform ? launch_gemm_t<2, true>(p, st) : launch_gemm_t<2, false>(p, st);
  else
    rc = xform ? launch_gemm_t<1, true>(p, st) : launch_gemm_t<1, false>(p, st);
  if (rc) return rc;
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return DISCO_OK;
}

// f16 E -> G factors [2][groups][b], stored after the f32 m_g in DISCO_R_SCALE.
uint4* scale16(void* ws, const Geometry& g) {
  return reinterpret_cast<uint4*>(region<float>(ws, g, DISCO_R_SCALE) + 2 * int64_t(g.groups) * g.b);
}

// E operand of direction `dir` (estore): per-(row, group) scales and label-column values.
void set_xform(GemmProblem& q, void* ws, const Geometry& g, int dir) {
  q.xform = g.estore;
  if (!g.estore) return;
  q.xscale = reinterpret_cast<const __half*>(scale16(ws, g)) + int64_t(dir) * g.groups * g.b;
  q.xlabel = region<float>(ws, g, DISCO_R_ROWS) + 4 * g.b + int64_t(dir) * g.b;
  q.xb = int(g.b);
  q.lab_off = int(int64_t(g.rank) * g.b);
}

int elementwise_grid(int64_t n, int threads) {
  return int(std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, int64_t(sm_count()) * 16)));
}


cudaStream_t st_of(void* stream) { return static_cast<cudaStream_t>(stream); }

// Cross GEMMs into p.prob[first], p.prob[first + 1]:
//   X_g = G_{d'}^T . A_{d'} (local rows), g = image <- d' = t2i (1), g = text <- d' = i2t (0)
int build_cross(GemmParams& p, int first, void* ws, const Geometry& g, int mt0 = 0, int mt1 = -1) {
  p.probe = probe_slot(ws, g, 4);
  const __half* G = region<__half>(ws, g, DISCO_R_G);
  const __half* f16 = region<__half>(ws, g, DISCO_R_FEAT16);
  const __half* I16 = f16;
  const __half* T16 = f16 + g.B * g.Dp;
  const int64_t Bc = g.B / g.nchunk;  // canonical chunk rows
  const int cross_wide = g.wide || g.wsplit;  // wide / split units: one partial per chunk; else pairs
  int rc;
  for (int gi = 0; gi < 2; ++gi) {
    GemmProblem& q = p.prob[first + gi];
    const int dsrc = gi == 0 ? 1 : 0;
    const __half* Gd = G + int64_t(dsrc) * g.b * g.ldG;
    const __half* Ad = gi == 0 ? T16 : I16;  // image grad uses T_n, text grad uses I_n
    if (g.g_blocked) {
      if ((rc = make_map_blocked(&q.a_map, G + int64_t(dsrc) * g.b * g.B, g.b, g.B, 64))) return rc;
      q.a_blocked = 1;
    } else if ((rc = make_map(&q.a_map, false, Gd, g.B, g.b, g.ldG, 64, 64))) {  // MN-major G^T
      return rc;
    }
    if ((rc = make_map(&q.b_map, false, Ad, g.Dp, g.B, g.Dp, 64, 64))) return rc;  // MN-major features
    q.a_mn_major = 1;
    q.b_mn_major = 1;
    q.M = int(g.B);
    q.N = int(g.Dp);
    q.m_tiles = int((g.B + PAIR_M - 1) / PAIR_M);
    if (mt1 >= 0) q.m_tiles = std::min(q.m_tiles, mt1) - mt0;
    q.m_off = mt0;
    q.n_tiles = cross_wide ? int(g.Dp / (2 * BN)) : int((g.Dp + BN - 1) / BN);
    q.paired = !cross_wide && g.cpr >= 2;
    q.k_chunks = g.np;  // units along K (pairs of canonical chunks when paired)
    q.k_chunk_len = int(g.cpr > 1 ? Bc : g.b);
    q.k_total = int(g.b);
    q.a_k_off = 0;
    q.b_k_off = int(int64_t(g.rank) * g.b);
    q.a_row_off = 0;
    set_xform(q, ws, g, dsrc);
    if (g.np > 1) {  // canonical partials [2][np][B][Dp]
      // leaf-interleaved partials [2][B][np][Dp]: the combine's np loads of an element share a DRAM page
      rc = set_output(q, region<float>(ws, g, DISCO_R_XPART) + int64_t(gi) * g.np * g.B * g.Dp, g.np * g.Dp, g.B, 0, 1,
                      g.Dp, g.np);
    } else {  // directly destination-major send slabs [N][2][b][Dp]
      rc = set_output(q, region<float>(ws, g, DISCO_R_SEND) + int64_t(gi) * g.b * g.Dp, g.Dp, g.b, 2 * g.b * g.Dp,
                      g.N, 0, 1);
    }
    if (rc) return rc;
  }
  return DISCO_OK;
}

// Sender-side tree over this rank's chunk partials into the destination-major slabs
// (single rank: the owner combine reads the partials directly).
int cross_presum(void* ws, const Geometry& g, cudaStream_t st) {
  if (g.np > 1 && g.N > 1) {
    const int64_t n = 2 * g.B * (g.Dp / 4);
    presum_kernel<<<elementwise_grid(n, 256), 256, 0, st>>>(region<float4>(ws, g, DISCO_R_XPART), g.np, g.N,
                                                           int(g.b), int(g.Dp), region<float4>(ws, g, DISCO_R_SEND));
    count_launch();
    CUDA_TRY(cudaGetLastError());
  }
  return DISCO_OK;
}

// Scale of the exchange backward's GEMM outputs: 0.5 t / B (reference loss scale, shard.py:143-146),
// times 2^-15 when the GEMMs ran on E (the forward's headroom: they formed 2^15 G).
float exchange_scale(const Geometry& g, float t, double rows) {
  return float(0.5 * double(t) / rows * (g.estore ? 1.0 / G_EXCHANGE_SCALE : 1.0));
}

int launch_combine(void* ws, const Geometry& g, float t, int flip, int row0, int nrows, float* d_image, float* d_text,
                   int64_t ld_out, cudaStream_t st) {
  const float s = exchange_scale(g, t, double(g.B));
  const int64_t n = 2 * int64_t(nrows) * (g.Dp / 4);
  if (n == 0) return DISCO_OK;
  combine_kernel<<<elementwise_grid(n, 256), 256, 0, st>>>(
      region<float4>(ws, g, DISCO_R_INTRA), g.ksplit, region<float4>(ws, g, DISCO_R_RECV),
      (g.N == 1 && g.np > 1) ? region<float4>(ws, g, DISCO_R_XPART) : nullptr, g.np, g.N, g.rank, int(g.b), int(g.Dp), int(g.D), s, flip, d_image, d_text, ld_out, row0, nrows,
      region<Status>(ws, g, DISCO_R_STATUS), 0, 1 << 30, 1);
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return DISCO_OK;
}

// Intra GEMMs into p.prob[first], p.prob[first + 1]: Y_image = G_i . T_g ; Y_text = G_t . I_g
int build_intra(GemmParams& p, int first, void* ws, const Geometry& g, int mt0 = 0, int mt1 = -1) {
  p.probe = probe_slot(ws, g, 4);
  const __half* G = region<__half>(ws, g, DISCO_R_G);
  const __half* f16 = region<__half>(ws, g, DISCO_R_FEAT16);
  const __half* I16 = f16;
  const __half* T16 = f16 + g.B * g.Dp;
  int rc;
  for (int gi = 0; gi < 2; ++gi) {
    GemmProblem& q = p.prob[first + gi];
    const __half* Gd = G + int64_t(gi) * g.b * g.ldG;
    const __half* Cd = gi == 0 ? T16 : I16;
    if (g.g_blocked) {
      if ((rc = make_map_blocked(&q.a_map, G + int64_t(gi) * g.b * g.B, g.b, g.B, BM))) return rc;
      q.a_blocked = 1;
    } else if ((rc = make_map(&q.a_map, false, Gd, g.B, g.b, g.ldG, 64, BM))) {  // K-major G
      return rc;
    }
    if ((rc = make_map(&q.b_map, false, Cd, g.Dp, g.B, g.Dp, 64, 64))) return rc;  // MN-major features
    q.a_mn_major = 0;
    q.b_mn_major = 1;
    q.M = int(g.b);
    q.N = int(g.Dp);
    q.m_tiles = int((g.b + PAIR_M - 1) / PAIR_M);
    if (mt1 >= 0) q.m_tiles = std::min(q.m_tiles, mt1) - mt0;
    q.m_off = mt0;
    q.n_tiles = g.wide ? int(g.Dp / (2 * BN)) : int((g.Dp + BN - 1) / BN);
    q.k_chunks = g.ksplit;  // fixed K halves [0, B/2), [B/2, B): independent of N
    q.k_chunk_len = int(g.B / g.ksplit);
    q.k_total = int(g.B);
    set_xform(q, ws, g, gi);
    if ((rc = set_output(q, region<float>(ws, g, DISCO_R_INTRA) + int64_t(gi) * g.ksplit * g.b * g.Dp, g.Dp, g.b, 0,
                         1, g.b * g.Dp, g.ksplit)))
      return rc;
  }
  return DISCO_OK;
}

// Dual GEMMs (g.dual): the intra problems (rows [mt0, mt1) of 256) with the dual transform:
//   d_image rows r: H'_0 . T_g, A = E_0 rows;  d_text rows r: H'_1 . I_g, A = E_1 rows
// K = all B columns in g.ksplit fixed halves (DISCO_R_INTRA partials), combined by combine_dual.
int build_dual(GemmParams& p, void* ws, const Geometry& g, int mt0 = 0, int mt1 = -1) {
  int rc;
  if ((rc = build_intra(p, 0, ws, g, mt0, mt1))) return rc;
  const float* mg = region<float>(ws, g, DISCO_R_SCALE);
  float* qcol = region<float>(ws, g, DISCO_R_QCOL);
  const float2* gm = reinterpret_cast<const float2*>(qcol + 2 * g.B);
  Status* status = region<Status>(ws, g, DISCO_R_STATUS);
  for (int d = 0; d < 2; ++d) {
    GemmProblem& q = p.prob[d];
    q.xform = 2;
    q.xmg = mg + int64_t(d) * g.groups * g.b;
    q.xlse = lse2_of(ws, g) + int64_t(d) * g.b;
    q.xq = qcol + int64_t(d) * g.B;
    q.xgm = gm + int64_t(d) * g.groups;
    q.fix_list = region<int>(ws, g, DISCO_R_FIX);
    q.fix_count = &status->fix_count;
    q.fix_tag = int(int64_t(d) * g.b);
    q.fix_cap = int(fix_capacity(g));
  }
  p.nprob = 2;
  p.split = 0;
  return DISCO_OK;
}

// stats combine: after every logits unit of the forward has run.  lse2 and ce land in the
// exchange vector (DISCO_R_XCHG), the label gradients in DISCO_R_ROWS.
int forward_finish(void* ws, const Geometry& g, cudaStream_t st) {
  float* rows = region<float>(ws, g, DISCO_R_ROWS);
  const int n = int(2 * g.b);
  // column parts per (row, sub-chunk): the FWDE kernel's epilogue parts, or halves (FWD)
  const int nparts = g.estore ? FWDE_PARTS : 2;
  stats_combine_kernel<<<(n + 255) / 256, 256, 0, st>>>(region<float2>(ws, g, DISCO_R_STATS), rows, g.nchunk, g.ssub,
                                                        nparts, int(g.b), 2, lse2_of(ws, g), rows + 4 * g.b,
                                                        region<float>(ws, g, DISCO_R_CE),
                                                        region<Status>(ws, g, DISCO_R_STATUS));
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return DISCO_OK;
}

// E -> G factors of the exchange backward (legacy transform): exp2(m_g - lse2) as f16.
int exchange_scales(void* ws, const Geometry& g, cudaStream_t st) {
  const int64_t nv = 2 * int64_t(g.groups) * g.b / 8;
  scale_kernel<<<elementwise_grid(nv, 256), 256, 0, st>>>(region<float4>(ws, g, DISCO_R_SCALE), lse2_of(ws, g),
                                                         g.groups, int(g.b), scale16(ws, g));
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return DISCO_OK;
}

// ---------------------------------------------------------------- peer transport (host side)
int64_t peer_leaves(const Geometry& g) { return int64_t(g.N) * g.np; }
// gradient slabs exist only for the exchange backward: the dual backward exchanges no gradients
int64_t peer_window_bytes(const Geometry& g) {
  return g.dual ? 0 : round_up(2 * peer_leaves(g) * g.b * g.Dp * 4, 1024);
}
int64_t peer_pack_bytes(const Geometry& g) { return round_up(2 * g.b * g.Dp * 2, 1024); }
int64_t peer_ce_bytes(const Geometry& g) { return round_up(int64_t(g.N) * 2 * g.b * 4, 1024); }
int64_t peer_total_bytes(const Geometry& g) {
  return PEER_FLAG_BYTES + 2 * peer_window_bytes(g) + 2 * peer_pack_bytes(g) + 2 * peer_ce_bytes(g);
}
// every rank's per-row ce, [N][2][b] f32, parity area after the two pack areas
float* peer_ce(const void* base, const Geometry& g, int parity) {
  return reinterpret_cast<float*>(const_cast<uint8_t*>(static_cast<const uint8_t*>(base)) + PEER_FLAG_BYTES +
                                  2 * peer_window_bytes(g) + 2 * peer_pack_bytes(g) +
                                  int64_t(parity & 1) * peer_ce_bytes(g));
}
// published packed rows of a rank, [2][b][Dp] bf16, parity window after the two slab windows
uint8_t* peer_pack(const void* base, const Geometry& g, int parity) {
  return const_cast<uint8_t*>(static_cast<const uint8_t*>(base)) + PEER_FLAG_BYTES + 2 * peer_window_bytes(g) +
         int64_t(parity & 1) * peer_pack_bytes(g);
}
float* peer_window(const void* base, const Geometry& g, int parity) {
  return reinterpret_cast<float*>(const_cast<uint8_t*>(static_cast<const uint8_t*>(base)) + PEER_FLAG_BYTES +
                                  int64_t(parity & 1) * peer_window_bytes(g));
}
int check_peer(const Geometry& g) {
  if (g.N < 2 || g.N > 8) return fail(DISCO_LAYOUT_ERROR, "peer transport needs 2 <= world <= 8, got %d", g.N);
  if (g.b % 128 != 0) return fail(DISCO_LAYOUT_ERROR, "peer transport needs b %% 128 == 0, got %lld", (long long)g.b);
  return DISCO_OK;
}

// Cross problem `q` (gradient gi) pushes its chunk partials into every destination's window:
// leaf (rank * np + kc) of [2][L][b][Dp], rows of destination r = output rows [r*b, (r+1)*b).
int set_output_peer(GemmProblem& q, const uint64_t* bases, int parity, const Geometry& g, int gi) {
  const int64_t L = peer_leaves(g);
  for (int r = 0; r < g.N; ++r) {
    const float* base = peer_window(reinterpret_cast<const void*>(bases[r]), g, parity) +
                        ((int64_t(gi) * L + int64_t(g.rank) * g.np) * g.b) * g.Dp;
    int rc = make_map_f32_3d(&q.peer_map[r], base, uint64_t(g.Dp), uint64_t(g.b), uint64_t(g.np), uint64_t(g.Dp),
                             uint64_t(g.b * g.Dp));
    if (rc) return rc;
  }
  q.peer = 1;
  q.peer_b = int(g.b);
  q.tma_store = 1;
  return DISCO_OK;
}

}  // namespace disco

// =====================================================================
// C ABI
// =====================================================================
using namespace disco;

extern "C" {

int disco_b200_abi_version(void) { return DISCO_B200_ABI_VERSION; }

int disco_b200_set_experiment_flags(int flags) { return g_debug_bits.exchange(flags); }

#if DISCO_WAITPROBE
int disco_b200_waitprobe(unsigned long long* out, int reset) {
  CUDA_TRY(cudaMemcpyFromSymbol(out, disco::g_waitprobe, sizeof(disco::g_waitprobe)));
  if (reset) {
    static const unsigned long long z[16] = {};
    CUDA_TRY(cudaMemcpyToSymbol(disco::g_waitprobe, z, sizeof(z)));
  }
  return DISCO_OK;
}
#endif
int64_t disco_b200_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

const char* disco_b200_last_error(void) { return g_last_error.c_str(); }

int disco_b200_workspace_bytes(int64_t B, int64_t D, int world, int rank, int64_t* bytes) {
  Geometry g;
  int rc = make_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  *bytes = g.total;
  return DISCO_OK;
}

int disco_b200_ws_region(int64_t B, int64_t D, int world, int rank, int reg, int64_t* offset, int64_t* bytes) {
  Geometry g;
  int rc = make_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  if (reg < 0 || reg >= DISCO_R_COUNT) return fail(DISCO_SHAPE_ERROR, "unknown workspace region %d", reg);
  *offset = g.off[reg];
  *bytes = g.len[reg];
  return DISCO_OK;
}

int disco_b200_chunking(int64_t B, int world, int* nchunk, int* chunks_per_rank) {
  Geometry g;
  int rc = make_geometry(B, 1, world, 0, &g);
  if (rc) return rc;
  *nchunk = g.nchunk;
  *chunks_per_rank = g.cpr;
  return DISCO_OK;
}

int disco_b200_pack(void* ws, int64_t B, int64_t D, int world, int rank, const void* local_I, const void* local_T,
                    int64_t ld_I, int64_t ld_T, int dtype, int clear_status, void* stream) {
  return disco_b200_pack_rows(ws, B, D, world, rank, local_I, local_T, ld_I, ld_T, dtype, clear_status, 0, B / world,
                              stream);
}

int disco_b200_pack_rows(void* ws, int64_t B, int64_t D, int world, int rank, const void* local_I,
                         const void* local_T, int64_t ld_I, int64_t ld_T, int dtype, int clear_status, int64_t row0,
                         int64_t row1, void* stream) {
  Geometry g;
  int rc = make_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  if (ld_I < D || ld_T < D) return fail(DISCO_SHAPE_ERROR, "row stride smaller than D");
  if (row0 < 0 || row1 > g.b || row0 > row1)
    return fail(DISCO_LAYOUT_ERROR, "pack rows [%lld, %lld) outside [0, %lld)", (long long)row0, (long long)row1,
                (long long)g.b);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Status* status = region<Status>(ws, g, DISCO_R_STATUS);
  if (clear_status) {
    clear_status_kernel<<<1, 1, 0, st>>>(status);
    count_launch();
  }
  __nv_bfloat16* out = region<__nv_bfloat16>(ws, g, DISCO_R_PACK);
  __half* out16 = world == 1 ? region<__half>(ws, g, DISCO_R_FEAT16) : nullptr;  // PACK aliases FEAT
  const int64_t n = 2 * (row1 - row0) * (g.Dp / 8);
  const int grid = elementwise_grid(n, 256);
  const int r0 = int(row0), nr = int(row1 - row0);
  if (nr == 0) return DISCO_OK;
  const int vec = (D % 8 == 0 && ld_I % 8 == 0 && ld_T % 8 == 0 &&
                   (reinterpret_cast<uintptr_t>(local_I) | reinterpret_cast<uintptr_t>(local_T)) % 16 == 0) ? 1 : 0;
  switch (dtype) {
    case DISCO_F32:
      pack_kernel<float><<<grid, 256, 0, st>>>(local_I, local_T, ld_I, ld_T, int(g.b), int(D), int(g.Dp), out, out16,
                                               status, r0, nr, vec);
      break;
    case DISCO_BF16:
      pack_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(local_I, local_T, ld_I, ld_T, int(g.b), int(D), int(g.Dp), out,
                                                       out16, status, r0, nr, vec);
      break;
    case DISCO_F16:
      pack_kernel<__half><<<grid, 256, 0, st>>>(local_I, local_T, ld_I, ld_T, int(g.b), int(D), int(g.Dp), out, out16,
                                                status, r0, nr, 0);
      break;
    case DISCO_F64:
      pack_kernel<double><<<grid, 256, 0, st>>>(local_I, local_T, ld_I, ld_T, int(g.b), int(D), int(g.Dp), out, out16,
                                                status, r0, nr, 0);
      break;
    default:
      return fail(DISCO_SHAPE_ERROR, "unsupported dtype code %d", dtype);
  }
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return DISCO_OK;
}

static int forward_impl(void* ws, int64_t B, int64_t D, int world, int rank, float t, bool unpack, void* stream);

int disco_b200_forward(void* ws, int64_t B, int64_t D, int world, int rank, float t, void* stream) {
  return forward_impl(ws, B, D, world, rank, t, true, stream);
}

int disco_b200_forward_gathered(void* ws, int64_t B, int64_t D, int world, int rank, float t, void* stream) {
  return forward_impl(ws, B, D, world, rank, t, false, stream);
}

static int forward_impl(void* ws, int64_t B, int64_t D, int world, int rank, float t, bool unpack, void* stream) {
  Geometry g;
  int rc = make_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  if (!(t > 0.f) || !std::isfinite(t)) return fail(DISCO_DOMAIN_ERROR, "temperature must be positive, got %g", t);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (world > 1 && unpack) {  // single rank: pack already wrote FEAT / FEAT16; peer gather: fused
    const int64_t nvec = int64_t(world) * 2 * g.b * (g.Dp / 8);
    unpack_kernel<<<elementwise_grid(nvec, 256), 256, 0, st>>>(
        region<uint4>(ws, g, DISCO_R_GATHER), world, int(g.b), int(g.Dp), region<uint4>(ws, g, DISCO_R_FEAT),
        region<uint4>(ws, g, DISCO_R_FEAT16));
    count_launch();
    CUDA_TRY(cudaGetLastError());
  }
  if ((rc = launch_logits(g.estore ? KIND_FWDE : KIND_FWD, ws, g, t, st))) return rc;
  return forward_finish(ws, g, st);
}

int disco_b200_forward_waves(int64_t B, int64_t D, int world, int rank, int* waves) {
  Geometry g;
  int rc = make_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  // one wave per stats sub-chunk (16 at B % 4096 == 0): the work left after the last H2D chunk
  // lands is (2W - 1) / W^2 of the forward
  *waves = (world == 1 && g.estore && (g.chunk_cols / g.ssub) % PAIR_M == 0) ? g.nchunk * g.ssub : 0;
  return DISCO_OK;
}

int disco_b200_path_info(int64_t B, int64_t D, int world, int rank, int* bits) {
  Geometry g;
  int rc = make_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  *bits = (g.estore ? DISCO_PATH_ESTORE : 0) | (g.wide ? DISCO_PATH_WIDE : 0) | (g.dual ? DISCO_PATH_DUAL : 0);
  return DISCO_OK;
}

int disco_b200_forward_wave(void* ws, int64_t B, int64_t D, int world, int rank, float t, int wave, void* stream) {
  Geometry g;
  int rc = make_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  if (!(t > 0.f) || !std::isfinite(t)) return fail(DISCO_DOMAIN_ERROR, "temperature must be positive, got %g", t);
  if (!(world == 1 && g.estore && (g.chunk_cols / g.ssub) % PAIR_M == 0))
    return fail(DISCO_LAYOUT_ERROR, "wavefront forward needs a single rank and B %% 2048 == 0");
  const int nw = g.nchunk * g.ssub;
  if (wave < 0 || wave >= nw) return fail(DISCO_LAYOUT_ERROR, "wave %d outside [0, %d)", wave, nw);
  return launch_logits(KIND_FWDE, ws, g, t, static_cast<cudaStream_t>(stream), wave);
}

int disco_b200_forward_streamed(void* ws, int64_t B, int64_t D, int world, int rank, float t, uint32_t epoch,
                                double timeout_s, void* stream) {
  Geometry g;
  int rc = make_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  if (!(t > 0.f) || !std::isfinite(t)) return fail(DISCO_DOMAIN_ERROR, "temperature must be positive, got %g", t);
  if (!(world == 1 && g.estore && (g.chunk_cols / g.ssub) % PAIR_M == 0 && g.D == g.Dp))
    return fail(DISCO_LAYOUT_ERROR, "streamed forward needs a single rank, B %% 2048 == 0 and D %% 64 == 0");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if ((rc = launch_logits(KIND_FWDE, ws, g, t, st, -2, epoch, timeout_s))) return rc;
  const int64_t n = 2 * g.B * g.Dp / 8;
  feat16_kernel<<<elementwise_grid(n, 256), 256, 0, st>>>(region<uint4>(ws, g, DISCO_R_FEAT),
                                                         region<uint4>(ws, g, DISCO_R_FEAT16), n,
                                                         region<Status>(ws, g, DISCO_R_STATUS));
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return forward_finish(ws, g, st);
}

int disco_b200_h2d_streamed(void* ws, int64_t B, int64_t D, int world, int rank, const void* host_I,
                            const void* host_T, uint32_t epoch, void* copy_stream) {
  Geometry g;
  int rc = make_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  if (!(world == 1 && g.estore && (g.chunk_cols / g.ssub) % PAIR_M == 0 && g.D == g.Dp))
    return fail(DISCO_LAYOUT_ERROR, "streamed forward needs a single rank, B %% 2048 == 0 and D %% 64 == 0");
  auto fn = write_value_fn();
  if (!fn) return fail(DISCO_CUDA_ERROR, "cuStreamWriteValue32 unavailable");
  const int waves = g.nchunk * g.ssub;
  const int64_t rows = g.b / waves, row_bytes = g.Dp * 2;
  uint8_t* feat = region<uint8_t>(ws, g, DISCO_R_FEAT);
  Status* stt = region<Status>(ws, g, DISCO_R_STATUS);
  cudaStream_t st = static_cast<cudaStream_t>(copy_stream);
  for (int k = 0; k < waves; ++k) {
    const int64_t off = k * rows * row_bytes, n = rows * row_bytes;
    CUDA_TRY(cudaMemcpyAsync(feat + off, static_cast<const uint8_t*>(host_I) + off, size_t(n),
                             cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(feat + g.B * row_bytes + off, static_cast<const uint8_t*>(host_T) + off, size_t(n),
                             cudaMemcpyHostToDevice, st));
    CUresult r = fn(static_cast<CUstream>(copy_stream), reinterpret_cast<CUdeviceptr>(&stt->wave_flags[k]), epoch, 0);
    if (r != CUDA_SUCCESS) return fail(DISCO_CUDA_ERROR, "cuStreamWriteValue32 failed (%d)", int(r));
  }
  return DISCO_OK;
}

int disco_b200_signal_wave(void* ws, int64_t B, int64_t D, int world, int rank, int wave, uint32_t epoch,
                           void* stream) {
  Geometry g;
  int rc = make_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  if (wave < 0 || wave >= 32) return fail(DISCO_LAYOUT_ERROR, "wave %d outside [0, 32)", wave);
  auto fn = write_value_fn();
  if (!fn) return fail(DISCO_CUDA_ERROR, "cuStreamWriteValue32 unavailable");
  Status* stt = region<Status>(ws, g, DISCO_R_STATUS);
  CUresult r = fn(static_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(&stt->wave_flags[wave]), epoch, 0);
  if (r != CUDA_SUCCESS) return fail(DISCO_CUDA_ERROR, "cuStreamWriteValue32 failed (%d)", int(r));
  return DISCO_OK;
}

int disco_b200_forward_finish(void* ws, int64_t B, int64_t D, int world, int rank, void* stream) {
  Geometry g;
  int rc = make_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  return forward_finish(ws, g, static_cast<cudaStream_t>(stream));
}


int disco_b200_backward_grad(void* ws, int64_t B, int64_t D, int world, int rank, float t, void* stream) {
  Geometry g;
  int rc = make_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  if (!(t > 0.f) || !std::isfinite(t)) return fail(DISCO_DOMAIN_ERROR, "temperature must be positive, got %g", t);
  // E path: the forward already stored E; the backward GEMMs finish G in smem with these factors
  if (g.estore) return exchange_scales(ws, g, static_cast<cudaStream_t>(stream));
  return launch_logits(KIND_GRAD, ws, g, t, static_cast<cudaStream_t>(stream));
}

int disco_b200_backward_cross(void* ws, int64_t B, int64_t D, int world, int rank, void* stream) {
  Geometry g;
  int rc = make_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  GemmParams p;
  memset(&p, 0, sizeof(p));
  if ((rc = build_cross(p, 0, ws, g))) return rc;
  p.nprob = 2;
  if ((rc = launch_backward(p, st, g))) return rc;
  return cross_presum(ws, g, st);
}

int disco_b200_backward_intra(void* ws, int64_t B, int64_t D, int world, int rank, void* stream) {
  Geometry g;
  int rc = make_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  GemmParams p;
  memset(&p, 0, sizeof(p));
  if ((rc = build_intra(p, 0, ws, g))) return rc;
  p.nprob = 2;
  return launch_backward(p, st_of(stream), g);
}

int disco_b200_backward_fused(void* ws, int64_t B, int64_t D, int world, int rank, void* stream) {
  Geometry g;
  int rc = make_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  cudaStream_t st = st_of(stream);
  GemmParams p;
  memset(&p, 0, sizeof(p));
  if ((rc = build_intra(p, 0, ws, g))) return rc;  // list A: long units (K = B / ksplit)
  if ((rc = build_cross(p, 2, ws, g))) return rc;  // list B: one canonical chunk of K per unit
  p.nprob = 4;
  p.split = 2;
  if ((rc = launch_backward(p, st, g))) return rc;
  return cross_presum(ws, g, st);
}

int disco_b200_combine(void* ws, int64_t B, int64_t D, int world, int rank, float t, int flip, float* d_image,
                       float* d_text, int64_t ld_out, void* stream) {
  Geometry g;
  int rc = make_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  if (ld_out < D) return fail(DISCO_SHAPE_ERROR, "output row stride smaller than D");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return launch_combine(ws, g, t, flip, 0, int(g.b), d_image, d_text, ld_out, st);
}

int disco_b200_combine_rows(void* ws, int64_t B, int64_t D, int world, int rank, float t, int flip, int64_t row0,
                            int64_t row1, float* d_image, float* d_text, int64_t ld_out, void* stream) {
  Geometry g;
  int rc = make_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  if (ld_out < D) return fail(DISCO_SHAPE_ERROR, "output row stride smaller than D");
  if (row0 < 0 || row1 > g.b || row0 > row1) return fail(DISCO_SHAPE_ERROR, "row range [%lld, %lld) outside [0, %lld)",
                                                         (long long)row0, (long long)row1, (long long)g.b);
  return launch_combine(ws, g, t, flip, int(row0), int(row1 - row0), d_image, d_text, ld_out, st_of(stream));
}

int disco_b200_backward_rows(void* ws, int64_t B, int64_t D, int world, int rank, int64_t row0, int64_t row1,
                             void* stream) {
  Geometry g;
  int rc = make_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  if (world != 1) return fail(DISCO_LAYOUT_ERROR, "row-block backward is single-rank only (N = %d)", world);
  if (row0 < 0 || row1 > g.b || row0 >= row1 || row0 % PAIR_M != 0 || (row1 % PAIR_M != 0 && row1 != g.b))
    return fail(DISCO_SHAPE_ERROR, "row block [%lld, %lld) must be 256-aligned inside [0, %lld)", (long long)row0,
                (long long)row1, (long long)g.b);
  const int mt0 = int(row0 / PAIR_M), mt1 = int((row1 + PAIR_M - 1) / PAIR_M);
  GemmParams p;
  memset(&p, 0, sizeof(p));
  if ((rc = build_intra(p, 0, ws, g, mt0, mt1))) return rc;
  if ((rc = build_cross(p, 2, ws, g, mt0, mt1))) return rc;
  p.nprob = 4;
  p.split = 2;
  return launch_backward(p, st_of(stream), g);
}

int disco_b200_contribution(void* ws, int64_t B, int64_t D, int world, int rank, float t, int flip,
                            float* d_image_full, float* d_text_full, int64_t ld_out, void* stream) {
  Geometry g;
  int rc = make_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  if (ld_out < D) return fail(DISCO_SHAPE_ERROR, "output row stride smaller than D");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const float s = exchange_scale(g, t, double(g.b));
  const int64_t n = 2 * g.B * (g.Dp / 4);
  contribution_kernel<<<elementwise_grid(n, 256), 256, 0, st>>>(
      region<float4>(ws, g, DISCO_R_INTRA), g.ksplit, region<float4>(ws, g, DISCO_R_SEND),
      (world == 1 && g.np > 1) ? region<float4>(ws, g, DISCO_R_XPART) : nullptr, g.np, world, rank, int(g.b),
      int(g.Dp), int(D), s, flip && world > 1, d_image_full, d_text_full, ld_out, region<Status>(ws, g, DISCO_R_STATUS));
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return DISCO_OK;
}

int disco_b200_loss_peer(void* ws, int64_t B, int64_t D, int world, int rank, const void* my_base, int parity,
                         void* stream) {
  Geometry g;
  int rc = make_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  if ((rc = check_peer(g))) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Status* status = region<Status>(ws, g, DISCO_R_STATUS);
  loss_partial_kernel<<<LOSS_BLOCKS, 256, 0, st>>>(peer_ce(my_base, g, parity), world, int(g.b),
                                                   status->loss_partial);
  loss_final_kernel<<<1, LOSS_BLOCKS, 0, st>>>(status->loss_partial, int64_t(2) * world * g.b, status);
  count_launch(2);
  CUDA_TRY(cudaGetLastError());
  return DISCO_OK;
}

int disco_b200_loss(void* ws, int64_t B, int64_t D, int world, int rank, int local_only, void* stream) {
  Geometry g;
  int rc = make_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool local = local_only == 1 || world == 1;
  const bool xall = local_only == 2 && !local;  // dual backward: ce of every rank in DISCO_R_XALL
  Status* status = region<Status>(ws, g, DISCO_R_STATUS);
  const int nw = local ? 1 : world;
  if (xall)
    loss_partial_kernel<<<LOSS_BLOCKS, 256, 0, st>>>(region<float>(ws, g, DISCO_R_XALL), nw, int(g.b),
                                                     status->loss_partial, 4, 2);
  else
    loss_partial_kernel<<<LOSS_BLOCKS, 256, 0, st>>>(region<float>(ws, g, local ? DISCO_R_CE : DISCO_R_CE_ALL), nw,
                                                     int(g.b), status->loss_partial);
  loss_final_kernel<<<1, LOSS_BLOCKS, 0, st>>>(status->loss_partial, int64_t(2) * nw * g.b, status);
  count_launch(2);
  CUDA_TRY(cudaGetLastError());
  return DISCO_OK;
}

int disco_b200_logit_scale_rows(void* ws, int64_t B, int64_t D, int world, int rank, const float* d_image,
                                const float* d_text, int64_t ld_out, void* stream) {
  Geometry g;
  int rc = make_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  if (ld_out < D) return fail(DISCO_SHAPE_ERROR, "output row stride smaller than D");
  const int64_t threads = g.b * 32;
  rowdot_kernel<<<int((threads + 255) / 256), 256, 0, st_of(stream)>>>(
      d_image, d_text, ld_out, region<__nv_bfloat16>(ws, g, DISCO_R_PACK), int(g.b), int(D), int(g.Dp),
      region<float>(ws, g, DISCO_R_RDOT));
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return DISCO_OK;
}

int disco_b200_logit_scale_grad(void* ws, int64_t B, int64_t D, int world, int rank, float t, void* stream) {
  Geometry g;
  int rc = make_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  if (!(t > 0.f) || !std::isfinite(t)) return fail(DISCO_DOMAIN_ERROR, "temperature must be positive, got %g", t);
  cudaStream_t st = st_of(stream);
  Status* status = region<Status>(ws, g, DISCO_R_STATUS);
  rowsum_partial_kernel<<<LOSS_BLOCKS, 256, 0, st>>>(region<float>(ws, g, DISCO_R_RDOT_ALL), g.B,
                                                     status->loss_partial);
  dlogit_final_kernel<<<1, LOSS_BLOCKS, 0, st>>>(status->loss_partial, 0.5 / double(t), status);
  count_launch(2);
  CUDA_TRY(cudaGetLastError());
  return DISCO_OK;
}

int disco_b200_l2norm_rows(const float* raw, int64_t ld_raw, int64_t rows, int64_t D, float* out, int64_t ld_out,
                           float* norms, int* flags, void* stream) {
  if (rows < 0 || D < 1 || ld_raw < D || ld_out < D) return fail(DISCO_SHAPE_ERROR, "bad l2norm geometry");
  if (rows == 0) return DISCO_OK;
  l2norm_rows_kernel<<<int((rows * 32 + 255) / 256), 256, 0, st_of(stream)>>>(raw, ld_raw, int(rows), int(D), out,
                                                                              ld_out, norms, flags);
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return DISCO_OK;
}

int disco_b200_l2norm_rows_backward(const float* raw, int64_t ld_raw, const float* grad, int64_t ld_grad, int64_t rows,
                                    int64_t D, float* out, int64_t ld_out, int* flags, void* stream) {
  if (rows < 0 || D < 1 || ld_raw < D || ld_grad < D || ld_out < D)
    return fail(DISCO_SHAPE_ERROR, "bad l2norm backward geometry");
  if (rows == 0) return DISCO_OK;
  l2norm_rows_backward_kernel<<<int((rows * 32 + 255) / 256), 256, 0, st_of(stream)>>>(
      raw, ld_raw, grad, ld_grad, int(rows), int(D), out, ld_out, flags);
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return DISCO_OK;
}

// ------------------------------------------------------------ dual backward
static int dual_geometry(int64_t B, int64_t D, int world, int rank, Geometry* g) {
  int rc = make_geometry(B, D, world, rank, g);
  if (rc) return rc;
  if (!g->dual)
    return fail(DISCO_LAYOUT_ERROR, "dual backward not available for B=%lld D=%lld N=%d (disco_b200_path_info)",
                (long long)B, (long long)D, world);
  return DISCO_OK;
}

int disco_b200_dual_prep(void* ws, int64_t B, int64_t D, int world, int rank, int flip, void* stream) {
  Geometry g;
  int rc = dual_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  float* qcol = region<float>(ws, g, DISCO_R_QCOL);
  const int warps = 2 * g.groups;
  dual_prep_kernel<<<(warps * 32 + 255) / 256, 256, 0, st_of(stream)>>>(
      region<float>(ws, g, DISCO_R_XALL), int(g.b), g.groups, rank, flip && world > 1, qcol,
      reinterpret_cast<float2*>(qcol + 2 * g.B));
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return DISCO_OK;
}

int disco_b200_backward_dual(void* ws, int64_t B, int64_t D, int world, int rank, int64_t row0, int64_t row1,
                             void* stream) {
  Geometry g;
  int rc = dual_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  if (row0 < 0 || row1 > g.b || row0 >= row1 || row0 % PAIR_M != 0 || (row1 % PAIR_M != 0 && row1 != g.b))
    return fail(DISCO_SHAPE_ERROR, "row block [%lld, %lld) must be 256-aligned inside [0, %lld)", (long long)row0,
                (long long)row1, (long long)g.b);
  GemmParams p;
  memset(&p, 0, sizeof(p));
  if ((rc = build_dual(p, ws, g, int(row0 / PAIR_M), int((row1 + PAIR_M - 1) / PAIR_M)))) return rc;
  return launch_backward(p, st_of(stream), g);
}

int disco_b200_combine_dual(void* ws, int64_t B, int64_t D, int world, int rank, float t, int64_t row0, int64_t row1,
                            float* d_image, float* d_text, int64_t ld_out, void* stream) {
  Geometry g;
  int rc = dual_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  if (ld_out < D) return fail(DISCO_SHAPE_ERROR, "output row stride smaller than D");
  if (row0 < 0 || row1 > g.b || row0 > row1) return fail(DISCO_SHAPE_ERROR, "row range [%lld, %lld) outside [0, %lld)",
                                                         (long long)row0, (long long)row1, (long long)g.b);
  const int64_t n = 2 * (row1 - row0) * (g.Dp / 4);
  if (n == 0) return DISCO_OK;
  combine_dual_kernel<<<elementwise_grid(n, 256), 256, 0, st_of(stream)>>>(
      region<float4>(ws, g, DISCO_R_INTRA), g.ksplit, region<float>(ws, g, DISCO_R_ROWS) + 4 * g.b,
      region<__nv_bfloat16>(ws, g, DISCO_R_PACK), int(g.b), int(g.Dp), int(D), float(0.5 * double(t) / double(g.B)),
      d_image, d_text, ld_out, int(row0), int(row1 - row0), region<Status>(ws, g, DISCO_R_STATUS));
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return DISCO_OK;
}

int disco_b200_dual_fixup(void* ws, int64_t B, int64_t D, int world, int rank, float t, int flip, float* d_image,
                          float* d_text, int64_t ld_out, void* stream) {
  Geometry g;
  int rc = dual_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  if (ld_out < D) return fail(DISCO_SHAPE_ERROR, "output row stride smaller than D");
  dual_fixup_kernel<<<sm_count(), FIX_THREADS, 0, st_of(stream)>>>(
      region<__nv_bfloat16>(ws, g, DISCO_R_FEAT), region<float>(ws, g, DISCO_R_XALL),
      region<float>(ws, g, DISCO_R_ROWS) + 4 * g.b, region<int>(ws, g, DISCO_R_FIX), region<Status>(ws, g, DISCO_R_STATUS),
      int(fix_capacity(g)), int(g.B), int(g.b), int(g.Dp), int(D), rank, t * LOG2E,
      float(0.5 * double(t) / double(g.B)), flip && world > 1, d_image, d_text, ld_out);
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return DISCO_OK;
}
int disco_b200_finish_dual_l2norm(void* ws, int64_t B, int64_t D, int world, int rank, float t, int flip,
                                  const float* raw_I, int64_t ld_raw_I, const float* raw_T, int64_t ld_raw_T,
                                  float* d_image, float* d_text, int64_t ld_out, float* dx_image, float* dx_text,
                                  int64_t ld_dx, int* norm_flags, void* stream) {
  Geometry g;
  int rc = dual_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  if (ld_out < D || ld_dx < D || ld_raw_I < D || ld_raw_T < D) return fail(DISCO_SHAPE_ERROR, "row stride smaller than D");
  cudaStream_t st = st_of(stream);
  TowerRows tw;
  tw.raw[0] = raw_I;
  tw.raw[1] = raw_T;
  tw.ld_raw[0] = ld_raw_I;
  tw.ld_raw[1] = ld_raw_T;
  tw.dx[0] = dx_image;
  tw.dx[1] = dx_text;
  tw.ld_dx = ld_dx;
  const float s = float(0.5 * double(t) / double(g.B));
  combine_dual_l2norm_kernel<<<int((2 * g.b * 32 + 255) / 256), 256, 0, st>>>(
      region<float>(ws, g, DISCO_R_INTRA), g.ksplit, region<float>(ws, g, DISCO_R_ROWS) + 4 * g.b,
      region<__nv_bfloat16>(ws, g, DISCO_R_PACK), int(g.b), int(g.Dp), int(D), s, d_image, d_text, ld_out, tw,
      region<Status>(ws, g, DISCO_R_STATUS), norm_flags);
  count_launch();
  if ((rc = disco_b200_dual_fixup(ws, B, D, world, rank, t, flip, d_image, d_text, ld_out, stream))) return rc;
  fixup_l2norm_kernel<<<sm_count(), 256, 0, st>>>(region<int>(ws, g, DISCO_R_FIX), region<Status>(ws, g, DISCO_R_STATUS),
                                                 int(fix_capacity(g)), int(g.b), int(D), d_image, d_text, ld_out, tw,
                                                 norm_flags);
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return DISCO_OK;
}

// ------------------------------------------------------------ peer transport
int disco_b200_peer_bytes(int64_t B, int64_t D, int world, int rank, int64_t* bytes) {
  Geometry g;
  int rc = make_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  if ((rc = check_peer(g))) return rc;
  *bytes = peer_total_bytes(g);
  return DISCO_OK;
}

int disco_b200_peer_alloc(int64_t bytes, void** ptr, void* ipc_handle) {
  if (bytes <= 0) return fail(DISCO_SHAPE_ERROR, "peer window size must be positive");
  CUDA_TRY(cudaMalloc(ptr, size_t(bytes)));
  CUDA_TRY(cudaMemset(*ptr, 0, size_t(PEER_FLAG_BYTES)));  // arrival flags start at epoch 0
  if (ipc_handle) {
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, *ptr);
    if (e != cudaSuccess) {
      cudaFree(*ptr);
      *ptr = nullptr;
      return fail(DISCO_CUDA_ERROR, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
    }
    memcpy(ipc_handle, &h, sizeof(h));
  }
  CUDA_TRY(cudaDeviceSynchronize());
  return DISCO_OK;
}

int disco_b200_peer_handle_bytes(void) { return int(sizeof(cudaIpcMemHandle_t)); }

int disco_b200_peer_open(const void* ipc_handle, void** ptr) {
  cudaIpcMemHandle_t h;
  memcpy(&h, ipc_handle, sizeof(h));
  CUDA_TRY(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return DISCO_OK;
}

int disco_b200_peer_close(void* ptr) {
  CUDA_TRY(cudaIpcCloseMemHandle(ptr));
  return DISCO_OK;
}

int disco_b200_peer_free(void* ptr) {
  CUDA_TRY(cudaFree(ptr));
  return DISCO_OK;
}

int disco_b200_backward_peer(void* ws, int64_t B, int64_t D, int world, int rank, const uint64_t* peer_bases,
                             int parity, uint32_t epoch, void* stream) {
  Geometry g;
  int rc = make_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  if ((rc = check_peer(g))) return rc;
  if (g.dual) return fail(DISCO_LAYOUT_ERROR, "peer gradient slabs need the exchange backward (DISCO_BACKWARD=exchange)");
  cudaStream_t st = st_of(stream);
  GemmParams p;
  memset(&p, 0, sizeof(p));
  if ((rc = build_intra(p, 0, ws, g))) return rc;  // list A: long units
  if ((rc = build_cross(p, 2, ws, g))) return rc;  // list B: cross units, pushed to the owners
  for (int gi = 0; gi < 2; ++gi)
    if ((rc = set_output_peer(p.prob[2 + gi], peer_bases, parity, g, gi))) return rc;
  p.nprob = 4;
  p.split = 2;
  if ((rc = launch_backward(p, st, g))) return rc;
  // the rank's per-row ce rides with the slabs: the owners' combine wait covers it too
  PeerDst pd;
  memset(&pd, 0, sizeof(pd));
  for (int r = 0; r < g.N; ++r)
    pd.ce[r] = peer_ce(reinterpret_cast<const void*>(peer_bases[r]), g, parity) + int64_t(rank) * 2 * g.b;
  const int n4 = int(2 * g.b / 4);
  peer_ce_push_kernel<<<std::max(1, std::min(n4 / 256 + 1, 64)), 256, 0, st>>>(region<float4>(ws, g, DISCO_R_CE), n4,
                                                                               pd, g.N);
  count_launch();
  PeerPtrs pp;
  memset(&pp, 0, sizeof(pp));
  for (int r = 0; r < g.N; ++r)
    pp.flag[r] = reinterpret_cast<uint32_t*>(peer_bases[r]) + rank;
  peer_signal_kernel<<<1, 32, 0, st>>>(pp, g.N, epoch);
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return DISCO_OK;
}

int disco_b200_peer_publish(void* ws, int64_t B, int64_t D, int world, int rank, const uint64_t* peer_bases,
                            int parity, uint32_t epoch, void* stream) {
  Geometry g;
  int rc = make_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  if ((rc = check_peer(g))) return rc;
  cudaStream_t st = st_of(stream);
  CUDA_TRY(cudaMemcpyAsync(peer_pack(reinterpret_cast<const void*>(peer_bases[rank]), g, parity),
                           region<uint8_t>(ws, g, DISCO_R_PACK), size_t(2 * g.b * g.Dp * 2), cudaMemcpyDeviceToDevice,
                           st));
  PeerPtrs pp;
  memset(&pp, 0, sizeof(pp));
  for (int r = 0; r < g.N; ++r)
    pp.flag[r] = reinterpret_cast<uint32_t*>(peer_bases[r]) + PEER_PACK_FLAG0 + rank;
  peer_signal_kernel<<<1, 32, 0, st>>>(pp, g.N, epoch);
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return DISCO_OK;
}

int disco_b200_peer_gather(void* ws, int64_t B, int64_t D, int world, int rank, const uint64_t* peer_bases,
                           int parity, uint32_t epoch, double timeout_s, void* stream) {
  Geometry g;
  int rc = make_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  if ((rc = check_peer(g))) return rc;
  cudaStream_t st = st_of(stream);
  peer_wait_kernel<<<1, 32, 0, st>>>(reinterpret_cast<const uint32_t*>(peer_bases[rank]) + PEER_PACK_FLAG0, g.N,
                                     epoch, region<Status>(ws, g, DISCO_R_STATUS), (unsigned long long)(timeout_s * 1e9));
  count_launch();
  PeerSrc src;
  memset(&src, 0, sizeof(src));
  for (int r = 0; r < g.N; ++r)
    src.pack[r] = reinterpret_cast<const uint4*>(peer_pack(reinterpret_cast<const void*>(peer_bases[r]), g, parity));
  const int64_t nvec = int64_t(g.N) * 2 * g.b * (g.Dp / 8);
  peer_gather_unpack_kernel<<<elementwise_grid(nvec, 256), 256, 0, st>>>(
      src, g.N, int(g.b), int(g.Dp), region<uint4>(ws, g, DISCO_R_FEAT), region<uint4>(ws, g, DISCO_R_FEAT16));
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return DISCO_OK;
}

int disco_b200_peer_gather_streamed(void* ws, int64_t B, int64_t D, int world, int rank, const uint64_t* peer_bases,
                                    int parity, uint32_t epoch, void* copy_stream) {
  Geometry g;
  int rc = make_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  if ((rc = check_peer(g))) return rc;
  if (!(g.estore && (g.nchunk * g.ssub) % g.N == 0))
    return fail(DISCO_LAYOUT_ERROR, "streamed peer gather needs canonical chunks");
  auto wfn = write_value_fn();
  auto wait = wait_value_fn();
  if (!wfn || !wait) return fail(DISCO_CUDA_ERROR, "stream memory operations unavailable");
  cudaStream_t st = static_cast<cudaStream_t>(copy_stream);
  const int64_t rank_bytes = g.b * g.Dp * 2;  // one direction of one rank's rows
  uint8_t* feat = region<uint8_t>(ws, g, DISCO_R_FEAT);
  Status* stt = region<Status>(ws, g, DISCO_R_STATUS);
  const uint32_t* my_flags = reinterpret_cast<const uint32_t*>(peer_bases[rank]) + PEER_PACK_FLAG0;
  for (int k = 0; k < g.N; ++k) {
    const int src = (rank + k) % g.N;
    const uint8_t* from = src == rank ? region<uint8_t>(ws, g, DISCO_R_PACK)
                                      : peer_pack(reinterpret_cast<const void*>(peer_bases[src]), g, parity);
    if (src != rank) {  // wait (copy engine, no SM) until that rank published this step's rows
      CUresult r = wait(static_cast<CUstream>(copy_stream), reinterpret_cast<CUdeviceptr>(my_flags + src), epoch,
                        0 /* CU_STREAM_WAIT_VALUE_GEQ */);
      if (r != CUDA_SUCCESS) return fail(DISCO_CUDA_ERROR, "cuStreamWaitValue32 failed (%d)", int(r));
    }
    for (int d = 0; d < 2; ++d)
      CUDA_TRY(cudaMemcpyAsync(feat + (int64_t(d) * g.B + int64_t(src) * g.b) * g.Dp * 2, from + d * rank_bytes,
                               size_t(rank_bytes), cudaMemcpyDeviceToDevice, st));
    CUresult r = wfn(static_cast<CUstream>(copy_stream), reinterpret_cast<CUdeviceptr>(&stt->wave_flags[k]), epoch, 0);
    if (r != CUDA_SUCCESS) return fail(DISCO_CUDA_ERROR, "cuStreamWriteValue32 failed (%d)", int(r));
  }
  return DISCO_OK;
}

int disco_b200_forward_peer_streamed(void* ws, int64_t B, int64_t D, int world, int rank, float t, uint32_t epoch,
                                     double timeout_s, void* stream) {
  Geometry g;
  int rc = make_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  if ((rc = check_peer(g))) return rc;
  if (!(t > 0.f) || !std::isfinite(t)) return fail(DISCO_DOMAIN_ERROR, "temperature must be positive, got %g", t);
  if (!(g.estore && (g.nchunk * g.ssub) % g.N == 0))
    return fail(DISCO_LAYOUT_ERROR, "streamed peer forward needs canonical chunks");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if ((rc = launch_logits(KIND_FWDE, ws, g, t, st, -3, epoch, timeout_s))) return rc;
  const int64_t n = 2 * g.B * g.Dp / 8;
  feat16_kernel<<<elementwise_grid(n, 256), 256, 0, st>>>(region<uint4>(ws, g, DISCO_R_FEAT),
                                                         region<uint4>(ws, g, DISCO_R_FEAT16), n,
                                                         region<Status>(ws, g, DISCO_R_STATUS));
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return forward_finish(ws, g, st);
}

int disco_b200_combine_peer(void* ws, int64_t B, int64_t D, int world, int rank, float t, int flip,
                            const void* my_base, int parity, uint32_t epoch, double timeout_s, float* d_image,
                            float* d_text, int64_t ld_out, void* stream) {
  Geometry g;
  int rc = make_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  if ((rc = check_peer(g))) return rc;
  if (g.dual) return fail(DISCO_LAYOUT_ERROR, "peer gradient slabs need the exchange backward (DISCO_BACKWARD=exchange)");
  if (ld_out < D) return fail(DISCO_SHAPE_ERROR, "output row stride smaller than D");
  cudaStream_t st = st_of(stream);
  Status* status = region<Status>(ws, g, DISCO_R_STATUS);
  peer_wait_kernel<<<1, 32, 0, st>>>(static_cast<const uint32_t*>(my_base), g.N, epoch, status,
                                     (unsigned long long)(timeout_s * 1e9));
  count_launch();
  CUDA_TRY(cudaGetLastError());
  const float s = exchange_scale(g, t, double(g.B));
  const int64_t n = 2 * g.b * (g.Dp / 4);
  const int L = int(peer_leaves(g));
  combine_kernel<<<elementwise_grid(n, 256), 256, 0, st>>>(
      region<float4>(ws, g, DISCO_R_INTRA), g.ksplit, nullptr,
      reinterpret_cast<const float4*>(peer_window(my_base, g, parity)), L, g.N, g.rank, int(g.b), int(g.Dp),
      int(g.D), s, flip, d_image, d_text, ld_out, 0, int(g.b), status, g.rank * g.np, (g.rank + 1) * g.np);
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return DISCO_OK;
}

// Clock probe readout (synchronous; profiling aid): the SM clock, in MHz, at which CTA 0 of the
// last logits kernel and of the last backward GEMM ran (clock64 cycles / globaltimer ns), 0 if
// the kernel has not run.
int disco_b200_clock_probe(void* ws, int64_t B, int64_t D, int world, int rank, double* mhz) {
  Geometry g;
  int rc = make_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  unsigned long long pr[10];
  CUDA_TRY(cudaMemcpy(pr, probe_slot(ws, g, 0), sizeof(pr), cudaMemcpyDeviceToHost));
  for (int k = 0; k < 2; ++k) {
    const unsigned long long* q = pr + 4 * k;
    mhz[k] = (q[3] > q[1] && q[2] > q[0]) ? double(q[2] - q[0]) / double(q[3] - q[1]) * 1e3 : 0.0;
  }
  // mhz[2]: mean accumulator drain (cycles per backward unit) since the last readout
  mhz[2] = pr[9] ? double(pr[8]) / double(pr[9]) : 0.0;
  CUDA_TRY(cudaMemset(probe_slot(ws, g, 8), 0, 2 * sizeof(unsigned long long)));
  return DISCO_OK;
}

}  // extern "C"
