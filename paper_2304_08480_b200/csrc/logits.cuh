// The forward logits kernel (tcgen05 CTA pairs; FWD / GRAD / FWDE epilogues).
// Part of the single translation unit disco_b200.cu (included there, in this order).
#pragma once

namespace disco {

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
  // wave k = the columns of source rank (rank + k) % N, all local row tiles), -4 = the H2D
  // wavefront of direction 1 with direction 0 only for waves k < k0 (each wave's direction-1 units
  // first), so direction 1 completes as early as the copies allow; -5 (not streamed) = one
  // rectangle of units: direction rect_dir, row tiles [rect_rt0, +rect_nrt), chunks [rect_ch0,
  // +rect_nch) -- the rest of direction 0 after -4, row block by row block.  Every mode walks the
  // same units (identical tiles, K order and outputs), so results are bit-identical.
  const bool streamed = wave == -2 || wave == -3 || wave == -4;
  const bool colwaves = wave == -3;
  const bool split = wave == -4;
  const bool rect = wave == -5;
  const int spr = colwaves ? p.nchunk / p.nwaves : 1;          // sub-chunks per source rank
  const int per_cwave = 2 * p.row_tiles * spr;                  // units per column wave
  const int per_dir = wave >= 0 ? p.rt_per_chunk * (2 * wave + 1)
                                : p.row_tiles * p.nchunk * (CHUNK_UNITS ? 1 : p.tiles_per_chunk);
  const int R = p.rt_per_chunk;
  // -4: waves before k hold R k^2 direction-1 units and R min(k, k0)^2 direction-0 units
  auto split_base = [&](int k) { return R * k * k + R * min(k, p.k0) * min(k, p.k0); };
  const int num_units = colwaves ? per_cwave * p.nwaves
                      : split    ? split_base(p.nwaves)
                      : rect     ? p.rect_nrt * p.rect_nch
                      : streamed ? NDIR * R * p.nwaves * p.nwaves : NDIR * per_dir;
  // -2: unit u belongs to wave k with 2 R k^2 <= u < 2 R (k+1)^2 (wave k holds 2 R (2k+1));
  auto wave_of = [&](int u) {
    if (colwaves) return u / per_cwave;
    if (split) {
      int k = 0;
      while (k + 1 < p.nwaves && split_base(k + 1) <= u) ++k;
      return k;
    }
    int k = int(sqrtf(float(u) / float(NDIR * R)));
    while (k > 0 && NDIR * R * k * k > u) --k;
    while (NDIR * R * (k + 1) * (k + 1) <= u) ++k;
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
    if (rect) {
      dir = p.rect_dir;
      rt = p.rect_rt0 + u / p.rect_nch;
      ch = p.rect_ch0 + u % p.rect_nch;
      t0 = 0;
      return;
    }
    int wv = wave, pd = per_dir;
    int rem;
    if (split) {  // wave wv: R (2 wv + 1) direction-1 units, then as many direction-0 units if wv < k0
      wv = wave_of(u);
      u -= split_base(wv);
      pd = R * (2 * wv + 1);
      dir = u < pd ? 1 : 0;
      rem = u < pd ? u : u - pd;
    } else {
      if (streamed) {
        wv = wave_of(u);
        u -= NDIR * R * wv * wv;
        pd = R * (2 * wv + 1);
      }
      dir = u / pd;
      rem = u - dir * pd;
    }
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

}  // namespace disco
