// The grouped backward GEMM (E-operand transforms, wide / narrow units, peer pushes).
// Part of the single translation unit disco_b200.cu (included there, in this order).
#pragma once

namespace disco {

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

}  // namespace disco
