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
#include "common.cuh"
#include "logits.cuh"
#include "gemm.cuh"
#include "tails.cuh"
#include "host.cuh"

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
int disco_b200_forward_streamed_split(void* ws, int64_t B, int64_t D, int world, int rank, float t, uint32_t epoch,
                                      double timeout_s, int k0, void* stream) {
  Geometry g;
  int rc = make_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  if (!(t > 0.f) || !std::isfinite(t)) return fail(DISCO_DOMAIN_ERROR, "temperature must be positive, got %g", t);
  if (!(world == 1 && g.estore && (g.chunk_cols / g.ssub) % PAIR_M == 0 && g.D == g.Dp))
    return fail(DISCO_LAYOUT_ERROR, "streamed forward needs a single rank, B %% 2048 == 0 and D %% 64 == 0");
  const int nw = g.nchunk * g.ssub;
  if (k0 < 0 || k0 > nw) return fail(DISCO_LAYOUT_ERROR, "k0 %d outside [0, %d]", k0, nw);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  UnitRange ur;
  ur.k0 = k0;
  if ((rc = launch_logits(KIND_FWDE, ws, g, t, st, -4, epoch, timeout_s, ur))) return rc;
  const int64_t n = 2 * g.B * g.Dp / 8;
  feat16_kernel<<<elementwise_grid(n, 256), 256, 0, st>>>(region<uint4>(ws, g, DISCO_R_FEAT),
                                                         region<uint4>(ws, g, DISCO_R_FEAT16), n,
                                                         region<Status>(ws, g, DISCO_R_STATUS));
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return forward_finish(ws, g, st, 1, 1);  // direction 1 is complete; direction 0 finishes per row block
}
int disco_b200_forward_rect(void* ws, int64_t B, int64_t D, int world, int rank, float t, int dir, int64_t row0,
                            int64_t row1, int ch0, int ch1, void* stream) {
  Geometry g;
  int rc = make_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  if (!(t > 0.f) || !std::isfinite(t)) return fail(DISCO_DOMAIN_ERROR, "temperature must be positive, got %g", t);
  if (!g.estore) return fail(DISCO_LAYOUT_ERROR, "unit rectangles need the E-storing forward (canonical shapes)");
  const int nch = g.nchunk * g.ssub;
  if (dir < 0 || dir > 1 || row0 < 0 || row1 > g.b || row0 >= row1 || row0 % PAIR_M || (row1 % PAIR_M && row1 != g.b) ||
      ch0 < 0 || ch1 > nch || ch0 >= ch1)
    return fail(DISCO_SHAPE_ERROR, "bad unit rectangle dir %d rows [%lld, %lld) chunks [%d, %d)", dir,
                (long long)row0, (long long)row1, ch0, ch1);
  UnitRange ur;
  ur.dir = dir;
  ur.rt0 = int(row0 / PAIR_M);
  ur.nrt = int((row1 + PAIR_M - 1) / PAIR_M) - ur.rt0;
  ur.ch0 = ch0;
  ur.nch = ch1 - ch0;
  return launch_logits(KIND_FWDE, ws, g, t, static_cast<cudaStream_t>(stream), -5, 0, 0.0, ur);
}
int disco_b200_stats_rows(void* ws, int64_t B, int64_t D, int world, int rank, int dir, int64_t row0, int64_t row1,
                          void* stream) {
  Geometry g;
  int rc = make_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  if (dir < 0 || dir > 1 || row0 < 0 || row1 > g.b || row0 > row1)
    return fail(DISCO_SHAPE_ERROR, "bad statistics rows dir %d [%lld, %lld)", dir, (long long)row0, (long long)row1);
  return forward_finish(ws, g, static_cast<cudaStream_t>(stream), dir, 1, row0, row1);
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
int disco_b200_dual_prep_dir(void* ws, int64_t B, int64_t D, int world, int rank, int dir, int flip, void* stream) {
  Geometry g;
  int rc = dual_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  if (dir < 0 || dir > 1) return fail(DISCO_SHAPE_ERROR, "direction %d outside {0, 1}", dir);
  float* qcol = region<float>(ws, g, DISCO_R_QCOL);
  const int warps = g.groups;
  dual_prep_kernel<<<(warps * 32 + 255) / 256, 256, 0, st_of(stream)>>>(
      region<float>(ws, g, DISCO_R_XALL), int(g.b), g.groups, rank, flip && world > 1, qcol,
      reinterpret_cast<float2*>(qcol + 2 * g.B), dir, 1);
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
int disco_b200_backward_dual_dir(void* ws, int64_t B, int64_t D, int world, int rank, int dir, int64_t row0,
                                 int64_t row1, void* stream) {
  Geometry g;
  int rc = dual_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  if (dir < 0 || dir > 1) return fail(DISCO_SHAPE_ERROR, "direction %d outside {0, 1}", dir);
  if (row0 < 0 || row1 > g.b || row0 >= row1 || row0 % PAIR_M != 0 || (row1 % PAIR_M != 0 && row1 != g.b))
    return fail(DISCO_SHAPE_ERROR, "row block [%lld, %lld) must be 256-aligned inside [0, %lld)", (long long)row0,
                (long long)row1, (long long)g.b);
  GemmParams p;
  memset(&p, 0, sizeof(p));
  if ((rc = build_dual(p, ws, g, int(row0 / PAIR_M), int((row1 + PAIR_M - 1) / PAIR_M)))) return rc;
  if (dir == 1) p.prob[0] = p.prob[1];  // one direction: the same problem (same tiles, K order, outputs)
  p.nprob = 1;
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
int disco_b200_combine_dual_dir(void* ws, int64_t B, int64_t D, int world, int rank, int dir, float t, int64_t row0,
                                int64_t row1, float* d_image, float* d_text, int64_t ld_out, void* stream) {
  Geometry g;
  int rc = dual_geometry(B, D, world, rank, &g);
  if (rc) return rc;
  if (dir < 0 || dir > 1) return fail(DISCO_SHAPE_ERROR, "direction %d outside {0, 1}", dir);
  if (ld_out < D) return fail(DISCO_SHAPE_ERROR, "output row stride smaller than D");
  if (row0 < 0 || row1 > g.b || row0 > row1) return fail(DISCO_SHAPE_ERROR, "row range [%lld, %lld) outside [0, %lld)",
                                                         (long long)row0, (long long)row1, (long long)g.b);
  const int64_t n = (row1 - row0) * (g.Dp / 4);
  if (n == 0) return DISCO_OK;
  combine_dual_kernel<<<elementwise_grid(n, 256), 256, 0, st_of(stream)>>>(
      region<float4>(ws, g, DISCO_R_INTRA), g.ksplit, region<float>(ws, g, DISCO_R_ROWS) + 4 * g.b,
      region<__nv_bfloat16>(ws, g, DISCO_R_PACK), int(g.b), int(g.Dp), int(D), float(0.5 * double(t) / double(g.B)),
      d_image, d_text, ld_out, int(row0), int(row1 - row0), region<Status>(ws, g, DISCO_R_STATUS), dir, 1);
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
