/*
 * disco_b200.h -- C ABI of the B200-native DisCo contrastive loss.
 *
 * This is the drop-in boundary for the reference package's hot path
 * (arxiv 2304.08480 reference, /root/reference/pkg/src/disco):
 *
 *   disco_step(endpoint, local_I, local_T, t, ...)            shard.py:169-208
 *   local_loss_and_grads(layout, I_gathered, T_gathered, t)   shard.py:98-166
 *
 * The reference is pure Python/numpy, so its "FFI" is the Python call
 * boundary; the entry points below are what a ctypes binding of that call
 * needs (INTEGRATION.md shows the stub).  The collectives that sit between
 * the phases (all_gather shard.py:190-191, all_reduce(AVG) shard.py:199-204,
 * all_reduce_scalar shard.py:205) are issued by the host through
 * torch.distributed (NCCL); this library never links NCCL.
 *
 * Conventions
 *  - Plain device pointers, int64 sizes, a cudaStream_t passed as void*.
 *  - Every call is stream-ordered and asynchronous; nothing allocates.
 *    All scratch lives in one caller-allocated workspace whose layout is
 *    described by disco_b200_ws_region().
 *  - Return value: DISCO_OK or one of the status codes below; a message is
 *    available from disco_b200_last_error() (thread-local).  The codes map
 *    onto the reference exception taxonomy (errors.py:4-20).
 *  - Problem geometry, per rank: global batch B, local batch b = B / N,
 *    feature dim D (padded internally to Dp = roundup(D, 64)), world size N,
 *    rank in [0, N).
 */
#ifndef DISCO_B200_H_
#define DISCO_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DISCO_B200_ABI_VERSION 3

enum disco_status {
  DISCO_OK = 0,
  DISCO_SHAPE_ERROR = 1,   /* errors.ShapeError   (errors.py:4)  */
  DISCO_LAYOUT_ERROR = 2,  /* errors.LayoutError  (errors.py:16) */
  DISCO_DOMAIN_ERROR = 3,  /* errors.DomainError  (errors.py:12) */
  DISCO_NONFINITE = 4,     /* ValueError("... non-finite ...") (matrix.py:43-45) */
  DISCO_CUDA_ERROR = 5     /* launch / driver failure */
};

/* Input element types accepted by disco_b200_pack. */
enum disco_dtype { DISCO_F32 = 0, DISCO_BF16 = 1, DISCO_F64 = 2, DISCO_F16 = 3 };

/* Workspace regions (see disco_b200_ws_region). */
enum disco_region {
  DISCO_R_PACK = 0,    /* bf16 [2][b][Dp]         local packed I_n, T_n (all_gather input)   */
  DISCO_R_GATHER = 1,  /* bf16 [N][2][b][Dp]      all_gather output                          */
  DISCO_R_FEAT = 2,    /* bf16 [2][B][Dp]         gathered I_g, T_g (forward GEMM operands)  */
  DISCO_R_FEAT16 = 3,  /* f16  [2][B][Dp]         gathered I_g, T_g (backward GEMM operands) */
  DISCO_R_STATS = 4,   /* f32x2 [2][nchunk*ssub][2][b] (max, sum-exp) per column sub-chunk and half */
  DISCO_R_ROWS = 5,    /* f32  [4][2][b]          target logit, spare, label gradient, spare */
  DISCO_R_CE = 6,      /* f32  [2][b]             per-row cross-entropy (loss all_gather in);
                          the second half of DISCO_R_XCHG                                     */
  DISCO_R_CE_ALL = 7,  /* f32  [N][2][b]          loss all_gather output                     */
  DISCO_R_G = 8,       /* f16  [2][b][ldG]        softmax-minus-one-hot blocks (unscaled)    */
  DISCO_R_XPART = 9,   /* f32  [2][B][cpr][Dp]    cross partials per canonical row chunk     */
  DISCO_R_SEND = 10,   /* f32  [N][2][b][Dp]      cross slabs by destination (all_to_all in) */
  DISCO_R_RECV = 11,   /* f32  [N][2][b][Dp]      cross slabs by source (all_to_all out)     */
  DISCO_R_INTRA = 12,  /* f32  [2][ksplit][b][Dp] intra-rank gradient terms (K-split halves) */
  DISCO_R_STATUS = 13, /* f64 loss, i32 flags, f64 dL/dt   host-visible step status           */
  DISCO_R_SCALE = 14,  /* f32  [2][B/64][b]       group offsets m_g, then
                          f16  [2][B/64][b]       E -> G factors exp2(m_g - lse2) per row and
                          64-column group (canonical shapes; empty otherwise)                 */
  DISCO_R_RDOT = 15,    /* f32  [b]               per-row <d_image, I_n> + <d_text, T_n>       */
  DISCO_R_RDOT_ALL = 16, /* f32  [N][b]           all_gather of DISCO_R_RDOT (alias at N = 1)  */
  DISCO_R_XCHG = 17,   /* f32  [4][b]             lse2 (i2t, t2i) then ce (i2t, t2i) of this rank's
                          rows: the dual backward's all_gather input                          */
  DISCO_R_XALL = 18,   /* f32  [N][4][b]          all_gather of DISCO_R_XCHG (alias at N = 1)  */
  DISCO_R_QCOL = 19,   /* f32  [2][B] column factors q_c, then f32x2 [2][B/64] (Q_g, min lse2) */
  DISCO_R_FIX = 20,    /* i32  [2][ksplit][b]     rows queued for disco_b200_dual_fixup        */
  DISCO_R_COUNT = 21
};

int disco_b200_abi_version(void);

/* Profiling experiments only (never needed for correct results): replaces the
 * DISCO_DEBUG_FLAGS bits read at load time, returns the previous value. */
int disco_b200_set_experiment_flags(int flags);
const char* disco_b200_last_error(void);

/* Number of CUDA kernels this library has launched in this process
 * (monotonic; used by bench.py to report gpu_launches). */
int64_t disco_b200_launch_count(void);

/* Validates the geometry exactly as ShardLayout (shard.py:38-49) does and
 * reports the workspace size in bytes. */
int disco_b200_workspace_bytes(int64_t B, int64_t D, int world, int rank, int64_t* bytes);

/* Byte offset and size of one region inside the workspace. */
int disco_b200_ws_region(int64_t B, int64_t D, int world, int rank, int region, int64_t* offset,
                         int64_t* bytes);

/* Number of canonical row/column chunks (8 when B % 1024 == 0 and N | 8,
 * else N) and chunks per rank.  Fixes every reduction order over B, which
 * makes results bitwise identical across world sizes that divide 8. */
int disco_b200_chunking(int64_t B, int world, int* nchunk, int* chunks_per_rank);

/* Step 0: round the rank's local features (b x D, row stride ld_*) to bf16
 * into DISCO_R_PACK, zero-padding D..Dp; clear_status != 0 first resets
 * DISCO_R_STATUS (the non-finite flags accumulate until the next reset).
 * Replaces the implicit dtype handling of matmul (matrix.py:57-78). */
int disco_b200_pack(void* ws, int64_t B, int64_t D, int world, int rank, const void* local_I,
                    const void* local_T, int64_t ld_I, int64_t ld_T, int dtype, int clear_status,
                    void* stream);

/* Rows [row0, row1) of disco_b200_pack (same layout, same non-finite flag); the
 * host-buffer single-rank path packs each canonical chunk as its H2D copy lands. */
int disco_b200_pack_rows(void* ws, int64_t B, int64_t D, int world, int rank, const void* local_I,
                         const void* local_T, int64_t ld_I, int64_t ld_T, int dtype, int clear_status, int64_t row0,
                         int64_t row1, void* stream);

/* Forward: unpack the gathered features, fused logits GEMM + online
 * log-sum-exp + target extraction (shard.py:134-141, matrix.py:103-118),
 * fixed-order chunk combine -> per-row lse / ce / label gradient.
 * Canonical shapes (B % 1024 == 0, N | 8): the same epilogue also stores
 * E = exp2(t*log2(e)*s - m_g) (f16, DISCO_R_G) with m_g the row max over its
 * 64-column group, and the combine turns m_g into exp2(m_g - lse2)
 * (DISCO_R_SCALE), so the backward needs no logit recompute. */
int disco_b200_forward(void* ws, int64_t B, int64_t D, int world, int rank, float t, void* stream);

/* Wavefront forward (single rank, canonical shapes with B % 2048 == 0; *waves = 0 otherwise):
 * disco_b200_forward == forward_wave(0) ... forward_wave(waves - 1) + forward_finish, bit for bit.
 * With W = *waves (16 when B % 4096 == 0, else 8) and rows split in W equal chunks, wave k
 * computes the logit units (row chunk, column chunk) with max(row chunk, column chunk) == k, i.e.
 * exactly those that became computable when rows [k*B/W, (k+1)*B/W) of I and T landed, so the
 * host->device copy of host features overlaps the logits GEMMs.  Waves may run on different
 * streams (they write disjoint outputs); forward_finish must follow all of them. */
int disco_b200_forward_waves(int64_t B, int64_t D, int world, int rank, int* waves);

/* Which implementation this geometry takes (bit mask; DISCO_BACKWARD is read now):
 * bit0 E stored by the forward (recompute-free backward), bit1 wide GEMM units (Dp % 512 == 0),
 * bit2 dual backward for disco_step (every N; DISCO_BACKWARD=exchange turns it off): one GEMM per
 * gradient over the rank's own E block on H = G_d + G_d'^T, 4*b*B*D backward flops instead of
 * 8*b*B*D, no gradient reduce-scatter (disco_b200_dual_prep / _backward_dual / _combine_dual /
 * _dual_fixup below). */
#define DISCO_PATH_ESTORE 1
#define DISCO_PATH_WIDE 2
#define DISCO_PATH_DUAL 4
int disco_b200_path_info(int64_t B, int64_t D, int world, int rank, int* bits);
int disco_b200_forward_wave(void* ws, int64_t B, int64_t D, int world, int rank, float t, int wave, void* stream);
int disco_b200_forward_finish(void* ws, int64_t B, int64_t D, int world, int rank, void* stream);
/* Split schedule of the host-buffer step (single rank, pinned bf16, D % 64 == 0; what disco_step
 * runs): the backward of one direction needs the other direction's statistics of EVERY row, so
 * direction 1 is finished first and direction 0 row block by row block, each block's d_image
 * gradients leaving for the host while the next block computes.
 *   forward_streamed_split  like disco_b200_forward_streamed, but the persistent launch walks each
 *                           wave's direction-1 units and, for waves < k0 only, its direction-0
 *                           units; then f16 operands and the direction-1 statistics
 *   forward_rect            the units (dir, 256-row tiles of [row0, row1), stats chunks [ch0, ch1))
 *   stats_rows              LSE / ce / label statistics of rows [row0, row1) of direction dir
 *                           (all of the row's chunks must have run)
 * Every unit is the one the one-launch forward runs (same tiles, K order, outputs): bit-identical.
 * The chunk index counts the forward's statistics sub-chunks (disco_b200_forward_waves of them). */
int disco_b200_forward_streamed_split(void* ws, int64_t B, int64_t D, int world, int rank, float t, uint32_t epoch,
                                      double timeout_s, int k0, void* stream);
int disco_b200_forward_rect(void* ws, int64_t B, int64_t D, int world, int rank, float t, int dir, int64_t row0,
                            int64_t row1, int ch0, int ch1, void* stream);
int disco_b200_stats_rows(void* ws, int64_t B, int64_t D, int world, int rank, int dir, int64_t row0, int64_t row1,
                          void* stream);

/* Streamed forward (host bf16 features, single rank, wavefront shape, D % 64 == 0): the caller
 * copies chunk k's rows of I and T straight into DISCO_R_FEAT on a copy stream and then calls
 * disco_b200_signal_wave(k, epoch) on that stream (cuStreamWriteValue32: no SM, ordered after
 * the copies).  disco_b200_forward_streamed launches ONE persistent logits kernel over all
 * waves in order whose producers wait for each wave's flag (bounded by timeout_s: status flag
 * 16 instead of a hang), then derives the f16 operands and the non-finite flag, then the stats.
 * Bit-identical to pack + disco_b200_forward; no per-wave launch tails.  Use a fresh epoch per
 * step; the flags live in DISCO_R_STATUS, which the caller zeroes once when allocating. */
int disco_b200_forward_streamed(void* ws, int64_t B, int64_t D, int world, int rank, float t, uint32_t epoch,
                                double timeout_s, void* stream);
int disco_b200_signal_wave(void* ws, int64_t B, int64_t D, int world, int rank, int wave, uint32_t epoch,
                           void* stream);
/* All of a step's chunk copies (pinned host bf16 [b][D] I and T -> DISCO_R_FEAT) and wave signals
 * enqueued on copy_stream in one call.  Enqueue them BEFORE launching disco_b200_forward_streamed:
 * streams may share a hardware queue, and a copy queued behind the spinning kernel could only run
 * after it (the producers' bounded wait then expires); copies first can at worst serialise. */
int disco_b200_h2d_streamed(void* ws, int64_t B, int64_t D, int world, int rank, const void* host_I,
                            const void* host_T, uint32_t epoch, void* copy_stream);

/* Backward part 1: recompute the logit tiles (bit-identical to the forward)
 * -> G = softmax - onehot, unscaled, f16 (shard.py:143-146, matrix.py:131-144).
 * Canonical shapes: no-op (G = E * scale, label column P_label - 1, is formed
 * inside the two backward GEMMs' shared-memory stages). */
int disco_b200_backward_grad(void* ws, int64_t B, int64_t D, int world, int rank, float t, void* stream);

/* Backward part 2: cross-rank gradient GEMMs G^T . local features
 * (shard.py:149, 151), canonical chunks pair-summed in the epilogue, reduced
 * over this rank's chunks into DISCO_R_SEND (destination-major slabs). */
int disco_b200_backward_cross(void* ws, int64_t B, int64_t D, int world, int rank, void* stream);

/* Backward part 3: intra-rank GEMMs G . gathered features (shard.py:150, 152)
 * into DISCO_R_INTRA.  Independent of the slab exchange, so it overlaps it. */
int disco_b200_backward_intra(void* ws, int64_t B, int64_t D, int world, int rank, void* stream);

/* Backward parts 2 + 3 in one persistent launch (single rank, where no slab
 * exchange has to overlap the intra GEMM): the intra and cross units are
 * interleaved in proportion to their counts.  Same outputs as
 * disco_b200_backward_cross followed by disco_b200_backward_intra. */
int disco_b200_backward_fused(void* ws, int64_t B, int64_t D, int world, int rank, void* stream);

/* Owner combine after the slab exchange (replaces all_reduce(AVG) +
 * row slice, shard.py:199-208): d = t*0.5/B * (intra + tree(recv slabs)),
 * fp32 b x D outputs with row stride ld_out.  flip != 0 negates the slabs
 * received from other ranks (the flip_cross_rank_sign hook, shard.py:158-162). */
int disco_b200_combine(void* ws, int64_t B, int64_t D, int world, int rank, float t, int flip,
                       float* d_image, float* d_text, int64_t ld_out, void* stream);

/* Row-block pipelining (single rank): backward GEMMs (intra + cross) restricted
 * to output rows [row0, row1) (256-aligned, or row1 == b), and the owner combine
 * of those rows.  Running block k's combine and device->host copy while block
 * k+1's GEMMs run hides the gradient read-back; the union over blocks equals
 * disco_b200_backward_fused + disco_b200_combine bit for bit. */
int disco_b200_backward_rows(void* ws, int64_t B, int64_t D, int world, int rank, int64_t row0, int64_t row1,
                             void* stream);
int disco_b200_combine_rows(void* ws, int64_t B, int64_t D, int world, int rank, float t, int flip, int64_t row0,
                            int64_t row1, float* d_image, float* d_text, int64_t ld_out, void* stream);

/* Peer transport: the cross-rank gradient exchange done by the backward GEMM
 * itself over NVLink peer memory instead of an NCCL all_to_all + sender presum.
 *
 * Every rank owns one peer window (disco_b200_peer_alloc: cudaMalloc'd, IPC-exportable):
 * u32 arrival flags (slab slots [0, N), pack-ready slots [64, 64 + N)), then two parity windows
 * of [2][L][b][Dp] f32 slabs, L = N * (chunk partials per rank), then two parity areas of
 * [2][b][Dp] bf16 published rows, then two parity areas of [N][2][b] f32 per-row ce.  disco_b200_backward_peer runs the intra and cross GEMMs as one persistent
 * launch; each cross tile's epilogue TMA-stores its fp32 chunk partial straight into the owning
 * rank's window (leaf rank*np + k), so the transfer overlaps the GEMM tile by tile; a one-warp
 * kernel then publishes `epoch` into every destination's flag slot [rank] (release, system
 * scope).  disco_b200_combine_peer waits (acquire) until all N slots of this rank's window hold
 * `epoch` (bounded by timeout_s: on expiry it sets status flag 8 instead of hanging), then runs
 * the owner combine over the L leaves with the same fixed tree as disco_b200_combine, so the
 * result is bit-identical to the all_to_all path and to N = 1.  Step s uses parity s & 1.
 * Requires 2 <= N <= 8 and b % 128 == 0.  peer_bases: host array of the N ranks' window bases
 * (this rank's own allocation at index rank, IPC-opened mappings of the others). */
int disco_b200_peer_bytes(int64_t B, int64_t D, int world, int rank, int64_t* bytes);
int disco_b200_peer_handle_bytes(void);
int disco_b200_peer_alloc(int64_t bytes, void** ptr, void* ipc_handle);
int disco_b200_peer_open(const void* ipc_handle, void** ptr);
int disco_b200_peer_close(void* ptr);
int disco_b200_peer_free(void* ptr);
/* Peer all-gather (replaces the NCCL all_gather + unpack at N > 1): publish copies this rank's
 * packed rows (DISCO_R_PACK, written by disco_b200_pack) into its window's parity pack area and
 * raises `epoch` in every window's pack-ready slot [rank]; gather waits (bounded, status flag 8)
 * for all N pack-ready slots, then reads every rank's packed rows straight from its window
 * (NVLink loads) into the forward (bf16) and backward (f16) operand layouts.  Follow it with
 * disco_b200_forward_gathered (the forward without its unpack step). */
int disco_b200_peer_publish(void* ws, int64_t B, int64_t D, int world, int rank, const uint64_t* peer_bases,
                            int parity, uint32_t epoch, void* stream);
int disco_b200_peer_gather(void* ws, int64_t B, int64_t D, int world, int rank, const uint64_t* peer_bases,
                           int parity, uint32_t epoch, double timeout_s, void* stream);
int disco_b200_forward_gathered(void* ws, int64_t B, int64_t D, int world, int rank, float t, void* stream);
/* Streamed alternative (all-gather overlapped with the logits GEMM, canonical shapes): after
 * disco_b200_peer_publish, peer_gather_streamed enqueues on a copy stream, for k = 0..N-1 and
 * src = (rank + k) % N, a cuStreamWaitValue32 on src's pack-ready slot (no SM), the copy of src's
 * rows (NVLink, copy engine) into the forward operands, and a stream write of wave flag k;
 * forward_peer_streamed (enqueued after it on the compute stream) is ONE persistent logits
 * launch whose producers take the column waves in that order, waiting on each flag (bounded:
 * status flag 16), then derives the f16 operands and the statistics.  Results are bit-identical
 * to the other gather paths.  Not for ranks sharing a GPU inside one process (the spinning
 * kernel can hold the SMs another rank's pack needs). */
int disco_b200_peer_gather_streamed(void* ws, int64_t B, int64_t D, int world, int rank, const uint64_t* peer_bases,
                                    int parity, uint32_t epoch, void* copy_stream);
int disco_b200_forward_peer_streamed(void* ws, int64_t B, int64_t D, int world, int rank, float t, uint32_t epoch,
                                     double timeout_s, void* stream);
int disco_b200_backward_peer(void* ws, int64_t B, int64_t D, int world, int rank, const uint64_t* peer_bases,
                             int parity, uint32_t epoch, void* stream);
/* Loss at N > 1 with the peer transport: disco_b200_backward_peer also pushes the rank's per-row
 * ce into every window's parity ce area ([N][2][b] f32, covered by the same arrival epoch), so
 * after disco_b200_combine_peer the loss needs no collective: same fixed-order f64 sum as
 * disco_b200_loss over the gathered ce. */
int disco_b200_loss_peer(void* ws, int64_t B, int64_t D, int world, int rank, const void* my_base, int parity,
                         void* stream);
int disco_b200_combine_peer(void* ws, int64_t B, int64_t D, int world, int rank, float t, int flip,
                            const void* my_base, int parity, uint32_t epoch, double timeout_s, float* d_image,
                            float* d_text, int64_t ld_out, void* stream);

/* Full-size per-rank contribution (LocalGradContribution, shard.py:61-80,
 * 153-162): t*0.5/b * (scatter(intra) + send slabs), B x D fp32 each. */
int disco_b200_contribution(void* ws, int64_t B, int64_t D, int world, int rank, float t, int flip,
                            float* d_image_full, float* d_text_full, int64_t ld_out, void* stream);

/* Dual backward (DISCO_PATH_DUAL; disco_step's backward for canonical shapes at every N).
 * The gradient of rank n's rows needs, besides its own softmax rows G_d[r, :], the other
 * direction's softmax at column r of every row c, G_d'[c, r] = exp2(y[r, c] - lse2_d'[c]) --
 * a logit rank n already holds in its own E block.  So after the forward (whose per-row lse2 and
 * ce land in DISCO_R_XCHG) the ranks all_gather DISCO_R_XCHG into DISCO_R_XALL (4 b floats per
 * rank; nothing to do at N = 1), and then:
 *   dual_prep      column factors from the gathered statistics (flip != 0: the flip hook's sign
 *                  on columns outside this rank's rows, shard.py:158-162);
 *   backward_dual  one GEMM per gradient, H'_d = 2^14 (G_d + G_d'^T) formed in shared memory
 *                  from E, rows [row0, row1) (256-aligned or row1 == b) into DISCO_R_INTRA;
 *   combine_dual   d = 0.5 t / B (2^-14 (K halves) + label term in fp32) for rows [row0, row1);
 *   dual_fixup     exact fp32 recompute of the rows whose E range could not carry a column term
 *                  (queued by backward_dual; the count is Status offset 12; normally none).
 * Together they replace the reference's all_reduce(AVG) + slice (shard.py:199-208) with results
 * bitwise independent of N (every reduction is a fixed function of B). */
int disco_b200_dual_prep(void* ws, int64_t B, int64_t D, int world, int rank, int flip, void* stream);
/* One direction of dual_prep / backward_dual / combine_dual (the split schedule above): dual_prep_dir(d)
 * needs the statistics of every row of direction 1 - d; backward_dual_dir / combine_dual_dir compute
 * exactly the direction-d part of backward_dual / combine_dual (same bits). */
int disco_b200_dual_prep_dir(void* ws, int64_t B, int64_t D, int world, int rank, int dir, int flip, void* stream);
int disco_b200_backward_dual_dir(void* ws, int64_t B, int64_t D, int world, int rank, int dir, int64_t row0,
                                 int64_t row1, void* stream);
int disco_b200_combine_dual_dir(void* ws, int64_t B, int64_t D, int world, int rank, int dir, float t, int64_t row0,
                                int64_t row1, float* d_image, float* d_text, int64_t ld_out, void* stream);
int disco_b200_backward_dual(void* ws, int64_t B, int64_t D, int world, int rank, int64_t row0, int64_t row1,
                             void* stream);
int disco_b200_combine_dual(void* ws, int64_t B, int64_t D, int world, int rank, float t, int64_t row0, int64_t row1,
                            float* d_image, float* d_text, int64_t ld_out, void* stream);
int disco_b200_dual_fixup(void* ws, int64_t B, int64_t D, int world, int rank, float t, int flip, float* d_image,
                          float* d_text, int64_t ld_out, void* stream);
/* Two-tower step: combine_dual + dual_fixup for rows [0, b) with the towers'
 * l2_normalize_rows_backward (matrix.py:178-195) fused into the combine: besides d_image / d_text
 * it writes dx = (d - (u . d) u) / ||raw|| per row (u = raw / ||raw||, f64 row sums, exactly the
 * arithmetic of disco_b200_l2norm_rows_backward), rows the fixup recomputes included.
 * norm_flags: bit0 non-finite dx, bit1 ||raw|| < 1e-12 (as disco_b200_l2norm_rows_backward). */
int disco_b200_finish_dual_l2norm(void* ws, int64_t B, int64_t D, int world, int rank, float t, int flip,
                                  const float* raw_I, int64_t ld_raw_I, const float* raw_T, int64_t ld_raw_T,
                                  float* d_image, float* d_text, int64_t ld_out, float* dx_image, float* dx_text,
                                  int64_t ld_dx, int* norm_flags, void* stream);

/* Loss: fixed-order f64 sum of the gathered per-row ce (DISCO_R_CE_ALL, or
 * DISCO_R_CE when world == 1 or local_only == 1) / (2 * rows) into DISCO_R_STATUS.
 * local_only=1 gives the rank's local_loss (shard.py:140-141); local_only=2 reads every rank's ce
 * from the dual backward's gathered statistics (DISCO_R_XALL). */
int disco_b200_loss(void* ws, int64_t B, int64_t D, int world, int rank, int local_only, void* stream);

/* Logit-scale gradient (the reference has none).
 * The logits are bilinear in (I, T), so dL/dt = (<dL/dI, I> + <dL/dT, T>) / (2t)
 * over the global batch.  _rows writes this rank's per-row terms (with the bf16
 * features the loss used) into DISCO_R_RDOT; after the host all_gathers them into
 * DISCO_R_RDOT_ALL (N > 1), _grad sums them in global-row order (f64, independent
 * of N) and stores dL/dt in the status block (f64 at byte offset 16). */
int disco_b200_logit_scale_rows(void* ws, int64_t B, int64_t D, int world, int rank, const float* d_image,
                                const float* d_text, int64_t ld_out, void* stream);
int disco_b200_logit_scale_grad(void* ws, int64_t B, int64_t D, int world, int rank, float t, void* stream);

/* Profiling aid (synchronous): the SM clock in MHz at which CTA 0 of the last logits kernel
 * (mhz[0]) and of the last backward GEMM (mhz[1]) ran, from clock64 / globaltimer stamps the
 * kernels write into the status block; 0 if not run.  Shows the power-capped effective clock. */
int disco_b200_clock_probe(void* ws, int64_t B, int64_t D, int world, int rank, double* mhz);
/*   mhz must hold 3 doubles: mhz[2] = mean cycles the backward GEMM's epilogue held its
 *   accumulators per unit (TMEM drain + stores) since the previous readout. */

/* Tower side of the two-tower trainer (reference towers.py:148-157):
 * row L2 normalisation of raw tower outputs (matrix.py:165-176) and its backward
 * (matrix.py:178-195), fp32, one warp per row.  flags (device int, may be NULL):
 * bit0 non-finite values, bit1 a row norm below 1e-12 (DegenerateInputError). */
int disco_b200_l2norm_rows(const float* raw, int64_t ld_raw, int64_t rows, int64_t D, float* out, int64_t ld_out,
                           float* norms, int* flags, void* stream);
int disco_b200_l2norm_rows_backward(const float* raw, int64_t ld_raw, const float* grad, int64_t ld_grad, int64_t rows,
                                    int64_t D, float* out, int64_t ld_out, int* flags, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* DISCO_B200_H_ */
