// Host side: geometry, workspace layout, tensor maps, launchers (everything the C ABI calls).
// Part of the single translation unit disco_b200.cu (included there, in this order).
#pragma once

namespace disco {

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

// unit selection of the split modes (wave -4: k0; wave -5: the rectangle)
struct UnitRange {
  int k0 = 0;
  int dir = 0, rt0 = 0, nrt = 0, ch0 = 0, nch = 0;
};

int launch_logits(int kind, void* ws, const Geometry& g, float t, cudaStream_t st, int wave = -1,
                  unsigned int epoch = 0, double timeout_s = 0.0, UnitRange ur = UnitRange()) {
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
  if (wave == -2 || wave == -3 || wave == -4) {
    Status* stt = region<Status>(ws, g, DISCO_R_STATUS);
    p.wave_flags = stt->wave_flags;
    p.status_flags = &stt->flags;
    p.nwaves = wave == -3 ? g.N : g.nchunk * g.ssub;
  }
  p.k0 = ur.k0;
  p.rect_dir = ur.dir;
  p.rect_rt0 = ur.rt0;
  p.rect_nrt = ur.nrt;
  p.rect_ch0 = ur.ch0;
  p.rect_nch = ur.nch;
  const int64_t ndir = 2;
  const int64_t R = p.rt_per_chunk;
  const int64_t units = wave == -3 ? int64_t(2) * p.row_tiles * p.nchunk
                      : wave == -4 ? R * p.nwaves * p.nwaves + R * ur.k0 * ur.k0
                      : wave == -5 ? int64_t(ur.nrt) * ur.nch
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
int forward_finish(void* ws, const Geometry& g, cudaStream_t st, int dir0 = 0, int ndir = 2, int64_t row0 = 0,
                   int64_t row1 = -1) {
  float* rows = region<float>(ws, g, DISCO_R_ROWS);
  if (row1 < 0) row1 = g.b;
  const int nrows = int(row1 - row0);
  const int n = ndir * nrows;
  if (n <= 0) return DISCO_OK;
  // column parts per (row, sub-chunk): the FWDE kernel's epilogue parts, or halves (FWD)
  const int nparts = g.estore ? FWDE_PARTS : 2;
  stats_combine_kernel<<<(n + 255) / 256, 256, 0, st>>>(region<float2>(ws, g, DISCO_R_STATS), rows, g.nchunk, g.ssub,
                                                        nparts, int(g.b), dir0, ndir, int(row0), nrows,
                                                        lse2_of(ws, g), rows + 4 * g.b,
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
