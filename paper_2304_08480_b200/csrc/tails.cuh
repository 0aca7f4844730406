// HBM-bound and latency-bound kernels: pack / unpack, statistics, combines, dual backward
// helpers, peer-transport kernels, loss, tower normalisation.
// Part of the single translation unit disco_b200.cu (included there, in this order).
#pragma once

namespace disco {

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
// rows [row0, row0 + nrows) of directions [dir0, dir0 + ndir)
__global__ void stats_combine_kernel(const float2* stats, const float* target, int nchunk, int ssub, int nparts,
                                     int b, int dir0, int ndir, int row0, int nrows, float* lse2_out,
                                     float* glabel_out, float* ce_out, Status* status) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= ndir * nrows) return;
  const int dir = dir0 + j / nrows, r = row0 + j % nrows;
  const int i = dir * b + r;
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
__global__ void dual_prep_kernel(const float* xall, int b, int groups, int rank, int flip, float* q, float2* gm,
                                 int d0 = 0, int nd = 2) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= nd * groups) return;
  const int d = d0 + w / groups, g = w % groups, e = 1 - d;
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
                                    int row0, int nrows, Status* status, int g0 = 0, int ng = 2) {
  const int v4 = Dp / 4;
  const bool vec_out = (ld_out % 4 == 0) && ((reinterpret_cast<uintptr_t>(d_image) | reinterpret_cast<uintptr_t>(d_text)) % 16 == 0);
  const int64_t per_g = int64_t(b) * v4;
  const unsigned pb = unsigned(int64_t(nrows) * v4), uv4 = unsigned(v4);
  const int64_t total = ng * int64_t(pb);
  bool bad = false;
  for (int64_t ii = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; ii < total; ii += int64_t(gridDim.x) * blockDim.x) {
    const unsigned iu = unsigned(ii);
    const int gl = int(iu / pb), g = g0 + gl;
    const int64_t rem = int64_t(iu - unsigned(gl) * pb) + int64_t(row0) * v4;
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

}  // namespace disco
