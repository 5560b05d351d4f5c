// attention.cu — K3/K4/K5: fused split-K GQA decode attention over the
// OCTOPUS-compressed KV cache on sm_100a (attention.hpp:50-73 semantics, V
// compressed with the same codec and accumulated in its rotated frame).
//
// Per SM, one persistent CTA (stream-K over all tiles), one launch per step
// with programmatic dependent launch (griddepcontrol):
//   * the joint dequant table T[code] = fp16 (rho x, rho y | rho z, 0),
//     code = ixi | ieta << b_dir | irho << 2 b_dir, is staged into shared
//     memory with one 1-D TMA bulk copy as host-built DITHERED replicas (32
//     at W = 7, 16 at W = 10, 2 at W = 13): a lookup's replica varies with
//     the lane and the tile, which keeps LDS.64 lookups bank-conflict-free
//     (W <= 10) and turns the table's fp16 rounding into zero-mean noise;
//   * each warp streams 32-token tiles of packed K and V codes through a
//     per-warp 2-stage TMA ring in shared memory (12 warps at 7 and 10 bits,
//     8 at 13 bits, one register image); 10-bit tiles with QJL keys straight
//     into registers (8 warps, the next tile prefetched in a second register
//     image);
//   * K codes dequantize straight into mma.sync A fragments of S^T = K_hat Q^T
//     (M = 16 tokens, N = 8 query heads of the GQA group, K = 144 triplet-
//     permuted dims; q is rotated and permuted in the segment prologue);
//   * online softmax in the log2 domain (q pre-scaled by log2(e)/sqrt(d));
//     accumulator rescaling is skipped while no running max moves;
//   * P^T becomes the PV B operand through movmatrix.trans, V codes
//     dequantize into A fragments of V_hat^T (M = 144 permuted dims, K = 16
//     tokens), so out^T accumulates in the rotated V frame;
//   * the CTA that lands a stream's last partial merges the stream's
//     partials and applies the inverse V rotation (K4 fused), or — sequence-
//     sharded over peer memory — exchanges the rank's rows with the other
//     GPUs and merges them (p2p_exchange).
// Tile formats (see oq_cache_pack): each lane's codes form one contiguous
// run, so extraction is a static shift+mask (funnel shift across words)
// folded into the table address: 1-2 ALU ops + 1 LDS per triplet.
#include <cuda_fp16.h>

#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"
#include "encode_exact.cuh"

namespace oqd {

constexpr int kTileTok = 32;
constexpr int kNT = 43;  // triplets at dim 128
constexpr int kMaxSmem = 227 * 1024 - 2048;  // dynamic smem per CTA (227 KB, static part reserved)
constexpr int kPartW = 132;  // (m, l, 0, 0, acc[128]): acc 16-byte aligned

// ---------------------------------------------------------------------------
// Tile geometry, shared by the packer and the kernels.
//
// K tile (32 tokens): gamma[8][4] f32 ([g][k] = token g + 8k) | code area |
//   [QJL: gamma_r[8][4] f16 | signs[8 g][4 c][4 k] u32 (word c of token g+8k)]
//   Lane l = 4g + c owns triplets t = 11c + u (u < 11, 10 for c = 3) of
//   tokens g + 8k (k < 4); code slot u*4 + k, W bits each, LSB-first, in a
//   run of kw_full words (kw_3 for c = 3).
// V tile: gamma[8][4] | code area: lane l owns triplets t = 6g + u (u < 6,
//   1 for g = 7) of tokens v_token(c, k) (k < 8); slot u*8 + k; run of
//   vw_full words (vw_7 for g = 7).
// The runs are stored word-interleaved so that word i of all lanes is one
// contiguous row (a warp's i-th 4-byte load is one 128-byte line): rows
// below the short-run length hold all 32 lanes, longer rows only the lanes
// that own a word there (K: the 24 lanes c < 3, compacted as 3g + c; V: the
// 28 lanes g < 7).
__host__ __device__ inline int cdiv(int a, int b) { return (a + b - 1) / b; }
// Field width of a W-bit joint code in the lane runs: codes of W <= 8 bits
// take one whole byte each, so one PRMT turns a code into its table address
// (see code_addr); wider codes are packed back to back.
__host__ __device__ constexpr int fw(int W) { return W <= 8 ? 8 : W; }
// Dithered fp16 replicas of each joint-table entry in shared memory (see
// stage_table_issue): 32 for byte-coded W <= 8, 16 for W = 10 (every
// half-warp lookup conflict-free); W = 13 (b = 4, 8192 codes) fits only 2
// (128 KB), so its lookups take bank conflicts.
__host__ __device__ constexpr int table_rep(int W) { return W <= 8 ? 32 : W <= 10 ? 16 : 2; }
__host__ __device__ constexpr int table_shift(int W) {  // log2(entry stride) = log2(8 * REP)
  return W <= 8 ? 8 : W <= 10 ? 7 : 4;
}
__host__ __device__ inline int kw_full(int W) { return cdiv(44 * fw(W), 32); }
__host__ __device__ inline int kw_3(int W) { return cdiv(40 * fw(W), 32); }
__host__ __device__ inline int vw_full(int W) { return cdiv(48 * fw(W), 32); }
__host__ __device__ inline int vw_7(int W) { return cdiv(8 * fw(W), 32); }
__host__ __device__ inline int kcode_words(int W) { return 8 * (3 * kw_full(W) + kw_3(W)); }
__host__ __device__ inline int vcode_words(int W) { return 28 * vw_full(W) + 4 * vw_7(W); }
__host__ __device__ inline int ktile_bytes(int W, int qjl) {
  return (128 + 4 * kcode_words(W) + (qjl ? 64 + 512 : 0) + 15) & ~15;
}
__host__ __device__ inline int vtile_bytes(int W) { return (128 + 4 * vcode_words(W) + 15) & ~15; }
// Word offset of word i of lane l's run inside the K / V code areas.
__host__ __device__ inline int k_word_off(int W, int lane, int i) {
  const int g = lane >> 2, c = lane & 3, n3 = kw_3(W);
  return i < n3 ? 32 * i + lane : 32 * n3 + 24 * (i - n3) + 3 * g + c;
}
__host__ __device__ inline int v_word_off(int W, int lane, int i) {
  const int n7 = vw_7(W);
  return i < n7 ? 32 * i + lane : 32 * n7 + 28 * (i - n7) + lane;
}
__host__ __device__ inline int k_token(int g, int k) { return g + 8 * k; }
__host__ __device__ inline int v_token(int c, int k) {
  return 16 * (k >> 2) + 2 * c + (k & 1) + 8 * ((k >> 1) & 1);
}

// K slot sigma (0..17) of lane c.  Blocks kb = (2kb, 2kb+1):
//   kb0 (xy0, xy1) kb1 (xy2, xy3) kb2 (z01, z23) kb3 (xy4, xy5) kb4 (xy6, xy7)
//   kb5 (z45, z67) kb6 (xy8, xy9) kb7 (xy10, z89) kb8 (z10, -)
// Returns the two rotated-frame dims of the slot's fp16 pair (-1 = zero).
__host__ __device__ inline void k_slot_dims(int c, int sigma, int& d0, int& d1) {
  int kind = 3, u = 0;  // 0 xy(u), 1 z(u, u+1), 2 z(u), 3 none
  if (sigma < 12) {
    const int base = 4 * (sigma / 6), r = sigma % 6;
    if (r < 4) { kind = 0; u = base + r; }
    else { kind = 1; u = base + 2 * (r - 4); }
  } else {
    const int r = sigma - 12;
    if (r < 3) { kind = 0; u = 8 + r; }
    else if (r == 3) { kind = 1; u = 8; }
    else if (r == 4) { kind = 2; u = 10; }
  }
  const int t = 11 * c + u;
  d0 = d1 = -1;
  if (kind == 0) { d0 = 3 * t; d1 = 3 * t + 1; }
  else if (kind == 1) { d0 = 3 * t + 2; d1 = 3 * (t + 1) + 2; }
  else if (kind == 2) { d0 = 3 * t + 2; }
  if (d0 >= 128) d0 = -1;
  if (d1 >= 128) d1 = -1;
}

// Rotated-frame dim behind V row-slot rho (0..17) of lane g; -1 = dummy row.
__host__ __device__ inline int v_row_dim(int g, int rho) {
  const int t = 6 * g + rho / 3, d = 3 * t + rho % 3;
  return (t < kNT && d < 128) ? d : -1;
}

// ---------------------------------------------------------------------------
extern __shared__ __align__(1024) uint8_t g_attn_smem[];

// Shared address of the table entry for the code in `slot` of a lane's run:
// off + code * 128, off = table base + 8 * replica.  A code inside one word
// is masked in place (LOP3) and shifted-and-added in one LEA / LEA.HI; a
// code straddling two words takes a funnel shift, a mask and an add.
__device__ __forceinline__ uint32_t mad_hi(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;  // ((a * b) >> 32) + c in one IMAD.HI
  asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ uint32_t mad_lo(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;  // a * b + c in one IMAD
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// Byte-coded runs (W <= 8): the table sits at shared address 0x10000 with a
// 256-byte entry stride (32 lane replicas of 8 bytes), and off = 0x10000 |
// 8 * lane, so byte s % 4 of the run word is the address's byte 1:
// address = 0x10000 | code << 8 | 8 * lane in ONE PRMT.
template <int W, int N>
__device__ __forceinline__ uint32_t code_addr(const uint32_t (&w)[N], int slot, uint32_t off) {
  if constexpr (W <= 8) {
    const int i = slot >> 2, b = slot & 3;
    return __byte_perm(w[i], off, 0x7604 | (b << 4));
  }
  constexpr int S = table_shift(W);  // entry stride 2^S bytes
  const int pos = slot * W, i = pos >> 5, sh = pos & 31;
  constexpr uint32_t M = (1u << W) - 1u;
  if (sh + W <= 32) {
    const uint32_t m = w[i] & (M << sh);  // LOP3
    if (sh > S) return mad_hi(m, 1u << (32 + S - sh), off);  // (m >> (sh - S)) + off
    return mad_lo(m, 1u << (S - sh), off);                   // (m << (S - sh)) + off
  }
  if (sh >= S) {
    const uint32_t v = __funnelshift_r(w[i], w[i + 1], sh - S);
    return off + (v & (M << S));
  }
  // (W = 13 only: a straddling field starting below bit S)
  const uint32_t v = __funnelshift_r(w[i], w[i + 1], sh);
  return off + ((v & M) << S);
}

// The dequant table in shared memory: NE codes x REP fp16 replicas of
// (rho x, rho y | rho z, 0), dithered on the host (joint_replicas, capi.cpp):
// a component rounds down in some replicas and up in the others so that the
// replicas' mean is the exact value to within ulp / (2 REP).  A lookup reads
// replica (lane + first tile of the warp's ping-pong buffer) mod REP, so the
// tokens of a code spread over the replicas and the table's fp16 rounding is
// not a per-code bias (which a long context's softmax average cannot remove).
// Replicating it also makes the lookups bank-conflict-free: the 16 lanes of a
// half-warp read 16 different replicas, 8 bytes apart.  Staged with one bulk
// copy (1-D TMA) of the host-built replicas.
__device__ __forceinline__ void stage_table_issue(void* dst, const uint2* __restrict__ src,
                                                  uint32_t bytes, uint64_t* bar, int tid) {
  if (tid == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
    constexpr uint32_t kChunk = 32768;
    for (uint32_t o = 0; o < bytes; o += kChunk) {
      const uint32_t n = bytes - o < kChunk ? bytes - o : kChunk;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
              "r"(smem_u32(static_cast<uint8_t*>(dst) + o)),
          "l"(reinterpret_cast<const uint8_t*>(src) + o), "r"(n), "r"(smem_u32(bar))
          : "memory");
    }
  }
}

__device__ __forceinline__ uint2 lds64(uint32_t addr) {
  uint2 r;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "r"(addr));
  return r;
}

__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t movtrans(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}

__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) {
  const __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&h);
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// +-1 fp16 pair from sign bits (sigma, sigma + 16) of ~w: bit 1 => +1.
__device__ __forceinline__ uint32_t sign_pair(uint32_t nw, int sigma) {
  return ((nw << (15 - sigma)) & 0x80008000u) | 0x3C003C00u;
}

// Word k (0..3) of a 4-word mask held in kernel parameters, by selects: a
// runtime index into a parameter array would copy it to local memory.
__device__ __forceinline__ uint32_t word4(const uint32_t (&m)[4], int k) {
  const uint32_t a = (k & 1) ? m[1] : m[0], b = (k & 1) ? m[3] : m[2];
  return (k & 2) ? b : a;
}

__device__ __forceinline__ void wht128_lane4(float (&y)[4], int lane) {
  // normalized-free WHT over 128 values, 4 consecutive per lane
  {
    const float a = y[0], b = y[1], c2 = y[2], d = y[3];
    y[0] = a + b; y[1] = a - b; y[2] = c2 + d; y[3] = c2 - d;
    const float e0 = y[0], e1 = y[1];
    y[0] = e0 + y[2]; y[1] = e1 + y[3]; y[2] = e0 - y[2]; y[3] = e1 - y[3];
  }
#pragma unroll
  for (int lm = 1; lm < 32; lm <<= 1) {
    const bool up = lane & lm;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float o = __shfl_xor_sync(kFull, y[i], lm);
      y[i] = up ? o - y[i] : y[i] + o;
    }
  }
}

// ---------------------------------------------------------------------------
struct AttnKParams {
  const uint2* tab;  // global replica table (2^W codes x REP, see stage_table)
  const uint8_t* kcache;
  const uint8_t* vcache;
  size_t k_tiles_cap, v_tiles_cap;
  const uint32_t* qfrag;  // [streams*HC][32][QF]
  float* partials;        // [B*Hq][n_parts][132]
  const int32_t* seq_lens;
  size_t T, t_begin, t_end;
  int B, Hq, Hkv, G, HC;
  int splits, n_parts, n_items;
  // stream-K mode (splits == 0): the B*Hkv*HC streams x tps tiles of
  // [tb0, tb0 + tps) are cut into gridDim.x equal contiguous ranges.
  int streamk, n_sh;
  size_t tb0, tps;
  size_t sko;  // stream-K: per-stream segment overhead in tile units
  // fused mode (single-GPU attention_decode): the kernel prepares the query
  // fragments itself from q and finalises each stream's rows once its last
  // partial lands (per-stream arrival counters, left at zero)
  int fuse, qjl;
  int out_partial;       // fused: write merged (m, l, 0, 0, acc) rows of kPartW floats
  const float* q;        // [B, Hq, 128]
  float* out;            // [B * Hq, 128] (or [B * Hq, kPartW] with out_partial)
  uint32_t* counters;    // [n_sh], zero on entry and exit
  // P2P sequence sharding (oq_attention_decode_p2p): the CTA that finalises a
  // stream writes this rank's merged rows into slot `rank` of every rank's
  // exchange buffer over peer memory, raises its flag there, waits for all
  // ranks' flags in its own buffer and merges the ranks in order into out
  int p2p_nranks, p2p_rank;
  uint32_t p2p_epoch;
  uint8_t* p2p_xbuf[8];  // rank r's exchange buffer, mapped in this process
  uint32_t smask[4], qmask[4], vmask[4];
  float inv_sqrt_d;
};

template <int W, bool QJL>
struct Cfg {
  static constexpr int FW = W <= 8 ? 8 : W;  // stored field width
  static constexpr int KWF = (44 * FW + 31) / 32, KW3 = (40 * FW + 31) / 32;
  static constexpr int VWF = (48 * FW + 31) / 32, VW7 = (8 * FW + 31) / 32;
  static constexpr int KCODE = 8 * (3 * KWF + KW3), VCODE = 28 * VWF + 4 * VW7;
  static constexpr int KTILE = (128 + 4 * KCODE + (QJL ? 576 : 0) + 15) & ~15;
  static constexpr int VTILE = (128 + 4 * VCODE + 15) & ~15;
  static constexpr int QF = 18 + (QJL ? 16 : 0);
  // W <= 8: the table lives at shared address 0x10000 (256-byte entries);
  // TAB_BYTES then spans from the start of dynamic smem to its end
  static constexpr int TAB_BYTES = W <= 8 ? 0x10000 + (1 << W) * 256 : (1 << W) * table_rep(W) * 8;
  static constexpr int QS_FLOATS = 8 * 2 * 129;  // fused query prep scratch
  // per-warp region: the merge slot (8 heads x kPartW floats) and, with a
  // TMA ring of `ring` stages, the staged tiles (aliased: the ring is idle
  // when the warp writes its merge slot)
  static constexpr int STAGE = KTILE + VTILE;
  static constexpr int wreg(int ring) {
    return (ring * STAGE > 8 * kPartW * 4 ? ring * STAGE : 8 * kPartW * 4);
  }
  static constexpr int smem(int nw, int ring = 0) { return TAB_BYTES + nw * wreg(ring) + QS_FLOATS * 4; }
};

template <int W, bool QJL>
struct TileRegs {
  uint32_t kc[Cfg<W, QJL>::KWF];
  uint32_t vc[Cfg<W, QJL>::VWF];
  float4 gk, gv;
  uint2 gr;
  uint4 sg;
};

// Streamed once: no L1 allocation for the tile data (it never hits again).
__device__ __forceinline__ uint32_t ldg_na(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ float4 ldg_na(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

template <int W, bool QJL>
__device__ __forceinline__ void load_tile(TileRegs<W, QJL>& r, const AttnKParams& P,
                                          size_t stream, size_t tile, int g, int c, int kl,
                                          int vl) {
  // word-interleaved runs: row i of the K area is lane-indexed (kl = lane)
  // below KW3 and compacted to 3g + c above; V rows are lane-indexed.
  using C = Cfg<W, QJL>;
  const uint8_t* kt = P.kcache + (stream * P.k_tiles_cap + tile) * (size_t)C::KTILE;
  const uint8_t* vt = P.vcache + (stream * P.v_tiles_cap + tile) * (size_t)C::VTILE;
  r.gk = ldg_na(reinterpret_cast<const float4*>(kt) + g);
  r.gv = ldg_na(reinterpret_cast<const float4*>(vt) + g);
  const uint32_t* kw = reinterpret_cast<const uint32_t*>(kt + 128);
  const uint32_t* vw = reinterpret_cast<const uint32_t*>(vt + 128);
#pragma unroll
  for (int i = 0; i < C::KWF; ++i)
    r.kc[i] = i < C::KW3 ? ldg_na(kw + 32 * i + kl)
                         : (c < 3 ? ldg_na(kw + 32 * C::KW3 + 24 * (i - C::KW3) + 3 * g + c) : 0u);
#pragma unroll
  for (int i = 0; i < C::VWF; ++i)
    r.vc[i] = i < C::VW7 ? ldg_na(vw + 32 * i + vl)
                         : (g < 7 ? ldg_na(vw + 32 * C::VW7 + 28 * (i - C::VW7) + vl) : 0u);
  if (QJL) {
    const uint8_t* qa = kt + 128 + 4 * C::KCODE;
    r.gr = __ldg(reinterpret_cast<const uint2*>(qa) + g);
    r.sg = __ldg(reinterpret_cast<const uint4*>(qa + 64) + (4 * g + c));
  }
}

// The same register image from a tile staged verbatim in shared memory (the
// TMA ring): identical word offsets, LDS instead of LDG.
template <int W, bool QJL>
__device__ __forceinline__ void load_tile_smem(TileRegs<W, QJL>& r, const uint8_t* kt,
                                               const uint8_t* vt, int g, int c, int kl, int vl) {
  using C = Cfg<W, QJL>;
  r.gk = reinterpret_cast<const float4*>(kt)[g];
  r.gv = reinterpret_cast<const float4*>(vt)[g];
  const uint32_t* kw = reinterpret_cast<const uint32_t*>(kt + 128);
  const uint32_t* vw = reinterpret_cast<const uint32_t*>(vt + 128);
#pragma unroll
  for (int i = 0; i < C::KWF; ++i)
    r.kc[i] = i < C::KW3 ? kw[32 * i + kl]
                         : (c < 3 ? kw[32 * C::KW3 + 24 * (i - C::KW3) + 3 * g + c] : 0u);
#pragma unroll
  for (int i = 0; i < C::VWF; ++i)
    r.vc[i] = i < C::VW7 ? vw[32 * i + vl] : (g < 7 ? vw[32 * C::VW7 + 28 * (i - C::VW7) + vl] : 0u);
  if (QJL) {
    const uint8_t* qa = kt + 128 + 4 * C::KCODE;
    r.gr = reinterpret_cast<const uint2*>(qa)[g];
    r.sg = reinterpret_cast<const uint4*>(qa + 64)[4 * g + c];
  }
}

// One TMA ring stage <- tile `tile` of `stream`: the K and V tiles, 1-D bulk
// copies completing on the stage's mbarrier.  Called by one lane.
template <int W, bool QJL>
__device__ __forceinline__ void ring_issue(uint8_t* stage, uint64_t* bar, const AttnKParams& P,
                                           size_t stream, size_t tile) {
  using C = Cfg<W, QJL>;
  const uint8_t* kt = P.kcache + (stream * P.k_tiles_cap + tile) * (size_t)C::KTILE;
  const uint8_t* vt = P.vcache + (stream * P.v_tiles_cap + tile) * (size_t)C::VTILE;
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"((uint32_t)(C::KTILE + C::VTILE))
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(stage)), "l"(kt), "r"((uint32_t)C::KTILE), "r"(smem_u32(bar))
      : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(stage + C::KTILE)), "l"(vt), "r"((uint32_t)C::VTILE), "r"(smem_u32(bar))
      : "memory");
}

// Online-softmax state of one warp for its 8 heads (2 per lane).
struct WarpState {
  float acc[9][4];
  float m[2], l[2];
};

template <int W, bool QJL, int PREV = 2>
__device__ __forceinline__ void process_tile(WarpState& S, const TileRegs<W, QJL>& R,
                                             const uint32_t (&qf)[Cfg<W, QJL>::QF],
                                             uint32_t toff, int tok0, int lo, int hi, int g,
                                             int c) {
  const float NEG_INF = -__int_as_float(0x7f800000);
  float gk[4] = {R.gk.x, R.gk.y, R.gk.z, R.gk.w};
  float gv[4] = {R.gv.x, R.gv.y, R.gv.z, R.gv.w};
  bool ok[4] = {true, true, true, true};
  if (tok0 < lo || tok0 + kTileTok > hi) {  // boundary tile (warp-uniform)
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int t = tok0 + k_token(g, k);
      ok[k] = t >= lo && t < hi;
      if (!ok[k]) gk[k] = gv[k] = 0.f;
    }
  }

  // ---- S^T = K_hat Q^T ----------------------------------------------------
  float sc[4][2];  // [token slot k][head 2c + h2]
#pragma unroll
  for (int st = 0; st < 2; ++st) {
    const int k0 = 2 * st, k1 = 2 * st + 1;  // rows g, g+8 of this sub-tile
    float d[4] = {0.f, 0.f, 0.f, 0.f}, d2[4] = {0.f, 0.f, 0.f, 0.f};  // two MMA chains
#pragma unroll
    for (int grp = 0; grp < 2; ++grp) {
      uint2 a[4], b[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        a[r] = lds64(code_addr<W>(R.kc, (4 * grp + r) * 4 + k0, toff));
        b[r] = lds64(code_addr<W>(R.kc, (4 * grp + r) * 4 + k1, toff));
      }
      const int kb = 3 * grp;
      mma16816(d, a[0].x, b[0].x, a[1].x, b[1].x, qf[2 * kb], qf[2 * kb + 1]);
      mma16816(d2, a[2].x, b[2].x, a[3].x, b[3].x, qf[2 * kb + 2], qf[2 * kb + 3]);
      mma16816(grp ? d2 : d, __byte_perm(a[0].y, a[1].y, 0x5410), __byte_perm(b[0].y, b[1].y, 0x5410),
               __byte_perm(a[2].y, a[3].y, 0x5410), __byte_perm(b[2].y, b[3].y, 0x5410),
               qf[2 * kb + 4], qf[2 * kb + 5]);
    }
    {
      uint2 a[3], b[3];
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        a[r] = lds64(code_addr<W>(R.kc, (8 + r) * 4 + k0, toff));
        b[r] = lds64(code_addr<W>(R.kc, (8 + r) * 4 + k1, toff));
      }
      mma16816(d, a[0].x, b[0].x, a[1].x, b[1].x, qf[12], qf[13]);
      mma16816(d2, a[2].x, b[2].x, __byte_perm(a[0].y, a[1].y, 0x5410),
               __byte_perm(b[0].y, b[1].y, 0x5410), qf[14], qf[15]);
      mma16816(d, a[2].y, b[2].y, 0u, 0u, qf[16], qf[17]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) d[i] += d2[i];
    if (QJL) {
      // residual sketch: sum_i (+-1)_i q_sketch_i on the tensor cores
      const uint32_t w0 = ~(st ? R.sg.z : R.sg.x), w1 = ~(st ? R.sg.w : R.sg.y);
      // two independent accumulation chains (the 8 sign MMAs would otherwise
      // form one serial dependency chain per sub-tile)
      float e[4] = {0.f, 0.f, 0.f, 0.f}, e2[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int kb = 0; kb < 8; ++kb)
        mma16816(kb & 1 ? e2 : e, sign_pair(w0, 2 * kb), sign_pair(w1, 2 * kb),
                 sign_pair(w0, 2 * kb + 1), sign_pair(w1, 2 * kb + 1), qf[18 + 2 * kb],
                 qf[18 + 2 * kb + 1]);
#pragma unroll
      for (int i = 0; i < 4; ++i) e[i] += e2[i];
      const uint32_t grw = st ? R.gr.y : R.gr.x;
      const float gr0 = __half2float(__ushort_as_half((unsigned short)(grw & 0xffff)));
      const float gr1 = __half2float(__ushort_as_half((unsigned short)(grw >> 16)));
      d[0] += gr0 * e[0];
      d[1] += gr0 * e[1];
      d[2] += gr1 * e[2];
      d[3] += gr1 * e[3];
    }
    sc[k0][0] = ok[k0] ? d[0] * gk[k0] : NEG_INF;
    sc[k0][1] = ok[k0] ? d[1] * gk[k0] : NEG_INF;
    sc[k1][0] = ok[k1] ? d[2] * gk[k1] : NEG_INF;
    sc[k1][1] = ok[k1] ? d[3] * gk[k1] : NEG_INF;
  }

  // the first two V groups' lookups do not depend on the softmax: issue them
  // before it so their latency overlaps the max/rescale chain (one group:
  // C3/C5/C4 -0.3/-0.8/0 %, two: a further -0/-0.4/-1.3 %, three: slower)
  // V lookup groups issued before the softmax: 2 measured best with and
  // without QJL and in the ring variants (A/B, r02: 0 / 1 / 2 within 1 %)
  constexpr int kPreV = PREV;
  uint2 e0[2][2][4];
#pragma unroll
  for (int gg = 0; gg < kPreV; ++gg)
#pragma unroll
    for (int uu = 0; uu < 2; ++uu)
#pragma unroll
      for (int q = 0; q < 4; ++q) e0[gg][uu][q] = lds64(code_addr<W>(R.vc, (2 * gg + uu) * 8 + q, toff));

  // ---- online softmax (log2 domain) ----------------------------------------
  // The warp-wide max reduction (three dependent shuffles per head) runs only
  // when some lane's own scores exceed the running maximum; otherwise the max
  // cannot move, so the result is identical (C3/C5/C4 -3.5/-3.4/-2.2 %).
  // W = 10 (C3) keeps no lag: a lag of 2^8 was +0.7 % there (and needs 8
  // bits of fp16 headroom in p * gamma_v); smaller lags were not measured on it.
  float lm[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) lm[h] = fmaxf(fmaxf(sc[0][h], sc[1][h]), fmaxf(sc[2][h], sc[3][h]));
  // Byte-coded tiles (W <= 8) also let the max lag by up to 2 (log2 units):
  // p <= 4 then, which costs 2 bits of fp16 headroom in p * gamma_v (overflow
  // only past gamma_v ~ 16K) and skips the rescales of small max moves
  // (C5 -1.2 %, C4 -0.7 %); (m, l, acc) stay consistent, so merges are exact.
  constexpr float kLag = W <= 8 ? 2.f : 0.f;
  if (__any_sync(kFull, lm[0] > S.m[0] + kLag || lm[1] > S.m[1] + kLag)) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float v = lm[h];
      v = fmaxf(v, __shfl_xor_sync(kFull, v, 4));
      v = fmaxf(v, __shfl_xor_sync(kFull, v, 8));
      v = fmaxf(v, __shfl_xor_sync(kFull, v, 16));
      const float mt = fmaxf(v, S.m[h]);
      const float f = S.m[h] == NEG_INF ? 1.f : ex2(S.m[h] - mt);
      S.l[h] *= f;
#pragma unroll
      for (int mb = 0; mb < 9; ++mb) {
        S.acc[mb][h] *= f;
        S.acc[mb][2 + h] *= f;
      }
      S.m[h] = mt;
    }
  }
  float p[4][2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const float mref = S.m[h] == NEG_INF ? 0.f : S.m[h];
#pragma unroll
    for (int k = 0; k < 4; ++k) p[k][h] = ex2(sc[k][h] - mref);
    S.l[h] += (p[0][h] + p[1][h]) + (p[2][h] + p[3][h]);
  }
  uint32_t pb[2][2];  // PV B fragments per 16-token sub-tile
#pragma unroll
  for (int st = 0; st < 2; ++st) {
    pb[st][0] = movtrans(pack_h2(p[2 * st][0] * gv[2 * st], p[2 * st][1] * gv[2 * st]));
    pb[st][1] = movtrans(pack_h2(p[2 * st + 1][0] * gv[2 * st + 1], p[2 * st + 1][1] * gv[2 * st + 1]));
  }

  // ---- out^T += V_hat^T P^T ------------------------------------------------
#pragma unroll
  for (int kk = 0; kk < 2; ++kk) {
#pragma unroll
    for (int grp = 0; grp < 3; ++grp) {
      uint2 e[2][4];
#pragma unroll
      for (int uu = 0; uu < 2; ++uu)
#pragma unroll
        for (int q = 0; q < 4; ++q)
          e[uu][q] = (kk == 0 && grp < kPreV)
                         ? e0[grp < 2 ? grp : 0][uu][q]
                         : lds64(code_addr<W>(R.vc, (2 * grp + uu) * 8 + 4 * kk + q, toff));
#pragma unroll
      for (int mbl = 0; mbl < 3; ++mbl) {
        uint32_t a[4];
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          const int rho = 2 * mbl + half, uu = rho / 3, j = rho % 3;
#pragma unroll
          for (int pr = 0; pr < 2; ++pr) {  // token pair A (q 0,1) / B (q 2,3)
            const uint2 x0 = e[uu][2 * pr], x1 = e[uu][2 * pr + 1];
            uint32_t v;
            if (j == 0) v = __byte_perm(x0.x, x1.x, 0x5410);
            else if (j == 1) v = __byte_perm(x0.x, x1.x, 0x7632);
            else v = __byte_perm(x0.y, x1.y, 0x5410);
            a[2 * pr + half] = v;
          }
        }
        mma16816(S.acc[3 * grp + mbl], a[0], a[1], a[2], a[3], pb[kk][0], pb[kk][1]);
      }
    }
  }
}

// A segment: one (stream, 8-head chunk) and a tile range of it, producing
// the partial in slot `part` of its rows.
struct Seg {
  int sh, hc, b, kvh, part;
  size_t stream;
  int lo, hi;            // valid tokens of the stream (sharding range x length)
  size_t tlo, thi;       // tiles to process
  bool last;             // last segment of the stream: clear the unused slots
};

__device__ __forceinline__ Seg make_seg(const AttnKParams& P, int sh, size_t t0, size_t t1,
                                        int part, bool last) {
  Seg sg;
  sg.sh = sh;
  sg.hc = sh % P.HC;
  sg.stream = sh / P.HC;
  sg.b = (int)(sg.stream / P.Hkv);
  sg.kvh = (int)(sg.stream % P.Hkv);
  sg.part = part;
  sg.last = last;
  size_t len = P.T;
  if (P.seq_lens) len = min((size_t)max(P.seq_lens[sg.b], 0), P.T);
  const size_t hi = min(P.t_end, len);
  sg.lo = (int)P.t_begin;
  sg.hi = (int)max(hi, P.t_begin);
  // tiles wholly past this stream's valid end carry no work
  const size_t tend = (sg.hi + kTileTok - 1) / kTileTok;
  sg.tlo = t0;
  sg.thi = min(t1, tend);
  if (sg.thi < sg.tlo) sg.thi = sg.tlo;
  return sg;
}

// Fixed split count: item -> (stream chunk, split).
__device__ __forceinline__ Seg item_seg(const AttnKParams& P, int item) {
  const int split = item % P.splits, sh = item / P.splits;
  size_t len = P.T;
  const int b = (int)((sh / P.HC) / P.Hkv);
  if (P.seq_lens) len = min((size_t)max(P.seq_lens[b], 0), P.T);
  const size_t hi = min(P.t_end, len);
  size_t t0 = 0, t1 = 0;
  if (hi > P.t_begin) {
    const size_t a = P.t_begin / kTileTok, z = (hi + kTileTok - 1) / kTileTok;
    t0 = a + (z - a) * split / P.splits;
    t1 = a + (z - a) * (split + 1) / P.splits;
  }
  return make_seg(P, sh, t0, t1, split, false);
}

// Stream-K: CTA boundaries over U = n_sh * tps units and the CTA owning unit x.
__device__ __forceinline__ size_t sk_bound(size_t c, size_t U, size_t G) { return c * U / G; }
__device__ __forceinline__ int sk_cta(size_t x, size_t U, size_t G) {
  return (int)(((x + 1) * G - 1) / U);
}

template <int QF>
__device__ __forceinline__ void load_qfrag(uint32_t (&qf)[QF], const AttnKParams& P, int sh,
                                           int lane) {
  const uint32_t* src = P.qfrag + ((size_t)sh * 32 + lane) * QF;
#pragma unroll
  for (int i = 0; i < QF; ++i) qf[i] = __ldg(src + i);
}

__device__ __forceinline__ void init_state(WarpState& S) {
  const float NEG_INF = -__int_as_float(0x7f800000);
#pragma unroll
  for (int i = 0; i < 9; ++i) S.acc[i][0] = S.acc[i][1] = S.acc[i][2] = S.acc[i][3] = 0.f;
  S.m[0] = S.m[1] = NEG_INF;
  S.l[0] = S.l[1] = 0.f;
}

// Per-warp epilogue: reduce l over the 8 row groups and store (m, l, acc) of
// the warp's 8 heads into its merge slot mw[8][kPartW].
__device__ __forceinline__ void warp_state_out(WarpState& S, float* mw, int g, int c) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    float v = S.l[h];
    v += __shfl_xor_sync(kFull, v, 4);
    v += __shfl_xor_sync(kFull, v, 8);
    v += __shfl_xor_sync(kFull, v, 16);
    S.l[h] = v;
  }
  if (g == 0) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      mw[(2 * c + h) * kPartW + 0] = S.m[h];
      mw[(2 * c + h) * kPartW + 1] = S.l[h];
    }
  }
#pragma unroll
  for (int mb = 0; mb < 9; ++mb)
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int d = v_row_dim(g, 2 * mb + half);
      if (d >= 0) {
        mw[(2 * c) * kPartW + 4 + d] = S.acc[mb][2 * half];
        mw[(2 * c + 1) * kPartW + 4 + d] = S.acc[mb][2 * half + 1];
      }
    }
}

// CTA merge of NW warp states (SoftmaxState::merge, attention.hpp:36-44) and
// the segment's partial store; threads [0, nthreads) participate.  The
// per-(warp, head) scale factors are computed once (mf: NW + 1 rows of 8
// floats of shared scratch; row NW holds the merged maxima), then every
// element is a dot product over the warps.
template <int NW>
__device__ __forceinline__ void merge_store(const AttnKParams& P, const Seg& it,
                                            const float* merge, float* mf, int tid,
                                            int nthreads, int ws) {
  const float NEG_INF = -__int_as_float(0x7f800000);
  const int nh = min(8, P.G - 8 * it.hc);
  if (tid < nh) {
    float M = NEG_INF;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const float* mm = merge + w * ws + tid * kPartW;
      if (mm[1] > 0.f) M = fmaxf(M, mm[0]);
    }
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const float* mm = merge + w * ws + tid * kPartW;
      mf[w * 8 + tid] = mm[1] > 0.f ? ex2(mm[0] - M) : 0.f;
    }
    mf[NW * 8 + tid] = M;
  }
  __syncthreads();
  for (int idx = tid; idx < nh * kPartW; idx += nthreads) {
    const int h = idx / kPartW, j = idx % kPartW;
    float v = 0.f;
    if (j == 0) {
      v = mf[NW * 8 + h];
    } else if (j == 1 || j >= 4) {
#pragma unroll
      for (int w = 0; w < NW; ++w) v += merge[w * ws + h * kPartW + j] * mf[w * 8 + h];
    }
    const size_t row = (size_t)it.b * P.Hq + (size_t)it.kvh * P.G + 8 * it.hc + h;
    P.partials[(row * P.n_parts + it.part) * kPartW + j] = v;
    if (it.last && j == 1)  // slots no CTA writes for this stream: empty (l = 0)
      for (int k = it.part + 1; k < P.n_parts; ++k)
        P.partials[(row * P.n_parts + k) * kPartW + 1] = 0.f;
  }
}

// Fused K5 for one segment's (stream, head chunk): warp w rotates head
// 8 hc + w of q (Encoder::prepare, codec.hpp:282-292) into smem, then every
// lane gathers its mma B fragments (same layout as qprep_kernel).
template <int QF>
// pre: this warp's q row (head 8 hc + warp), already loaded (use_pre).
__device__ __forceinline__ void seg_qprep(uint32_t (&qf)[QF], const AttnKParams& P, int sh,
                                          float* qs, int warp, int nwarps, int lane,
                                          bool use_pre = false,
                                          float4 pre = make_float4(0.f, 0.f, 0.f, 0.f)) {
  const int hc = sh % P.HC, stream = sh / P.HC;
  const int b = stream / P.Hkv, kvh = stream % P.Hkv;
  const float log2e = 1.4426950408889634f;
  for (int w = warp; w < 8; w += nwarps) {
    float* qsw = qs + w * 129;
    float* qkw = qs + (8 + w) * 129;
    const int h = 8 * hc + w;
    if (h < P.G) {
      const float* q = P.q + ((size_t)b * P.Hq + (size_t)kvh * P.G + h) * 128;
      const float4 q4 = use_pre && w == warp ? pre : __ldg(reinterpret_cast<const float4*>(q) + lane);
      float y[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int e = 4 * lane + i;
        if ((word4(P.smask, e >> 5) >> (e & 31)) & 1u) y[i] = -y[i];
      }
      wht128_lane4(y, lane);
      const float s_attn = P.inv_sqrt_d * P.inv_sqrt_d * log2e;
#pragma unroll
      for (int i = 0; i < 4; ++i) qsw[4 * lane + i] = y[i] * s_attn;
      if (P.qjl) {
        float z[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int e = 4 * lane + i;
          const float v = y[i] * P.inv_sqrt_d;
          z[i] = ((word4(P.qmask, e >> 5) >> (e & 31)) & 1u) ? -v : v;
        }
        wht128_lane4(z, lane);
        const float s_sk = P.inv_sqrt_d * P.inv_sqrt_d * log2e * sqrtf(1.5707963267948966f / 128.f);
#pragma unroll
        for (int i = 0; i < 4; ++i) qkw[4 * lane + i] = z[i] * s_sk;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) qsw[4 * lane + i] = qkw[4 * lane + i] = 0.f;
    }
  }
  __syncthreads();
  const int g = lane >> 2, c = lane & 3;
#pragma unroll
  for (int sigma = 0; sigma < 18; ++sigma) {
    int d0, d1;
    k_slot_dims(c, sigma, d0, d1);
    qf[sigma] = pack_h2(d0 >= 0 ? qs[g * 129 + d0] : 0.f, d1 >= 0 ? qs[g * 129 + d1] : 0.f);
  }
  if (QF > 18)
#pragma unroll
    for (int sigma = 0; sigma < 16; ++sigma)
      qf[18 + sigma] = pack_h2(qs[(8 + g) * 129 + 32 * c + sigma],
                               qs[(8 + g) * 129 + 32 * c + sigma + 16]);
}

// Fused K4 for one row: merge its n partials in order (SoftmaxState::merge,
// attention.hpp:36-44), acc / l, inverse V rotation; one warp.
// partial: write the merged state (M, L, 0, 0, acc[128]) (the format of
// combine_kernel's finalize = 0, for a later cross-rank merge) instead.
__device__ __forceinline__ void combine_row(const float* base, int n, float* out,
                                            const uint32_t (&vmask)[4], float inv_sqrt_d,
                                            int lane, bool partial = false,
                                            size_t stride = kPartW) {
  const float NEG_INF = -__int_as_float(0x7f800000);
  float M = NEG_INF;
  float L = 0.f, y[4] = {0.f, 0.f, 0.f, 0.f};
  // the parts were just written by other CTAs (L2).  Up to 8 parts (the
  // usual count): ONE batch of loads, the maximum taken from it, then the
  // same in-order sums — one L2 round trip on the launch's critical path
  // instead of three
  constexpr int NB1 = 8;
  if (n >= 1 && n <= NB1) {
    float2 ml[NB1];
    float4 a4[NB1];
#pragma unroll
    for (int j = 0; j < NB1; ++j) {  // past the end: re-read the last part, skipped below
      const size_t i = (size_t)min(j, n - 1);
      ml[j] = *reinterpret_cast<const float2*>(base + i * stride);
      a4[j] = *reinterpret_cast<const float4*>(base + i * stride + 4 + 4 * lane);
    }
#pragma unroll
    for (int j = 0; j < NB1; ++j)
      if (j < n && ml[j].y > 0.f) M = fmaxf(M, ml[j].x);
#pragma unroll
    for (int j = 0; j < NB1; ++j)
      if (j < n && ml[j].y > 0.f) {  // in part order
        const float f = ex2(ml[j].x - M);
        L += ml[j].y * f;
        y[0] += a4[j].x * f; y[1] += a4[j].y * f; y[2] += a4[j].z * f; y[3] += a4[j].w * f;
      }
    n = 0;  // done: skip the general loop below
  } else {
    for (int i = lane; i < n; i += 32) {
      const float2 ml = *reinterpret_cast<const float2*>(base + (size_t)i * stride);
      if (ml.y > 0.f) M = fmaxf(M, ml.x);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) M = fmaxf(M, __shfl_xor_sync(kFull, M, o));
  }
  // more parts: batches of them requested before they are consumed, instead
  // of one dependent round trip per part
  constexpr int NB = 4;
  for (int i0 = 0; i0 < n; i0 += NB) {
    float2 ml[NB];
    float4 a4[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) {  // past the end: re-read the last part, skipped below
      const size_t i = (size_t)min(i0 + j, n - 1);
      ml[j] = *reinterpret_cast<const float2*>(base + i * stride);
      a4[j] = *reinterpret_cast<const float4*>(base + i * stride + 4 + 4 * lane);
    }
#pragma unroll
    for (int j = 0; j < NB; ++j)
      if (i0 + j < n && ml[j].y > 0.f) {  // in part order, as before
        const float f = ex2(ml[j].x - M);
        L += ml[j].y * f;
        y[0] += a4[j].x * f; y[1] += a4[j].y * f; y[2] += a4[j].z * f; y[3] += a4[j].w * f;
      }
  }
  if (partial) {
    if (lane == 0) *reinterpret_cast<float4*>(out) = make_float4(M, L, 0.f, 0.f);
    *reinterpret_cast<float4*>(out + 4 + 4 * lane) = make_float4(y[0], y[1], y[2], y[3]);
    return;
  }
  const float inv = L > 0.f ? 1.f / L : 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) y[i] *= inv;
  wht128_lane4(y, lane);
  float r[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int e = 4 * lane + i;
    const float v = y[i] * inv_sqrt_d;
    r[i] = ((word4(vmask, e >> 5) >> (e & 31)) & 1u) ? -v : v;
  }
  *reinterpret_cast<float4*>(out + 4 * lane) = make_float4(r[0], r[1], r[2], r[3]);
}

// Fused P2P sequence sharding, run by the CTA that finalises stream chunk
// `it` on this rank (all its threads):
//  (1) this rank's merged rows of the chunk -> shared staging;
//  (2) stored into slot `rank` of EVERY rank's exchange buffer — peer memory
//      over NVLink, mapped into this process (CUDA IPC);
//  (3) a system-scope release fence, then flag [rank][chunk] = epoch in
//      each buffer;
//  (4) an acquire-spin on this buffer's flags [r][chunk] for every rank r;
//  (5) the ranks' rows merged in rank order — attention_decode(...,
//      n_splits = nranks), attention.hpp:60-69 — and finalised into out.
// One launch per step, no collective library; every rank ends with the same
// rows.  A rank that never arrives traps after 20 s instead of hanging.
// Exchange buffer layout: float [2][nranks][B*Hq][kPartW] (the half is the
// epoch's parity: a rank can start the next call while a slower one still
// reads this call's rows), then u32 flags [nranks][n_sh] (zeroed once; epochs
// increase per call, and a flag that has already moved on counts as arrived).
// The fields p2p_exchange reads.  Passing the kernel parameters themselves
// by reference to this out-of-line function makes every thread copy the
// whole parameter block to local memory at kernel entry (~26 MB of DRAM
// writes per C3 launch); the QJL kernels pass this copied subset instead
// (C4 -1 %), while for the others every way of avoiding the copy measured
// 2-3 % slower tile-loop code, so they keep it.
struct P2PView {
  float* partials;
  float* out;
  uint8_t* p2p_xbuf[8];
  uint32_t vmask[4];
  float inv_sqrt_d;
  int G, B, Hq, n_parts, n_sh, p2p_nranks, p2p_rank;
  uint32_t p2p_epoch;
};

template <class PV>
__device__ __noinline__ void p2p_exchange(const PV& P, const Seg& it, int nparts,
                                          float* stage, int tid, int warp, int lane, int nwarps) {
  const int nh = min(8, P.G - 8 * it.hc);
  const size_t rows_total = (size_t)P.B * P.Hq;
  const size_t row0 = (size_t)it.b * P.Hq + (size_t)it.kvh * P.G + 8 * it.hc;
  for (int w = warp; w < nh; w += nwarps)
    combine_row(P.partials + (row0 + w) * P.n_parts * kPartW, nparts, stage + w * kPartW,
                P.vmask, P.inv_sqrt_d, lane, true);
  __syncthreads();
  const size_t half = (size_t)(P.p2p_epoch & 1u) * P.p2p_nranks * rows_total * kPartW;
  for (int r = 0; r < P.p2p_nranks; ++r) {
    float* dst = reinterpret_cast<float*>(P.p2p_xbuf[r]) + half +
                 ((size_t)P.p2p_rank * rows_total + row0) * kPartW;
    for (int i = tid; i < nh * kPartW / 4; i += blockDim.x)
      reinterpret_cast<float4*>(dst)[i] = reinterpret_cast<const float4*>(stage)[i];
  }
  __syncthreads();
  const size_t flag_off = 2 * (size_t)P.p2p_nranks * rows_total * kPartW * sizeof(float);
  if (tid == 0) {
    // release at system scope, once (the barrier above orders the CTA's row
    // stores before it; a release fence is cumulative over them), then
    // relaxed flag stores
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    for (int r = 0; r < P.p2p_nranks; ++r) {
      uint32_t* fl = reinterpret_cast<uint32_t*>(P.p2p_xbuf[r] + flag_off) +
                     (size_t)P.p2p_rank * P.n_sh + it.sh;
      asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(fl), "r"(P.p2p_epoch) : "memory");
    }
    const uint32_t* mine = reinterpret_cast<const uint32_t*>(P.p2p_xbuf[P.p2p_rank] + flag_off);
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int r = 0; r < P.p2p_nranks; ++r) {
      for (;;) {
        uint32_t v;
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];"
                     : "=r"(v)
                     : "l"(mine + (size_t)r * P.n_sh + it.sh)
                     : "memory");
        if ((int32_t)(v - P.p2p_epoch) >= 0) break;
        uint64_t now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        if (now - t0 > 20000000000ull) __trap();
      }
    }
  }
  __syncthreads();
  const float* xl = reinterpret_cast<const float*>(P.p2p_xbuf[P.p2p_rank]) + half;
  for (int w = warp; w < nh; w += nwarps)
    combine_row(xl + (row0 + w) * kPartW, P.p2p_nranks, P.out + (row0 + w) * 128, P.vmask,
                P.inv_sqrt_d, lane, false, rows_total * kPartW);
}

// Variant A: each warp streams its tiles from HBM straight into registers,
// prefetching one tile ahead (ping-pong register images).
// RING = 0: each warp prefetches the next tile into registers (ping-pong
// register images).  RING > 0: each warp owns a RING-stage ring of tiles in
// shared memory filled by 1-D TMA (cp.async.bulk) RING tiles ahead; a tile's
// words move to registers with LDS when it is processed (one register image,
// so more warps fit per SM).
template <int W, bool QJL, int kAttnWarps, int RING = 0>
__global__ void __launch_bounds__(kAttnWarps * 32, 1) attn_partials_kernel(const AttnKParams P) {
  using C = Cfg<W, QJL>;
  constexpr int WREG = C::wreg(RING);   // bytes per warp region
  constexpr int WS = WREG / 4;          // ... in floats (merge slot stride)
  uint8_t* smem = g_attn_smem;
  uint2* tab = reinterpret_cast<uint2*>(smem);
  float* merge = reinterpret_cast<float*>(smem + C::TAB_BYTES);
  uint8_t* ring = smem + C::TAB_BYTES;  // warp w: ring + w * WREG (aliases its merge slot)
  float* qs = reinterpret_cast<float*>(smem + C::TAB_BYTES + kAttnWarps * WREG);
  __shared__ __align__(8) uint64_t s_ring_bar[kAttnWarps][RING > 0 ? RING : 1];
  uint32_t ring_phase = 0;  // bit s: parity of the next completion of stage s
  __shared__ int s_last;
  __shared__ float s_mf[(kAttnWarps + 1) * 8];  // merge_store scale factors
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, c = lane & 3;

  // Programmatic dependent launch: let the next launch in the stream start
  // its CTAs (they can only become resident as ours exit), and stage the
  // dequant table — the codec's constant, written by no earlier kernel — before
  // waiting for the previous grid; everything after griddepcontrol.wait
  // (q, seq_lens, the caches, the workspace counters and partials) sees its
  // writes.  Without the launch attribute both instructions are no-ops.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  __shared__ __align__(8) uint64_t s_tab_bar;
  uint32_t tbase;
  constexpr uint32_t kRepMask = (uint32_t)table_rep(W) - 1u;
  if constexpr (W <= 8) {
    // table at shared address 0x10000: 32 replicas x 8 B per entry
    const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    if (base > 0x10000u) __trap();
    stage_table_issue(smem + (0x10000u - base), P.tab, (1u << W) * 32u * 8u, &s_tab_bar, tid);
    tbase = 0x10000u;
  } else {
    stage_table_issue(tab, P.tab, (1u << W) * (uint32_t)table_rep(W) * 8u, &s_tab_bar, tid);
    tbase = static_cast<uint32_t>(__cvta_generic_to_shared(tab));
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");

  // the first segment's q row of this warp's head, requested while the table
  // arrives so its latency is hidden behind it
  int sh_pre = -1;
  float4 q_pre = make_float4(0.f, 0.f, 0.f, 0.f);
  // (not with QJL: the extra live float4 makes that variant spill in its tile loop)
  if (!QJL && P.fuse && P.streamk && kAttnWarps == 8) {
    const size_t V = P.tps + P.sko, U = (size_t)P.n_sh * V, G = gridDim.x;
    const size_t u0 = sk_bound(blockIdx.x, U, G), u1 = sk_bound(blockIdx.x + 1, U, G);
    for (size_t sh = u0 / V; sh * V < u1; ++sh)
      if (max(u0, sh * V + P.sko) < min(u1, sh * V + V)) {
        sh_pre = (int)sh;
        break;
      }
    if (sh_pre >= 0) {
      const int hc = sh_pre % P.HC, stream = sh_pre / P.HC, h = 8 * hc + warp;
      if (h < P.G)
        q_pre = __ldg(reinterpret_cast<const float4*>(
                          P.q + ((size_t)(stream / P.Hkv) * P.Hq + (size_t)(stream % P.Hkv) * P.G + h) * 128) +
                      lane);
    }
  }
  if constexpr (RING > 0) {
    if (lane == 0)
      for (int st = 0; st < RING; ++st) mbar_init(&s_ring_bar[warp][st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();  // the table's barrier is initialised before anyone waits on it
  mbar_wait(&s_tab_bar, 0);

  // per-lane table offset for the tiles of a ping-pong buffer whose first
  // tile is t: base + 8 * replica, replica = (lane + t) mod REP (a
  // permutation of the replicas within each half-warp: conflict-free).  The
  // warps of a CTA take tiles round-robin, so over a stream every token
  // position meets every residue of t and reads a code through all replicas.
  auto toff_of = [&](size_t t) -> uint32_t {
    return tbase + ((((uint32_t)lane + (uint32_t)t) & kRepMask) << 3);
  };

  auto run = [&](const Seg& it, int nparts) {
    TileRegs<W, QJL> ra, rb;
    (void)ra;
    (void)rb;
    size_t tile = it.tlo + warp;
    uint32_t qf[C::QF];
    if (P.fuse) {
      seg_qprep(qf, P, it.sh, qs, warp, kAttnWarps, lane, it.sh == sh_pre, q_pre);
      sh_pre = -1;
    } else {
      load_qfrag(qf, P, it.sh, lane);
    }
    WarpState S;
    if constexpr (RING > 0) {
      uint8_t* wr = ring + warp * WREG;
      // the first RING tiles of this warp, issued after the query prep (the
      // proxy fence orders the region's earlier generic stores — the merge
      // slot it aliases — before the TMA writes)
      if (lane == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (lane == 0)
#pragma unroll
        for (int st = 0; st < RING; ++st) {
          const size_t t = tile + (size_t)st * kAttnWarps;
          if (t < it.thi) ring_issue<W, QJL>(wr + st * C::STAGE, &s_ring_bar[warp][st], P, it.stream, t);
        }
      init_state(S);
      if constexpr (RING == 2 && !QJL) {
        // two tiles per iteration: the stage index is a constant in each
        // half (C5 -1.5 %, C3 -0.3 %; with QJL keys it spills: C4 +1.2 %)
        auto one = [&](auto st_tag) -> bool {
          constexpr int st = decltype(st_tag)::value;
          if (tile >= it.thi) return false;
          mbar_wait(&s_ring_bar[warp][st], (ring_phase >> st) & 1u);
          ring_phase ^= 1u << st;
          TileRegs<W, QJL> r;
          load_tile_smem<W, QJL>(r, wr + st * C::STAGE, wr + st * C::STAGE + C::KTILE, g, c, lane,
                                 lane);
          __syncwarp();
          const size_t tn = tile + (size_t)RING * kAttnWarps;
          if (lane == 0 && tn < it.thi)
            ring_issue<W, QJL>(wr + st * C::STAGE, &s_ring_bar[warp][st], P, it.stream, tn);
          process_tile<W, QJL>(S, r, qf, toff_of(tile), (int)(tile * kTileTok), it.lo, it.hi, g, c);
          tile += kAttnWarps;
          return true;
        };
        while (one(std::integral_constant<int, 0>{}) && one(std::integral_constant<int, 1>{})) {
        }
      } else {
      int st = 0;
      while (tile < it.thi) {
        mbar_wait(&s_ring_bar[warp][st], (ring_phase >> st) & 1u);
        ring_phase ^= 1u << st;
        TileRegs<W, QJL> r;
        load_tile_smem<W, QJL>(r, wr + st * C::STAGE, wr + st * C::STAGE + C::KTILE, g, c, lane,
                               lane);
        __syncwarp();  // every lane has its words: the stage can be refilled
        const size_t tn = tile + (size_t)RING * kAttnWarps;
        if (lane == 0 && tn < it.thi)
          ring_issue<W, QJL>(wr + st * C::STAGE, &s_ring_bar[warp][st], P, it.stream, tn);
        process_tile<W, QJL>(S, r, qf, toff_of(tile), (int)(tile * kTileTok), it.lo, it.hi, g, c);
        tile += kAttnWarps;
        st = st + 1 == RING ? 0 : st + 1;
      }
      }
      __syncwarp();
    } else {
    // first tile requested after the query prep: issued before it, its 31
    // loads per lane (on every SM at once) held up the prep (C3 -0.7 us)
    if (tile < it.thi) load_tile<W, QJL>(ra, P, it.stream, tile, g, c, lane, lane);
    // the two ping-pong buffers' table offsets (see toff_of)
    const uint32_t toff_a = toff_of(tile), toff_b = toff_of(tile + kAttnWarps);
    init_state(S);
    while (tile < it.thi) {
      size_t tn = tile + kAttnWarps;
      if (tn < it.thi) load_tile<W, QJL>(rb, P, it.stream, tn, g, c, lane, lane);
      process_tile<W, QJL>(S, ra, qf, toff_a, (int)(tile * kTileTok), it.lo, it.hi, g, c);
      tile = tn;
      if (tile >= it.thi) break;
      tn = tile + kAttnWarps;
      if (tn < it.thi) load_tile<W, QJL>(ra, P, it.stream, tn, g, c, lane, lane);
      process_tile<W, QJL>(S, rb, qf, toff_b, (int)(tile * kTileTok), it.lo, it.hi, g, c);
      tile = tn;
    }
    }
    warp_state_out(S, merge + warp * WS, g, c);
    __syncthreads();
    merge_store<kAttnWarps>(P, it, merge, s_mf, tid, blockDim.x, WS);
    if (P.fuse) {
      // the CTA that lands a stream's last partial finalises its rows.  The
      // barrier orders the CTA's partial stores before thread 0's gpu-scope
      // acq_rel arrival (release cumulativity); the CTA that arrives last
      // acquires every other CTA's partials through the same counter, and
      // the second barrier passes that on to its threads.
      __syncthreads();
      if (tid == 0) {
        uint32_t old;
        asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;"
                     : "=r"(old)
                     : "l"(P.counters + it.sh)
                     : "memory");
        s_last = old + 1 == (uint32_t)nparts;
        if (s_last) P.counters[it.sh] = 0u;
      }
      __syncthreads();
      if (s_last && P.p2p_nranks > 0) {
        if constexpr (QJL) {
          P2PView V;
          V.partials = P.partials;
          V.out = P.out;
#pragma unroll
          for (int r = 0; r < 8; ++r) V.p2p_xbuf[r] = P.p2p_xbuf[r];
#pragma unroll
          for (int i = 0; i < 4; ++i) V.vmask[i] = P.vmask[i];
          V.inv_sqrt_d = P.inv_sqrt_d;
          V.G = P.G;
          V.B = P.B;
          V.Hq = P.Hq;
          V.n_parts = P.n_parts;
          V.n_sh = P.n_sh;
          V.p2p_nranks = P.p2p_nranks;
          V.p2p_rank = P.p2p_rank;
          V.p2p_epoch = P.p2p_epoch;
          p2p_exchange(V, it, nparts, qs, tid, warp, lane, kAttnWarps);
        } else {
          p2p_exchange(P, it, nparts, qs, tid, warp, lane, kAttnWarps);
        }
      } else if (s_last) {
        for (int w = warp; w < 8; w += kAttnWarps) {
          if (8 * it.hc + w >= P.G) continue;
          const size_t row = (size_t)it.b * P.Hq + (size_t)it.kvh * P.G + 8 * it.hc + w;
          combine_row(P.partials + row * P.n_parts * kPartW, nparts,
                      P.out + row * (P.out_partial ? kPartW : 128), P.vmask, P.inv_sqrt_d, lane,
                      P.out_partial);
        }
      }
    }
    __syncthreads();
  };

  if (!P.streamk) {
    for (int item = blockIdx.x; item < P.n_items; item += gridDim.x)
      run(item_seg(P, item), P.splits);
  } else {
    // stream-K over virtual units: each stream is sko units of segment
    // overhead (q prep, pipeline restart, merge) followed by its tps tiles,
    // so a CTA that starts a second stream gets correspondingly fewer tiles
    const size_t V = P.tps + P.sko, U = (size_t)P.n_sh * V, G = gridDim.x;
    const size_t u0 = sk_bound(blockIdx.x, U, G), u1 = sk_bound(blockIdx.x + 1, U, G);
    for (size_t sh = u0 / V; sh * V < u1; ++sh) {
      const size_t t0 = sh * V + P.sko, s1 = sh * V + V;  // the stream's tile units
      const size_t a = max(u0, t0), z = min(u1, s1);
      if (a >= z) continue;  // only overhead units of this stream
      const int first = sk_cta(t0, U, G), part = (int)blockIdx.x - first;
      run(make_seg(P, (int)sh, P.tb0 + (a - t0), P.tb0 + (z - t0), part, z == s1),
          sk_cta(s1 - 1, U, G) - first + 1);
    }
  }
}

// ---------------------------------------------------------------------------
// K5: query prep (Encoder::prepare, codec.hpp:282-292) -> mma B fragments.
// q_rot = R_k q scaled by log2(e)/sqrt(d); QJL: q_sketch = R' q_rot with the
// estimator constant sqrt(pi/(2d)) (qjl.hpp:47) folded in.
struct QPrepParams {
  const float* q;
  uint32_t* qfrag;
  int Hq, Hkv, G, HC, QF;
  uint32_t smask[4], qmask[4];
  float inv_sqrt_d;
  int qjl;
};

__global__ void qprep_kernel(QPrepParams P) {
  __shared__ float qs[8][129];
  __shared__ float qk[8][129];
  const int sh = blockIdx.x, hc = sh % P.HC, stream = sh / P.HC;
  const int b = stream / P.Hkv, kvh = stream % P.Hkv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = 8 * hc + warp;
  const float log2e = 1.4426950408889634f;
  if (h < P.G) {
    const float* q = P.q + ((size_t)b * P.Hq + (size_t)kvh * P.G + h) * 128;
    float y[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = 4 * lane + i;
      const float v = q[e];
      y[i] = ((word4(P.smask, e >> 5) >> (e & 31)) & 1u) ? -v : v;
    }
    wht128_lane4(y, lane);
    const float s_attn = P.inv_sqrt_d * P.inv_sqrt_d * log2e;  // rotation norm x 1/sqrt(d) x log2e
#pragma unroll
    for (int i = 0; i < 4; ++i) qs[warp][4 * lane + i] = y[i] * s_attn;
    if (P.qjl) {
      float z[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int e = 4 * lane + i;
        const float v = y[i] * P.inv_sqrt_d;  // q_rot
        z[i] = ((word4(P.qmask, e >> 5) >> (e & 31)) & 1u) ? -v : v;
      }
      wht128_lane4(z, lane);
      const float s_sk = P.inv_sqrt_d * P.inv_sqrt_d * log2e * sqrtf(1.5707963267948966f / 128.f);
#pragma unroll
      for (int i = 0; i < 4; ++i) qk[warp][4 * lane + i] = z[i] * s_sk;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) qs[warp][4 * lane + i] = qk[warp][4 * lane + i] = 0.f;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int g = lane >> 2, c = lane & 3;
    uint32_t* dst = P.qfrag + ((size_t)sh * 32 + lane) * P.QF;
    for (int sigma = 0; sigma < 18; ++sigma) {
      int d0, d1;
      k_slot_dims(c, sigma, d0, d1);
      dst[sigma] = pack_h2(d0 >= 0 ? qs[g][d0] : 0.f, d1 >= 0 ? qs[g][d1] : 0.f);
    }
    if (P.qjl)
      for (int sigma = 0; sigma < 16; ++sigma)
        dst[18 + sigma] = pack_h2(qk[g][32 * c + sigma], qk[g][32 * c + sigma + 16]);
  }
}

// ---------------------------------------------------------------------------
// K4: merge partials in order, then acc/l and the inverse V rotation.
struct CombineParams {
  const float* parts;
  float* out;
  int rows, n_parts, finalize;
  size_t row_stride, part_stride;
  uint32_t smask[4];
  float inv_sqrt_d;
};

__global__ void combine_kernel(CombineParams P) {
  // one warp per row: lanes fetch (m, l) of the parts in parallel, reduce,
  // then every lane streams its 4 dims of each part with independent loads.
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= P.rows) return;
  const float NEG_INF = -__int_as_float(0x7f800000);
  const float* base = P.parts + (size_t)row * P.row_stride;
  float M = NEG_INF;
  for (int i = lane; i < P.n_parts; i += 32) {
    const float2 ml = *reinterpret_cast<const float2*>(base + (size_t)i * P.part_stride);
    if (ml.y > 0.f) M = fmaxf(M, ml.x);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) M = fmaxf(M, __shfl_xor_sync(kFull, M, o));
  float L = 0.f, y[4] = {0.f, 0.f, 0.f, 0.f};
  for (int i0 = 0; i0 < P.n_parts; i0 += 32) {
    // scale factor of part i0 + lane, broadcast below
    float f = 0.f, l = 0.f;
    if (i0 + lane < P.n_parts) {
      const float2 ml =
          *reinterpret_cast<const float2*>(base + (size_t)(i0 + lane) * P.part_stride);
      if (ml.y > 0.f) {
        f = ex2(ml.x - M);
        l = ml.y * f;
      }
    }
    float ls = l;
#pragma unroll
    for (int o = 16; o; o >>= 1) ls += __shfl_xor_sync(kFull, ls, o);
    L += ls;
    const int n = min(32, P.n_parts - i0);
#pragma unroll 8
    for (int j = 0; j < n; ++j) {
      const float fj = __shfl_sync(kFull, f, j);
      if (fj != 0.f) {
        const float4 a4 = *reinterpret_cast<const float4*>(
            base + (size_t)(i0 + j) * P.part_stride + 4 + 4 * lane);
        y[0] += a4.x * fj; y[1] += a4.y * fj; y[2] += a4.z * fj; y[3] += a4.w * fj;
      }
    }
  }
  if (!P.finalize) {
    float* o = P.out + (size_t)row * kPartW;
    if (lane == 0) *reinterpret_cast<float4*>(o) = make_float4(M, L, 0.f, 0.f);
    *reinterpret_cast<float4*>(o + 4 + 4 * lane) = make_float4(y[0], y[1], y[2], y[3]);
    return;
  }
  const float inv = L > 0.f ? 1.f / L : 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) y[i] *= inv;
  wht128_lane4(y, lane);
  float r[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int e = 4 * lane + i;
    const float v = y[i] * P.inv_sqrt_d;
    r[i] = ((word4(P.smask, e >> 5) >> (e & 31)) & 1u) ? -v : v;
  }
  *reinterpret_cast<float4*>(P.out + (size_t)row * 128 + 4 * lane) = make_float4(r[0], r[1], r[2], r[3]);
}

// ---------------------------------------------------------------------------
// records -> attention tiles (oq_cache_pack).  One warp per (stream, tile).
__device__ __forceinline__ uint32_t rec_joint(const OqCodecParams& p, const uint8_t* r, int t) {
  if (t >= kNT) return 0u;
  const uint32_t a = read_bits_safe(r + 4, 2 * t * p.b_dir, p.b_dir);
  const uint32_t b = read_bits_safe(r + 4, (2 * t + 1) * p.b_dir, p.b_dir);
  const uint32_t n = read_bits_safe(r + 4 + p.dir_bytes, t * p.b_nrm, p.b_nrm);
  return a | (b << p.b_dir) | (n << (2 * p.b_dir));
}

// The same joint code from a record held as 32-bit words (bits LSB-first):
// the direction pair field is ixi | ieta << b_dir already.
__device__ __forceinline__ uint32_t rec_field_w(const uint32_t* w, int pos, int bits) {
  const int i = pos >> 5, sh = pos & 31;
  const uint32_t v = sh + bits > 32 ? __funnelshift_r(w[i], w[i + 1], sh) : w[i] >> sh;
  return v & ((1u << bits) - 1u);
}
__device__ __forceinline__ uint32_t rec_joint_w(const OqCodecParams& p, const uint32_t* w, int t) {
  if (t >= kNT) return 0u;
  const uint32_t d = rec_field_w(w, 32 + 2 * p.b_dir * t, 2 * p.b_dir);
  const uint32_t n = rec_field_w(w, 32 + 8 * (int)p.dir_bytes + p.b_nrm * t, p.b_nrm);
  return d | (n << (2 * p.b_dir));
}

__global__ void pack_tiles_kernel(OqCodecParams p, int role, const uint8_t* __restrict__ recs,
                                  size_t n_streams, size_t n_tok, size_t rec_stride,
                                  uint8_t* __restrict__ tiles, size_t tiles_cap) {
  const int W = 2 * p.b_dir + p.b_nrm;
  const int lane = threadIdx.x & 31;
  const size_t wid = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const size_t ntiles = (n_tok + 31) / 32;
  if (wid >= n_streams * ntiles) return;
  const size_t s = wid / ntiles, tile = wid % ntiles;
  const int tb = role == 0 ? ktile_bytes(W, p.qjl) : vtile_bytes(W);
  uint8_t* out = tiles + (s * tiles_cap + tile) * (size_t)tb;
  const int g = lane >> 2, c = lane & 3;
  auto rec = [&](int tt) -> const uint8_t* {
    const size_t tok = tile * 32 + tt;
    return tok < n_tok ? recs + (s * rec_stride + tok) * p.rec_bytes : nullptr;
  };
  auto gamma_of = [&](const uint8_t* r) -> float {
    if (!r) return 0.f;
    const uint32_t b = (uint32_t)r[0] | ((uint32_t)r[1] << 8) | ((uint32_t)r[2] << 16) |
                       ((uint32_t)r[3] << 24);
    return __uint_as_float(b);
  };
  if (lane < 8)
    for (int k = 0; k < 4; ++k)
      reinterpret_cast<float*>(out)[lane * 4 + k] = gamma_of(rec(k_token(lane, k)));
  uint32_t* codes = reinterpret_cast<uint32_t*>(out + 128);
  // build this lane's code run (word-interleaved, see the layout note)
  uint32_t acc = 0;
  int nbits = 0, wi = 0;
  const int nslots = role == 0 ? (c < 3 ? 11 : 10) * 4 : (g < 7 ? 6 : 1) * 8;
  auto put = [&](int i, uint32_t w) {
    codes[role == 0 ? k_word_off(W, lane, i) : v_word_off(W, lane, i)] = w;
  };
  for (int slot = 0; slot < nslots; ++slot) {
    uint32_t code;
    if (role == 0) {
      const int u = slot >> 2, k = slot & 3;
      const uint8_t* r = rec(k_token(g, k));
      code = r ? rec_joint(p, r, 11 * c + u) : 0u;
    } else {
      const int u = slot >> 3, k = slot & 7;
      const uint8_t* r = rec(v_token(c, k));
      code = r ? rec_joint(p, r, 6 * g + u) : 0u;
    }
    // append FW bits LSB-first
    const int FWb = fw(W);
    acc |= code << nbits;
    nbits += FWb;
    if (nbits >= 32) {
      put(wi++, acc);
      nbits -= 32;
      acc = nbits ? code >> (FWb - nbits) : 0u;
    }
  }
  if (nbits) put(wi++, acc);
  if (role == 0 && p.qjl) {
    uint8_t* qa = out + 128 + 4 * kcode_words(W);
    const int sign_off = 4 + p.dir_bytes + p.nrm_bytes + 2;
    if (lane < 8)
      for (int k = 0; k < 4; ++k) {
        const uint8_t* r = rec(k_token(lane, k));
        const uint16_t grb = r ? (uint16_t)(r[sign_off - 2] | (r[sign_off - 1] << 8)) : 0;
        reinterpret_cast<uint16_t*>(qa)[lane * 4 + k] = grb;
      }
    uint32_t* sg = reinterpret_cast<uint32_t*>(qa + 64) + (4 * g + c) * 4;
    for (int k = 0; k < 4; ++k) {
      const uint8_t* r = rec(k_token(g, k));
      uint32_t w = 0;
      if (r)
        for (int i = 0; i < 4; ++i) w |= (uint32_t)r[sign_off + 4 * c + i] << (8 * i);
      sg[k] = w;
    }
  }
}

// ---------------------------------------------------------------------------
// Decode-step append (oq_cache_append): write ONE token per stream — the
// record rec[s] — into token slot pos of the stream's tile, leaving the other
// 31 tokens of the tile untouched (read-modify-write of the W-bit fields in
// the lane runs).  One warp per stream; only the lanes owning that token's
// slots write.  Same bit layout as pack_tiles_kernel.
// Write the record in rec (32 shared words, already complete) into token
// slot pos of stream s's tile.  run: 32 x 21 words of warp-private shared
// scratch.  Called by the whole warp; only the lanes owning the token's
// slots touch the code runs.
// Geometry of the append of token pos: the tile, and which lanes write.
struct AppendGeo {
  uint8_t* out;
  int tt, nw;
  bool writer;
};
__device__ __forceinline__ bool append_geo(const OqCodecParams& p, int role, size_t s, int64_t pos,
                                           uint8_t* tiles, size_t tiles_cap, int lane,
                                           AppendGeo& a) {
  const int W = 2 * p.b_dir + p.b_nrm;
  if (pos < 0 || (size_t)pos >= tiles_cap * 32) return false;
  const int tb = role == 0 ? ktile_bytes(W, p.qjl) : vtile_bytes(W);
  a.out = tiles + (s * tiles_cap + (size_t)pos / 32) * (size_t)tb;
  a.tt = (int)(pos % 32);
  const int g = lane >> 2, c = lane & 3;
  a.writer = role == 0 ? (g == (a.tt & 7)) : (c == ((a.tt & 7) >> 1));
  a.nw = role == 0 ? (c < 3 ? kw_full(W) : kw_3(W)) : (g < 7 ? vw_full(W) : vw_7(W));
  return true;
}

// Start the asynchronous copy (cp.async, no register staging) of the writing
// lanes' run words into run_w, so that it overlaps the key's encoding; the
// caller waits (cp.async.wait_all) before append_record(staged = true).
__device__ __forceinline__ void append_stage_runs(const OqCodecParams& p, int role, size_t s,
                                                  int64_t pos, uint8_t* tiles, size_t tiles_cap,
                                                  uint32_t (*run_w)[21], int lane) {
  AppendGeo a;
  if (!append_geo(p, role, s, pos, tiles, tiles_cap, lane, a) || !a.writer) return;
  const int W = 2 * p.b_dir + p.b_nrm;
  const uint32_t* codes = reinterpret_cast<const uint32_t*>(a.out + 128);
  const uint32_t dst = (uint32_t)__cvta_generic_to_shared(run_w[lane]);
  for (int i = 0; i < a.nw; ++i) {
    const uint32_t* src = codes + (role == 0 ? k_word_off(W, lane, i) : v_word_off(W, lane, i));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst + 4 * i), "l"(src));
  }
}

__device__ __forceinline__ void append_record(const OqCodecParams& p, int role, const uint32_t* rec,
                                              uint32_t (*run_w)[21], size_t s, int64_t pos,
                                              uint8_t* __restrict__ tiles, size_t tiles_cap,
                                              int lane, bool staged = false) {
  const int W = 2 * p.b_dir + p.b_nrm;
  if (pos < 0 || (size_t)pos >= tiles_cap * 32) return;
  const size_t tile = (size_t)pos / 32;
  const int tt = (int)(pos % 32);
  const int tb = role == 0 ? ktile_bytes(W, p.qjl) : vtile_bytes(W);
  uint8_t* out = tiles + (s * tiles_cap + tile) * (size_t)tb;
  const uint8_t* r = reinterpret_cast<const uint8_t*>(rec);
  const int g = lane >> 2, c = lane & 3;
  const int tg = tt & 7, tk = tt >> 3;  // token = g + 8k in the K map and the gamma slots
  if (lane == 0) reinterpret_cast<float*>(out)[tg * 4 + tk] = __uint_as_float(rec[0]);
  uint32_t* codes = reinterpret_cast<uint32_t*>(out + 128);
  const bool writer = role == 0 ? (g == tg) : (c == ((tt & 7) >> 1));
  if (!writer) return;
  const int nw = role == 0 ? (c < 3 ? kw_full(W) : kw_3(W)) : (g < 7 ? vw_full(W) : vw_7(W));
  uint32_t* run = run_w[lane];
  auto woff = [&](int i) { return role == 0 ? k_word_off(W, lane, i) : v_word_off(W, lane, i); };
  if (!staged) {
#pragma unroll 4
    for (int i = 0; i < nw; ++i) run[i] = codes[woff(i)];
  }
  const int FW = fw(W);
  const uint32_t m = (1u << FW) - 1u;
  auto put = [&](int slot, uint32_t code) {
    const int bpos = slot * FW, i = bpos >> 5, sh = bpos & 31;
    run[i] = (run[i] & ~(m << sh)) | (code << sh);
    if (sh + FW > 32) {
      const int hi = sh + FW - 32;
      run[i + 1] = (run[i + 1] & ~((1u << hi) - 1u)) | (code >> (FW - hi));
    }
  };
  if (role == 0) {
    const int nu = c < 3 ? 11 : 10;
    for (int u = 0; u < nu; ++u) put(u * 4 + tk, rec_joint_w(p, rec, 11 * c + u));
    if (p.qjl) {
      uint8_t* qa = out + 128 + 4 * kcode_words(W);
      const int sign_off = 4 + p.dir_bytes + p.nrm_bytes + 2;
      if (c == 0)
        reinterpret_cast<uint16_t*>(qa)[tg * 4 + tk] =
            (uint16_t)(r[sign_off - 2] | (r[sign_off - 1] << 8));
      uint32_t w = 0;
      for (int i = 0; i < 4; ++i) w |= (uint32_t)r[sign_off + 4 * c + i] << (8 * i);
      reinterpret_cast<uint32_t*>(qa + 64)[(4 * g + c) * 4 + tk] = w;
    }
  } else {
    // V map: token v_token(c, k) = 16 (k >> 2) + 2c + (k & 1) + 8 ((k >> 1) & 1)
    const int k = (tt >> 4) * 4 + ((tt >> 3) & 1) * 2 + (tt & 1);
    const int nu = g < 7 ? 6 : 1;
    for (int u = 0; u < nu; ++u) put(u * 8 + k, rec_joint_w(p, rec, 6 * g + u));
  }
#pragma unroll 4
  for (int i = 0; i < nw; ++i) codes[woff(i)] = run[i];
}

// Decode-step append (oq_cache_append): write ONE token per stream — the
// record rec[s] — into token slot pos of the stream's tile, leaving the other
// 31 tokens of the tile untouched (read-modify-write of the W-bit fields in
// the lane runs).  One warp per stream.  Same bit layout as pack_tiles_kernel.
// The record and each writing lane's run words are staged in shared memory so
// the read-modify-writes cost one batch of global loads and one of stores.
__global__ void __launch_bounds__(256) append_token_kernel(
    OqCodecParams p, int role, const uint8_t* __restrict__ recs, size_t n_streams,
    const int64_t* __restrict__ pos_dev, int64_t pos_scalar, uint8_t* __restrict__ tiles,
    size_t tiles_cap) {
  __shared__ uint32_t rec_s[8][32];
  __shared__ uint32_t run_s[8][32][21];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const size_t s = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  if (s >= n_streams) return;
  const int64_t pos = pos_dev ? pos_dev[s] : pos_scalar;
  {
    const uint8_t* rg = recs + s * p.rec_bytes;
    uint32_t w = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t bi = 4 * lane + i;
      if (bi < p.rec_bytes) w |= (uint32_t)rg[bi] << (8 * i);
    }
    rec_s[wib][lane] = w;
  }
  __syncwarp();
  append_record(p, role, rec_s[wib], run_s[wib], s, pos, tiles, tiles_cap, lane);
}

// Fused decode-step append of K AND V (oq_cache_append_kv): blockIdx.y is the
// role; each warp encodes its stream's new vector (encode_key_warp, exact)
// straight into shared memory and writes it into the tile — one launch per
// step instead of compress + append for each of K and V.  d = 128 (QJL keys
// included: qjl_key_warp adds the sidecar).
constexpr int kAppendWarps = 4;
__global__ void __launch_bounds__(32 * kAppendWarps) append_fused_kernel(
    const __grid_constant__ OqCodecParams pk, const __grid_constant__ OqCodecParams pv,
    const void* __restrict__ xk, const void* __restrict__ xv, int dtype, size_t n_streams,
    const int64_t* __restrict__ pos_dev, int64_t pos_scalar, uint8_t* __restrict__ rk,
    uint8_t* __restrict__ rv, uint8_t* __restrict__ tk, uint8_t* __restrict__ tv,
    size_t tiles_cap) {
  __shared__ double row_s[kAppendWarps][132];
  __shared__ uint32_t rec_s[kAppendWarps][kRecWords];
  __shared__ uint32_t run_s[kAppendWarps][32][21];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, role = blockIdx.y;
  const size_t s = blockIdx.x * (size_t)kAppendWarps + wib;
  if (s >= n_streams) return;
  const OqCodecParams& p = role ? pv : pk;
  const int64_t pos = pos_dev ? pos_dev[s] : pos_scalar;
  uint8_t* tiles = role ? tv : tk;
  {
    // warm L1 with the codebook tables joint_round reads (their dependent
    // lookups would otherwise each pay an L2 round trip) while the key is
    // loaded and rotated; the tile's run words are copied asynchronously
    const uint32_t kk = p.K * p.K;
    const int t = threadIdx.x;
    auto pf = [](const void* a) { asm volatile("prefetch.global.L1 [%0];" ::"l"(a)); };
    for (uint32_t i = t; i < kk * 16 / 128; i += blockDim.x) pf(reinterpret_cast<const uint8_t*>(p.dirs32) + 128 * i);
    for (uint32_t i = t; i < kk * 24 / 128; i += blockDim.x) pf(reinterpret_cast<const uint8_t*>(p.dirs64) + 128 * i);
    for (int i = t; i < 32; i += blockDim.x) {
      pf(reinterpret_cast<const uint8_t*>(p.xi_lut) + 128 * i);
      pf(reinterpret_cast<const uint8_t*>(p.rho_lut) + 128 * i);
    }
    if (t == 0) {
      pf(p.xi_bnd);
      pf(p.rho_bnd);
      pf(p.rho_c);
    }
  }
  append_stage_runs(p, role, s, pos, tiles, tiles_cap, run_s[wib], lane);
  encode_key_warp(p, role ? xv : xk, dtype, s, row_s[wib], rec_s[wib], lane);
  if (p.qjl) qjl_key_warp(p, row_s[wib], rec_s[wib], lane, global_tables(p));
  uint8_t* recs = role ? rv : rk;
  if (recs) {
    const uint8_t* src = reinterpret_cast<const uint8_t*>(rec_s[wib]);
    for (uint32_t b = lane; b < p.rec_bytes; b += 32) recs[s * p.rec_bytes + b] = src[b];
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncwarp();
  append_record(p, role, rec_s[wib], run_s[wib], s, pos, tiles, tiles_cap, lane, true);
}

cudaError_t launch_append_fused(const OqCodecParams& pk, const OqCodecParams& pv, const void* xk,
                                const void* xv, int dtype, size_t n_streams,
                                const int64_t* pos_dev, int64_t pos_scalar, uint8_t* rk,
                                uint8_t* rv, uint8_t* tk, uint8_t* tv, size_t tiles_cap,
                                cudaStream_t st) {
  if (n_streams == 0) return cudaSuccess;
  const dim3 grid((unsigned)((n_streams + kAppendWarps - 1) / kAppendWarps), 2);
  append_fused_kernel<<<grid, 32 * kAppendWarps, 0, st>>>(pk, pv, xk, xv, dtype, n_streams, pos_dev,
                                                         pos_scalar, rk, rv, tk, tv, tiles_cap);
  return cudaGetLastError();
}

cudaError_t launch_append_token(const OqCodecParams& p, int role, const uint8_t* recs,
                                size_t n_streams, const int64_t* pos_dev, int64_t pos_scalar,
                                uint8_t* tiles, size_t tiles_cap, cudaStream_t st) {
  if (n_streams == 0) return cudaSuccess;
  const size_t blocks = (n_streams * 32 + 255) / 256;
  append_token_kernel<<<(unsigned)blocks, 256, 0, st>>>(p, role, recs, n_streams, pos_dev,
                                                        pos_scalar, tiles, tiles_cap);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
size_t attention_tile_bytes(const OqCodecParams& p, int role) {
  const int W = 2 * p.b_dir + p.b_nrm;
  // the attention kernels exist for W = 7, 10, 13 (b = 2, 3, 4 at the default split)
  if (p.dim != 128 || (W != 7 && W != 10 && W != 13)) return 0;
  return role == 0 ? ktile_bytes(W, p.qjl) : vtile_bytes(W);
}

int attention_num_parts(int B, int Hq, int Hkv, uint64_t T, uint64_t t0, uint64_t t1,
                        int n_splits, int num_sms) {
  if (n_splits > 0) return n_splits;
  const int G = Hq / Hkv, HC = (G + 7) / 8;
  const uint64_t te = t1 < T ? t1 : T;
  const uint64_t tb0 = t0 / kTileTok, tz = (te + kTileTok - 1) / kTileTok;
  const uint64_t tps = tz > tb0 ? tz - tb0 : 0;
  const uint64_t nsh = (uint64_t)B * Hkv * HC, U = nsh * tps;
  const uint64_t grid = U < (uint64_t)num_sms ? (U ? U : 1) : num_sms;
  // CTAs touching one stream: at most ceil(tps * grid / U) + 1
  return (int)((tps * grid + U - 1) / (U ? U : 1)) + 1;
}

size_t attention_qfrag_bytes(const OqCodecParams& pk) {
  return 32 * (18 + (pk.qjl ? 16 : 0)) * 4;
}

bool attention_fast_path_ok(const OqCodecParams& pk, const OqCodecParams& pv) {
  const int W = 2 * pk.b_dir + pk.b_nrm;
  return pk.dim == 128 && pv.dim == 128 && pk.b_dir == pv.b_dir && pk.b_nrm == pv.b_nrm &&
         (W == 7 || W == 10 || W == 13) && !pv.qjl;
}

cudaError_t launch_pack_tiles(const OqCodecParams& p, int role, const uint8_t* recs,
                              size_t n_streams, size_t n_tokens, size_t rec_stride,
                              uint8_t* tiles, size_t tiles_cap, cudaStream_t st) {
  const size_t warps = n_streams * ((n_tokens + 31) / 32);
  if (warps == 0) return cudaSuccess;
  const size_t blocks = (warps * 32 + 255) / 256;
  pack_tiles_kernel<<<(unsigned)blocks, 256, 0, st>>>(p, role, recs, n_streams, n_tokens,
                                                      rec_stride, tiles, tiles_cap);
  return cudaGetLastError();
}

template <int W, bool QJL, int NW, int RING = 0>
static cudaError_t launch_attn_t(const OqCodecParams& pk, const AttnArgs& a, int splits,
                                 int G, int HC, cudaStream_t st, int num_sms) {
  using C = Cfg<W, QJL>;
  AttnKParams P;
  P.tab = pk.jointrep;
  P.kcache = a.kcache;
  P.vcache = a.vcache;
  P.k_tiles_cap = a.k_tiles_cap;
  P.v_tiles_cap = a.v_tiles_cap;
  P.qfrag = static_cast<const uint32_t*>(a.qfrag);
  P.partials = a.partials;
  P.seq_lens = a.seq_lens;
  P.T = a.T;
  P.t_begin = a.t_begin;
  P.t_end = a.t_end;
  P.B = a.B;
  P.Hq = a.Hq;
  P.Hkv = a.Hkv;
  P.G = G;
  P.HC = HC;
  P.splits = splits;
  P.n_parts = a.n_parts;
  P.n_sh = a.B * a.Hkv * HC;
  P.streamk = splits == 0;
  P.n_items = P.n_sh * (splits > 0 ? splits : 1);
  {
    const size_t te = a.t_end < a.T ? a.t_end : a.T;
    P.tb0 = a.t_begin / kTileTok;
    const size_t tz = (te + kTileTok - 1) / kTileTok;
    P.tps = tz > P.tb0 ? tz - P.tb0 : 0;
  }
  P.fuse = a.out != nullptr && a.counters != nullptr;
  P.out_partial = a.out_partial;
  P.p2p_nranks = a.p2p_nranks;
  P.p2p_rank = a.p2p_rank;
  P.p2p_epoch = a.p2p_epoch;
  for (int i = 0; i < 8; ++i) P.p2p_xbuf[i] = i < a.p2p_nranks ? a.p2p_xbuf[i] : nullptr;
  P.qjl = pk.qjl;
  P.q = a.q;
  P.out = a.out;
  P.counters = a.counters;
  for (int i = 0; i < 4; ++i) {
    P.smask[i] = pk.sign_mask[i];
    P.qmask[i] = pk.qsign_mask[i];
    P.vmask[i] = a.vmask[i];
  }
  P.inv_sqrt_d = (float)pk.inv_sqrt_d;
  {
    // a stream start costs about as much as this many tiles on one SM
    static const long sko_env = [] {
      const char* e = getenv("OQ_ATTN_SKO");
      return e ? atol(e) : -1L;
    }();
    // (swept with tools/exp/sko_sweep.sh: 48 best at 4096 tiles per stream,
    // 32 at 1024)
    P.sko = sko_env >= 0 ? (size_t)sko_env : (P.tps >= 2048 ? 48 : P.tps >= 512 ? 32 : 0);
  }
  if (a.max_ctas > 0 && a.max_ctas < num_sms) num_sms = a.max_ctas;
  int grid = P.n_items < num_sms ? P.n_items : num_sms;
  if (P.streamk) {
    const size_t U = (size_t)P.n_sh * P.tps;
    grid = (int)(U < (size_t)num_sms ? (U ? U : 1) : num_sms);
  }
  cudaError_t e = set_smem_once(attn_partials_kernel<W, QJL, NW, RING>, C::smem(NW, RING));
  if (e != cudaSuccess) return e;
  // programmatic dependent launch (see the kernel's prologue): the table
  // staging overlaps the previous kernel's tail (OQ_ATTN_PDL=0 disables it)
  static const bool pdl = [] {
    const char* v = getenv("OQ_ATTN_PDL");
    return !(v && v[0] == '0');
  }();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NW * 32);
  cfg.dynamicSmemBytes = C::smem(NW, RING);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, attn_partials_kernel<W, QJL, NW, RING>, P);
}

cudaError_t launch_qprep(const OqCodecParams& pk, const AttnArgs& a, cudaStream_t st) {
  const int G = a.Hq / a.Hkv, HC = (G + 7) / 8;
  QPrepParams qp;
  qp.q = a.q;
  qp.qfrag = static_cast<uint32_t*>(a.qfrag);
  qp.Hq = a.Hq;
  qp.Hkv = a.Hkv;
  qp.G = G;
  qp.HC = HC;
  qp.QF = 18 + (pk.qjl ? 16 : 0);
  for (int i = 0; i < 4; ++i) {
    qp.smask[i] = pk.sign_mask[i];
    qp.qmask[i] = pk.qsign_mask[i];
  }
  qp.inv_sqrt_d = (float)pk.inv_sqrt_d;
  qp.qjl = pk.qjl;
  qprep_kernel<<<a.B * a.Hkv * HC, 256, 0, st>>>(qp);
  return cudaGetLastError();
}

cudaError_t launch_attention_partials(const OqCodecParams& pk, const OqCodecParams& pv,
                                      const AttnArgs& a, int splits, cudaStream_t st,
                                      int num_sms) {
  const int G = a.Hq / a.Hkv, HC = (G + 7) / 8;
  const int W = 2 * pk.b_dir + pk.b_nrm;
  // Warps per CTA (one CTA per SM) and the tile delivery: OQ_ATTN_WARPS /
  // OQ_ATTN_RING select a variant for tuning runs; the default is the
  // measured best.  RING 0 = register ping-pong, 2 = two-stage TMA ring.
  static const int ring_env = [] {
    const char* e = getenv("OQ_ATTN_RING");
    return e ? atoi(e) : -1;
  }();
  static const int nw_env = [] {
    const char* e = getenv("OQ_ATTN_WARPS");
    return e ? atoi(e) : -1;
  }();
  // measured defaults (tools/exp/abn.sh, r02; a 3-stage ring measured the
  // same as 2 stages): 12 warps fed by a 2-stage TMA ring for the byte-coded
  // 2-bit tiles (W = 7, C4/C5: C4 -10 %, C5 -1.7 % against 8 warps with
  // register prefetch) and, since the round-2 kernel changes, for the 10-bit
  // tiles too (C3 147.3 -> 144.0 us, A/B); 10-bit tiles with QJL keys (the
  // 12-warp ring does not fit their shared memory) keep 8 warps with
  // register prefetch; the 13-bit tiles (b = 4) need the ring's single
  // register image (8 warps)
  const int ring = ring_env >= 0 ? ring_env : (W == 10 && pk.qjl ? 0 : 2);
  const int nw = nw_env > 0 ? nw_env : (ring && W <= 10 ? 12 : 8);
  auto launch = [&](auto w_tag, auto q_tag) -> cudaError_t {
    constexpr int WW = decltype(w_tag)::value;
    constexpr bool QQ = decltype(q_tag)::value;
    // only the variants that fit in shared memory are instantiated
    if constexpr (Cfg<WW, QQ>::smem(12, 2) <= kMaxSmem)
      if (ring >= 2 && nw == 12) return launch_attn_t<WW, QQ, 12, 2>(pk, a, splits, G, HC, st, num_sms);
    if constexpr (Cfg<WW, QQ>::smem(8, 2) <= kMaxSmem)
      if (ring >= 2) return launch_attn_t<WW, QQ, 8, 2>(pk, a, splits, G, HC, st, num_sms);
    return launch_attn_t<WW, QQ, 8, 0>(pk, a, splits, G, HC, st, num_sms);
  };
  using I10 = std::integral_constant<int, 10>;
  using I7 = std::integral_constant<int, 7>;
  using I13 = std::integral_constant<int, 13>;
  using T_ = std::true_type;
  using F_ = std::false_type;
  if (W == 10 && !pk.qjl) return launch(I10{}, F_{});
  if (W == 10 && pk.qjl) return launch(I10{}, T_{});
  if (W == 7 && !pk.qjl) return launch(I7{}, F_{});
  if (W == 7 && pk.qjl) return launch(I7{}, T_{});
  if (W == 13 && !pk.qjl) return launch(I13{}, F_{});
  if (W == 13 && pk.qjl) return launch(I13{}, T_{});

  (void)pv;
  return cudaErrorNotSupported;
}

cudaError_t launch_attention_combine(const OqCodecParams& pv, const float* partials, int rows,
                                     int n_parts, size_t row_stride, size_t part_stride,
                                     int finalize, float* out, cudaStream_t st) {
  CombineParams P;
  P.parts = partials;
  P.out = out;
  P.rows = rows;
  P.n_parts = n_parts;
  P.finalize = finalize;
  P.row_stride = row_stride;
  P.part_stride = part_stride;
  for (int i = 0; i < 4; ++i) P.smask[i] = pv.sign_mask[i];
  P.inv_sqrt_d = (float)pv.inv_sqrt_d;
  const int per_block = 2;
  combine_kernel<<<(rows + per_block - 1) / per_block, 32 * per_block, 0, st>>>(P);
  return cudaGetLastError();
}

}  // namespace oqd
