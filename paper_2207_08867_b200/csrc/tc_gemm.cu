// tc_gemm.cu -- hand-written tcgen05 int8 GEMM for sm_100a (the residue GEMMs
// of the MCF_FAST tensor-core contraction, mm_ozaki.cu).
//
//   C_b (m x n, int32) = A_b (m x kp, int8, K contiguous) . B_b (n x kp)^T
//   for b < batch; epilogue either writes C_b (int32) or, for the CRT scheme,
//   C_b mod m_b as symmetric int8 residues (the reconstruction then reads a
//   quarter of the bytes and no reduction is left to do).
//
// Structure (one CTA per SM, persistent over (b, row block, column block)
// tiles of 128 x 256):
//   warp 0      TMA producer: 128-byte K blocks of A (128 rows) and B (256
//               rows) into a 4-stage shared-memory ring, SWIZZLE_128B,
//               mbarrier transaction counts;
//   warp 1      MMA issuer: one elected thread issues tcgen05.mma
//               .cta_group::1.kind::i8 (M 128, N 256, K 32; four per stage)
//               into one of two TMEM accumulators (2 x 256 columns), and
//               tcgen05.commit frees the stage / hands the accumulator over;
//   warps 2-5   epilogue: tcgen05.ld 32x32b.x32 (each warp its 32 TMEM lanes
//               = rows), exact int32 -> residue reduction, 32-byte stores,
//               then releases the accumulator (double buffering overlaps a
//               tile's epilogue with the next tile's MMAs).
// int32 accumulation of int8 products is exact (|C| <= K 2^14 < 2^31 for
// K < 2^17).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <mutex>

#include "mcf_runtime.h"

namespace mcfg {
namespace tc {
namespace {

constexpr int BM = 128, BN = 256, BK = 128;  // BK: bytes (= int8 elements) per stage per row
constexpr int kStages = 4;
constexpr int kABytes = BM * BK, kBBytes = BN * BK, kStageBytes = kABytes + kBBytes;
constexpr int kThreads = 192;
constexpr int kTmemCols = 512;
constexpr int kMaxBatch = 32;
constexpr float kMagic = 12582912.0f;  // 1.5 2^23

struct Params {
  int stages;  // pair kernel: depth of the shared-memory ring (<= kStages2)
  int raster;  // row blocks per raster group (tile_coords)
  int m, n, kp, batch, tiles_m, tiles_n;
  int64_t ldo;           // output row stride (elements)
  int mode;              // 0: int32 C, 1: int8 residues C mod m_b
  void* out;             // [batch][m][ldo]
  float mod[kMaxBatch];  // modulus of batch entry b (mode 1)
  float inv[kMaxBatch];  // RN32(1 / m_b)
  float c14[kMaxBatch];  // 2^14 mod m_b, symmetric
  int big;               // |C| may exceed 2^28 (K > 2^14): two-step reduction
  // segment mode (nseg > 0, int32 output, pair kernel): batch entry b reads
  // K bytes [seg_ka[b], + 128 seg_kblk[b]) of every row of a and [seg_kb[b],
  // ...) of every row of b (one 2-D operand each, rows of any stride): the
  // diagonal GEMMs of the digit-plane schemes, one launch for all diagonals
  int nseg;
  int seg_ka[kMaxBatch], seg_kb[kMaxBatch], seg_kblk[kMaxBatch];
};

// Tile order inside one batch entry (modulus / segment): row blocks in groups
// of kRaster, and within a group the column block outermost -- the ~74 tiles
// in flight then cover kRaster row blocks x ~9 column blocks instead of one
// row block x every column block, so a wave re-reads a few operand panels
// from L2 instead of streaming the whole B plane from HBM (16384^3: 14.7 GB
// per modulus down to 2.3 GB).  r in [0, tiles_m * tiles_n).
__device__ __forceinline__ void tile_coords(int r, int tiles_m, int tiles_n, int raster, int& mb, int& nb) {
  const int per_group = raster * tiles_n;
  const int g = r / per_group, q = r - g * per_group;
  const int rows = tiles_m - g * raster < raster ? tiles_m - g * raster : raster;  // the last group may be short
  nb = q / rows;
  mb = g * raster + (q - nb * rows);
}

// ---- PTX helpers ----

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// K-major operand in the canonical SWIZZLE_128B layout (8-row atoms of 128 B,
// atoms 1024 B apart): start >> 4, LBO 1 (16 B, unused when swizzled), SBO
// 1024 >> 4, version 1 (sm_100), layout type 2 = SWIZZLE_128B
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) |
         ((uint64_t)2 << 61);
}
// kind::i8 instruction descriptor: D s32 (c_format 2), A / B s8 (format 1),
// both K-major, N >> 3 at bit 17, M >> 4 at bit 24
constexpr uint32_t kIdesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ void umma_i8(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(kIdesc), "r"(accumulate)
      : "memory");
}

#define TMEM_LD32(taddr, v)                                                                                     \
  asm volatile(                                                                                                 \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17," \
      "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                        \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),        \
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),   \
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),              \
        "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),              \
        "=r"(v[30]), "=r"(v[31])                                                                                \
      : "r"(taddr))

// C mod m (symmetric) of an exact int32 sum, as kMagic + r (low byte = r as
// int8); the same arithmetic as mm_ozaki.cu's mod_c (CPU-pinned in
// tests/test_crt_scheme.py)
__device__ __forceinline__ uint32_t mod_bits(int c, float m, float inv, float c14, bool big) {
  const int cl = ((c + 8192) & 16383) - 8192, ch = (c - cl) >> 14;
  const float fl = __fsub_rn(__int_as_float(cl + 0x4B400000), kMagic);
  const float fh = __fsub_rn(__int_as_float(ch + 0x4B400000), kMagic);
  float s = __fmaf_rn(fh, c14, fl);
  if (big) {
    const float q0 = __fsub_rn(__fmaf_rn(s, inv, kMagic), kMagic);
    s = __fmaf_rn(-q0, m, s);
  }
  const float q = __fsub_rn(__fmaf_rn(s, inv, kMagic), kMagic);
  return __float_as_uint(__fmaf_rn(-q, m, __fadd_rn(s, kMagic)));
}

__global__ void __launch_bounds__(kThreads, 1)
    k_tc_gemm_s8(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, const Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment for the SWIZZLE_128B atoms
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;
  uint8_t* sb = smem + kStages * kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ta)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tb)) : "memory");
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull + a, 1);
      mbar_init(tempty + a, 4);  // one arrival per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;

  const int per_b = p.tiles_m * p.tiles_n;
  const int total = per_b * p.batch;
  const int kblocks = (p.kp + BK - 1) / BK;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
        const int b = tile / per_b, r = tile - b * per_b;
        int mb, nb;
        tile_coords(r, p.tiles_m, p.tiles_n, p.raster, mb, nb);
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(empty + stage, phase ^ 1);
          mbar_expect_tx(full + stage, kStageBytes);
          tma_load_3d(sa + stage * kABytes, &ta, kb * BK, mb * BM, b, full + stage);
          tma_load_3d(sb + stage * kBBytes, &tb, kb * BK, nb * BN, b, full + stage);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int stage = 0, acc = 0;
      uint32_t phase = 0, aphase = 0;
      for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
        mbar_wait(tempty + acc, aphase ^ 1);
        fence_after();
        const uint32_t d = tmem + acc * BN;
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(full + stage, phase);
          fence_after();
          const uint32_t a0 = smem_u32(sa + stage * kABytes), b0 = smem_u32(sb + stage * kBBytes);
#pragma unroll
          for (int kk = 0; kk < BK / 32; ++kk)
            umma_i8(d, smem_desc(a0 + kk * 32), smem_desc(b0 + kk * 32), (kb | kk) != 0);
          umma_commit(empty + stage);  // the stage is free once these MMAs have read it
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(tfull + acc);  // accumulator complete
        if (++acc == 2) {
          acc = 0;
          aphase ^= 1;
        }
      }
    }
  } else {
    // epilogue: warp w reads TMEM lanes 32 (w % 4) .. + 31 = tile rows
    const int q = warp & 3;
    const int row_in_tile = q * 32 + lane;
    int acc = 0;
    uint32_t aphase = 0;
    for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
      const int b = tile / per_b, r = tile - b * per_b;
      int mb, nb;
      tile_coords(r, p.tiles_m, p.tiles_n, p.raster, mb, nb);
      mbar_wait(tfull + acc, aphase);
      fence_after();
      const int row = mb * BM + row_in_tile;
      const bool row_ok = row < p.m;
      const float fm = p.mod[b < kMaxBatch ? b : 0], fi = p.inv[b < kMaxBatch ? b : 0],
                  fc = p.c14[b < kMaxBatch ? b : 0];
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t v[32];
        TMEM_LD32(tmem + ((uint32_t)(q * 32) << 16) + acc * BN + c * 32, v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const int col = nb * BN + c * 32;
        if (!row_ok || col >= p.n) continue;
        if (p.mode == 0) {
          int* o = static_cast<int*>(p.out) + ((int64_t)b * p.m + row) * p.ldo + col;
#pragma unroll
          for (int u = 0; u < 32; u += 4)
            if (col + u < p.n) *reinterpret_cast<int4*>(o + u) = make_int4(v[u], v[u + 1], v[u + 2], v[u + 3]);
        } else {
          uint32_t w[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const uint32_t r0 = mod_bits((int)v[4 * u], fm, fi, fc, p.big),
                           r1 = mod_bits((int)v[4 * u + 1], fm, fi, fc, p.big),
                           r2 = mod_bits((int)v[4 * u + 2], fm, fi, fc, p.big),
                           r3 = mod_bits((int)v[4 * u + 3], fm, fi, fc, p.big);
            w[u] = __byte_perm(__byte_perm(r0, r1, 0x0040), __byte_perm(r2, r3, 0x0040), 0x5410);
          }
          int8_t* o = static_cast<int8_t*>(p.out) + ((int64_t)b * p.m + row) * p.ldo + col;
          *reinterpret_cast<uint4*>(o) = make_uint4(w[0], w[1], w[2], w[3]);
          if (col + 16 < p.n) *reinterpret_cast<uint4*>(o + 16) = make_uint4(w[4], w[5], w[6], w[7]);
        }
      }
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty + acc);
      if (++acc == 2) {
        acc = 0;
        aphase ^= 1;
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
  }
}

// ---- CTA-pair variant (cta_group::2): one 256 x 256 tile per pair of SMs ----
//
// The two CTAs of a cluster share each MMA: CTA r stages rows r*128.. of the
// tile's A and rows r*128.. of its B (N) half, so per SM the stage is 32 KB
// (six stages) and the tensor core reads half of B from the peer.  The
// leader (rank 0) issues tcgen05.mma.cta_group::2 (M 256, N 256); both CTAs'
// TMA loads complete on the leader's full barrier (peer bit cleared), the
// leader's commits multicast to both CTAs' empty / accumulator-full
// barriers, and both CTAs' epilogue warps release the accumulator on the
// leader's barrier (8 arrivals).  Each CTA's TMEM holds its own 128 rows.
constexpr int kStages2 = 7;  // 7 x 32 KB + alignment + barriers fit the 227 KB
constexpr int kHalfBytes = 128 * BK;  // 16 KB: 128 rows x 128 bytes
constexpr int kStage2 = 2 * kHalfBytes;
constexpr uint32_t kIdesc2 =
    (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_3d_pair(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                                 uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
      "%4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar) & 0xFEFFFFFFu)
      : "memory");
}
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void umma_i8_pair(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(kIdesc2), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(0));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    k_tc_gemm_s8_pair(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, const Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int nst = p.stages;  // ring depth: 7 fills the SM's shared memory, fewer leave room for co-resident kernels
  uint8_t* sa = smem;
  uint8_t* sb = smem + nst * kHalfBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + nst * kStage2);
  uint64_t* empty = full + nst;
  uint64_t* tfull = empty + nst;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cta_rank();
  const bool leader = rank == 0;
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ta)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tb)) : "memory");
    for (int s = 0; s < nst; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull + a, 1);
      mbar_init(tempty + a, 8);  // four epilogue warps in each CTA of the pair
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  fence_before();
  cluster_sync();
  fence_after();
  const uint32_t tmem = *tmem_slot;

  const int tiles_m2 = (p.m + 255) / 256;
  const int per_b = tiles_m2 * p.tiles_n;
  const int total = per_b * p.batch;
  const int kblocks = (p.kp + BK - 1) / BK;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = pair; tile < total; tile += npairs) {
        const int b = tile / per_b, r = tile - b * per_b;
        int mb, nb;
        tile_coords(r, tiles_m2, p.tiles_n, p.raster, mb, nb);
        const int kbl = p.nseg ? p.seg_kblk[b] : kblocks, ka0 = p.nseg ? p.seg_ka[b] : 0,
                  kb0 = p.nseg ? p.seg_kb[b] : 0, zb = p.nseg ? 0 : b;
        for (int kb = 0; kb < kbl; ++kb) {
          mbar_wait(empty + stage, phase ^ 1);
          if (leader) mbar_expect_tx(full + stage, 2 * kStage2);
          tma_load_3d_pair(sa + stage * kHalfBytes, &ta, ka0 + kb * BK, mb * 256 + (int)rank * 128, zb, full + stage);
          tma_load_3d_pair(sb + stage * kHalfBytes, &tb, kb0 + kb * BK, nb * 256 + (int)rank * 128, zb, full + stage);
          if (++stage == nst) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      int stage = 0, acc = 0;
      uint32_t phase = 0, aphase = 0;
      for (int tile = pair; tile < total; tile += npairs) {
        const int kbl = p.nseg ? p.seg_kblk[tile / per_b] : kblocks;
        mbar_wait(tempty + acc, aphase ^ 1);
        fence_after();
        const uint32_t d = tmem + acc * BN;
        for (int kb = 0; kb < kbl; ++kb) {
          mbar_wait(full + stage, phase);
          fence_after();
          const uint32_t a0 = smem_u32(sa + stage * kHalfBytes), b0 = smem_u32(sb + stage * kHalfBytes);
#pragma unroll
          for (int kk = 0; kk < BK / 32; ++kk)
            umma_i8_pair(d, smem_desc(a0 + kk * 32), smem_desc(b0 + kk * 32), (kb | kk) != 0);
          umma_commit_pair(empty + stage);
          if (++stage == nst) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_pair(tfull + acc);
        if (++acc == 2) {
          acc = 0;
          aphase ^= 1;
        }
      }
    }
  } else {
    const int q = warp & 3;
    const int row_in_tile = (int)rank * 128 + q * 32 + lane;
    int acc = 0;
    uint32_t aphase = 0;
    for (int tile = pair; tile < total; tile += npairs) {
      const int b = tile / per_b, r = tile - b * per_b;
      int mb, nb;
      tile_coords(r, tiles_m2, p.tiles_n, p.raster, mb, nb);
      mbar_wait(tfull + acc, aphase);
      fence_after();
      const int row = mb * 256 + row_in_tile;
      const bool row_ok = row < p.m;
      const float fm = p.mod[b < kMaxBatch ? b : 0], fi = p.inv[b < kMaxBatch ? b : 0],
                  fc = p.c14[b < kMaxBatch ? b : 0];
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t v[32];
        TMEM_LD32(tmem + ((uint32_t)(q * 32) << 16) + acc * BN + c * 32, v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const int col = nb * BN + c * 32;
        if (!row_ok || col >= p.n) continue;
        if (p.mode == 0) {
          int* o = static_cast<int*>(p.out) + ((int64_t)b * p.m + row) * p.ldo + col;
#pragma unroll
          for (int u = 0; u < 32; u += 4)
            if (col + u < p.n) *reinterpret_cast<int4*>(o + u) = make_int4(v[u], v[u + 1], v[u + 2], v[u + 3]);
        } else {
          uint32_t w[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const uint32_t r0 = mod_bits((int)v[4 * u], fm, fi, fc, p.big),
                           r1 = mod_bits((int)v[4 * u + 1], fm, fi, fc, p.big),
                           r2 = mod_bits((int)v[4 * u + 2], fm, fi, fc, p.big),
                           r3 = mod_bits((int)v[4 * u + 3], fm, fi, fc, p.big);
            w[u] = __byte_perm(__byte_perm(r0, r1, 0x0040), __byte_perm(r2, r3, 0x0040), 0x5410);
          }
          int8_t* o = static_cast<int8_t*>(p.out) + ((int64_t)b * p.m + row) * p.ldo + col;
          *reinterpret_cast<uint4*>(o) = make_uint4(w[0], w[1], w[2], w[3]);
          if (col + 16 < p.n) *reinterpret_cast<uint4*>(o + 16) = make_uint4(w[4], w[5], w[6], w[7]);
        }
      }
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_leader(tempty + acc);
      if (++acc == 2) {
        acc = 0;
        aphase ^= 1;
      }
    }
  }
  fence_before();
  cluster_sync();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

// [batch][rows][kp] int8, box 128 (K bytes) x box_rows x 1, SWIZZLE_128B
bool make_map(CUtensorMap* map, const int8_t* base, int64_t rows, int64_t kp, int batch, int box_rows) {
  auto enc = encode_fn();
  if (!enc) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)kp, (cuuint64_t)rows, (cuuint64_t)batch};
  const cuuint64_t strides[2] = {(cuuint64_t)kp, (cuuint64_t)(rows * kp)};
  const cuuint32_t box[3] = {(cuuint32_t)BK, (cuuint32_t)box_rows, 1u};
  const cuuint32_t estr[3] = {1u, 1u, 1u};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace
}  // namespace tc
}  // namespace mcfg

namespace mcfr {

// row blocks per raster group (MCF_TC_RASTER; default 8).  Measured on B200
// (r02, 16384^3 x 20 moduli): DRAM reads per modulus 10.1 GB at 8 and 8.3 GB at
// 16 against ~14 GB unrastered (ncu), the product 99.9 -> 87-91 ms; at that
// size the GEMM is limited by the sustained power cap (a 4-modulus run of the
// same shape reaches 3.1 POPS, the 20-modulus run 2.3 POPS at 1.16 GHz), which
// the DRAM traffic shares.  Config 2 (everything L2-resident) is unchanged.
static int raster_rows() {
  static const int n = [] {
    const char* e = getenv("MCF_TC_RASTER");
    const int v = e ? atoi(e) : 8;
    return v < 1 ? 1 : (v > 64 ? 64 : v);
  }();
  return n;
}

// ring depth of the pair kernel (MCF_TC_STAGES, 5..7; default 7).  Measured
// on B200 (r02, config 2): 5, 6 and 7 stages all give 1.33 ms per product, and
// the shallower rings (which leave shared memory for the residue /
// reconstruction kernels of other row blocks to share the SMs, MCF_OZ_PIPE)
// do not make the pipelined product faster (2 blocks 1.34 ms, 4 blocks 1.37).
static int pair_stages() {
  static const int n = [] {
    const char* e = getenv("MCF_TC_STAGES");
    const int v = e ? atoi(e) : mcfg::tc::kStages2;
    return v < 5 ? 5 : (v > mcfg::tc::kStages2 ? mcfg::tc::kStages2 : v);
  }();
  return n;
}

// C_b = A_b . B_b^T (b < batch) on the hand-written tcgen05 kernel.
// a: [batch][m][kp], b: [batch][b_rows][kp] int8 (the first n rows used) (kp % 16 == 0, 16-byte aligned
// bases); out: [batch][m][ldo] int32 (moduli == nullptr) or int8 residues
// C_b mod moduli[b] (symmetric).  MCF_ERR_UNSUPPORTED when the shape or the
// driver's tensor-map entry point is unavailable.
mcf_status tc_gemm_s8(const int8_t* a, const int8_t* b, void* out, int64_t m, int64_t n, int64_t kp, int batch,
                      int64_t ldo, const int* moduli, cudaStream_t s, int64_t b_rows) {
  if (b_rows < n) b_rows = n;  // rows per plane of b (>= n: padded columns)
  using namespace mcfg::tc;
  if (m <= 0 || n <= 0 || kp <= 0 || kp % 16 != 0 || batch < 1 || (moduli && batch > kMaxBatch) ||
      kp >= (int64_t(1) << 17) || m >= (int64_t(1) << 31) || n >= (int64_t(1) << 31))
    return MCF_ERR_UNSUPPORTED;
  // the epilogue's 16-byte stores: int32 rows a multiple of 4 elements,
  // residue rows of 16 bytes, 16-byte aligned bases
  if (ldo < n || ldo % (moduli ? 16 : 4) != 0 || (reinterpret_cast<uintptr_t>(out) & 15) ||
      (reinterpret_cast<uintptr_t>(a) & 15) || (reinterpret_cast<uintptr_t>(b) & 15))
    return MCF_ERR_UNSUPPORTED;
  CUtensorMap ta, tb;
  if (!make_map(&ta, a, m, kp, batch, BM) || !make_map(&tb, b, b_rows, kp, batch, BN)) return MCF_ERR_UNSUPPORTED;
  Params p{};
  p.m = (int)m;
  p.n = (int)n;
  p.kp = (int)kp;
  p.batch = batch;
  p.tiles_m = (int)((m + BM - 1) / BM);
  p.tiles_n = (int)((n + BN - 1) / BN);
  p.ldo = ldo;
  p.mode = moduli ? 1 : 0;
  p.out = out;
  p.big = kp > 16384;
  p.raster = raster_rows();
  if (moduli)
    for (int i = 0; i < batch; ++i) {
      const int mm = moduli[i];
      int p14 = 1;
      for (int t = 0; t < 14; ++t) p14 = p14 * 2 % mm;
      if (p14 > mm / 2) p14 -= mm;
      p.mod[i] = (float)mm;
      p.inv[i] = 1.0f / (float)mm;
      p.c14[i] = (float)p14;
    }
  // MCF_TC_PAIR=0 selects the single-CTA kernel (A/B measurement)
  static const bool pair = [] {
    const char* e = getenv("MCF_TC_PAIR");
    return !(e && atoi(e) == 0);
  }();
  if (pair) {
    CUtensorMap tb2;
    if (!make_map(&tb2, b, b_rows, kp, batch, 128)) return MCF_ERR_UNSUPPORTED;
    p.stages = pair_stages();
    const int smem = p.stages * kStage2 + 1024 + 256;
    per_device_once(kOnceTcGemm, [&] {
      cudaFuncSetAttribute(k_tc_gemm_s8_pair, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           kStages2 * kStage2 + 1024 + 256);
    });
    const int64_t tiles = (int64_t)((m + 255) / 256) * p.tiles_n * batch;
    const int grid = 2 * (int)std::min<int64_t>(tiles, sm_count() / 2);
    // a.k.a. TMA box of 128 rows for both operands (each CTA loads half the tile)
    CUtensorMap ta2;
    if (!make_map(&ta2, a, m, kp, batch, 128)) return MCF_ERR_UNSUPPORTED;
    k_tc_gemm_s8_pair<<<grid, kThreads, smem, s>>>(ta2, tb2, p);
  } else {
    const int smem = kStages * kStageBytes + 1024 + 256;
    per_device_once(kOnceTcGemm + 8, [&] {
      cudaFuncSetAttribute(k_tc_gemm_s8, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    });
    const int64_t tiles = (int64_t)p.tiles_m * p.tiles_n * batch;
    const int grid = (int)std::min<int64_t>(tiles, sm_count());
    k_tc_gemm_s8<<<grid, kThreads, smem, s>>>(ta, tb, p);
  }
  note_launch();
  return check_launch("tcgen05 int8 GEMM");
}

// The diagonal GEMMs of a digit-plane scheme in one launch (pair kernel,
// int32 output): for d < nseg, out_d (m x n, row stride ldo) = A_d . B_d^T
// with A_d = bytes [ka[d], ka[d] + kd[d]) of each of a's m rows (row stride
// lda bytes) and B_d likewise from b (n used of b_rows rows, stride ldb).
// ka, kb, kd multiples of 128 (a segment's last K block must not read the
// next segment's bytes); MCF_ERR_UNSUPPORTED otherwise.
mcf_status tc_gemm_s8_seg(const int8_t* a, int64_t lda, const int8_t* b, int64_t ldb, int* out, int64_t m, int64_t n,
                          int64_t b_rows, int nseg, const int* ka, const int* kb, const int* kd, int64_t ldo,
                          cudaStream_t s) {
  using namespace mcfg::tc;
  if (b_rows < n) b_rows = n;
  if (m <= 0 || n <= 0 || nseg < 1 || nseg > kMaxBatch || lda % 16 || ldb % 16 || ldo < n || ldo % 4 ||
      (reinterpret_cast<uintptr_t>(out) & 15) || (reinterpret_cast<uintptr_t>(a) & 15) ||
      (reinterpret_cast<uintptr_t>(b) & 15) || m >= (int64_t(1) << 31) || n >= (int64_t(1) << 31))
    return MCF_ERR_UNSUPPORTED;
  Params p{};
  p.m = (int)m;
  p.n = (int)n;
  p.kp = BK;
  p.batch = nseg;
  p.tiles_m = (int)((m + BM - 1) / BM);
  p.tiles_n = (int)((n + BN - 1) / BN);
  p.ldo = ldo;
  p.mode = 0;
  p.out = out;
  p.nseg = nseg;
  p.raster = raster_rows();
  for (int d = 0; d < nseg; ++d) {
    if (ka[d] % BK || kb[d] % BK || kd[d] % BK || kd[d] <= 0 || ka[d] + kd[d] > lda || kb[d] + kd[d] > ldb ||
        kd[d] >= (1 << 17))
      return MCF_ERR_UNSUPPORTED;
    p.seg_ka[d] = ka[d];
    p.seg_kb[d] = kb[d];
    p.seg_kblk[d] = kd[d] / BK;
  }
  CUtensorMap ta2, tb2;
  if (!make_map(&ta2, a, m, lda, 1, 128) || !make_map(&tb2, b, b_rows, ldb, 1, 128)) return MCF_ERR_UNSUPPORTED;
  p.stages = pair_stages();
  const int smem = p.stages * kStage2 + 1024 + 256;
  per_device_once(kOnceTcGemm, [&] {
    cudaFuncSetAttribute(k_tc_gemm_s8_pair, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kStages2 * kStage2 + 1024 + 256);
  });
  const int64_t tiles = (int64_t)((m + 255) / 256) * p.tiles_n * nseg;
  const int grid = 2 * (int)std::min<int64_t>(tiles, sm_count() / 2);
  k_tc_gemm_s8_pair<<<grid, kThreads, smem, s>>>(ta2, tb2, p);
  note_launch();
  return check_launch("tcgen05 int8 GEMM (segments)");
}

}  // namespace mcfr

extern "C" {

// probe / test entry point: int32 products (moduli == null) or residues
mcf_status mcf_tc_gemm_s8(const void* a, const void* b, void* out, int64_t m, int64_t n, int64_t kp, int batch,
                          int64_t ldo, const int* moduli, mcf_stream stream) {
  if (!a || !b || !out) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "tc_gemm_s8: null argument");
  const mcf_status st = mcfr::tc_gemm_s8(static_cast<const int8_t*>(a), static_cast<const int8_t*>(b), out, m, n, kp,
                                         batch, ldo, moduli, static_cast<cudaStream_t>(stream));
  if (st == MCF_ERR_UNSUPPORTED) return mcfr::fail(st, "tc_gemm_s8: shape or driver entry point unsupported");
  return st;
}

}  // extern "C"
