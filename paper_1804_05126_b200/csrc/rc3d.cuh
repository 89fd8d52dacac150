// rc3d.cuh -- the config-4 fused IOP pass (Alg. 2) in
// the RECOMPUTE form, fed by TMA tensor-map loads, on a ghost-padded grid layout.
//
// Pass k completes Alg. 2 iteration k-1 and starts iteration k WITHOUT a stored
// r_{k-1} = (A~ x_{k-1})_top: every CTA recomputes it on the halo-1 ring of its tile
// from the halo-2 tile of x_{k-1}, so the pass moves the SURVEY 8(d) MINIMUM
// (q+1+p+c) 8N bytes -- read x_{k-1}, x_{k-2}, B (p vectors), kappa; write x_k --
// instead of the lazy form's (q+3+p+c) 8N (805 vs 1074 MB at 256^3, p = 2):
//
//   stage 1, plane L (halo-1 ring + interior):
//     r_{k-1} = A x_{k-1} + nu B t_{k-1}                         (Thm 1)
//     x_k     = a0 r_{k-1} - a1 x_{k-1} - a2 x_{k-2}               (l.7-10, l.17 folded)
//   stage 2, plane L-1 (interior):
//     r_k = A x_k + nu B t_k ;  S = x_k.x_k, G = x_{k-1}.x_k, E1 = x_{k-1}.r_k,
//     E2 = x_k.r_k, R = r_k.r_k  (block partials; the grid reduction and the
//     finalisation are the persistent loop's, inner.cuh) ; store x_k.
//
// with A the 7-point variable-kappa operator (A u)_i = 1/h^2 sum_faces kappa_f
// (u_nb - u_i), kappa_f = (kappa_i + kappa_nb)/2 (BJ config 4, reading D6), evaluated
// as 0.5/h^2 sum (kappa_i + kappa_nb)(u_nb - u_i) in the lazy kernels' operand order.
//
// Layout ("padded mode"): every vector the pass reads is stored with
// two ghost columns / rows on each side of every xy plane, (nx+4) x (ny+4) x nz,
// index (x+2) + (nx+4) ((y+2) + (ny+4) z); ghosts hold the periodic images, so a
// tile's halo box is ONE rectangular TMA box with no wrap.  z wraps through the TMA
// coordinate.  The basis slots, the B copies and the kappa copy form one 4-D tensor
// [nx+4][ny+4][nz][slot] (slot stride ldN doubles) described by two tensor maps
// (box 68 x (HM+4) for the halo-2 operands x_{k-1}, kappa; 68 x (HM+2) for the halo-1
// operands x_{k-2}, B).  The pass writes x_k's interior AND its ghost images.
//
// Decomposition: tiles of 64 x hb points (hb <= HM, balanced bands) x z-parts, one
// unit per CTA per wave (config 4: 4 x 37 tiles, 148 CTAs, one z-part, the full
// periodic z column), every CTA marching z in lock-step with the others (halo rows
// shared by neighbouring tiles are read at about the same time: L2 hits), direction
// alternating with the pass parity.  Per CTA: a ring of RS = D + 2 plane slots
// filled by one thread with 2 + 1 + p TMA boxes per plane (mbarrier complete_tx),
// D planes ahead; threads own 16-byte pairs: interior pairs in full warps (one warp
// = one 64-point row), the halo ring in the last warps; x_k of plane L is published
// in a 2-plane shared exchange ring for the in-plane neighbours of stage 2; z
// neighbours and the face sums of stage 2 stay in registers (carried from stage 1 of
// the previous plane).  ONE __syncthreads per plane.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

// KIOPS_BOUNDS_CHECK (debug builds, scripts/sanitize_run.py): device asserts on every
// shared-memory offset, ring slot, TMA coordinate and global store offset of the pass
// (compute-sanitizer is not available on this GPU pool).
#ifdef KIOPS_BOUNDS_CHECK
#include <cassert>
#define RC3_ASSERT(c) assert(c)
#else
#define RC3_ASSERT(c) do { } while (0)
#endif

#ifndef RC3_PRODUCER
#define RC3_PRODUCER 0  // the thread that issues the TMA boxes
#endif
#ifndef RC3_FFORM
#define RC3_FFORM 1  // stencil as sum_f k_f x_f - (sum_f k_f) x_c, the diagonal sum F carried to stage 2
                     // (stage 2 saves the six differences per point: 164.5 vs 167.3 us per pass,
                     // microbenchmark; folding a0 into the scalars and fma-chain dots measured slower)
#endif
#ifndef RC3_SPLIT
#define RC3_SPLIT 1
#endif
#ifndef RC3_ROLEMAP
#define RC3_ROLEMAP 1
#endif

namespace rc3 {

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "RC3_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra RC3_WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
// 4-D tensor-map box load global -> shared, completion on the mbarrier
__device__ __forceinline__ void tma_load4(void *dst, const void *tmap, int c0, int c1, int c2, int c3, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const void *tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
}
__device__ __forceinline__ double2 ld2(const double *p) { return *reinterpret_cast<const double2 *>(p); }

// Frozen geometry of the padded-mode 3D operator (identical in every pass).
struct Geom {
  int nx, ny, nz;          // grid (nx even, nx, ny >= 4)
  int Xp, Yp;              // padded extents nx + 4, ny + 4
  long long ldN;           // slot stride of the 4-D tensor (doubles)
  int ntx, nb, zsplit;     // 64-wide x tiles, y bands, z parts
  int slot_kappa, slot_B;  // 4-D slot of the kappa copy and of B column 0 (= u_p copy)
  const void *mapA, *mapB; // tensor maps (global memory): halo-2 box, halo-1 box
  double *V;               // slot 0 of the 4-D tensor
  double hh;               // 0.5 / h^2
};

// Per-pass arguments (identical in every CTA).
template <int PM>
struct PassArgs {
  int k;
  int slot_prev, slot_pp;  // 4-D slots of x_{k-1}, x_{k-2} (slot_pp < 0: none)
  double *xout;            // x_k (padded; NULL: x_1 is the start vector itself)
  double a0, a1, a2;       // x_k = a0 r_{k-1} - a1 x_{k-1} - a2 x_{k-2}
  double btp[PM > 0 ? PM : 1], btc[PM > 0 ? PM : 1];  // nu t_{k-1}, nu t_k
  int use_r;               // k >= 2
};

// Tile rule (host and device): ntx columns of 64 points; nb bands of <= hm rows
// giving about `ctas` tiles; z parts filling the CTAs (>= 2 planes each).
__host__ __device__ inline void tiles(int nx, int ny, int nz, int ctas, int hm, int *ntx, int *nb, int *zs) {
  const int tx = (nx + 63) / 64;
  int b = ctas / tx;
  if (b < 1) b = 1;
  if (b > ny) b = ny;
  const int bmin = (ny + hm - 1) / hm;
  if (b < bmin) b = bmin;
  int z = ctas / (tx * b);
  if (z < 1) z = 1;
  if (z > nz / 2) z = nz / 2 > 0 ? nz / 2 : 1;
  *ntx = tx;
  *nb = b;
  *zs = z;
}

template <int PM, int HM, int D>
struct Cfg {
  static constexpr int W = 68;                 // box row: 64 + 2 halo columns each side (doubles)
  static constexpr int RA = HM + 4, RB = HM + 2;  // box rows: halo-2 / halo-1
  static constexpr unsigned BYTES_A = W * RA * 8, BYTES_B = W * RB * 8;
  static constexpr int SA = (BYTES_A + 127) / 128 * 16, SB = (BYTES_B + 127) / 128 * 16;  // doubles, 128-B multiples
  static constexpr int SLOT = 2 * SA + (1 + PM) * SB;  // X, kappa, x_{k-2}, B_0..B_{PM-1}
  static constexpr int RS = D + 2;
  static constexpr int EXP = 34 * (HM + 2);    // exchange ring: pairs per plane
  static constexpr int NT = (32 * HM + 2 * 34 + 2 * HM + 31) / 32 * 32;
  static constexpr size_t smem_bytes = 128 + (size_t)RS * SLOT * 8 + 2 * (size_t)(EXP + 32) * 16 + 8 * (size_t)RS;
};

// Shared-memory carve-up: [ring RS x SLOT doubles][exchange 2 x EXP pairs][RS mbarriers]
template <int PM, int HM, int D>
__device__ __forceinline__ double *smem_base() {
  extern __shared__ __align__(128) unsigned char rc3_dsm[];
  return reinterpret_cast<double *>(rc3_dsm);
}
template <int PM, int HM, int D>
__device__ __forceinline__ uint64_t *bars(double *sm) {
  using C = Cfg<PM, HM, D>;
  return reinterpret_cast<uint64_t *>(sm + (size_t)C::RS * C::SLOT + 4 * (size_t)(C::EXP + 32));
}
// Once per kernel launch, before the first pass (thread 0 inits, then a barrier).
template <int PM, int HM, int D>
__device__ __forceinline__ void init(const Geom &G) {
  double *sm = smem_base<PM, HM, D>();
  uint64_t *b = bars<PM, HM, D>(sm);
  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg<PM, HM, D>::RS; s++) mbar_init(b + s, 1);
    fence_mbar_init();
    tma_prefetch_desc(G.mapA);
    tma_prefetch_desc(G.mapB);
  }
  __syncthreads();
}

// One work unit (tile x z-part) of a pass: tile origin, band height, interior pairs,
// z range, march direction (alternating with the pass parity) and the physical plane
// of logical plane 0.
struct UnitGeo {
  int ox, oy, hb, tw, zlo, zhi, nzc, dz, z0;
};
__device__ __forceinline__ UnitGeo unit_geo(const Geom &G, int w, int k) {
  UnitGeo U;
  const int ntx = G.ntx, nb = G.nb;
  const int tile = w % (ntx * nb), part = w / (ntx * nb);
  U.ox = (tile % ntx) * 64;
  const int band = tile / ntx;
  U.oy = (int)((long long)band * G.ny / nb);
  U.hb = (int)((long long)(band + 1) * G.ny / nb) - U.oy;
  U.tw = min(32, (G.nx - U.ox) / 2);
  U.zlo = (int)((long long)part * G.nz / G.zsplit);
  U.zhi = (int)((long long)(part + 1) * G.nz / G.zsplit);
  U.nzc = U.zhi - U.zlo;
  const bool down = ((part ^ k) & 1) != 0;
  U.dz = down ? -1 : 1;
  U.z0 = down ? U.zhi - 1 : U.zlo;
  return U;
}
// physical plane of logical plane L (>= -2) of a unit
__device__ __forceinline__ int plane_z(const UnitGeo &U, int nz, int L) {
  int z = (U.z0 + L * U.dz) % nz;
  return z < 0 ? z + nz : z;
}
// The TMA boxes of one plane into ring slot `slot`: which & 1: kappa, x_{k-2} (slot_pp
// >= 0), B (with the barrier's expected byte count for all boxes); which & 2: x_{k-1}.

template <int PM, int HM, int D>
__device__ __forceinline__ void issue_boxes(const Geom &G, const UnitGeo &U, int z, int slot, int slot_prev, int slot_pp,
                                            int which) {
  using C = Cfg<PM, HM, D>;
  double *sm = smem_base<PM, HM, D>();
  double *dst = sm + (size_t)slot * C::SLOT;
  uint64_t *b = bars<PM, HM, D>(sm) + slot;
  if (which & 1) {
    mbar_expect_tx(b, 2 * C::BYTES_A + (unsigned)PM * C::BYTES_B + (slot_pp >= 0 ? C::BYTES_B : 0u));
    tma_load4(dst + C::SA, G.mapA, U.ox, U.oy, z, G.slot_kappa, b);
    if (slot_pp >= 0) tma_load4(dst + 2 * C::SA, G.mapB, U.ox, U.oy + 1, z, slot_pp, b);
#pragma unroll
    for (int c = 0; c < PM; c++) tma_load4(dst + 2 * C::SA + (1 + c) * C::SB, G.mapB, U.ox, U.oy + 1, z, G.slot_B + c, b);
  }
  if (which & 2) tma_load4(dst, G.mapA, U.ox, U.oy, z, slot_prev, b);
}
// Pass-boundary prefetch (persistent loop, RC_PREFETCH): the producer issues the first
// ring planes of this CTA's first unit of pass k while pass k-1's grid reduction runs:
// which = 1 before the grid barrier (kappa, B and x_{k-2} boxes: independent of pass
// k-1), which = 2 after it (x_{k-1} boxes: pass k-1's output).  Returns the number of
// planes (identical in every thread); pre = that number in the producer thread.
template <int PM, int HM, int D>
__device__ __forceinline__ int preissue(const Geom &G, int k, int slot_prev, int slot_pp, unsigned nl, int which,
                                        int &pre) {
  using C = Cfg<PM, HM, D>;
  if ((int)blockIdx.x >= G.ntx * G.nb * G.zsplit) return 0;
  const UnitGeo U = unit_geo(G, blockIdx.x, k);
  const int n = min(C::RS, U.nzc + 4);
  if (threadIdx.x == RC3_PRODUCER) {
    for (int q = 0; q < n; q++)
      issue_boxes<PM, HM, D>(G, U, plane_z(U, G.nz, q - 2), (int)((nl + (unsigned)q) % (unsigned)C::RS), slot_prev,
                             slot_pp, which);
    pre = n;
  }
  return n;
}
// Planes pre-issued for a pass that does not take place (the Alg. 2 run ended): wait
// for them in every thread (keeps the barrier phases in step) and advance the ring.
template <int PM, int HM, int D>
__device__ __forceinline__ void drain(unsigned &nl, int n) {
  using C = Cfg<PM, HM, D>;
  uint64_t *b = bars<PM, HM, D>(smem_base<PM, HM, D>());
  for (int q = 0; q < n; q++) {
    const unsigned c = nl + (unsigned)q;
    mbar_wait(b + c % (unsigned)C::RS, (c / (unsigned)C::RS) & 1u);
  }
  nl += (unsigned)n;
}

// sum_f kappa_f (x_f - x_c) over the six faces of one point (x-, x+, y-, y+, z-, z+
// in the lazy kernels' operand order).  RC3_SPLIT: two interleaved partial sums
// (dependency depth 3 + 1 instead of 6), the same terms.
__device__ __forceinline__ double face_sum(double f0, double d0, double f1, double d1, double f2, double d2, double f3,
                                           double d3, double f4, double d4, double f5, double d5) {
#if RC3_SPLIT
  double a = f0 * d0, b = f1 * d1;
  a = fma(f2, d2, a);
  b = fma(f3, d3, b);
  a = fma(f4, d4, a);
  b = fma(f5, d5, b);
  return a + b;
#else
  double a = f0 * d0;
  a = fma(f1, d1, a);
  a = fma(f2, d2, a);
  a = fma(f3, d3, a);
  a = fma(f4, d4, a);
  return fma(f5, d5, a);
#endif
}

// sum_f kappa_f x_f over the six faces (F form: the diagonal part -(sum_f kappa_f) x_c is
// applied by the caller); two interleaved partial sums.
__device__ __forceinline__ double face_prod(double f0, double x0, double f1, double x1, double f2, double x2, double f3,
                                           double x3, double f4, double x4, double f5, double x5) {
  double a = f0 * x0, b = f1 * x1;
  a = fma(f2, x2, a);
  b = fma(f3, x3, b);
  a = fma(f4, x4, a);
  b = fma(f5, x5, b);
  return a + b;
}

// Stage-1 results of one plane at this thread's pair, carried to stage 2 of the next
// step (and its x_{k-1} / kappa centre to stage 1 of the next plane as the z-1 terms).
struct Rec {
  double2 xk, bk;     // x_k ; nu B t_k
  double fl, fi, fr;  // kappa sums of the x faces: left, inside the pair, right
  double2 fs, fn, fm; // kappa sums of the y-, y+, z- faces (per point)
  double2 xc, kc;     // x_{k-1}, kappa centre
  double2 F;          // RC3_FFORM: sum of the six face kappa sums (the stencil's diagonal, x 2)
};

// Warp roles.  Warp w runs on scheduler w % 4; interior warps run stage 1 + stage 2,
// halo warps stage 1 only (about half the work).  For HM = 7 (10 warps: 7 interior
// rows, 3 halo) the halo warps are 4, 8, 9 so that no scheduler carries more than
// I + I + H (schedulers 0-3: I H H | I I H | I I | I I), instead of three full warps
// on two of them.  Returns the interior row (>= 0) or -1 - halo warp index.
template <int HM>
__host__ __device__ constexpr int role_of(int w) {
#if RC3_ROLEMAP
  if (HM == 7) {
    return w == 4 ? -1 : w == 8 ? -2 : w == 9 ? -3 : (w < 4 ? w : w - 1);
  }
#endif
  return w < HM ? w : -1 - (w - HM);
}

// One pass over this CTA's units.  nl: planes this CTA has loaded so far (the ring's
// running fill count: slot = count % RS, phase parity = (count / RS) & 1), identical
// in every thread and carried across passes by the caller.
//
// UR: k >= 2 (x_k is formed from the recomputed r_{k-1}); UPP: k >= 3 (x_{k-2} term).
// Every thread runs both stages on every plane with no data-dependent branches (threads
// without a pair read a valid dummy location and write a dummy exchange slot; halo
// threads' stage-2 results are discarded), so stage 1 of plane L and stage 2 of plane
// L-1 form ONE basic block the compiler can interleave.
template <int PM, int HM, int D, bool UR, bool UPP>
__device__ __forceinline__ void march(const Geom &G, const PassArgs<PM> &Q, double (&v)[5], unsigned &nl, int &pre) {
  using C = Cfg<PM, HM, D>;
  constexpr int W = C::W, SA = C::SA, SB = C::SB, SLOT = C::SLOT, RS = C::RS, EXP = C::EXP;
  double *const sm = smem_base<PM, HM, D>();
  double2 *const ex = reinterpret_cast<double2 *>(sm + (size_t)RS * SLOT);
  uint64_t *const bar = bars<PM, HM, D>(sm);
  const int t = threadIdx.x, lane = t & 31;
  const int nx = G.nx, ny = G.ny, nz = G.nz, ntx = G.ntx, nb = G.nb;
  const int units = ntx * nb * G.zsplit;
  const long long plane = (long long)G.Xp * G.Yp;
  const double a0 = Q.a0, a1 = Q.a1, a2 = Q.a2, hh = G.hh;
  double btp[PM > 0 ? PM : 1], btc[PM > 0 ? PM : 1];
#pragma unroll
  for (int c = 0; c < PM; c++) {
    btp[c] = Q.btp[c];
    btc[c] = Q.btc[c];
  }
  double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0, v4 = 0.0;

  for (int w = blockIdx.x; w < units; w += gridDim.x) {
    const int tile = w % (ntx * nb), part = w / (ntx * nb);
    const int ox = (tile % ntx) * 64, band = tile / ntx;
    const int oy = (int)((long long)band * ny / nb), hb = (int)((long long)(band + 1) * ny / nb) - oy;
    const int tw = min(32, (nx - ox) / 2);
    const int zlo = (int)((long long)part * nz / G.zsplit), zhi = (int)((long long)(part + 1) * nz / G.zsplit);
    const int nzc = zhi - zlo;
    const bool down = ((part ^ Q.k) & 1) != 0;
    // thread -> pair (px, py) of the halo-1 plane: px 0..tw+1, py 0..hb+1; interior pairs
    // (1..tw, 1..hb) in full warps (one warp per row), the halo ring after them
    int px = -1, py = -1;
    bool s2 = false;
    const int wr = role_of<HM>(t >> 5);  // >= 0: interior row; < 0: halo warp -1 - index
    const bool hwarp = wr < 0;
    if (!hwarp) {
      if (wr < hb && lane < tw) {
        px = 1 + lane;
        py = 1 + wr;
        s2 = true;
      }
    } else {
      int h = (-1 - wr) * 32 + lane;
      const int rw = tw + 2;
      if (h < rw) { px = h; py = 0; }
      else if ((h -= rw) < rw) { px = h; py = hb + 1; }
      else if ((h -= rw) < hb) { px = 0; py = 1 + h; }
      else if ((h -= hb) < hb) { px = tw + 1; py = 1 + h; }
    }
    const bool s1 = px >= 0;
    // threads without a pair compute on pair (1, 1) and publish into the pad slot EXP
    const int qx = s1 ? px : 1, qy = s1 ? py : 1;
    const int offA = (qy + 1) * W + 2 * qx, offB = qy * W + 2 * qx;
    const int ew = s1 ? qy * 34 + qx : EXP, er = s2 ? ew : 35;
    RC3_ASSERT(offA - W >= 0 && offA - 1 >= 0 && offA + W + 1 < C::RA * W);  // halo-2 box: x +-1, y +-1
    RC3_ASSERT(offB >= 0 && offB + 1 < C::RB * W);
    RC3_ASSERT(ew >= 0 && ew < EXP + 32 && er - 34 >= 0 && er + 34 < EXP && er - 1 >= 0);
    RC3_ASSERT(qx <= 33 && qy <= HM + 1);
    // x-neighbour values from the neighbouring lanes when they hold the adjacent pair
    const int key = s1 ? py * 64 + px : -1000 - t;
    const int kl = __shfl_up_sync(0xffffffffu, key, 1), kr = __shfl_down_sync(0xffffffffu, key, 1);
    const bool shl = lane > 0 && s1 && kl == key - 1, shr = lane < 31 && s1 && kr == key + 1;
    // padded-plane offsets of this pair and of its periodic ghost images (interior pairs)
    const int gx = ox - 2 + 2 * qx, gy = oy - 1 + qy;
    const int o0 = (gx + 2) + G.Xp * (gy + 2);  // (a padded plane has < 2^31 points)
    int og0 = -1, og1 = -1, og2 = -1;
    if (s2) {
      const int gxg = gx < 2 ? gx + nx : (gx >= nx - 2 ? gx - nx : -99);
      const int gyg = gy < 2 ? gy + ny : (gy >= ny - 2 ? gy - ny : -99);
      if (gxg != -99) og0 = (gxg + 2) + G.Xp * (gy + 2);
      if (gyg != -99) og1 = (gx + 2) + G.Xp * (gyg + 2);
      if (gxg != -99 && gyg != -99) og2 = (gxg + 2) + G.Xp * (gyg + 2);
    }
    const bool st = s2 && Q.xout != nullptr;
    const int dz = down ? -1 : 1;
    auto wrapz = [&](int z) { return z < 0 ? z + nz : (z >= nz ? z - nz : z); };
    const UnitGeo U = unit_geo(G, w, Q.k);
    const int z0 = U.z0;
    const int last = nzc + 1;  // logical planes -2 .. nzc+1
    // producer: next plane to issue, its slot and physical plane; the first `pre` planes
    // of the CTA's first unit may have been issued by preissue() already
    const bool prod = t == RC3_PRODUCER;
    const int npre = (prod && w == (int)blockIdx.x) ? pre : 0;
    int iL = -2 + npre, isl = (int)((nl + (unsigned)npre) % (unsigned)RS), iz = plane_z(U, nz, -2 + npre);
    auto issue = [&]() {
      RC3_ASSERT(iz >= 0 && iz < nz && isl >= 0 && isl < RS && iL >= -2 && iL <= last);
      issue_boxes<PM, HM, D>(G, U, iz, isl, Q.slot_prev, UPP ? Q.slot_pp : -1, 3);
      iL++;
      isl = isl + 1 == RS ? 0 : isl + 1;
      iz = wrapz(iz + dz);
    };
    __syncthreads();  // the previous unit / pass is done with the ring and the exchange
    if (prod) {
      pre = 0;
      for (int q = npre; q < RS && iL <= last; q++) issue();
    }
    // consumer ring position: slot / parity of the plane to wait for next (plane -2)
    int wsl = (int)(nl % (unsigned)RS);
    unsigned wpar = (nl / (unsigned)RS) & 1u;
    auto wait_next = [&]() -> int {
      const int s = wsl;
      mbar_wait(bar + s, wpar);
      wsl = wsl + 1 == RS ? 0 : wsl + 1;
      if (wsl == 0) wpar ^= 1u;
      return s;
    };
    // prologue: plane -2 (x_{k-1}, kappa centre below the first stage-1 plane), plane -1
    const int sm2 = wait_next();
    int sl = wait_next();  // slot of the stage-1 plane L (= -1 at step 0)
    Rec ra, rb;            // ra: plane L-1 at even steps; rb: at odd steps (ping-pong)
    ra.xc = ld2(sm + (size_t)sm2 * SLOT + offA);
    ra.kc = ld2(sm + (size_t)sm2 * SLOT + SA + offA);
    ra.xk = ra.bk = ra.fs = ra.fn = ra.fm = make_double2(0.0, 0.0);
    ra.fl = ra.fi = ra.fr = 0.0;
    ra.F = make_double2(0.0, 0.0);
    rb = ra;
    double2 xq = ld2(sm + (size_t)sl * SLOT + offA), kq = ld2(sm + (size_t)sl * SLOT + SA + offA);  // centre of plane L
    __syncthreads();
    if (prod && iL <= last) issue();  // into the slot of plane -2
    int zo = z0;                        // physical plane of the stage-2 output (logical L-1)

    // one step: stage 1 on plane L = i-1 (into cu, which held plane L-2), stage 2 on
    // plane L-1 (pv) when S2
    auto step = [&](auto s2tag, int i, Rec &pv, Rec &cu) {
      constexpr bool S2 = decltype(s2tag)::value;
      const int sq = wait_next();  // plane L+1
      const double *Xs = sm + (size_t)sl * SLOT, *Xq = sm + (size_t)sq * SLOT;
      // ---- stage 1, plane L
      const double *XL = Xs + offA, *KL = Xs + SA + offA, *BL = Xs + 2 * SA + SB + offB;
      const double2 xc = xq, kc = kq;
      const double2 xqn = ld2(Xq + offA), kqn = ld2(Xq + SA + offA);
      const double2 ks = ld2(KL - W), kn = ld2(KL + W);
      double kl = __shfl_up_sync(0xffffffffu, kc.y, 1), kr = __shfl_down_sync(0xffffffffu, kc.x, 1);
      if (!shl) kl = KL[-1];
      if (!shr) kr = KL[2];
      const double fl = kc.x + kl, fi = kc.x + kc.y, fr = kc.y + kr;
      const double2 fs = make_double2(kc.x + ks.x, kc.y + ks.y), fn = make_double2(kc.x + kn.x, kc.y + kn.y);
      const double2 fm = make_double2(kc.x + pv.kc.x, kc.y + pv.kc.y), fp = make_double2(kc.x + kqn.x, kc.y + kqn.y);
      double2 xk = xc;
      double2 Fn = make_double2(0.0, 0.0);  // RC3_FFORM: face-sum diagonal of plane L
#if RC3_FFORM
      if (!UR)  // (k = 1: no stage-1 stencil, but stage 2 of the next plane needs F)
        Fn = make_double2(((fl + fi) + (fs.x + fn.x)) + (fm.x + fp.x), ((fr + fi) + (fs.y + fn.y)) + (fm.y + fp.y));
#endif
      if (UR) {
        const double2 xs = ld2(XL - W), xn = ld2(XL + W);
        double xl = __shfl_up_sync(0xffffffffu, xc.y, 1), xr = __shfl_down_sync(0xffffffffu, xc.x, 1);
        if (!shl) xl = XL[-1];
        if (!shr) xr = XL[2];
        double2 bt = {0.0, 0.0};
#pragma unroll
        for (int c = 0; c < PM; c++) {
          const double2 b = ld2(BL + c * SB);
          bt.x = fma(b.x, btp[c], bt.x);
          bt.y = fma(b.y, btp[c], bt.y);
        }
        const double2 xm = pv.xc;
#if RC3_FFORM
        Fn = make_double2(((fl + fi) + (fs.x + fn.x)) + (fm.x + fp.x), ((fr + fi) + (fs.y + fn.y)) + (fm.y + fp.y));
        const double ra_ = fma(-Fn.x, xc.x, face_prod(fl, xl, fi, xc.y, fs.x, xs.x, fn.x, xn.x, fm.x, xm.x, fp.x, xqn.x));
        const double rb_ = fma(-Fn.y, xc.y, face_prod(fr, xr, fi, xc.x, fs.y, xs.y, fn.y, xn.y, fm.y, xm.y, fp.y, xqn.y));
#else
        const double ra_ = face_sum(fl, xl - xc.x, fi, xc.y - xc.x, fs.x, xs.x - xc.x, fn.x, xn.x - xc.x, fm.x,
                                    xm.x - xc.x, fp.x, xqn.x - xc.x);
        const double rb_ = face_sum(fr, xr - xc.y, fi, xc.x - xc.y, fs.y, xs.y - xc.y, fn.y, xn.y - xc.y, fm.y,
                                    xm.y - xc.y, fp.y, xqn.y - xc.y);
#endif
        const double r0 = fma(ra_, hh, bt.x), r1 = fma(rb_, hh, bt.y);
        xk.x = a0 * r0 - a1 * xc.x;
        xk.y = a0 * r1 - a1 * xc.y;
        if (UPP) {
          const double2 pp = ld2(Xs + 2 * SA + offB);
          xk.x -= a2 * pp.x;
          xk.y -= a2 * pp.y;
        }
      }
      double2 bk = {0.0, 0.0};
#pragma unroll
      for (int c = 0; c < PM; c++) {
        const double2 b = ld2(BL + c * SB);
        bk.x = fma(b.x, btc[c], bk.x);
        bk.y = fma(b.y, btc[c], bk.y);
      }
      ex[(i & 1) * (EXP + 32) + ew] = xk;
      // ---- stage 2, plane L-1: r_k = A x_k + nu B t_k, dots, store x_k
      if (S2) {
        const double2 *E = ex + ((i - 1) & 1) * (EXP + 32);
        const double2 c0 = pv.xk, xkm = cu.xk;  // x_k at L-1, L-2
        double xl = __shfl_up_sync(0xffffffffu, c0.y, 1), xr = __shfl_down_sync(0xffffffffu, c0.x, 1);
        if (!shl) xl = E[er - 1].y;
        if (!shr) xr = E[er + 1].x;
        const double2 xs = E[er - 34], xn = E[er + 34];
        // (the upper face of plane L-1 is the lower face fm of plane L)
#if RC3_FFORM
        const double ra_ = fma(-pv.F.x, c0.x, face_prod(pv.fl, xl, pv.fi, c0.y, pv.fs.x, xs.x, pv.fn.x, xn.x, pv.fm.x,
                                                        xkm.x, fm.x, xk.x));
        const double rb_ = fma(-pv.F.y, c0.y, face_prod(pv.fr, xr, pv.fi, c0.x, pv.fs.y, xs.y, pv.fn.y, xn.y, pv.fm.y,
                                                        xkm.y, fm.y, xk.y));
#else
        const double ra_ = face_sum(pv.fl, xl - c0.x, pv.fi, c0.y - c0.x, pv.fs.x, xs.x - c0.x, pv.fn.x, xn.x - c0.x,
                                    pv.fm.x, xkm.x - c0.x, fm.x, xk.x - c0.x);
        const double rb_ = face_sum(pv.fr, xr - c0.y, pv.fi, c0.x - c0.y, pv.fs.y, xs.y - c0.y, pv.fn.y, xn.y - c0.y,
                                    pv.fm.y, xkm.y - c0.y, fm.y, xk.y - c0.y);
#endif
        const double r0 = fma(ra_, hh, pv.bk.x), r1 = fma(rb_, hh, pv.bk.y);
        const double2 xm = pv.xc;  // x_{k-1} at L-1
        const double d0 = fma(c0.x, c0.x, c0.y * c0.y), d1 = fma(xm.x, c0.x, xm.y * c0.y);
        const double d2 = fma(xm.x, r0, xm.y * r1), d3 = fma(c0.x, r0, c0.y * r1), d4 = fma(r0, r0, r1 * r1);
        if (s2) {
          v0 += d0; v1 += d1; v2 += d2; v3 += d3; v4 += d4;
        }
        if (st) {
          RC3_ASSERT(zo >= 0 && zo < nz && o0 >= 0 && o0 + 1 < plane && og0 + 1 < plane && og1 + 1 < plane &&
                     og2 + 1 < plane);
          double *xo = Q.xout + (long long)zo * plane;
          *reinterpret_cast<double2 *>(xo + o0) = c0;
          if (og0 >= 0) *reinterpret_cast<double2 *>(xo + og0) = c0;
          if (og1 >= 0) *reinterpret_cast<double2 *>(xo + og1) = c0;
          if (og2 >= 0) *reinterpret_cast<double2 *>(xo + og2) = c0;
        }
        zo = wrapz(zo + dz);
      }
      cu.xk = xk; cu.bk = bk;
      cu.fl = fl; cu.fi = fi; cu.fr = fr;
      cu.fs = fs; cu.fn = fn; cu.fm = fm;
      cu.xc = xc; cu.kc = kc;
      cu.F = Fn;
      xq = xqn;
      kq = kqn;
      sl = sq;
      __syncthreads();  // slot of plane L and exchange (i-1)&1 fully read
      if (prod && iL <= last) issue();  // plane L + RS into the slot of plane L
    };
    using F = std::integral_constant<bool, false>;
    using T = std::integral_constant<bool, true>;
    // steps i = 0 .. nzc+1: stage 2 from i = 2; ra holds plane L-1 at even i
    step(F{}, 0, ra, rb);
    step(F{}, 1, rb, ra);
    int i = 2;
    for (; i + 1 <= last; i += 2) {
      step(T{}, i, ra, rb);
      step(T{}, i + 1, rb, ra);
    }
    if (i <= last) step(T{}, i, ra, rb);
    nl += (unsigned)(nzc + 4);
  }
  // the stage-2 sums use v += d (not fma chains) -- same values as the fma form up to rounding
  v[0] += v0; v[1] += v1; v[2] += v2; v[3] += v3; v[4] += v4;
}

template <int PM, int HM, int D>
__device__ __forceinline__ void body(const Geom &G, const PassArgs<PM> &Q, double (&v)[5], unsigned &nl, int &pre) {
  if (Q.slot_pp >= 0)
    march<PM, HM, D, true, true>(G, Q, v, nl, pre);
  else if (Q.use_r)
    march<PM, HM, D, true, false>(G, Q, v, nl, pre);
  else
    march<PM, HM, D, false, false>(G, Q, v, nl, pre);
}

}  // namespace rc3
