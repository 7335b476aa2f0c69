// AMR cell-level FMM gravity over a forest (rows a12/a13 of SURVEY.md §8).
//
// Our specification (the reference has no gravity code), restated
// in oracle/gravity_amr_oracle.c and matched bitwise (-fmad=false): the
// classic adaptive FMM (U, V, W, X lists) on the cell tree of the forest,
// with the operators of the uniform solver (gravity_common.cuh). Layout: every
// forest node (leaf or internal) at level l is one 8^3 patch of cells at cell
// depth l + 3, AoS [node*512 + (k*8+j)*8+i][10] moments / locals per level;
// cell depths 0..2 are three tiny dense levels above the root patch.
//
//   amr_p2m     leaf cells: (m, 0, 0)                      one launch
//   amr_m2m     internal patches from their 8 child patches, per level
//   dense       depths 2..0: M2M, depth-2 M2L, depth-3 L2L (uniform kernels)
//   amr_m2l     per level, 4 CTAs per patch (8x4x4 targets each): the 12x8x8
//               source window gathered from the 27 neighbour patches into
//               shared memory (missing neighbours = zero moments), the 189-cell
//               V stencil with tabulated geometry, then the
//               target's W/X pairs (CSR) — fused, one write of the locals
//   amr_l2l     per level, parent local shifted + own M2L sum
//   amr_l2p     leaf cells: L2P + same-depth P2P over the 26 neighbours that
//               are leaf cells + cross-depth U pairs (CSR)
//   am_*        angular-momentum correction (our rigid-rotation
//               specification, tmo_grav_am_correct): per-slot adjacent-pair
//               tree (shuffles + shared memory), one-CTA tree over slots,
//               3x3 solve, apply
#include <algorithm>
#include <type_traits>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "comm.h"
#include "gravity_amr_plan.h"
#include "gravity_common.cuh"
#include "peer.cuh"

namespace tmgpu {

struct GLv {
  double* mom;
  double* loc;
  const int* ijk;
  const int* nbr;
  const int* child;
  const int* parent;
  const int* leaf_slot;
  const long long* moff;
  const long long* ment;
  const long long* poff;
  const long long* pent;
  const int* mgeo;  // W/X entry -> row of the W/X geometry table
  const int* pgeo;  // cross-depth U entry -> row of the P2P geometry table
  double* unm;      // cross-depth U entry -> -(source mass), gathered per solve (amr_u_gather_kernel)
  long long nu;     // cross-depth U entries of this level
  // leaf-mass indices (slot * 512 + cell, global slots) of the W/X entries
  // whose source is a leaf cell (-1 otherwise) and of the U entries: with the
  // leaf-mass array these replace the moment arrays' m of leaf cells (one GPU)
  const int* mmi;
  const int* pmi;
};

// P2P geometry of the 26 same-depth lattice offsets at unit spacing (depth 0):
// at depth d the table is this one scaled exactly by 2^d (1/r) and 2^2d
// (R/r^3) — every operation of p2p_geom commutes with power-of-two scaling —
// so L2P scales the neighbour masses instead and reads the geometry from the
// constant bank (no shared-memory traffic)
__constant__ double c_p2p_unit[27][4];
// cell volume h^3 of a level-l leaf patch's cells (h = 1 / (8 * 2^l), a power of
// two: exact however computed), for the masses m = rho * h^3
constexpr int kMaxLevels = 48;
__constant__ double c_level_dv[kMaxLevels];

namespace {

// ((double)gi + 0.5) / 2^d as the oracle writes it; dividing by a power of two
// is exact, so multiplying by the exact 2^-d gives the same bits without a
// division sequence
__device__ __forceinline__ double centre(long long gi, int d) {
  return ((double)gi + 0.5) * __longlong_as_double((long long)(1023 - d) << 52);
}

// arena slots 0..nslots-1 are the canonical slots lo.. (distributed: the owned range)
// V > 0: density from a ghosted arena [slot][V][12^3]; V == 0: from a compact
// density at slot stride cstride (the stage's provisional density [slot][512],
// 6-solve cadence; or var 0 of compact interiors [slot][V][512])
__global__ void amr_mass_kernel(const double* __restrict__ arena, int V, long long nslots,
                                long long lo, const int* __restrict__ slot_level,
                                double* __restrict__ mass, long long cstride = 512) {
  const long long total = nslots * 512;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long s = t >> 9;
    const int c = (int)(t & 511);
    const int i = c & 7, j = (c >> 3) & 7, k = c >> 6;
    const double dV = c_level_dv[slot_level[lo + s]];
    const double rho = V ? arena[s * V * 1728 + ((k + 2) * 12 + (j + 2)) * 12 + (i + 2)] : arena[s * cstride + c];
    mass[lo * 512 + t] = rho * dV;
  }
}

// leaf cells: moments (m, 0, ..., 0). The moment arrays are zeroed when the
// solver is created and nothing writes a leaf patch's D and Q afterwards (M2M
// writes internal patches; received patches arrive with their owner's +0s),
// so P2M stores only m; slots lo .. lo+nslots
__global__ void amr_p2m_kernel(const double* __restrict__ mass, long long nslots, long long lo,
                               const int* __restrict__ slot_level, const int* __restrict__ slot_node,
                               const GLv* __restrict__ L) {
  const long long total = nslots * 512;
  for (long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x; u < total;
       u += (long long)gridDim.x * blockDim.x) {
    const long long t = lo * 512 + u;
    const long long s = t >> 9;
    const int c = (int)(t & 511);
    L[slot_level[s]].mom[((long long)slot_node[s] * 512 + c) * 10] = mass[t];
  }
}

// LET moment exchange: whole patches (512 cells x 10 moments) between the
// moment arrays and a contiguous buffer (block j of `list` <-> buffer block
// blk ? blk[j] : j); one CTA per patch
__global__ void pack_patches_kernel(const GLv* __restrict__ Lv, const int2* __restrict__ list,
                                    const int* __restrict__ blk, double* __restrict__ buf) {
  const int2 p = list[blockIdx.x];
  const double2* src = reinterpret_cast<const double2*>(Lv[p.x].mom + (long long)p.y * 5120);
  double2* dst = reinterpret_cast<double2*>(buf + (long long)(blk ? blk[blockIdx.x] : blockIdx.x) * 5120);
  for (int q = threadIdx.x; q < 2560; q += blockDim.x) dst[q] = src[q];
}

__global__ void unpack_patches_kernel(const GLv* __restrict__ Lv, const int2* __restrict__ list,
                                      const int* __restrict__ blk, const double* __restrict__ buf) {
  const int2 p = list[blockIdx.x];
  const double2* src =
      reinterpret_cast<const double2*>(buf + (long long)(blk ? blk[blockIdx.x] : blockIdx.x) * 5120);
  double2* dst = reinterpret_cast<double2*>(Lv[p.x].mom + (long long)p.y * 5120);
  for (int q = threadIdx.x; q < 2560; q += blockDim.x) dst[q] = src[q];
}

// masses of received leaf patches (their P2P sources) from their monopoles
__global__ void halo_mass_kernel(const GLv* __restrict__ Lv, const int* __restrict__ slots, long long n,
                                 const int* __restrict__ slot_level, const int* __restrict__ slot_node,
                                 double* __restrict__ mass) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n * 512;
       t += (long long)gridDim.x * blockDim.x) {
    const int s = slots[t >> 9], c = (int)(t & 511);
    mass[(long long)s * 512 + c] = Lv[slot_level[s]].mom[((long long)slot_node[s] * 512 + c) * 10];
  }
}

// mass (one GPU, else null): leaf children's m from the leaf-mass array
// (the same values P2M would store, read coalesced)
__global__ void amr_m2m_kernel(const GLv* __restrict__ L, int l, const int* __restrict__ internal,
                               long long n_int, const double* __restrict__ mass = nullptr) {
  const GLv P = L[l], Ch = L[l + 1];
  const double hc = 1.0 / (double)(1LL << (l + 4));
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n_int * 512;
       t += (long long)gridDim.x * blockDim.x) {
    const int n = internal[t >> 9];
    const int c = (int)(t & 511);
    const int I = c & 7, J = (c >> 3) & 7, K = c >> 6;
    const int cn = P.child[n * 8 + ((K >> 2) * 2 + (J >> 2)) * 2 + (I >> 2)];
    const double* base = Ch.mom + (long long)cn * 512 * 10;
    double o[10];
#pragma unroll
    for (int q = 0; q < 10; ++q) o[q] = 0.0;
    const int lsl = Ch.leaf_slot[cn];
    if (lsl >= 0) {
      // leaf child cells carry (m, +0, ..., +0): read only m. Dropping the +0
      // terms can only turn a +0 term into -0, and a sum started at +0 is the
      // same either way, so the result is tmo_grav_m2m's bit for bit.
      // the 8 children's masses loaded together (one round trip), then summed in order
      double Ms[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int a = q & 1, b = (q >> 1) & 1, cc = q >> 2;
        const int cc8 = ((((2 * K) & 7) + cc) * 8 + ((2 * J) & 7) + b) * 8 + ((2 * I) & 7) + a;
        Ms[q] = mass ? mass[(long long)lsl * 512 + cc8] : base[cc8 * 10];
      }
#pragma unroll
      for (int cc = 0; cc < 2; ++cc)
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
          for (int a = 0; a < 2; ++a) {
            const double s[3] = {(a - 0.5) * hc, (b - 0.5) * hc, (cc - 0.5) * hc};
            const double M = Ms[(cc * 2 + b) * 2 + a];
            o[0] += M;
#pragma unroll
            for (int i = 0; i < 3; ++i) o[1 + i] += M * s[i];
#pragma unroll
            for (int i = 0; i < 3; ++i)
#pragma unroll
              for (int j = i; j < 3; ++j) o[4 + s2(i, j)] += M * s[i] * s[j];
          }
      double2* out = reinterpret_cast<double2*>(P.mom + ((long long)n * 512 + c) * 10);
#pragma unroll
      for (int h = 0; h < 5; ++h) out[h] = make_double2(o[2 * h], o[2 * h + 1]);
      continue;
    }
    // the 8 children's 80-byte records (five 16-byte loads each) loaded
    // together, then summed in order
    double2 rec[8][5];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int a = q & 1, b = (q >> 1) & 1, cc = q >> 2;
      const double2* c2 = reinterpret_cast<const double2*>(
          base + (((((2 * K) & 7) + cc) * 8 + ((2 * J) & 7) + b) * 8 + ((2 * I) & 7) + a) * 10);
#pragma unroll
      for (int h = 0; h < 5; ++h) rec[q][h] = c2[h];
    }
#pragma unroll
    for (int cc = 0; cc < 2; ++cc)
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int a = 0; a < 2; ++a) {
          const double s[3] = {(a - 0.5) * hc, (b - 0.5) * hc, (cc - 0.5) * hc};
          double ch[10];
#pragma unroll
          for (int h = 0; h < 5; ++h) {
            ch[2 * h] = rec[(cc * 2 + b) * 2 + a][h].x;
            ch[2 * h + 1] = rec[(cc * 2 + b) * 2 + a][h].y;
          }
          const double M = ch[0];
          o[0] += M;
#pragma unroll
          for (int i = 0; i < 3; ++i) o[1 + i] += ch[1 + i] + M * s[i];
#pragma unroll
          for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = i; j < 3; ++j)
              o[4 + s2(i, j)] += ch[4 + s2(i, j)] + ch[1 + i] * s[j] + s[i] * ch[1 + j] + M * s[i] * s[j];
        }
    double2* out = reinterpret_cast<double2*>(P.mom + ((long long)n * 512 + c) * 10);
#pragma unroll
    for (int h = 0; h < 5; ++h) out[h] = make_double2(o[2 * h], o[2 * h + 1]);
  }
}

// ---- M2L, all levels in one launch -----------------------------------------
// CTA = one patch (8^3 targets), 256 threads, one CTA per SM (197 KB smem).
// Warp w = target parity class (b, c) = (w & 1, w >> 1 & 1) in y, z and source
// half h = w >> 2 (the lower / upper three source planes of the spec's two
// partial sums); lane = (a, Y, Z) = (lane & 1, lane >> 1 & 3, lane >> 3): the
// thread owns the four targets x = a + 2k (k = 0..3), y = 2Y + b, z = 2Z + c,
// over its half of the source planes. All 8 siblings of a
// parent share the 6x6x6 children of the parent's neighbours as sources (the
// 189-cell list is that box minus the target's 27 near cells), so per source
// row (dy, dz) — warp-uniform — the thread keeps the geometry of its six x
// offsets in registers (G[jj], jj = j + 2, dx = j - a) and streams the row's 12
// sources once, applying each to every target k with jj = sx - 2k in [0, 5]:
// ~1.3 shared loads per interaction instead of 20. In the nine near rows the
// offsets j = 0, 1 (near for both a) are skipped; j = -1 (a = 0) and j = 2
// (a = 1) use zeroed near geometry: an exact no-op, because a sum that starts
// at +0 never becomes -0 and x + (+-0) = x (finite moments).
// Window: 12^3 sources (27-patch neighbourhood; missing patches are zero
// moments) filled by cp.async, split into 4 (y, z)-parity sub-grids of 6 x 6
// rows of 12 with pitches 13 / 84: a warp's 16 distinct source addresses
// (Y, Z) fall in 16 distinct bank pairs.
// Accumulation per target: two partial sums (lower / upper source planes),
// dz, dy, dx ascending, added; the W/X pairs follow in amr_wx_kernel —
// tmo_grav_amr_solve's order, so the result is bitwise the oracle's.
constexpr int kM2lThreads = 256;
constexpr int kWPY = 13, kWPZ = 84, kWSub = 6 * kWPZ;  // the mono kernel's mass window
// The fused kernel's window: one 80-byte record (the 10 moments, as the global
// AoS layout) per source cell, addressed in 16-byte chunks: rows of 12 records
// at a pitch of 65 chunks (= 1 mod 8), 6 rows per z plane of a parity sub-grid
// at 396 chunks (= 4 mod 8) — a warp's 16 distinct (Y, Z) sources then fill the
// eight 16-byte bank groups exactly twice (conflict-free LDS.128), and the fill
// copies 16-byte chunks.
constexpr int kFRec = 5, kFPY = 65, kFPZ = 396, kFSub = 6 * kFPZ;  // chunks
constexpr int kWinDoubles = 2 * 4 * kFSub;                          // 19,008
constexpr int kTabP = 14;  // shared-memory table entry: 13 doubles + pad (16-byte rows)
constexpr int kTabDoubles = kOff3 * kTabP;                                // 4,802
constexpr size_t kM2lSmem = (size_t)(kWinDoubles + kTabDoubles) * sizeof(double);  // 199,856 B

// One V-list term (m2l_acc's operations) with raw window moments; NOUT = 4
// drops the L_ij terms (leaf targets: the other components are unaffected).
template <int NOUT>
__device__ __forceinline__ void m2l_term(const double (&m)[10], const double (&e)[kTab], double (&o)[10]) {
  const double nM = -m[0];
  double t = nM * e[0];
  t = fma(m[1], e[1], t);
  t = fma(m[2], e[2], t);
  t = fma(m[3], e[3], t);
  t = fma(-m[4], e[10], t);
  t = fma(-m[5], e[5], t);
  t = fma(-m[6], e[6], t);
  t = fma(-m[7], e[11], t);
  t = fma(-m[8], e[8], t);
  t = fma(-m[9], e[12], t);
  o[0] = o[0] + t;
  o[1] = fma(m[3], e[6], fma(m[2], e[5], fma(m[1], e[4], fma(nM, e[1], o[1]))));
  o[2] = fma(m[3], e[8], fma(m[2], e[7], fma(m[1], e[5], fma(nM, e[2], o[2]))));
  o[3] = fma(m[3], e[9], fma(m[2], e[8], fma(m[1], e[6], fma(nM, e[3], o[3]))));
#pragma unroll
  for (int q = 0; q < NOUT - 4; ++q) o[4 + q] = fma(nM, e[4 + q], o[4 + q]);
}

// One source row, in the specification's order per target: the sources with
// even window x first, then odd (dx ascending within each). Per parity pass
// the three x-offsets' geometry (39 registers) is loaded once and the row's six
// sources of that parity are streamed once, each applied to every target it
// reaches (jj = sx - 2k in {pe, pe+2, pe+4}): ~6 shared loads per interaction.
// Near rows skip jj = 2, 3 (near for both x parities); jj = 1 (a = 0) and
// jj = 4 (a = 1) use zeroed near geometry (exact no-ops, see above).
// The same term for a source whose D and Q are +0 (a leaf cell, or a missing
// cell's zero moments): every dropped operation is an exact no-op (see
// amr_m2l_mono_kernel), so this is m2l_term's result bit for bit.
template <int NOUT>
__device__ __forceinline__ void m2l_term_mono(const double nM, const double (&e)[kTab], double (&o)[10]) {
  o[0] = o[0] + nM * e[0];
  o[1] = fma(nM, e[1], o[1]);
  o[2] = fma(nM, e[2], o[2]);
  o[3] = fma(nM, e[3], o[3]);
#pragma unroll
  for (int q = 0; q < NOUT - 4; ++q) o[4 + q] = fma(nM, e[4 + q], o[4 + q]);
}

// full[0..2]: does any lane of the warp take a source of this row from an
// internal patch at x-offset -1, 0, +1 (warp votes; a warp whose sources in a
// group are all leaf cells runs the monopole term for the group)
template <bool NEAR, int NOUT>
__device__ __forceinline__ void m2l_row_par(const double2* __restrict__ src,
                                            const double* __restrict__ trow, double (&acc)[4][10],
                                            const bool (&full)[3]) {
#pragma unroll
  for (int pe = 0; pe < 2; ++pe) {
    double G[3][kTab];
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      if (NEAR && t == 1) continue;
      const int jj = pe + 2 * t;
      const double2* t2 = reinterpret_cast<const double2*>(trow + jj * kTabP);
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        const double2 v = t2[q];
        G[t][2 * q] = v.x;
        G[t][2 * q + 1] = v.y;
      }
      G[t][12] = trow[jj * kTabP + 12];
    }
    // sources in x-groups sharing a neighbour patch (mi = 0 | 1..4 | 5):
    // one branch per group, so a group's independent term chains share a
    // basic block (the scheduler overlaps them); per target the sources still
    // arrive in ascending mi
    auto group = [&](auto lo_c, auto hi_c, bool f) {
      constexpr int lo = decltype(lo_c)::value, hi = decltype(hi_c)::value;
      if (f) {
#pragma unroll
        for (int mi = lo; mi <= hi; ++mi) {
          const int sx = pe + 2 * mi;
          double m[10];
#pragma unroll
          for (int q = 0; q < kFRec; ++q) {
            const double2 v = src[sx * kFRec + q];
            m[2 * q] = v.x;
            m[2 * q + 1] = v.y;
          }
#pragma unroll
          for (int t = 0; t < 3; ++t) {
            const int k = mi - t;
            if (k < 0 || k > 3) continue;
            if (NEAR && t == 1) continue;
            m2l_term<NOUT>(m, G[t], acc[k]);
          }
        }
      } else {
#pragma unroll
        for (int mi = lo; mi <= hi; ++mi) {
          const double nM = -reinterpret_cast<const double*>(src + (pe + 2 * mi) * kFRec)[0];
#pragma unroll
          for (int t = 0; t < 3; ++t) {
            const int k = mi - t;
            if (k < 0 || k > 3) continue;
            if (NEAR && t == 1) continue;
            m2l_term_mono<NOUT>(nM, G[t], acc[k]);
          }
        }
      }
    };
    group(std::integral_constant<int, 0>{}, std::integral_constant<int, 0>{}, full[0]);
    group(std::integral_constant<int, 1>{}, std::integral_constant<int, 4>{}, full[1]);
    group(std::integral_constant<int, 5>{}, std::integral_constant<int, 5>{}, full[2]);
  }
}

__device__ __forceinline__ void cp_async16(double* smem, const double* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}

// 16 bytes of which the first `bytes` (0, 8 or 16) are copied, the rest zero-filled
__device__ __forceinline__ void cp_async16n(double* smem, const double* gmem, int bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(bytes) : "memory");
}

// 16 bytes, zero-filled when !valid
__device__ __forceinline__ void cp_async16z(double* smem, const double* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(valid ? 16 : 0)
               : "memory");
}

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem),
               "r"(valid ? 8 : 0)
               : "memory");
}

// V-list sums of one patch from the staged window: NOUT = 10 (internal
// patch, all locals into loc[node]) or 4 (leaf patch: L0, L_i into the
// compact leaf locals [4][512]).
template <int NOUT>
__device__ __forceinline__ void m2l_patch(double* __restrict__ win, const double* __restrict__ tabs,
                                          double* __restrict__ loc, int n, double* __restrict__ lloc,
                                          unsigned internal27) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = warp & 1, c = (warp >> 1) & 1, half = warp >> 2;
  const int a = lane & 1, Y = (lane >> 1) & 3, Z = lane >> 3;
  double acc[4][10];
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int q = 0; q < 10; ++q) acc[k][q] = 0.0;
  // table row base of this lane's x parity: entry (dx + 3) = jj + 1 - a
  const double* tab_lane = tabs + (1 - a) * kTabP;
  // this warp's half of the source planes: iz = dz + 2 + c in [3 half, 3 half + 2]
  for (int iz = 3 * half; iz < 3 * half + 3; ++iz) {
    const int dz = iz - 2 - c;
    for (int iy = 0; iy < 6; ++iy) {
      const int dy = iy - 2 - b;
      const double* trow = tab_lane + ((dz + 3) * kOff + (dy + 3)) * kOff * kTabP;
      // source row: window y = 2Y + iy, z = 2Z + iz (parent-aligned, parity-free)
      const double2* src = reinterpret_cast<const double2*>(win) + ((iz & 1) * 2 + (iy & 1)) * kFSub +
                           (Z + (iz >> 1)) * kFPZ + (Y + (iy >> 1)) * kFPY;
      // this lane's source row lies in neighbour row (oy, oz); internal patches there?
      const int wy = 2 * Y + iy, wz = 2 * Z + iz;
      const int oy = wy < 2 ? 0 : (wy > 9 ? 2 : 1), oz = wz < 2 ? 0 : (wz > 9 ? 2 : 1);
      const unsigned rowbits = (internal27 >> ((oz * 3 + oy) * 3)) & 7u;
      const bool full[3] = {__any_sync(0xffffffffu, rowbits & 1u) != 0,
                            __any_sync(0xffffffffu, rowbits & 2u) != 0,
                            __any_sync(0xffffffffu, rowbits & 4u) != 0};
      if (dz >= -1 && dz <= 1 && dy >= -1 && dy <= 1)
        m2l_row_par<true, NOUT>(src, trow, acc, full);
      else
        m2l_row_par<false, NOUT>(src, trow, acc, full);
    }
  }
  // upper-half warps hand their partial sums to the lower-half warps (the
  // window is dead after the barrier): V = lower + upper, as the oracle adds
  __syncthreads();
  const int pair = threadIdx.x & 127;
  if (half) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int q = 0; q < NOUT; ++q) win[(k * 10 + q) * 128 + pair] = acc[k][q];
  }
  __syncthreads();
  if (half) return;
  const int y = 2 * Y + b, z = 2 * Z + c;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int cell = (z * 8 + y) * 8 + a + 2 * k;
    double v[NOUT];
#pragma unroll
    for (int q = 0; q < NOUT; ++q) v[q] = acc[k][q] + win[(k * 10 + q) * 128 + pair];
    if constexpr (NOUT == 10) {
      double2* out = reinterpret_cast<double2*>(loc + ((long long)n * 512 + cell) * 10);
#pragma unroll
      for (int h = 0; h < 5; ++h) out[h] = make_double2(v[2 * h], v[2 * h + 1]);
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) lloc[q * 512 + cell] = v[q];
    }
  }
}

// mass (one GPU, else null): a leaf neighbour's window cells take m from the
// leaf-mass array and zero-filled D, Q (its moments are (m, +0, ..., +0))
__global__ void __launch_bounds__(kM2lThreads, 1) amr_m2l_fused_kernel(
    const GLv* __restrict__ Lv, const int2* __restrict__ work, const double* __restrict__ tabp_all,
    double* __restrict__ lloc, long long lo, const double* __restrict__ mass) {
  extern __shared__ double sm[];
  __shared__ int s_nb[27], s_ls[27];
  __shared__ unsigned s_int27;
  double* win = sm;
  double* tabs = sm + kWinDoubles;
  const int2 wk = work[blockIdx.x];
  const int l = wk.x, n = wk.y;
  const GLv L = Lv[l];
  const int* nb27 = L.nbr + (long long)n * 27;
  // asynchronous fill (cp.async): the depth's geometry table, already in its
  // shared-memory layout (tabp_all: 14-double rows, the 27 near rows zero)
  const double* tabp = tabp_all + (long long)(l + 3) * kTabDoubles;
  for (int q = threadIdx.x; q < kTabDoubles / 2; q += kM2lThreads) cp_async16(tabs + 2 * q, tabp + 2 * q);
  // the 27 neighbour patches and their leaf slots, once; bit o of
  // internal27: neighbour o exists and is internal (full moments)
  if (threadIdx.x < 32) {
    const int o = threadIdx.x;
    const int nb = o < 27 ? nb27[o] : -1;
    const int ls = nb >= 0 ? L.leaf_slot[nb] : -1;
    const unsigned bits = __ballot_sync(0xffffffffu, nb >= 0 && ls < 0);
    if (o < 27) s_nb[o] = nb, s_ls[o] = ls;
    if (o == 0) s_int27 = bits;
  }
  __syncthreads();
  // task = (window row (wy, wz), component), component fastest: a warp's
  // copies of one x position read ~3 consecutive cells' 80-byte moments;
  // h = the 16-byte chunk of the records
  for (int task = threadIdx.x; task < 144 * kFRec; task += kM2lThreads) {
    const int h = task % kFRec, row = task / kFRec;
    const int wy = row % 12, wz = row / 12;
    int ly = wy - 2, lz = wz - 2;
    const int oy = ly < 0 ? -1 : (ly > 7 ? 1 : 0), oz = lz < 0 ? -1 : (lz > 7 ? 1 : 0);
    ly -= 8 * oy, lz -= 8 * oz;
    const int r3 = ((oz + 1) * 3 + (oy + 1)) * 3;
    const int nbs[3] = {s_nb[r3], s_nb[r3 + 1], s_nb[r3 + 2]};
    int lsl[3] = {-1, -1, -1};
    if (mass)
#pragma unroll
      for (int q = 0; q < 3; ++q) lsl[q] = s_ls[r3 + q];
    double* dst = win + 2 * (((wz & 1) * 2 + (wy & 1)) * kFSub + (wz >> 1) * kFPZ + (wy >> 1) * kFPY + h);
    const long long rowoff = (long long)(lz * 8 + ly) * 8;
#pragma unroll
    for (int wx = 0; wx < 12; ++wx) {
      const int ox = wx < 2 ? -1 : (wx > 9 ? 1 : 0), lx = wx - 2 - 8 * ox;
      const int nb = nbs[ox + 1], ls = lsl[ox + 1];
      double* d = dst + 2 * kFRec * wx;
      if (ls >= 0 && h == 0) {  // leaf neighbour (mass given): chunk 0 = (m, +0) (the mass is 8-byte aligned)
        cp_async8(d, mass + (long long)ls * 512 + rowoff + lx, true);
        cp_async8(d + 1, mass, false);
      } else if (ls >= 0 || nb < 0) {  // its other chunks, and missing patches: +0s
        cp_async16n(d, L.mom, 0);
      } else {
        cp_async16n(d, L.mom + ((long long)nb * 512 + rowoff + lx) * 10 + 2 * h, 16);
      }
    }
  }
  const unsigned internal27 = s_int27;
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
  const int leaf = L.leaf_slot[n];
  // leaf patch below the root: L0, L_i into the compact leaf locals (L2P's
  // input); a leaf root keeps all ten (the dense levels' L2L adds into them)
  if (leaf >= 0 && l > 0)
    m2l_patch<4>(win, tabs, L.loc, n, lloc + (long long)(leaf - lo) * 2048, internal27);
  else
    m2l_patch<10>(win, tabs, L.loc, n, nullptr, internal27);
}

// ---- M2L of leaf patches among leaf patches (monopole sources) -------------
// A leaf patch whose existing 27 neighbours are all leaf patches (5,000 of the
// 6,729 patches on C3) has only leaf cells as V sources, and a leaf cell's
// moments are (m, +0, ..., +0). Every D/Q term of the specification's M2L term
// is then an exact no-op (fma(+-0, e, x) = x for x != 0, and an accumulator that
// starts at +0 never becomes -0; the same argument as amr_m2m_kernel's leaf
// children), so per interaction only
//   t = -m * e0;  L0 = L0 + t;  L_i = fma(-m, e_i, L_i)        (i = 1..3)
// remain — 5 of the 23 operations into a leaf target, bit for bit the full
// term's result. The source window is then the 12^3 masses (from the compact
// [slot][512] mass array, not the 80-byte moments), 16 KB instead of 161 KB,
// so several CTAs share an SM (2 at 98 registers: faster per step than 4 at
// 64, 3.92 vs 3.97 ms on C3). Thread mapping, source order and the two
// partial sums are m2l_patch's.
constexpr int kMonoWin = 2048;  // >= 4 * kWSub + 2 (window) and the 4 x 4 x 128 partial sums
constexpr size_t kMonoSmem = (size_t)(kMonoWin + kOff3 * 4) * sizeof(double);  // 27,360 B

template <bool NEAR>
__device__ __forceinline__ void mono_row(const double* __restrict__ src, const double* __restrict__ trow,
                                         double (&acc)[4][4]) {
#pragma unroll
  for (int pe = 0; pe < 2; ++pe) {
    double G[3][4];
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      if (NEAR && t == 1) continue;
      const double2* t2 = reinterpret_cast<const double2*>(trow + (pe + 2 * t) * 4);
      const double2 u = t2[0], v = t2[1];
      G[t][0] = u.x, G[t][1] = u.y, G[t][2] = v.x, G[t][3] = v.y;
    }
#pragma unroll
    for (int mi = 0; mi < 6; ++mi) {
      const double nM = -src[pe + 2 * mi];
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        const int k = mi - t;
        if (k < 0 || k > 3) continue;
        if (NEAR && t == 1) continue;
        acc[k][0] = acc[k][0] + nM * G[t][0];
        acc[k][1] = fma(nM, G[t][1], acc[k][1]);
        acc[k][2] = fma(nM, G[t][2], acc[k][2]);
        acc[k][3] = fma(nM, G[t][3], acc[k][3]);
      }
    }
  }
}

__global__ void __launch_bounds__(kM2lThreads, 2) amr_m2l_mono_kernel(
    const long long* __restrict__ slots, const int* __restrict__ slot_level, const double* __restrict__ mass,
    const int* __restrict__ slot_nbs, const double* __restrict__ tab4p_all, double* __restrict__ lloc,
    long long lo) {
  extern __shared__ double sm[];
  double* win = sm;
  double* tabs = sm + kMonoWin;
  const long long s = slots[blockIdx.x];
  const int l = slot_level[s];
  // the depth's monopole table (4 values per offset, near rows zero)
  const double* tab4p = tab4p_all + (long long)(l + 3) * kOff3 * 4;
  for (int q = threadIdx.x; q < kOff3 * 2; q += kM2lThreads) cp_async16(tabs + 2 * q, tab4p + 2 * q);
  __shared__ int s_nb[27];
  if (threadIdx.x < 27) s_nb[threadIdx.x] = slot_nbs[s * 27 + threadIdx.x];
  __syncthreads();
  for (int t = threadIdx.x; t < 1728; t += kM2lThreads) {
    const int row = t / 12, wx = t - 12 * row, wz = row / 12, wy = row - 12 * wz;
    const int ox = wx < 2 ? -1 : (wx > 9 ? 1 : 0), oy = wy < 2 ? -1 : (wy > 9 ? 1 : 0),
              oz = wz < 2 ? -1 : (wz > 9 ? 1 : 0);
    const int nb = s_nb[((oz + 1) * 3 + (oy + 1)) * 3 + ox + 1];
    const int lx = wx - 2 - 8 * ox, ly = wy - 2 - 8 * oy, lz = wz - 2 - 8 * oz;
    double* dst = win + ((wz & 1) * 2 + (wy & 1)) * kWSub + (wz >> 1) * kWPZ + (wy >> 1) * kWPY + wx;
    cp_async8(dst, mass + ((long long)(nb < 0 ? s : nb) * 512 + (lz * 8 + ly) * 8 + lx), nb >= 0);
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = warp & 1, c = (warp >> 1) & 1, half = warp >> 2;
  const int a = lane & 1, Y = (lane >> 1) & 3, Z = lane >> 3;
  double acc[4][4];
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[k][q] = 0.0;
  const double* tab_lane = tabs + (1 - a) * 4;
  for (int iz = 3 * half; iz < 3 * half + 3; ++iz) {
    const int dz = iz - 2 - c;
#pragma unroll 2
    for (int iy = 0; iy < 6; ++iy) {
      const int dy = iy - 2 - b;
      const double* trow = tab_lane + ((dz + 3) * kOff + (dy + 3)) * kOff * 4;
      const double* src = win + ((iz & 1) * 2 + (iy & 1)) * kWSub + (Z + (iz >> 1)) * kWPZ + (Y + (iy >> 1)) * kWPY;
      if (dz >= -1 && dz <= 1 && dy >= -1 && dy <= 1)
        mono_row<true>(src, trow, acc);
      else
        mono_row<false>(src, trow, acc);
    }
  }
  __syncthreads();  // the window is dead: the upper half hands over its partial sums
  const int pair = threadIdx.x & 127;
  if (half) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int q = 0; q < 4; ++q) win[(k * 4 + q) * 128 + pair] = acc[k][q];
  }
  __syncthreads();
  if (half) return;
  const int y = 2 * Y + b, z = 2 * Z + c;
  double* out = lloc + (s - lo) * 2048;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int cell = (z * 8 + y) * 8 + a + 2 * k;
#pragma unroll
    for (int q = 0; q < 4; ++q) out[q * 512 + cell] = acc[k][q] + win[(k * 4 + q) * 128 + pair];
  }
}

// W/X pairs (AMR level jumps) after the V-list sums, in the list's sorted
// order, one thread per target with entries (targets in patch order);
// geometry from the plan's separation table (m2l_geom of each distinct R).
// mgeo[e] < 0 marks an entry whose source is a leaf cell (moments (m, +0, ...)):
// its geometry row is ~mgeo[e] and the monopole term is applied (bit for bit
// the full term, see amr_m2l_mono_kernel), reading 1 moment and 4 geometry
// values instead of 10 and 13.
template <int NOUT>
__device__ __forceinline__ void wx_mono(double nM, const double* __restrict__ e, double* acc) {
  acc[0] = acc[0] + nM * __ldg(e);
  acc[1] = fma(nM, __ldg(e + 1), acc[1]);
  acc[2] = fma(nM, __ldg(e + 2), acc[2]);
  acc[3] = fma(nM, __ldg(e + 3), acc[3]);
#pragma unroll
  for (int q = 0; q < NOUT - 4; ++q) acc[4 + q] = fma(nM, __ldg(e + 4 + q), acc[4 + q]);
}

template <int NOUT>
__device__ __forceinline__ void wx_entries(const GLv* __restrict__ Lv, const long long* __restrict__ ment,
                                           const int* __restrict__ mgeo, const int* __restrict__ mmi,
                                           const double* __restrict__ mass, long long e0, long long e1,
                                           const double* __restrict__ geo, double* acc) {
  auto mom_of = [&](long long enc) { return Lv[enc >> 40].mom + (enc & ((1LL << 40) - 1)) * 10; };
  auto apply = [&](long long e, int gi, double m0) {
    if (gi < 0) {
      wx_mono<NOUT>(-m0, geo + (long long)(~gi) * kTab, acc);
    } else {
      const double* pm = mom_of(__ldg(ment + e));
      if constexpr (NOUT == 10) m2l_tab(pm, geo + (long long)gi * kTab, acc);
      else m2l_tab4(pm, geo + (long long)gi * kTab, acc);
    }
  };
  long long e = e0;
  if (mass) {  // leaf sources' m from the leaf-mass array (mmi >= 0 exactly when gi < 0)
    for (; e + 3 < e1; e += 4) {  // four entries' loads in flight, applied in order
      int gi[4], mi[4];
      double m0[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) gi[u] = __ldg(mgeo + e + u), mi[u] = __ldg(mmi + e + u);
#pragma unroll
      for (int u = 0; u < 4; ++u) m0[u] = mi[u] >= 0 ? __ldg(mass + mi[u]) : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u) apply(e + u, gi[u], m0[u]);
    }
    for (; e < e1; ++e) {
      const int gi = __ldg(mgeo + e), mi = __ldg(mmi + e);
      apply(e, gi, mi >= 0 ? __ldg(mass + mi) : 0.0);
    }
    return;
  }
  for (; e + 3 < e1; e += 4) {
    long long enc[4];
    int gi[4];
    double m0[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) enc[u] = __ldg(ment + e + u), gi[u] = __ldg(mgeo + e + u);
#pragma unroll
    for (int u = 0; u < 4; ++u) m0[u] = __ldg(mom_of(enc[u]));
#pragma unroll
    for (int u = 0; u < 4; ++u) apply(e + u, gi[u], m0[u]);
  }
  for (; e < e1; ++e) {
    const int gi = __ldg(mgeo + e);
    apply(e, gi, __ldg(mom_of(__ldg(ment + e))));
  }
}

// A leaf target's entries with the leaf-mass array (one GPU): eight entries'
// loads in flight — index and geometry row, then the mass and the row's 4
// monopole values (geo4, two 16-byte loads) — applied in order; the terms are
// wx_mono<4>'s operations (an internal source's entry takes m2l_tab4).
__device__ __forceinline__ void wx_leaf_entries(const GLv* __restrict__ Lv, const long long* __restrict__ ment,
                                                const int* __restrict__ mgeo, const int* __restrict__ mmi,
                                                const double* __restrict__ mass, long long e0, long long e1,
                                                const double* __restrict__ geo, const double* __restrict__ geo4,
                                                double* acc) {
  constexpr int D = 8;
  const double2* g2 = reinterpret_cast<const double2*>(geo4);
  auto full = [&](long long e, int gi) {
    const long long enc = __ldg(ment + e);
    m2l_tab4(Lv[enc >> 40].mom + (enc & ((1LL << 40) - 1)) * 10, geo + (long long)gi * kTab, acc);
  };
  long long e = e0;
  // software pipeline: the next batch's indices load while this batch's
  // masses and geometry rows are in flight (one round trip per batch)
  int gi[D], mi[D];
  if (e + D - 1 < e1) {
#pragma unroll
    for (int u = 0; u < D; ++u) gi[u] = __ldg(mgeo + e + u), mi[u] = __ldg(mmi + e + u);
  }
  for (; e + D - 1 < e1; e += D) {
    double m0[D];
    double2 ga[D], gb[D];
#pragma unroll
    for (int u = 0; u < D; ++u) {
      const bool mono = gi[u] < 0;
      const long long row = mono ? ~gi[u] : 0;
      m0[u] = mono ? __ldg(mass + mi[u]) : 0.0;
      ga[u] = __ldg(g2 + 2 * row);
      gb[u] = __ldg(g2 + 2 * row + 1);
    }
    int gc[D];
#pragma unroll
    for (int u = 0; u < D; ++u) gc[u] = gi[u];
    if (e + 2 * D - 1 < e1) {
#pragma unroll
      for (int u = 0; u < D; ++u) gi[u] = __ldg(mgeo + e + D + u), mi[u] = __ldg(mmi + e + D + u);
    }
#pragma unroll
    for (int u = 0; u < D; ++u) {
      if (gc[u] < 0) {
        const double nM = -m0[u];
        acc[0] = acc[0] + nM * ga[u].x;
        acc[1] = fma(nM, ga[u].y, acc[1]);
        acc[2] = fma(nM, gb[u].x, acc[2]);
        acc[3] = fma(nM, gb[u].y, acc[3]);
      } else {
        full(e + u, gc[u]);
      }
    }
  }
  for (; e < e1; ++e) {
    const int gi = __ldg(mgeo + e);
    if (gi < 0) {
      const double nM = -__ldg(mass + __ldg(mmi + e));
      const double2 a = __ldg(g2 + 2 * (long long)~gi), b = __ldg(g2 + 2 * (long long)~gi + 1);
      acc[0] = acc[0] + nM * a.x;
      acc[1] = fma(nM, a.y, acc[1]);
      acc[2] = fma(nM, b.x, acc[2]);
      acc[3] = fma(nM, b.y, acc[3]);
    } else {
      full(e, gi);
    }
  }
}

// W/X pairs (AMR level jumps) after the V-list sums, in the list's sorted
// order, one thread per target with entries (targets in patch order);
// geometry from the plan's separation table (m2l_geom of each distinct R).
// Leaf-patch targets update their compact L0, L_i only.
// A W/X target resolved with the plan: its entry range, and where its locals
// live (leaf: the compact leaf locals at `off`; internal: level l's loc at
// flat `off`) — one 32-byte load instead of a chain of dependent lookups.
struct WxTarget {
  long long e0, e1, off;
  int level, leaf;
};

__global__ void __launch_bounds__(128, 4) amr_wx_kernel(const GLv* __restrict__ Lv,
                                                        const WxTarget* __restrict__ targets, long long ntarget,
                                                        const double* __restrict__ geo,
                                                        double* __restrict__ lloc,
                                                        const double* __restrict__ mass,
                                                        const double* __restrict__ geo4) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < ntarget;
       t += (long long)gridDim.x * blockDim.x) {
    const WxTarget d = targets[t];
    const int l = d.level;
    const long long e0 = d.e0, e1 = d.e1, flat = d.off;
    if (d.leaf) {
      double* p = lloc + d.off;
      double acc[4] = {p[0], p[512], p[1024], p[1536]};
      if (mass)
        wx_leaf_entries(Lv, Lv[l].ment, Lv[l].mgeo, Lv[l].mmi, mass, e0, e1, geo, geo4, acc);
      else
        wx_entries<4>(Lv, Lv[l].ment, Lv[l].mgeo, Lv[l].mmi, mass, e0, e1, geo, acc);
#pragma unroll
      for (int q = 0; q < 4; ++q) p[q * 512] = acc[q];
    } else {
      double* loc = Lv[l].loc + flat * 10;
      double acc[10];
#pragma unroll
      for (int h = 0; h < 5; ++h) {
        const double2 v = reinterpret_cast<const double2*>(loc)[h];
        acc[2 * h] = v.x;
        acc[2 * h + 1] = v.y;
      }
      wx_entries<10>(Lv, Lv[l].ment, Lv[l].mgeo, Lv[l].mmi, mass, e0, e1, geo, acc);
#pragma unroll
      for (int h = 0; h < 5; ++h)
        reinterpret_cast<double2*>(loc)[h] = make_double2(acc[2 * h], acc[2 * h + 1]);
    }
  }
}

// The M2L geometry table in the kernels' shared-memory layouts, per depth:
// tabp [343][14] (13 values + a zero pad) and tab4p [343][4] (the monopole
// values), the 27 near offsets' rows zero
__global__ void pad_tables_kernel(const double* __restrict__ tab, int D, double* __restrict__ tabp,
                                  double* __restrict__ tab4p) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)(D + 1) * kOff3 * kTabP) return;
  const long long row = t / kTabP;
  const int q = (int)(t % kTabP), o = (int)(row % kOff3);
  const int dx = o % kOff - 3, dy = (o / kOff) % kOff - 3, dz = o / (kOff * kOff) - 3;
  const bool near = dx >= -1 && dx <= 1 && dy >= -1 && dy <= 1 && dz >= -1 && dz <= 1;
  const double v = (near || q >= kTab) ? 0.0 : tab[row * kTab + q];
  tabp[t] = v;
  if (q < 4) tab4p[row * 4 + q] = v;
}

// P2P geometry of the 26 same-depth lattice offsets at every cell depth
// (p2p_geom, the per-pair operations): [depth][27][4], centre entry zero
__global__ void p2p_table_kernel(double* __restrict__ tab, int D) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (D + 1) * 27) return;
  const int dpt = t / 27, o = t % 27;
  const int dx = o % 3 - 1, dy = (o / 3) % 3 - 1, dz = o / 9 - 1;
  double* e = tab + (long long)t * 4;
  if (o == 13) {
    for (int q = 0; q < 4; ++q) e[q] = 0.0;
    return;
  }
  const double h = 1.0 / (double)(1LL << dpt);
  p2p_geom(-(double)dx * h, -(double)dy * h, -(double)dz * h, e);
}

__global__ void sep_geom_kernel(const double* __restrict__ sep, long long n, double* __restrict__ geo,
                                int p2p) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= n) return;
  const double x = sep[3 * t], y = sep[3 * t + 1], z = sep[3 * t + 2];
  if (p2p) {
    double w[4];
    p2p_geom(x, y, z, w);
    for (int q = 0; q < 4; ++q) geo[4 * t + q] = w[q];
  } else {
    m2l_geom(x, y, z, geo + t * kTab);
  }
}

// parent local (Lp, 10) shifted to the child centre s (tmo_grav_l2l): the
// first NOUT components (L2P needs only L0 and L_i)
template <int NOUT>
__device__ __forceinline__ void l2l_shift(const double* __restrict__ Lp, const double s[3],
                                          double sh[NOUT]) {
  double Lm[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) Lm[a][b] = Lp[4 + s2(a, b)];
  double t1 = 0.0, t2 = 0.0;
#pragma unroll
  for (int a = 0; a < 3; ++a) t1 += Lp[1 + a] * s[a];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) t2 += Lm[a][b] * s[a] * s[b];
  sh[0] = Lp[0] + t1 + 0.5 * t2;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double u = 0.0;
#pragma unroll
    for (int b = 0; b < 3; ++b) u += Lm[a][b] * s[b];
    sh[1 + a] = Lp[1 + a] + u;
  }
#pragma unroll
  for (int q = 4; q < NOUT; ++q) sh[q] = Lp[q];
}

// parent's cell and the child-centre offset of cell c of node n at level l
__device__ __forceinline__ const double* l2l_parent(const GLv& L, const GLv& P, long long n, int c,
                                                   double h, double s[3]) {
  const int i = c & 7, j = (c >> 3) & 7, k = c >> 6;
  const int pn = L.parent[n];
  const int pi = (L.ijk[3 * n] & 1) * 4 + (i >> 1), pj = (L.ijk[3 * n + 1] & 1) * 4 + (j >> 1),
            pk = (L.ijk[3 * n + 2] & 1) * 4 + (k >> 1);
  s[0] = ((i & 1) - 0.5) * h;
  s[1] = ((j & 1) - 0.5) * h;
  s[2] = ((k & 1) - 0.5) * h;
  return P.loc + ((long long)pn * 512 + (pk * 8 + pj) * 8 + pi) * 10;
}

// L2L of the internal patches of level l (leaf patches get theirs inside L2P)
__global__ void amr_l2l_kernel(const GLv* __restrict__ Lv, int l, long long nnodes,
                               const int* __restrict__ nodes) {
  const GLv L = Lv[l], P = Lv[l - 1];
  const double h = 1.0 / (double)(1LL << (l + 3));
  for (long long tt = blockIdx.x * (long long)blockDim.x + threadIdx.x; tt < nnodes * 512;
       tt += (long long)gridDim.x * blockDim.x) {
    const long long n = nodes[tt >> 9];
    const int c = (int)(tt & 511);
    double s[3], sh[10], lp[10], cur[10];
    const double2* p2 = reinterpret_cast<const double2*>(l2l_parent(L, P, n, c, h, s));
    double2* o2 = reinterpret_cast<double2*>(L.loc + (n * 512 + c) * 10);
#pragma unroll
    for (int q = 0; q < 5; ++q) {  // 80-byte records as five 16-byte loads
      const double2 a = p2[q], b = o2[q];
      lp[2 * q] = a.x, lp[2 * q + 1] = a.y, cur[2 * q] = b.x, cur[2 * q + 1] = b.y;
    }
    l2l_shift<10>(lp, s, sh);
#pragma unroll
    for (int q = 0; q < 5; ++q) o2[q] = make_double2(sh[2 * q] + cur[2 * q], sh[2 * q + 1] + cur[2 * q + 1]);
  }
}

// -(source mass) of every cross-depth U entry, gathered in parallel over the
// entries before L2P (whose per-target loop then reads them contiguously
// instead of chasing entry -> moment); grid.y = level
__global__ void amr_u_gather_kernel(const GLv* __restrict__ Lv, const double* __restrict__ mass) {
  const GLv L = Lv[blockIdx.y];
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < L.nu;
       e += (long long)gridDim.x * blockDim.x) {
    if (mass) {
      L.unm[e] = -__ldg(mass + __ldg(L.pmi + e));
    } else {
      const long long enc = __ldg(L.pent + e);
      L.unm[e] = -__ldg(Lv[enc >> 40].mom + (enc & ((1LL << 40) - 1)) * 10);
    }
  }
}

// L2P + P2P at the leaf cells, output by local slot: phi[s*512 + c],
// g[q*ncell + s*512 + c]. CTA = one slot (512 cells). The leaf patch's L2L is
// done here (L_q = shift(parent)_q + own M2L sum_q for q = 0..3, the only
// components L2P uses; level-0 leaves have their final locals). The 26
// same-depth offsets' P2P geometry (p2p_geom of the lattice offset, the same
// operations as per pair) and the 27 neighbour slots are resolved once into
// shared memory; neighbour masses come from the leaf-mass array (coalesced),
// cross-depth U pairs from the plan's geometry table. Term order: 26 offsets
// dz, dy, dx ascending, then the U pairs. With `part`, the slot's 16
// angular-momentum sums follow (am_block_sums2: the per-slot pair tree).
__device__ __forceinline__ void cell_pos(const GLv* __restrict__ Lv, int l, int n, int c, double x[3]);
__device__ __forceinline__ void am_block_sums2(double m0, const double x0[3], const double g0[3], double m1,
                                               const double x1[3], const double g1[3], double* __restrict__ out16);

constexpr int kL2pThreads = 256;  // two cells per thread: 5 CTAs per SM (48 registers) overlap their prologues

__global__ void __launch_bounds__(kL2pThreads, 5) amr_l2p_kernel(const GLv* __restrict__ Lv, long long nslots,
                                                      long long lo, const int* __restrict__ slot_level,
                                                      const int* __restrict__ slot_node,
                                                      const double* __restrict__ mass,
                                                      const double* __restrict__ ugeo,
                                                      const double* __restrict__ lloc,
                                                      const double* __restrict__ p2p_tab,
                                                      const int* __restrict__ slot_nbs,
                                                      double* __restrict__ phi, double* __restrict__ g,
                                                      double* __restrict__ part) {
  // everything the cell needs from memory is staged up front by cp.async, so
  // the loads overlap each other instead of forming per-thread chains:
  //   mw   masses of the patch and its one-cell halo, [z 10][y 10][x pitch 24],
  //        x = -1..8 at offsets 1..10 (interior 16-byte aligned; pitch 24: the
  //        two rows of a half-warp fall in disjoint banks)
  //   ll   the leaf's compact V + W/X locals [4][512]
  //   pl   the 4^3 parent cells above the patch, [cell][10] (the L2L input)
  __shared__ double w26[27][4];
  __shared__ __align__(16) double mw[10 * 240];
  __shared__ __align__(16) double ll[2048];
  __shared__ __align__(16) double pl[640];
  __shared__ unsigned valid27;  // bit o: same-depth neighbour leaf patch o exists
  __shared__ int nbs[27];
  const long long ls = blockIdx.x;  // local slot
  const long long s = lo + ls;
  const int l = slot_level[s], n = slot_node[s];
  const GLv L = Lv[l];
  const int d = l + 3;
  const double h = 1.0 / (double)(1LL << d);
  // the patch's cell-grid origin (8 ijk), for the angular-momentum sums' positions
  const long long g0[3] = {8LL * L.ijk[3 * n], 8LL * L.ijk[3 * n + 1], 8LL * L.ijk[3 * n + 2]};
  if (threadIdx.x < 27) {  // the 27 neighbour slots, resolved once
    const int o = threadIdx.x;
    const int nb = slot_nbs[s * 27 + o];
    nbs[o] = nb;
    const unsigned bit = __ballot_sync(0x07ffffffu, nb >= 0);
    if (o == 0) valid27 = bit;
  }
  __syncthreads();
  // window rows (wy, wz) of x = -1..8 at offsets 1..10: the 8 interior x as
  // four 16-byte copies from one neighbour row, the two halo cells as 8 bytes
  for (int t = threadIdx.x; t < 600; t += blockDim.x) {
    const bool interior = t < 400;
    const int row = interior ? (t >> 2) : ((t - 400) >> 1), q = interior ? (t & 3) : ((t - 400) & 1);
    const int wy = row % 10, wz = row / 10;
    const int oy = wy < 1 ? -1 : (wy > 8 ? 1 : 0), oz = wz < 1 ? -1 : (wz > 8 ? 1 : 0);
    const int ox = interior ? 0 : (q ? 1 : -1);
    const int nb = nbs[((oz + 1) * 3 + (oy + 1)) * 3 + ox + 1];
    const int ly = wy - 1 - 8 * oy, lz = wz - 1 - 8 * oz;
    const double* src = mass + (long long)(nb < 0 ? s : nb) * 512 + (lz * 8 + ly) * 8;
    if (interior)
      cp_async16z(mw + row * 24 + 2 + 2 * q, src + 2 * q, nb >= 0);
    else
      cp_async8(mw + row * 24 + (q ? 10 : 1), src + (q ? 0 : 7), nb >= 0);
  }
  if (l > 0) {
    const double* src = lloc + ls * 2048;
    for (int t = threadIdx.x; t < 1024; t += blockDim.x) cp_async16(ll + 2 * t, src + 2 * t);
    const GLv P = Lv[l - 1];
    const int pn = L.parent[n];
    const int bx = (L.ijk[3 * n] & 1) * 4, by = (L.ijk[3 * n + 1] & 1) * 4, bz = (L.ijk[3 * n + 2] & 1) * 4;
    for (int t = threadIdx.x; t < 320; t += blockDim.x) {  // 16 rows of 4 cells x 10 = 20 x 16 B
      const int row = t / 20, q = t % 20;
      const double* r = P.loc + ((long long)pn * 512 + ((bz + (row >> 2)) * 8 + (by + (row & 3))) * 8 + bx) * 10;
      cp_async16(pl + row * 40 + 2 * q, r + 2 * q);
    }
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
  // masses scaled by 2^d at use for the unit-spacing constant geometry (exact)
  const double sc1 = (double)(1LL << d);
  const long long ncell = nslots * 512;
  double keep[2][3];  // the two cells' g for the angular-momentum sums
#pragma unroll
  for (int hc = 0; hc < 2; ++hc) {
  const int c = threadIdx.x + hc * kL2pThreads;
  const int i = c & 7, j = (c >> 3) & 7, k = c >> 6;
  const long long flat = (long long)n * 512 + c;
  double loc4[4];
  if (l == 0) {  // a leaf root: the full locals, with the dense levels' L2L already added
    const double* Lr = L.loc + flat * 10;
#pragma unroll
    for (int q = 0; q < 4; ++q) loc4[q] = Lr[q];
  } else {  // compact leaf locals (V + W/X sums) + the parent's shift (l2l_parent's cell)
#pragma unroll
    for (int q = 0; q < 4; ++q) loc4[q] = ll[q * 512 + c];
    const double sv[3] = {((i & 1) - 0.5) * h, ((j & 1) - 0.5) * h, ((k & 1) - 0.5) * h};
    double sh[4];
    l2l_shift<4>(pl + (((k >> 1) * 4 + (j >> 1)) * 4 + (i >> 1)) * 10, sv, sh);
#pragma unroll
    for (int q = 0; q < 4; ++q) loc4[q] = sh[q] + loc4[q];
  }
  double p = loc4[0], gx = -loc4[1], gy = -loc4[2], gz = -loc4[3];
  // the 26 same-depth neighbours; a neighbour in a missing patch is skipped —
  // a check needed only when some of the 27 patches is missing (valid27 is
  // the same for the whole CTA, so the branch does not diverge)
  auto p2p = [&](auto check_c) {
    constexpr bool CHECK = decltype(check_c)::value;
#pragma unroll
    for (int dz = -1; dz <= 1; ++dz)
#pragma unroll
      for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
        for (int dx = -1; dx <= 1; ++dx) {
          if (!dx && !dy && !dz) continue;
          const int lx = i + dx, ly = j + dy, lz = k + dz;
          if (CHECK) {
            const int ox = lx < 0 ? -1 : (lx > 7 ? 1 : 0), oy = ly < 0 ? -1 : (ly > 7 ? 1 : 0),
                      oz = lz < 0 ? -1 : (lz > 7 ? 1 : 0);
            if (!((valid27 >> (((oz + 1) * 3 + (oy + 1)) * 3 + ox + 1)) & 1u)) continue;
          }
          // -m 2^d and -m 2^2d against the unit geometry: p2p_geom's terms exactly
          const double nm1 = -(mw[((lz + 1) * 10 + (ly + 1)) * 24 + lx + 2] * sc1), nm2 = nm1 * sc1;
          const int o = ((dz + 1) * 3 + (dy + 1)) * 3 + dx + 1;
          p = fma(nm1, c_p2p_unit[o][0], p);
          gx = fma(nm2, c_p2p_unit[o][1], gx);
          gy = fma(nm2, c_p2p_unit[o][2], gy);
          gz = fma(nm2, c_p2p_unit[o][3], gz);
        }
  };
  if (valid27 == 0x7ffffffu)
    p2p(std::integral_constant<bool, false>{});
  else
    p2p(std::integral_constant<bool, true>{});
  const long long e0 = L.poff[flat], e1 = L.poff[flat + 1];
  long long e = e0;
  for (; e + 3 < e1; e += 4) {  // cross-depth U pairs, sorted by source: 4 entries' loads in flight
    double nm[4], w[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      nm[u] = __ldg(L.unm + e + u);
      const double2* w2 = reinterpret_cast<const double2*>(ugeo + (long long)__ldg(L.pgeo + e + u) * 4);
      const double2 a = __ldg(w2), b = __ldg(w2 + 1);
      w[u][0] = a.x, w[u][1] = a.y, w[u][2] = b.x, w[u][3] = b.y;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      p = fma(nm[u], w[u][0], p);
      gx = fma(nm[u], w[u][1], gx);
      gy = fma(nm[u], w[u][2], gy);
      gz = fma(nm[u], w[u][3], gz);
    }
  }
  for (; e < e1; ++e) {
    const double nm = L.unm[e];
    const double* w = ugeo + (long long)L.pgeo[e] * 4;
    p = fma(nm, w[0], p);
    gx = fma(nm, w[1], gx);
    gy = fma(nm, w[2], gy);
    gz = fma(nm, w[3], gz);
  }
  const long long t = ls * 512 + c;
  phi[t] = p;
  g[t] = gx;
  g[ncell + t] = gy;
  g[2 * ncell + t] = gz;
  keep[hc][0] = gx, keep[hc][1] = gy, keep[hc][2] = gz;
  }
  if (part) {  // the two cells' masses from the window, positions from the patch origin (cell_pos's values)
    const int c0 = threadIdx.x, i = c0 & 7, j = (c0 >> 3) & 7, k = c0 >> 6;  // c1 = c0 + 256: k + 4
    const double x0[3] = {centre(g0[0] + i, d), centre(g0[1] + j, d), centre(g0[2] + k, d)};
    const double x1[3] = {x0[0], x0[1], centre(g0[2] + k + 4, d)};
    const double m0 = mw[((k + 1) * 10 + (j + 1)) * 24 + i + 2], m1 = mw[((k + 5) * 10 + (j + 1)) * 24 + i + 2];
    am_block_sums2(m0, x0, keep[0], m1, x1, keep[1], part + s * 16);
  }
}

// The dense depth-2 M2L (4^3 cells, every cell exists; m2l_kernel's loop
// order and arithmetic) with the 64 cells' moments and the depth's geometry
// table staged in shared memory; thread t < 64 sums target t's lower source
// planes, thread t + 64 its upper ones (the specification's two partial sums),
// added as o[0] + o[1]. One CTA.
__global__ void __launch_bounds__(128) dense_m2l_staged_kernel(const double* __restrict__ mom,
                                                               double* __restrict__ loc,
                                                               const double* __restrict__ tab) {
  __shared__ double s_mom[64 * 10];
  __shared__ double s_tab[kOff3 * kTab];
  __shared__ double s_up[64 * 10];
  for (int q = threadIdx.x; q < 64 * 10; q += blockDim.x) s_mom[q] = mom[q];
  for (int q = threadIdx.x; q < kOff3 * kTab; q += blockDim.x) s_tab[q] = tab[q];
  __syncthreads();
  const int t = threadIdx.x & 63, upper = threadIdx.x >> 6;
  const int i = t & 3, j = (t >> 2) & 3, k = t >> 4;
  double o[10];
#pragma unroll
  for (int q = 0; q < 10; ++q) o[q] = 0.0;
  for (int dz = -2 - (k & 1); dz <= 3 - (k & 1); ++dz) {
    if ((dz + (k & 1) >= 1) != (upper != 0)) continue;
    for (int dy = -2 - (j & 1); dy <= 3 - (j & 1); ++dy)
      for (int pe = 0; pe < 2; ++pe)  // even source x, then odd
        for (int dx = -2 - (i & 1) + pe; dx <= 3 - (i & 1); dx += 2) {
          if (dx >= -1 && dx <= 1 && dy >= -1 && dy <= 1 && dz >= -1 && dz <= 1) continue;
          const int si = i + dx, sj = j + dy, sk = k + dz;
          if (si < 0 || sj < 0 || sk < 0 || si >= 4 || sj >= 4 || sk >= 4) continue;
          m2l_tab(s_mom + ((sk * 4 + sj) * 4 + si) * 10, s_tab + (((dz + 3) * kOff + (dy + 3)) * kOff + (dx + 3)) * kTab,
                  o);
        }
  }
  if (upper)
#pragma unroll
    for (int q = 0; q < 10; ++q) s_up[t * 10 + q] = o[q];
  __syncthreads();
  if (!upper)
#pragma unroll
    for (int q = 0; q < 10; ++q) loc[t * 10 + q] = o[q] + s_up[t * 10 + q];
}

// The dense top's three M2M levels (4^3 <- level-0 patch, 2^3, 1) in one CTA
__global__ void __launch_bounds__(128) top_m2m_kernel(const double* __restrict__ lv0, double* __restrict__ d2,
                                                      double* __restrict__ d1, double* __restrict__ d0) {
  if (threadIdx.x < 64) m2m_cell(lv0, d2, 4, 1.0 / 8.0, threadIdx.x);
  __syncthreads();
  if (threadIdx.x < 8) m2m_cell(d2, d1, 2, 1.0 / 4.0, threadIdx.x);
  __syncthreads();
  if (threadIdx.x == 0) m2m_cell(d1, d0, 1, 1.0 / 2.0, 0);
}

// ---- angular-momentum correction (tmo_grav_am_correct) ---------------------

__device__ __forceinline__ void cell_pos(const GLv* __restrict__ Lv, int l, int n, int c, double x[3]) {
  const GLv L = Lv[l];
  const int d = l + 3;
  x[0] = centre(8LL * L.ijk[3 * n] + (c & 7), d);
  x[1] = centre(8LL * L.ijk[3 * n + 1] + ((c >> 3) & 7), d);
  x[2] = centre(8LL * L.ijk[3 * n + 2] + (c >> 6), d);
}

// The slot's 16 angular-momentum sums for 256 threads holding cells t and
// t + 256: an adjacent-pair tree over the 512 cells in slot order (warp trees
// over cells [32w, 32w + 32), then a tree over the 16 warp sums).
// The warp tree is transposed: at level st the lane pair (l, l ^ st) holds the
// same values for two adjacent subtrees; each lane keeps half of them and
// receives the partner's half (8 + 4 + 2 + 1 shuffles, then one for the two
// 16-lane halves) — every partial sum is the same (left subtree + right
// subtree) as the plain tree's, and IEEE addition is commutative, so the sums
// are bitwise the plain tree's with 16 shuffles instead of 80. Returns on
// lanes 0..15 the warp sum of value am_lane_value(lane).
__device__ __forceinline__ int am_lane_value(int lane) {
  return ((lane & 1) << 3) | ((lane & 2) << 1) | ((lane & 4) >> 1) | ((lane & 8) >> 3);
}

__device__ __forceinline__ double am_warp_tree(double m, const double x[3], const double gg[3]) {
  double v[16];
  v[0] = m;
  v[1] = m * x[0];
  v[2] = m * x[1];
  v[3] = m * x[2];
  v[4] = m * gg[0];
  v[5] = m * gg[1];
  v[6] = m * gg[2];
  v[7] = m * (x[1] * gg[2] - x[2] * gg[1]);
  v[8] = m * (x[2] * gg[0] - x[0] * gg[2]);
  v[9] = m * (x[0] * gg[1] - x[1] * gg[0]);
  v[10] = v[1] * x[0];
  v[11] = v[1] * x[1];
  v[12] = v[1] * x[2];
  v[13] = v[2] * x[1];
  v[14] = v[2] * x[2];
  v[15] = v[3] * x[2];
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  double a[8], b[4], c[2];
  const bool h1 = lane & 1, h2 = lane & 2, h4 = lane & 4, h8 = lane & 8;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double r = __shfl_xor_sync(full, h1 ? v[k] : v[8 + k], 1);
    a[k] = (h1 ? v[8 + k] : v[k]) + r;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double r = __shfl_xor_sync(full, h2 ? a[k] : a[4 + k], 2);
    b[k] = (h2 ? a[4 + k] : a[k]) + r;
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const double r = __shfl_xor_sync(full, h4 ? b[k] : b[2 + k], 4);
    c[k] = (h4 ? b[2 + k] : b[k]) + r;
  }
  const double d = (h8 ? c[1] : c[0]) + __shfl_xor_sync(full, h8 ? c[0] : c[1], 8);
  return d + __shfl_xor_sync(full, d, 16);
}

__device__ __forceinline__ void am_block_sums2(double m0, const double x0[3], const double g0[3], double m1,
                                               const double x1[3], const double g1[3], double* __restrict__ out16) {
  __shared__ double red[16][16];  // [warp of 32 cells][value]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double s0 = am_warp_tree(m0, x0, g0);
  const double s1 = am_warp_tree(m1, x1, g1);
  if (lane < 16) {
    red[warp][am_lane_value(lane)] = s0;
    red[warp + 8][am_lane_value(lane)] = s1;
  }
  __syncthreads();
  if (threadIdx.x < 16) {
    const int c = threadIdx.x;
    double w[16];
#pragma unroll
    for (int a = 0; a < 16; ++a) w[a] = red[a][c];
#pragma unroll
    for (int st = 1; st < 16; st <<= 1)
#pragma unroll
      for (int a = 0; a < 16; a += 2 * st) w[a] = w[a] + w[a + st];
    out16[c] = w[0];
  }
}

// adjacent-pair tree over n (power of two) entries of 16 sums: each CTA
// reduces a chunk of min(n, 256) consecutive entries (the first levels of the
// global tree) into out[blockIdx.x]
__device__ __forceinline__ void am_solve(const double* __restrict__ S, double* __restrict__ rw);

// rw (the last pass: one CTA over the whole remaining n): thread 0 solves
// for the rigid-rotation field from the root sums (am_solve) instead of
// storing them
__global__ void __launch_bounds__(256) am_tree_pass_kernel(const double* __restrict__ in,
                                                           double* __restrict__ out, long long n,
                                                           double* __restrict__ rw = nullptr) {
  __shared__ double v[256][17];
  const int chunk = n < 256 ? (int)n : 256;
  const long long base = (long long)blockIdx.x * chunk;
  const int t = threadIdx.x;
  if (t < chunk)
#pragma unroll
    for (int q = 0; q < 16; ++q) v[t][q] = in[(base + t) * 16 + q];
  __syncthreads();
  for (int st = 1; st < chunk; st <<= 1) {
    if (t < chunk && (t & (2 * st - 1)) == 0)
#pragma unroll
      for (int q = 0; q < 16; ++q) v[t][q] = v[t][q] + v[t + st][q];
    __syncthreads();
  }
  if (rw) {
    if (t == 0) am_solve(v[0], rw);
  } else if (t < 16) {
    out[(long long)blockIdx.x * 16 + t] = v[0][t];
  }
}

// the 3x3 solve of tmo_grav_am_solve on the total sums S -> rw = (R, w, S)
__device__ __forceinline__ void am_solve(const double* __restrict__ S, double* __restrict__ rw) {
  double R[3], w[3];
  const double M = S[0];
  R[0] = S[1] / M;
  R[1] = S[2] / M;
  R[2] = S[3] / M;
  const double F[3] = {S[4], S[5], S[6]};
  const double tau[3] = {S[7] - (R[1] * F[2] - R[2] * F[1]), S[8] - (R[2] * F[0] - R[0] * F[2]),
                         S[9] - (R[0] * F[1] - R[1] * F[0])};
  const double cxx = S[10] - (M * R[0]) * R[0], cxy = S[11] - (M * R[0]) * R[1],
               cxz = S[12] - (M * R[0]) * R[2], cyy = S[13] - (M * R[1]) * R[1],
               cyz = S[14] - (M * R[1]) * R[2], czz = S[15] - (M * R[2]) * R[2];
  const double tr = (cxx + cyy) + czz;
  const double j00 = tr - cxx, j11 = tr - cyy, j22 = tr - czz, j01 = -cxy, j02 = -cxz, j12 = -cyz;
  const double a00 = j11 * j22 - j12 * j12, a01 = j02 * j12 - j01 * j22, a02 = j01 * j12 - j02 * j11,
               a11 = j00 * j22 - j02 * j02, a12 = j01 * j02 - j00 * j12, a22 = j00 * j11 - j01 * j01;
  const double det = (j00 * a00 + j01 * a01) + j02 * a02;
  if (!(det > 0.0)) {
    w[0] = w[1] = w[2] = 0.0;
  } else {
    const double b0 = -tau[0], b1 = -tau[1], b2 = -tau[2];
    w[0] = ((a00 * b0 + a01 * b1) + a02 * b2) / det;
    w[1] = ((a01 * b0 + a11 * b1) + a12 * b2) / det;
    w[2] = ((a02 * b0 + a12 * b1) + a22 * b2) / det;
  }
  for (int q = 0; q < 3; ++q) rw[q] = R[q], rw[3 + q] = w[q];
  for (int q = 0; q < 16; ++q) rw[6 + q] = S[q];
}

__global__ void am_solve_kernel(const double* __restrict__ part, double* __restrict__ rw) {
  if (threadIdx.x == 0) am_solve(part, rw);
}

__global__ void am_apply_kernel(const GLv* __restrict__ Lv, long long nslots, long long lo,
                                const int* __restrict__ slot_level, const int* __restrict__ slot_node,
                                const double* __restrict__ rw, double* __restrict__ g) {
  const long long ncell = nslots * 512;
  const double R0 = rw[0], R1 = rw[1], R2 = rw[2], w0 = rw[3], w1 = rw[4], w2 = rw[5];
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < ncell;
       t += (long long)gridDim.x * blockDim.x) {
    const long long s = lo + (t >> 9);
    double x[3];
    cell_pos(Lv, slot_level[s], slot_node[s], (int)(t & 511), x);
    const double dx = x[0] - R0, dy = x[1] - R1, dz = x[2] - R2;
    g[t] = g[t] + (w1 * dz - w2 * dy);
    g[ncell + t] = g[ncell + t] + (w2 * dx - w0 * dz);
    g[2 * ncell + t] = g[2 * ncell + t] + (w0 * dy - w1 * dx);
  }
}

template <class T>
cudaError_t upload(const std::vector<T>& v, T** out) {
  *out = nullptr;
  if (v.empty()) return cudaSuccess;
  cudaError_t e = cudaMalloc(out, v.size() * sizeof(T));
  if (e == cudaSuccess) e = cudaMemcpy(*out, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
  return e;
}

}  // namespace

// Algorithmic work of one solve (bench roofline): interactions with an
// existing source, counted per neighbour-patch offset from the plan.
// need: per-level node lists this GPU evaluates M2L for (nullptr = all);
// [lo, hi): the canonical slots it evaluates L2P/P2P for.
constexpr int kWorkCounts = 16;

void count_work(const GravPlan& P, const std::vector<std::vector<int>>* need, long long lo,
                long long hi, long long out[kWorkCounts]) {
  long long vtab[27] = {0}, ptab[27] = {0};
  for (int c = 0; c < 512; ++c) {
    const int i = c & 7, j = (c >> 3) & 7, k = c >> 6;
    for (int dz = -2 - (k & 1); dz <= 3 - (k & 1); ++dz)
      for (int dy = -2 - (j & 1); dy <= 3 - (j & 1); ++dy)
        for (int dx = -2 - (i & 1); dx <= 3 - (i & 1); ++dx) {
          const bool near = dx >= -1 && dx <= 1 && dy >= -1 && dy <= 1 && dz >= -1 && dz <= 1;
          const int ox = (i + dx + 8) / 8 - 1, oy = (j + dy + 8) / 8 - 1, oz = (k + dz + 8) / 8 - 1;
          const int o = ((oz + 1) * 3 + (oy + 1)) * 3 + ox + 1;
          if (!near) ++vtab[o];
          else if (dx || dy || dz) ++ptab[o];
        }
  }
  long long v = 0, vk = 0, p = 0, wx = 0, u = 0, vleaf = 0, wxleaf = 0, vmono = 0;
  long long vt[4] = {0, 0, 0, 0}, wt[4] = {0, 0, 0, 0};  // by (target internal?, source internal?)
  for (int l = 0; l < P.nlevels; ++l) {
    const GravLevel& L = P.lv[l];
    auto node = [&](int n) {
      vk += 512 * 189;  // the kernel's 189 offsets x 512 targets
      long long vn = 0;
      const int ti = L.leaf_slot[n] >= 0 ? 0 : 2;
      for (int o = 0; o < 27; ++o) {
        const int nb = L.nbr[(size_t)n * 27 + o];
        if (nb < 0) continue;
        vn += vtab[o];
        vt[ti + (L.leaf_slot[nb] >= 0 ? 0 : 1)] += vtab[o];
      }
      const long long wn = L.moff[(size_t)(n + 1) * 512] - L.moff[(size_t)n * 512];
      for (long long e = L.moff[(size_t)n * 512]; e < L.moff[(size_t)(n + 1) * 512]; ++e) {
        const long long enc = L.ment[(size_t)e];
        const GravLevel& S = P.lv[enc >> 40];
        wt[ti + (S.leaf_slot[(size_t)((enc & ((1LL << 40) - 1)) >> 9)] >= 0 ? 0 : 1)] += 1;
      }
      v += vn;
      wx += wn;
      // amr_m2l_mono_kernel's patches (leaf below the root, existing neighbours all leaves)
      bool mono = l > 0 && L.leaf_slot[n] >= 0;
      for (int o = 0; o < 27 && mono; ++o) {
        const int nb = L.nbr[(size_t)n * 27 + o];
        if (nb >= 0 && L.leaf_slot[nb] < 0) mono = false;
      }
      if (mono) vmono += vn;
      if (L.leaf_slot[n] >= 0) vleaf += vn, wxleaf += wn;  // L0, L_i only
    };
    if (need)
      for (int n : (*need)[l]) node(n);
    else
      for (int n = 0; n < L.n; ++n) node(n);
  }
  for (long long s = lo; s < hi; ++s) {
    const GravLevel& L = P.lv[P.slot_level[s]];
    const int n = P.slot_node[s];
    for (int o = 0; o < 27; ++o) {
      const int nb = L.nbr[(size_t)n * 27 + o];
      if (nb >= 0 && L.leaf_slot[nb] >= 0) p += ptab[o];
    }
    u += L.poff[(size_t)(n + 1) * 512] - L.poff[(size_t)n * 512];
  }
  // dense depth 2 (4^3 cells, every cell exists): the uniform 189-stencil
  for (int t = 0; t < 64; ++t) {
    const int i = t & 3, j = (t >> 2) & 3, k = t >> 4;
    for (int dz = -2 - (k & 1); dz <= 3 - (k & 1); ++dz)
      for (int dy = -2 - (j & 1); dy <= 3 - (j & 1); ++dy)
        for (int dx = -2 - (i & 1); dx <= 3 - (i & 1); ++dx) {
          if (dx >= -1 && dx <= 1 && dy >= -1 && dy <= 1 && dz >= -1 && dz <= 1) continue;
          if (i + dx >= 0 && i + dx < 4 && j + dy >= 0 && j + dy < 4 && k + dz >= 0 && k + dz < 4) ++v;
        }
  }
  out[0] = v;
  out[1] = wx;
  out[2] = p;
  out[3] = u;
  out[4] = vk;
  out[5] = vleaf;
  out[6] = wxleaf;
  for (int q = 0; q < 4; ++q) out[7 + q] = vt[q], out[11 + q] = wt[q];
  out[15] = vmono;
}

constexpr int kMaxLetPeers = 8;

// per-phase device timing of solves (bench): events at the phase boundaries
constexpr int kGravPhases = 6;  // up (P2M + owned M2M), let (moment exchange + top), m2l, l2l, l2p, am
constexpr int kGravKernels = 3;  // the M2L kernels alone: mono, fused, W/X
struct GravTimingRec {
  cudaEvent_t ev[kGravPhases + 1];
  cudaEvent_t k[kGravKernels + 1];  // brackets of the M2L kernels (serialised when timing)
};

struct LetPeer {
  unsigned long long* flags[kMaxLetPeers];  // peers' flag words (IPC-mapped)
  double* part[kMaxLetPeers];               // peers' AM sum arrays (IPC-mapped)
  unsigned long long* mine;                 // this rank's flag words (GravAmrWork::pflags)
  unsigned long long* seqp;                 // this rank's solve sequence number (pflags[4R])
  int n_push[kMaxLetPeers];                 // push CTAs per destination
  int me, world, nl;
  unsigned recv_mask;                       // ranks that store patches into this one
  unsigned am_mask;                         // ranks that store AM sums into this one
  long long seg_at, seg_n;                  // this rank's AM sums: part[seg_at, seg_at + seg_n)
  unsigned long long spin_ns;               // flag-wait limit (peer_spin_ns(); 0 = none)
};
constexpr int kAmPushCtas = 16;  // CTAs per destination of am_push_kernel

struct GravAmrWork {
  GravPlan plan;
  long long work[kWorkCounts] = {};
  bool timing = false;
  std::vector<GravTimingRec> pending;
  double phase_ms[kGravPhases + kGravKernels] = {};
  long long timed_solves = 0;
  std::vector<GLv> host_lv;
  std::vector<void*> allocs;
  GLv* dev_lv = nullptr;
  int* slot_level = nullptr;
  int* slot_node = nullptr;
  std::vector<int*> internal;
  double* dmom[3] = {nullptr, nullptr, nullptr};
  double* dloc[3] = {nullptr, nullptr, nullptr};
  double* tab = nullptr;
  double* tabp = nullptr;   // tab in amr_m2l_fused_kernel's shared layout (pad_tables_kernel)
  double* tab4p = nullptr;  // tab's monopole values in amr_m2l_mono_kernel's layout
  double* mass = nullptr;
  double* lloc = nullptr;   // [slot - lo][4][512] leaf locals L0, L_i (leaf patches only)
  double* p2p_tab = nullptr;  // [depth][27][4] same-depth P2P geometry
  int* slot_nbs = nullptr;    // [slot][27] same-depth neighbour leaf slot or -1
  double* part = nullptr;   // [P][16] + rw[22]
  double* part2 = nullptr;  // [P/256 + 1][16] tree scratch
  long long nslots = 0, P = 1;
  long long nodes = 0;
  // distributed (tmgpu_gravity_amr_distribute): this rank owns canonical
  // slots [lo, hi); M2L/L2L run over the owned leaves' ancestors only
  tmgpu_comm* comm = nullptr;
  long long lo = 0, hi = 0;
  std::vector<long long> seg_lo, seg_cnt;  // per rank (slots)
  long long seg_max = 0;                   // largest rank segment (slots)
  // locally essential tree (grav_let_plan): device lists and buffers
  bool let = false;
  unsigned long long version = 0;  // bumped by distribute / set_peer (a forest's cached step graph keys on it)
  bool root_leaf = false;  // a level-0 patch is a leaf (the dense top M2M reads its moments)
  std::vector<int*> let_owned, let_top;    // per level internal patch lists
  std::vector<long long> n_owned, n_top;
  int2* roots_all = nullptr;               // every rank's subtree roots, rank-major
  int* roots_blk = nullptr;                //   their blocks in roots_buf ([rank][max_roots])
  long long n_roots_all = 0, my_roots_at = 0, n_my_roots = 0, max_roots = 0;
  double* roots_buf = nullptr;
  int2* send_list = nullptr;               // peer-major; recv likewise
  int2* recv_list = nullptr;
  long long n_send = 0, n_recv = 0;
  std::vector<long long> send_off, send_cnt, recv_off, recv_cnt;  // in doubles, per peer
  double* send_buf = nullptr;
  double* recv_buf = nullptr;
  int* halo_slots = nullptr;
  long long n_halo_slots = 0;
  double* gather = nullptr;                // [world][seg_max][512] all-gather staging
  std::vector<int*> need;                  // per level device node list (nullptr = all)
  std::vector<long long> nneed;
  std::vector<int*> l2l_nodes;      // per level: internal patches needing L2L
  std::vector<long long> nl2l;
  int2* m2l_work = nullptr;  // fused M2L launch: (level, node) per CTA
  long long m2l_ctas = 0;
  long long* mono_slots = nullptr;  // amr_m2l_mono_kernel: leaf patches among leaf patches (slot)
  long long mono_ctas = 0;
  long long mono_local = 0;  // the first mono_local have only this rank's leaves as neighbours
  long long m2l_local = 0;   // the first m2l_local fused patches read only this rank's subtrees
  cudaEvent_t ev_up = nullptr, ev_fl = nullptr;  // owned upward pass done; local fused M2L done
  long long u_max = 0;  // most cross-depth U entries of a level
  WxTarget* wx_targets_dev = nullptr;  // W/X kernel targets: internal ones, then leaf ones, in patch order
  long long wx_n_int = 0;              // the internal targets (their locals feed L2L)
  cudaEvent_t ev_wx = nullptr, ev_wxl = nullptr;  // V sums done; leaf targets' W/X done
  long long wx_targets = 0;

  double* wx_geo = nullptr;  // [distinct W/X separations][13]
  double* wx_geo4 = nullptr;  // the same rows' first 4 values (a leaf target's monopole term), 32-byte rows
  double* u_geo = nullptr;   // [distinct cross-depth U separations][4]
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaStream_t side2 = nullptr;  // the mono M2L, concurrent with the fused one
  cudaEvent_t ev_fork2 = nullptr, ev_join2 = nullptr;
  // peer-memory LET exchange (tmgpu_gravity_amr_set_peer): subtree roots and
  // halo patches stored straight into the peers' level moment arrays
  bool peer = false;
  LetPeer pt{};
  // [0,R) moment arrival, [R,2R) consumption, [2R,3R) push counters, [3R,4R) AM-sum arrival
  unsigned long long* pflags = nullptr;
  int4* push = nullptr;                  // (level, node, destination rank) per CTA
  long long n_push = 0;
  double** peer_mom = nullptr;           // [R][nlevels] peers' moment arrays
  std::vector<void*> peer_opened;
};

// Peer LET exchange: one CTA per (patch, destination) copies the patch's 512
// cells x 10 moments into the destination's moment array at the same (level,
// node) — after the destination has consumed the previous solve's patches —
// and the last CTA for a destination raises its arrival flag.
__global__ void __launch_bounds__(256) let_push_kernel(const GLv* __restrict__ Lv,
                                                       const int4* __restrict__ items,
                                                       double* const* __restrict__ peer_mom, LetPeer t) {
  const unsigned long long seq = *t.seqp;  // this solve's (let_bump_kernel ran before on the stream)
  const int4 it = items[blockIdx.x];
  const int q = it.z;
  if (threadIdx.x == 0) spin_geq(t.mine + t.world + q, seq - 1, t.spin_ns);
  __syncthreads();
  const double2* src = reinterpret_cast<const double2*>(Lv[it.x].mom + (long long)it.y * 5120);
  double2* dst = reinterpret_cast<double2*>(peer_mom[q * t.nl + it.x] + (long long)it.y * 5120);
  for (int k = threadIdx.x; k < 2560; k += blockDim.x) dst[k] = src[k];
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long* cnt = t.mine + 2 * t.world + q;
    if (atomicAdd(cnt, 1ull) == (unsigned long long)t.n_push[q] - 1) {
      *cnt = 0;
      __threadfence_system();
      st_release_sys(t.flags[q] + t.me, seq);
    }
  }
}

__global__ void let_wait_kernel(LetPeer t) {
  const unsigned long long seq = *t.seqp;
  if (threadIdx.x == 0)
    for (int s = 0; s < t.world; ++s)
      if (t.recv_mask >> s & 1u) spin_geq(t.mine + s, seq, t.spin_ns);
}

// after the solve's last reader of received patches and AM sums: every rank
// that stores into this one may store the next solve's
__global__ void let_done_kernel(LetPeer t) {
  const unsigned long long seq = *t.seqp;
  if (threadIdx.x == 0) {
    __threadfence_system();
    const unsigned from = t.recv_mask | t.am_mask;
    for (int s = 0; s < t.world; ++s)
      if (from >> s & 1u) st_release_sys(t.flags[s] + t.world + t.me, seq);
  }
}

// AM sums: this rank's slot segment of `part` to every peer (same offsets),
// kAmPushCtas CTAs per destination; arrival flags at [3R + me].
__global__ void __launch_bounds__(256) am_push_kernel(const double* __restrict__ part, LetPeer t) {
  const unsigned long long seq = *t.seqp;
  int q = blockIdx.x / kAmPushCtas;
  q += q >= t.me;
  const int c = blockIdx.x % kAmPushCtas;
  if (threadIdx.x == 0) spin_geq(t.mine + t.world + q, seq - 1, t.spin_ns);
  __syncthreads();
  const long long per = (t.seg_n + kAmPushCtas - 1) / kAmPushCtas;
  const long long b = t.seg_at + c * per, e = min(t.seg_at + t.seg_n, b + per);
  for (long long k = b + threadIdx.x; k < e; k += blockDim.x) t.part[q][k] = part[k];
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long* cnt = t.mine + 2 * t.world + q;
    if (atomicAdd(cnt, 1ull) == (unsigned long long)kAmPushCtas - 1) {
      *cnt = 0;
      __threadfence_system();
      st_release_sys(t.flags[q] + 3 * t.world + t.me, seq);
    }
  }
}

// the next solve's sequence number (one thread, stream-ordered)
__global__ void let_bump_kernel(unsigned long long* p) { *p += 1; }

__global__ void am_wait_kernel(LetPeer t) {
  const unsigned long long seq = *t.seqp;
  if (threadIdx.x == 0)
    for (int s = 0; s < t.world; ++s)
      if (t.am_mask >> s & 1u) spin_geq(t.mine + 3 * t.world + s, seq, t.spin_ns);
}

// collective (tmgpu_gravity_amr_set_peer on every rank): barrier, unmap the
// peers' buffers, barrier, then free what this rank exported (see the forest's
// peer_close); otherwise a local release (destroy)
static void let_peer_close(GravAmrWork& w, bool collective = false) {
  if (w.pflags || w.peer) cudaDeviceSynchronize();
  const bool coll = collective && w.peer && w.comm && comm_world(w.comm) > 1;
  std::string why;
  if (coll) comm_barrier(w.comm, &why);
  for (void* p : w.peer_opened)
    if (p) cudaIpcCloseMemHandle(p);
  w.peer_opened.clear();
  if (coll) comm_barrier(w.comm, &why);
  for (void* p : {(void*)w.pflags, (void*)w.push, (void*)w.peer_mom})
    if (p) cudaFree(p);
  w.pflags = nullptr;
  w.push = nullptr;
  w.peer_mom = nullptr;
  w.n_push = 0;
  w.pt = LetPeer{};
  w.peer = false;
}

// Distributed: base[slot * per_slot ..] of every rank's slot range to every
// rank — one ncclAllGather of the padded per-rank segments through the
// staging buffer, then each remote segment into place.
static int allgather_slots(GravAmrWork& w, double* base, int per_slot, cudaStream_t st, cudaError_t* e,
                           std::string* why) {
  const int R = (int)w.seg_lo.size(), me = comm_rank(w.comm);
  const size_t per = (size_t)w.seg_max * per_slot;
  double* mine = w.gather + (size_t)me * per;
  *e = cudaMemcpyAsync(mine, base + w.lo * per_slot, (size_t)(w.hi - w.lo) * per_slot * sizeof(double),
                       cudaMemcpyDeviceToDevice, st);
  if (*e != cudaSuccess) return TMGPU_OK;
  int rc = comm_allgather(w.comm, mine, w.gather, per, st, why);
  for (int r = 0; r < R && *e == cudaSuccess && rc == TMGPU_OK; ++r)
    if (r != me && w.seg_cnt[r])
      *e = cudaMemcpyAsync(base + w.seg_lo[r] * per_slot, w.gather + (size_t)r * per,
                           (size_t)w.seg_cnt[r] * per_slot * sizeof(double), cudaMemcpyDeviceToDevice, st);
  return rc;
}

// device side of grav_let_plan (tmgpu_gravity_amr_distribute)
static cudaError_t build_let(GravAmrWork& w, const std::vector<long long>& bounds, int me) {
  const GravPlan& P = w.plan;
  const GravLetPlan G = grav_let_plan(P, bounds, me);
  const int R = (int)bounds.size() - 1;
  auto own = [&w](void* p) {
    if (p) w.allocs.push_back(p);
  };
  cudaError_t e = cudaSuccess;
  w.let_owned.assign(P.nlevels, nullptr);
  w.let_top.assign(P.nlevels, nullptr);
  w.n_owned.assign(P.nlevels, 0);
  w.n_top.assign(P.nlevels, 0);
  for (int l = 0; l < P.nlevels && e == cudaSuccess; ++l) {
    w.n_owned[l] = (long long)G.owned_internal[l].size();
    w.n_top[l] = (long long)G.top_internal[l].size();
    e = upload(G.owned_internal[l], &w.let_owned[l]);
    own(w.let_owned[l]);
    if (e == cudaSuccess) e = upload(G.top_internal[l], &w.let_top[l]), own(w.let_top[l]);
  }
  std::vector<int2> roots;
  std::vector<int> blk;
  w.max_roots = 1;
  for (int r = 0; r < R; ++r) w.max_roots = std::max(w.max_roots, (long long)G.roots[r].size());
  for (int r = 0; r < R; ++r) {
    if (r == me) w.my_roots_at = (long long)roots.size(), w.n_my_roots = (long long)G.roots[r].size();
    for (size_t i = 0; i < G.roots[r].size(); ++i) {
      roots.push_back(make_int2(G.roots[r][i].level, G.roots[r][i].node));
      blk.push_back((int)(r * w.max_roots + (long long)i));
    }
  }
  w.n_roots_all = (long long)roots.size();
  if (e == cudaSuccess) e = upload(roots, &w.roots_all), own(w.roots_all);
  if (e == cudaSuccess) e = upload(blk, &w.roots_blk), own(w.roots_blk);
  if (e == cudaSuccess)
    e = cudaMalloc(&w.roots_buf, (size_t)R * w.max_roots * 5120 * sizeof(double)), own(w.roots_buf);
  std::vector<int2> sl, rl;
  w.send_off.assign(R, 0), w.send_cnt.assign(R, 0), w.recv_off.assign(R, 0), w.recv_cnt.assign(R, 0);
  for (int q = 0; q < R; ++q) {
    w.send_off[q] = (long long)sl.size() * 5120;
    w.send_cnt[q] = (long long)G.send[q].size() * 5120;
    for (const PatchRef& p : G.send[q]) sl.push_back(make_int2(p.level, p.node));
    w.recv_off[q] = (long long)rl.size() * 5120;
    w.recv_cnt[q] = (long long)G.recv[q].size() * 5120;
    for (const PatchRef& p : G.recv[q]) rl.push_back(make_int2(p.level, p.node));
  }
  w.n_send = (long long)sl.size();
  w.n_recv = (long long)rl.size();
  if (e == cudaSuccess) e = upload(sl, &w.send_list), own(w.send_list);
  if (e == cudaSuccess) e = upload(rl, &w.recv_list), own(w.recv_list);
  if (e == cudaSuccess)
    e = cudaMalloc(&w.send_buf, (size_t)(w.n_send ? w.n_send : 1) * 5120 * sizeof(double)), own(w.send_buf);
  if (e == cudaSuccess)
    e = cudaMalloc(&w.recv_buf, (size_t)(w.n_recv ? w.n_recv : 1) * 5120 * sizeof(double)), own(w.recv_buf);
  w.n_halo_slots = (long long)G.halo_leaf_slots.size();
  if (e == cudaSuccess) e = upload(G.halo_leaf_slots, &w.halo_slots), own(w.halo_slots);
  if (e == cudaSuccess) w.let = true;
  return e;
}

// internal patches that need the L2L pass, per level (leaf patches: in L2P)
static cudaError_t build_l2l_lists(GravAmrWork& w, const std::vector<std::vector<int>>* need) {
  const GravPlan& P = w.plan;
  for (auto* p : w.l2l_nodes)
    if (p) {
      cudaFree(p);
      w.allocs.erase(std::find(w.allocs.begin(), w.allocs.end(), (void*)p));
    }
  w.l2l_nodes.assign(P.nlevels, nullptr);
  w.nl2l.assign(P.nlevels, 0);
  cudaError_t e = cudaSuccess;
  for (int l = 1; l < P.nlevels && e == cudaSuccess; ++l) {
    std::vector<int> ids;
    if (need) {
      for (int n : (*need)[l])
        if (P.lv[l].leaf_slot[n] < 0) ids.push_back(n);
    } else {
      ids = P.lv[l].internal;
    }
    w.nl2l[l] = (long long)ids.size();
    e = upload(ids, &w.l2l_nodes[l]);
    if (w.l2l_nodes[l]) w.allocs.push_back(w.l2l_nodes[l]);
  }
  return e;
}

// (level, node) list of the fused M2L launch: every needed node of every level
static cudaError_t build_m2l_work(GravAmrWork& w, const std::vector<std::vector<int>>* need) {
  std::vector<int2> wk, wk_all;
  std::vector<long long> mono;
  for (int l = 0; l < w.plan.nlevels; ++l) {
    if (need) {
      for (int n : (*need)[l]) wk_all.push_back(make_int2(l, n));
    } else {
      for (int n = 0; n < w.plan.lv[l].n; ++n) wk_all.push_back(make_int2(l, n));
    }
  }
  // leaf patches (below the root) whose existing neighbours are all leaf
  // patches go to the monopole-source kernel; the rest to the fused kernel
  const bool mono_on = std::getenv("TMGPU_M2L_MONO") == nullptr || std::getenv("TMGPU_M2L_MONO")[0] != '0';
  for (const int2& x : wk_all) {
    const GravLevel& L = w.plan.lv[x.x];
    bool all_leaf = mono_on && x.x > 0 && L.leaf_slot[x.y] >= 0;
    for (int o = 0; o < 27 && all_leaf; ++o) {
      const int nb = L.nbr[(size_t)x.y * 27 + o];
      if (nb >= 0 && L.leaf_slot[nb] < 0) all_leaf = false;
    }
    if (all_leaf)
      mono.push_back(L.leaf_slot[x.y]);
    else
      wk.push_back(x);
  }
  // distributed: the mono patches whose neighbours are all this rank's own
  // leaves first — they need only local masses and start with the solve,
  // beside the upward pass and the moment exchange (w.mono_local of them)
  auto local_mono = [&](long long slot) {
    const GravLevel& L = w.plan.lv[w.plan.slot_level[(size_t)slot]];
    const int n = w.plan.slot_node[(size_t)slot];
    for (int o = 0; o < 27; ++o) {
      const int nb = L.nbr[(size_t)n * 27 + o];
      if (nb < 0) continue;
      const long long ls = L.leaf_slot[(size_t)nb];
      if (ls < w.lo || ls >= w.hi) return false;
    }
    return true;
  };
  w.mono_local = std::stable_partition(mono.begin(), mono.end(), local_mono) - mono.begin();
  // distributed: the patches whose existing neighbours all lie in this rank's
  // own subtrees first (their sources' moments come from the owned upward
  // pass, their leaf sources' masses are local): they run beside the moment
  // exchange (w.m2l_local of them). A patch is this rank's when every leaf of
  // its subtree is (leaf slots are a Morton DFS, so subtrees are slot ranges)
  std::vector<std::vector<char>> mine(w.plan.nlevels);
  for (int l = w.plan.nlevels - 1; l >= 0; --l) {
    const GravLevel& L = w.plan.lv[l];
    mine[l].assign(L.n, 0);
    for (int n = 0; n < L.n; ++n) {
      if (L.leaf_slot[n] >= 0) {
        mine[l][n] = L.leaf_slot[n] >= w.lo && L.leaf_slot[n] < w.hi;
        continue;
      }
      bool all = true;
      for (int c = 0; c < 8 && all; ++c) all = mine[l + 1][L.child[(size_t)n * 8 + c]] != 0;
      mine[l][n] = all;
    }
  }
  auto local_patch = [&](const int2& x) {
    const GravLevel& L = w.plan.lv[x.x];
    for (int o = 0; o < 27; ++o) {
      const int nb = L.nbr[(size_t)x.y * 27 + o];
      if (nb >= 0 && !mine[x.x][nb]) return false;
    }
    return true;
  };
  const auto split = need ? std::stable_partition(wk.begin(), wk.end(), local_patch) : wk.begin();
  w.m2l_local = split - wk.begin();
  // within each part the heavier internal patches (all ten locals) first: the
  // last waves are then the lighter leaf patches, and the concurrent mono
  // kernel fills the tail
  auto internal_first = [&](const int2& x) { return w.plan.lv[x.x].leaf_slot[x.y] < 0 || x.x == 0; };
  std::stable_partition(wk.begin(), split, internal_first);
  std::stable_partition(split, wk.end(), internal_first);
  auto drop = [&w](void*& p) {
    if (!p) return;
    cudaFree(p);
    w.allocs.erase(std::find(w.allocs.begin(), w.allocs.end(), p));
    p = nullptr;
  };
  drop(reinterpret_cast<void*&>(w.m2l_work));
  drop(reinterpret_cast<void*&>(w.mono_slots));
  w.mono_ctas = (long long)mono.size();
  drop(reinterpret_cast<void*&>(w.wx_targets_dev));

  w.m2l_ctas = (long long)wk.size();
  // targets with W/X entries among the M2L patches, in patch order (source locality)
  std::vector<std::pair<long long, std::pair<int, long long>>> tg;
  for (const int2& x : wk_all) {
    const GravLevel& L = w.plan.lv[x.x];
    for (int c = 0; c < 512; ++c) {
      const long long f = (long long)x.y * 512 + c;
      const long long cnt = L.moff[f + 1] - L.moff[f];
      if (cnt) tg.push_back({-cnt, {x.x, f}});
    }
  }
  std::vector<WxTarget> td(tg.size());
  for (size_t i = 0; i < tg.size(); ++i) {
    const int l = tg[i].second.first;
    const long long f = tg[i].second.second;
    const GravLevel& L = w.plan.lv[l];
    const int leaf = L.leaf_slot[(size_t)(f >> 9)];
    const bool lt = leaf >= 0 && l > 0;
    td[i] = WxTarget{L.moff[(size_t)f], L.moff[(size_t)f + 1], lt ? (long long)(leaf - w.lo) * 2048 + (f & 511) : f,
                     l, lt ? 1 : 0};
  }
  // internal targets first (L2L reads their locals), then the leaf targets
  // (only L2P reads theirs: their W/X runs beside the L2L chain)
  std::stable_partition(td.begin(), td.end(), [](const WxTarget& t) { return !t.leaf; });
  w.wx_targets = (long long)tg.size();
  w.wx_n_int = (long long)std::count_if(td.begin(), td.end(), [](const WxTarget& t) { return !t.leaf; });

  cudaError_t e = upload(wk, &w.m2l_work);
  if (w.m2l_work) w.allocs.push_back(w.m2l_work);
  if (e == cudaSuccess) e = upload(mono, &w.mono_slots);
  if (w.mono_slots) w.allocs.push_back(w.mono_slots);
  if (e == cudaSuccess) e = upload(td, &w.wx_targets_dev);
  if (w.wx_targets_dev) w.allocs.push_back(w.wx_targets_dev);
  return e;
}

}  // namespace tmgpu

using namespace tmgpu;

struct tmgpu_gravity_amr {
  GravAmrWork w;
};

extern "C" {

void tmgpu_gravity_amr_destroy(tmgpu_gravity_amr* G) {
  if (!G) return;
  for (auto& r : G->w.pending) {
    for (auto& e : r.ev) cudaEventDestroy(e);
    for (auto& e : r.k) cudaEventDestroy(e);
  }
  if (G->w.ev_fork) cudaEventDestroy(G->w.ev_fork);
  if (G->w.ev_join) cudaEventDestroy(G->w.ev_join);
  if (G->w.side) cudaStreamDestroy(G->w.side);
  if (G->w.side2) cudaStreamDestroy(G->w.side2);
  if (G->w.ev_join2) cudaEventDestroy(G->w.ev_join2);
  if (G->w.ev_fork2) cudaEventDestroy(G->w.ev_fork2);
  if (G->w.ev_up) cudaEventDestroy(G->w.ev_up);
  if (G->w.ev_fl) cudaEventDestroy(G->w.ev_fl);
  if (G->w.ev_wx) cudaEventDestroy(G->w.ev_wx);
  if (G->w.ev_wxl) cudaEventDestroy(G->w.ev_wxl);
  let_peer_close(G->w);
  for (void* p : G->w.allocs)
    if (p) cudaFree(p);
  delete G;
}

tmgpu_gravity_amr* tmgpu_gravity_amr_create(const int* leaves, long long nleaves, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  auto* G = new tmgpu_gravity_amr;
  GravAmrWork& w = G->w;
  std::string why;
  if (!build_grav_plan(leaves, nleaves, w.plan, &why)) {
    set_err(err, TMGPU_ERR_INVALID, why.c_str());
    delete G;
    return nullptr;
  }
  const GravPlan& P = w.plan;
  count_work(P, nullptr, 0, nleaves, w.work);
  if ((long long)nleaves * 512 > INT32_MAX) {
    set_err(err, TMGPU_ERR_INVALID, "gravity_amr: more than 2^31 leaf cells");
    delete G;
    return nullptr;
  }
  if (P.nlevels > kMaxLevels) {
    set_err(err, TMGPU_ERR_INVALID, "gravity_amr: more than 48 refinement levels");
    delete G;
    return nullptr;
  }
  w.root_leaf = false;
  for (int ls : P.lv[0].leaf_slot) w.root_leaf |= ls >= 0;
  w.nslots = nleaves;
  w.hi = nleaves;
  while (w.P < nleaves) w.P <<= 1;
  cudaError_t e = cudaSuccess;
  auto track = [&](void* p) { w.allocs.push_back(p); };
  w.host_lv.resize(P.nlevels);
  w.internal.assign(P.nlevels, nullptr);
  w.need.assign(P.nlevels, nullptr);
  w.nneed.assign(P.nlevels, 0);
  for (int l = 0; l < P.nlevels; ++l) w.nneed[l] = P.lv[l].n;
  for (int l = 0; l < P.nlevels && e == cudaSuccess; ++l) {
    const GravLevel& L = P.lv[l];
    GLv& g = w.host_lv[l];
    std::memset(&g, 0, sizeof(g));
    const size_t ncell = (size_t)L.n * 512;
    w.nodes += L.n;
    e = cudaMalloc(&g.mom, ncell * 10 * sizeof(double));
    track(g.mom);
    if (e == cudaSuccess) e = cudaMemset(g.mom, 0, ncell * 10 * sizeof(double));  // leaf D, Q stay +0
    if (e == cudaSuccess) e = cudaMalloc(&g.loc, ncell * 10 * sizeof(double)), track(g.loc);
    int *ijk, *nbr, *child, *parent, *slot, *inter;
    long long *moff, *ment, *poff, *pent;
    if (e == cudaSuccess) e = upload(L.ijk, &ijk), track(ijk);
    if (e == cudaSuccess) e = upload(L.nbr, &nbr), track(nbr);
    if (e == cudaSuccess) e = upload(L.child, &child), track(child);
    if (e == cudaSuccess) e = upload(L.parent, &parent), track(parent);
    if (e == cudaSuccess) e = upload(L.leaf_slot, &slot), track(slot);
    if (e == cudaSuccess) e = upload(L.internal, &inter), track(inter);
    static_assert(sizeof(long long) == sizeof(int64_t), "int64");
    if (e == cudaSuccess)
      e = upload(reinterpret_cast<const std::vector<long long>&>(L.moff), &moff), track(moff);
    if (e == cudaSuccess)
      e = upload(reinterpret_cast<const std::vector<long long>&>(L.ment), &ment), track(ment);
    if (e == cudaSuccess)
      e = upload(reinterpret_cast<const std::vector<long long>&>(L.poff), &poff), track(poff);
    if (e == cudaSuccess)
      e = upload(reinterpret_cast<const std::vector<long long>&>(L.pent), &pent), track(pent);
    int *mgeo = nullptr, *pgeo = nullptr;
    if (e == cudaSuccess) {  // leaf-cell sources marked ~row (monopole term in amr_wx_kernel)
      std::vector<int> mg(L.mgeo);
      for (size_t q = 0; q < mg.size(); ++q) {
        const long long enc = L.ment[q];
        const GravLevel& S = P.lv[enc >> 40];
        if (S.leaf_slot[(size_t)((enc & ((1LL << 40) - 1)) >> 9)] >= 0) mg[q] = ~mg[q];
      }
      e = upload(mg, &mgeo), track(mgeo);
    }
    if (e == cudaSuccess) e = upload(L.pgeo, &pgeo), track(pgeo);
    int *mmi = nullptr, *pmi = nullptr;
    if (e == cudaSuccess) {  // leaf-mass indices of leaf-cell W/X sources and of U sources
      auto mass_index = [&](long long enc) -> int {
        const GravLevel& S = P.lv[enc >> 40];
        const long long flat = enc & ((1LL << 40) - 1);
        const int ls = S.leaf_slot[(size_t)(flat >> 9)];
        return ls >= 0 ? (int)((long long)ls * 512 + (flat & 511)) : -1;
      };
      std::vector<int> mi(L.ment.size()), pi(L.pent.size());
      for (size_t q = 0; q < mi.size(); ++q) mi[q] = mass_index(L.ment[q]);
      for (size_t q = 0; q < pi.size(); ++q) pi[q] = mass_index(L.pent[q]);
      e = upload(mi, &mmi), track(mmi);
      if (e == cudaSuccess) e = upload(pi, &pmi), track(pmi);
    }
    if (e != cudaSuccess) break;
    g.mmi = mmi, g.pmi = pmi;
    g.ijk = ijk, g.nbr = nbr, g.child = child, g.parent = parent, g.leaf_slot = slot;
    g.moff = moff, g.ment = ment, g.poff = poff, g.pent = pent, g.mgeo = mgeo, g.pgeo = pgeo;
    g.nu = (long long)L.pent.size();
    w.u_max = std::max(w.u_max, g.nu);
    if (e == cudaSuccess) e = cudaMalloc(&g.unm, (size_t)(g.nu ? g.nu : 1) * sizeof(double)), track(g.unm);
    w.internal[l] = inter;
  }
  if (e == cudaSuccess) e = cudaMalloc(&w.dev_lv, P.nlevels * sizeof(GLv)), track(w.dev_lv);
  if (e == cudaSuccess)
    e = cudaMemcpy(w.dev_lv, w.host_lv.data(), P.nlevels * sizeof(GLv), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = upload(P.slot_level, &w.slot_level), track(w.slot_level);
  if (e == cudaSuccess) e = upload(P.slot_node, &w.slot_node), track(w.slot_node);
  for (int d = 0; d < 3 && e == cudaSuccess; ++d) {
    const size_t n3 = (size_t)1 << (3 * d);
    e = cudaMalloc(&w.dmom[d], n3 * 10 * sizeof(double));
    track(w.dmom[d]);
    if (e == cudaSuccess) e = cudaMalloc(&w.dloc[d], n3 * 10 * sizeof(double)), track(w.dloc[d]);
  }
  const int Dmax = P.nlevels - 1 + 3;
  if (e == cudaSuccess) e = cudaMalloc(&w.tab, (size_t)(Dmax + 1) * kOff3 * kTab * sizeof(double)), track(w.tab);
  if (e == cudaSuccess) e = cudaMalloc(&w.mass, (size_t)w.nslots * 512 * sizeof(double)), track(w.mass);
  if (e == cudaSuccess) e = cudaMalloc(&w.lloc, (size_t)w.nslots * 2048 * sizeof(double)), track(w.lloc);
  if (e == cudaSuccess) {
    std::vector<int> nbs((size_t)nleaves * 27, -1);
    for (long long sl = 0; sl < nleaves; ++sl) {
      const GravLevel& L = P.lv[P.slot_level[sl]];
      const int nd = P.slot_node[sl];
      for (int o = 0; o < 27; ++o) {
        const int nb = L.nbr[(size_t)nd * 27 + o];
        nbs[(size_t)sl * 27 + o] = nb >= 0 ? L.leaf_slot[nb] : -1;
      }
    }
    e = upload(nbs, &w.slot_nbs), track(w.slot_nbs);
  }
  if (e == cudaSuccess) e = cudaMalloc(&w.part, ((size_t)w.P * 16 + 22) * sizeof(double)), track(w.part);
  if (e == cudaSuccess) e = cudaMalloc(&w.part2, ((size_t)w.P / 256 + 1) * 16 * sizeof(double)), track(w.part2);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(amr_m2l_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)kM2lSmem);
  if (e == cudaSuccess) e = build_m2l_work(w, nullptr);
  if (e == cudaSuccess) e = build_l2l_lists(w, nullptr);
  // the one-CTA dense top M2L on a high-priority stream: its CTA takes the first
  // free SM instead of queueing behind every CTA of the concurrent patch M2L
  int prio_lo = 0, prio_hi = 0;
  if (e == cudaSuccess) e = cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&w.side, cudaStreamNonBlocking, prio_hi);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&w.ev_fork, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&w.ev_join, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&w.side2, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&w.ev_join2, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&w.ev_fork2, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&w.ev_up, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&w.ev_fl, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&w.ev_wx, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&w.ev_wxl, cudaEventDisableTiming);

  for (int kind = 0; kind < 2 && e == cudaSuccess; ++kind) {
    const std::vector<double>& sep = kind == 0 ? P.wx_sep : P.u_sep;
    const long long ns = (long long)sep.size() / 3;
    double** geo = kind == 0 ? &w.wx_geo : &w.u_geo;
    double* dsep = nullptr;
    e = cudaMalloc(geo, (size_t)(ns ? ns : 1) * (kind == 0 ? kTab : 4) * sizeof(double));
    track(*geo);
    if (e == cudaSuccess && ns) e = upload(sep, &dsep);
    if (e == cudaSuccess && ns) {
      sep_geom_kernel<<<(unsigned)((ns + 127) / 128), 128>>>(dsep, ns, *geo, kind);
      g_launches.fetch_add(1, std::memory_order_relaxed);
      e = cudaDeviceSynchronize();
    }
    if (e == cudaSuccess && kind == 0) {
      e = cudaMalloc(&w.wx_geo4, (size_t)(ns ? ns : 1) * 4 * sizeof(double));
      track(w.wx_geo4);
      if (e == cudaSuccess && ns)
        e = cudaMemcpy2D(w.wx_geo4, 4 * sizeof(double), w.wx_geo, kTab * sizeof(double), 4 * sizeof(double),
                         (size_t)ns, cudaMemcpyDeviceToDevice);
    }
    if (dsep) cudaFree(dsep);
  }
  if (e == cudaSuccess) e = cudaMalloc(&w.p2p_tab, (size_t)(Dmax + 1) * 27 * 4 * sizeof(double)), track(w.p2p_tab);
  if (e == cudaSuccess) {
    p2p_table_kernel<<<((Dmax + 1) * 27 + 127) / 128, 128>>>(w.p2p_tab, Dmax);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    e = cudaMemcpyToSymbol(c_p2p_unit, w.p2p_tab, 27 * 4 * sizeof(double), 0, cudaMemcpyDeviceToDevice);
    double dv[kMaxLevels];
    for (int l = 0; l < kMaxLevels; ++l) {
      const double h = 1.0 / (double)(8LL << l);
      dv[l] = h * h * h;
    }
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_level_dv, dv, sizeof(dv));
    stencil_table_kernel<<<((Dmax + 1) * kOff3 + 127) / 128, 128>>>(w.tab, Dmax);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    e = cudaMalloc(&w.tabp, (size_t)(Dmax + 1) * kTabDoubles * sizeof(double));
    track(w.tabp);
    if (e == cudaSuccess) e = cudaMalloc(&w.tab4p, (size_t)(Dmax + 1) * kOff3 * 4 * sizeof(double)), track(w.tab4p);
    if (e == cudaSuccess) {
      pad_tables_kernel<<<(unsigned)(((long long)(Dmax + 1) * kTabDoubles + 255) / 256), 256>>>(w.tab, Dmax, w.tabp,
                                                                                             w.tab4p);
      g_launches.fetch_add(1, std::memory_order_relaxed);
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
  }
  if (e != cudaSuccess) {
    cuda_err(err, e, "tmgpu_gravity_amr_create");
    tmgpu_gravity_amr_destroy(G);
    return nullptr;
  }
  return G;
}

int tmgpu_gravity_amr_info(const tmgpu_gravity_amr* G, long long* out) {
  if (!G || !out) return TMGPU_ERR_INVALID;
  out[0] = G->w.plan.nlevels;
  out[1] = G->w.nodes;
  out[2] = G->w.plan.m_entries;
  out[3] = G->w.plan.p_entries;
  return TMGPU_OK;
}

// Host-only (tests): per-level counts of the patches a rank owning canonical
// slots [lo, hi) evaluates M2L/L2L for (grav_owned_ancestors); returns levels.
int tmgpu_gravity_amr_plan_need(const int* leaves, long long nleaves, long long lo, long long hi,
                                long long* counts, int max_levels, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  GravPlan P;
  std::string why;
  if (!build_grav_plan(leaves, nleaves, P, &why)) return -set_err(err, TMGPU_ERR_INVALID, why.c_str());
  if (lo < 0 || hi > nleaves || lo > hi) return -set_err(err, TMGPU_ERR_INVALID, "slot range");
  const auto lists = grav_owned_ancestors(P, lo, hi);
  for (int l = 0; l < P.nlevels && l < max_levels; ++l) counts[l] = (long long)lists[l].size();
  return P.nlevels;
}

// Host-only (tests, diagnostics): the LET plan of rank `me` of `world` with
// canonical slot bounds[world + 1]: out[0..3] = owned internal, shared top,
// own subtree roots, halo leaf patches; send[q] / recv[q] = patch counts and
// send_hash[q] / recv_hash[q] = an order-sensitive hash of the patch lists
// (rank r's send list to q must equal q's receive list from r).
int tmgpu_gravity_amr_let_plan(const int* leaves, long long nleaves, const long long* bounds, int world,
                               int me, long long* out, long long* send, long long* recv,
                               long long* send_hash, long long* recv_hash, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  GravPlan P;
  std::string why;
  if (!build_grav_plan(leaves, nleaves, P, &why)) return set_err(err, TMGPU_ERR_INVALID, why.c_str());
  const GravLetPlan G = grav_let_plan(P, std::vector<long long>(bounds, bounds + world + 1), me);
  out[0] = out[1] = 0;
  for (int l = 0; l < P.nlevels; ++l) {
    out[0] += (long long)G.owned_internal[l].size();
    out[1] += (long long)G.top_internal[l].size();
  }
  out[2] = (long long)G.roots[me].size();
  out[3] = (long long)G.halo_leaf_slots.size();
  auto hash = [](const std::vector<PatchRef>& v) {
    unsigned long long h = 1469598103934665603ULL;
    for (const PatchRef& p : v) h = (h ^ (unsigned long long)(p.level * 1000003LL + p.node)) * 1099511628211ULL;
    return (long long)(h >> 1);
  };
  for (int q = 0; q < world; ++q) {
    send[q] = (long long)G.send[q].size();
    recv[q] = (long long)G.recv[q].size();
    send_hash[q] = hash(G.send[q]);
    recv_hash[q] = hash(G.recv[q]);
  }
  return TMGPU_OK;
}

// Host-only: build the plan and report info[4] without touching the GPU.
int tmgpu_gravity_amr_plan_info(const int* leaves, long long nleaves, long long* out,
                                tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  GravPlan P;
  std::string why;
  if (!build_grav_plan(leaves, nleaves, P, &why)) return set_err(err, TMGPU_ERR_INVALID, why.c_str());
  long long nodes = 0;
  for (const auto& L : P.lv) nodes += L.n;
  out[0] = P.nlevels;
  out[1] = nodes;
  out[2] = P.m_entries;
  out[3] = P.p_entries;
  return TMGPU_OK;
}

int tmgpu_gravity_amr_mass_from_arena(tmgpu_gravity_amr* G, const double* arena, int vars,
                                      void* stream, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  GravAmrWork& w = G->w;
  cudaStream_t st = as_stream(stream);
  amr_mass_kernel<<<grid_for((w.hi - w.lo) * 512), 128, 0, st>>>(arena, vars, w.hi - w.lo, w.lo,
                                                                 w.slot_level, w.mass);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cuda_err(err, cudaGetLastError(), "tmgpu_gravity_amr_mass_from_arena");
}

int tmgpu_gravity_amr_mass_from_density(tmgpu_gravity_amr* G, const double* rho, void* stream,
                                        tmgpu_error* err) {
  return tmgpu_gravity_amr_mass_from_compact(G, rho, 512, stream, err);
}

int tmgpu_gravity_amr_mass_from_compact(tmgpu_gravity_amr* G, const double* rho, long long slot_stride,
                                        void* stream, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (!G || !rho || slot_stride < 512) return set_err(err, TMGPU_ERR_INVALID, "gravity mass_from_compact: bad argument");
  GravAmrWork& w = G->w;
  cudaStream_t st = as_stream(stream);
  amr_mass_kernel<<<grid_for((w.hi - w.lo) * 512), 128, 0, st>>>(rho, 0, w.hi - w.lo, w.lo, w.slot_level,
                                                                 w.mass, slot_stride);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cuda_err(err, cudaGetLastError(), "tmgpu_gravity_amr_mass_from_density");
}

int tmgpu_gravity_amr_solve(tmgpu_gravity_amr* G, const double* mass, double* phi, double* g,
                            int flags, void* stream, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  GravAmrWork& w = G->w;
  const GravPlan& P = w.plan;
  cudaStream_t st = as_stream(stream);
  const long long nloc = w.hi - w.lo;  // output slots (all of them on one GPU)
  const long long ncell = w.nslots * 512, nout = nloc * 512;
  const bool host = (flags & TMGPU_HOST_PTRS) != 0;
  cudaError_t e = cudaSuccess;
  std::string why;
  double *dphi = phi, *dg = g;
  if (mass)  // this rank's masses (all of them on one GPU)
    e = cudaMemcpyAsync(w.mass + w.lo * 512, mass, nout * sizeof(double),
                        host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st);
  if (host && e == cudaSuccess) {
    e = cudaMallocAsync(&dphi, nout * sizeof(double), st);
    if (e == cudaSuccess) e = cudaMallocAsync(&dg, 3 * nout * sizeof(double), st);
  }
  GravTimingRec rec;
  const bool timed = w.timing && e == cudaSuccess;
  if (timed) {
    for (auto& ev : rec.ev) cudaEventCreate(&ev);
    for (auto& ev : rec.k) cudaEventCreate(&ev);
    cudaEventRecord(rec.ev[0], st);
  }
  int rc = TMGPU_OK;
  // the mono M2L needs only the leaf masses (and, distributed, the halo
  // leaves' masses that come with the moment exchange): on one GPU it starts
  // now on its own stream and overlaps the whole upward pass
  // (a timed solve runs the three M2L kernels one after another on `st`
  // instead, each between its own events: their durations measured alone)
  const bool mono_early = !w.let && w.mono_ctas > 0 && !timed;
  // distributed: the mono patches with only local neighbours start now too
  const long long mono_pre = (w.let && !timed && !w.root_leaf) ? w.mono_local : 0;
  // (one GPU) the U sources' masses are gathered there too, off the critical path
  const bool u_side = mono_early && w.u_max && !w.root_leaf;
  if (e == cudaSuccess && mono_pre) {
    cudaEventRecord(w.ev_fork2, st);
    cudaStreamWaitEvent(w.side2, w.ev_fork2, 0);
    amr_m2l_mono_kernel<<<(unsigned)mono_pre, kM2lThreads, kMonoSmem, w.side2>>>(
        w.mono_slots, w.slot_level, w.mass, w.slot_nbs, w.tab4p, w.lloc, w.lo);
    g_launches.fetch_add(1, std::memory_order_relaxed);
  }
  if (e == cudaSuccess && mono_early) {
    cudaEventRecord(w.ev_fork2, st);
    cudaStreamWaitEvent(w.side2, w.ev_fork2, 0);
    if (u_side) {
      amr_u_gather_kernel<<<dim3((unsigned)std::min<long long>((w.u_max + 255) / 256, 1184), P.nlevels), 256, 0,
                            w.side2>>>(w.dev_lv, w.mass);
      g_launches.fetch_add(1, std::memory_order_relaxed);
    }
    amr_m2l_mono_kernel<<<(unsigned)w.mono_ctas, kM2lThreads, kMonoSmem, w.side2>>>(
        w.mono_slots, w.slot_level, w.mass, w.slot_nbs, w.tab4p, w.lloc, w.lo);
    cudaEventRecord(w.ev_join2, w.side2);
    g_launches.fetch_add(1, std::memory_order_relaxed);
  }
  if (e == cudaSuccess && rc == TMGPU_OK) {
    long long launches = 0;
    bool wx_beside = false;  // the leaf targets' W/X runs on the side stream (joined before L2P)
    // leaf cells' m is read from the leaf-mass array wherever a leaf moment
    // would be: the owned-subtree M2M (owned leaves), and after the moment
    // exchange the fused window, W/X and U (the masses of every other rank's
    // leaf patch this rank reads arrive with it: halo_mass_kernel). One GPU
    // skips P2M; distributed, leaf moments travel in the exchange (and the
    // shared-top M2M reads them), so P2M stays
    const double* lmass = !w.root_leaf ? w.mass : nullptr;
    if (nloc && (w.let || !lmass)) {
      amr_p2m_kernel<<<grid_for(nout), 128, 0, st>>>(w.mass, nloc, w.lo, w.slot_level, w.slot_node,
                                                     w.dev_lv);
      ++launches;
    }
    for (int l = P.nlevels - 2; l >= 0; --l) {  // own subtrees (all of the tree on one GPU)
      const long long ni = w.let ? w.n_owned[l] : (long long)P.lv[l].internal.size();
      if (!ni) continue;
      amr_m2m_kernel<<<grid_for(ni * 512), 128, 0, st>>>(w.dev_lv, l, w.let ? w.let_owned[l] : w.internal[l],
                                                         ni, lmass);
      ++launches;
    }
    // distributed: the fused M2L of patches that read only this rank's
    // subtrees runs now on the side stream, beside the moment exchange
    const long long m2l_pre = (w.let && !timed && !w.root_leaf) ? w.m2l_local : 0;
    if (m2l_pre) {
      cudaEventRecord(w.ev_up, st);
      cudaStreamWaitEvent(w.side, w.ev_up, 0);
      amr_m2l_fused_kernel<<<(unsigned)m2l_pre, kM2lThreads, kM2lSmem, w.side>>>(w.dev_lv, w.m2l_work, w.tabp,
                                                                                w.lloc, w.lo, lmass);
      cudaEventRecord(w.ev_fl, w.side);
      ++launches;
    }
    if (timed) cudaEventRecord(rec.ev[1], st);
    if (w.peer) {
      // roots to every peer and halo patches to their readers, straight into
      // the peers' moment arrays; then the shared top as below
      let_bump_kernel<<<1, 1, 0, st>>>(w.pt.seqp);  // device-side: a captured solve replays
      ++launches;
      if (w.n_push)
        let_push_kernel<<<(unsigned)w.n_push, 256, 0, st>>>(w.dev_lv, w.push, w.peer_mom, w.pt);
      let_wait_kernel<<<1, 32, 0, st>>>(w.pt);
      launches += 2;
      for (int l = P.nlevels - 2; l >= 0; --l) {
        if (!w.n_top[l]) continue;
        amr_m2m_kernel<<<grid_for(w.n_top[l] * 512), 128, 0, st>>>(w.dev_lv, l, w.let_top[l], w.n_top[l]);
        ++launches;
      }
      if (w.n_halo_slots) {
        halo_mass_kernel<<<grid_for(w.n_halo_slots * 512), 128, 0, st>>>(
            w.dev_lv, w.halo_slots, w.n_halo_slots, w.slot_level, w.slot_node, w.mass);
        ++launches;
      }
    } else if (w.let) {
      // LET moment exchange: subtree roots to everyone, the shared top by M2M,
      // then the owned patches other ranks read, point to point
      if (w.n_my_roots)
        pack_patches_kernel<<<(unsigned)w.n_my_roots, 256, 0, st>>>(
            w.dev_lv, w.roots_all + w.my_roots_at, w.roots_blk + w.my_roots_at, w.roots_buf);
      const size_t per = (size_t)w.max_roots * 5120;
      rc = comm_allgather(w.comm, w.roots_buf + (size_t)comm_rank(w.comm) * per, w.roots_buf, per, st, &why);
      if (rc == TMGPU_OK && w.n_roots_all)
        unpack_patches_kernel<<<(unsigned)w.n_roots_all, 256, 0, st>>>(w.dev_lv, w.roots_all, w.roots_blk,
                                                                       w.roots_buf);
      for (int l = P.nlevels - 2; l >= 0 && rc == TMGPU_OK; --l) {
        if (!w.n_top[l]) continue;
        amr_m2m_kernel<<<grid_for(w.n_top[l] * 512), 128, 0, st>>>(w.dev_lv, l, w.let_top[l], w.n_top[l]);
        ++launches;
      }
      if (rc == TMGPU_OK && w.n_send)
        pack_patches_kernel<<<(unsigned)w.n_send, 256, 0, st>>>(w.dev_lv, w.send_list, nullptr, w.send_buf);
      if (rc == TMGPU_OK)
        rc = comm_exchange(w.comm, w.send_buf, w.send_off, w.send_cnt, w.recv_buf, w.recv_off, w.recv_cnt,
                           st, &why);
      if (rc == TMGPU_OK && w.n_recv)
        unpack_patches_kernel<<<(unsigned)w.n_recv, 256, 0, st>>>(w.dev_lv, w.recv_list, nullptr, w.recv_buf);
      if (rc == TMGPU_OK && w.n_halo_slots)
        halo_mass_kernel<<<grid_for(w.n_halo_slots * 512), 128, 0, st>>>(
            w.dev_lv, w.halo_slots, w.n_halo_slots, w.slot_level, w.slot_node, w.mass);
      launches += 5;
    }
    top_m2m_kernel<<<1, 128, 0, st>>>(w.host_lv[0].mom, w.dmom[2], w.dmom[1], w.dmom[0]);
    // the dense depth-2 M2L (one small CTA) overlaps the patch M2L on a side stream
    cudaEventRecord(w.ev_fork, st);
    cudaStreamWaitEvent(w.side, w.ev_fork, 0);
    dense_m2l_staged_kernel<<<1, 128, 0, w.side>>>(w.dmom[2], w.dloc[2], w.tab + 2LL * kOff3 * kTab);
    cudaEventRecord(w.ev_join, w.side);
    launches += 2;
    if (timed) cudaEventRecord(rec.ev[2], st);
    {
      // the fused kernel (1 CTA/SM) first on the solve's stream, the mono kernel
      // (2 CTAs/SM, independent outputs) on a second stream: its CTAs take the
      // SMs the fused kernel's last waves leave idle; both join before W/X
      if (timed) {
        cudaEventRecord(rec.k[0], st);
        if (w.mono_ctas)
          amr_m2l_mono_kernel<<<(unsigned)w.mono_ctas, kM2lThreads, kMonoSmem, st>>>(
              w.mono_slots, w.slot_level, w.mass, w.slot_nbs, w.tab4p, w.lloc, w.lo);
        cudaEventRecord(rec.k[1], st);
        launches += w.mono_ctas ? 1 : 0;
      }
      if (w.m2l_ctas > m2l_pre) {
        amr_m2l_fused_kernel<<<(unsigned)(w.m2l_ctas - m2l_pre), kM2lThreads, kM2lSmem, st>>>(
            w.dev_lv, w.m2l_work + m2l_pre, w.tabp, w.lloc, w.lo, lmass);
        ++launches;
      }
      if (timed) cudaEventRecord(rec.k[2], st);
      if (w.mono_ctas && !mono_early && !timed) {  // leaf patches among leaf patches: monopole sources
        cudaStreamWaitEvent(w.side2, w.ev_fork, 0);
        if (w.mono_ctas > mono_pre) {  // (distributed: those not started at the solve's start)
          amr_m2l_mono_kernel<<<(unsigned)(w.mono_ctas - mono_pre), kM2lThreads, kMonoSmem, w.side2>>>(
              w.mono_slots + mono_pre, w.slot_level, w.mass, w.slot_nbs, w.tab4p, w.lloc, w.lo);
          ++launches;
        }
        cudaEventRecord(w.ev_join2, w.side2);
      }
      if (w.mono_ctas && !timed) cudaStreamWaitEvent(st, w.ev_join2, 0);
      if (m2l_pre) cudaStreamWaitEvent(st, w.ev_fl, 0);  // W/X follows every V sum
      const long long nwx_leaf = w.wx_targets - w.wx_n_int;
      wx_beside = !timed && nwx_leaf > 0;
      if (wx_beside) {  // the leaf targets' W/X on the side stream, beside the L2L chain
        cudaEventRecord(w.ev_wx, st);
        cudaStreamWaitEvent(w.side2, w.ev_wx, 0);
        amr_wx_kernel<<<grid_for(nwx_leaf), 128, 0, w.side2>>>(w.dev_lv, w.wx_targets_dev + w.wx_n_int, nwx_leaf,
                                                                w.wx_geo, w.lloc, lmass, w.wx_geo4);
        cudaEventRecord(w.ev_wxl, w.side2);
        ++launches;
      }
      const long long nwx_st = wx_beside ? w.wx_n_int : w.wx_targets;
      if (nwx_st) {
        amr_wx_kernel<<<grid_for(nwx_st), 128, 0, st>>>(w.dev_lv, w.wx_targets_dev, nwx_st, w.wx_geo, w.lloc,
                                                        lmass, w.wx_geo4);
        ++launches;
      }
      if (timed) cudaEventRecord(rec.k[3], st);
    }
    cudaStreamWaitEvent(st, w.ev_join, 0);
    if (timed) cudaEventRecord(rec.ev[3], st);
    l2l_kernel<<<grid_for(512), 128, 0, st>>>(w.dloc[2], w.host_lv[0].loc, 8, 1.0 / 8.0);
    ++launches;
    for (int l = 1; l < P.nlevels; ++l) {
      if (!w.nl2l[l]) continue;
      amr_l2l_kernel<<<grid_for(w.nl2l[l] * 512), 128, 0, st>>>(w.dev_lv, l, w.nl2l[l], w.l2l_nodes[l]);
      ++launches;
    }
    if (timed) cudaEventRecord(rec.ev[4], st);
    const bool am = (flags & TMGPU_GRAV_AM) != 0;
    // peer mode: peers store their segments straight into `part`; zero ours only
    if (am && w.peer)
      e = cudaMemsetAsync(w.part + w.lo * 16, 0, (size_t)(w.hi - w.lo) * 16 * sizeof(double), st);
    else if (am)
      e = cudaMemsetAsync(w.part, 0, (size_t)w.P * 16 * sizeof(double), st);
    if (w.u_max && !u_side) {  // U entries' source masses, gathered in parallel
      amr_u_gather_kernel<<<dim3((unsigned)std::min<long long>((w.u_max + 255) / 256, 1184), P.nlevels), 256, 0, st>>>(
          w.dev_lv, lmass);
      ++launches;
    }
    if (wx_beside) cudaStreamWaitEvent(st, w.ev_wxl, 0);  // the leaf locals are complete
    if (nloc)
      amr_l2p_kernel<<<(unsigned)nloc, kL2pThreads, 0, st>>>(w.dev_lv, nloc, w.lo, w.slot_level, w.slot_node,
                                                     w.mass, w.u_geo, w.lloc, w.p2p_tab, w.slot_nbs, dphi, dg,
                                                     am ? w.part : nullptr);
    ++launches;
    if (timed) cudaEventRecord(rec.ev[5], st);
    if (am) {  // the per-slot sums came with L2P
      if (w.peer && e == cudaSuccess) {  // identical global pair tree on every rank
        am_push_kernel<<<(unsigned)((w.pt.world - 1) * kAmPushCtas), 256, 0, st>>>(w.part, w.pt);
        am_wait_kernel<<<1, 32, 0, st>>>(w.pt);
        launches += 2;
      } else if (w.comm && e == cudaSuccess) {
        rc = allgather_slots(w, w.part, 16, st, &e, &why);
      }
      double* bufs[2] = {w.part, w.part2};
      int cur = 0;
      bool solved = false;  // the last pass (one CTA) solves for the field
      for (long long n = w.P; n > 1;) {
        const long long chunk = n < 256 ? n : 256;
        const bool last = n == chunk;
        am_tree_pass_kernel<<<(unsigned)(n / chunk), 256, 0, st>>>(bufs[cur], bufs[cur ^ 1], n,
                                                                   last ? w.part + w.P * 16 : nullptr);
        solved |= last;
        n /= chunk;
        cur ^= 1;
        ++launches;
      }
      if (!solved) {
        am_solve_kernel<<<1, 32, 0, st>>>(bufs[cur], w.part + w.P * 16);
        ++launches;
      }
      am_apply_kernel<<<grid_for(nout), 128, 0, st>>>(w.dev_lv, nloc, w.lo, w.slot_level, w.slot_node,
                                                      w.part + w.P * 16, dg);
      launches += 1;
    }
    if (w.peer) {  // every received patch and AM sum has been read
      let_done_kernel<<<1, 32, 0, st>>>(w.pt);
      ++launches;
    }
    g_launches.fetch_add(launches, std::memory_order_relaxed);
    if (e == cudaSuccess) e = cudaGetLastError();
  }
  if (timed) {
    cudaEventRecord(rec.ev[kGravPhases], st);
    w.pending.push_back(rec);
  }
  if (host) {
    if (e == cudaSuccess) e = cudaMemcpyAsync(phi, dphi, nout * sizeof(double), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(g, dg, 3 * nout * sizeof(double), cudaMemcpyDeviceToHost, st);
    if (dphi && dphi != phi) cudaFreeAsync(dphi, st);
    if (dg && dg != g) cudaFreeAsync(dg, st);
    cudaError_t e2 = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = e2;
  } else if (!(flags & TMGPU_ASYNC)) {
    cudaError_t e2 = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = e2;
  }
  if (rc != TMGPU_OK) return set_err(err, rc, why.c_str());
  return cuda_err(err, e, "tmgpu_gravity_amr_solve");
}

// Distributed solve: rank comm_rank(comm) owns canonical slots
// [slot_bounds[r], slot_bounds[r+1]) (contiguous ranges, partition_leaves).
// Locally essential tree (grav_let_plan): each rank computes its owned
// subtrees' moments, all-gathers the subtree roots, computes the shared top,
// and receives the owned patches of others it reads (point to point); M2L and
// L2L run only over the ancestors of the owned leaves, L2P and the AM
// correction's per-slot sums only over the owned slots (the sums are
// all-gathered, so every rank reduces the identical global pair tree).
// Outputs (phi, g) and masses are then by local slot; the result equals the
// one-GPU solve bit for bit.
int tmgpu_gravity_amr_distribute(tmgpu_gravity_amr* G, tmgpu_comm* comm, const long long* slot_bounds,
                                 tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (!G || !comm || !slot_bounds) return set_err(err, TMGPU_ERR_INVALID, "gravity distribute: null argument");
  GravAmrWork& w = G->w;
  ++w.version;
  const GravPlan& P = w.plan;
  const int R = comm_world(comm), me = comm_rank(comm);
  if (slot_bounds[0] != 0 || slot_bounds[R] != w.nslots)
    return set_err(err, TMGPU_ERR_INVALID, "gravity distribute: slot bounds must cover [0, nslots)");
  for (int r = 0; r < R; ++r)
    if (slot_bounds[r + 1] < slot_bounds[r])
      return set_err(err, TMGPU_ERR_INVALID, "gravity distribute: slot bounds not ascending");
  let_peer_close(w);  // a new distribution needs a new tmgpu_gravity_amr_set_peer
  w.comm = comm;
  w.lo = slot_bounds[me];
  w.hi = slot_bounds[me + 1];
  w.seg_lo.assign(slot_bounds, slot_bounds + R);
  w.seg_cnt.resize(R);
  w.seg_max = 0;
  for (int r = 0; r < R; ++r) {
    w.seg_cnt[r] = slot_bounds[r + 1] - slot_bounds[r];
    w.seg_max = std::max(w.seg_max, w.seg_cnt[r]);
  }
  if (w.gather) {
    cudaFree(w.gather);
    w.allocs.erase(std::find(w.allocs.begin(), w.allocs.end(), (void*)w.gather));
    w.gather = nullptr;
  }
  {
    cudaError_t e0 = cudaMalloc(&w.gather, (size_t)R * (w.seg_max ? w.seg_max : 1) * 512 * sizeof(double));
    if (e0 != cudaSuccess) return cuda_err(err, e0, "tmgpu_gravity_amr_distribute");
    w.allocs.push_back(w.gather);
  }
  cudaError_t e = cudaSuccess;
  std::vector<std::vector<int>> lists = grav_owned_ancestors(P, w.lo, w.hi);
  for (int l = 0; l < P.nlevels && e == cudaSuccess; ++l) {
    const std::vector<int>& ids = lists[l];
    if (w.need[l]) {  // an earlier distribute
      cudaFree(w.need[l]);
      w.allocs.erase(std::find(w.allocs.begin(), w.allocs.end(), (void*)w.need[l]));
    }
    w.need[l] = nullptr;
    w.nneed[l] = (long long)ids.size();
    e = upload(ids, &w.need[l]);
    if (w.need[l]) w.allocs.push_back(w.need[l]);
  }
  if (e == cudaSuccess) e = build_m2l_work(w, &lists);
  if (e == cudaSuccess) e = build_l2l_lists(w, &lists);
  if (e == cudaSuccess) e = build_let(w, std::vector<long long>(slot_bounds, slot_bounds + R + 1), me);
  count_work(P, &lists, w.lo, w.hi, w.work);  // this GPU's share (bench roofline)
  return cuda_err(err, e, "tmgpu_gravity_amr_distribute");
}

// Peer-memory LET moment exchange (collective over the solver's communicator):
// exports every level's moment array and the flag words by CUDA IPC and
// replaces the root all-gather + halo send/recv with let_push_kernel. on = 0
// returns to NCCL. Re-call after tmgpu_gravity_amr_distribute.
int tmgpu_gravity_amr_set_peer(tmgpu_gravity_amr* G, int on, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (!G) return set_err(err, TMGPU_ERR_INVALID, "null gravity solver");
  GravAmrWork& w = G->w;
  ++w.version;
  let_peer_close(w, /*collective=*/true);
  if (!on) return TMGPU_OK;
  if (!w.let || !w.comm) return set_err(err, TMGPU_ERR_INVALID, "gravity peer exchange: call distribute first");
  const GravPlan& P = w.plan;
  const int R = comm_world(w.comm), me = comm_rank(w.comm), nl = P.nlevels;
  if (R < 2 || R > kMaxLetPeers)
    return set_err(err, TMGPU_ERR_INVALID, "gravity peer exchange supports 2..8 ranks");
  std::vector<long long> bounds(R + 1);
  for (int r = 0; r < R; ++r) bounds[r] = w.seg_lo[r];
  bounds[R] = w.seg_lo[R - 1] + w.seg_cnt[R - 1];
  const GravLetPlan L = grav_let_plan(P, bounds, me);
  // per rank: flag handle, AM-sum handle, one moment-array handle per level (8 doubles
  // each), status
  const int rec_n = 8 * (2 + nl) + 1, k_ok = rec_n - 1;
  std::vector<double> rec(rec_n, 0.0), all((size_t)rec_n * R, 0.0);
  double* dbuf = nullptr;
  cudaError_t e = cudaMalloc((void**)&dbuf, sizeof(double) * rec_n * (R + 1));
  if (e != cudaSuccess) return cuda_err(err, e, "tmgpu_gravity_amr_set_peer");
  std::string why = "gravity peer exchange: setup failed on a rank";
  // every rank takes part in both all-gathers and all agree on the outcome
  auto agree = [&](bool ok, double* out) {
    rec[k_ok] = ok ? 1.0 : 0.0;
    cudaError_t ce = cudaMemcpy(dbuf, rec.data(), sizeof(double) * rec_n, cudaMemcpyHostToDevice);
    if (ce == cudaSuccess) ce = cudaDeviceSynchronize();
    int rc = ce == cudaSuccess ? comm_allgather(w.comm, dbuf, dbuf + rec_n, rec_n, nullptr, &why) : TMGPU_ERR_CUDA;
    if (rc == TMGPU_OK) ce = cudaMemcpy(out, dbuf + rec_n, sizeof(double) * rec_n * R, cudaMemcpyDeviceToHost);
    if (rc != TMGPU_OK || ce != cudaSuccess) return false;
    for (int q = 0; q < R; ++q)
      if (out[(size_t)q * rec_n + k_ok] != 1.0) return false;
    return true;
  };
  // flag words [0, 4R) and this rank's sequence counter at [4R]
  e = cudaMalloc((void**)&w.pflags, (4 * R + 1) * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemset(w.pflags, 0, (4 * R + 1) * sizeof(unsigned long long));
  cudaIpcMemHandle_t h{};
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, w.pflags);
  std::memcpy(&rec[0], &h, 64);
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, w.part);
  std::memcpy(&rec[8], &h, 64);
  for (int l = 0; l < nl && e == cudaSuccess; ++l) {
    e = cudaIpcGetMemHandle(&h, w.host_lv[l].mom);
    std::memcpy(&rec[8 * (2 + l)], &h, 64);
  }
  bool ok = agree(e == cudaSuccess, all.data());
  LetPeer t{};
  t.spin_ns = peer_spin_ns();
  t.mine = w.pflags;
  t.seqp = w.pflags + 4 * R;
  t.me = me;
  t.world = R;
  t.nl = nl;
  t.seg_at = w.lo * 16;
  t.seg_n = (w.hi - w.lo) * 16;
  std::vector<double*> pm((size_t)R * nl, nullptr);
  for (int q = 0; q < R && ok && e == cudaSuccess; ++q) {
    if (q == me) continue;
    if (!L.roots[q].empty() || !L.recv[q].empty()) t.recv_mask |= 1u << q;
    t.am_mask |= 1u << q;
    for (int k = 0; k < nl + 2 && e == cudaSuccess; ++k) {
      std::memcpy(&h, &all[(size_t)q * rec_n + 8 * k], 64);
      void* p = nullptr;
      e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) break;
      w.peer_opened.push_back(p);
      if (k == 0)
        t.flags[q] = static_cast<unsigned long long*>(p);
      else if (k == 1)
        t.part[q] = static_cast<double*>(p);
      else
        pm[(size_t)q * nl + (k - 2)] = static_cast<double*>(p);
    }
  }
  if (ok) {
    std::vector<int4> items;
    for (int q = 0; q < R; ++q) {
      if (q == me) continue;
      for (const PatchRef& r : L.roots[me]) items.push_back(make_int4(r.level, r.node, q, 0));
      for (const PatchRef& r : L.send[q]) items.push_back(make_int4(r.level, r.node, q, 0));
      t.n_push[q] = (int)(L.roots[me].size() + L.send[q].size());
    }
    w.n_push = (long long)items.size();
    if (e == cudaSuccess && !items.empty()) e = upload(items, &w.push);
    if (e == cudaSuccess) e = upload(pm, &w.peer_mom);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    // every rank has zeroed its flags and mapped its peers before anyone pushes
    std::vector<double> all2((size_t)rec_n * R);
    ok = agree(e == cudaSuccess, all2.data());
  }
  cudaFree(dbuf);
  if (!ok) {
    let_peer_close(w);
    return e != cudaSuccess ? cuda_err(err, e, "tmgpu_gravity_amr_set_peer") : set_err(err, TMGPU_ERR_CUDA, why.c_str());
  }
  w.pt = t;
  w.peer = true;
  return TMGPU_OK;
}

// AM-correction sums of the last solve with TMGPU_GRAV_AM: out[0..2] centre of
// mass, [3..5] w, [6..21] the 16 sums (tests).
int tmgpu_gravity_amr_am_stats(tmgpu_gravity_amr* G, double* out) {
  if (!G || !out) return TMGPU_ERR_INVALID;
  return cudaMemcpy(out, G->w.part + G->w.P * 16, 22 * sizeof(double), cudaMemcpyDeviceToHost) ==
                 cudaSuccess
             ? TMGPU_OK
             : TMGPU_ERR_CUDA;
}

// Algorithmic work of one solve on this GPU (after tmgpu_gravity_amr_distribute:
// its share): [0] V-list M2L pairs with an existing source (incl. the dense
// depth-2 level), [1] W/X M2L entries, [2] same-depth P2P pairs, [3] cross-depth
// U entries, [4] V-list pairs the kernel evaluates (missing neighbour patches as
// zero moments), [5] of [0] into leaf patches, [6] of [1] into leaf patches
// (those evaluate only L0 and L_i).
int tmgpu_gravity_amr_work(const tmgpu_gravity_amr* G, long long* out) {
  if (!G || !out) return TMGPU_ERR_INVALID;
  for (int q = 0; q < kWorkCounts; ++q) out[q] = G->w.work[q];
  return TMGPU_OK;
}

// Per-phase device timing (CUDA events on the solve's stream): on != 0 starts
// recording (and clears the totals); tmgpu_gravity_amr_timing syncs on the
// recorded events and returns ms totals [comm, up, m2l, l2l, l2p, am] and the count.
int tmgpu_gravity_amr_set_timing(tmgpu_gravity_amr* G, int on) {
  if (!G) return TMGPU_ERR_INVALID;
  GravAmrWork& w = G->w;
  w.timing = on != 0;
  if (on) {
    for (auto& r : w.pending) {
      for (auto& e : r.ev) cudaEventDestroy(e);
      for (auto& e : r.k) cudaEventDestroy(e);
    }
    w.pending.clear();
    for (double& x : w.phase_ms) x = 0.0;
    w.timed_solves = 0;
  }
  return TMGPU_OK;
}

int tmgpu_gravity_amr_timing(tmgpu_gravity_amr* G, double* ms, long long* solves) {
  if (!G) return TMGPU_ERR_INVALID;
  GravAmrWork& w = G->w;
  for (auto& r : w.pending) {
    if (cudaEventSynchronize(r.ev[kGravPhases]) != cudaSuccess) return TMGPU_ERR_CUDA;
    for (int q = 0; q < kGravPhases; ++q) {
      float t = 0.f;
      cudaEventElapsedTime(&t, r.ev[q], r.ev[q + 1]);
      w.phase_ms[q] += t;
    }
    for (int q = 0; q < kGravKernels; ++q) {
      float t = 0.f;
      cudaEventElapsedTime(&t, r.k[q], r.k[q + 1]);
      w.phase_ms[kGravPhases + q] += t;
    }
    for (auto& e : r.ev) cudaEventDestroy(e);
    for (auto& e : r.k) cudaEventDestroy(e);
    ++w.timed_solves;
  }
  w.pending.clear();
  if (ms)
    for (int q = 0; q < kGravPhases + kGravKernels; ++q) ms[q] = w.phase_ms[q];
  if (solves) *solves = w.timed_solves;
  return TMGPU_OK;
}

// Whether a solve enqueues the same work every call with no host-side state
// (so a CUDA graph may capture it): not timing (distributed solves qualify:
// their peer sequence numbers are in device memory, their NCCL calls capture).
bool tmgpu_gravity_amr_graph_safe(const tmgpu_gravity_amr* G) {
  return G && !G->w.timing;
}

unsigned long long tmgpu_gravity_amr_version(const tmgpu_gravity_amr* G) { return G ? G->w.version : 0; }

// Leaf-cell masses currently in the workspace ([slot][512], device pointer).
const double* tmgpu_gravity_amr_mass_ptr(const tmgpu_gravity_amr* G) { return G ? G->w.mass : nullptr; }

}  // extern "C"
