// Acoustic leapfrog step in float64 for B200 (sm_100a) + C ABI.
//
// the precision_bytes = 8 path of the reference's cost model
// (/root/reference/pkg/src/fdroof/equations.py:74-78; 32 B per point instead
// of 16, so half the operational intensity).  The per-point sequence is the
// reference step's (kernel.py:194-211) with every value in IEEE double, one
// rounding per operation and no contraction (explicit __dadd_rn / __dmul_rn /
// __ddiv_rn):
//   lap = w0 c; lap = lap + wj (c[+j] + c[-j]) for x, then y, then z;
//   s = coef lap; s = s / m; out = (2c - prev) + s; out *= (gx gy) gz;
// then the source adds series[it] and receivers sample the new level.  The
// parity oracle is oracle/acoustic.py's numpy restatement run on float64
// levels (tests/test_fp64.py).
//
// a64_queue (AUTO, QUEUE): the TMA-fed register-queue kernel of the float32
// path, one double2 per thread (below).  a64_stream (variant TMA, kept for
// comparison): a 32(z) x 8(y) tile of one point per thread streams along x.
// The 2r+1 x-neighbours of a thread's column live in a register queue; the
// y/z taps read a shared-memory box of the centre plane (zero halo written
// explicitly), double-buffered: the box of plane x+1, the queue's next value
// and this plane's prev / m are loaded into registers before plane x is
// computed, so their latency overlaps the arithmetic; one barrier per plane.
// FP64 on B200 is half the FP32 rate and the step is HBM-bound (OI 1.8).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <type_traits>

#include "../../include/b200fd.h"
#include "fdr_common.cuh"

#ifndef FDR_Q64PLAIN
#define FDR_Q64PLAIN 1  // plain / no-taper copies of the float64 plane loop (0: one general loop)
#endif

namespace fdr64 {

using fdr::cuda_fail;
using fdr::fail;

struct A64Step {
  const double* cur;
  const double* prev;
  double* out;
  const double* m;
  int nx, ny, nz, pitch_y;
  long long pitch_x;
  double w[FDR_MAX_RADIUS + 1];
  double coef;
  double m_scalar;
  int m_mode;
  int radius;
  const double* gx;
  const double* gy;
  const double* gz;
  const double* series;
  int n_series, it;
  int sx, sy, sz;
  const int* rec;
  int n_rec;
  double* traces;
  int gather_row;
  int chunk;
};

#define A64_DEV __device__ __forceinline__

A64_DEV double tapd(double lap, double w, double a, double b) {
  return __dadd_rn(lap, __dmul_rn(w, __dadd_rn(a, b)));
}

// s = coef lap / m; out = (2c - prev) + s; sponge; source
A64_DEV double finish(const A64Step& a, double c, double prev, double lap, double m, double g,
                      bool src) {
  double s = __dmul_rn(a.coef, lap);
  if (a.m_mode == FDR_M_GRID) s = __ddiv_rn(s, m);
  else if (a.m_mode == FDR_M_SCALAR) s = __ddiv_rn(s, a.m_scalar);
  double out = __dadd_rn(__dsub_rn(__dadd_rn(c, c), prev), s);
  if (a.gx) out = __dmul_rn(out, g);
  if (src) out = __dadd_rn(out, a.series[a.it]);
  return out;
}

// traces[gather_row] = cur[rec] (the previous step's new level), by the first threads
A64_DEV void gather(const A64Step& a) {
  if (a.gather_row < 0) return;
  const int nthr = blockDim.x * blockDim.y;
  const int b = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  const int stride = nthr * (int)(gridDim.x * gridDim.y * gridDim.z);
  for (int i = b * nthr + threadIdx.x + blockDim.x * threadIdx.y; i < a.n_rec; i += stride) {
    const int* r = a.rec + 3 * i;
    a.traces[(size_t)a.gather_row * a.n_rec + i] =
        a.cur[(size_t)r[0] * a.pitch_x + (size_t)r[1] * a.pitch_y + r[2]];
  }
}

__global__ void a64_gather_kernel(const double* level, const int* rec, int n_rec, double* traces,
                                  int row, int pitch_y, long long pitch_x) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_rec) {
    const int* r = rec + 3 * i;
    traces[(size_t)row * n_rec + i] = level[(size_t)r[0] * pitch_x + (size_t)r[1] * pitch_y + r[2]];
  }
}

// One thread per point (any radius): the checker variant.
__global__ void __launch_bounds__(256) a64_direct(const A64Step a) {
  gather(a);
  const int z = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  const int x = blockIdx.z;
  if (z >= a.nz || y >= a.ny) return;
  auto at = [&](int xx, int yy, int zz) -> double {
    if (xx < 0 || xx >= a.nx || yy < 0 || yy >= a.ny || zz < 0 || zz >= a.nz) return 0.0;
    return a.cur[(size_t)xx * a.pitch_x + (size_t)yy * a.pitch_y + zz];
  };
  const size_t p = (size_t)x * a.pitch_x + (size_t)y * a.pitch_y + z;
  const double c = a.cur[p];
  double lap = __dmul_rn(a.w[0], c);
  for (int j = 1; j <= a.radius; ++j) lap = tapd(lap, a.w[j], at(x + j, y, z), at(x - j, y, z));
  for (int j = 1; j <= a.radius; ++j) lap = tapd(lap, a.w[j], at(x, y + j, z), at(x, y - j, z));
  for (int j = 1; j <= a.radius; ++j) lap = tapd(lap, a.w[j], at(x, y, z + j), at(x, y, z - j));
  const double g = a.gx ? __dmul_rn(__dmul_rn(a.gx[x], a.gy[y]), a.gz[z]) : 1.0;
  const bool src = x == a.sx && y == a.sy && z == a.sz && a.it < a.n_series;
  a.out[p] = finish(a, c, a.prev[p], lap, a.m_mode == FDR_M_GRID ? a.m[p] : 1.0, g, src);
}

#ifndef FDR64_TY
#define FDR64_TY 8
#endif
constexpr int TZ = 32, TY = FDR64_TY, NT = TZ * TY;

template <int R>
struct Geo {
  static constexpr int BZ = TZ + 2 * R, BY = TY + 2 * R, BOX = BZ * BY;
  static constexpr int NL = (BOX + NT - 1) / NT;  // box elements per thread
  static constexpr int MINB = R <= 4 ? 2 * (512 / NT) : 512 / NT;
};

template <int R, bool SPONGE>
__global__ void __launch_bounds__(NT, Geo<R>::MINB) a64_stream(const A64Step a) {
  using G = Geo<R>;
  __shared__ double box[2][G::BOX];
  gather(a);
  const int tz = threadIdx.x, ty = threadIdx.y, tid = ty * TZ + tz;
  const int zt = blockIdx.x * TZ, yt = blockIdx.y * TY;
  const int z = zt + tz, y = yt + ty;
  const int xb = blockIdx.z * a.chunk;
  const int nx = a.nx;
  const int xe = min(nx, xb + a.chunk);
  if (xb >= xe) return;
  const bool inb = z < a.nz && y < a.ny;
  const long long px = a.pitch_x;
  const int own = inb ? y * a.pitch_y + z : 0;
  // loop-invariant box element offsets within a plane (-1: outside, reads 0)
  int boff[G::NL];
#pragma unroll
  for (int l = 0; l < G::NL; ++l) {
    const int e = tid + l * NT;
    const int by = e / G::BZ, bz = e - by * G::BZ;
    const int gy = yt - R + by, gz = zt - R + bz;
    boff[l] = (e < G::BOX && gy >= 0 && gy < a.ny && gz >= 0 && gz < a.nz) ? gy * a.pitch_y + gz : -1;
  }
  const double gyv = (SPONGE && inb) ? a.gy[y] : 1.0, gzv = (SPONGE && inb) ? a.gz[z] : 1.0;
  const bool src_col = inb && y == a.sy && z == a.sz && a.it < a.n_series;
  const int sx = src_col ? a.sx : -1;
  const bool grid_m = a.m_mode == FDR_M_GRID;

  // column pointers at plane xb; they advance one plane per iteration
  const double* cur0 = a.cur + own;
  double q[2 * R + 1];
#pragma unroll
  for (int i = 0; i < 2 * R; ++i) {
    const int x = xb - R + i;
    q[i] = (inb && x >= 0 && x < nx) ? cur0[x * px] : 0.0;
  }
  const double* lead_p = cur0 + (xb + R) * px;       // queue head: plane x + R
  const double* plane_p = a.cur + xb * px;           // box source: plane x
  const double* prev_p = a.prev + own + xb * px;
  const double* m_p = (grid_m ? a.m : a.cur) + own + xb * px;
  double* out_p = a.out + own + xb * px;
  double bv[G::NL];
#pragma unroll
  for (int l = 0; l < G::NL; ++l) bv[l] = boff[l] >= 0 ? plane_p[boff[l]] : 0.0;
#pragma unroll
  for (int l = 0; l < G::NL; ++l)
    if (tid + l * NT < G::BOX) box[0][tid + l * NT] = bv[l];
  double lead = (inb && xb + R < nx) ? *lead_p : 0.0;
  __syncthreads();
  const int cbox = (ty + R) * G::BZ + tz + R;
#pragma unroll 1
  for (int x = xb, i = 0; x < xe; ++x, ++i) {
    q[2 * R] = lead;
    const bool more = x + 1 < xe;
    plane_p += px;
    lead_p += px;
    if (more) {
#pragma unroll
      for (int l = 0; l < G::NL; ++l) bv[l] = boff[l] >= 0 ? plane_p[boff[l]] : 0.0;
      lead = (inb && x + 1 + R < nx) ? *lead_p : 0.0;
    }
    const double pv = inb ? *prev_p : 0.0;
    const double mv = (grid_m && inb) ? *m_p : 1.0;
    const double* b = box[i & 1];
    const double c = q[R];
    double lap = __dmul_rn(a.w[0], c);
#pragma unroll
    for (int j = 1; j <= R; ++j) lap = tapd(lap, a.w[j], q[R + j], q[R - j]);
#pragma unroll
    for (int j = 1; j <= R; ++j) lap = tapd(lap, a.w[j], b[cbox + j * G::BZ], b[cbox - j * G::BZ]);
#pragma unroll
    for (int j = 1; j <= R; ++j) lap = tapd(lap, a.w[j], b[cbox + j], b[cbox - j]);
    if (inb) {
      const double g = SPONGE ? __dmul_rn(__dmul_rn(__ldg(a.gx + x), gyv), gzv) : 1.0;
      *out_p = finish(a, c, pv, lap, mv, g, x == sx);
    }
    prev_p += px;
    m_p += px;
    out_p += px;
#pragma unroll
    for (int k = 0; k < 2 * R; ++k) q[k] = q[k + 1];
    if (more) {
#pragma unroll
      for (int l = 0; l < G::NL; ++l)
        if (tid + l * NT < G::BOX) box[(i + 1) & 1][tid + l * NT] = bv[l];
    }
    __syncthreads();
  }
}

// ------------------------------------------------------- TMA queue kernel
// The float64 counterpart of acoustic_queue (acoustic.cu): 256 threads own a
// 32(z) x 16(y) tile, one double2 (2 z points) each, and stream it along x.
// Stage p (filled by TMA NS-1 planes ahead, float64 tensor maps, out-of-bound
// zero fill = the reference halo) holds the newest plane's tile (register
// queue along x: 2r+U double2), the centre plane's box with y/z halo, and its
// prev / m tiles.  Barrier-free recycling: the warp completing a stage's
// "empty" phase refills it.  Arithmetic in IEEE double, one rounding per op.
constexpr int QTZ = 32, QTY = 16, QNTZ = QTZ / 2, QNT = QNTZ * QTY;

template <int R>
struct QG64 {
  static constexpr int LZ = (R + 1) / 2 * 2;  // z halo in doubles, 16-byte aligned
  static constexpr int BZ = QTZ + 2 * LZ;
  static constexpr int BY = QTY + 2 * R;
  static constexpr int BOX_BYTES = BZ * BY * 8;
  static constexpr int BOX = (BOX_BYTES + 127) / 128 * 16;  // doubles, 128-B aligned
  static constexpr int TILE = QTZ * QTY;
  static constexpr int TILE_BYTES = TILE * 8;
  static constexpr int OFF_BOX = TILE, OFF_PREV = TILE + BOX, OFF_M = OFF_PREV + TILE;
  static constexpr int STAGE = OFF_M + TILE;
  static constexpr int NS = 4;
  static constexpr int QD = 2 * R + 1;
#ifdef FDR_A64_U
  static constexpr int U = FDR_A64_U;
#else
  // re-measured after the carried addresses (512^3 random levels, GPts/s):
  // order 4 U = 1 205.2 vs whole-queue 201.0; orders 8 / 12 / 16 U = 3
  // 169.0 / 141.8 / 124.8 vs U = 2 167.8 / 140.3 / 123.7 and U = 1 166.7 / 140.6 / 122.2
  static constexpr int U = R <= 1 ? QD : (R == 2 ? 1 : 3);
#endif
  static constexpr int NQ = 1 + LZ;  // double2 loads of the own z-row window
  static constexpr int NWARPS = QNT / 32;
  static constexpr size_t SMEM = size_t(NS) * STAGE * 8 + 2 * NS * 8;
};

A64_DEV double2 lds2(const double* p) { return *reinterpret_cast<const double2*>(p); }
// from a 32-bit shared-window address (volatile: stays after the stage wait)
A64_DEV double2 lds2a(uint32_t a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}

A64_DEV void stg2_stream(double* p, double2 v) {
  asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}

A64_DEV bool arrive_is_last_a(uint32_t bar) {
  uint64_t state;
  uint32_t pending;
  asm volatile("mbarrier.arrive.shared::cta.b64 %0, [%1];" : "=l"(state) : "r"(bar) : "memory");
  asm volatile("mbarrier.pending_count.b64 %0, %1;" : "=r"(pending) : "l"(state));
  return pending == 1;
}
A64_DEV bool arrive_is_last(uint64_t* bar) { return arrive_is_last_a(fdr::smem_u32(bar)); }

// Correctly rounded s / m in double without __ddiv_rn's slow path for tiny
// dividends.  In float64 the numerical precursor ahead of a wavefront decays
// through ~1e-300 instead of underflowing to zero, and __ddiv_rn's operand
// check sends every such dividend to its slow-path subroutine (ncu: one CALL
// per division early in a run).  The float32 path's scaled scheme, in double:
// s' = s 2^600 (exact, subnormals included); r = 1/m from MUFU.RCP64H and two
// Newton steps; q = s' r plus one exact-remainder correction (correctly
// rounded while q is normal and nothing overflows); y = q 2^-600.  The
// downscale is exact unless y is subnormal; then d = q - y 2^600 (exact) is
// the rounding error, |d| <= 2^-475 (half a subnormal ulp, scaled).  y is the
// correctly rounded quotient unless q 2^-600 sat exactly on a midpoint of the
// subnormal grid (|d| = 2^-475): there the double rounding may have gone the
// wrong way, and the sign of the exact remainder e = s' - m q (Q - q has the
// sign of e) decides: when e and d have the same sign the true quotient lies
// past the midpoint, and y moves one subnormal ulp toward q.  Anything else
// (overflow, inf/NaN: d is NaN; m outside [2^-500, 2^500], or below 2^-400
// at a midpoint) takes __ddiv_rn.
// Before the subnormal handling every subnormal quotient took __ddiv_rn,
// whose slow path the float64 precursor ahead of a wavefront hits in bulk.
// fdr_selftest_division64 checks the bits against __ddiv_rn (midpoints
// included, seed bit 31).
A64_DEV double rcp_approx64(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return r;
}
A64_DEV double ddiv_scaled(double s, double m, bool* fast, bool* mid = nullptr) {
  const double sp = __dmul_rn(s, 0x1p600);
  double r = rcp_approx64(m);
  r = __fma_rn(r, __fma_rn(-m, r, 1.0), r);
  r = __fma_rn(r, __fma_rn(-m, r, 1.0), r);
  const double q0 = __dmul_rn(sp, r);
  const double q = __fma_rn(r, __fma_rn(-m, q0, sp), q0);
  // m > 0 on the fast path, so the quotient carries the sign of s; this only
  // changes s = -0 (the remainder step returns +0 there, IEEE gives -0)
  double y = copysign(__dmul_rn(q, 0x1p-600), s);
  const double d = __fma_rn(y, -0x1p600, q);
  const double ad = fabs(d);
  // NaN d fails; the midpoint correction needs an exact remainder (m >= 2^-400)
  *fast = ad <= 0x1p-475 && m >= (ad == 0x1p-475 ? 0x1p-400 : 0x1p-500) && m <= 0x1p500;
  if (ad == 0x1p-475) {  // exact midpoint of the subnormal grid (rare)
    const double e = __fma_rn(-m, q, sp);  // exact: q correctly rounded, m >= 2^-400
    if (e != 0.0 && ((e > 0.0) == (d > 0.0))) y = __dadd_rn(y, __dmul_rn(d, 0x1p-599));
    if (mid) *mid = true;
  }
  return y;
}
// Out of line on purpose: inline, the compiler if-converts the select and
// evaluates __ddiv_rn (and its slow-path call on zero dividends) for every
// lane (ncu: one CALL per division early in a run).
__device__ __noinline__ double ddiv_fallback(double s, double m) { return __ddiv_rn(s, m); }
A64_DEV double ddiv_exact(double s, double m) {
  bool fast;
  const double y = ddiv_scaled(s, m, &fast);
  return fast ? y : ddiv_fallback(s, m);
}

template <bool GRID_M>
A64_DEV double divide64(const A64Step& a, double s, double m) {
  if (GRID_M) return ddiv_exact(s, m);
  if (a.m_mode == FDR_M_SCALAR) return ddiv_exact(s, a.m_scalar);
  return s;
}

template <int R, bool GRID_M, bool SPONGE>
__global__ void __launch_bounds__(QNT, 2)
    a64_queue(const __grid_constant__ CUtensorMap tm_box, const __grid_constant__ CUtensorMap tm_tile,
              const __grid_constant__ CUtensorMap tm_prev, const __grid_constant__ CUtensorMap tm_m,
              const A64Step a) {
  using G = QG64<R>;
  using namespace fdr;
  extern __shared__ __align__(128) double dsm[];
  double* ring = dsm;
  uint64_t* full = reinterpret_cast<uint64_t*>(dsm + G::NS * G::STAGE);
  uint64_t* empty = full + G::NS;

  gather(a);
  const int tid = threadIdx.x;
  const int tz = tid % QNTZ, ty = tid / QNTZ;
  const int zt = blockIdx.x * QTZ, yt = blockIdx.y * QTY;
  const int xb = blockIdx.z * a.chunk;
  const int xe = min(a.nx, xb + a.chunk);
  if (xb >= xe) return;
  const int n = xe - xb;
  const int nplanes = n + 2 * R;  // stream plane p: newest x = xb - R + p

  auto issue = [&](int p, int sl) {
    double* st = ring + sl * G::STAGE;
    const bool compute = p >= 2 * R;
    const uint32_t bytes = G::TILE_BYTES + (compute ? G::BOX_BYTES + (GRID_M ? 2 : 1) * G::TILE_BYTES : 0);
    mbar_arrive_expect_tx(&full[sl], bytes);
    tma_load_3d(st, &tm_tile, &full[sl], zt, yt, xb - R + p);
    if (compute) {
      const int xc = xb - 2 * R + p;
      tma_load_3d(st + G::OFF_BOX, &tm_box, &full[sl], zt - G::LZ, yt - R, xc);
      tma_load_3d(st + G::OFF_PREV, &tm_prev, &full[sl], zt, yt, xc);
      if (GRID_M) tma_load_3d(st + G::OFF_M, &tm_m, &full[sl], zt, yt, xc);
    }
  };
  if (tid == 0) {
    prefetch_tensormap(&tm_box);
    prefetch_tensormap(&tm_tile);
    prefetch_tensormap(&tm_prev);
    if (GRID_M) prefetch_tensormap(&tm_m);
    for (int sl = 0; sl < G::NS; ++sl) {
      mbar_init(&full[sl], 1);
      mbar_init(&empty[sl], G::NWARPS);
    }
    fence_barrier_init();
    for (int p = 0; p < G::NS && p < nplanes; ++p) issue(p, p);
  }
  __syncthreads();

  const int y = yt + ty;
  const int zb = zt + 2 * tz;
  const bool row_ok = y < a.ny;
  const bool vec_ok = row_ok && zb + 1 < a.nz;
  const int bcen = G::OFF_BOX + (ty + R) * G::BZ + G::LZ + 2 * tz;
  const int tcol = ty * QTZ + 2 * tz;
  double gyz0 = 1.0, gyz1 = 1.0, gyv = 1.0;
  if (SPONGE && row_ok) {
    gyv = a.gy[y];
    gyz0 = zb < a.nz ? a.gz[zb] : 1.0;
    gyz1 = zb + 1 < a.nz ? a.gz[zb + 1] : 1.0;
  }
  int src_k = 0, kinj = -1;
  double qsrc = 0.0;
  if (a.sx >= 0 && y == a.sy && a.sz >= zb && a.sz < zb + 2 && a.it < a.n_series) {
    src_k = a.sz - zb;
    kinj = a.sx - xb;
    qsrc = a.series[a.it];
  }
  double* outp = a.out + (size_t)xb * a.pitch_x + (size_t)y * a.pitch_y + zb;
  // r <= 6: at r = 8 the extra copies measured 3% slower (instruction cache)
  const bool cta_plain = (FDR_Q64PLAIN && R <= 6) ? (__syncthreads_and(vec_ok && kinj < 0) != 0) : false;
  bool cta_nosp = false;
  if (FDR_Q64PLAIN && SPONGE && cta_plain) {  // every taper factor of this CTA's tile and chunk is 1?
    bool one = gyv == 1.0 && gyz0 == 1.0 && gyz1 == 1.0;
    for (int i = threadIdx.x; i < xe - xb; i += blockDim.x) one &= __ldg(a.gx + xb + i) == 1.0;
    cta_nosp = __syncthreads_and(one) != 0;
  }

  int slot = 0;
  uint32_t phase = 0;
  // own-column / own-box-row / full-barrier shared addresses of stage `slot`,
  // carried across planes (no thread-index rematerialisation per plane, as in
  // the float32 kernel)
  constexpr uint32_t SB = G::STAGE * 8u;
  uint32_t ac = fdr::smem_u32(ring + tcol), ab = fdr::smem_u32(ring + bcen);
  uint32_t af = fdr::smem_u32(full);  // empty[slot] is 8 NS bytes further
  auto finish = [&](int p) {
    __syncwarp();
    if (fdr::elect_one() && arrive_is_last_a(af + 8u * G::NS)) {
      fdr::mbar_wait_a(af + 8u * G::NS, phase);
      fence_proxy_async();  // generic-proxy reads of the stage before the TMA refill (cross-proxy WAR)
      if (p + G::NS < nplanes) issue(p + G::NS, slot);
    }
    ac += SB;
    ab += SB;
    af += 8u;
    if (++slot == G::NS) {
      slot = 0;
      phase ^= 1u;
      ac -= G::NS * SB;
      ab -= G::NS * SB;
      af -= 8u * G::NS;
    }
  };

  constexpr bool ROTATE = G::U % G::QD == 0;
  double2 qw[2 * R + G::U];
#pragma unroll
  for (int p = 0; p < 2 * R; ++p) {
    fdr::mbar_wait_a(af, phase);
    qw[p] = lds2a(ac);
    finish(p);
  }

  // As in acoustic_queue (FDR_QPLAIN / FDR_QNOSP): copies of the plane loop
  // without the source test and with unconditional vector stores for CTAs
  // that need neither, and without the taper code outside the sponge.
  auto main_loop = [&](auto plain_tag, auto nosp_tag) {
  constexpr bool PLAIN = decltype(plain_tag)::value;
  constexpr bool NOSP = decltype(nosp_tag)::value;
#pragma unroll 1
  for (int p0 = 2 * R; p0 < nplanes; p0 += G::U) {
#pragma unroll
    for (int u = 0; u < G::U; ++u) {
      const int p = p0 + u;
      if (p >= nplanes) break;
      const int k = p - 2 * R;
      fdr::mbar_wait_a(af, phase);
      qw[ROTATE ? (2 * R + u) % G::QD : 2 * R + u] = lds2a(ac);
      double zr[2 + 2 * G::LZ];
#pragma unroll
      for (int qd = 0; qd < G::NQ; ++qd) {
        const double2 v = lds2a(ab + 8u * (2 * qd - G::LZ));
        zr[2 * qd] = v.x;
        zr[2 * qd + 1] = v.y;
      }
      const double c0 = zr[G::LZ], c1 = zr[G::LZ + 1];
      double l0 = __dmul_rn(a.w[0], c0), l1 = __dmul_rn(a.w[0], c1);
#pragma unroll
      for (int j = 1; j <= R; ++j) {  // x taps from the register queue
        const double2 pp = qw[ROTATE ? (R + u + j) % G::QD : R + u + j];
        const double2 mm = qw[ROTATE ? (R + u - j + G::QD) % G::QD : R + u - j];
        l0 = tapd(l0, a.w[j], pp.x, mm.x);
        l1 = tapd(l1, a.w[j], pp.y, mm.y);
      }
#pragma unroll
      for (int j = 1; j <= R; ++j) {  // y taps from the centre box
        const double2 pp = lds2a(ab + 8u * (j * G::BZ));
        const double2 mm = lds2a(ab - 8u * (j * G::BZ));
        l0 = tapd(l0, a.w[j], pp.x, mm.x);
        l1 = tapd(l1, a.w[j], pp.y, mm.y);
      }
#pragma unroll
      for (int j = 1; j <= R; ++j) {  // z taps from the own row window
        l0 = tapd(l0, a.w[j], zr[G::LZ + j], zr[G::LZ - j]);
        l1 = tapd(l1, a.w[j], zr[G::LZ + 1 + j], zr[G::LZ + 1 - j]);
      }
      const double2 pv = lds2a(ac + 8u * G::OFF_PREV);
      double2 mv = make_double2(1.0, 1.0);
      if (GRID_M) mv = lds2a(ac + 8u * G::OFF_M);
      finish(p);
      double o0 = __dadd_rn(__dsub_rn(__dadd_rn(c0, c0), pv.x),
                            divide64<GRID_M>(a, __dmul_rn(a.coef, l0), mv.x));
      double o1 = __dadd_rn(__dsub_rn(__dadd_rn(c1, c1), pv.y),
                            divide64<GRID_M>(a, __dmul_rn(a.coef, l1), mv.y));
      if (SPONGE && !NOSP) {
        const double gxy = __dmul_rn(__ldg(a.gx + xb + k), gyv);
        o0 = __dmul_rn(o0, __dmul_rn(gxy, gyz0));
        o1 = __dmul_rn(o1, __dmul_rn(gxy, gyz1));
      }
      if (!PLAIN && k == kinj) {
        if (src_k == 0) o0 = __dadd_rn(o0, qsrc);
        else o1 = __dadd_rn(o1, qsrc);
      }
      double* dst = outp + (size_t)k * a.pitch_x;
      if (PLAIN || vec_ok) {
        stg2_stream(dst, make_double2(o0, o1));
      } else if (row_ok && zb < a.nz) {
        dst[0] = o0;
      }
    }
    if (!ROTATE) {
#pragma unroll
      for (int i = 0; i < 2 * R; ++i) qw[i] = qw[i + G::U];
    }
  }
  };
  if (FDR_Q64PLAIN && R <= 6 && cta_plain) {
    if (SPONGE && cta_nosp) main_loop(std::true_type{}, std::true_type{});
    else main_loop(std::true_type{}, std::false_type{});
  } else {
    main_loop(std::false_type{}, std::false_type{});
  }
}

typedef CUresult (*A64EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                CUtensorMapFloatOOBfill);

static int encode64(CUtensorMap* map, const double* base, const A64Step& s, int box_z, int box_y) {
  static A64EncodeFn enc = nullptr;
  if (!enc) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return fail(FDR_ECUDA, "cuTensorMapEncodeTiled unavailable");
    enc = reinterpret_cast<A64EncodeFn>(fn);
  }
  cuuint64_t dims[3] = {(cuuint64_t)s.nz, (cuuint64_t)s.ny, (cuuint64_t)s.nx};
  cuuint64_t strides[2] = {(cuuint64_t)s.pitch_y * 8, (cuuint64_t)s.pitch_x * 8};
  cuuint32_t box[3] = {(cuuint32_t)box_z, (cuuint32_t)box_y, 1}, es[3] = {1, 1, 1};
  const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims,
                         strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? FDR_OK : fail(FDR_ECUDA, "cuTensorMapEncodeTiled (float64) failed (%d)", (int)r);
}

struct Maps64 {
  CUtensorMap box[3], tile[3], m;
};

template <int R, bool GRID_M, bool SPONGE>
static int queue_inst(const A64Step& s, const Maps64& mp, int k, cudaStream_t st, int* chunk_cache) {
  using G = QG64<R>;
  auto kern = a64_queue<R, GRID_M, SPONGE>;
  // occupancy facts per (kernel, device), cached under a lock (concurrent
  // callers on several devices share launch_facts' table)
  int occ = 0, nsm = 0;
  const int frc = fdr::launch_facts(reinterpret_cast<const void*>(kern), QNT, G::SMEM, &occ, &nsm);
  if (frc != FDR_OK) return frc;
  const int tzn = (s.nz + QTZ - 1) / QTZ, tyn = (s.ny + QTY - 1) / QTY;
  if (*chunk_cache <= 0) {
    const long tiles = (long)tzn * tyn, slots = (long)occ * nsm;
    double best = 1e30;
    int best_c = 1;
    for (int c = 1; c <= std::max(1, s.nx / (2 * R)); ++c) {
      const int len = (s.nx + c - 1) / c;
      const int cc = (s.nx + len - 1) / len;
      const long waves = (tiles * cc + slots - 1) / slots;
      const double t = (double)waves * (len + 0.3 * 2 * R);
      if (t < best * 0.999) {
        best = t;
        best_c = cc;
      }
    }
    *chunk_cache = (s.nx + best_c - 1) / best_c;
  }
  A64Step t = s;
  t.chunk = *chunk_cache;
  const int cur = (2 + k) % 3, prev = (1 + k) % 3;
  dim3 grid(tzn, tyn, (s.nx + t.chunk - 1) / t.chunk);
  kern<<<grid, QNT, G::SMEM, st>>>(mp.box[cur], mp.tile[cur], mp.tile[prev], mp.m, t);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? FDR_OK : cuda_fail(e, "a64_queue launch");
}

template <int R>
static int queue_r(const A64Step& s, const Maps64& mp, int k, cudaStream_t st, int* cc) {
  const bool gm = s.m_mode == FDR_M_GRID, sp = s.gx != nullptr;
  if (gm && sp) return queue_inst<R, true, true>(s, mp, k, st, cc);
  if (gm) return queue_inst<R, true, false>(s, mp, k, st, cc);
  if (sp) return queue_inst<R, false, true>(s, mp, k, st, cc);
  return queue_inst<R, false, false>(s, mp, k, st, cc);
}

static int queue_step(const A64Step& s, const Maps64& mp, int k, cudaStream_t st, int* cc) {
  switch (s.radius) {
    case 1: return queue_r<1>(s, mp, k, st, cc);
    case 2: return queue_r<2>(s, mp, k, st, cc);
    case 3: return queue_r<3>(s, mp, k, st, cc);
    case 4: return queue_r<4>(s, mp, k, st, cc);
    case 5: return queue_r<5>(s, mp, k, st, cc);
    case 6: return queue_r<6>(s, mp, k, st, cc);
    case 7: return queue_r<7>(s, mp, k, st, cc);
    case 8: return queue_r<8>(s, mp, k, st, cc);
    default: return fail(FDR_EINVAL, "float64 queue kernel supports radius <= 8, got %d", s.radius);
  }
}

template <int R>
static int stream_launch(const A64Step& s, cudaStream_t st, int* chunk_cache) {
  using G = Geo<R>;
  const bool sponge = s.gx != nullptr;
  auto kern = sponge ? a64_stream<R, true> : a64_stream<R, false>;
  int occ_s = 0, nsm = 0;
  const int frc = fdr::launch_facts(reinterpret_cast<const void*>(kern), NT, 0, &occ_s, &nsm);
  if (frc != FDR_OK) return frc;
  int occ[2] = {occ_s, occ_s};
  cudaError_t e = cudaSuccess;
  const int tzn = (s.nz + TZ - 1) / TZ, tyn = (s.ny + TY - 1) / TY;
  if (*chunk_cache <= 0) {  // fewest waves x (planes + the 2r-plane queue fill)
    const long tiles = (long)tzn * tyn, slots = (long)occ[sponge] * nsm;
    double best = 1e30;
    int best_c = 1;
    for (int c = 1; c <= std::max(1, s.nx / (2 * R)); ++c) {
      const int len = (s.nx + c - 1) / c;
      const int cc = (s.nx + len - 1) / len;
      const long waves = (tiles * cc + slots - 1) / slots;
      const double t = (double)waves * (len + 0.5 * 2 * R);
      if (t < best * 0.999) {
        best = t;
        best_c = cc;
      }
    }
    *chunk_cache = (s.nx + best_c - 1) / best_c;
  }
  A64Step t = s;
  t.chunk = *chunk_cache;
  dim3 grid(tzn, tyn, (s.nx + t.chunk - 1) / t.chunk);
  kern<<<grid, dim3(TZ, TY), 0, st>>>(t);
  e = cudaGetLastError();
  return e == cudaSuccess ? FDR_OK : cuda_fail(e, "a64_stream launch");
}

static int stream_step(const A64Step& s, cudaStream_t st, int* chunk_cache) {
  switch (s.radius) {
    case 1: return stream_launch<1>(s, st, chunk_cache);
    case 2: return stream_launch<2>(s, st, chunk_cache);
    case 3: return stream_launch<3>(s, st, chunk_cache);
    case 4: return stream_launch<4>(s, st, chunk_cache);
    case 5: return stream_launch<5>(s, st, chunk_cache);
    case 6: return stream_launch<6>(s, st, chunk_cache);
    case 7: return stream_launch<7>(s, st, chunk_cache);
    case 8: return stream_launch<8>(s, st, chunk_cache);
    default: return fail(FDR_EINVAL, "fp64 stream kernel supports radius <= 8, got %d", s.radius);
  }
}

static int validate(const fdr_acoustic64_args* a) {
  if (!a) return fail(FDR_EINVAL, "args is NULL");
  if (a->abi_version != FDR_ABI_VERSION)
    return fail(FDR_EINVAL, "abi_version %d != library %d", a->abi_version, FDR_ABI_VERSION);
  if (a->order < 2 || a->order % 2 || a->order > 2 * FDR_MAX_RADIUS)
    return fail(FDR_EINVAL, "order must be even and within [2, %d], got %d", 2 * FDR_MAX_RADIUS,
                a->order);
  const int r = a->order / 2;
  if (a->nx < 2 * r + 1 || a->ny < 2 * r + 1 || a->nz < 2 * r + 1)
    return fail(FDR_EINVAL, "interior dims (%d, %d, %d) too small for halo width %d", a->nx, a->ny,
                a->nz, r);
  if (a->pitch_y < a->nz || a->pitch_y % 2 || a->pitch_x < (int64_t)a->ny * a->pitch_y)
    return fail(FDR_EINVAL, "bad pitches (pitch_y %d, pitch_x %lld)", a->pitch_y,
                (long long)a->pitch_x);
  if (a->n_steps < 0 || a->it0 < 0) return fail(FDR_EINVAL, "n_steps and it0 must be >= 0");
  for (int i = 0; i < 3; ++i)
    if (!a->levels[i]) return fail(FDR_EINVAL, "level pointer %d is NULL", i);
  if (a->m_mode < FDR_M_NONE || a->m_mode > FDR_M_GRID)
    return fail(FDR_EINVAL, "unknown m_mode %d", a->m_mode);
  if (a->m_mode == FDR_M_GRID && !a->m) return fail(FDR_EINVAL, "m_mode GRID needs an m grid");
  if (a->sponge_x && (!a->sponge_y || !a->sponge_z))
    return fail(FDR_EINVAL, "sponge needs all three profiles");
  if (a->src_x >= 0 && (a->src_x >= a->nx || a->src_y < 0 || a->src_y >= a->ny || a->src_z < 0 ||
                        a->src_z >= a->nz))
    return fail(FDR_EINVAL, "source location outside interior");
  if (a->src_x >= 0 && a->n_series > 0 && !a->series)
    return fail(FDR_EINVAL, "source series pointer NULL");
  if (a->n_rec < 0 || (a->n_rec > 0 && (!a->rec_xyz || !a->traces)))
    return fail(FDR_EINVAL, "receiver coordinates or trace buffer NULL");
  if (a->variant < FDR_VARIANT_AUTO || a->variant > FDR_VARIANT_QUEUE)
    return fail(FDR_EINVAL, "fp64 variant must be AUTO, DIRECT, TMA or QUEUE, got %d", a->variant);
  if ((a->variant == FDR_VARIANT_QUEUE || a->variant == FDR_VARIANT_TMA) && r > 8)
    return fail(FDR_EINVAL, "fp64 streaming kernels support order <= 16, got %d", a->order);
  if (a->variant != FDR_VARIANT_DIRECT &&
      ((uintptr_t)a->levels[0] % 16 || (uintptr_t)a->levels[1] % 16 || (uintptr_t)a->levels[2] % 16 ||
       (a->m_mode == FDR_M_GRID && (uintptr_t)a->m % 16)))
    return fail(FDR_EINVAL, "fp64 streaming kernels need 16-byte aligned levels and m");
  return FDR_OK;
}

static void fill(A64Step& s, const fdr_acoustic64_args* a, int k) {
  memset(&s, 0, sizeof(s));
  s.out = a->levels[(0 + k) % 3];
  s.prev = a->levels[(1 + k) % 3];
  s.cur = a->levels[(2 + k) % 3];
  s.m = a->m;
  s.nx = a->nx;
  s.ny = a->ny;
  s.nz = a->nz;
  s.pitch_y = a->pitch_y;
  s.pitch_x = a->pitch_x;
  for (int j = 0; j <= FDR_MAX_RADIUS; ++j) s.w[j] = a->weights[j];
  s.coef = a->coef;
  s.m_scalar = a->m_scalar;
  s.m_mode = a->m_mode;
  s.radius = a->order / 2;
  s.gx = a->sponge_x;
  s.gy = a->sponge_y;
  s.gz = a->sponge_z;
  s.series = a->series;
  s.n_series = (a->src_x >= 0 && a->series) ? a->n_series : 0;
  s.it = a->it0 + k;
  s.sx = a->src_x;
  s.sy = a->src_y;
  s.sz = a->src_z;
  s.rec = a->rec_xyz;
  s.n_rec = a->n_rec;
  s.traces = a->traces;
  const int row = s.it - 1;
  s.gather_row = (k > 0 && a->n_rec > 0 && a->traces && row < a->trace_rows) ? row : -1;
}

static int run(const fdr_acoustic64_args* a, cudaStream_t st) {
  const int r = a->order / 2;
  const bool queue = a->variant == FDR_VARIANT_QUEUE || (a->variant == FDR_VARIANT_AUTO && r <= 8);
  const bool stream = a->variant == FDR_VARIANT_TMA;  // plain-load streaming kernel
  Maps64 mp;
  if (queue && a->n_steps > 0) {
    A64Step s0;
    fill(s0, a, 0);
    const int lz = (r + 1) / 2 * 2;
    for (int i = 0; i < 3; ++i) {
      int rc = encode64(&mp.box[i], a->levels[i], s0, QTZ + 2 * lz, QTY + 2 * r);
      if (rc == FDR_OK) rc = encode64(&mp.tile[i], a->levels[i], s0, QTZ, QTY);
      if (rc != FDR_OK) return rc;
    }
    const int rc = encode64(&mp.m, a->m_mode == FDR_M_GRID ? a->m : a->levels[0], s0, QTZ, QTY);
    if (rc != FDR_OK) return rc;
  }
  int chunk = 0;
  for (int k = 0; k < a->n_steps; ++k) {
    A64Step s;
    fill(s, a, k);
    if (queue) {
      const int rc = queue_step(s, mp, k, st, &chunk);
      if (rc != FDR_OK) return rc;
    } else if (stream) {
      const int rc = stream_step(s, st, &chunk);
      if (rc != FDR_OK) return rc;
    } else {
      dim3 block(64, 4, 1), grid((a->nz + 63) / 64, (a->ny + 3) / 4, a->nx);
      a64_direct<<<grid, block, 0, st>>>(s);
      const cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return cuda_fail(e, "a64_direct launch");
    }
  }
  const int last = a->it0 + a->n_steps - 1;
  if (a->n_steps > 0 && a->n_rec > 0 && a->traces && last < a->trace_rows) {
    a64_gather_kernel<<<(a->n_rec + 255) / 256, 256, 0, st>>>(
        a->levels[(2 + a->n_steps) % 3], a->rec_xyz, a->n_rec, a->traces, last, a->pitch_y,
        a->pitch_x);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "a64 gather launch");
  }
  return (2 + a->n_steps) % 3;
}

__device__ __forceinline__ uint32_t hmix(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

// ddiv_exact vs __ddiv_rn on n hashed pairs: |s| log-uniform over
// [2^-1080, 2^520] (random mantissas, both signs, zeros, subnormals, edge
// values), m log-uniform over [m_lo, m_hi]; counts mismatching bits and the
// pairs that took the fast path.  With seed bit 31 set every pair is a
// constructed subnormal-midpoint candidate and the second count is the pairs
// the fast path resolved through its midpoint correction.
__global__ void div64_selftest_kernel(long long n, double m_lo, double m_hi, unsigned seed,
                                      unsigned long long* bad, unsigned long long* fast) {
  unsigned long long nb = 0, nf = 0;
  const double lmlo = log2(m_lo), lmhi = log2(m_hi);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const uint32_t h1 = hmix((uint32_t)i * 2654435761u ^ seed);
    const uint32_t h2 = hmix(h1 ^ 0x9e3779b9u);
    const uint32_t h3 = hmix(h2 + 0x85ebca6bu);
    const uint32_t h4 = hmix(h3 ^ 0x27d4eb2fu);
    double s = exp2(-1080.0 + 1600.0 * (h1 >> 8) * (1.0 / 16777216.0));
    const unsigned long long mant = ((unsigned long long)h3 << 20) ^ h4;
    s = __longlong_as_double((__double_as_longlong(s) & 0xfff0000000000000ull) | (mant & 0x000fffffffffffffull));
    if ((h3 >> 24) == 0) s = 0.0;
    if ((h3 >> 24) == 1) s = 0x1p-1074;
    if ((h3 >> 24) == 2) s = __longlong_as_double(0x000fffffffffffffull);  // largest subnormal
    if ((h3 >> 24) == 3) s = __longlong_as_double(0x0010000000000000ull);  // smallest normal
    if (h2 & 1u) s = -s;
    double m = exp2(lmlo + (lmhi - lmlo) * (h2 >> 8) * (1.0 / 16777216.0));
    m = __longlong_as_double((__double_as_longlong(m) & 0xfff0000000000000ull) |
                             (((unsigned long long)hmix(h4) << 21 ^ h1) & 0x000fffffffffffffull));
    m = fmin(fmax(m, m_lo), m_hi);
    if (seed & 0x80000000u) {
      // midpoint candidates: s = j 2^-1074 (exact subnormal) and m = RN(2j / k)
      // with k odd (up to 2^40), so s'/m is within a relative 2^-53 of the
      // subnormal-grid midpoint k 2^-1075 (scaled: k 2^-475) and q often
      // rounds onto it exactly; the sign of the remainder then varies
      const double k = (double)((((unsigned long long)h4 << 8) ^ h1) & 0xffffffffffull) * 2.0 + 1.0;
      const double j = fmin(fmax(floor(k * m * 0.5), 1.0), 4503599627370495.0);
      s = (h2 & 1u ? -j : j) * 0x1p-1074;
      m = fmin(fmax(__ddiv_rn(2.0 * j, k), m_lo), m_hi);
    }
    bool f, mid = false;
    const double y = ddiv_scaled(s, m, &f, &mid);
    nf += (seed & 0x80000000u) ? (f && mid) : f;
    const double q = f ? y : __ddiv_rn(s, m);
    if (__double_as_longlong(q) != __double_as_longlong(__ddiv_rn(s, m))) ++nb;
  }
  atomicAdd(bad, nb);
  atomicAdd(fast, nf);
}


// ------------------------------------------------- oracle_step (float64)
// The reference's independent verification step, kernel.py:225-254: the
// update as an explicit float64 convolution over the star stencil's points
// in stencil_geometry("star") order (stencils.py:161-179: the centre with
// weight 3 w0, then for j = 1..r and sign +/-: x, y, z), accumulated from
// acc = 0 with one rounding per product and per sum (numpy, no FMA);
// upd = (2 c - prev) + (coef acc) / m in float64; one rounding to float32
// into the scratch level; the on-grid source added to the new value in
// float32 (kernel.py:167-173).  One thread per interior point.
__global__ void __launch_bounds__(256) conv64_step(const float* cur, const float* prev, float* out,
                                                   const float* m, const double* m64,
                                                   double m_scalar, int nx, int ny,
                                                   int nz, int pitch_y, long long pitch_x, int r,
                                                   const double* __restrict__ w, double coef,
                                                   int sx, int sy, int sz, float q) {
  const int z = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  const int x = blockIdx.z;
  if (z >= nz) return;
  const size_t p = (size_t)x * pitch_x + (size_t)y * pitch_y + z;
  auto at = [&](int xx, int yy, int zz) -> double {
    const bool in = (unsigned)xx < (unsigned)nx && (unsigned)yy < (unsigned)ny && (unsigned)zz < (unsigned)nz;
    return in ? (double)cur[(size_t)xx * pitch_x + (size_t)yy * pitch_y + zz] : 0.0;
  };
  const double c = (double)cur[p];
  double acc = __dadd_rn(0.0, __dmul_rn(w[0], c));
  for (int j = 1; j <= r; ++j) {
    for (int sgn = 1; sgn >= -1; sgn -= 2) {
      const int o = sgn * j;
      acc = __dadd_rn(acc, __dmul_rn(w[j], at(x + o, y, z)));
      acc = __dadd_rn(acc, __dmul_rn(w[j], at(x, y + o, z)));
      acc = __dadd_rn(acc, __dmul_rn(w[j], at(x, y, z + o)));
    }
  }
  const double mm = m64 ? m64[p] : m ? (double)m[p] : m_scalar;
  const double upd = __dadd_rn(__dsub_rn(__dmul_rn(2.0, c), (double)prev[p]),
                               __ddiv_rn(__dmul_rn(coef, acc), mm));
  float v = __double2float_rn(upd);
  if (x == sx && y == sy && z == sz) v = __fadd_rn(v, q);
  out[p] = v;
}
}  // namespace fdr64

extern "C" {

int64_t fdr_selftest_division64(int64_t n, double m_lo, double m_hi, uint32_t seed,
                                int64_t* n_fast) {
  using fdr64::cuda_fail;
  using fdr64::fail;
  if (n <= 0 || !(m_lo > 0.0) || !(m_hi >= m_lo)) return fail(FDR_EINVAL, "bad self-test range");
  unsigned long long* d = nullptr;
  cudaError_t e = cudaMalloc(&d, 2 * sizeof(unsigned long long));
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc");
  e = cudaMemset(d, 0, 2 * sizeof(unsigned long long));
  if (e == cudaSuccess) {
    fdr64::div64_selftest_kernel<<<148 * 8, 256>>>(n, m_lo, m_hi, seed, d, d + 1);
    e = cudaGetLastError();
  }
  unsigned long long h[2] = {0, 0};
  if (e == cudaSuccess) e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return cuda_fail(e, "float64 division self-test");
  if (n_fast) *n_fast = (int64_t)h[1];
  return (int64_t)h[0];
}


int fdr_acoustic_oracle_step(const fdr_acoustic_args* a, const double* weights64, double coef64,
                             double m_scalar64, const double* m64, void* stream) {
  using fdr64::cuda_fail;
  using fdr64::fail;
  if (!a || a->abi_version != FDR_ABI_VERSION) return fail(FDR_EINVAL, "ABI version mismatch");
  if (a->order < 2 || a->order > 2 * FDR_MAX_RADIUS || a->order % 2)
    return fail(FDR_EINVAL, "order must be even in 2..%d", 2 * FDR_MAX_RADIUS);
  if (a->nx < 1 || a->ny < 1 || a->nz < 1 || a->pitch_y < a->nz ||
      a->pitch_x < (int64_t)a->ny * a->pitch_y || a->ny > 65535 || a->nx > 65535)
    return fail(FDR_EINVAL, "bad extents or pitches");
  if (!a->levels[0] || !a->levels[1] || !a->levels[2] || !weights64)
    return fail(FDR_EINVAL, "null level or weight pointer");
  if (a->m_mode == FDR_M_GRID && !a->m) return fail(FDR_EINVAL, "m_mode grid needs m");
  if (a->src_w || a->rec_w) return fail(FDR_EINVAL, "oracle_step takes an on-grid source only");
  const int r = a->order / 2;
  double* dw = nullptr;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMallocAsync(&dw, sizeof(double) * (r + 1), st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync");
  e = cudaMemcpyAsync(dw, weights64, sizeof(double) * (r + 1), cudaMemcpyHostToDevice, st);
  const bool inject = a->src_x >= 0 && a->series && a->it0 < a->n_series;
  float q = 0.0f;
  if (e == cudaSuccess && inject)
    e = cudaMemcpyAsync(&q, a->series + a->it0, sizeof(float), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);  // q is read on the host
  if (e == cudaSuccess) {
    dim3 grid((a->nz + 255) / 256, a->ny, a->nx);
    fdr64::conv64_step<<<grid, 256, 0, st>>>(
        a->levels[2], a->levels[1], a->levels[0], a->m_mode == FDR_M_GRID ? a->m : nullptr, m64,
        m_scalar64, a->nx, a->ny, a->nz, a->pitch_y, a->pitch_x,
        r, dw, coef64, inject ? a->src_x : -1, a->src_y, a->src_z, q);
    e = cudaGetLastError();
  }
  cudaFreeAsync(dw, st);
  if (e != cudaSuccess) return cuda_fail(e, "oracle_step");
  return FDR_OK;
}

size_t fdr_acoustic64_args_size(void) { return sizeof(fdr_acoustic64_args); }

int fdr_acoustic64_run(const fdr_acoustic64_args* args, void* stream) {
  const int rc = fdr64::validate(args);
  if (rc != FDR_OK) return rc;
  return fdr64::run(args, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
