// TTI pseudo-acoustic (coupled p/r) step kernels for B200 (sm_100a) + C ABI.
//
// BASELINE config 4.  The reference only catalogues this kernel's cost
// (/root/reference/pkg/src/fdroof/equations.py:144-155) and states the system
// (PAPER.md:804-829); the float32 operation sequence is defined by the parity
// oracle oracle/tti_ref.c and reproduced here bit for bit:
//   D2_a(u) = w2[0] u + sum_j fma(w2[j], u[+j] + u[-j])           (fma chain)
//   D1_a(u) = w1[1] (u[+1]-u[-1]) + sum_{j>=2} fma(w1[j], u[+j] - u[-j])
//   dxy = D1_x(D1_y u), dxz = D1_x(D1_z u), dyz = D1_y(D1_z u)   (inner first)
//   G = cxz dxz + (cxy dxy + (cxx dxx + (cyz dyz + (czz dzz + cyy dyy))))   (fma)
//   L = (dyy + dzz) + dxx;  H = L - G
//   p' = fma(k, fma(a, H(p), b G(r)), fma(2, p, -p_prev))
//   r' = fma(k, fma(b, H(p), G(r)),   fma(2, r, -r_prev))
//   then taper, source injection into p and r, receivers sample p.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/b200fd.h"
#include "fdr_common.cuh"

namespace fdr_tti {

using namespace fdr;

struct TTIStep {
  const float* p;
  const float* pp;
  float* pn;
  const float* r;
  const float* rp;
  float* rn;
  const float* prm[9];  // k a b cxx cyy czz cxy cyz cxz
  int nx, ny, nz, pitch_y;
  long long pitch_x;
  int radius;
  float w2[FDR_MAX_RADIUS + 1];
  float w1[FDR_MAX_RADIUS + 1];
  const float* gx;
  const float* gy;
  const float* gz;
  const float* series;
  int n_series, it;
  int sx, sy, sz;
  const int* rec;
  int n_rec;
  float* traces;
  int gather_row;
  int gather_pad_chunk;  // x-planes per CTA (stream kernel)
  int es;                // floats between consecutive points: 1 separate p/r, 2 interleaved
};

__device__ __forceinline__ float at(const float* u, const TTIStep& a, int x, int y, int z) {
  if (x < 0 || x >= a.nx || y < 0 || y >= a.ny || z < 0 || z >= a.nz) return 0.0f;
  return u[a.es * ((size_t)x * a.pitch_x + (size_t)y * a.pitch_y + z)];
}

// first derivative along axis `ax` (0 x, 1 y, 2 z) at (x, y, z)
__device__ float d1(const float* u, const TTIStep& a, int x, int y, int z, int ax) {
  const int dx = ax == 0, dy = ax == 1, dz = ax == 2;
  float d = __fmul_rn(a.w1[1], __fsub_rn(at(u, a, x + dx, y + dy, z + dz),
                                         at(u, a, x - dx, y - dy, z - dz)));
  for (int j = 2; j <= a.radius; ++j)
    d = __fmaf_rn(a.w1[j], __fsub_rn(at(u, a, x + j * dx, y + j * dy, z + j * dz),
                                     at(u, a, x - j * dx, y - j * dy, z - j * dz)), d);
  return d;
}

__device__ float d2(const float* u, const TTIStep& a, int x, int y, int z, int ax) {
  const int dx = ax == 0, dy = ax == 1, dz = ax == 2;
  float d = __fmul_rn(a.w2[0], at(u, a, x, y, z));
  for (int j = 1; j <= a.radius; ++j)
    d = __fmaf_rn(a.w2[j], __fadd_rn(at(u, a, x + j * dx, y + j * dy, z + j * dz),
                                     at(u, a, x - j * dx, y - j * dy, z - j * dz)), d);
  return d;
}

// outer D1 along `ao` of the inner D1 along `ai`
__device__ float d11(const float* u, const TTIStep& a, int x, int y, int z, int ao, int ai) {
  const int dx = ao == 0, dy = ao == 1, dz = ao == 2;
  float d = __fmul_rn(a.w1[1], __fsub_rn(d1(u, a, x + dx, y + dy, z + dz, ai),
                                         d1(u, a, x - dx, y - dy, z - dz, ai)));
  for (int j = 2; j <= a.radius; ++j)
    d = __fmaf_rn(a.w1[j], __fsub_rn(d1(u, a, x + j * dx, y + j * dy, z + j * dz, ai),
                                     d1(u, a, x - j * dx, y - j * dy, z - j * dz, ai)), d);
  return d;
}

__device__ void gl_op(const float* u, const TTIStep& a, int x, int y, int z, const float* c,
                      float* G, float* L) {
  const float dxx = d2(u, a, x, y, z, 0), dyy = d2(u, a, x, y, z, 1), dzz = d2(u, a, x, y, z, 2);
  const float dxy = d11(u, a, x, y, z, 0, 1), dxz = d11(u, a, x, y, z, 0, 2);
  const float dyz = d11(u, a, x, y, z, 1, 2);
  const float gin = __fmaf_rn(c[4], dyz, __fmaf_rn(c[2], dzz, __fmul_rn(c[1], dyy)));
  const float lin = __fadd_rn(dyy, dzz);
  *G = __fmaf_rn(c[5], dxz, __fmaf_rn(c[3], dxy, __fmaf_rn(c[0], dxx, gin)));
  *L = __fadd_rn(lin, dxx);
}

__device__ void gather(const TTIStep& a) {
  if (a.gather_row < 0) return;
  const int nthr = blockDim.x * blockDim.y * blockDim.z;
  const int b = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  const int t = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
  const int stride = nthr * (int)(gridDim.x * gridDim.y * gridDim.z);
  for (int i = b * nthr + t; i < a.n_rec; i += stride) {
    const int* c = a.rec + 3 * i;
    a.traces[(size_t)a.gather_row * a.n_rec + i] =
        a.p[a.es * ((size_t)c[0] * a.pitch_x + (size_t)c[1] * a.pitch_y + c[2])];
  }
}

// One thread per point; the checker variant.
__global__ void __launch_bounds__(256) tti_direct(const TTIStep a) {
  gather(a);
  const int z = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  const int x = blockIdx.z;
  if (z >= a.nz || y >= a.ny) return;
  const size_t o = (size_t)x * a.pitch_x + (size_t)y * a.pitch_y + z;
  const size_t e = (size_t)a.es * o;  // level element of the point
  const float k = a.prm[0][o], pa = a.prm[1][o], pb = a.prm[2][o];
  const float c[6] = {a.prm[3][o], a.prm[4][o], a.prm[5][o], a.prm[6][o], a.prm[7][o], a.prm[8][o]};
  float Gp, Lp, Gr, Lr;
  gl_op(a.p, a, x, y, z, c, &Gp, &Lp);
  gl_op(a.r, a, x, y, z, c, &Gr, &Lr);
  const float Hp = __fsub_rn(Lp, Gp);
  float pn = __fmaf_rn(k, __fmaf_rn(pa, Hp, __fmul_rn(pb, Gr)), __fmaf_rn(2.0f, a.p[e], -a.pp[e]));
  float rn = __fmaf_rn(k, __fmaf_rn(pb, Hp, Gr), __fmaf_rn(2.0f, a.r[e], -a.rp[e]));
  if (a.gx) {
    const float g = __fmul_rn(__fmul_rn(a.gx[x], a.gy[y]), a.gz[z]);
    pn = __fmul_rn(pn, g);
    rn = __fmul_rn(rn, g);
  }
  if (x == a.sx && y == a.sy && z == a.sz && a.it < a.n_series) {
    pn = __fadd_rn(pn, a.series[a.it]);
    rn = __fadd_rn(rn, a.series[a.it]);
  }
  a.pn[e] = pn;
  a.rn[e] = rn;
}

__global__ void tti_gather_kernel(const float* p, const int* rec, int n_rec, float* traces, int row,
                                  int pitch_y, long long pitch_x, int es) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_rec) {
    const int* c = rec + 3 * i;
    traces[(size_t)row * n_rec + i] = p[es * ((size_t)c[0] * pitch_x + (size_t)c[1] * pitch_y + c[2])];
  }
}

#define TTI_CUDA(call)                                    \
  do {                                                    \
    cudaError_t e_ = (call);                              \
    if (e_ != cudaSuccess) return fdr::cuda_fail(e_, #call); \
  } while (0)

// ============================================================ stream kernel
// 2.5D streaming TTI step.  A CTA of 512 threads owns a 32(z) x 16(y) column
// tile (one point per thread, a warp = one z row) and streams it along x.
// Stream plane p (x_n = xb - R + p) arrives by TMA in one ring stage holding
//   the p and r boxes of x_n (y/z halo: the in-plane derivatives),
//   the in-plane Gzz coefficients cyy, czz, cyz of x_n,
//   and, for the plane computed at this iteration (x_c = x_n - R), its
//   k, a, b, cxx, cxy, cxz and the prev levels of p and r.
// When x_n arrives each thread forms u, D1y u, D1z u, dyy, dzz and (through a
// shared D1z buffer over the box rows) dyz, and the in-plane partial sums
// gin = cyz dyz + (czz dzz + cyy dyy) and lin = dyy + dzz; x-direction values
// travel in register windows (u, D1y u, D1z u: 2R+1 planes; gin, lin: R+1),
// so the x derivatives dxx, dxy = D1x(D1y u), dxz = D1x(D1z u) of x_c need no
// shared memory.  Stages are recycled by the last warp to release them (empty
// mbarrier, as in acoustic_queue); one __syncthreads per plane orders the
// D1z buffer.
#ifndef FDR_TTI_TY
#define FDR_TTI_TY 16
#endif
#ifndef FDR_TTI_TZ
#define FDR_TTI_TZ 32
#endif
constexpr int TTZ = FDR_TTI_TZ, TTY = FDR_TTI_TY, TNT = TTZ * TTY;
constexpr int TMINB = TTY <= 8 ? 2 : 1;  // CTAs per SM the tile is sized for

template <int R>
struct TGeo {
  static constexpr int LZ = (R + 3) / 4 * 4;
  static constexpr int BZ = TTZ + 2 * LZ;
  static constexpr int BY = TTY + 2 * R;
  static constexpr int BOX_BYTES = BZ * BY * 4;
  static constexpr int BOX = (BOX_BYTES + 127) / 128 * 32;  // floats, 128-B aligned
  static constexpr int TILE = TTY * TTZ;                     // 2 KB
  static constexpr int DZ = BY * TTZ;                        // D1z rows of the box
  // stage layout (floats)
  static constexpr int O_BP = 0, O_BR = BOX, O_DZP = 2 * BOX, O_DZR = O_DZP + DZ;
  static constexpr int O_IN = O_DZR + DZ;                    // cyy czz cyz (3 tiles)
  static constexpr int O_CEN = O_IN + 3 * TILE;              // k a b cxx cxy cxz prev_p prev_r
  static constexpr int STAGE = O_CEN + 8 * TILE;
#ifdef FDR_TTI_NS
  static constexpr int NS = FDR_TTI_NS;
#else
  static constexpr int NS = 4;
#endif
#ifdef FDR_TTI_U
  static constexpr int U = FDR_TTI_U;
#else
  // planes per unrolled round: the whole window period 2R+1, so tti_pack's
  // windows rotate by renaming (no shifts; measured 81.2 against 78.5 GPts/s
  // for U = 2 with shifts at config 4, which had beaten U = 1 and U = 3)
  static constexpr int U = 2 * R + 1;
#endif
  static constexpr int QW = 2 * R + U;                       // x-window length
  static constexpr int GW = R + U;                           // delayed in-plane window
  static constexpr int NWARPS = TNT / 32;
  static constexpr size_t SMEM = size_t(NS) * STAGE * 4 + 3 * NS * 8;  // full, empty, D1z-ready
};

struct TTIMaps {
  CUtensorMap box_p, box_r;   // current levels, boxes with halo
  CUtensorMap prev_p, prev_r; // previous levels, tiles
  CUtensorMap prm[9];         // k a b cxx cyy czz cxy cyz cxz, tiles
};

FDR_DEV void mbar_arrive_ta(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
FDR_DEV void mbar_arrive_t(uint64_t* bar) { mbar_arrive_ta(smem_u32(bar)); }

FDR_DEV bool mbar_arrive_last_a(uint32_t bar) {
  uint64_t state;
  uint32_t pending;
  asm volatile("mbarrier.arrive.shared::cta.b64 %0, [%1];" : "=l"(state) : "r"(bar) : "memory");
  asm volatile("mbarrier.pending_count.b64 %0, %1;" : "=r"(pending) : "l"(state));
  return pending == 1;
}
FDR_DEV bool mbar_arrive_last(uint64_t* bar) { return mbar_arrive_last_a(smem_u32(bar)); }

template <int R>
FDR_DEV float d1_row(const float* row, const float* w1) {  // D1 along z at row[0]
  float d = __fmul_rn(w1[1], __fsub_rn(row[1], row[-1]));
#pragma unroll
  for (int j = 2; j <= R; ++j) d = __fmaf_rn(w1[j], __fsub_rn(row[j], row[-j]), d);
  return d;
}

template <int R, bool SPONGE>
__global__ void __launch_bounds__(TNT, TMINB) tti_stream(const __grid_constant__ TTIMaps maps,
                                                     const TTIStep a) {
  using G = TGeo<R>;
  extern __shared__ __align__(128) float smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + G::NS * G::STAGE);
  uint64_t* empty = full + G::NS;

  gather(a);
  const int tid = threadIdx.x;
  const int tz = tid % TTZ, ty = tid / TTZ;
  const int zt = blockIdx.x * TTZ, yt = blockIdx.y * TTY;
  const int xb = blockIdx.z * a.gather_pad_chunk;
  const int xe = min(a.nx, xb + a.gather_pad_chunk);
  if (xb >= xe) return;
  const int n = xe - xb;
  const int nplanes = n + 2 * R;
  const bool leader = (tid & 31) == 0;

  auto issue = [&](int p, int s) {
    float* st = smem + s * G::STAGE;
    const int xn = xb - R + p;
    const bool cen = p >= 2 * R;
    const uint32_t bytes = 2 * G::BOX_BYTES + 3 * G::TILE * 4 + (cen ? 8 * G::TILE * 4 : 0);
    mbar_arrive_expect_tx(&full[s], bytes);
    tma_load_3d(st + G::O_BP, &maps.box_p, &full[s], zt - G::LZ, yt - R, xn);
    tma_load_3d(st + G::O_BR, &maps.box_r, &full[s], zt - G::LZ, yt - R, xn);
    tma_load_3d(st + G::O_IN + 0 * G::TILE, &maps.prm[4], &full[s], zt, yt, xn);  // cyy
    tma_load_3d(st + G::O_IN + 1 * G::TILE, &maps.prm[5], &full[s], zt, yt, xn);  // czz
    tma_load_3d(st + G::O_IN + 2 * G::TILE, &maps.prm[7], &full[s], zt, yt, xn);  // cyz
    if (cen) {
      const int xc = xn - R;
      const int src[6] = {0, 1, 2, 3, 6, 8};  // k a b cxx cxy cxz
#pragma unroll
      for (int i = 0; i < 6; ++i)
        tma_load_3d(st + G::O_CEN + i * G::TILE, &maps.prm[src[i]], &full[s], zt, yt, xc);
      tma_load_3d(st + G::O_CEN + 6 * G::TILE, &maps.prev_p, &full[s], zt, yt, xc);
      tma_load_3d(st + G::O_CEN + 7 * G::TILE, &maps.prev_r, &full[s], zt, yt, xc);
    }
  };
  if (tid == 0) {
    prefetch_tensormap(&maps.box_p);
    prefetch_tensormap(&maps.box_r);
    for (int s = 0; s < G::NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], G::NWARPS);
    }
    fence_barrier_init();
    for (int p = 0; p < G::NS && p < nplanes; ++p) issue(p, p);
  }
  __syncthreads();

  const int y = yt + ty, z = zt + tz;
  const bool ok = y < a.ny && z < a.nz;
  const int bown = (ty + R) * G::BZ + G::LZ + tz;  // own point in a box
  const int town = ty * TTZ + tz;                   // own point in a tile
  // halo rows of the D1z buffer this thread fills (box rows 0..R-1, TY+R..)
  const int hrow = ty < R ? ty : (ty < 2 * R ? TTY + ty : -1);
  float gy = 1.0f, gz = 1.0f;
  if (SPONGE && ok) {
    gy = a.gy[y];
    gz = a.gz[z];
  }
  const bool src_here = a.sx >= 0 && y == a.sy && z == a.sz && a.it < a.n_series;
  const float qsrc = src_here ? a.series[a.it] : 0.0f;
  const int kinj = src_here ? a.sx - xb : -1;
  const uint32_t px32 = (uint32_t)a.pitch_x;
  const uint32_t oidx0 = (uint32_t)xb * px32 + (uint32_t)y * (uint32_t)a.pitch_y + (uint32_t)z;

  // x-direction windows: at round base p0, index i <-> stream plane p0 - 2R + i
  float pu[G::QW], py[G::QW], pz[G::QW], ru[G::QW], ry[G::QW], rz[G::QW];
  // delayed in-plane sums: index i <-> stream plane p0 - R + i
  float pg[G::GW], pl[G::GW], rg[G::GW];
#pragma unroll
  for (int i = 0; i < G::QW; ++i) pu[i] = py[i] = pz[i] = ru[i] = ry[i] = rz[i] = 0.0f;
#pragma unroll
  for (int i = 0; i < G::GW; ++i) pg[i] = pl[i] = rg[i] = 0.0f;

  int slot = 0;
  uint32_t phase = 0;
#pragma unroll 1
  for (int p0 = 0; p0 < nplanes; p0 += G::U) {
#pragma unroll
    for (int u = 0; u < G::U; ++u) {
      const int p = p0 + u;
      if (p >= nplanes) break;
      mbar_wait(&full[slot], phase);
      float* st = smem + slot * G::STAGE;
      // ---- in-plane work on the newest plane, both fields
#pragma unroll
      for (int f = 0; f < 2; ++f) {
        const float* box = st + (f == 0 ? G::O_BP : G::O_BR);
        float* dzb = st + (f == 0 ? G::O_DZP : G::O_DZR);
        const float* c0 = box + bown;
        const float uo = c0[0];
        float dy1 = __fmul_rn(a.w1[1], __fsub_rn(c0[G::BZ], c0[-G::BZ]));
        float dyy = __fmul_rn(a.w2[0], uo);
#pragma unroll
        for (int j = 1; j <= R; ++j) {
          const float up = c0[j * G::BZ], um = c0[-j * G::BZ];
          if (j >= 2) dy1 = __fmaf_rn(a.w1[j], __fsub_rn(up, um), dy1);
          dyy = __fmaf_rn(a.w2[j], __fadd_rn(up, um), dyy);
        }
        float dz1 = __fmul_rn(a.w1[1], __fsub_rn(c0[1], c0[-1]));
        float dzz = __fmul_rn(a.w2[0], uo);
#pragma unroll
        for (int j = 1; j <= R; ++j) {
          const float up = c0[j], um = c0[-j];
          if (j >= 2) dz1 = __fmaf_rn(a.w1[j], __fsub_rn(up, um), dz1);
          dzz = __fmaf_rn(a.w2[j], __fadd_rn(up, um), dzz);
        }
        dzb[(ty + R) * TTZ + tz] = dz1;
        if (hrow >= 0) dzb[hrow * TTZ + tz] = d1_row<R>(box + hrow * G::BZ + G::LZ + tz, a.w1);
        if (f == 0) {
          pu[2 * R + u] = uo; py[2 * R + u] = dy1; pz[2 * R + u] = dz1;
          pl[R + u] = __fadd_rn(dyy, dzz);
        } else {
          ru[2 * R + u] = uo; ry[2 * R + u] = dy1; rz[2 * R + u] = dz1;
        }
        // gin = fma(cyz, dyz, fma(czz, dzz, cyy dyy)): the dyz term follows the barrier
        if (f == 0) pg[R + u] = __fmaf_rn(st[G::O_IN + 1 * G::TILE + town], dzz,
                                          __fmul_rn(st[G::O_IN + town], dyy));
        else rg[R + u] = __fmaf_rn(st[G::O_IN + 1 * G::TILE + town], dzz,
                                   __fmul_rn(st[G::O_IN + town], dyy));
      }
      __syncthreads();  // the D1z rows of both boxes are complete
#pragma unroll
      for (int f = 0; f < 2; ++f) {
        const float* dzb = st + (f == 0 ? G::O_DZP : G::O_DZR) + (ty + R) * TTZ + tz;
        float dyz = __fmul_rn(a.w1[1], __fsub_rn(dzb[TTZ], dzb[-TTZ]));
#pragma unroll
        for (int j = 2; j <= R; ++j) dyz = __fmaf_rn(a.w1[j], __fsub_rn(dzb[j * TTZ], dzb[-j * TTZ]), dyz);
        const float cyz = st[G::O_IN + 2 * G::TILE + town];
        if (f == 0) pg[R + u] = __fmaf_rn(cyz, dyz, pg[R + u]);
        else rg[R + u] = __fmaf_rn(cyz, dyz, rg[R + u]);
      }
      // ---- the plane R behind: x derivatives and the update
      const int k = p - 2 * R;
      float vk = 0.f, va = 0.f, vb = 0.f, cxx = 0.f, cxy = 0.f, cxz = 0.f, ppv = 0.f, rpv = 0.f;
      if (k >= 0) {
        const float* cen = st + G::O_CEN + town;
        vk = cen[0]; va = cen[G::TILE]; vb = cen[2 * G::TILE];
        cxx = cen[3 * G::TILE]; cxy = cen[4 * G::TILE]; cxz = cen[5 * G::TILE];
        ppv = cen[6 * G::TILE]; rpv = cen[7 * G::TILE];
      }
      // release the stage (every read of it is above)
      __syncwarp();
      if (leader && mbar_arrive_last(&empty[slot])) {
        mbar_wait(&empty[slot], phase);
        fence_proxy_async();  // generic-proxy reads of the stage before the TMA refill (cross-proxy WAR)
        if (p + G::NS < nplanes) issue(p + G::NS, slot);
      }
      if (++slot == G::NS) {
        slot = 0;
        phase ^= 1u;
      }
      if (k >= 0) {
        // window index of the centre plane (stream plane p - R): u + R
        float Gf[2], Lp = 0.f;
#pragma unroll
        for (int f = 0; f < 2; ++f) {
          const float* qu = f == 0 ? pu : ru;
          const float* qy = f == 0 ? py : ry;
          const float* qz = f == 0 ? pz : rz;
          const int c = u + R;
          float dxx = __fmul_rn(a.w2[0], qu[c]);
          float dxy = __fmul_rn(a.w1[1], __fsub_rn(qy[c + 1], qy[c - 1]));
          float dxz = __fmul_rn(a.w1[1], __fsub_rn(qz[c + 1], qz[c - 1]));
#pragma unroll
          for (int j = 1; j <= R; ++j) {
            dxx = __fmaf_rn(a.w2[j], __fadd_rn(qu[c + j], qu[c - j]), dxx);
            if (j >= 2) {
              dxy = __fmaf_rn(a.w1[j], __fsub_rn(qy[c + j], qy[c - j]), dxy);
              dxz = __fmaf_rn(a.w1[j], __fsub_rn(qz[c + j], qz[c - j]), dxz);
            }
          }
          const float gin = f == 0 ? pg[u] : rg[u];
          Gf[f] = __fmaf_rn(cxz, dxz, __fmaf_rn(cxy, dxy, __fmaf_rn(cxx, dxx, gin)));
          if (f == 0) Lp = __fadd_rn(pl[u], dxx);
        }
        const float Hp = __fsub_rn(Lp, Gf[0]);
        const float pc = pu[u + R], rc = ru[u + R];
        float pn = __fmaf_rn(vk, __fmaf_rn(va, Hp, __fmul_rn(vb, Gf[1])), __fmaf_rn(2.0f, pc, -ppv));
        float rn = __fmaf_rn(vk, __fmaf_rn(vb, Hp, Gf[1]), __fmaf_rn(2.0f, rc, -rpv));
        if (SPONGE) {
          const float g = __fmul_rn(__fmul_rn(__ldg(a.gx + xb + k), gy), gz);
          pn = __fmul_rn(pn, g);
          rn = __fmul_rn(rn, g);
        }
        if (k == kinj) {
          pn = __fadd_rn(pn, qsrc);
          rn = __fadd_rn(rn, qsrc);
        }
        if (ok) {
          const uint32_t o = oidx0 + (uint32_t)k * px32;
          a.pn[o] = pn;
          a.rn[o] = rn;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 2 * R; ++i) {
      pu[i] = pu[i + G::U]; py[i] = py[i + G::U]; pz[i] = pz[i + G::U];
      ru[i] = ru[i + G::U]; ry[i] = ry[i + G::U]; rz[i] = rz[i + G::U];
    }
#pragma unroll
    for (int i = 0; i < R; ++i) {
      pg[i] = pg[i + G::U]; pl[i] = pl[i + G::U]; rg[i] = rg[i + G::U];
    }
  }
}

// ============================================================ packed kernel
// tti_pack<R, SPONGE>: tti_stream with the two fields in the two lanes of
// packed f32x2 registers (lane 0: p, lane 1: r).  Both fields run the same
// derivative chains with the same weights and G coefficients, so every
// in-plane and x derivative, window entry and G partial sum is one packed
// value: half the arithmetic instructions at the same register count.  The
// D1z buffer interleaves (p, r) per point.  Only L(p) and the two final
// updates are per field (scalar, in the oracle's order).
FDR_DEV f2 bcast(float w) { return pk(w, w); }
FDR_DEV f2 ldpr(const float* p, const float* r, int off) { return pk(p[off], r[off]); }
// The same from a 32-bit shared address of the p element; the r box is `dr`
// bytes further.
FDR_DEV f2 ldpra(uint32_t ap, uint32_t dr, int off) {
  return pk(lds32a(ap + 4 * off), lds32a(ap + dr + 4 * off));
}
template <int R>
FDR_DEV f2 d1_row2a(uint32_t hp, uint32_t dr, const float* w1) {  // D1z, both fields
  f2 d = mul2(bcast(w1[1]), sub2(ldpra(hp, dr, 1), ldpra(hp, dr, -1)));
#pragma unroll
  for (int j = 2; j <= R; ++j) d = fma2(bcast(w1[j]), sub2(ldpra(hp, dr, j), ldpra(hp, dr, -j)), d);
  return d;
}
#ifndef FDR_TTI_ROT
#define FDR_TTI_ROT 1  // rotating windows (config 4: 78.5 -> 81.2 GPts/s)
#endif
#ifdef FDR_TTI_CARRY
constexpr bool TTI_CARRY = FDR_TTI_CARRY != 0;
#else
constexpr bool TTI_CARRY = true;
#endif
// Deferred dyz: plane p's D1z rows are consumed at iteration p + 1, so the
// wait for every warp's rows has a whole plane of slack (ncu: the per-plane
// wait on the D1z-ready barrier was the top stall; the 8 warps with halo rows
// arrive late every plane).  The rows live in the stage's D1z area, which TMA
// never writes, so releasing the stage at the end of iteration p stays safe;
// the area is rewritten at iteration p + NS, after every warp has arrived on
// the barrier of plane p + 2 (waited at p + 3), i.e. after its reads at p + 1.
#ifdef FDR_TTI_DEFER
constexpr bool TTI_DEFER = FDR_TTI_DEFER != 0;
#else
constexpr bool TTI_DEFER = true;
#endif
// With DEFER: the halo D1z rows (2R of them per plane) rotate over groups of
// 2R warps plane by plane instead of always falling to warps 0 .. 2R-1, so
// every warp does the same work over NG planes and the one-plane slack of the
// deferred wait absorbs the per-plane difference.
#ifdef FDR_TTI_HALT
constexpr bool TTI_HALT = FDR_TTI_HALT != 0;
#else
constexpr bool TTI_HALT = true;
#endif

// D1z of an interleaved (p, r) row from the 32-bit shared address of the
// own pair: one 8-byte load per tap
template <int R>
FDR_DEV f2 d1_row2i(uint32_t hp, const float* w1) {
  f2 d = mul2(bcast(w1[1]), sub2(lds64a(hp + 8), lds64a(hp - 8)));
#pragma unroll
  for (int j = 2; j <= R; ++j) d = fma2(bcast(w1[j]), sub2(lds64a(hp + 8 * j), lds64a(hp - 8 * j)), d);
  return d;
}

template <int R>
FDR_DEV f2 d1_row2(const float* hp, const float* hr, const float* w1) {  // D1z, both fields
  f2 d = mul2(bcast(w1[1]), sub2(ldpr(hp, hr, 1), ldpr(hp, hr, -1)));
#pragma unroll
  for (int j = 2; j <= R; ++j) d = fma2(bcast(w1[j]), sub2(ldpr(hp, hr, j), ldpr(hp, hr, -j)), d);
  return d;
}

template <int R, bool SPONGE, bool IL>
__global__ void __launch_bounds__(TNT, TMINB) tti_pack(const __grid_constant__ TTIMaps maps,
                                                       const TTIStep a) {
  using G = TGeo<R>;
  extern __shared__ __align__(128) float smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + G::NS * G::STAGE);
  uint64_t* empty = full + G::NS;
  uint64_t* dzrdy = empty + G::NS;  // per stage: every warp's D1z rows are written

  gather(a);
  const int tid = threadIdx.x;
  const int tz = tid % TTZ, ty = tid / TTZ;
  const int zt = blockIdx.x * TTZ, yt = blockIdx.y * TTY;
  const int xb = blockIdx.z * a.gather_pad_chunk;
  const int xe = min(a.nx, xb + a.gather_pad_chunk);
  if (xb >= xe) return;
  const int n = xe - xb;
  const int nplanes = n + 2 * R;
  const bool leader = (tid & 31) == 0;

  auto issue = [&](int p, int s) {
    float* st = smem + s * G::STAGE;
    const int xn = xb - R + p;
    const bool cen = p >= 2 * R;
    const uint32_t bytes = 2 * G::BOX_BYTES + 3 * G::TILE * 4 + (cen ? 8 * G::TILE * 4 : 0);
    mbar_arrive_expect_tx(&full[s], bytes);
    if (IL) {  // one box of (p, r) pairs: twice the z extent in floats
      tma_load_3d(st + G::O_BP, &maps.box_p, &full[s], 2 * (zt - G::LZ), yt - R, xn);
    } else {
      tma_load_3d(st + G::O_BP, &maps.box_p, &full[s], zt - G::LZ, yt - R, xn);
      tma_load_3d(st + G::O_BR, &maps.box_r, &full[s], zt - G::LZ, yt - R, xn);
    }
    tma_load_3d(st + G::O_IN + 0 * G::TILE, &maps.prm[4], &full[s], zt, yt, xn);  // cyy
    tma_load_3d(st + G::O_IN + 1 * G::TILE, &maps.prm[5], &full[s], zt, yt, xn);  // czz
    tma_load_3d(st + G::O_IN + 2 * G::TILE, &maps.prm[7], &full[s], zt, yt, xn);  // cyz
    if (cen) {
      const int xc = xn - R;
      const int src[6] = {0, 1, 2, 3, 6, 8};  // k a b cxx cxy cxz
#pragma unroll
      for (int i = 0; i < 6; ++i)
        tma_load_3d(st + G::O_CEN + i * G::TILE, &maps.prm[src[i]], &full[s], zt, yt, xc);
      if (IL) {  // (p, r) pairs of the previous level
        tma_load_3d(st + G::O_CEN + 6 * G::TILE, &maps.prev_p, &full[s], 2 * zt, yt, xc);
      } else {
        tma_load_3d(st + G::O_CEN + 6 * G::TILE, &maps.prev_p, &full[s], zt, yt, xc);
        tma_load_3d(st + G::O_CEN + 7 * G::TILE, &maps.prev_r, &full[s], zt, yt, xc);
      }
    }
  };
  if (tid == 0) {
    prefetch_tensormap(&maps.box_p);
    if (!IL) prefetch_tensormap(&maps.box_r);
    for (int s = 0; s < G::NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], G::NWARPS);
      mbar_init(&dzrdy[s], G::NWARPS);
    }
    fence_barrier_init();
    for (int p = 0; p < G::NS && p < nplanes; ++p) issue(p, p);
  }
  __syncthreads();

  const int y = yt + ty, z = zt + tz;
  const bool ok = y < a.ny && z < a.nz;
  const int bown = (ty + R) * G::BZ + G::LZ + tz;
  const int town = ty * TTZ + tz;
  constexpr bool DEFER = TTI_DEFER && TTI_CARRY && G::NS >= 4;
  constexpr int HG = 2 * R, NG = TTY / HG;  // halo-row warp groups (ALT)
  constexpr bool ALT = DEFER && TTI_HALT && NG >= 2;
  const int hgrp = ty / HG, hh = ty % HG;
  const int hrow = ALT ? (hgrp < NG ? (hh < R ? hh : TTY + hh) : -1)
                       : (ty < R ? ty : (ty < 2 * R ? TTY + ty : -1));
  int hturn = 0;  // ALT: the group computing the halo rows of this plane
  float gy = 1.0f, gz = 1.0f;
  if (SPONGE && ok) {
    gy = a.gy[y];
    gz = a.gz[z];
  }
  const bool src_here = a.sx >= 0 && y == a.sy && z == a.sz && a.it < a.n_series;
  const float qsrc = src_here ? a.series[a.it] : 0.0f;
  const int kinj = src_here ? a.sx - xb : -1;
  const uint32_t px32 = (uint32_t)a.pitch_x;
  const uint32_t oidx0 = (uint32_t)xb * px32 + (uint32_t)y * (uint32_t)a.pitch_y + (uint32_t)z;

  // x windows (u, D1y u, D1z u; lane 0 p, lane 1 r): index i <-> plane p0 - 2R + i
  // FDR_TTI_ROT: the windows are rings of period 2R+1 walked by a round of
  // U = 2R+1 planes (pure register renaming, no shifts); otherwise shifted
  // by U at the end of each round
  constexpr bool ROT = FDR_TTI_ROT != 0 && G::U == 2 * R + 1;
  constexpr int PER = 2 * R + 1;
  constexpr int NQW = ROT ? PER : G::QW, NGW = ROT ? PER : G::GW;
  f2 qu[NQW], qy[NQW], qz[NQW];
  // delayed in-plane sums: G partial (both fields), L partial (p): plane p0 - R + i
  f2 gq[NGW];
  float pl[NGW];
#pragma unroll
  for (int i = 0; i < NQW; ++i) qu[i] = qy[i] = qz[i] = 0ull;
#pragma unroll
  for (int i = 0; i < NGW; ++i) {
    gq[i] = 0ull;
    pl[i] = 0.0f;
  }

  int slot = 0;
  uint32_t phase = 0;
  // 32-bit shared addresses of this thread's elements in stage `slot`,
  // carried across planes so ptxas cannot rematerialise them from the thread
  // index every plane (as in acoustic_queue)
  constexpr bool CA = TTI_CARRY;
  constexpr uint32_t SB = G::STAGE * 4u, DR = (G::O_BR - G::O_BP) * 4u;
  const int hr0 = hrow >= 0 ? hrow : 0;
  // IL: (p, r) pairs, the own point at float 2 * bown of the box
  uint32_t ab = smem_u32(smem + G::O_BP + (IL ? 2 : 1) * bown), at = smem_u32(smem + town);
  uint32_t adz = smem_u32(smem + G::O_DZP + 2 * ((ty + R) * TTZ + tz));
  uint32_t ah = smem_u32(smem + G::O_BP + (IL ? 2 : 1) * (hr0 * G::BZ + G::LZ + tz));
  uint32_t ahdz = smem_u32(smem + G::O_DZP + 2 * (hr0 * TTZ + tz));
  uint32_t af = smem_u32(full);  // full[slot]; empty[] and dzrdy[] follow
  // DEFER: the previous plane's D1z rows (own address), barrier, parity and cyz
  uint32_t adzp = 0, afp = 0, phasep = 0;
  float cyzp = 0.0f;
  auto dyz_at = [&](uint32_t adr) {
    auto ldz = [&](int rows) { return lds64a(adr + 8 * rows * TTZ); };
    f2 d = mul2(bcast(a.w1[1]), sub2(ldz(1), ldz(-1)));
#pragma unroll
    for (int j = 2; j <= R; ++j) d = fma2(bcast(a.w1[j]), sub2(ldz(j), ldz(-j)), d);
    return d;
  };
#pragma unroll 1
  for (int p0 = 0; p0 < nplanes; p0 += G::U) {
#pragma unroll
    for (int u = 0; u < G::U; ++u) {
      const int p = p0 + u;
      if (p >= nplanes) break;
      if (CA) mbar_wait_a(af, phase); else mbar_wait(&full[slot], phase);
      float* st = smem + slot * G::STAGE;
      auto lp = [&](int off) -> f2 {
        if (IL) return CA ? lds64a(ab + 8 * off) : *reinterpret_cast<const f2*>(st + G::O_BP + 2 * (bown + off));
        return CA ? ldpra(ab, DR, off) : ldpr(st + G::O_BP + bown, st + G::O_BR + bown, off);
      };
      auto lt = [&](int off) { return CA ? lds32a(at + 4 * off) : st[town + off]; };
      // ---- in-plane work on the newest plane, both fields packed
      const f2 uo = lp(0);
      f2 dy1 = mul2(bcast(a.w1[1]), sub2(lp(G::BZ), lp(-G::BZ)));
      f2 dyy = mul2(bcast(a.w2[0]), uo);
#pragma unroll
      for (int j = 1; j <= R; ++j) {
        const f2 up = lp(j * G::BZ), um = lp(-j * G::BZ);
        if (j >= 2) dy1 = fma2(bcast(a.w1[j]), sub2(up, um), dy1);
        dyy = fma2(bcast(a.w2[j]), add2(up, um), dyy);
      }
      f2 dz1 = mul2(bcast(a.w1[1]), sub2(lp(1), lp(-1)));
      f2 dzz = mul2(bcast(a.w2[0]), uo);
#pragma unroll
      for (int j = 1; j <= R; ++j) {
        const f2 up = lp(j), um = lp(-j);
        if (j >= 2) dz1 = fma2(bcast(a.w1[j]), sub2(up, um), dz1);
        dzz = fma2(bcast(a.w2[j]), add2(up, um), dzz);
      }
      float* dzb = st + G::O_DZP;  // interleaved (p, r) D1z rows, 2 * BY * TTZ floats
      if (CA) {
        sts64a(adz, dz1);
        if (ALT ? hgrp == hturn : hrow >= 0) sts64a(ahdz, IL ? d1_row2i<R>(ah, a.w1) : d1_row2a<R>(ah, DR, a.w1));
      } else {
        *reinterpret_cast<f2*>(dzb + 2 * ((ty + R) * TTZ + tz)) = dz1;
        if (hrow >= 0)
          *reinterpret_cast<f2*>(dzb + 2 * (hrow * TTZ + tz)) =
              IL ? d1_row2i<R>(smem_u32(st + G::O_BP + 2 * (hrow * G::BZ + G::LZ + tz)), a.w1)
                 : d1_row2<R>(st + G::O_BP + hrow * G::BZ + G::LZ + tz, st + G::O_BR + hrow * G::BZ + G::LZ + tz, a.w1);
      }
      auto QI = [](int i) { return ROT ? i % PER : i; };  // window slot (compile-time after unrolling)
      qu[QI(2 * R + u)] = uo;
      qy[QI(2 * R + u)] = dy1;
      qz[QI(2 * R + u)] = dz1;
      pl[QI(R + u)] = __fadd_rn(lo(dyy), lo(dzz));
      // gin = fma(cyz, dyz, fma(czz, dzz, cyy dyy)): the dyz term follows the barrier
      gq[QI(R + u)] = fma2(bcast(lt(G::O_IN + 1 * G::TILE)), dzz, mul2(bcast(lt(G::O_IN)), dyy));
      // Split barrier: announce this warp's D1z rows, update the plane R
      // behind (which needs no D1z row of this plane), then wait for every
      // warp's rows.  The warps' skew is absorbed by useful work instead of a
      // __syncthreads.
      __syncwarp();
      if (CA ? elect_one() : leader) {
        if (CA) mbar_arrive_ta(af + 16u * G::NS); else mbar_arrive_t(&dzrdy[slot]);
      }
      // DEFER: dyz of the previous plane completes its G partial sum
      // (gin = fma(cyz, dyz, ...)); at R = 1 the update below needs it
      auto deferred = [&]() {
        if (p > 0) {
          mbar_wait_a(afp + 16u * G::NS, phasep);
          gq[QI(R + u - 1 + (ROT ? PER : 0))] = fma2(bcast(cyzp), dyz_at(adzp), gq[QI(R + u - 1 + (ROT ? PER : 0))]);
        }
      };
      if constexpr (DEFER && R == 1) deferred();
      // ---- the plane R behind: x derivatives and the update
      const int k = p - 2 * R;
      if (k >= 0) {
        const float vk = lt(G::O_CEN), va = lt(G::O_CEN + G::TILE), vb = lt(G::O_CEN + 2 * G::TILE);
        const float cxx = lt(G::O_CEN + 3 * G::TILE), cxy = lt(G::O_CEN + 4 * G::TILE);
        const float cxz = lt(G::O_CEN + 5 * G::TILE);
        float ppv, rpv;
        if (IL) {  // one 8-byte load of the (p, r) pair
          const f2 pr = CA ? lds64a(at + 4u * (G::O_CEN + 6 * G::TILE + town))
                           : *reinterpret_cast<const f2*>(st + G::O_CEN + 6 * G::TILE + 2 * town);
          ppv = lo(pr);
          rpv = hi(pr);
        } else {
          ppv = lt(G::O_CEN + 6 * G::TILE);
          rpv = lt(G::O_CEN + 7 * G::TILE);
        }
        const int c = u + R;
        f2 dxx = mul2(bcast(a.w2[0]), qu[QI(c)]);
        f2 dxy = mul2(bcast(a.w1[1]), sub2(qy[QI(c + 1)], qy[QI(c - 1)]));
        f2 dxz = mul2(bcast(a.w1[1]), sub2(qz[QI(c + 1)], qz[QI(c - 1)]));
#pragma unroll
        for (int j = 1; j <= R; ++j) {
          dxx = fma2(bcast(a.w2[j]), add2(qu[QI(c + j)], qu[QI(c - j)]), dxx);
          if (j >= 2) {
            dxy = fma2(bcast(a.w1[j]), sub2(qy[QI(c + j)], qy[QI(c - j)]), dxy);
            dxz = fma2(bcast(a.w1[j]), sub2(qz[QI(c + j)], qz[QI(c - j)]), dxz);
          }
        }
        const f2 gf = fma2(bcast(cxz), dxz, fma2(bcast(cxy), dxy, fma2(bcast(cxx), dxx, gq[QI(u)])));
        const float Lp = __fadd_rn(pl[QI(u)], lo(dxx));
        const float Hp = __fsub_rn(Lp, lo(gf));
        const float Gr = hi(gf);
        const float pc = lo(qu[QI(c)]), rc = hi(qu[QI(c)]);
        float pn = __fmaf_rn(vk, __fmaf_rn(va, Hp, __fmul_rn(vb, Gr)), __fmaf_rn(2.0f, pc, -ppv));
        float rn = __fmaf_rn(vk, __fmaf_rn(vb, Hp, Gr), __fmaf_rn(2.0f, rc, -rpv));
        if (SPONGE) {
          const float g = __fmul_rn(__fmul_rn(__ldg(a.gx + xb + k), gy), gz);
          pn = __fmul_rn(pn, g);
          rn = __fmul_rn(rn, g);
        }
        if (k == kinj) {
          pn = __fadd_rn(pn, qsrc);
          rn = __fadd_rn(rn, qsrc);
        }
        if (ok) {
          const uint32_t o = oidx0 + (uint32_t)k * px32;
          if (IL) {
            asm volatile("st.global.v2.f32 [%0], {%1, %2};" ::"l"(a.pn + 2u * o), "f"(pn), "f"(rn) : "memory");
          } else {
            a.pn[o] = pn;
            a.rn[o] = rn;
          }
        }
      }
      if constexpr (DEFER) {
        if constexpr (R > 1) deferred();
        cyzp = lt(G::O_IN + 2 * G::TILE);  // this plane's cyz, read before the stage is released
      } else {
      // the D1z rows are complete
      if (CA) mbar_wait_a(af + 16u * G::NS, phase); else mbar_wait(&dzrdy[slot], phase);
        const float* db = dzb + 2 * ((ty + R) * TTZ + tz);
        auto ldz = [&](int rows) {
          return CA ? lds64a(adz + 8 * rows * TTZ) : *reinterpret_cast<const f2*>(db + 2 * rows * TTZ);
        };
        f2 dyz = mul2(bcast(a.w1[1]), sub2(ldz(1), ldz(-1)));
#pragma unroll
        for (int j = 2; j <= R; ++j) dyz = fma2(bcast(a.w1[j]), sub2(ldz(j), ldz(-j)), dyz);
        gq[QI(R + u)] = fma2(bcast(lt(G::O_IN + 2 * G::TILE)), dyz, gq[QI(R + u)]);
      }
      // release the stage (every read of it is above)
      __syncwarp();
      if (CA ? (elect_one() && mbar_arrive_last_a(af + 8u * G::NS))
             : (leader && mbar_arrive_last(&empty[slot]))) {
        if (CA) mbar_wait_a(af + 8u * G::NS, phase); else mbar_wait(&empty[slot], phase);
        fence_proxy_async();  // generic-proxy reads of the stage before the TMA refill (cross-proxy WAR)
        if (p + G::NS < nplanes) issue(p + G::NS, slot);
      }
      if constexpr (DEFER) {
        adzp = adz;
        afp = af;
        phasep = phase;
      }
      if constexpr (ALT) {
        if (++hturn == NG) hturn = 0;
      }
      if (CA) {
        ab += SB; at += SB; adz += SB; ah += SB; ahdz += SB; af += 8u;
      }
      if (++slot == G::NS) {
        slot = 0;
        phase ^= 1u;
        if (CA) {
          ab -= G::NS * SB; at -= G::NS * SB; adz -= G::NS * SB;
          ah -= G::NS * SB; ahdz -= G::NS * SB; af -= 8u * G::NS;
        }
      }
    }
    if (!ROT) {
#pragma unroll
      for (int i = 0; i < 2 * R; ++i) {
        qu[i] = qu[i + G::U];
        qy[i] = qy[i + G::U];
        qz[i] = qz[i + G::U];
      }
#pragma unroll
      for (int i = 0; i < R; ++i) {
        gq[i] = gq[i + G::U];
        pl[i] = pl[i + G::U];
      }
    }
  }
}

static int tti_encode(CUtensorMap* map, const float* base, const fdr_tti_args* a, int bz, int by,
                      int es = 1) {
  typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                          const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                          CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                          CUtensorMapFloatOOBfill);
  const Enc enc = reinterpret_cast<Enc>(fdr::tensor_map_encoder());
  if (!enc) return fail(FDR_ECUDA, "cuTensorMapEncodeTiled unavailable");
  // es = 2: (p, r) pairs, i.e. a tensor with twice the z extent in floats
  cuuint64_t dims[3] = {(cuuint64_t)a->nz * es, (cuuint64_t)a->ny, (cuuint64_t)a->nx};
  cuuint64_t strides[2] = {(cuuint64_t)a->pitch_y * 4 * es, (cuuint64_t)a->pitch_x * 4 * es};
  cuuint32_t box[3] = {(cuuint32_t)(bz * es), (cuuint32_t)by, 1}, els[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides,
                   box, els, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(FDR_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return FDR_OK;
}

template <int R, bool PACK>
static int stream_inst(const TTIStep& s, const fdr_tti_args* a, int k, cudaStream_t st,
                       int* chunk_cache) {
  using G = TGeo<R>;
  const bool sponge = s.gx != nullptr;
  const bool il = a->interleaved != 0;
  auto kern = PACK ? (il ? (sponge ? tti_pack<R, true, true> : tti_pack<R, false, true>)
                         : (sponge ? tti_pack<R, true, false> : tti_pack<R, false, false>))
                   : (sponge ? tti_stream<R, true> : tti_stream<R, false>);
  int occ = 0, nsm = 0;
  const int frc = fdr::launch_facts(reinterpret_cast<const void*>(kern), TNT, G::SMEM, &occ, &nsm);
  if (frc != FDR_OK) return frc;
  TTIMaps maps;
  const int cur = (2 + k) % 3, prev = (1 + k) % 3;
  int rc = FDR_OK;
  if (il) {  // r[i] == p[i] + 1: the p maps cover the pairs; the r maps are unused
    rc = tti_encode(&maps.box_p, a->p[cur], a, G::BZ, G::BY, 2);
    if (rc == FDR_OK) rc = tti_encode(&maps.prev_p, a->p[prev], a, TTZ, TTY, 2);
    maps.box_r = maps.box_p;
    maps.prev_r = maps.prev_p;
  } else {
    rc = tti_encode(&maps.box_p, a->p[cur], a, G::BZ, G::BY);
    if (rc == FDR_OK) rc = tti_encode(&maps.box_r, a->r[cur], a, G::BZ, G::BY);
    if (rc == FDR_OK) rc = tti_encode(&maps.prev_p, a->p[prev], a, TTZ, TTY);
    if (rc == FDR_OK) rc = tti_encode(&maps.prev_r, a->r[prev], a, TTZ, TTY);
  }
  for (int i = 0; i < 9 && rc == FDR_OK; ++i) rc = tti_encode(&maps.prm[i], a->params[i], a, TTZ, TTY);
  if (rc != FDR_OK) return rc;
  TTIStep t = s;
  const int tzn = (a->nz + TTZ - 1) / TTZ, tyn = (a->ny + TTY - 1) / TTY;
  if (*chunk_cache <= 0) {
    const long tiles = (long)tzn * tyn, slots = (long)occ * nsm;
    double best = 1e30;
    int best_c = 1;
    for (int c = 1; c <= std::max(1, a->nx / (2 * R)); ++c) {
      const int len = (a->nx + c - 1) / c;
      const int cc = (a->nx + len - 1) / len;
      const long waves = (tiles * cc + slots - 1) / slots;
      const double tt = (double)waves * (len + 0.3 * 2 * R);
      if (tt < best * 0.999) {
        best = tt;
        best_c = cc;
      }
    }
    *chunk_cache = (a->nx + best_c - 1) / best_c;
  }
  t.gather_pad_chunk = *chunk_cache;
  dim3 grid(tzn, tyn, (a->nx + t.gather_pad_chunk - 1) / t.gather_pad_chunk);
  kern<<<grid, TNT, G::SMEM, st>>>(maps, t);
  TTI_CUDA(cudaGetLastError());
  return FDR_OK;
}

int tti_stream_launch(const TTIStep& s, const fdr_tti_args* a, int k, cudaStream_t st,
                      int* chunk_cache, bool pack) {
  switch (a->order / 2) {
    case 1: return pack ? stream_inst<1, true>(s, a, k, st, chunk_cache) : stream_inst<1, false>(s, a, k, st, chunk_cache);
    case 2: return pack ? stream_inst<2, true>(s, a, k, st, chunk_cache) : stream_inst<2, false>(s, a, k, st, chunk_cache);
    case 3: return pack ? stream_inst<3, true>(s, a, k, st, chunk_cache) : stream_inst<3, false>(s, a, k, st, chunk_cache);
    case 4: return pack ? stream_inst<4, true>(s, a, k, st, chunk_cache) : stream_inst<4, false>(s, a, k, st, chunk_cache);
    default: return fail(FDR_EINVAL, "TTI stream kernel supports orders 2..8, got %d", a->order);
  }
}

int tti_stream_prepare(const fdr_tti_args* a) {
  if ((uint64_t)a->nx * (uint64_t)a->pitch_x * (a->interleaved ? 2u : 1u) >= (1ull << 32))
    return fail(FDR_EINVAL, "the TTI stream kernel indexes grids of < 2^32 elements");
  return FDR_OK;
}

static int validate(const fdr_tti_args* a) {
  if (!a) return fail(FDR_EINVAL, "args is NULL");
  if (a->abi_version != FDR_ABI_VERSION)
    return fail(FDR_EINVAL, "abi_version %d != library %d", a->abi_version, FDR_ABI_VERSION);
  if (a->order < 2 || a->order % 2 || a->order > 16)
    return fail(FDR_EINVAL, "TTI order must be even and within [2, 16], got %d", a->order);
  const int r = a->order / 2;
  if (a->nx < 2 * r + 1 || a->ny < 2 * r + 1 || a->nz < 2 * r + 1)
    return fail(FDR_EINVAL, "interior dims (%d, %d, %d) too small for halo width %d", a->nx,
                a->ny, a->nz, r);
  if (a->pitch_y < a->nz || a->pitch_y % 4 || a->pitch_x < (int64_t)a->ny * a->pitch_y ||
      a->pitch_x % 4)
    return fail(FDR_EINVAL, "bad pitches");
  if (a->n_steps < 0 || a->it0 < 0) return fail(FDR_EINVAL, "n_steps and it0 must be >= 0");
  for (int i = 0; i < 3; ++i)
    if (!a->p[i] || !a->r[i]) return fail(FDR_EINVAL, "level pointer NULL");
  if (a->interleaved != 0 && a->interleaved != 1)
    return fail(FDR_EINVAL, "interleaved must be 0 or 1, got %d", a->interleaved);
  if (a->interleaved)
    for (int i = 0; i < 3; ++i)
      if (a->r[i] != a->p[i] + 1)
        return fail(FDR_EINVAL, "interleaved levels need r[i] == p[i] + 1 (level %d)", i);
  if (a->interleaved && a->variant == FDR_VARIANT_TMA)
    return fail(FDR_EINVAL, "the TMA (tti_stream) variant takes separate p/r levels (interleaved = 0)");
  for (int i = 0; i < 9; ++i)
    if (!a->params[i]) return fail(FDR_EINVAL, "parameter grid %d is NULL", i);
  if (a->sponge_x && (!a->sponge_y || !a->sponge_z))
    return fail(FDR_EINVAL, "sponge needs all three profiles");
  if (a->src_x >= 0 && (a->src_x >= a->nx || a->src_y < 0 || a->src_y >= a->ny ||
                        a->src_z < 0 || a->src_z >= a->nz))
    return fail(FDR_EINVAL, "source location outside interior");
  if (a->n_rec > 0 && (!a->rec_xyz || !a->traces))
    return fail(FDR_EINVAL, "receiver coordinates or trace buffer NULL");
  if (a->variant < 0 || a->variant > FDR_VARIANT_QUEUE)
    return fail(FDR_EINVAL, "unknown TTI variant %d", a->variant);
  return FDR_OK;
}

void fill(TTIStep& s, const fdr_tti_args* a, int k) {
  memset(&s, 0, sizeof(s));
  s.pn = a->p[(0 + k) % 3];
  s.pp = a->p[(1 + k) % 3];
  s.p = a->p[(2 + k) % 3];
  s.rn = a->r[(0 + k) % 3];
  s.rp = a->r[(1 + k) % 3];
  s.r = a->r[(2 + k) % 3];
  for (int i = 0; i < 9; ++i) s.prm[i] = a->params[i];
  s.nx = a->nx;
  s.ny = a->ny;
  s.nz = a->nz;
  s.pitch_y = a->pitch_y;
  s.pitch_x = a->pitch_x;
  s.radius = a->order / 2;
  for (int j = 0; j <= FDR_MAX_RADIUS; ++j) {
    s.w2[j] = a->w2[j];
    s.w1[j] = a->w1[j];
  }
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
  s.es = a->interleaved ? 2 : 1;
}

static int run(const fdr_tti_args* a, cudaStream_t st) {
  int variant = a->variant;
  // the streaming kernels index levels with 32-bit element offsets (twice
  // the points for interleaved (p, r) levels)
  const uint64_t elems = (uint64_t)a->nx * (uint64_t)a->pitch_x * (a->interleaved ? 2u : 1u);
  if (variant == FDR_VARIANT_AUTO)
    variant = (a->order <= 8 && elems < (1ull << 32)) ? FDR_VARIANT_QUEUE : FDR_VARIANT_DIRECT;
  if ((variant == FDR_VARIANT_QUEUE || variant == FDR_VARIANT_TMA) && a->n_steps > 0) {
    int rc = tti_stream_prepare(a);
    if (rc != FDR_OK) return rc;
  }
  int chunk = 0;
  for (int k = 0; k < a->n_steps; ++k) {
    TTIStep s;
    fill(s, a, k);
    if (variant == FDR_VARIANT_QUEUE || variant == FDR_VARIANT_TMA) {
      // QUEUE: tti_pack (fields packed in f32x2 lanes); TMA: tti_stream
      int rc = tti_stream_launch(s, a, k, st, &chunk, variant == FDR_VARIANT_QUEUE);
      if (rc != FDR_OK) return rc;
    } else {
      dim3 block(64, 4, 1), grid((a->nz + 63) / 64, (a->ny + 3) / 4, a->nx);
      tti_direct<<<grid, block, 0, st>>>(s);
      TTI_CUDA(cudaGetLastError());
    }
  }
  const int last = a->it0 + a->n_steps - 1;
  if (a->n_steps > 0 && a->n_rec > 0 && a->traces && last < a->trace_rows) {
    tti_gather_kernel<<<(a->n_rec + 255) / 256, 256, 0, st>>>(
        a->p[(2 + a->n_steps) % 3], a->rec_xyz, a->n_rec, a->traces, last, a->pitch_y, a->pitch_x,
        a->interleaved ? 2 : 1);
    TTI_CUDA(cudaGetLastError());
  }
  return (2 + a->n_steps) % 3;
}


// ========================================================= float64 path
// fdr_tti64_run: the direct kernel's per-point sequence (= oracle/tti_ref.c)
// with every value in IEEE double, on separate p and r levels.  The float64
// reference the float32 path's error is reported against (SURVEY.md §8(f)3
// for TTI; precision_bytes = 8, equations.py:74-78).
struct TTIStep64 {
  const double *p, *pp, *r, *rp;
  double *pn, *rn;
  const double* prm[9];
  int nx, ny, nz, pitch_y;
  long long pitch_x;
  int radius;
  double w2[FDR_MAX_RADIUS + 1];
  double w1[FDR_MAX_RADIUS + 1];
  const double *gx, *gy, *gz, *series;
  int n_series, it, sx, sy, sz;
  const int* rec;
  int n_rec;
  double* traces;
  int gather_row;
};

__device__ __forceinline__ double at64(const double* u, const TTIStep64& a, int x, int y, int z) {
  if (x < 0 || x >= a.nx || y < 0 || y >= a.ny || z < 0 || z >= a.nz) return 0.0;
  return u[(size_t)x * a.pitch_x + (size_t)y * a.pitch_y + z];
}
__device__ double d1_64(const double* u, const TTIStep64& a, int x, int y, int z, int ax) {
  const int dx = ax == 0, dy = ax == 1, dz = ax == 2;
  double d = __dmul_rn(a.w1[1], __dsub_rn(at64(u, a, x + dx, y + dy, z + dz), at64(u, a, x - dx, y - dy, z - dz)));
  for (int j = 2; j <= a.radius; ++j)
    d = __fma_rn(a.w1[j], __dsub_rn(at64(u, a, x + j * dx, y + j * dy, z + j * dz),
                                    at64(u, a, x - j * dx, y - j * dy, z - j * dz)), d);
  return d;
}
__device__ double d2_64(const double* u, const TTIStep64& a, int x, int y, int z, int ax) {
  const int dx = ax == 0, dy = ax == 1, dz = ax == 2;
  double d = __dmul_rn(a.w2[0], at64(u, a, x, y, z));
  for (int j = 1; j <= a.radius; ++j)
    d = __fma_rn(a.w2[j], __dadd_rn(at64(u, a, x + j * dx, y + j * dy, z + j * dz),
                                    at64(u, a, x - j * dx, y - j * dy, z - j * dz)), d);
  return d;
}
__device__ double d11_64(const double* u, const TTIStep64& a, int x, int y, int z, int ao, int ai) {
  const int dx = ao == 0, dy = ao == 1, dz = ao == 2;
  double d = __dmul_rn(a.w1[1], __dsub_rn(d1_64(u, a, x + dx, y + dy, z + dz, ai),
                                          d1_64(u, a, x - dx, y - dy, z - dz, ai)));
  for (int j = 2; j <= a.radius; ++j)
    d = __fma_rn(a.w1[j], __dsub_rn(d1_64(u, a, x + j * dx, y + j * dy, z + j * dz, ai),
                                    d1_64(u, a, x - j * dx, y - j * dy, z - j * dz, ai)), d);
  return d;
}
__device__ void gl_op64(const double* u, const TTIStep64& a, int x, int y, int z, const double* c,
                        double* G, double* L) {
  const double dxx = d2_64(u, a, x, y, z, 0), dyy = d2_64(u, a, x, y, z, 1), dzz = d2_64(u, a, x, y, z, 2);
  const double dxy = d11_64(u, a, x, y, z, 0, 1), dxz = d11_64(u, a, x, y, z, 0, 2);
  const double dyz = d11_64(u, a, x, y, z, 1, 2);
  const double gin = __fma_rn(c[4], dyz, __fma_rn(c[2], dzz, __dmul_rn(c[1], dyy)));
  const double lin = __dadd_rn(dyy, dzz);
  *G = __fma_rn(c[5], dxz, __fma_rn(c[3], dxy, __fma_rn(c[0], dxx, gin)));
  *L = __dadd_rn(lin, dxx);
}

__global__ void __launch_bounds__(256) tti_direct64(const TTIStep64 a) {
  if (a.gather_row >= 0) {  // the previous step's p (cur here, read-only) at the receivers
    const int nthr = blockDim.x * blockDim.y;
    const int b = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    const int t = threadIdx.x + blockDim.x * threadIdx.y;
    for (int i = b * nthr + t; i < a.n_rec; i += nthr * (int)(gridDim.x * gridDim.y * gridDim.z)) {
      const int* c = a.rec + 3 * i;
      a.traces[(size_t)a.gather_row * a.n_rec + i] =
          a.p[(size_t)c[0] * a.pitch_x + (size_t)c[1] * a.pitch_y + c[2]];
    }
  }
  const int z = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  const int x = blockIdx.z;
  if (z >= a.nz || y >= a.ny) return;
  const size_t o = (size_t)x * a.pitch_x + (size_t)y * a.pitch_y + z;
  const double k = a.prm[0][o], pa = a.prm[1][o], pb = a.prm[2][o];
  const double c[6] = {a.prm[3][o], a.prm[4][o], a.prm[5][o], a.prm[6][o], a.prm[7][o], a.prm[8][o]};
  double Gp, Lp, Gr, Lr;
  gl_op64(a.p, a, x, y, z, c, &Gp, &Lp);
  gl_op64(a.r, a, x, y, z, c, &Gr, &Lr);
  const double Hp = __dsub_rn(Lp, Gp);
  double pn = __fma_rn(k, __fma_rn(pa, Hp, __dmul_rn(pb, Gr)), __fma_rn(2.0, a.p[o], -a.pp[o]));
  double rn = __fma_rn(k, __fma_rn(pb, Hp, Gr), __fma_rn(2.0, a.r[o], -a.rp[o]));
  if (a.gx) {
    const double g = __dmul_rn(__dmul_rn(a.gx[x], a.gy[y]), a.gz[z]);
    pn = __dmul_rn(pn, g);
    rn = __dmul_rn(rn, g);
  }
  if (x == a.sx && y == a.sy && z == a.sz && a.it < a.n_series) {
    pn = __dadd_rn(pn, a.series[a.it]);
    rn = __dadd_rn(rn, a.series[a.it]);
  }
  a.pn[o] = pn;
  a.rn[o] = rn;
}

__global__ void tti_gather64(const double* p, const int* rec, int n_rec, double* traces, int row,
                             int pitch_y, long long pitch_x) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_rec) {
    const int* c = rec + 3 * i;
    traces[(size_t)row * n_rec + i] = p[(size_t)c[0] * pitch_x + (size_t)c[1] * pitch_y + c[2]];
  }
}

static int validate64(const fdr_tti64_args* a) {
  if (!a) return fail(FDR_EINVAL, "args is NULL");
  if (a->abi_version != FDR_ABI_VERSION)
    return fail(FDR_EINVAL, "abi_version %d != library %d", a->abi_version, FDR_ABI_VERSION);
  if (a->order < 2 || a->order % 2 || a->order > 16)
    return fail(FDR_EINVAL, "TTI order must be even and within [2, 16], got %d", a->order);
  const int r = a->order / 2;
  if (a->nx < 2 * r + 1 || a->ny < 2 * r + 1 || a->nz < 2 * r + 1)
    return fail(FDR_EINVAL, "interior dims (%d, %d, %d) too small for halo width %d", a->nx,
                a->ny, a->nz, r);
  if (a->pitch_y < a->nz || a->pitch_x < (int64_t)a->ny * a->pitch_y)
    return fail(FDR_EINVAL, "bad pitches");
  if (a->n_steps < 0 || a->it0 < 0) return fail(FDR_EINVAL, "n_steps and it0 must be >= 0");
  for (int i = 0; i < 3; ++i)
    if (!a->p[i] || !a->r[i]) return fail(FDR_EINVAL, "level pointer NULL");
  for (int i = 0; i < 9; ++i)
    if (!a->params[i]) return fail(FDR_EINVAL, "parameter grid %d is NULL", i);
  if (a->sponge_x && (!a->sponge_y || !a->sponge_z))
    return fail(FDR_EINVAL, "sponge needs all three profiles");
  if (a->src_x >= 0 && (a->src_x >= a->nx || a->src_y < 0 || a->src_y >= a->ny ||
                        a->src_z < 0 || a->src_z >= a->nz))
    return fail(FDR_EINVAL, "source location outside interior");
  if (a->n_rec > 0 && (!a->rec_xyz || !a->traces))
    return fail(FDR_EINVAL, "receiver coordinates or trace buffer NULL");
  return FDR_OK;
}

static int run64(const fdr_tti64_args* a, cudaStream_t st) {
  for (int k = 0; k < a->n_steps; ++k) {
    TTIStep64 s;
    memset(&s, 0, sizeof(s));
    s.pn = a->p[k % 3];
    s.pp = a->p[(1 + k) % 3];
    s.p = a->p[(2 + k) % 3];
    s.rn = a->r[k % 3];
    s.rp = a->r[(1 + k) % 3];
    s.r = a->r[(2 + k) % 3];
    for (int i = 0; i < 9; ++i) s.prm[i] = a->params[i];
    s.nx = a->nx;
    s.ny = a->ny;
    s.nz = a->nz;
    s.pitch_y = a->pitch_y;
    s.pitch_x = a->pitch_x;
    s.radius = a->order / 2;
    for (int j = 0; j <= FDR_MAX_RADIUS; ++j) {
      s.w2[j] = a->w2[j];
      s.w1[j] = a->w1[j];
    }
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
    dim3 block(64, 4, 1), grid((a->nz + 63) / 64, (a->ny + 3) / 4, a->nx);
    tti_direct64<<<grid, block, 0, st>>>(s);
    TTI_CUDA(cudaGetLastError());
  }
  const int last = a->it0 + a->n_steps - 1;
  if (a->n_steps > 0 && a->n_rec > 0 && a->traces && last < a->trace_rows) {
    tti_gather64<<<(a->n_rec + 255) / 256, 256, 0, st>>>(a->p[(2 + a->n_steps) % 3], a->rec_xyz,
                                                        a->n_rec, a->traces, last, a->pitch_y,
                                                        a->pitch_x);
    TTI_CUDA(cudaGetLastError());
  }
  return (2 + a->n_steps) % 3;
}

}  // namespace fdr_tti

extern "C" {

size_t fdr_tti_args_size(void) { return sizeof(fdr_tti_args); }

int fdr_tti_run(const fdr_tti_args* args, void* stream) {
  int rc = fdr_tti::validate(args);
  if (rc != FDR_OK) return rc;
  return fdr_tti::run(args, static_cast<cudaStream_t>(stream));
}

size_t fdr_tti64_args_size(void) { return sizeof(fdr_tti64_args); }

int fdr_tti64_run(const fdr_tti64_args* args, void* stream) {
  int rc = fdr_tti::validate64(args);
  if (rc != FDR_OK) return rc;
  return fdr_tti::run64(args, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
