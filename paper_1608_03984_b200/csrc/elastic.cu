// Isotropic elastic velocity-stress kernels for B200 (sm_100a) + C ABI.
//
// BASELINE config 5.  The reference has no velocity-stress kernel (its
// elastic catalogue is displacement-form anisotropic, equations.py:156-177);
// the float32 sequence is defined by the parity oracle oracle/elastic_ref.c
// and reproduced here bit for bit (staggered Virieux grid, one velocity pass
// and one stress pass per step, fields updated in place):
//   F(f)[i] = c1 (f[i+1]-f[i]) + sum_{k>=2} fma(c_k, f[i+k]-f[i+1-k])
//   B(f)[i] = c1 (f[i]-f[i-1]) + sum_{k>=2} fma(c_k, f[i+k-1]-f[i-k])
//   vx = fma(bs, (By sxy + Bz sxz) + Fx sxx, vx)   (vy, vz likewise)
//   sxx = fma(lam, ey + ez, fma(l2m, ex, sxx)), l2m = fma(2, mu, lam)
//   sxy = fma(mu, Fy vx + Fx vy, sxy)              (sxz, syz likewise)
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/b200fd.h"
#include "fdr_common.cuh"

namespace fdr_el {

using namespace fdr;

enum { VX, VY, VZ, SXX, SYY, SZZ, SXY, SXZ, SYZ };

struct ElStep {
  float* f[9];
  const float* bs;
  const float* lam;
  const float* mu;
  int nx, ny, nz, pitch_y;
  long long pitch_x;
  int radius;
  float c[FDR_MAX_RADIUS + 1];
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
  int chunk;
  // x range of this launch (the whole grid except in the windowed schedule,
  // el_window_step) and whether the velocity stores stay in L2 (plain stores
  // instead of streaming ones) for the stress launch that follows closely
  int x0, x1;
  int keep_v;
};

__device__ __forceinline__ float at(const float* u, const ElStep& a, int x, int y, int z) {
  if (x < 0 || x >= a.nx || y < 0 || y >= a.ny || z < 0 || z >= a.nz) return 0.0f;
  return u[(size_t)x * a.pitch_x + (size_t)y * a.pitch_y + z];
}

// forward / backward staggered differences along axis ax at (x, y, z)
__device__ float dF(const float* u, const ElStep& a, int x, int y, int z, int ax) {
  const int dx = ax == 0, dy = ax == 1, dz = ax == 2;
  float d = __fmul_rn(a.c[1], __fsub_rn(at(u, a, x + dx, y + dy, z + dz), at(u, a, x, y, z)));
  for (int k = 2; k <= a.radius; ++k)
    d = __fmaf_rn(a.c[k], __fsub_rn(at(u, a, x + k * dx, y + k * dy, z + k * dz),
                                    at(u, a, x + (1 - k) * dx, y + (1 - k) * dy, z + (1 - k) * dz)), d);
  return d;
}

__device__ float dB(const float* u, const ElStep& a, int x, int y, int z, int ax) {
  const int dx = ax == 0, dy = ax == 1, dz = ax == 2;
  float d = __fmul_rn(a.c[1], __fsub_rn(at(u, a, x, y, z), at(u, a, x - dx, y - dy, z - dz)));
  for (int k = 2; k <= a.radius; ++k)
    d = __fmaf_rn(a.c[k], __fsub_rn(at(u, a, x + (k - 1) * dx, y + (k - 1) * dy, z + (k - 1) * dz),
                                    at(u, a, x - k * dx, y - k * dy, z - k * dz)), d);
  return d;
}

__device__ void gather_vz(const ElStep& a) {
  if (a.gather_row < 0) return;
  const int nthr = blockDim.x * blockDim.y * blockDim.z;
  const int b = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  const int t = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
  const int stride = nthr * (int)(gridDim.x * gridDim.y * gridDim.z);
  for (int i = b * nthr + t; i < a.n_rec; i += stride) {
    const int* q = a.rec + 3 * i;
    if (q[0] < a.x0 || q[0] >= a.x1) continue;  // another window's launch samples it
    a.traces[(size_t)a.gather_row * a.n_rec + i] =
        a.f[VZ][(size_t)q[0] * a.pitch_x + (size_t)q[1] * a.pitch_y + q[2]];
  }
}

__device__ __forceinline__ float taper(const ElStep& a, int x, int y, int z) {
  return __fmul_rn(__fmul_rn(a.gx[x], a.gy[y]), a.gz[z]);
}

// velocity pass, one thread per point (checker variant)
__global__ void __launch_bounds__(256) el_vel_direct(const ElStep a) {
  const int z = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  const int x = blockIdx.z;
  if (z >= a.nz || y >= a.ny) return;
  const size_t o = (size_t)x * a.pitch_x + (size_t)y * a.pitch_y + z;
  const float b = a.bs[o];
  const float ax = __fadd_rn(__fadd_rn(dB(a.f[SXY], a, x, y, z, 1), dB(a.f[SXZ], a, x, y, z, 2)),
                             dF(a.f[SXX], a, x, y, z, 0));
  const float ay = __fadd_rn(__fadd_rn(dF(a.f[SYY], a, x, y, z, 1), dB(a.f[SYZ], a, x, y, z, 2)),
                             dB(a.f[SXY], a, x, y, z, 0));
  const float az = __fadd_rn(__fadd_rn(dB(a.f[SYZ], a, x, y, z, 1), dF(a.f[SZZ], a, x, y, z, 2)),
                             dB(a.f[SXZ], a, x, y, z, 0));
  float vx = __fmaf_rn(b, ax, a.f[VX][o]), vy = __fmaf_rn(b, ay, a.f[VY][o]);
  float vz = __fmaf_rn(b, az, a.f[VZ][o]);
  if (a.gx) {
    const float g = taper(a, x, y, z);
    vx = __fmul_rn(vx, g);
    vy = __fmul_rn(vy, g);
    vz = __fmul_rn(vz, g);
  }
  a.f[VX][o] = vx;
  a.f[VY][o] = vy;
  a.f[VZ][o] = vz;
}

// stress pass, one thread per point (checker variant)
__global__ void __launch_bounds__(256) el_str_direct(const ElStep a) {
  gather_vz(a);  // vz is final for this step and not written by the stress pass
  const int z = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  const int x = blockIdx.z;
  if (z >= a.nz || y >= a.ny) return;
  const size_t o = (size_t)x * a.pitch_x + (size_t)y * a.pitch_y + z;
  const float lam = a.lam[o], mu = a.mu[o];
  const float l2m = __fmaf_rn(2.0f, mu, lam);
  const float ex = dB(a.f[VX], a, x, y, z, 0), ey = dB(a.f[VY], a, x, y, z, 1);
  const float ez = dB(a.f[VZ], a, x, y, z, 2);
  float s[6];
  s[0] = __fmaf_rn(lam, __fadd_rn(ey, ez), __fmaf_rn(l2m, ex, a.f[SXX][o]));
  s[1] = __fmaf_rn(lam, __fadd_rn(ez, ex), __fmaf_rn(l2m, ey, a.f[SYY][o]));
  s[2] = __fmaf_rn(lam, __fadd_rn(ey, ex), __fmaf_rn(l2m, ez, a.f[SZZ][o]));
  s[3] = __fmaf_rn(mu, __fadd_rn(dF(a.f[VX], a, x, y, z, 1), dF(a.f[VY], a, x, y, z, 0)), a.f[SXY][o]);
  s[4] = __fmaf_rn(mu, __fadd_rn(dF(a.f[VX], a, x, y, z, 2), dF(a.f[VZ], a, x, y, z, 0)), a.f[SXZ][o]);
  s[5] = __fmaf_rn(mu, __fadd_rn(dF(a.f[VY], a, x, y, z, 2), dF(a.f[VZ], a, x, y, z, 1)), a.f[SYZ][o]);
  if (a.gx) {
    const float g = taper(a, x, y, z);
#pragma unroll
    for (int i = 0; i < 6; ++i) s[i] = __fmul_rn(s[i], g);
  }
  if (x == a.sx && y == a.sy && z == a.sz && a.it < a.n_series) {
    const float q = a.series[a.it];
    s[0] = __fadd_rn(s[0], q);
    s[1] = __fadd_rn(s[1], q);
    s[2] = __fadd_rn(s[2], q);
  }
#pragma unroll
  for (int i = 0; i < 6; ++i) a.f[SXX + i][o] = s[i];
}

#define EL_CUDA(call)                                        \
  do {                                                       \
    cudaError_t e_ = (call);                                 \
    if (e_ != cudaSuccess) return fdr::cuda_fail(e_, #call); \
  } while (0)

int el_stream_step(const ElStep& s, const fdr_elastic_args* a, cudaStream_t st, int* chunk_cache);
// Per-run state of the queue path: the x-chunk choice and, for the fused
// schedule, the ticket/flag buffer (stream-ordered allocation) and step count.
struct ElRunState {
  int chunk = 0;
  unsigned* fuse_buf = nullptr;
  int fuse_step = 0;
};
int el_queue_step(const ElStep& s, const fdr_elastic_args* a, cudaStream_t st, ElRunState* rs);
void el_queue_refresh_knobs();

static int validate(const fdr_elastic_args* a) {
  if (!a) return fail(FDR_EINVAL, "args is NULL");
  if (a->abi_version != FDR_ABI_VERSION)
    return fail(FDR_EINVAL, "abi_version %d != library %d", a->abi_version, FDR_ABI_VERSION);
  if (a->order < 2 || a->order % 2 || a->order > 16)
    return fail(FDR_EINVAL, "elastic order must be even and within [2, 16], got %d", a->order);
  const int r = a->order / 2;
  if (a->nx < 2 * r + 1 || a->ny < 2 * r + 1 || a->nz < 2 * r + 1)
    return fail(FDR_EINVAL, "interior dims (%d, %d, %d) too small for halo width %d", a->nx,
                a->ny, a->nz, r);
  if (a->pitch_y < a->nz || a->pitch_y % 4 || a->pitch_x < (int64_t)a->ny * a->pitch_y ||
      a->pitch_x % 4)
    return fail(FDR_EINVAL, "bad pitches");
  if (a->n_steps < 0 || a->it0 < 0) return fail(FDR_EINVAL, "n_steps and it0 must be >= 0");
  for (int i = 0; i < 9; ++i)
    if (!a->fields[i]) return fail(FDR_EINVAL, "field %d is NULL", i);
  for (int i = 0; i < 3; ++i)
    if (!a->params[i]) return fail(FDR_EINVAL, "parameter grid %d is NULL", i);
  if (a->sponge_x && (!a->sponge_y || !a->sponge_z))
    return fail(FDR_EINVAL, "sponge needs all three profiles");
  if (a->src_x >= 0 && (a->src_x >= a->nx || a->src_y < 0 || a->src_y >= a->ny ||
                        a->src_z < 0 || a->src_z >= a->nz))
    return fail(FDR_EINVAL, "source location outside interior");
  if (a->n_rec > 0 && (!a->rec_xyz || !a->traces))
    return fail(FDR_EINVAL, "receiver coordinates or trace buffer NULL");
  if (a->variant < 0 || a->variant > FDR_VARIANT_QUEUE)
    return fail(FDR_EINVAL, "unknown elastic variant %d", a->variant);
  return FDR_OK;
}

static void fill(ElStep& s, const fdr_elastic_args* a, int k) {
  memset(&s, 0, sizeof(s));
  for (int i = 0; i < 9; ++i) s.f[i] = a->fields[i];
  s.bs = a->params[0];
  s.lam = a->params[1];
  s.mu = a->params[2];
  s.nx = a->nx;
  s.ny = a->ny;
  s.nz = a->nz;
  s.pitch_y = a->pitch_y;
  s.pitch_x = a->pitch_x;
  s.radius = a->order / 2;
  for (int j = 0; j <= FDR_MAX_RADIUS; ++j) s.c[j] = a->c[j];
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
  // receivers sample vz at the start of the stress pass (vz is final for
  // step `it` there and the stress pass does not write it)
  s.gather_row = (a->n_rec > 0 && a->traces && s.it < a->trace_rows) ? s.it : -1;
  s.x0 = 0;
  s.x1 = a->nx;
}

static int run(const fdr_elastic_args* a, cudaStream_t st) {
  int variant = a->variant;
  const bool small_index = (uint64_t)a->nx * (uint64_t)a->pitch_x < (1ull << 32);
  if (variant == FDR_VARIANT_AUTO)
    variant = (a->order <= 8 && small_index) ? FDR_VARIANT_QUEUE : FDR_VARIANT_DIRECT;
  if ((variant == FDR_VARIANT_QUEUE || variant == FDR_VARIANT_TMA) && (!small_index || a->order > 8))
    return fail(FDR_EINVAL, "the elastic streaming kernels need order <= 8 and < 2^32 elements");
  ElRunState rs;
  int& chunk = rs.chunk;
  if (variant == FDR_VARIANT_QUEUE) el_queue_refresh_knobs();
  struct FreeFuse {  // the fused schedule's buffer goes back in stream order
    ElRunState& r;
    cudaStream_t st;
    ~FreeFuse() {
      if (r.fuse_buf) cudaFreeAsync(r.fuse_buf, st);
    }
  } free_fuse{rs, st};
  for (int k = 0; k < a->n_steps; ++k) {
    ElStep s;
    fill(s, a, k);
    if (variant == FDR_VARIANT_QUEUE) {  // el_queue (production)
      int rc = el_queue_step(s, a, st, &rs);
      if (rc != FDR_OK) return rc;
    } else if (variant == FDR_VARIANT_TMA) {  // el_stream (previous design)
      int rc = el_stream_step(s, a, st, &chunk);
      if (rc != FDR_OK) return rc;
    } else {
      dim3 block(64, 4, 1), grid((a->nz + 63) / 64, (a->ny + 3) / 4, a->nx);
      el_vel_direct<<<grid, block, 0, st>>>(s);
      EL_CUDA(cudaGetLastError());
      el_str_direct<<<grid, block, 0, st>>>(s);
      EL_CUDA(cudaGetLastError());
    }
  }
  return FDR_OK;
}

// ============================================================ stream kernels
// 2.5D streaming velocity and stress passes.  A CTA of 512 threads owns a
// 32(z) x 16(y) column tile (one point per thread) and streams it along x.
// Stream plane p (x_n = xb - R + p) arrives by TMA in one ring stage with the
// boxes (y/z halo) of the fields whose y/z derivatives the pass needs, and the
// halo-free tiles of the plane computed at this iteration (x_c = x_n - R):
// the fields it updates in place and its parameters.  In-plane derivative
// sums are formed on arrival and delayed R planes in registers; the x
// derivatives read register windows of own-column values.  Stages are
// recycled by the last warp to release them (empty mbarrier).
#ifndef FDR_EL_TY
#define FDR_EL_TY 8
#endif
constexpr int ETZ = 32, ETY = FDR_EL_TY, ENT = ETZ * ETY;
constexpr int EMINB = ETY <= 8 ? 2 : 1;  // CTAs per SM the tile is sized for

template <int R, int NBOX, int NTILE>
struct EGeo {
  static constexpr int LZ = (R + 3) / 4 * 4;
  static constexpr int BZ = ETZ + 2 * LZ;
  static constexpr int BY = ETY + 2 * R;
  static constexpr int BOX_BYTES = BZ * BY * 4;
  static constexpr int BOX = (BOX_BYTES + 127) / 128 * 32;
  static constexpr int TILE = ETY * ETZ;
  static constexpr int O_TILE = NBOX * BOX;
  static constexpr int STAGE = O_TILE + NTILE * TILE;
  static constexpr int NS = 4;
  static constexpr int U = R <= 2 ? 2 * R + 1 : 3;
  static constexpr int QW = 2 * R + U;
  static constexpr int GW = R + U;
  static constexpr int NWARPS = ENT / 32;
  static constexpr size_t SMEM = size_t(NS) * STAGE * 4 + 2 * NS * 8;
};

struct ElMaps {
  CUtensorMap box[5];   // velocity pass: sxy sxz syy syz szz; stress pass: vx vy vz
  CUtensorMap tile[9];  // velocity pass: sxx vx vy vz bs; stress: sxx..syz lam mu
};

FDR_DEV bool el_arrive_last_a(uint32_t bar) {
  uint64_t state;
  uint32_t pending;
  asm volatile("mbarrier.arrive.shared::cta.b64 %0, [%1];" : "=l"(state) : "r"(bar) : "memory");
  asm volatile("mbarrier.pending_count.b64 %0, %1;" : "=r"(pending) : "l"(state));
  return pending == 1;
}
FDR_DEV bool el_arrive_last(uint64_t* bar) { return el_arrive_last_a(smem_u32(bar)); }

// staggered differences on a strided line (p points at the own element)
template <int R>
FDR_DEV float sF(const float* p, int s, const float* c) {
  float d = __fmul_rn(c[1], __fsub_rn(p[s], p[0]));
#pragma unroll
  for (int k = 2; k <= R; ++k) d = __fmaf_rn(c[k], __fsub_rn(p[k * s], p[(1 - k) * s]), d);
  return d;
}
template <int R>
FDR_DEV float sB(const float* p, int s, const float* c) {
  float d = __fmul_rn(c[1], __fsub_rn(p[0], p[-s]));
#pragma unroll
  for (int k = 2; k <= R; ++k) d = __fmaf_rn(c[k], __fsub_rn(p[(k - 1) * s], p[-k * s]), d);
  return d;
}
// the same on a register window w (centre index c)
template <int R>
FDR_DEV float wF(const float* w, int c, const float* cc) {
  float d = __fmul_rn(cc[1], __fsub_rn(w[c + 1], w[c]));
#pragma unroll
  for (int k = 2; k <= R; ++k) d = __fmaf_rn(cc[k], __fsub_rn(w[c + k], w[c + 1 - k]), d);
  return d;
}
template <int R>
FDR_DEV float wB(const float* w, int c, const float* cc) {
  float d = __fmul_rn(cc[1], __fsub_rn(w[c], w[c - 1]));
#pragma unroll
  for (int k = 2; k <= R; ++k) d = __fmaf_rn(cc[k], __fsub_rn(w[c + k - 1], w[c - k]), d);
  return d;
}

// PASS 0: velocity (boxes sxy sxz syy syz szz; tiles sxx [newest], vx vy vz bs [centre])
// PASS 1: stress   (boxes vx vy vz;            tiles sxx syy szz sxy sxz syz lam mu [centre])
template <int R, int PASS, bool SPONGE>
__global__ void __launch_bounds__(ENT, EMINB) el_stream(const __grid_constant__ ElMaps maps,
                                                    const ElStep a) {
  constexpr int NBOX = PASS == 0 ? 5 : 3;
  constexpr int NTILE = PASS == 0 ? 5 : 8;
  using G = EGeo<R, NBOX, NTILE>;
  extern __shared__ __align__(128) float smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + G::NS * G::STAGE);
  uint64_t* empty = full + G::NS;

  if (PASS == 1) gather_vz(a);
  const int tid = threadIdx.x;
  const int tz = tid % ETZ, ty = tid / ETZ;
  const int zt = blockIdx.x * ETZ, yt = blockIdx.y * ETY;
  const int xb = blockIdx.z * a.chunk;
  const int xe = min(a.nx, xb + a.chunk);
  if (xb >= xe) return;
  const int n = xe - xb;
  const int nplanes = n + 2 * R;
  const bool leader = (tid & 31) == 0;

  auto issue = [&](int pl, int s) {
    float* st = smem + s * G::STAGE;
    const int xn = xb - R + pl;
    const bool cen = pl >= 2 * R;
    const int ncen = PASS == 0 ? 4 : 8;  // centre tiles
    const uint32_t bytes = NBOX * G::BOX_BYTES + (PASS == 0 ? G::TILE * 4 : 0) +
                           (cen ? ncen * G::TILE * 4 : 0);
    mbar_arrive_expect_tx(&full[s], bytes);
#pragma unroll
    for (int b = 0; b < NBOX; ++b)
      tma_load_3d(st + b * G::BOX, &maps.box[b], &full[s], zt - G::LZ, yt - R, xn);
    if (PASS == 0) tma_load_3d(st + G::O_TILE, &maps.tile[0], &full[s], zt, yt, xn);
    if (cen) {
      const int t0 = PASS == 0 ? 1 : 0;
#pragma unroll
      for (int t = 0; t < (PASS == 0 ? 4 : 8); ++t)
        tma_load_3d(st + G::O_TILE + (t0 + t) * G::TILE, &maps.tile[t0 + t], &full[s], zt, yt,
                    xn - R);
    }
  };
  if (tid == 0) {
    for (int b = 0; b < NBOX; ++b) prefetch_tensormap(&maps.box[b]);
    for (int s = 0; s < G::NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], G::NWARPS);
    }
    fence_barrier_init();
    for (int pl = 0; pl < G::NS && pl < nplanes; ++pl) issue(pl, pl);
  }
  __syncthreads();

  const int y = yt + ty, z = zt + tz;
  const bool ok = y < a.ny && z < a.nz;
  const int bown = (ty + R) * G::BZ + G::LZ + tz;
  const int town = ty * ETZ + tz;
  float gyz = 1.0f, gy = 1.0f, gz = 1.0f;
  if (SPONGE && ok) {
    gy = a.gy[y];
    gz = a.gz[z];
  }
  (void)gyz;
  const bool src_here = PASS == 1 && a.sx >= 0 && y == a.sy && z == a.sz && a.it < a.n_series;
  const float qsrc = src_here ? a.series[a.it] : 0.0f;
  const int kinj = src_here ? a.sx - xb : -1;
  const uint32_t px32 = (uint32_t)a.pitch_x;
  const uint32_t oidx0 = (uint32_t)xb * px32 + (uint32_t)y * (uint32_t)a.pitch_y + (uint32_t)z;

  // x windows (index i <-> stream plane p0 - 2R + i) and delayed in-plane
  // values (index i <-> stream plane p0 - R + i)
  float w0[G::QW], w1[G::QW], w2[G::QW];
  constexpr int ND = PASS == 0 ? 3 : 5;
  float dly[ND][G::GW];
#pragma unroll
  for (int i = 0; i < G::QW; ++i) w0[i] = w1[i] = w2[i] = 0.0f;
#pragma unroll
  for (int d = 0; d < ND; ++d)
#pragma unroll
    for (int i = 0; i < G::GW; ++i) dly[d][i] = 0.0f;

  int slot = 0;
  uint32_t phase = 0;
#pragma unroll 1
  for (int p0 = 0; p0 < nplanes; p0 += G::U) {
#pragma unroll
    for (int u = 0; u < G::U; ++u) {
      const int pl = p0 + u;
      if (pl >= nplanes) break;
      mbar_wait(&full[slot], phase);
      const float* st = smem + slot * G::STAGE;
      const int qn = 2 * R + u, gn = R + u;
      if (PASS == 0) {
        const float* sxy = st + 0 * G::BOX + bown;
        const float* sxz = st + 1 * G::BOX + bown;
        const float* syy = st + 2 * G::BOX + bown;
        const float* syz = st + 3 * G::BOX + bown;
        const float* szz = st + 4 * G::BOX + bown;
        w0[qn] = st[G::O_TILE + town];  // sxx
        w1[qn] = sxy[0];
        w2[qn] = sxz[0];
        dly[0][gn] = __fadd_rn(sB<R>(sxy, G::BZ, a.c), sB<R>(sxz, 1, a.c));
        dly[1][gn] = __fadd_rn(sF<R>(syy, G::BZ, a.c), sB<R>(syz, 1, a.c));
        dly[2][gn] = __fadd_rn(sB<R>(syz, G::BZ, a.c), sF<R>(szz, 1, a.c));
      } else {
        const float* vx = st + 0 * G::BOX + bown;
        const float* vy = st + 1 * G::BOX + bown;
        const float* vz = st + 2 * G::BOX + bown;
        w0[qn] = vx[0];
        w1[qn] = vy[0];
        w2[qn] = vz[0];
        dly[0][gn] = sB<R>(vy, G::BZ, a.c);                            // ey
        dly[1][gn] = sB<R>(vz, 1, a.c);                                // ez
        dly[2][gn] = sF<R>(vx, G::BZ, a.c);                            // Fy vx
        dly[3][gn] = sF<R>(vx, 1, a.c);                                // Fz vx
        dly[4][gn] = __fadd_rn(sF<R>(vy, 1, a.c), sF<R>(vz, G::BZ, a.c));  // Fz vy + Fy vz
      }
      const int k = pl - 2 * R;
      float cen[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) cen[t] = 0.0f;
      if (k >= 0) {
        const float* ct = st + G::O_TILE + (PASS == 0 ? G::TILE : 0) + town;
#pragma unroll
        for (int t = 0; t < (PASS == 0 ? 4 : 8); ++t) cen[t] = ct[t * G::TILE];
      }
      __syncwarp();
      if (leader && el_arrive_last(&empty[slot])) {
        mbar_wait(&empty[slot], phase);
        fence_proxy_async();  // generic-proxy reads of the stage before the TMA refill (cross-proxy WAR)
        if (pl + G::NS < nplanes) issue(pl + G::NS, slot);
      }
      if (++slot == G::NS) {
        slot = 0;
        phase ^= 1u;
      }
      if (k >= 0) {
        const int c = u + R;
        const uint32_t o = oidx0 + (uint32_t)k * px32;
        const float g = SPONGE ? __fmul_rn(__fmul_rn(__ldg(a.gx + xb + k), gy), gz) : 1.0f;
        if (PASS == 0) {
          const float b = cen[3];
          float vx = __fmaf_rn(b, __fadd_rn(dly[0][u], wF<R>(w0, c, a.c)), cen[0]);
          float vy = __fmaf_rn(b, __fadd_rn(dly[1][u], wB<R>(w1, c, a.c)), cen[1]);
          float vz = __fmaf_rn(b, __fadd_rn(dly[2][u], wB<R>(w2, c, a.c)), cen[2]);
          if (SPONGE) {
            vx = __fmul_rn(vx, g);
            vy = __fmul_rn(vy, g);
            vz = __fmul_rn(vz, g);
          }
          if (ok) {
            a.f[VX][o] = vx;
            a.f[VY][o] = vy;
            a.f[VZ][o] = vz;
          }
        } else {
          const float lam = cen[6], mu = cen[7];
          const float l2m = __fmaf_rn(2.0f, mu, lam);
          const float ex = wB<R>(w0, c, a.c);
          const float ey = dly[0][u], ez = dly[1][u];
          float sv[6];
          sv[0] = __fmaf_rn(lam, __fadd_rn(ey, ez), __fmaf_rn(l2m, ex, cen[0]));
          sv[1] = __fmaf_rn(lam, __fadd_rn(ez, ex), __fmaf_rn(l2m, ey, cen[1]));
          sv[2] = __fmaf_rn(lam, __fadd_rn(ey, ex), __fmaf_rn(l2m, ez, cen[2]));
          sv[3] = __fmaf_rn(mu, __fadd_rn(dly[2][u], wF<R>(w1, c, a.c)), cen[3]);
          sv[4] = __fmaf_rn(mu, __fadd_rn(dly[3][u], wF<R>(w2, c, a.c)), cen[4]);
          sv[5] = __fmaf_rn(mu, dly[4][u], cen[5]);
          if (SPONGE) {
#pragma unroll
            for (int i = 0; i < 6; ++i) sv[i] = __fmul_rn(sv[i], g);
          }
          if (k == kinj) {
            sv[0] = __fadd_rn(sv[0], qsrc);
            sv[1] = __fadd_rn(sv[1], qsrc);
            sv[2] = __fadd_rn(sv[2], qsrc);
          }
          if (ok) {
#pragma unroll
            for (int i = 0; i < 6; ++i) a.f[SXX + i][o] = sv[i];
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 2 * R; ++i) {
      w0[i] = w0[i + G::U];
      w1[i] = w1[i + G::U];
      w2[i] = w2[i + G::U];
    }
#pragma unroll
    for (int d = 0; d < ND; ++d)
#pragma unroll
      for (int i = 0; i < R; ++i) dly[d][i] = dly[d][i + G::U];
  }
}

static int el_encode(CUtensorMap* map, const float* base, const fdr_elastic_args* a, int bz, int by) {
  typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                          const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                          CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                          CUtensorMapFloatOOBfill);
  const Enc enc = reinterpret_cast<Enc>(fdr::tensor_map_encoder());
  if (!enc) return fail(FDR_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)a->nz, (cuuint64_t)a->ny, (cuuint64_t)a->nx};
  cuuint64_t strides[2] = {(cuuint64_t)a->pitch_y * 4, (cuuint64_t)a->pitch_x * 4};
  cuuint32_t box[3] = {(cuuint32_t)bz, (cuuint32_t)by, 1}, es[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides,
                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(FDR_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return FDR_OK;
}

// ======================================================= queue kernels
// el_queue<R, PASS, SPONGE>: the acoustic_queue design for the two elastic
// passes.  256 threads own a 32(z) x 16(y) tile, one float2 (2 z points) each,
// and stream it along x.  Stage p (TMA, NS-1 planes ahead) holds
//   - the newest plane's tiles of the three fields differentiated along x
//     (velocity pass: sxx sxy sxz; stress pass: vx vy vz), appended to
//     per-thread register queues of 2r+U float2;
//   - the centre plane's (x = newest - r) boxes, each with only the halo its
//     in-plane derivatives need (y-only, z-only or both), and its tiles.
// All in-plane derivatives are formed from the centre boxes when the centre
// plane is computed, so nothing is carried across planes but the x queues.
// Same float32 sequence as el_stream / oracle/elastic_ref.c.
constexpr int QZ = 32, QY = 16, QNZ = QZ / 2, QN = QNZ * QY;

template <int R, int PASS>
struct QGeoE {
  // z halo in floats: the TMA box must start on a 16-byte boundary (a 2-float
  // halo, i.e. an 8-byte offset, faults with an illegal instruction)
  static constexpr int LZ = (R + 3) / 4 * 4;
  static constexpr int ZB = QZ + 2 * LZ, YB = QY + 2 * R;    // boxed extents
  static constexpr int TILE = QZ * QY;
  static constexpr int al(int f) { return (f + 31) / 32 * 32; }  // 128-byte aligned regions
  static constexpr int YBOX = al(QZ * YB), ZBOX = al(ZB * QY), FBOX = al(ZB * YB);
  static constexpr int NY = PASS == 0 ? 2 : 0, NZB = PASS == 0 ? 2 : 0, NF = PASS == 0 ? 1 : 3;
  static constexpr int NC = PASS == 0 ? 4 : 8;               // centre tiles
  static constexpr int O_WIN = 0;
  static constexpr int O_Y = 3 * TILE;
  static constexpr int O_Z = O_Y + NY * YBOX;
  static constexpr int O_F = O_Z + NZB * ZBOX;
  static constexpr int O_C = O_F + NF * FBOX;
  static constexpr int STAGE = O_C + NC * TILE;
#ifdef FDR_EL_NS
  static constexpr int NS = FDR_EL_NS;
#else
  static constexpr int NS = 3;
#endif
  static constexpr int QD = 2 * R + 1;
#ifdef FDR_ELQ_U
  static constexpr int U = FDR_ELQ_U;
#else
  static constexpr int U = R <= 2 ? QD : 2;
#endif
  static constexpr int NWARPS = QN / 32;
  static constexpr size_t SMEM = size_t(NS) * STAGE * 4 + 2 * NS * 8;
  static constexpr uint32_t WIN_BYTES = 3 * TILE * 4;
  static constexpr uint32_t CEN_BYTES = (NY * QZ * YB + NZB * ZB * QY + NF * ZB * YB + NC * TILE) * 4;
};

struct ElQMaps {
  CUtensorMap win[3];   // newest-plane tiles of the x-differentiated fields
  CUtensorMap ybox[2];  // velocity pass: sxy syy
  CUtensorMap zbox[2];  // velocity pass: sxz szz
  CUtensorMap fbox[3];  // velocity pass: syz; stress pass: vx vy vz
  CUtensorMap ctile[8]; // velocity: vx vy vz bs; stress: sxx syy szz sxy sxz syz lam mu
};

// Staggered differences for the two lanes (2 z points of one field) in
// packed f32x2: the oracle's per-lane sequence (mul, then fma chain; each bare
// product feeds only an fma operand, so nothing can be contracted).
FDR_DEV f2 f2of(float2 v) { return pk(v.x, v.y); }
FDR_DEV float2 f2to(f2 v) { return make_float2(lo(v), hi(v)); }
FDR_DEV f2 bcw(float c) { return pk(c, c); }
FDR_DEV f2 ldf2(const float* p) { return *reinterpret_cast<const f2*>(p); }
// A 32-bit shared-window address in float units of offset, so the strided
// helpers below run on addresses the queue kernel carries across planes
// (ptxas then cannot rematerialise them from the thread index every plane).
struct SAddr {
  uint32_t a;
};
FDR_DEV SAddr operator+(SAddr p, int off) { return {p.a + 4u * (uint32_t)off}; }
FDR_DEV SAddr operator-(SAddr p, int off) { return {p.a - 4u * (uint32_t)off}; }
FDR_DEV f2 ldf2(SAddr p) { return lds64a(p.a); }

// p points at the own pair, s = the element stride of the differenced axis
template <int R, class P>
FDR_DEV float2 pF2(P p, int s, const float* c) {
  f2 d = mul2(bcw(c[1]), sub2(ldf2(p + s), ldf2(p)));
#pragma unroll
  for (int k = 2; k <= R; ++k) d = fma2(bcw(c[k]), sub2(ldf2(p + k * s), ldf2(p + (1 - k) * s)), d);
  return f2to(d);
}
template <int R, class P>
FDR_DEV float2 pB2(P p, int s, const float* c) {
  f2 d = mul2(bcw(c[1]), sub2(ldf2(p), ldf2(p - s)));
#pragma unroll
  for (int k = 2; k <= R; ++k) d = fma2(bcw(c[k]), sub2(ldf2(p + (k - 1) * s), ldf2(p - k * s)), d);
  return f2to(d);
}
// along z within one row window w[] (w[LZ] = the own pair's first point); the
// odd-offset pairs are misaligned, so the lane differences are scalar
template <int R, int LZ>
FDR_DEV float2 zF2(const float* w, const float* c) {
  f2 d = mul2(bcw(c[1]), pk(__fsub_rn(w[LZ + 1], w[LZ]), __fsub_rn(w[LZ + 2], w[LZ + 1])));
#pragma unroll
  for (int k = 2; k <= R; ++k)
    d = fma2(bcw(c[k]), pk(__fsub_rn(w[LZ + k], w[LZ + 1 - k]), __fsub_rn(w[LZ + 1 + k], w[LZ + 2 - k])), d);
  return f2to(d);
}
template <int R, int LZ>
FDR_DEV float2 zB2(const float* w, const float* c) {
  f2 d = mul2(bcw(c[1]), pk(__fsub_rn(w[LZ], w[LZ - 1]), __fsub_rn(w[LZ + 1], w[LZ])));
#pragma unroll
  for (int k = 2; k <= R; ++k)
    d = fma2(bcw(c[k]), pk(__fsub_rn(w[LZ + k - 1], w[LZ - k]), __fsub_rn(w[LZ + k], w[LZ + 1 - k])), d);
  return f2to(d);
}
// along x from a register queue of float2 (centre index cidx)
template <int R, int QD, bool ROT>
FDR_DEV float2 xF2(const float2* q, int cidx, const float* c) {
  auto at = [&](int i) -> f2 { return f2of(q[ROT ? (i + QD) % QD : i]); };
  f2 d = mul2(bcw(c[1]), sub2(at(cidx + 1), at(cidx)));
#pragma unroll
  for (int k = 2; k <= R; ++k) d = fma2(bcw(c[k]), sub2(at(cidx + k), at(cidx + 1 - k)), d);
  return f2to(d);
}
template <int R, int QD, bool ROT>
FDR_DEV float2 xB2(const float2* q, int cidx, const float* c) {
  auto at = [&](int i) -> f2 { return f2of(q[ROT ? (i + QD) % QD : i]); };
  f2 d = mul2(bcw(c[1]), sub2(at(cidx), at(cidx - 1)));
#pragma unroll
  for (int k = 2; k <= R; ++k) d = fma2(bcw(c[k]), sub2(at(cidx + k - 1), at(cidx - k)), d);
  return f2to(d);
}
FDR_DEV float2 add2f(float2 a, float2 b) { return f2to(add2(f2of(a), f2of(b))); }
FDR_DEV float2 fma2f(float2 a, float2 b, float2 c) { return f2to(fma2(f2of(a), f2of(b), f2of(c))); }
FDR_DEV void stg2cs(float* p, float2 v) {
  asm volatile("st.global.cs.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v.x), "f"(v.y) : "memory");
}

#ifndef FDR_EL_CARRY_STRESS
#define FDR_EL_CARRY_STRESS 0
#endif
// One (tile, x range) of a pass: the whole work of an el_queue CTA, also the
// item of the fused persistent kernel (el_fused), which re-initialises the
// ring's mbarriers for every item (`reinit`).
template <int R, int PASS, bool SPONGE>
FDR_DEV void el_queue_body(const ElQMaps& maps, const ElStep& a, const int zt, const int yt,
                           const int xb, const int xe, float* smem, const bool reinit) {
  using G = QGeoE<R, PASS>;
  constexpr int LZ = G::LZ;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + G::NS * G::STAGE);
  uint64_t* empty = full + G::NS;
  const int tid = threadIdx.x;
  const int tz = tid % QNZ, ty = tid / QNZ;
  const int n = xe - xb;
  const int nplanes = n + 2 * R;

  auto issue = [&](int pl, int sl) {
    float* st = smem + sl * G::STAGE;
    const int xn = xb - R + pl;
    const bool cen = pl >= 2 * R;
    mbar_arrive_expect_tx(&full[sl], G::WIN_BYTES + (cen ? G::CEN_BYTES : 0));
#pragma unroll
    for (int f = 0; f < 3; ++f) tma_load_3d(st + G::O_WIN + f * G::TILE, &maps.win[f], &full[sl], zt, yt, xn);
    if (cen) {
      const int xc = xn - R;
#pragma unroll
      for (int b = 0; b < G::NY; ++b) tma_load_3d(st + G::O_Y + b * G::YBOX, &maps.ybox[b], &full[sl], zt, yt - R, xc);
#pragma unroll
      for (int b = 0; b < G::NZB; ++b) tma_load_3d(st + G::O_Z + b * G::ZBOX, &maps.zbox[b], &full[sl], zt - LZ, yt, xc);
#pragma unroll
      for (int b = 0; b < G::NF; ++b) tma_load_3d(st + G::O_F + b * G::FBOX, &maps.fbox[b], &full[sl], zt - LZ, yt - R, xc);
#pragma unroll
      for (int t = 0; t < G::NC; ++t) tma_load_3d(st + G::O_C + t * G::TILE, &maps.ctile[t], &full[sl], zt, yt, xc);
    }
  };
  if (tid == 0) {
    for (int f = 0; f < 3; ++f) prefetch_tensormap(&maps.win[f]);
    for (int sl = 0; sl < G::NS; ++sl) {
      if (reinit) {
        mbar_inval(&full[sl]);
        mbar_inval(&empty[sl]);
      }
      mbar_init(&full[sl], 1);
      mbar_init(&empty[sl], G::NWARPS);
    }
    fence_barrier_init();
    for (int pl = 0; pl < G::NS && pl < nplanes; ++pl) issue(pl, pl);
  }
  __syncthreads();

  const int y = yt + ty, zb = zt + 2 * tz;
  const bool row_ok = y < a.ny;
  const bool vec_ok = row_ok && zb + 1 < a.nz;
  const int tcol = ty * QZ + 2 * tz;                    // own pair in a tile
  const int ycol = (ty + R) * QZ + 2 * tz;              // in a y-box
  const int zrow = ty * G::ZB + 2 * tz;                 // own row window start in a z-box
  const int frow = (ty + R) * G::ZB + 2 * tz;           // own row window start in a full box
  // the same as 32-bit shared addresses in stage `slot`, carried across planes
  // in the velocity pass; the stress pass (at the 128-register cap, where three
  // carried addresses spill) re-forms them from the slot every plane
  constexpr bool CA = PASS == 0 || FDR_EL_CARRY_STRESS;
  const SAddr s0{smem_u32(smem)};
  SAddr at_ = s0 + tcol, ay = s0 + ycol, az = s0 + zrow, afr = s0 + frow;
  uint32_t af = smem_u32(full);  // full[slot]; empty[slot] is 8 NS bytes on
  float gy = 1.0f, gz0 = 1.0f, gz1 = 1.0f;
  if (SPONGE && row_ok) {
    gy = a.gy[y];
    gz0 = zb < a.nz ? a.gz[zb] : 1.0f;
    gz1 = zb + 1 < a.nz ? a.gz[zb + 1] : 1.0f;
  }
  int kinj = -1, src_l = 0;
  float qsrc = 0.0f;
  if (PASS == 1 && a.sx >= 0 && y == a.sy && a.sz >= zb && a.sz < zb + 2 && a.it < a.n_series) {
    kinj = a.sx - xb;
    src_l = a.sz - zb;
    qsrc = a.series[a.it];
  }
  // 32-bit element offsets (the queue kernels take grids of < 2^32 elements)
  const uint32_t px32 = (uint32_t)a.pitch_x;
  const uint32_t obase = (uint32_t)xb * px32 + (uint32_t)y * (uint32_t)a.pitch_y + (uint32_t)zb;

  int slot = 0;
  uint32_t phase = 0;
  constexpr bool ROT = G::U % G::QD == 0;
  float2 q0[2 * R + G::U], q1[2 * R + G::U], q2[2 * R + G::U];

#pragma unroll 1
  for (int p0 = 0; p0 < nplanes; p0 += G::U) {
#pragma unroll
    for (int u = 0; u < G::U; ++u) {
      const int pl = p0 + u;
      if (pl >= nplanes) break;
      if (!CA) {
        const SAddr sl0 = s0 + slot * G::STAGE;
        at_ = sl0 + tcol;
        ay = sl0 + ycol;
        az = sl0 + zrow;
        afr = sl0 + frow;
        af = smem_u32(full + slot);
      }
      mbar_wait_a(af, phase);
      auto ld2 = [](SAddr p) { return f2to(ldf2(p)); };
      // queue slot of the newest plane: index 2R + u of this round (plane p0 - 2R + i at i)
      const int qn = ROT ? (2 * R + u) % G::QD : 2 * R + u;
      q0[qn] = ld2(at_ + G::O_WIN);
      q1[qn] = ld2(at_ + (G::O_WIN + G::TILE));
      q2[qn] = ld2(at_ + (G::O_WIN + 2 * G::TILE));
      const int k = pl - 2 * R;
      float2 out[6];
      if (k >= 0) {
        const int ci = R + u;  // queue index of the centre plane
        if (PASS == 0) {
          const SAddr sxy = ay + G::O_Y;
          const SAddr syy = ay + (G::O_Y + G::YBOX);
          float zw[2 + 2 * LZ], zw2[2 + 2 * LZ], fw[2 + 2 * LZ];
#pragma unroll
          for (int i = 0; i < 1 + LZ; ++i) {
            const float2 v = ld2(az + (G::O_Z + 2 * i));
            const float2 w = ld2(az + (G::O_Z + G::ZBOX + 2 * i));
            const float2 f = ld2(afr + (G::O_F + 2 * i));
            zw[2 * i] = v.x; zw[2 * i + 1] = v.y;
            zw2[2 * i] = w.x; zw2[2 * i + 1] = w.y;
            fw[2 * i] = f.x; fw[2 * i + 1] = f.y;
          }
          const SAddr syz = afr + (G::O_F + LZ);
          const float2 d0 = add2f(pB2<R>(sxy, QZ, a.c), zB2<R, LZ>(zw, a.c));     // By sxy + Bz sxz
          const float2 d1 = add2f(pF2<R>(syy, QZ, a.c), zB2<R, LZ>(fw, a.c));     // Fy syy + Bz syz
          const float2 d2 = add2f(pB2<R>(syz, G::ZB, a.c), zF2<R, LZ>(zw2, a.c)); // By syz + Fz szz
          const SAddr ct = at_ + G::O_C;
          const float2 vx = ld2(ct);
          const float2 vy = ld2(ct + G::TILE);
          const float2 vz = ld2(ct + 2 * G::TILE);
          const float2 bs = ld2(ct + 3 * G::TILE);
          out[0] = fma2f(bs, add2f(d0, xF2<R, G::QD, ROT>(q0, ci, a.c)), vx);
          out[1] = fma2f(bs, add2f(d1, xB2<R, G::QD, ROT>(q1, ci, a.c)), vy);
          out[2] = fma2f(bs, add2f(d2, xB2<R, G::QD, ROT>(q2, ci, a.c)), vz);
        } else {
          float xw[2 + 2 * LZ], yw[2 + 2 * LZ], zw[2 + 2 * LZ];
#pragma unroll
          for (int i = 0; i < 1 + LZ; ++i) {
            const float2 v0 = ld2(afr + (G::O_F + 2 * i));
            const float2 v1 = ld2(afr + (G::O_F + G::FBOX + 2 * i));
            const float2 v2 = ld2(afr + (G::O_F + 2 * G::FBOX + 2 * i));
            xw[2 * i] = v0.x; xw[2 * i + 1] = v0.y;
            yw[2 * i] = v1.x; yw[2 * i + 1] = v1.y;
            zw[2 * i] = v2.x; zw[2 * i + 1] = v2.y;
          }
          const SAddr vxb = afr + (G::O_F + LZ);
          const SAddr vyb = vxb + G::FBOX;
          const SAddr vzb = vxb + 2 * G::FBOX;
          const float2 ey = pB2<R>(vyb, G::ZB, a.c);
          const float2 ez = zB2<R, LZ>(zw, a.c);
          const float2 fyvx = pF2<R>(vxb, G::ZB, a.c);
          const float2 fzvx = zF2<R, LZ>(xw, a.c);
          const float2 d4 = add2f(zF2<R, LZ>(yw, a.c), pF2<R>(vzb, G::ZB, a.c));  // Fz vy + Fy vz
          const float2 ex = xB2<R, G::QD, ROT>(q0, ci, a.c);
          const SAddr ct = at_ + G::O_C;
          float2 cv[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) cv[t] = ld2(ct + t * G::TILE);
          const float2 lam = cv[6], mu = cv[7];
          const float2 l2m = make_float2(__fmaf_rn(2.0f, mu.x, lam.x), __fmaf_rn(2.0f, mu.y, lam.y));
          out[0] = fma2f(lam, add2f(ey, ez), fma2f(l2m, ex, cv[0]));
          out[1] = fma2f(lam, add2f(ez, ex), fma2f(l2m, ey, cv[1]));
          out[2] = fma2f(lam, add2f(ey, ex), fma2f(l2m, ez, cv[2]));
          out[3] = fma2f(mu, add2f(fyvx, xF2<R, G::QD, ROT>(q1, ci, a.c)), cv[3]);
          out[4] = fma2f(mu, add2f(fzvx, xF2<R, G::QD, ROT>(q2, ci, a.c)), cv[4]);
          out[5] = fma2f(mu, d4, cv[5]);
        }
      }
      // release the stage (every read of it is above)
      __syncwarp();
      if (elect_one() && el_arrive_last_a(af + 8u * G::NS)) {
        mbar_wait_a(af + 8u * G::NS, phase);
        fence_proxy_async();  // generic-proxy reads of the stage before the TMA refill (cross-proxy WAR)
        if (pl + G::NS < nplanes) issue(pl + G::NS, slot);
      }
      if (CA) {
        at_ = at_ + G::STAGE; ay = ay + G::STAGE; az = az + G::STAGE; afr = afr + G::STAGE;
        af += 8u;
      }
      if (++slot == G::NS) {
        slot = 0;
        phase ^= 1u;
        if (CA) {
          at_ = at_ - G::NS * G::STAGE; ay = ay - G::NS * G::STAGE;
          az = az - G::NS * G::STAGE; afr = afr - G::NS * G::STAGE;
          af -= 8u * G::NS;
        }
      }
      if (k >= 0) {
        constexpr int NO = PASS == 0 ? 3 : 6;
        if (SPONGE) {
          const float gxy = __fmul_rn(__ldg(a.gx + xb + k), gy);
          const float g0 = __fmul_rn(gxy, gz0), g1 = __fmul_rn(gxy, gz1);
#pragma unroll
          for (int i = 0; i < NO; ++i) out[i] = f2to(mul2(f2of(out[i]), pk(g0, g1)));
        }
        if (PASS == 1 && k == kinj) {
#pragma unroll
          for (int i = 0; i < 3; ++i) {
            if (src_l == 0) out[i].x = __fadd_rn(out[i].x, qsrc);
            else out[i].y = __fadd_rn(out[i].y, qsrc);
          }
        }
        const uint32_t o = obase + (uint32_t)k * px32;
#pragma unroll
        for (int i = 0; i < NO; ++i) {
          float* dst = a.f[(PASS == 0 ? VX : SXX) + i] + o;
          if (vec_ok) {
            if (PASS == 0 && a.keep_v) *reinterpret_cast<float2*>(dst) = out[i];
            else stg2cs(dst, out[i]);
          }
          else if (row_ok && zb < a.nz) dst[0] = out[i].x;
        }
      }
    }
    if (!ROT) {
#pragma unroll
      for (int i = 0; i < 2 * R; ++i) {
        q0[i] = q0[i + G::U];
        q1[i] = q1[i + G::U];
        q2[i] = q2[i + G::U];
      }
    }
  }
}

template <int R, int PASS, bool SPONGE>
#ifndef FDR_EL_MINB
#define FDR_EL_MINB 2
#endif
__global__ void __launch_bounds__(QN, FDR_EL_MINB) el_queue(const __grid_constant__ ElQMaps maps, const ElStep a) {
  extern __shared__ __align__(128) float smem[];
  if (PASS == 1) gather_vz(a);
  const int xb = a.x0 + blockIdx.z * a.chunk;
  const int xe = min(a.x1, xb + a.chunk);
  if (xb >= xe) return;
  el_queue_body<R, PASS, SPONGE>(maps, a, blockIdx.x * QZ, blockIdx.y * QY, xb, xe, smem, false);
}

// ============================================================ fused step
// el_fused: one persistent launch per time step runs both passes as items
// (pass, window k of C x-planes, tile t) handed out by a ticket counter, so the
// stress item of a window finds the new velocities and the stresses of its
// window still in L2 (windowed schedule above, without the launches).
//   - Ticket order: the velocity items in (k, t) order; the stress items in
//     the same order, each placed `lag` velocity items after V(k+1, t), i.e.
//     after every velocity item it depends on was handed out.
//   - S(k, t) reads the new velocities of windows k-1 .. k+1 on its tile's halo
//     and overwrites the stresses those velocity items read: it waits until
//     V(k-1 .. k+1) of the tile and its 8 neighbours have published (a stamp
//     per velocity item, st.release.gpu after the CTA's stores; relaxed polls +
//     fence.acq_rel.gpu + fence.proxy.async.global before the TMA reads).
//   - Velocity items wait for nothing: their inputs are final since the previous
//     launch.  Every dependency points to an earlier ticket and a CTA takes its
//     tickets in order, so the schedule cannot deadlock; a wait that exceeds
//     wait_cycles gives up and reports through the error word.
struct ElFuse {
  unsigned* ticket;   // monotonic across the run's launches
  unsigned base;      // ticket value of this launch's item 0
  unsigned* flags;    // [K][T] stamp of the last launch that finished V(k, t)
  unsigned stamp;     // this launch's stamp
  int C, K, T, tzn, tyn, lag;
  long long wait_cycles;
  unsigned* err;
};

FDR_DEV unsigned el_ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int R, bool SPONGE>
__global__ void __launch_bounds__(QN, FDR_EL_MINB)
    el_fused(const __grid_constant__ ElQMaps mv, const __grid_constant__ ElQMaps ms, const ElStep a,
             const ElFuse f) {
  extern __shared__ __align__(128) float smem[];
  __shared__ int item[3];  // pass (-1: no more items), window, tile
  const int NV = f.K * f.T, P = f.T + f.lag, total = 2 * NV;
  for (bool first = true;; first = false) {
    if (threadIdx.x == 0) {
      const int tk = (int)(atomicAdd(f.ticket, 1u) - f.base);
      int pass = -1, idx = 0;
      if (tk < total) {
        if (tk < P) {
          pass = 0;
          idx = tk;
        } else {
          const int j = tk - P, rem = NV - P;
          if (j < 2 * rem) {
            pass = (j & 1) ? 0 : 1;
            idx = (j & 1) ? P + (j >> 1) : (j >> 1);
          } else {
            pass = 1;
            idx = rem + (j - 2 * rem);
          }
        }
      }
      const int k = idx / f.T, t = idx - k * f.T;
      if (pass == 1) {
        const int tzi = t % f.tzn, tyi = t / f.tzn;
        long long t0 = 0;
        for (int spin = 0;; ++spin) {
          bool all = true;
          for (int dk = -1; dk <= 1; ++dk) {
            const int kk = k + dk;
            if (kk < 0 || kk >= f.K) continue;
            for (int dy = -1; dy <= 1; ++dy) {
              const int yy = tyi + dy;
              if (yy < 0 || yy >= f.tyn) continue;
#pragma unroll
              for (int dz = -1; dz <= 1; ++dz) {
                const int zz = tzi + dz;
                if (zz < 0 || zz >= f.tzn) continue;
                all &= el_ld_relaxed(f.flags + (size_t)kk * f.T + yy * f.tzn + zz) == f.stamp;
              }
            }
          }
          if (all) break;
          if (spin == 0) t0 = clock64();
          else if (clock64() - t0 > f.wait_cycles) {
            atomicAdd_system(f.err, 1u);
            break;
          }
        }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        asm volatile("fence.proxy.async.global;" ::: "memory");
      }
      item[0] = pass;
      item[1] = k;
      item[2] = t;
    }
    __syncthreads();  // also: every warp is done with the previous item's ring
    const int pass = item[0], k = item[1], t = item[2];
    if (pass < 0) break;
    const int zt = (t % f.tzn) * QZ, yt = (t / f.tzn) * QY;
    const int xb = k * f.C, xe = min(a.nx, xb + f.C);
    if (pass == 0) {
      el_queue_body<R, 0, SPONGE>(mv, a, zt, yt, xb, xe, smem, !first);
      __syncthreads();  // the CTA's velocity stores, then one release for all of them
      if (threadIdx.x == 0) {
        __threadfence();
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f.flags + (size_t)k * f.T + t),
                     "r"(f.stamp)
                     : "memory");
      }
    } else {
      el_queue_body<R, 1, SPONGE>(ms, a, zt, yt, xb, xe, smem, !first);
    }
    __syncthreads();  // item[] is rewritten next
  }
}

// vz at the receivers after a fused step (the two-pass kernels gather at the
// start of the stress launch)
__global__ void el_gather_kernel(const ElStep a) { gather_vz(a); }

// The tensor maps of one pass (velocity: PASS 0, stress: PASS 1).
template <int R, int PASS>
static int elq_maps(const fdr_elastic_args* a, ElQMaps* out) {
  using G = QGeoE<R, PASS>;
  ElQMaps& maps = *out;
  int rc = FDR_OK;
  const int ZBW = QZ + 2 * G::LZ, YBH = QY + 2 * R;
  if (PASS == 0) {
    const int win[3] = {SXX, SXY, SXZ};
    for (int f = 0; f < 3 && rc == FDR_OK; ++f) rc = el_encode(&maps.win[f], a->fields[win[f]], a, QZ, QY);
    if (rc == FDR_OK) rc = el_encode(&maps.ybox[0], a->fields[SXY], a, QZ, YBH);
    if (rc == FDR_OK) rc = el_encode(&maps.ybox[1], a->fields[SYY], a, QZ, YBH);
    if (rc == FDR_OK) rc = el_encode(&maps.zbox[0], a->fields[SXZ], a, ZBW, QY);
    if (rc == FDR_OK) rc = el_encode(&maps.zbox[1], a->fields[SZZ], a, ZBW, QY);
    if (rc == FDR_OK) rc = el_encode(&maps.fbox[0], a->fields[SYZ], a, ZBW, YBH);
    const float* ct[4] = {a->fields[VX], a->fields[VY], a->fields[VZ], a->params[0]};
    for (int t = 0; t < 4 && rc == FDR_OK; ++t) rc = el_encode(&maps.ctile[t], ct[t], a, QZ, QY);
  } else {
    const int win[3] = {VX, VY, VZ};
    for (int f = 0; f < 3 && rc == FDR_OK; ++f) rc = el_encode(&maps.win[f], a->fields[win[f]], a, QZ, QY);
    for (int f = 0; f < 3 && rc == FDR_OK; ++f) rc = el_encode(&maps.fbox[f], a->fields[win[f]], a, ZBW, YBH);
    const float* ct[8] = {a->fields[SXX], a->fields[SYY], a->fields[SZZ], a->fields[SXY],
                          a->fields[SXZ], a->fields[SYZ], a->params[1], a->params[2]};
    for (int t = 0; t < 8 && rc == FDR_OK; ++t) rc = el_encode(&maps.ctile[t], ct[t], a, QZ, QY);
  }
  return rc;
}

template <int R, int PASS>
static int elq_launch(const ElStep& s, const fdr_elastic_args* a, cudaStream_t st, int* chunk_cache) {
  using G = QGeoE<R, PASS>;
  const bool sponge = s.gx != nullptr;
  auto kern = sponge ? el_queue<R, PASS, true> : el_queue<R, PASS, false>;
  int occ_s = 0, nsm_s = 0;
  const int frc = fdr::launch_facts(reinterpret_cast<const void*>(kern), QN, G::SMEM, &occ_s, &nsm_s);
  if (frc != FDR_OK) return frc;
  int occ[2] = {occ_s, occ_s};
  int dev = 0;
  EL_CUDA(cudaGetDevice(&dev));
  const int tzn = (a->nz + QZ - 1) / QZ, tyn = (a->ny + QY - 1) / QY;
  if (*chunk_cache <= 0) {
    int nsm = 148;
    EL_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    const long tiles = (long)tzn * tyn, slots = (long)nsm * occ[sponge];
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
  ElQMaps maps;
  int rc = elq_maps<R, PASS>(a, &maps);
  if (rc != FDR_OK) return rc;
  ElStep t = s;
  t.chunk = *chunk_cache;
  dim3 grid(tzn, tyn, (a->nx + t.chunk - 1) / t.chunk);
  kern<<<grid, QN, G::SMEM, st>>>(maps, t);
  EL_CUDA(cudaGetLastError());
  return FDR_OK;
}

// ---- windowed schedule (experiment, B200FD_EL_WINDOW=C planes) ----
// The two passes of a step are launched alternately on windows of C x-planes,
// V(k+1) before S(k), so that the stress launch of window k finds the new
// velocities and the stresses of its window still in L2 (the two full-grid
// passes re-read both from HBM: 120 B/pt moved against 84 B/pt algorithmic).
// V(k+1) before S(k) also keeps the in-place update exact: V(k+1) reads the old
// stresses of window k's last R planes before S(k) overwrites them, and S(k)
// needs the new velocities of window k+1's first R planes.  C >= R.
// B200FD_EL_WINDOW_STREAMS=2 runs the stress launches on a second stream
// (V(k+2) and S(k) are independent), V(k+LEAD) held until S(k) is done.
struct ElWindowCtl {
  int planes = 0, streams = 1, lead = 3, sub = 1;
  int fuse = 0, fuse_lag = 160;  // B200FD_EL_FUSE (window planes of el_fused), B200FD_EL_FUSE_LAG
  cudaStream_t aux = nullptr;
  std::vector<cudaEvent_t> ev_v, ev_s;
};
static ElWindowCtl& el_window_ctl() {
  static ElWindowCtl c;
  return c;
}
// Re-read the knobs (once per run; tests flip them inside one process).
static void el_window_refresh() {
  ElWindowCtl& w = el_window_ctl();
  const char* e = getenv("B200FD_EL_WINDOW");
  w.planes = e ? atoi(e) : 0;
  e = getenv("B200FD_EL_WINDOW_STREAMS");
  w.streams = e ? atoi(e) : 1;
  e = getenv("B200FD_EL_WINDOW_LEAD");
  w.lead = e ? std::max(2, atoi(e)) : 3;
  e = getenv("B200FD_EL_WINDOW_SUB");
  w.sub = e ? std::max(1, atoi(e)) : 1;
  e = getenv("B200FD_EL_FUSE");
  w.fuse = e ? atoi(e) : 0;
  e = getenv("B200FD_EL_FUSE_LAG");
  w.fuse_lag = e ? std::max(0, atoi(e)) : 160;
}

template <int R, int PASS>
static int elq_fire(const ElQMaps& maps, const ElStep& s, const fdr_elastic_args* a, int x0, int x1,
                    int sub, cudaStream_t st) {
  using G = QGeoE<R, PASS>;
  const bool sponge = s.gx != nullptr;
  auto kern = sponge ? el_queue<R, PASS, true> : el_queue<R, PASS, false>;
  int occ = 0, nsm = 0;
  const int frc = fdr::launch_facts(reinterpret_cast<const void*>(kern), QN, G::SMEM, &occ, &nsm);
  if (frc != FDR_OK) return frc;
  ElStep t = s;
  t.x0 = x0;
  t.x1 = x1;
  t.keep_v = 1;
  t.chunk = (x1 - x0 + sub - 1) / sub;
  dim3 grid((a->nz + QZ - 1) / QZ, (a->ny + QY - 1) / QY, (x1 - x0 + t.chunk - 1) / t.chunk);
  kern<<<grid, QN, G::SMEM, st>>>(maps, t);
  EL_CUDA(cudaGetLastError());
  return FDR_OK;
}

template <int R>
static int el_window_step(const ElStep& s, const fdr_elastic_args* a, cudaStream_t st) {
  ElWindowCtl& w = el_window_ctl();
  const int C = std::max(w.planes, R);
  const int K = (a->nx + C - 1) / C;
  const int sub = w.sub;
  ElQMaps mv, ms;
  int rc = elq_maps<R, 0>(a, &mv);
  if (rc == FDR_OK) rc = elq_maps<R, 1>(a, &ms);
  if (rc != FDR_OK) return rc;
  auto lo = [&](int k) { return k * C; };
  auto hi = [&](int k) { return std::min(a->nx, (k + 1) * C); };
  if (w.streams < 2) {
    rc = elq_fire<R, 0>(mv, s, a, lo(0), hi(0), sub, st);
    for (int k = 0; k < K && rc == FDR_OK; ++k) {
      if (k + 1 < K) rc = elq_fire<R, 0>(mv, s, a, lo(k + 1), hi(k + 1), sub, st);
      if (rc == FDR_OK) rc = elq_fire<R, 1>(ms, s, a, lo(k), hi(k), sub, st);
    }
    return rc;
  }
  // the helper stream and the event pool are process-wide: one windowed step at a time
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (!w.aux) EL_CUDA(cudaStreamCreateWithFlags(&w.aux, cudaStreamNonBlocking));
  while ((int)w.ev_v.size() < K) {
    cudaEvent_t e1, e2;
    EL_CUDA(cudaEventCreateWithFlags(&e1, cudaEventDisableTiming));
    EL_CUDA(cudaEventCreateWithFlags(&e2, cudaEventDisableTiming));
    w.ev_v.push_back(e1);
    w.ev_s.push_back(e2);
  }
  // velocity launches on st, stress launches on aux
  int s_done = 0;  // stress launches issued so far
  auto stress = [&](int k) -> int {
    EL_CUDA(cudaStreamWaitEvent(w.aux, w.ev_v[std::min(k + 1, K - 1)], 0));
    int r2 = elq_fire<R, 1>(ms, s, a, lo(k), hi(k), sub, w.aux);
    if (r2 != FDR_OK) return r2;
    EL_CUDA(cudaEventRecord(w.ev_s[k], w.aux));
    return FDR_OK;
  };
  for (int k = 0; k < K && rc == FDR_OK; ++k) {
    if (k >= w.lead) EL_CUDA(cudaStreamWaitEvent(st, w.ev_s[k - w.lead], 0));
    rc = elq_fire<R, 0>(mv, s, a, lo(k), hi(k), sub, st);
    if (rc != FDR_OK) break;
    EL_CUDA(cudaEventRecord(w.ev_v[k], st));
    if (k >= 1) {
      rc = stress(k - 1);
      ++s_done;
    }
  }
  if (rc == FDR_OK) rc = stress(K - 1);
  if (rc == FDR_OK) EL_CUDA(cudaStreamWaitEvent(st, w.ev_s[K - 1], 0));  // join
  (void)s_done;
  return rc;
}

// One time step as one el_fused launch (+ the receiver gather).  Returns
// FDR_OK with *done = false when the grid is too small for the schedule.
template <int R>
static int el_fused_step(const ElStep& s, const fdr_elastic_args* a, cudaStream_t st, ElRunState* rs,
                         bool* done) {
  *done = false;
  ElWindowCtl& w = el_window_ctl();
  const int C = std::max(w.fuse, R);
  const int K = (a->nx + C - 1) / C;
  const int tzn = (a->nz + QZ - 1) / QZ, tyn = (a->ny + QY - 1) / QY;
  const int T = tzn * tyn;
  const int lag = std::min(std::max(w.fuse_lag, tzn + 2), T);
  if (K < 3) return FDR_OK;
  const bool sponge = s.gx != nullptr;
  auto kern = sponge ? el_fused<R, true> : el_fused<R, false>;
  const size_t smem = std::max(QGeoE<R, 0>::SMEM, QGeoE<R, 1>::SMEM);
  int occ = 0, nsm = 0;
  int rc = fdr::launch_facts(reinterpret_cast<const void*>(kern), QN, smem, &occ, &nsm);
  if (rc != FDR_OK) return rc;
  const size_t nflags = (size_t)K * T;
  if (!rs->fuse_buf) {
    EL_CUDA(cudaMallocAsync(&rs->fuse_buf, (nflags + 1) * sizeof(unsigned), st));
    EL_CUDA(cudaMemsetAsync(rs->fuse_buf, 0, (nflags + 1) * sizeof(unsigned), st));
    rs->fuse_step = 0;
  }
  ElQMaps mv, ms;
  rc = elq_maps<R, 0>(a, &mv);
  if (rc == FDR_OK) rc = elq_maps<R, 1>(a, &ms);
  if (rc != FDR_OK) return rc;
  int dev = 0;
  EL_CUDA(cudaGetDevice(&dev));
  ElFuse f;
  f.ticket = rs->fuse_buf + nflags;
  f.flags = rs->fuse_buf;
  const long long total = 2ll * K * T;
  const int grid = (int)std::min<long long>(total, (long long)nsm * occ);
  // every CTA takes one ticket beyond the last item before it exits
  f.base = (unsigned)((unsigned long long)rs->fuse_step * (unsigned long long)(total + grid));
  f.stamp = (unsigned)rs->fuse_step + 1u;
  f.C = C;
  f.K = K;
  f.T = T;
  f.tzn = tzn;
  f.tyn = tyn;
  f.lag = lag;
  const char* wc = getenv("B200FD_WAIT_CYCLES");
  f.wait_cycles = wc ? atoll(wc) : (1ll << 31);
  rc = fdr::err_word(dev, &f.err);
  if (rc != FDR_OK) return rc;
  ElStep t = s;
  t.keep_v = 1;
  kern<<<grid, QN, smem, st>>>(mv, ms, t, f);
  EL_CUDA(cudaGetLastError());
  if (t.gather_row >= 0) {
    el_gather_kernel<<<std::max(1, std::min(64, (t.n_rec + 255) / 256)), 256, 0, st>>>(t);
    EL_CUDA(cudaGetLastError());
  }
  ++rs->fuse_step;
  *done = true;
  return FDR_OK;
}

void el_queue_refresh_knobs() { el_window_refresh(); }

int el_queue_step(const ElStep& s, const fdr_elastic_args* a, cudaStream_t st, ElRunState* rs) {
  int rc = FDR_OK;
  int* chunk_cache = &rs->chunk;
  if (el_window_ctl().fuse > 0) {
    bool done = false;
    switch (a->order / 2) {
      case 1: rc = el_fused_step<1>(s, a, st, rs, &done); break;
      case 2: rc = el_fused_step<2>(s, a, st, rs, &done); break;
      case 3: rc = el_fused_step<3>(s, a, st, rs, &done); break;
      case 4: rc = el_fused_step<4>(s, a, st, rs, &done); break;
      default: return fail(FDR_EINVAL, "elastic queue kernel supports orders 2..8, got %d", a->order);
    }
    if (rc != FDR_OK || done) return rc;
  }
  if (el_window_ctl().planes > 0) {
    switch (a->order / 2) {
      case 1: return el_window_step<1>(s, a, st);
      case 2: return el_window_step<2>(s, a, st);
      case 3: return el_window_step<3>(s, a, st);
      case 4: return el_window_step<4>(s, a, st);
      default: return fail(FDR_EINVAL, "elastic queue kernel supports orders 2..8, got %d", a->order);
    }
  }
  switch (a->order / 2) {
    case 1: rc = elq_launch<1, 0>(s, a, st, chunk_cache); if (rc == FDR_OK) rc = elq_launch<1, 1>(s, a, st, chunk_cache); break;
    case 2: rc = elq_launch<2, 0>(s, a, st, chunk_cache); if (rc == FDR_OK) rc = elq_launch<2, 1>(s, a, st, chunk_cache); break;
    case 3: rc = elq_launch<3, 0>(s, a, st, chunk_cache); if (rc == FDR_OK) rc = elq_launch<3, 1>(s, a, st, chunk_cache); break;
    case 4: rc = elq_launch<4, 0>(s, a, st, chunk_cache); if (rc == FDR_OK) rc = elq_launch<4, 1>(s, a, st, chunk_cache); break;
    default: return fail(FDR_EINVAL, "elastic queue kernel supports orders 2..8, got %d", a->order);
  }
  return rc;
}

template <int R, int PASS>
static int el_launch(const ElStep& s, const fdr_elastic_args* a, cudaStream_t st, int chunk) {
  constexpr int NBOX = PASS == 0 ? 5 : 3;
  constexpr int NTILE = PASS == 0 ? 5 : 8;
  using G = EGeo<R, NBOX, NTILE>;
  const bool sponge = s.gx != nullptr;
  auto kern = sponge ? el_stream<R, PASS, true> : el_stream<R, PASS, false>;
  static int configured[2] = {-1, -1};
  int dev = 0;
  EL_CUDA(cudaGetDevice(&dev));
  if (configured[sponge] != dev) {
    EL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM));
    configured[sponge] = dev;
  }
  ElMaps maps;
  const int boxes0[5] = {SXY, SXZ, SYY, SYZ, SZZ}, boxes1[3] = {VX, VY, VZ};
  int rc = FDR_OK;
  for (int b = 0; b < NBOX && rc == FDR_OK; ++b)
    rc = el_encode(&maps.box[b], a->fields[PASS == 0 ? boxes0[b] : boxes1[b]], a, G::BZ, G::BY);
  if (PASS == 0) {
    const float* t[5] = {a->fields[SXX], a->fields[VX], a->fields[VY], a->fields[VZ], a->params[0]};
    for (int i = 0; i < 5 && rc == FDR_OK; ++i) rc = el_encode(&maps.tile[i], t[i], a, ETZ, ETY);
  } else {
    const float* t[8] = {a->fields[SXX], a->fields[SYY], a->fields[SZZ], a->fields[SXY],
                         a->fields[SXZ], a->fields[SYZ], a->params[1], a->params[2]};
    for (int i = 0; i < 8 && rc == FDR_OK; ++i) rc = el_encode(&maps.tile[i], t[i], a, ETZ, ETY);
  }
  if (rc != FDR_OK) return rc;
  ElStep t = s;
  t.chunk = chunk;
  dim3 grid((a->nz + ETZ - 1) / ETZ, (a->ny + ETY - 1) / ETY, (a->nx + chunk - 1) / chunk);
  kern<<<grid, ENT, G::SMEM, st>>>(maps, t);
  EL_CUDA(cudaGetLastError());
  return FDR_OK;
}

template <int R>
static int el_step_r(const ElStep& s, const fdr_elastic_args* a, cudaStream_t st, int* chunk_cache) {
  if (*chunk_cache <= 0) {
    int nsm = 148;
    int dev = 0;
    EL_CUDA(cudaGetDevice(&dev));
    EL_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    const long tiles = (long)((a->nz + ETZ - 1) / ETZ) * ((a->ny + ETY - 1) / ETY),
               slots = (long)nsm * EMINB;
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
  int rc = el_launch<R, 0>(s, a, st, *chunk_cache);
  if (rc == FDR_OK) rc = el_launch<R, 1>(s, a, st, *chunk_cache);
  return rc;
}

int el_stream_step(const ElStep& s, const fdr_elastic_args* a, cudaStream_t st, int* chunk_cache) {
  switch (a->order / 2) {
    case 1: return el_step_r<1>(s, a, st, chunk_cache);
    case 2: return el_step_r<2>(s, a, st, chunk_cache);
    case 3: return el_step_r<3>(s, a, st, chunk_cache);
    case 4: return el_step_r<4>(s, a, st, chunk_cache);
    default: return fail(FDR_EINVAL, "elastic stream kernel supports orders 2..8, got %d", a->order);
  }
}


// ========================================================= float64 path
// fdr_elastic64_run: el_vel_direct / el_str_direct (= oracle/elastic_ref.c)
// in IEEE double: the float64 reference of the float32 path's error.
struct ElStep64 {
  double* f[9];
  const double *bs, *lam, *mu;
  int nx, ny, nz, pitch_y;
  long long pitch_x;
  int radius;
  double c[FDR_MAX_RADIUS + 1];
  const double *gx, *gy, *gz, *series;
  int n_series, it, sx, sy, sz;
  const int* rec;
  int n_rec;
  double* traces;
  int gather_row;
};

__device__ __forceinline__ double at64(const double* u, const ElStep64& a, int x, int y, int z) {
  if (x < 0 || x >= a.nx || y < 0 || y >= a.ny || z < 0 || z >= a.nz) return 0.0;
  return u[(size_t)x * a.pitch_x + (size_t)y * a.pitch_y + z];
}
__device__ double dF64(const double* u, const ElStep64& a, int x, int y, int z, int ax) {
  const int dx = ax == 0, dy = ax == 1, dz = ax == 2;
  double d = __dmul_rn(a.c[1], __dsub_rn(at64(u, a, x + dx, y + dy, z + dz), at64(u, a, x, y, z)));
  for (int k = 2; k <= a.radius; ++k)
    d = __fma_rn(a.c[k], __dsub_rn(at64(u, a, x + k * dx, y + k * dy, z + k * dz),
                                   at64(u, a, x + (1 - k) * dx, y + (1 - k) * dy, z + (1 - k) * dz)), d);
  return d;
}
__device__ double dB64(const double* u, const ElStep64& a, int x, int y, int z, int ax) {
  const int dx = ax == 0, dy = ax == 1, dz = ax == 2;
  double d = __dmul_rn(a.c[1], __dsub_rn(at64(u, a, x, y, z), at64(u, a, x - dx, y - dy, z - dz)));
  for (int k = 2; k <= a.radius; ++k)
    d = __fma_rn(a.c[k], __dsub_rn(at64(u, a, x + (k - 1) * dx, y + (k - 1) * dy, z + (k - 1) * dz),
                                   at64(u, a, x - k * dx, y - k * dy, z - k * dz)), d);
  return d;
}
__device__ __forceinline__ double taper64(const ElStep64& a, int x, int y, int z) {
  return __dmul_rn(__dmul_rn(a.gx[x], a.gy[y]), a.gz[z]);
}

__global__ void __launch_bounds__(256) el_vel_direct64(const ElStep64 a) {
  const int z = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  const int x = blockIdx.z;
  if (z >= a.nz || y >= a.ny) return;
  const size_t o = (size_t)x * a.pitch_x + (size_t)y * a.pitch_y + z;
  const double b = a.bs[o];
  const double ax = __dadd_rn(__dadd_rn(dB64(a.f[SXY], a, x, y, z, 1), dB64(a.f[SXZ], a, x, y, z, 2)),
                              dF64(a.f[SXX], a, x, y, z, 0));
  const double ay = __dadd_rn(__dadd_rn(dF64(a.f[SYY], a, x, y, z, 1), dB64(a.f[SYZ], a, x, y, z, 2)),
                              dB64(a.f[SXY], a, x, y, z, 0));
  const double az = __dadd_rn(__dadd_rn(dB64(a.f[SYZ], a, x, y, z, 1), dF64(a.f[SZZ], a, x, y, z, 2)),
                              dB64(a.f[SXZ], a, x, y, z, 0));
  double vx = __fma_rn(b, ax, a.f[VX][o]), vy = __fma_rn(b, ay, a.f[VY][o]);
  double vz = __fma_rn(b, az, a.f[VZ][o]);
  if (a.gx) {
    const double g = taper64(a, x, y, z);
    vx = __dmul_rn(vx, g);
    vy = __dmul_rn(vy, g);
    vz = __dmul_rn(vz, g);
  }
  a.f[VX][o] = vx;
  a.f[VY][o] = vy;
  a.f[VZ][o] = vz;
}

__global__ void __launch_bounds__(256) el_str_direct64(const ElStep64 a) {
  if (a.gather_row >= 0) {  // vz is final for this step and not written here
    const int nthr = blockDim.x * blockDim.y;
    const int bi = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    const int t = threadIdx.x + blockDim.x * threadIdx.y;
    for (int i = bi * nthr + t; i < a.n_rec; i += nthr * (int)(gridDim.x * gridDim.y * gridDim.z)) {
      const int* q = a.rec + 3 * i;
      a.traces[(size_t)a.gather_row * a.n_rec + i] =
          a.f[VZ][(size_t)q[0] * a.pitch_x + (size_t)q[1] * a.pitch_y + q[2]];
    }
  }
  const int z = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  const int x = blockIdx.z;
  if (z >= a.nz || y >= a.ny) return;
  const size_t o = (size_t)x * a.pitch_x + (size_t)y * a.pitch_y + z;
  const double lam = a.lam[o], mu = a.mu[o];
  const double l2m = __fma_rn(2.0, mu, lam);
  const double ex = dB64(a.f[VX], a, x, y, z, 0), ey = dB64(a.f[VY], a, x, y, z, 1);
  const double ez = dB64(a.f[VZ], a, x, y, z, 2);
  double s[6];
  s[0] = __fma_rn(lam, __dadd_rn(ey, ez), __fma_rn(l2m, ex, a.f[SXX][o]));
  s[1] = __fma_rn(lam, __dadd_rn(ez, ex), __fma_rn(l2m, ey, a.f[SYY][o]));
  s[2] = __fma_rn(lam, __dadd_rn(ey, ex), __fma_rn(l2m, ez, a.f[SZZ][o]));
  s[3] = __fma_rn(mu, __dadd_rn(dF64(a.f[VX], a, x, y, z, 1), dF64(a.f[VY], a, x, y, z, 0)), a.f[SXY][o]);
  s[4] = __fma_rn(mu, __dadd_rn(dF64(a.f[VX], a, x, y, z, 2), dF64(a.f[VZ], a, x, y, z, 0)), a.f[SXZ][o]);
  s[5] = __fma_rn(mu, __dadd_rn(dF64(a.f[VY], a, x, y, z, 2), dF64(a.f[VZ], a, x, y, z, 1)), a.f[SYZ][o]);
  if (a.gx) {
    const double g = taper64(a, x, y, z);
#pragma unroll
    for (int i = 0; i < 6; ++i) s[i] = __dmul_rn(s[i], g);
  }
  if (x == a.sx && y == a.sy && z == a.sz && a.it < a.n_series) {
    const double q = a.series[a.it];
    s[0] = __dadd_rn(s[0], q);
    s[1] = __dadd_rn(s[1], q);
    s[2] = __dadd_rn(s[2], q);
  }
#pragma unroll
  for (int i = 0; i < 6; ++i) a.f[SXX + i][o] = s[i];
}

static int validate64(const fdr_elastic64_args* a) {
  if (!a) return fail(FDR_EINVAL, "args is NULL");
  if (a->abi_version != FDR_ABI_VERSION)
    return fail(FDR_EINVAL, "abi_version %d != library %d", a->abi_version, FDR_ABI_VERSION);
  if (a->order < 2 || a->order % 2 || a->order > 16)
    return fail(FDR_EINVAL, "elastic order must be even and within [2, 16], got %d", a->order);
  const int r = a->order / 2;
  if (a->nx < 2 * r + 1 || a->ny < 2 * r + 1 || a->nz < 2 * r + 1)
    return fail(FDR_EINVAL, "interior dims (%d, %d, %d) too small for halo width %d", a->nx,
                a->ny, a->nz, r);
  if (a->pitch_y < a->nz || a->pitch_x < (int64_t)a->ny * a->pitch_y)
    return fail(FDR_EINVAL, "bad pitches");
  if (a->n_steps < 0 || a->it0 < 0) return fail(FDR_EINVAL, "n_steps and it0 must be >= 0");
  for (int i = 0; i < 9; ++i)
    if (!a->fields[i]) return fail(FDR_EINVAL, "field %d is NULL", i);
  for (int i = 0; i < 3; ++i)
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

static int run64(const fdr_elastic64_args* a, cudaStream_t st) {
  for (int k = 0; k < a->n_steps; ++k) {
    ElStep64 s;
    memset(&s, 0, sizeof(s));
    for (int i = 0; i < 9; ++i) s.f[i] = a->fields[i];
    s.bs = a->params[0];
    s.lam = a->params[1];
    s.mu = a->params[2];
    s.nx = a->nx;
    s.ny = a->ny;
    s.nz = a->nz;
    s.pitch_y = a->pitch_y;
    s.pitch_x = a->pitch_x;
    s.radius = a->order / 2;
    for (int j = 0; j <= FDR_MAX_RADIUS; ++j) s.c[j] = a->c[j];
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
    s.gather_row = (a->n_rec > 0 && a->traces && s.it < a->trace_rows) ? s.it : -1;
    dim3 block(64, 4, 1), grid((a->nz + 63) / 64, (a->ny + 3) / 4, a->nx);
    el_vel_direct64<<<grid, block, 0, st>>>(s);
    EL_CUDA(cudaGetLastError());
    el_str_direct64<<<grid, block, 0, st>>>(s);
    EL_CUDA(cudaGetLastError());
  }
  return FDR_OK;
}

}  // namespace fdr_el

extern "C" {

size_t fdr_elastic_args_size(void) { return sizeof(fdr_elastic_args); }

int fdr_elastic_run(const fdr_elastic_args* args, void* stream) {
  int rc = fdr_el::validate(args);
  if (rc != FDR_OK) return rc;
  return fdr_el::run(args, static_cast<cudaStream_t>(stream));
}

size_t fdr_elastic64_args_size(void) { return sizeof(fdr_elastic64_args); }

int fdr_elastic64_run(const fdr_elastic64_args* args, void* stream) {
  int rc = fdr_el::validate64(args);
  if (rc != FDR_OK) return rc;
  return fdr_el::run64(args, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
