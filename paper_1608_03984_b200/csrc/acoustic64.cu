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
// a64_stream: a 32(z) x 8(y) tile of one point per thread streams along x.
// The 2r+1 x-neighbours of a thread's column live in a register queue; the
// y/z taps read a shared-memory box of the centre plane (zero halo written
// explicitly), double-buffered: the box of plane x+1, the queue's next value
// and this plane's prev / m are loaded into registers before plane x is
// computed, so their latency overlaps the arithmetic; one barrier per plane.
// FP64 on B200 is half the FP32 rate and the step is HBM-bound (OI 1.8).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include "../../include/b200fd.h"
#include "fdr_common.cuh"

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
  const int i = b * nthr + threadIdx.x + blockDim.x * threadIdx.y;
  if (i < a.n_rec) {
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

template <int R>
static int stream_launch(const A64Step& s, cudaStream_t st, int* chunk_cache) {
  using G = Geo<R>;
  const bool sponge = s.gx != nullptr;
  auto kern = sponge ? a64_stream<R, true> : a64_stream<R, false>;
  static int occ[2] = {0, 0}, nsm = 0, cfg_dev[2] = {-1, -1};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  if (cfg_dev[sponge] != dev) {
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[sponge], kern, NT, 0);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return cuda_fail(e, "fp64 stream kernel occupancy");
    if (occ[sponge] < 1) return fail(FDR_ECUDA, "fp64 stream kernel (r=%d) cannot be resident", R);
    cfg_dev[sponge] = dev;
  }
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
  if (a->variant != FDR_VARIANT_AUTO && a->variant != FDR_VARIANT_DIRECT &&
      a->variant != FDR_VARIANT_QUEUE)
    return fail(FDR_EINVAL, "fp64 variant must be AUTO, DIRECT or QUEUE, got %d", a->variant);
  if (a->variant == FDR_VARIANT_QUEUE && r > 8)
    return fail(FDR_EINVAL, "fp64 streaming kernel supports order <= 16, got %d", a->order);
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
  const bool stream = a->variant == FDR_VARIANT_QUEUE || (a->variant == FDR_VARIANT_AUTO && r <= 8);
  int chunk = 0;
  for (int k = 0; k < a->n_steps; ++k) {
    A64Step s;
    fill(s, a, k);
    if (stream) {
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

}  // namespace fdr64

extern "C" {

size_t fdr_acoustic64_args_size(void) { return sizeof(fdr_acoustic64_args); }

int fdr_acoustic64_run(const fdr_acoustic64_args* args, void* stream) {
  const int rc = fdr64::validate(args);
  if (rc != FDR_OK) return rc;
  return fdr64::run(args, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
