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
#include <cstring>

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
  const int i = b * nthr + t;
  if (i < a.n_rec) {
    const int* q = a.rec + 3 * i;
    a.traces[(size_t)a.gather_row * a.n_rec + i] =
        a.f[VZ][(size_t)q[0] * a.pitch_x + (size_t)q[1] * a.pitch_y + q[2]];
  }
}

__device__ __forceinline__ float taper(const ElStep& a, int x, int y, int z) {
  return __fmul_rn(__fmul_rn(a.gx[x], a.gy[y]), a.gz[z]);
}

// velocity pass, one thread per point (checker variant)
__global__ void __launch_bounds__(256) el_vel_direct(const ElStep a) {
  gather_vz(a);
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

__global__ void el_gather_kernel(const float* vz, const int* rec, int n_rec, float* traces, int row,
                                 int pitch_y, long long pitch_x) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_rec) {
    const int* q = rec + 3 * i;
    traces[(size_t)row * n_rec + i] = vz[(size_t)q[0] * pitch_x + (size_t)q[1] * pitch_y + q[2]];
  }
}

#define EL_CUDA(call)                                        \
  do {                                                       \
    cudaError_t e_ = (call);                                 \
    if (e_ != cudaSuccess) return fdr::cuda_fail(e_, #call); \
  } while (0)

int el_stream_step(const ElStep& s, const fdr_elastic_args* a, cudaStream_t st, int* chunk_cache);

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
  if (a->variant < 0 || a->variant > FDR_VARIANT_QUEUE || a->variant == FDR_VARIANT_TMA)
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
  const int row = s.it - 1;
  s.gather_row = (k > 0 && a->n_rec > 0 && a->traces && row < a->trace_rows) ? row : -1;
}

static int run(const fdr_elastic_args* a, cudaStream_t st) {
  int variant = a->variant;
  const bool small_index = (uint64_t)a->nx * (uint64_t)a->pitch_x < (1ull << 32);
  if (variant == FDR_VARIANT_AUTO)
    variant = (a->order <= 8 && small_index) ? FDR_VARIANT_QUEUE : FDR_VARIANT_DIRECT;
  if (variant == FDR_VARIANT_QUEUE && (!small_index || a->order > 8))
    return fail(FDR_EINVAL, "the elastic stream kernel needs order <= 8 and < 2^32 elements");
  int chunk = 0;
  for (int k = 0; k < a->n_steps; ++k) {
    ElStep s;
    fill(s, a, k);
    if (variant == FDR_VARIANT_QUEUE) {
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
  const int last = a->it0 + a->n_steps - 1;
  if (a->n_steps > 0 && a->n_rec > 0 && a->traces && last < a->trace_rows) {
    el_gather_kernel<<<(a->n_rec + 255) / 256, 256, 0, st>>>(a->fields[VZ], a->rec_xyz, a->n_rec,
                                                             a->traces, last, a->pitch_y, a->pitch_x);
    EL_CUDA(cudaGetLastError());
  }
  return FDR_OK;
}

int el_stream_step(const ElStep&, const fdr_elastic_args*, cudaStream_t, int*) {
  return fail(FDR_EINVAL, "elastic stream kernel not built yet");
}

}  // namespace fdr_el

extern "C" {

size_t fdr_elastic_args_size(void) { return sizeof(fdr_elastic_args); }

int fdr_elastic_run(const fdr_elastic_args* args, void* stream) {
  int rc = fdr_el::validate(args);
  if (rc != FDR_OK) return rc;
  return fdr_el::run(args, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
