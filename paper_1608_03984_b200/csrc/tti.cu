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
};

__device__ __forceinline__ float at(const float* u, const TTIStep& a, int x, int y, int z) {
  if (x < 0 || x >= a.nx || y < 0 || y >= a.ny || z < 0 || z >= a.nz) return 0.0f;
  return u[(size_t)x * a.pitch_x + (size_t)y * a.pitch_y + z];
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
  const int i = b * nthr + t;
  if (i < a.n_rec) {
    const int* c = a.rec + 3 * i;
    a.traces[(size_t)a.gather_row * a.n_rec + i] =
        a.p[(size_t)c[0] * a.pitch_x + (size_t)c[1] * a.pitch_y + c[2]];
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
  const float k = a.prm[0][o], pa = a.prm[1][o], pb = a.prm[2][o];
  const float c[6] = {a.prm[3][o], a.prm[4][o], a.prm[5][o], a.prm[6][o], a.prm[7][o], a.prm[8][o]};
  float Gp, Lp, Gr, Lr;
  gl_op(a.p, a, x, y, z, c, &Gp, &Lp);
  gl_op(a.r, a, x, y, z, c, &Gr, &Lr);
  const float Hp = __fsub_rn(Lp, Gp);
  float pn = __fmaf_rn(k, __fmaf_rn(pa, Hp, __fmul_rn(pb, Gr)), __fmaf_rn(2.0f, a.p[o], -a.pp[o]));
  float rn = __fmaf_rn(k, __fmaf_rn(pb, Hp, Gr), __fmaf_rn(2.0f, a.r[o], -a.rp[o]));
  if (a.gx) {
    const float g = __fmul_rn(__fmul_rn(a.gx[x], a.gy[y]), a.gz[z]);
    pn = __fmul_rn(pn, g);
    rn = __fmul_rn(rn, g);
  }
  if (x == a.sx && y == a.sy && z == a.sz && a.it < a.n_series) {
    pn = __fadd_rn(pn, a.series[a.it]);
    rn = __fadd_rn(rn, a.series[a.it]);
  }
  a.pn[o] = pn;
  a.rn[o] = rn;
}

__global__ void tti_gather_kernel(const float* p, const int* rec, int n_rec, float* traces, int row,
                                  int pitch_y, long long pitch_x) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_rec) {
    const int* c = rec + 3 * i;
    traces[(size_t)row * n_rec + i] = p[(size_t)c[0] * pitch_x + (size_t)c[1] * pitch_y + c[2]];
  }
}

#define TTI_CUDA(call)                                    \
  do {                                                    \
    cudaError_t e_ = (call);                              \
    if (e_ != cudaSuccess) return fdr::cuda_fail(e_, #call); \
  } while (0)

int tti_stream_launch(const TTIStep&, const fdr_tti_args*, int, cudaStream_t, int*) {
  return fail(FDR_EINVAL, "TTI stream kernel not built yet");
}
int tti_stream_prepare(const fdr_tti_args*) { return FDR_OK; }

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
  for (int i = 0; i < 9; ++i)
    if (!a->params[i]) return fail(FDR_EINVAL, "parameter grid %d is NULL", i);
  if (a->sponge_x && (!a->sponge_y || !a->sponge_z))
    return fail(FDR_EINVAL, "sponge needs all three profiles");
  if (a->src_x >= 0 && (a->src_x >= a->nx || a->src_y < 0 || a->src_y >= a->ny ||
                        a->src_z < 0 || a->src_z >= a->nz))
    return fail(FDR_EINVAL, "source location outside interior");
  if (a->n_rec > 0 && (!a->rec_xyz || !a->traces))
    return fail(FDR_EINVAL, "receiver coordinates or trace buffer NULL");
  if (a->variant < 0 || a->variant > FDR_VARIANT_QUEUE || a->variant == FDR_VARIANT_TMA)
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
}

static int run(const fdr_tti_args* a, cudaStream_t st) {
  int variant = a->variant == FDR_VARIANT_AUTO ? FDR_VARIANT_DIRECT : a->variant;
  if (variant == FDR_VARIANT_QUEUE && a->n_steps > 0) {
    int rc = tti_stream_prepare(a);
    if (rc != FDR_OK) return rc;
  }
  int chunk = 0;
  for (int k = 0; k < a->n_steps; ++k) {
    TTIStep s;
    fill(s, a, k);
    if (variant == FDR_VARIANT_QUEUE) {
      int rc = tti_stream_launch(s, a, k, st, &chunk);
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
        a->p[(2 + a->n_steps) % 3], a->rec_xyz, a->n_rec, a->traces, last, a->pitch_y, a->pitch_x);
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

}  // extern "C"
