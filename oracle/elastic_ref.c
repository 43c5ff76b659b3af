/*
 * Elastic velocity-stress oracle (exact float32 restatement) -- TEST INFRASTRUCTURE ONLY.
 *
 * BASELINE config 5 has no reference implementation: the reference's elastic
 * catalogue entries are a displacement-form anisotropic kernel
 * (equations.py:156-177).  This file defines the isotropic
 * velocity-stress staggered-grid system (Virieux 1986, order-2R staggered
 * weights c_k from the exact Taylor solve on offsets +-(k-1/2)) whose float32
 * operation sequence the CUDA kernels reproduce bit for bit.  Accuracy is
 * checked against the independent float64 oracle in oracle/elastic.py.
 *
 * Staggering (array index -> position): vx (i+1/2,j,k), vy (i,j+1/2,k),
 * vz (i,j,k+1/2); sxx, syy, szz (i,j,k); sxy (i+1/2,j+1/2,k),
 * sxz (i+1/2,j,k+1/2), syz (i,j+1/2,k+1/2).  Undivided staggered differences
 * along an axis (fma chains, one rounding each):
 *   F(f)[i] = c1*(f[i+1]-f[i])   + sum_{k>=2} fma(c_k, f[i+k]-f[i+1-k])
 *   B(f)[i] = c1*(f[i]-f[i-1])   + sum_{k>=2} fma(c_k, f[i+k-1]-f[i-k])
 * Velocity pass (bs = f32(dt/(h rho))), in-plane terms first:
 *   vx = fma(bs, (By(sxy) + Bz(sxz)) + Fx(sxx), vx)
 *   vy = fma(bs, (Fy(syy) + Bz(syz)) + Bx(sxy), vy)
 *   vz = fma(bs, (By(syz) + Fz(szz)) + Bx(sxz), vz);   v *= taper
 * Stress pass (lam = f32(dt lambda/h), mu = f32(dt mu/h), l2m = fma(2, mu, lam)):
 *   ex = Bx(vx), ey = By(vy), ez = Bz(vz)
 *   sxx = fma(lam, ey + ez, fma(l2m, ex, sxx))
 *   syy = fma(lam, ez + ex, fma(l2m, ey, syy))
 *   szz = fma(lam, ey + ex, fma(l2m, ez, szz))
 *   sxy = fma(mu, Fy(vx) + Fx(vy), sxy)
 *   sxz = fma(mu, Fz(vx) + Fx(vz), sxz)
 *   syz = fma(mu, Fz(vy) + Fy(vz), syz);   s *= taper
 * then sxx, syy, szz += f32(series[it]) at the source (explosive source) and
 * receivers record vz.  Fields outside the interior are zero.  Parameters are
 * the integer-point values for every staggered component (no averaging).
 *
 * Layout: 9 zero-padded (nx+2R, ny+2R, nz+2R) float32 fields (vx vy vz sxx
 * syy szz sxy sxz syz), 3 interior-shaped parameter grids (bs lam mu).
 */
#include <math.h>
#include <pthread.h>
#include <stdlib.h>

enum { VX, VY, VZ, SXX, SYY, SZZ, SXY, SXZ, SYZ };

typedef struct {
  int r, nx, ny, nz, pass;
  long sy, sx;
  float* f[9];
  const float *bs, *lam, *mu, *c;
  const float *gx, *gy, *gz;
  int x_lo, x_hi;
} el_job;

static inline float dF(const float* f, long s, const float* c, int r) {
  float d = c[1] * (f[s] - f[0]);
  for (int k = 2; k <= r; ++k) d = fmaf(c[k], f[k * s] - f[(1 - k) * s], d);
  return d;
}

static inline float dB(const float* f, long s, const float* c, int r) {
  float d = c[1] * (f[0] - f[-s]);
  for (int k = 2; k <= r; ++k) d = fmaf(c[k], f[(k - 1) * s] - f[-k * s], d);
  return d;
}

static void* run_slab(void* arg) {
  const el_job* j = (const el_job*)arg;
  const int r = j->r;
  const long sx = j->sx, sy = j->sy;
  for (int x = j->x_lo; x < j->x_hi; ++x)
    for (int y = 0; y < j->ny; ++y) {
      const long base = (long)(x + r) * sx + (long)(y + r) * sy + r;
      const long ib = ((long)x * j->ny + y) * j->nz;
      const float gxy = j->gx ? j->gx[x] * j->gy[y] : 1.0f;
      for (int z = 0; z < j->nz; ++z) {
        const long o = base + z, i = ib + z;
        float* const* f = j->f;
        const float g = j->gx ? gxy * j->gz[z] : 1.0f;
        if (j->pass == 0) {
          const float b = j->bs[i];
          const float ax = (dB(f[SXY] + o, sy, j->c, r) + dB(f[SXZ] + o, 1, j->c, r)) +
                           dF(f[SXX] + o, sx, j->c, r);
          const float ay = (dF(f[SYY] + o, sy, j->c, r) + dB(f[SYZ] + o, 1, j->c, r)) +
                           dB(f[SXY] + o, sx, j->c, r);
          const float az = (dB(f[SYZ] + o, sy, j->c, r) + dF(f[SZZ] + o, 1, j->c, r)) +
                           dB(f[SXZ] + o, sx, j->c, r);
          float vx = fmaf(b, ax, f[VX][o]), vy = fmaf(b, ay, f[VY][o]), vz = fmaf(b, az, f[VZ][o]);
          if (j->gx) {
            vx = vx * g;
            vy = vy * g;
            vz = vz * g;
          }
          /* stored in the pass's own output slots (read-only fields differ) */
          f[VX][o] = vx;
          f[VY][o] = vy;
          f[VZ][o] = vz;
        } else {
          const float lam = j->lam[i], mu = j->mu[i];
          const float l2m = fmaf(2.0f, mu, lam);
          const float ex = dB(f[VX] + o, sx, j->c, r), ey = dB(f[VY] + o, sy, j->c, r);
          const float ez = dB(f[VZ] + o, 1, j->c, r);
          float sxx = fmaf(lam, ey + ez, fmaf(l2m, ex, f[SXX][o]));
          float syy = fmaf(lam, ez + ex, fmaf(l2m, ey, f[SYY][o]));
          float szz = fmaf(lam, ey + ex, fmaf(l2m, ez, f[SZZ][o]));
          float sxy = fmaf(mu, dF(f[VX] + o, sy, j->c, r) + dF(f[VY] + o, sx, j->c, r), f[SXY][o]);
          float sxz = fmaf(mu, dF(f[VX] + o, 1, j->c, r) + dF(f[VZ] + o, sx, j->c, r), f[SXZ][o]);
          float syz = fmaf(mu, dF(f[VY] + o, 1, j->c, r) + dF(f[VZ] + o, sy, j->c, r), f[SYZ][o]);
          if (j->gx) {
            sxx = sxx * g;
            syy = syy * g;
            szz = szz * g;
            sxy = sxy * g;
            sxz = sxz * g;
            syz = syz * g;
          }
          f[SXX][o] = sxx;
          f[SYY][o] = syy;
          f[SZZ][o] = szz;
          f[SXY][o] = sxy;
          f[SXZ][o] = sxz;
          f[SYZ][o] = syz;
        }
      }
    }
  return 0;
}

static void run_pass(el_job* jobs, pthread_t* tid, int threads, int pass) {
  char* started = (char*)malloc(threads);
  for (int t = 0; t < threads; ++t) {
    jobs[t].pass = pass;
    /* a slab whose thread cannot be created runs inline (never skipped) */
    started[t] = threads > 1 && pthread_create(&tid[t], 0, run_slab, &jobs[t]) == 0;
    if (!started[t]) run_slab(&jobs[t]);
  }
  for (int t = 0; t < threads; ++t)
    if (started[t]) pthread_join(tid[t], 0);
  free(started);
}

/* The velocity pass reads stresses only (plus its own v), the stress pass
 * velocities only (plus its own s): in-place updates are race-free across
 * slab threads. */
int fdo_elastic_run(int order, int nx, int ny, int nz, const float* c, const float* bs,
                    const float* lam, const float* mu, float* const* fields, const float* gx,
                    const float* gy, const float* gz, const float* series, int n_series, int sx_,
                    int sy_, int sz_, int n_rec, const int* rec, float* traces, int trace_rows,
                    int it0, int n_steps, int threads) {
  const int r = order / 2;
  const long sy = nz + 2 * r, sx = (long)(ny + 2 * r) * sy;
  if (threads < 1) threads = 1;
  if (threads > nx) threads = nx;
  pthread_t* tid = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  el_job* jobs = (el_job*)malloc(sizeof(el_job) * threads);
  for (int t = 0; t < threads; ++t) {
    el_job* j = &jobs[t];
    j->r = r;
    j->nx = nx;
    j->ny = ny;
    j->nz = nz;
    j->sx = sx;
    j->sy = sy;
    for (int i = 0; i < 9; ++i) j->f[i] = fields[i];
    j->bs = bs;
    j->lam = lam;
    j->mu = mu;
    j->c = c;
    j->gx = gx;
    j->gy = gy;
    j->gz = gz;
    j->x_lo = (int)((long)t * nx / threads);
    j->x_hi = (int)((long)(t + 1) * nx / threads);
  }
  for (int k = 0; k < n_steps; ++k) {
    run_pass(jobs, tid, threads, 0);
    run_pass(jobs, tid, threads, 1);
    const int it = it0 + k;
    if (sx_ >= 0 && series && it < n_series) {
      const long o = (long)(sx_ + r) * sx + (long)(sy_ + r) * sy + (sz_ + r);
      fields[SXX][o] = fields[SXX][o] + series[it];
      fields[SYY][o] = fields[SYY][o] + series[it];
      fields[SZZ][o] = fields[SZZ][o] + series[it];
    }
    if (n_rec > 0 && traces && it < trace_rows)
      for (int i = 0; i < n_rec; ++i) {
        const int* q = rec + 3 * i;
        traces[(long)it * n_rec + i] = fields[VZ][(long)(q[0] + r) * sx + (long)(q[1] + r) * sy + q[2] + r];
      }
  }
  free(tid);
  free(jobs);
  return 0;
}
