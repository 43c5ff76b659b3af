/*
 * C restatement of the reference acoustic step -- TEST INFRASTRUCTURE ONLY.
 *
 * Same arithmetic as /root/reference/pkg/src/fdroof/kernel.py:194-211 on the
 * reference's zero-padded float32 levels (kernel.py:119-123), one IEEE
 * rounding per operation: compiled with -ffp-contract=off and without
 * -ffast-math so no multiply-add is fused and nothing is re-associated.
 * Per interior point:
 *   lap = centre * c
 *   for axis x, y, z: for j = 1..r: lap = lap + w[j] * (c[+j] + c[-j])
 *   s = coef * lap;  s = s / m  (grid / scalar / none)
 *   out = (2c - prev) + s;  out = out * ((gx*gy)*gz)  [sponge extension]
 * then rotation (kernel.py:219), injection of series[it] (kernel.py:167-173),
 * receiver sampling after injection.  Threads split the x range into slabs
 * exactly like kernel.py:190-217 (disjoint writes, bit-identical results).
 *
 * Pinned by tests/test_oracle.py against goldens produced by the real
 * reference (tests/golden/make_golden.py).  Used by tests as a fast checker
 * for large GPU parity cases; never linked into the product library.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int r, nx, ny, nz;
  long sy, sx; /* padded strides (floats) */
  const float* cur;
  const float* prev;
  float* out;
  const float* w; /* w[0] = centre, w[1..r] taps */
  float coef;
  int m_mode; /* 0 none, 1 scalar, 2 grid (interior C order) */
  float m_scalar;
  const float* m;
  const float* gx;
  const float* gy;
  const float* gz;
  int x_lo, x_hi;
} slab_job;

static void* run_slab(void* p) {
  const slab_job* j = (const slab_job*)p;
  const int r = j->r;
  for (int x = j->x_lo; x < j->x_hi; ++x) {
    for (int y = 0; y < j->ny; ++y) {
      const long base = (long)(x + r) * j->sx + (long)(y + r) * j->sy + r;
      const float* c = j->cur + base;
      const float* pv = j->prev + base;
      float* o = j->out + base;
      const float* mrow = j->m_mode == 2 ? j->m + ((long)x * j->ny + y) * j->nz : 0;
      const float gxy = j->gx ? j->gx[x] * j->gy[y] : 1.0f;
      for (int z = 0; z < j->nz; ++z) {
        float lap = j->w[0] * c[z];
        for (int k = 1; k <= r; ++k) lap = lap + j->w[k] * (c[z + k * j->sx] + c[z - k * j->sx]);
        for (int k = 1; k <= r; ++k) lap = lap + j->w[k] * (c[z + k * j->sy] + c[z - k * j->sy]);
        for (int k = 1; k <= r; ++k) lap = lap + j->w[k] * (c[z + k] + c[z - k]);
        float s = j->coef * lap;
        if (j->m_mode == 2)
          s = s / mrow[z];
        else if (j->m_mode == 1)
          s = s / j->m_scalar;
        float v = (2.0f * c[z] - pv[z]) + s;
        if (j->gx) v = v * (gxy * j->gz[z]);
        o[z] = v;
      }
    }
  }
  return 0;
}

/* Advance n_steps; levels[3] are padded (nx+2r)(ny+2r)(nz+2r) arrays in
 * Wavefield.grids order.  Returns the index of the newest level. */
int fdo_acoustic_run(int order, int nx, int ny, int nz, const float* w, float coef, int m_mode,
                     float m_scalar, const float* m, float* g0, float* g1, float* g2,
                     const float* gx, const float* gy, const float* gz, const float* series,
                     int n_series, int sx_, int sy_, int sz_, int n_rec, const int* rec,
                     float* traces, int trace_rows, int it0, int n_steps, int threads) {
  const int r = order / 2;
  const long sz = 1, sy = nz + 2 * r, sx = (long)(ny + 2 * r) * sy;
  (void)sz;
  float* lv[3] = {g0, g1, g2};
  if (threads < 1) threads = 1;
  if (threads > nx) threads = nx;
  pthread_t* tid = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  slab_job* jobs = (slab_job*)malloc(sizeof(slab_job) * threads);
  char* started = (char*)malloc(threads);
  for (int k = 0; k < n_steps; ++k) {
    float* out = lv[(0 + k) % 3];
    const float* prev = lv[(1 + k) % 3];
    const float* cur = lv[(2 + k) % 3];
    for (int t = 0; t < threads; ++t) {
      slab_job* j = &jobs[t];
      j->r = r;
      j->nx = nx;
      j->ny = ny;
      j->nz = nz;
      j->sy = sy;
      j->sx = sx;
      j->cur = cur;
      j->prev = prev;
      j->out = out;
      j->w = w;
      j->coef = coef;
      j->m_mode = m_mode;
      j->m_scalar = m_scalar;
      j->m = m;
      j->gx = gx;
      j->gy = gy;
      j->gz = gz;
      j->x_lo = (int)((long)t * nx / threads);
      j->x_hi = (int)((long)(t + 1) * nx / threads);
      /* a slab whose thread cannot be created runs inline (never skipped) */
      started[t] = threads > 1 && pthread_create(&tid[t], 0, run_slab, j) == 0;
      if (!started[t]) run_slab(j);
    }
    for (int t = 0; t < threads; ++t)
      if (started[t]) pthread_join(tid[t], 0);
    const int it = it0 + k;
    if (sx_ >= 0 && series && it < n_series) {
      float* p = out + (long)(sx_ + r) * sx + (long)(sy_ + r) * sy + (sz_ + r);
      *p = *p + series[it];
    }
    if (n_rec > 0 && traces && it < trace_rows) {
      for (int i = 0; i < n_rec; ++i) {
        const int* q = rec + 3 * i;
        traces[(long)it * n_rec + i] = out[(long)(q[0] + r) * sx + (long)(q[1] + r) * sy + q[2] + r];
      }
    }
  }
  free(tid);
  free(jobs);
  free(started);
  return (2 + n_steps) % 3;
}
