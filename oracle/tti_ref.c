/*
 * TTI pseudo-acoustic oracle (exact float32 restatement) -- TEST INFRASTRUCTURE ONLY.
 *
 * The reference has no TTI time stepping: equations.py:144-155 only catalogues
 * its cost (15 fields, factor 2, 3 second + 3 cross derivatives) and
 * PAPER.md:804-829 states the coupled system (Liu 2009)
 *   m p_tt = (1+2eps) (Gxx+Gyy) p + sqrt(1+2delta) Gzz r + q
 *   m r_tt = sqrt(1+2delta) (Gxx+Gyy) p + Gzz r + q
 * with Gzz = (c.grad)^2, c = (cos(phi) sin(theta), sin(phi) sin(theta), cos(theta)).
 * Gxx + Gyy = lap - Gzz (App. B of SURVEY.md; the paper's Gyy cross term
 * carries a sign typo).  Parity for this system is therefore pinned by this
 * file, whose float32 operation sequence the CUDA kernels reproduce bit for
 * bit, and checked for accuracy against the independent float64 numpy oracle
 * in oracle/tti.py.
 *
 * Per interior point, for u in {p, r} (undivided differences, h folded into k;
 * w2 second-derivative and w1 first-derivative weights, f32 of the exact
 * rationals; fmaf = one rounding):
 *   D2_a(u) = w2[0]*u; for j=1..R: D2 = fmaf(w2[j], u[+j] + u[-j], D2)   (axis a)
 *   D1_a(u) = w1[1]*(u[+1] - u[-1]); for j=2..R: D1 = fmaf(w1[j], u[+j] - u[-j], D1)
 *   dxx = D2_x u, dyy = D2_y u, dzz = D2_z u
 *   dxy = D1_x(D1_y u), dxz = D1_x(D1_z u), dyz = D1_y(D1_z u)   (inner first)
 *   gin = fmaf(cyz, dyz, fmaf(czz, dzz, cyy*dyy));  lin = dyy + dzz
 *   G   = fmaf(cxz, dxz, fmaf(cxy, dxy, fmaf(cxx, dxx, gin)));  L = lin + dxx
 *   H   = L - G
 * then with Hp = H(p), Gr = G(r):
 *   p_new = fmaf(k, fmaf(a, Hp, b*Gr), fmaf(2, p, -p_prev))
 *   r_new = fmaf(k, fmaf(b, Hp, Gr),   fmaf(2, r, -r_prev))
 *   p_new *= taper; r_new *= taper;  p_new += q; r_new += q  (source point)
 * k = f32(dt^2/(h^2 m)), a = f32(1+2eps), b = f32(sqrt(1+2delta)), c** the
 * f32 Gzz coefficients; receivers record p_new after injection.
 *
 * Layout: zero-padded (nx+2R, ny+2R, nz+2R) float32 levels for p and r, the
 * 9 parameter grids interior-shaped, C order.
 */
#include <math.h>
#include <pthread.h>
#include <stdlib.h>

#define MAXR 8

typedef struct {
  int r, nx, ny, nz;
  long sy, sx;
  const float *p, *pp, *q, *qp; /* p cur, p prev, r cur, r prev (padded) */
  float *pn, *qn;                /* new levels (padded) */
  const float* prm[9];           /* k a b cxx cyy czz cxy cyz cxz (interior) */
  const float *w2, *w1;
  const float *gx, *gy, *gz;
  int x_lo, x_hi;
} tti_job;

static inline float d2(const float* u, long s, const float* w2, int r) {
  float d = w2[0] * u[0];
  for (int j = 1; j <= r; ++j) d = fmaf(w2[j], u[j * s] + u[-j * s], d);
  return d;
}

static inline float d1(const float* u, long s, const float* w1, int r) {
  float d = w1[1] * (u[s] - u[-s]);
  for (int j = 2; j <= r; ++j) d = fmaf(w1[j], u[j * s] - u[-j * s], d);
  return d;
}

/* D1 along axis (stride so) of the inner D1 along axis (stride si), both at u */
static inline float d11(const float* u, long so, long si, const float* w1, int r) {
  float d = w1[1] * (d1(u + so, si, w1, r) - d1(u - so, si, w1, r));
  for (int j = 2; j <= r; ++j)
    d = fmaf(w1[j], d1(u + j * so, si, w1, r) - d1(u - j * so, si, w1, r), d);
  return d;
}

static void op(const float* u, long sx, long sy, const float* w2, const float* w1, int r,
               const float* c, float* G, float* L) {
  /* c = {cxx, cyy, czz, cxy, cyz, cxz} */
  const float dxx = d2(u, sx, w2, r), dyy = d2(u, sy, w2, r), dzz = d2(u, 1, w2, r);
  const float dxy = d11(u, sx, sy, w1, r), dxz = d11(u, sx, 1, w1, r);
  const float dyz = d11(u, sy, 1, w1, r);
  const float gin = fmaf(c[4], dyz, fmaf(c[2], dzz, c[1] * dyy));
  const float lin = dyy + dzz;
  *G = fmaf(c[5], dxz, fmaf(c[3], dxy, fmaf(c[0], dxx, gin)));
  *L = lin + dxx;
}

static void* run_slab(void* arg) {
  const tti_job* j = (const tti_job*)arg;
  const int r = j->r;
  for (int x = j->x_lo; x < j->x_hi; ++x)
    for (int y = 0; y < j->ny; ++y) {
      const long base = (long)(x + r) * j->sx + (long)(y + r) * j->sy + r;
      const long ib = ((long)x * j->ny + y) * j->nz;
      const float gxy = j->gx ? j->gx[x] * j->gy[y] : 1.0f;
      for (int z = 0; z < j->nz; ++z) {
        const long o = base + z, i = ib + z;
        const float k = j->prm[0][i], a = j->prm[1][i], b = j->prm[2][i];
        const float c[6] = {j->prm[3][i], j->prm[4][i], j->prm[5][i],
                            j->prm[6][i], j->prm[7][i], j->prm[8][i]};
        float Gp, Lp, Gr, Lr;
        op(j->p + o, j->sx, j->sy, j->w2, j->w1, r, c, &Gp, &Lp);
        op(j->q + o, j->sx, j->sy, j->w2, j->w1, r, c, &Gr, &Lr);
        (void)Lr;
        const float Hp = Lp - Gp;
        float pn = fmaf(k, fmaf(a, Hp, b * Gr), fmaf(2.0f, j->p[o], -j->pp[o]));
        float qn = fmaf(k, fmaf(b, Hp, Gr), fmaf(2.0f, j->q[o], -j->qp[o]));
        if (j->gx) {
          const float g = gxy * j->gz[z];
          pn = pn * g;
          qn = qn * g;
        }
        j->pn[o] = pn;
        j->qn[o] = qn;
      }
    }
  return 0;
}

/* levels: P[3], Q[3] padded in Wavefield order [scratch, prev, cur]; returns
 * the newest index (2 + n_steps) % 3. */
int fdo_tti_run(int order, int nx, int ny, int nz, const float* w2, const float* w1,
                const float* const* prm, float* P0, float* P1, float* P2, float* Q0, float* Q1,
                float* Q2, const float* gx, const float* gy, const float* gz,
                const float* series, int n_series, int sx_, int sy_, int sz_, int n_rec,
                const int* rec, float* traces, int trace_rows, int it0, int n_steps,
                int threads) {
  const int r = order / 2;
  const long sy = nz + 2 * r, sx = (long)(ny + 2 * r) * sy;
  float* P[3] = {P0, P1, P2};
  float* Q[3] = {Q0, Q1, Q2};
  if (threads < 1) threads = 1;
  if (threads > nx) threads = nx;
  pthread_t* tid = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  tti_job* jobs = (tti_job*)malloc(sizeof(tti_job) * threads);
  char* started = (char*)malloc(threads);
  for (int k = 0; k < n_steps; ++k) {
    const int io = (0 + k) % 3, ip = (1 + k) % 3, ic = (2 + k) % 3;
    for (int t = 0; t < threads; ++t) {
      tti_job* j = &jobs[t];
      j->r = r;
      j->nx = nx;
      j->ny = ny;
      j->nz = nz;
      j->sx = sx;
      j->sy = sy;
      j->p = P[ic];
      j->pp = P[ip];
      j->q = Q[ic];
      j->qp = Q[ip];
      j->pn = P[io];
      j->qn = Q[io];
      for (int i = 0; i < 9; ++i) j->prm[i] = prm[i];
      j->w2 = w2;
      j->w1 = w1;
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
    const long o = (long)(sx_ + r) * sx + (long)(sy_ + r) * sy + (sz_ + r);
    if (sx_ >= 0 && series && it < n_series) {
      P[io][o] = P[io][o] + series[it];
      Q[io][o] = Q[io][o] + series[it];
    }
    if (n_rec > 0 && traces && it < trace_rows)
      for (int i = 0; i < n_rec; ++i) {
        const int* c = rec + 3 * i;
        traces[(long)it * n_rec + i] = P[io][(long)(c[0] + r) * sx + (long)(c[1] + r) * sy + c[2] + r];
      }
  }
  free(tid);
  free(jobs);
  free(started);
  return (2 + n_steps) % 3;
}
