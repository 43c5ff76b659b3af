/*
 * A plain C99 host program driving libb200fd.so through include/b200fd.h
 * only -- the way a non-Python host (or the C side of a cgo / JNI / N-API
 * binding) would use the library.  No Python, no torch: the program builds a
 * small acoustic problem (m grid, sponge, Ricker source, a receiver line),
 * sizes and allocates the device workspace itself, runs the whole simulation
 * with one fdr_acoustic_run_host call and writes inputs and outputs to a
 * binary file.  tests/test_c_consumer.py compiles it (CPU: header is valid C,
 * every used symbol links) and, on a GPU, runs it and checks the output
 * bit for bit against the C oracle fed the same inputs.
 *
 * usage: consumer ORDER NX NY NZ N_STEPS DT H OUT.bin
 * exit 0 on success; 1 bad usage; 2 library / CUDA error (message on stderr)
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "b200fd.h"

/* second-derivative central weights w_0..w_r as exact rationals (the
 * Fornberg weights of fdroof/stencils.py for these orders) */
static int weights_for(int order, double* w) {
  static const double o2[] = {-2.0, 1.0};
  static const double o4[] = {-5.0 / 2.0, 4.0 / 3.0, -1.0 / 12.0};
  static const double o8[] = {-205.0 / 72.0, 8.0 / 5.0, -1.0 / 5.0, 8.0 / 315.0, -1.0 / 560.0};
  const double* src = order == 2 ? o2 : order == 4 ? o4 : order == 8 ? o8 : NULL;
  int j;
  if (!src) return -1;
  for (j = 0; j <= order / 2; ++j) w[j] = src[j];
  return 0;
}

static unsigned int rng_state = 12345u;
static double uniform01(void) { /* xorshift32 */
  rng_state ^= rng_state << 13;
  rng_state ^= rng_state >> 17;
  rng_state ^= rng_state << 5;
  return (rng_state >> 8) * (1.0 / 16777216.0);
}

static float taper(int i, int n) { /* Cerjan-style profile, width 4 */
  const int w = 4;
  const int d = i < n - 1 - i ? i : n - 1 - i;
  if (d >= w) return 1.0f;
  return (float)exp(-pow(0.1 * (w - d), 2.0));
}

static int put(FILE* f, const void* p, size_t bytes) { return fwrite(p, 1, bytes, f) == bytes ? 0 : -1; }

int main(int argc, char** argv) {
  fdr_acoustic_args a, bad;
  double w[FDR_MAX_RADIUS + 1];
  int order, nx, ny, nz, n_steps, r, j, x, y, z, n_rec, rc, hdr[8], src[3];
  double dt, h, f0 = 15.0, t0;
  size_t npts, ws_bytes;
  float *m, *gx, *gy, *gz, *series, *final_, *traces;
  int32_t* rec;
  void* ws = NULL;
  FILE* out;

  if (argc != 9) {
    fprintf(stderr, "usage: %s ORDER NX NY NZ N_STEPS DT H OUT.bin\n", argv[0]);
    return 1;
  }
  order = atoi(argv[1]);
  nx = atoi(argv[2]);
  ny = atoi(argv[3]);
  nz = atoi(argv[4]);
  n_steps = atoi(argv[5]);
  dt = atof(argv[6]);
  h = atof(argv[7]);
  r = order / 2;
  if (weights_for(order, w) != 0 || nx < 1 || ny < 1 || nz < 1 || n_steps < 1) {
    fprintf(stderr, "unsupported arguments\n");
    return 1;
  }
  if (fdr_abi_version() != FDR_ABI_VERSION) {
    fprintf(stderr, "library ABI %d, header ABI %d\n", fdr_abi_version(), FDR_ABI_VERSION);
    return 2;
  }
  if (fdr_acoustic_args_size() != sizeof(fdr_acoustic_args)) {
    fprintf(stderr, "fdr_acoustic_args size mismatch\n");
    return 2;
  }

  /* inputs */
  npts = (size_t)nx * ny * nz;
  n_rec = nx;
  m = (float*)malloc(npts * sizeof(float));
  gx = (float*)malloc(nx * sizeof(float));
  gy = (float*)malloc(ny * sizeof(float));
  gz = (float*)malloc(nz * sizeof(float));
  series = (float*)malloc(n_steps * sizeof(float));
  rec = (int32_t*)malloc(3 * (size_t)n_rec * sizeof(int32_t));
  final_ = (float*)malloc(npts * sizeof(float));
  traces = (float*)malloc((size_t)n_steps * n_rec * sizeof(float));
  if (!m || !gx || !gy || !gz || !series || !rec || !final_ || !traces) return 2;
  for (x = 0; x < (int)npts; ++x) {
    const double v = 2000.0 + 1000.0 * uniform01();
    m[x] = (float)(1.0 / (v * v));
  }
  for (x = 0; x < nx; ++x) gx[x] = taper(x, nx);
  for (y = 0; y < ny; ++y) gy[y] = taper(y, ny);
  for (z = 0; z < nz; ++z) gz[z] = taper(z, nz);
  t0 = 1.0 / f0;
  for (j = 0; j < n_steps; ++j) {
    const double a2 = pow(3.14159265358979323846 * f0 * (j * dt - t0), 2.0);
    series[j] = (float)(1e3 * (1.0 - 2.0 * a2) * exp(-a2));
  }
  for (j = 0; j < n_rec; ++j) {
    rec[3 * j] = j;
    rec[3 * j + 1] = ny > 1 ? 1 : 0;
    rec[3 * j + 2] = nz > 2 ? 2 : 0;
  }
  src[0] = nx / 2;
  src[1] = ny / 2;
  src[2] = nz / 2;

  /* the run description: weights[0] = f32(3 w0), weights[j] = f32(w_j),
   * coef = f32(dt*dt/(h*h)) formed in double (b200fd.h) */
  memset(&a, 0, sizeof(a));
  a.abi_version = FDR_ABI_VERSION;
  a.order = order;
  a.nx = nx;
  a.ny = ny;
  a.nz = nz;
  a.pitch_y = (nz + 3) / 4 * 4;
  a.pitch_x = (int64_t)ny * a.pitch_y;
  a.weights[0] = (float)(3.0 * w[0]);
  for (j = 1; j <= r; ++j) a.weights[j] = (float)w[j];
  a.coef = (float)(dt * dt / (h * h));
  a.m_mode = FDR_M_GRID;
  a.m_lo = 0.0f; /* unknown: the library reduces the bounds itself */
  a.n_series = n_steps;
  a.src_x = src[0];
  a.src_y = src[1];
  a.src_z = src[2];
  a.n_rec = n_rec;
  a.trace_rows = n_steps;
  a.it0 = 0;
  a.n_steps = n_steps;
  a.variant = FDR_VARIANT_AUTO;

  /* the error path: a wrong ABI version is rejected with a message */
  bad = a;
  bad.abi_version = FDR_ABI_VERSION + 100;
  if (fdr_acoustic_workspace_bytes(&bad) != 0 || fdr_last_error()[0] == '\0') {
    fprintf(stderr, "bad ABI version not rejected\n");
    return 2;
  }
  printf("rejected: %s\n", fdr_last_error());

  ws_bytes = fdr_acoustic_workspace_bytes(&a);
  if (ws_bytes == 0) {
    fprintf(stderr, "workspace size: %s\n", fdr_last_error());
    return 2;
  }
  if (cudaMalloc(&ws, ws_bytes) != cudaSuccess) {
    fprintf(stderr, "cudaMalloc(%zu) failed\n", ws_bytes);
    return 2;
  }
  rc = fdr_acoustic_run_host(&a, m, gx, gy, gz, series, rec, final_, traces, ws, ws_bytes, NULL);
  if (rc < 0) {
    fprintf(stderr, "fdr_acoustic_run_host: %d %s\n", rc, fdr_last_error());
    return 2;
  }
  printf("ok: newest level %d, launches %lld\n", rc, (long long)fdr_last_launch_count());
  cudaFree(ws);

  out = fopen(argv[8], "wb");
  if (!out) return 2;
  hdr[0] = order;
  hdr[1] = nx;
  hdr[2] = ny;
  hdr[3] = nz;
  hdr[4] = n_steps;
  hdr[5] = n_rec;
  hdr[6] = rc;
  hdr[7] = a.pitch_y;
  if (put(out, hdr, sizeof(hdr)) || put(out, a.weights, (r + 1) * sizeof(float)) ||
      put(out, &a.coef, sizeof(float)) || put(out, m, npts * sizeof(float)) ||
      put(out, gx, nx * sizeof(float)) || put(out, gy, ny * sizeof(float)) ||
      put(out, gz, nz * sizeof(float)) || put(out, series, n_steps * sizeof(float)) ||
      put(out, rec, 3 * (size_t)n_rec * sizeof(int32_t)) || put(out, src, sizeof(src)) ||
      put(out, final_, npts * sizeof(float)) ||
      put(out, traces, (size_t)n_steps * n_rec * sizeof(float)))
    return 2;
  fclose(out);
  free(m);
  free(gx);
  free(gy);
  free(gz);
  free(series);
  free(rec);
  free(final_);
  free(traces);
  return 0;
}
