// Included by acoustic.cu after the queue kernel (uses its tile geometry,
// packed-pair helpers and the exact scaled division).
//
// ======================================================= queue2 kernel
// The queue kernel with two adjacent y rows per thread (variant QUEUE2).
// Same tiles, TMA ring and stage layout as acoustic_queue (QGeo<R>), but a
// CTA of 128 threads covers the 64(z) x 16(y) tile: thread (tz, tp) owns the
// z-quad 4tz..4tz+3 of rows 2tp and 2tp+1.  What the second row buys:
//   - the y taps of both rows come from 2r + 2 box rows instead of 4r (the
//     rows y+j of row 0 and y+1-j of row 1 are the ones loaded for the other
//     row one tap earlier, and the own centre rows are already in registers):
//     shared-memory wavefronts per quad fall from 6 + 2r to 5 + r;
//   - the per-plane control (stage wait and release, carried addresses, the
//     division test, sponge and source tests) is paid once per 8 points;
//   - four independent accumulation chains per thread instead of two, which
//     hides the FADD2 latency of the exact serial tap order at 8 warps/SM.
// The price is two register queues: at most 255 registers per thread (two
// CTAs of four warps per SM).
// The per-point operation sequence is the queue kernel's exactly (the
// reference order, kernel.py:199-211), so the results are bit-identical.
#ifndef FDR_Q2_UNROLL
#define FDR_Q2_UNROLL 0
#endif

constexpr int NT2 = NTZ * TY / 2;  // 128 threads: 16 z-quads x 8 row pairs

template <int R>
struct Q2Geo {
  using G = QGeo<R>;
  static constexpr int QD = G::QD;
  // planes per unrolled round (whole-queue rotation for small r)
  static constexpr int U = FDR_Q2_UNROLL > 0 ? FDR_Q2_UNROLL : (R <= 2 ? QD : (R <= 4 ? 3 : 2));
  static constexpr int NWARPS = NT2 / 32;
};

template <int R, bool GRID_M, bool SPONGE>
__global__ void __launch_bounds__(NT2, 2)
    acoustic_queue2(const __grid_constant__ CUtensorMap tm_box,
                    const __grid_constant__ CUtensorMap tm_tile,
                    const __grid_constant__ CUtensorMap tm_prev,
                    const __grid_constant__ CUtensorMap tm_m, const AcousticStep a) {
  using G = QGeo<R>;
  using Q = Q2Geo<R>;
  extern __shared__ __align__(128) float smem[];
  float* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + G::NS * G::STAGE_FLOATS);

  gather_receivers(a);
  const int tid = threadIdx.x;
  const int tz = tid % NTZ, tp = tid / NTZ;
  const int zt = blockIdx.x * TZ, yt = blockIdx.y * TY;
  const int xb = a.x0 + blockIdx.z * a.chunk;
  const int xe = min(a.x1, xb + a.chunk);
  if (xb >= xe) return;
  const int n = xe - xb;
  const int nplanes = n + 2 * R;  // stream planes p: newest x = xb - R + p

  auto issue = [&](int p, int s) {
    float* st = ring + s * G::STAGE_FLOATS;
    const bool compute = p >= 2 * R;
    const uint32_t bytes = G::TILE_BYTES +
        (compute ? G::BOX_BYTES + (GRID_M ? 2 : 1) * G::TILE_BYTES : 0);
    mbar_arrive_expect_tx(&full[s], bytes);
    tma_load_3d(st, &tm_tile, &full[s], zt, yt, xb - R + p);
    if (compute) {
      const int xc = xb - 2 * R + p;
      tma_load_3d(st + G::OFF_BOX, &tm_box, &full[s], zt - G::LZ, yt - R, xc);
      tma_load_3d(st + G::OFF_PREV, &tm_prev, &full[s], zt, yt, xc);
      if (GRID_M) tma_load_3d(st + G::OFF_M, &tm_m, &full[s], zt, yt, xc);
    }
  };
  if (tid == 0) {
    prefetch_tensormap(&tm_box);
    prefetch_tensormap(&tm_tile);
    prefetch_tensormap(&tm_prev);
    if (GRID_M) prefetch_tensormap(&tm_m);
    for (int s = 0; s < G::NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&full[G::NS + s], Q::NWARPS);  // empty[s]
    }
    fence_barrier_init();
    for (int p = 0; p < G::NS && p < nplanes; ++p) issue(p, p);
  }
  __syncthreads();

  const int y0 = yt + 2 * tp;  // rows y0 (a) and y0 + 1 (b)
  const int zb = zt + 4 * tz;
  const bool ok_a = y0 < a.ny, ok_b = y0 + 1 < a.ny;
  const bool zfull = zb + 3 < a.nz;
  const int bcen = G::OFF_BOX + (2 * tp + R) * G::BZ + G::LZ + 4 * tz;  // row a, box centre
  const int tcol = 2 * tp * TZ + 4 * tz;  // row a's column within a halo-free tile

  float gya = 1.0f, gyb = 1.0f, gz[4] = {1.0f, 1.0f, 1.0f, 1.0f};
  bool tile_one = true;
  if (SPONGE) {
    if (ok_a) gya = a.gy[y0];
    if (ok_b) gyb = a.gy[y0 + 1];
#pragma unroll
    for (int k = 0; k < 4; ++k) gz[k] = (zb + k < a.nz) ? a.gz[zb + k] : 1.0f;
    tile_one = __syncthreads_and(gya == 1.0f && gyb == 1.0f && gz[0] == 1.0f && gz[1] == 1.0f &&
                                 gz[2] == 1.0f && gz[3] == 1.0f);
  }
  const f2 gz01 = pk(gz[0], gz[1]), gz23 = pk(gz[2], gz[3]);
  float gx_next = SPONGE ? __ldg(a.gx + xb) : 1.0f;
  // source: the one thread whose row pair holds the source column adds q at
  // plane kinj of row src_b (0: row a, 1: row b)
  int src_k = 0, kinj = -1, src_b = 0;
  float qsrc = 0.0f;
  if (a.sx >= 0 && (a.sy == y0 || a.sy == y0 + 1) && a.sz >= zb && a.sz < zb + 4 &&
      a.it < a.n_series) {
    src_k = a.sz - zb;
    src_b = a.sy - y0;
    kinj = a.sx - xb;
    qsrc = a.series[a.it];
  }
  const float div_hi = a.div_hi;
  const f2 nz = pk(a.nzero, a.nzero);
  const uint32_t px32 = (uint32_t)a.pitch_x, py32 = (uint32_t)a.pitch_y;
  const uint32_t oidx0 = (uint32_t)(xb - a.x0) * px32 + (uint32_t)y0 * py32 + (uint32_t)zb;

  int slot = 0;
  uint32_t phase = 0;
  constexpr uint32_t SB = G::STAGE_FLOATS * 4u;
  uint32_t ac = smem_u32(ring + tcol), ab = smem_u32(ring + bcen), af = smem_u32(full);
  auto finish = [&](int p) {
    __syncwarp();
    const uint32_t ae = af + 8u * G::NS;  // empty[slot]
    if (elect_one() && mbar_arrive_is_last_a(ae)) {
      mbar_wait_a(ae, phase);  // acquire: every warp's reads are done
      fence_proxy_async();     // cross-proxy WAR (see acoustic_queue)
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
      af -= G::NS * 8u;
    }
  };
  auto ldc = [&](int off) { return lds128a(ac + 4u * off); };
  auto ldb = [&](int off) { return lds128a(ab + 4u * off); };

  constexpr bool ROTATE = Q::U % Q::QD == 0;
  float4 qa[2 * R + Q::U], qb[2 * R + Q::U];

#pragma unroll
  for (int p = 0; p < 2 * R; ++p) {
    mbar_wait_a(af, phase);
    qa[p] = ldc(0);
    qb[p] = ldc(TZ);
    finish(p);
  }

#pragma unroll 1
  for (int p0 = 2 * R; p0 < nplanes; p0 += Q::U) {
#pragma unroll
    for (int u = 0; u < Q::U; ++u) {
      const int p = p0 + u;
      if (p >= nplanes) break;
      const int k = p - 2 * R;  // computing x = xb + k
      mbar_wait_a(af, phase);
      const int qn = ROTATE ? (2 * R + u) % Q::QD : 2 * R + u;
      qa[qn] = ldc(0);
      qb[qn] = ldc(TZ);
      // own row windows of the centre box (z taps), rows a and b
      float za[4 + 2 * G::LZ], zr[4 + 2 * G::LZ];
#pragma unroll
      for (int qd = 0; qd < G::NQ; ++qd) {
        const float4 v = ldb(4 * qd - G::LZ);
        za[4 * qd + 0] = v.x;
        za[4 * qd + 1] = v.y;
        za[4 * qd + 2] = v.z;
        za[4 * qd + 3] = v.w;
        const float4 w = ldb(G::BZ + 4 * qd - G::LZ);
        zr[4 * qd + 0] = w.x;
        zr[4 * qd + 1] = w.y;
        zr[4 * qd + 2] = w.z;
        zr[4 * qd + 3] = w.w;
      }
      const f2 ca01 = pk(za[G::LZ + 0], za[G::LZ + 1]), ca23 = pk(za[G::LZ + 2], za[G::LZ + 3]);
      const f2 cb01 = pk(zr[G::LZ + 0], zr[G::LZ + 1]), cb23 = pk(zr[G::LZ + 2], zr[G::LZ + 3]);
      f2 la01 = prod2(a.w[0], ca01, nz), la23 = prod2(a.w[0], ca23, nz);
      f2 lb01 = prod2(a.w[0], cb01, nz), lb23 = prod2(a.w[0], cb23, nz);
#pragma unroll
      for (int j = 1; j <= R; ++j) {  // x taps from the register queues
        const int ip = ROTATE ? (R + u + j) % Q::QD : R + u + j;
        const int im = ROTATE ? (R + u - j + Q::QD) % Q::QD : R + u - j;
        const float4 pa = qa[ip], ma = qa[im], pb = qb[ip], mb = qb[im];
        la01 = tap2(la01, a.w[j], pk(pa.x, pa.y), pk(ma.x, ma.y), nz);
        la23 = tap2(la23, a.w[j], pk(pa.z, pa.w), pk(ma.z, ma.w), nz);
        lb01 = tap2(lb01, a.w[j], pk(pb.x, pb.y), pk(mb.x, mb.y), nz);
        lb23 = tap2(lb23, a.w[j], pk(pb.z, pb.w), pk(mb.z, mb.w), nz);
      }
      // y taps: box rows -R .. R+1 relative to row a, each loaded once;
      // yr[R] and yr[R+1] are the own centre rows
      float4 yr[2 * R + 2];
      yr[R] = make_float4(za[G::LZ + 0], za[G::LZ + 1], za[G::LZ + 2], za[G::LZ + 3]);
      yr[R + 1] = make_float4(zr[G::LZ + 0], zr[G::LZ + 1], zr[G::LZ + 2], zr[G::LZ + 3]);
#pragma unroll
      for (int j = 1; j <= R; ++j) {
        yr[R - j] = ldb(-j * G::BZ);
        yr[R + 1 + j] = ldb((1 + j) * G::BZ);
        const float4 pa = yr[R + j], ma = yr[R - j], pb = yr[R + 1 + j], mb = yr[R + 1 - j];
        la01 = tap2(la01, a.w[j], pk(pa.x, pa.y), pk(ma.x, ma.y), nz);
        la23 = tap2(la23, a.w[j], pk(pa.z, pa.w), pk(ma.z, ma.w), nz);
        lb01 = tap2(lb01, a.w[j], pk(pb.x, pb.y), pk(mb.x, mb.y), nz);
        lb23 = tap2(lb23, a.w[j], pk(pb.z, pb.w), pk(mb.z, mb.w), nz);
      }
#pragma unroll
      for (int j = 1; j <= R; ++j) {  // z taps from the own row windows
        if (j % 2 == 0) {  // even shifts keep the register pairs aligned
          la01 = tap2(la01, a.w[j], pk(za[G::LZ + j], za[G::LZ + 1 + j]),
                      pk(za[G::LZ - j], za[G::LZ + 1 - j]), nz);
          la23 = tap2(la23, a.w[j], pk(za[G::LZ + 2 + j], za[G::LZ + 3 + j]),
                      pk(za[G::LZ + 2 - j], za[G::LZ + 3 - j]), nz);
          lb01 = tap2(lb01, a.w[j], pk(zr[G::LZ + j], zr[G::LZ + 1 + j]),
                      pk(zr[G::LZ - j], zr[G::LZ + 1 - j]), nz);
          lb23 = tap2(lb23, a.w[j], pk(zr[G::LZ + 2 + j], zr[G::LZ + 3 + j]),
                      pk(zr[G::LZ + 2 - j], zr[G::LZ + 3 - j]), nz);
        } else {  // odd shifts: scalar pair sums, packed accumulation
          float ta[4], tb[4];
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            ta[kk] = __fadd_rn(za[G::LZ + kk + j], za[G::LZ + kk - j]);
            tb[kk] = __fadd_rn(zr[G::LZ + kk + j], zr[G::LZ + kk - j]);
          }
          la01 = add2(la01, prod2(a.w[j], pk(ta[0], ta[1]), nz));
          la23 = add2(la23, prod2(a.w[j], pk(ta[2], ta[3]), nz));
          lb01 = add2(lb01, prod2(a.w[j], pk(tb[0], tb[1]), nz));
          lb23 = add2(lb23, prod2(a.w[j], pk(tb[2], tb[3]), nz));
        }
      }
      const float4 pva = ldc(G::OFF_PREV), pvb = ldc(G::OFF_PREV + TZ);
      float4 mva = make_float4(1.f, 1.f, 1.f, 1.f), mvb = mva;
      if (GRID_M) {
        mva = ldc(G::OFF_M);
        mvb = ldc(G::OFF_M + TZ);
      }
      finish(p);  // this warp is done with the stage
      f2 sa01 = prod2(a.coef, la01, nz), sa23 = prod2(a.coef, la23, nz);
      f2 sb01 = prod2(a.coef, lb01, nz), sb23 = prod2(a.coef, lb23, nz);
      if (GRID_M || a.m_mode == FDR_M_SCALAR) {
        const f2 ma01 = GRID_M ? pk(mva.x, mva.y) : pk(a.m_scalar, a.m_scalar);
        const f2 ma23 = GRID_M ? pk(mva.z, mva.w) : pk(a.m_scalar, a.m_scalar);
        const f2 mb01 = GRID_M ? pk(mvb.x, mvb.y) : pk(a.m_scalar, a.m_scalar);
        const f2 mb23 = GRID_M ? pk(mvb.z, mvb.w) : pk(a.m_scalar, a.m_scalar);
        const f2 up = 0x5f8000005f800000ull;    // 2^64, both lanes
        const f2 down = 0x9f8000009f800000ull;  // -2^-64 (the quotients are negated)
        const f2 qa01 = div2_fast_neg(mul2(sa01, up), ma01);
        const f2 qa23 = div2_fast_neg(mul2(sa23, up), ma23);
        const f2 qb01 = div2_fast_neg(mul2(sb01, up), mb01);
        const f2 qb23 = div2_fast_neg(mul2(sb23, up), mb23);
        const f2 ya01 = fma2(qa01, down, nz), ya23 = fma2(qa23, down, nz);
        const f2 yb01 = fma2(qb01, down, nz), yb23 = fma2(qb23, down, nz);
        const f2 da01 = fma2(ya01, up, qa01), da23 = fma2(ya23, up, qa23);
        const f2 db01 = fma2(yb01, up, qb01), db23 = fma2(yb23, up, qb23);
        const f2 dor = da01 | da23 | db01 | db23;
        if (((uint32_t)dor | (uint32_t)(dor >> 32)) == 0u) {
          sa01 = ya01;
          sa23 = ya23;
          sb01 = yb01;
          sb23 = yb23;
        } else {  // rare (subnormal quotients at wavefront precursors): div_fix
#ifdef FDR_COUNT_SLOW
          atomicAdd(&g_slow_quads, 1ull);
#endif
          const ulonglong2 fa = div_fix4(sa01, sa23, qa01, qa23, ma01, ma23, div_hi);
          const ulonglong2 fb = div_fix4(sb01, sb23, qb01, qb23, mb01, mb23, div_hi);
          sa01 = fa.x;
          sa23 = fa.y;
          sb01 = fb.x;
          sb23 = fb.y;
        }
      }
      // out = (2c - prev) + s
      f2 oa01 = add2(sub2(add2(ca01, ca01), pk(pva.x, pva.y)), sa01);
      f2 oa23 = add2(sub2(add2(ca23, ca23), pk(pva.z, pva.w)), sa23);
      f2 ob01 = add2(sub2(add2(cb01, cb01), pk(pvb.x, pvb.y)), sb01);
      f2 ob23 = add2(sub2(add2(cb23, cb23), pk(pvb.z, pvb.w)), sb23);
      if (SPONGE) {
        const float gxv = gx_next;
        if (k + 1 < n) gx_next = __ldg(a.gx + xb + k + 1);
        if (!(tile_one && gxv == 1.0f)) {  // out * ((gx*gy)*gz), products only
          const float gxya = __fmul_rn(gxv, gya), gxyb = __fmul_rn(gxv, gyb);
          const f2 ga = pk(gxya, gxya), gb = pk(gxyb, gxyb);
          oa01 = mul2(oa01, mul2(ga, gz01));
          oa23 = mul2(oa23, mul2(ga, gz23));
          ob01 = mul2(ob01, mul2(gb, gz01));
          ob23 = mul2(ob23, mul2(gb, gz23));
        }
      }
      float o[2][4] = {{lo(oa01), hi(oa01), lo(oa23), hi(oa23)},
                       {lo(ob01), hi(ob01), lo(ob23), hi(ob23)}};
      if (k == kinj) {
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            o[b][kk] = (b == src_b && kk == src_k) ? __fadd_rn(o[b][kk], qsrc) : o[b][kk];
      }
      float* dst = a.out + (oidx0 + (uint32_t)k * px32);
      if (zfull && ok_b) {
        stg_stream(dst, make_float4(o[0][0], o[0][1], o[0][2], o[0][3]));
        stg_stream(dst + py32, make_float4(o[1][0], o[1][1], o[1][2], o[1][3]));
      } else {
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          if (b == 0 ? ok_a : ok_b) {
            float* d = dst + b * py32;
            if (zfull) {
              stg_stream(d, make_float4(o[b][0], o[b][1], o[b][2], o[b][3]));
            } else {
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)
                if (zb + kk < a.nz) d[kk] = o[b][kk];
            }
          }
        }
      }
    }
    if (!ROTATE) {
#pragma unroll
      for (int i = 0; i < 2 * R; ++i) {
        qa[i] = qmov(qa[i + Q::U]);
        qb[i] = qmov(qb[i + Q::U]);
      }
    }
  }
}
