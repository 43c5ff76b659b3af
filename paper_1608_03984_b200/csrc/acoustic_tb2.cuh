// Two leapfrog steps per launch (temporal blocking) -- included by acoustic.cu.
//
// acoustic_tb2<R, GRID_M, SPONGE> advances u_{t-1}, u_t to u_{t+1}, u_{t+2}
// in one pass over HBM: every point still takes the reference's exact
// float32 sequence (kernel.py:199-211, as acoustic_queue) in both steps, so
// the result is bit-identical to two acoustic_queue launches.
//
//   step A (time step it):   u_{t+1} = A(u_t, u_{t-1}, m)  -> level `out`
//   step B (time step it+1): u_{t+2} = B(u_{t+1}, u_t, m)  -> level `prev`
//
// HBM traffic per point and pair of steps: u_t, u_{t-1} and m read, u_{t+1}
// and u_{t+2} written = 20 B, i.e. 10 B per point-step against 16 B for the
// single-step kernel (a ceiling of 655 instead of 410 GPts/s at 6.55 TB/s).
//
// Each CTA owns a 64(z) x TB_TY(y) column tile for both steps and streams it
// along x through the whole grid (no x-chunks).  Step A runs as in
// acoustic_queue (TMA ring A: newest u_t tile for the register queue, the
// u_t box of the plane pa being computed, its prev and m tiles).  Step B of
// plane pb = pa - R - D needs u_{t+1} at pb +- R along x -- this thread's own
// A results, kept in a thread-private shared-memory ring -- and the u_{t+1}
// box of plane pb, whose y/z halo belongs to the neighbouring tiles: ring B
// loads it from the `out` level (L2: it was written microseconds earlier)
// once the four neighbours (and this CTA) have published A-progress > pb.
// Progress is a per-tile counter in global memory (st.release.gpu after the
// plane's stores; ld.acquire.gpu + fence.proxy.async before the TMA that
// reads it).  Every tile is resident at once (cooperative launch: the host
// only takes this kernel when tiles <= resident CTA slots, 8 x 37 = 296 at
// 512^2 with two CTAs per SM), so the waits cannot deadlock; a wait still
// gives up after ~1 s and reports through the error word (pending_error).
//
// No level is read and written in the same launch except through the
// progress counters: A reads u_t (cur) and u_{t-1} (prev, own tile only, R+D
// planes before B overwrites that plane with u_{t+2}); B reads u_{t+1} (out)
// behind the counters and u_t (cur).  Receivers are recorded by a separate
// two-row gather after the launch (run_device).

#ifndef FDR_TB2_WAIT
#define FDR_TB2_WAIT 2  // 0: no waits (timing experiments only), 1: serial polls, 2: batched polls
#endif
#ifndef FDR_TB2_PUB
#define FDR_TB2_PUB 1  // publish A progress every FDR_TB2_PUB planes (0: never; timing experiments)
#endif
#ifndef FDR_TB2_FENCE
#define FDR_TB2_FENCE 1  // __threadfence before the progress release
#endif
constexpr int TB_TY = 14;                // y rows per tile (8 x 37 = 296 tiles at 512^2)
constexpr int TB_NT = NTZ * TB_TY;       // 224 threads, 7 warps

template <int R>
struct TBGeo {
  static_assert(R >= 1 && R <= 4, "two-step kernel: radius 1..4");
  static constexpr int LZ = 4;                 // z halo of the boxes (16-byte TMA rows)
  static constexpr int BZ = TZ + 2 * LZ;       // 72
  static constexpr int BY = TB_TY + 2 * R;
  static constexpr int BOX_BYTES = BZ * BY * 4;
  static constexpr int BOX_FLOATS = (BOX_BYTES + 127) / 128 * 32;
  static constexpr int TILE_FLOATS = TZ * TB_TY;
  static constexpr int TILE_BYTES = TILE_FLOATS * 4;
  // ring A stage: [newest u_t tile][u_t box of pa][prev tile of pa][m tile of pa]
  static constexpr int A_BOX = TILE_FLOATS;
  static constexpr int A_PREV = A_BOX + BOX_FLOATS;
  static constexpr int A_M = A_PREV + TILE_FLOATS;
  static constexpr int A_STAGE = A_M + TILE_FLOATS;
  // ring B stage: [u_{t+1} box of pb][u_t tile of pb][m tile of pb]
  static constexpr int B_UT = BOX_FLOATS;
  static constexpr int B_M = B_UT + TILE_FLOATS;
  static constexpr int B_STAGE = B_M + TILE_FLOATS;
  static constexpr int NA = 3;                 // ring A stages
  static constexpr int NB = 2;                 // ring B stages
  // extra lag of B behind A (planes): the B box of plane q is issued NB
  // planes ahead, when this tile's A has reached q + R + D - NB + 1; D keeps
  // that >= 2 planes of slack over the neighbours (R >= 4: none needed)
  static constexpr int PUBK = FDR_TB2_PUB > 1 ? FDR_TB2_PUB : 1;
  static constexpr int D = NB + 1 + PUBK - R > 0 ? NB + 1 + PUBK - R : 0;
  static constexpr int QB = 2 * R + 1 + D;     // own-column u_{t+1} ring (planes)
  static constexpr int QD = 2 * R + 1;         // A register queue depth
  static constexpr int U = R <= 2 ? QD : 2;    // A planes per unrolled round
  static constexpr int NWARPS = TB_NT / 32;   // compute warps (plus one producer warp)
  static constexpr int OFF_B = NA * A_STAGE;
  static constexpr int OFF_Q = OFF_B + NB * B_STAGE;
  static constexpr int OFF_BAR = OFF_Q + QB * TB_NT * 4;
  static constexpr size_t SMEM = size_t(OFF_BAR) * 4 + (3 * NA + 2 * NB) * 8;
};

struct TB2Run {
  unsigned* flags;       // per tile: A-progress counter (base + planes done)
  unsigned base;         // counter value of "no plane done" for this launch
  long long wait_cycles; // give-up bound of a neighbour wait (clock64 cycles)
  unsigned* err;         // host-mapped error word (pending_error)
};

FDR_DEV void mbar_arrive_ta_acq(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

FDR_DEV unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Wait until every tile in `tiles` (this one and its y/z neighbours) has
// published A-progress >= need; then order the async proxy (the TMA that
// reads their u_{t+1}) after the acquires.  Returns false on a timeout.
FDR_DEV unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
FDR_DEV bool tb2_wait(const TB2Run& run, const int* tiles, int nt, unsigned need) {
  bool ok = true;
#if FDR_TB2_WAIT == 1
  for (int i = 0; i < nt; ++i) {
    const unsigned* f = run.flags + tiles[i];
    if (ld_acquire_u32(f) >= need) continue;
    const long long t0 = clock64();
    while (ld_acquire_u32(f) < need) {
      if (clock64() - t0 > run.wait_cycles) {
        ok = false;
        break;
      }
    }
  }
#elif FDR_TB2_WAIT == 2
  // all counters in flight at once (one L2 round trip when they are ready),
  // relaxed polls, then one acquire fence for the lot
  long long t0 = 0;
  for (int pass = 0;; ++pass) {
    unsigned v[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) v[i] = i < nt ? ld_relaxed_u32(run.flags + tiles[i]) : need;
    bool all = true;
#pragma unroll
    for (int i = 0; i < 5; ++i) all &= v[i] >= need;
    if (all) break;
    if (pass == 0) t0 = clock64();
    else if (clock64() - t0 > run.wait_cycles) {
      ok = false;
      break;
    }
  }
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
#endif
  asm volatile("fence.proxy.async.global;" ::: "memory");
  return ok;
}

// The y and z taps of a quad from a box row-centre address (both steps).
template <int R, int BZ, int LZ>
FDR_DEV void lap_yz(f2& l01, f2& l23, uint32_t ab, const AcousticStep& a, f2 nz, f2& c01, f2& c23) {
  constexpr int NQ = 1 + 2 * LZ / 4;
  float zr[4 + 2 * LZ];
#pragma unroll
  for (int qd = 0; qd < NQ; ++qd) {
    const float4 v = lds128a(ab + 4u * (4 * qd - LZ));
    zr[4 * qd + 0] = v.x;
    zr[4 * qd + 1] = v.y;
    zr[4 * qd + 2] = v.z;
    zr[4 * qd + 3] = v.w;
  }
  c01 = pk(zr[LZ + 0], zr[LZ + 1]);
  c23 = pk(zr[LZ + 2], zr[LZ + 3]);
  (void)c01;
#pragma unroll
  for (int j = 1; j <= R; ++j) {  // y taps
    const float4 pp = lds128a(ab + 4u * (j * BZ));
    const float4 mm = lds128a(ab - 4u * (j * BZ));
    l01 = tap2(l01, a.w[j], pk(pp.x, pp.y), pk(mm.x, mm.y), nz);
    l23 = tap2(l23, a.w[j], pk(pp.z, pp.w), pk(mm.z, mm.w), nz);
  }
#pragma unroll
  for (int j = 1; j <= R; ++j) {  // z taps
    if (j % 2 == 0) {
      l01 = tap2(l01, a.w[j], pk(zr[LZ + j], zr[LZ + 1 + j]), pk(zr[LZ - j], zr[LZ + 1 - j]), nz);
      l23 = tap2(l23, a.w[j], pk(zr[LZ + 2 + j], zr[LZ + 3 + j]), pk(zr[LZ + 2 - j], zr[LZ + 3 - j]), nz);
    } else {
      float t[4];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) t[kk] = __fadd_rn(zr[LZ + kk + j], zr[LZ + kk - j]);
      l01 = add2(l01, prod2(a.w[j], pk(t[0], t[1]), nz));
      l23 = add2(l23, prod2(a.w[j], pk(t[2], t[3]), nz));
    }
  }
}

// s = coef * lap, s / m (exact), out = (2c - prev) + s, sponge: as acoustic_queue.
template <bool GRID_M, bool SPONGE>
FDR_DEV float4 tb2_update(f2 l01, f2 l23, f2 c01, f2 c23, float4 pvv, float4 mvv, float gxv, float gy,
                          f2 gz01, f2 gz23, bool tile_one, const AcousticStep& a, f2 nz) {
  f2 s01 = prod2(a.coef, l01, nz);
  f2 s23 = prod2(a.coef, l23, nz);
  if (GRID_M || a.m_mode == FDR_M_SCALAR) {
    const f2 m01 = GRID_M ? pk(mvv.x, mvv.y) : pk(a.m_scalar, a.m_scalar);
    const f2 m23 = GRID_M ? pk(mvv.z, mvv.w) : pk(a.m_scalar, a.m_scalar);
    const f2 up = 0x5f8000005f800000ull;
    const f2 down = 0x9f8000009f800000ull;
    const f2 q01 = div2_fast_neg(mul2(s01, up), m01);
    const f2 q23 = div2_fast_neg(mul2(s23, up), m23);
    const f2 y01 = fma2(q01, down, nz), y23 = fma2(q23, down, nz);
    const f2 d01 = fma2(y01, up, q01), d23 = fma2(y23, up, q23);
    if (((uint32_t)d01 | (uint32_t)(d01 >> 32) | (uint32_t)d23 | (uint32_t)(d23 >> 32)) == 0u) {
      s01 = y01;
      s23 = y23;
    } else {
      const ulonglong2 f = div_fix4(s01, s23, q01, q23, m01, m23, a.div_hi);
      s01 = f.x;
      s23 = f.y;
    }
  }
  f2 o01 = add2(sub2(add2(c01, c01), pk(pvv.x, pvv.y)), s01);
  f2 o23 = add2(sub2(add2(c23, c23), pk(pvv.z, pvv.w)), s23);
  if (SPONGE && !(tile_one && gxv == 1.0f)) {
    const float gxy = __fmul_rn(gxv, gy);
    const f2 gxy2 = pk(gxy, gxy);
    o01 = mul2(o01, mul2(gxy2, gz01));
    o23 = mul2(o23, mul2(gxy2, gz23));
  }
  return make_float4(lo(o01), hi(o01), lo(o23), hi(o23));
}

FDR_DEV void stg128(float* p, float4 v) {  // plain (L2-allocating) 16-byte store
  asm volatile("st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}
FDR_DEV void sts128a(uint32_t ad, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(ad), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}

template <int R, bool GRID_M, bool SPONGE>
__global__ void __launch_bounds__(TB_NT + 32, 2)
    acoustic_tb2(const __grid_constant__ CUtensorMap tm_box,   // u_t, BZ x BY boxes
                 const __grid_constant__ CUtensorMap tm_tile,  // u_t, tiles
                 const __grid_constant__ CUtensorMap tm_prev,  // u_{t-1}, tiles
                 const __grid_constant__ CUtensorMap tm_m,     // m, tiles
                 const __grid_constant__ CUtensorMap tm_box1,  // u_{t+1} (out), boxes
                 const AcousticStep a, const TB2Run run) {
  using G = TBGeo<R>;
  extern __shared__ __align__(128) float smem[];
  float* ringA = smem;
  float* ringB = smem + G::OFF_B;
  // barriers: fullA[NA] emptyA[NA] doneA[NA] fullB[NB] emptyB[NB]
  uint64_t* fullA = reinterpret_cast<uint64_t*>(smem + G::OFF_BAR);
  uint64_t* emptyA = fullA + G::NA;
  uint64_t* doneA = emptyA + G::NA;
  uint64_t* fullB = doneA + G::NA;
  uint64_t* emptyB = fullB + G::NB;

  const int tid = threadIdx.x;
  const int zt = blockIdx.x * TZ, yt = blockIdx.y * TB_TY;
  const int nx = a.nx;
  const int nst = nx + 3 * R + G::D;  // stream iterations s: newest u_t plane s - R

  auto issueA = [&](int s, int slot) {
    float* st = ringA + slot * G::A_STAGE;
    const int pa = s - 2 * R;
    const bool comp = pa >= 0 && pa < nx;
    const uint32_t bytes = G::TILE_BYTES + (comp ? G::BOX_BYTES + (GRID_M ? 2 : 1) * G::TILE_BYTES : 0);
    mbar_arrive_expect_tx(&fullA[slot], bytes);
    tma_load_3d(st, &tm_tile, &fullA[slot], zt, yt, s - R);
    if (comp) {
      tma_load_3d(st + G::A_BOX, &tm_box, &fullA[slot], zt - G::LZ, yt - R, pa);
      tma_load_3d(st + G::A_PREV, &tm_prev, &fullA[slot], zt, yt, pa);
      if (GRID_M) tma_load_3d(st + G::A_M, &tm_m, &fullA[slot], zt, yt, pa);
    }
  };

  // own-column u_{t+1} ring (thread-private): plane p in slot p mod QB;
  // slots of planes < 0 stay zero (the reference halo)
  const uint32_t aq0 = smem_u32(smem + G::OFF_Q) + 16u * (uint32_t)tid;
  constexpr uint32_t QSTRIDE = 16u * TB_NT;
  if (tid < TB_NT) {
#pragma unroll
    for (int i = 0; i < G::QB; ++i) sts128a(aq0 + i * QSTRIDE, make_float4(0.f, 0.f, 0.f, 0.f));
  }
  if (tid == 0) {
    prefetch_tensormap(&tm_box);
    prefetch_tensormap(&tm_tile);
    prefetch_tensormap(&tm_prev);
    prefetch_tensormap(&tm_box1);
    if (GRID_M) prefetch_tensormap(&tm_m);
    for (int s = 0; s < G::NA; ++s) {
      mbar_init(&fullA[s], 1);
      mbar_init(&emptyA[s], G::NWARPS);
      mbar_init(&doneA[s], G::NWARPS);
    }
    for (int s = 0; s < G::NB; ++s) {
      mbar_init(&fullB[s], 1);
      mbar_init(&emptyB[s], G::NWARPS);
    }
    fence_barrier_init();
    for (int s = 0; s < G::NA && s < nst; ++s) issueA(s, s);
  }
  // sponge factors of this thread's column (producer lanes: none)
  const int tz = tid % NTZ, ty = tid / NTZ;
  const int y = yt + ty;
  const int zb = zt + 4 * tz;
  const bool row_ok = tid < TB_NT && y < a.ny;
  const bool vec_ok = row_ok && zb + 3 < a.nz;
  float gy = 1.0f, gz[4] = {1.0f, 1.0f, 1.0f, 1.0f};
  bool tile_one = true;
  if (SPONGE) {
    if (row_ok) {
      gy = a.gy[y];
#pragma unroll
      for (int k = 0; k < 4; ++k) gz[k] = (zb + k < a.nz) ? a.gz[zb + k] : 1.0f;
    }
    tile_one = __syncthreads_and(gy == 1.0f && gz[0] == 1.0f && gz[1] == 1.0f && gz[2] == 1.0f &&
                                 gz[3] == 1.0f);
  } else {
    __syncthreads();
  }

  if (tid >= TB_NT) {
    // ---------------- producer warp: TMA refills, progress, B boxes --------
    if (!elect_one()) return;
    const int me = blockIdx.x + gridDim.x * blockIdx.y;
    // this tile and its y/z neighbours (the B boxes' halo owners)
    int nb[5];
    int nnb = 0;
    nb[nnb++] = me;
    if (blockIdx.x > 0) nb[nnb++] = me - 1;
    if (blockIdx.x + 1 < gridDim.x) nb[nnb++] = me + 1;
    if (blockIdx.y > 0) nb[nnb++] = me - gridDim.x;
    if (blockIdx.y + 1 < gridDim.y) nb[nnb++] = me + gridDim.x;
    int slot = 0;
    uint32_t ph = 0;
    for (int t = 0; t < nst; ++t) {
      // stage t read by every compute warp: refill it with stream plane t + NA
      mbar_wait(&emptyA[slot], ph);
      fence_proxy_async();  // the warps' generic reads of the stage before the TMA refill
      if (t + G::NA < nst) issueA(t + G::NA, slot);
      // A of plane t - 2R stored by every compute warp: publish the progress
      mbar_wait(&doneA[slot], ph);
      const int pa = t - 2 * R;
      if (FDR_TB2_PUB > 0 && pa >= 0 && pa < nx && ((pa + 1) % (FDR_TB2_PUB > 0 ? FDR_TB2_PUB : 1) == 0 || pa == nx - 1)) {
        if (FDR_TB2_FENCE) __threadfence();
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(run.flags + me),
                     "r"(run.base + (unsigned)pa + 1u)
                     : "memory");
      }
      // B of plane pb read: refill its slot with plane pb + NB once every
      // halo owner's A has passed it (the first NB planes: no earlier use)
      const int pb = t - 3 * R - G::D, q = pb + G::NB;
      if (q >= 0 && q < nx) {
        if (pb >= 0) {
          mbar_wait(&emptyB[pb % G::NB], (uint32_t)(pb / G::NB) & 1u);
          fence_proxy_async();  // as above, for ring B
        }
#if FDR_TB2_WAIT
        if (!tb2_wait(run, nb, nnb, run.base + (unsigned)q + 1u)) atomicAdd_system(run.err, 1u);
#endif
        const int sb = q % G::NB;
        float* st = ringB + sb * G::B_STAGE;
        mbar_arrive_expect_tx(&fullB[sb], G::BOX_BYTES + (GRID_M ? 2 : 1) * G::TILE_BYTES);
        tma_load_3d(st, &tm_box1, &fullB[sb], zt - G::LZ, yt - R, q);
        tma_load_3d(st + G::B_UT, &tm_tile, &fullB[sb], zt, yt, q);
        if (GRID_M) tma_load_3d(st + G::B_M, &tm_m, &fullB[sb], zt, yt, q);
      }
      if (++slot == G::NA) {
        slot = 0;
        ph ^= 1u;
      }
    }
    return;
  }

  // ---------------- compute warps ------------------------------------------
  const f2 gz01 = pk(gz[0], gz[1]), gz23 = pk(gz[2], gz[3]);
  // sources: step A injects series[it] at plane sx, step B series[it + 1]
  int src_k = -1;
  if (a.sx >= 0 && y == a.sy && a.sz >= zb && a.sz < zb + 4) src_k = a.sz - zb;
  const bool injA = src_k >= 0 && a.it < a.n_series;
  const bool injB = src_k >= 0 && a.it + 1 < a.n_series;
  const float qA = injA ? a.series[a.it] : 0.0f;
  const float qB = injB ? a.series[a.it + 1] : 0.0f;
  const f2 nz = pk(a.nzero, a.nzero);
  const uint32_t px32 = (uint32_t)a.pitch_x;
  const uint32_t oidx0 = (uint32_t)y * (uint32_t)a.pitch_y + (uint32_t)zb;
  const int bcen = (ty + R) * G::BZ + G::LZ + 4 * tz;  // own box-row centre
  const int tcol = ty * TZ + 4 * tz;                   // own column in a tile

  auto store_quad = [&](float* base, int plane, float4 v) {
    float* dst = base + (oidx0 + (uint32_t)plane * px32);
    if (vec_ok) {
      stg128(dst, v);
    } else if (row_ok) {
      const float o[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        if (zb + kk < a.nz) dst[kk] = o[kk];
    }
  };
  auto inject = [&](float4 v, float q) {
    float o[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) o[kk] = kk == src_k ? __fadd_rn(o[kk], q) : o[kk];
    return make_float4(o[0], o[1], o[2], o[3]);
  };

  int slotA = 0;
  uint32_t phA = 0;
  constexpr uint32_t SBA = G::A_STAGE * 4u;
  const uint32_t ringA_u = smem_u32(ringA), ringB_u = smem_u32(ringB), bar_u = smem_u32(fullA);
  uint32_t ac = ringA_u + 4u * tcol, ab = ringA_u + 4u * (G::A_BOX + bcen);
  uint32_t afa = bar_u;  // fullA[slotA]; emptyA / doneA are 8 * NA and 16 * NA bytes further

  float4 qw[2 * R + G::U];
#pragma unroll
  for (int i = 0; i < 2 * R + G::U; ++i) qw[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  constexpr bool ROTATE = G::U % G::QD == 0;
  auto arrive = [&](uint32_t bar) {
    __syncwarp();
    if (elect_one()) mbar_arrive_ta_acq(bar);
  };

  // one stream iteration: A of plane s - 2R, then B of plane s - 3R - D
  auto iter = [&](int s, int u) {
    const int pa = s - 2 * R;
    mbar_wait_a(afa, phA);
    const int qn = ROTATE ? (2 * R + u) % G::QD : 2 * R + u;
    qw[qn] = lds128a(ac);
    float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
    if (pa >= 0 && pa < nx) {
      f2 c01, c23;
      f2 l01, l23;
      {  // lap = w0 c (the queue's centre column is the box centre)
        const float4 cc = qw[ROTATE ? (R + u) % G::QD : R + u];
        c01 = pk(cc.x, cc.y);
        c23 = pk(cc.z, cc.w);
        l01 = prod2(a.w[0], c01, nz);
        l23 = prod2(a.w[0], c23, nz);
      }
#pragma unroll
      for (int j = 1; j <= R; ++j) {  // x taps from the register queue
        const float4 pp = qw[ROTATE ? (R + u + j) % G::QD : R + u + j];
        const float4 mm = qw[ROTATE ? (R + u - j + G::QD) % G::QD : R + u - j];
        l01 = tap2(l01, a.w[j], pk(pp.x, pp.y), pk(mm.x, mm.y), nz);
        l23 = tap2(l23, a.w[j], pk(pp.z, pp.w), pk(mm.z, mm.w), nz);
      }
      f2 cb01, cb23;
      lap_yz<R, G::BZ, G::LZ>(l01, l23, ab, a, nz, cb01, cb23);
      const float4 pvv = lds128a(ac + 4u * G::A_PREV);
      const float4 mvv = GRID_M ? lds128a(ac + 4u * G::A_M) : make_float4(1.f, 1.f, 1.f, 1.f);
      arrive(afa + 8u * G::NA);  // stage A read: the producer may refill it
      const float gxv = SPONGE ? __ldg(a.gx + pa) : 1.0f;
      o = tb2_update<GRID_M, SPONGE>(l01, l23, c01, c23, pvv, mvv, gxv, gy, gz01, gz23, tile_one, a, nz);
      if (injA && pa == a.sx) o = inject(o, qA);
      store_quad(a.out, pa, o);
    } else {
      arrive(afa + 8u * G::NA);
    }
    // own column of u_{t+1} (zero beyond the last plane: the halo)
    if (pa >= 0) sts128a(aq0 + (uint32_t)(pa % G::QB) * QSTRIDE, o);
    arrive(afa + 16u * G::NA);  // A stores of this plane issued (doneA)
    ac += SBA;
    ab += SBA;
    afa += 8u;
    if (++slotA == G::NA) {
      slotA = 0;
      phA ^= 1u;
      ac -= G::NA * SBA;
      ab -= G::NA * SBA;
      afa -= G::NA * 8u;
    }

    // ---- step B of plane pb
    const int pb = s - 3 * R - G::D;
    if (pb >= 0 && pb < nx) {
      const int slotB = pb % G::NB;
      const uint32_t phB = (uint32_t)(pb / G::NB) & 1u;  // uses of this slot so far
      const uint32_t stb = ringB_u + 4u * (uint32_t)(slotB * G::B_STAGE);
      const uint32_t fb = bar_u + 8u * (3 * G::NA + slotB);
      mbar_wait_a(fb, phB);
      f2 c01, c23;
      f2 l01, l23;
      {
        const float4 cc = lds128a(aq0 + (uint32_t)(pb % G::QB) * QSTRIDE);
        c01 = pk(cc.x, cc.y);
        c23 = pk(cc.z, cc.w);
        l01 = prod2(a.w[0], c01, nz);
        l23 = prod2(a.w[0], c23, nz);
      }
#pragma unroll
      for (int j = 1; j <= R; ++j) {  // x taps from the own-column ring
        const float4 pp = lds128a(aq0 + (uint32_t)((pb + j) % G::QB) * QSTRIDE);
        const float4 mm = lds128a(aq0 + (uint32_t)((pb - j + G::QB) % G::QB) * QSTRIDE);
        l01 = tap2(l01, a.w[j], pk(pp.x, pp.y), pk(mm.x, mm.y), nz);
        l23 = tap2(l23, a.w[j], pk(pp.z, pp.w), pk(mm.z, mm.w), nz);
      }
      f2 cb01, cb23;
      lap_yz<R, G::BZ, G::LZ>(l01, l23, stb + 4u * bcen, a, nz, cb01, cb23);
      const float4 pvv = lds128a(stb + 4u * (G::B_UT + tcol));
      const float4 mvv = GRID_M ? lds128a(stb + 4u * (G::B_M + tcol)) : make_float4(1.f, 1.f, 1.f, 1.f);
      arrive(fb + 8u * G::NB);  // stage B read
      const float gxv = SPONGE ? __ldg(a.gx + pb) : 1.0f;
      float4 ob = tb2_update<GRID_M, SPONGE>(l01, l23, c01, c23, pvv, mvv, gxv, gy, gz01, gz23, tile_one, a, nz);
      if (injB && pb == a.sx) ob = inject(ob, qB);
      store_quad(const_cast<float*>(a.prev), pb, ob);
    }
  };

#pragma unroll 1
  for (int s0 = 0; s0 < nst; s0 += G::U) {
#pragma unroll
    for (int u = 0; u < G::U; ++u) {
      if (s0 + u < nst) iter(s0 + u, u);
    }
    if (!ROTATE) {
#pragma unroll
      for (int i = 0; i < 2 * R; ++i) qw[i] = qmov(qw[i + G::U]);
    }
  }
}

// Receiver rows it and it + 1 after a two-step launch.
__global__ void gather2_kernel(const float* l1, const float* l2, const int* rec, const float* rec_w,
                               int n_rec, float* traces, int row, int rows, int nx, int ny, int nz,
                               int pitch_y, long long pitch_x) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_rec) return;
  if (row < rows)
    traces[(size_t)row * n_rec + i] = receiver_sample(l1, rec, rec_w, i, nx, ny, nz, pitch_y, pitch_x);
  if (row + 1 < rows)
    traces[(size_t)(row + 1) * n_rec + i] = receiver_sample(l2, rec, rec_w, i, nx, ny, nz, pitch_y, pitch_x);
}
