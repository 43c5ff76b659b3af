// Shared device helpers for the b200fd kernels (sm_100a).
//
// Exact-arithmetic helpers: the reference computes with numpy float32 ufuncs
// (/root/reference/pkg/src/fdroof/kernel.py:199-211), i.e. one IEEE
// round-to-nearest rounding per operation and never a fused multiply-add.
// The __f*_rn intrinsics are never contracted by nvcc, so every helper below
// emits exactly one rounding per reference operation.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define FDR_DEV __device__ __forceinline__

namespace fdr {

// Library-wide error reporting (acoustic.cu): sets the thread-local message
// returned by fdr_last_error() and returns `code`.
int fail(int code, const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* what);

// Resident CTAs per SM (*occ) and SM count (*nsm) of `kern` with `threads`
// threads and `smem` dynamic shared bytes on the current device (also sets
// the kernel's dynamic shared-memory limit).  Computed once per (kernel,
// device, threads, smem) under a lock, so host threads driving several
// devices never see another device's answer.  FDR_OK or an error code.
int launch_facts(const void* kern, int threads, size_t smem, int* occ, int* nsm);

// Device pointer (*d) of the host-mapped error word of device `dev`: kernels
// whose bounded waits time out add to it, and the next fdr_pending_error() /
// host-buffer run reports FDR_ECUDA (acoustic.cu).
int err_word(int dev, unsigned** d);

// The driver's cuTensorMapEncodeTiled, resolved once under std::call_once
// (safe from concurrent host threads); nullptr when the driver lacks it.
void* tensor_map_encoder();

// lap + w * (a + b): one tap pair of kernel.py:205 (three roundings).
FDR_DEV float tap(float lap, float w, float a, float b) {
  return __fadd_rn(lap, __fmul_rn(w, __fadd_rn(a, b)));
}

// (2c - prev) + s: kernel.py:211.  2*c == c + c exactly in IEEE arithmetic.
FDR_DEV float leapfrog(float c, float prev, float s) {
  return __fadd_rn(__fsub_rn(__fadd_rn(c, c), prev), s);
}

// ---------------------------------------------------------------- mbarrier
FDR_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

FDR_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

FDR_DEV void mbar_inval(uint64_t* bar) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

FDR_DEV void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

FDR_DEV void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

FDR_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

// try_wait suspends the warp until the phase completes or a time limit
// passes; every expiry costs a SYNCS + BRA issue slot in the spin loop.  A
// suspend-time hint (ns, FDR_MBAR_SUSPEND_NS; 0 = the hardware default)
// lengthens the sleep so waiting warps spin less.
#ifndef FDR_MBAR_SUSPEND_NS
#define FDR_MBAR_SUSPEND_NS 0
#endif
FDR_DEV void mbar_wait_a(uint32_t addr, uint32_t parity) {
#if FDR_MBAR_SUSPEND_NS > 0
  asm volatile(
      "{\n\t.reg .pred done;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1, %2;\n\t"
      "@!done bra WAIT_%=;\n}" ::"r"(addr),
      "r"(parity), "r"((uint32_t)FDR_MBAR_SUSPEND_NS)
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred done;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra WAIT_%=;\n}" ::"r"(addr),
      "r"(parity)
      : "memory");
#endif
}
FDR_DEV void mbar_wait(uint64_t* bar, uint32_t parity) { mbar_wait_a(smem_u32(bar), parity); }

// 3D TMA tile load global -> shared, completing on `bar` (complete_tx bytes).
// Coordinates are element indices (z, y, x) and may be negative / beyond the
// extents: those elements are zero-filled, which is the reference's
// zero-Dirichlet halo (kernel.py:5-6).
FDR_DEV void tma_load_3d(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                         int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

FDR_DEV void prefetch_tensormap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// Streaming (read-once) 16-byte global load that does not allocate in L1.
FDR_DEV float4 ldg_stream(const float* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

// Streaming 16-byte store (evict-first).
FDR_DEV void stg_stream(float* p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}

FDR_DEV float4 lds128(const float* p) { return *reinterpret_cast<const float4*>(p); }

// 16-byte shared load from a 32-bit shared-window address.  Volatile: the
// loads must stay after the stage's mbarrier wait (also a volatile asm).
FDR_DEV float4 lds128a(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(a));
  return v;
}

FDR_DEV float lds32a(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}

FDR_DEV unsigned long long lds64a(uint32_t a) {
  unsigned long long v;
  asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(a));
  return v;
}
FDR_DEV void sts64a(uint32_t a, unsigned long long v) {
  asm volatile("st.shared.b64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}

// One lane of a converged warp (elect.sync): no thread-index read.
FDR_DEV bool elect_one() {
  uint32_t e;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(e));
  return e != 0u;
}

// Register copy pinned to the ALU pipe.  ptxas emits plain copies as
// IMAD.MOV (FMA pipe, 2 cycles per warp instruction) about half the time;
// in the streaming kernels the FMA pipe carries all the arithmetic, so the
// register-queue shifts go through an identity PRMT instead (ALU pipe).
FDR_DEV float alu_mov(float x) {
  uint32_t r;
  asm volatile("prmt.b32 %0, %1, 0, 0x3210;" : "=r"(r) : "r"(__float_as_uint(x)));
  return __uint_as_float(r);
}
FDR_DEV float4 alu_mov4(float4 v) {
  return make_float4(alu_mov(v.x), alu_mov(v.y), alu_mov(v.z), alu_mov(v.w));
}
// Queue-shift copy of the float32 acoustic kernel; -DFDR_PLAIN_QMOV builds
// plain copies for A/B.  Measured: +1-3% at acoustic orders
// 8-16; the same change cost TTI 10% and float64 2%, so those keep plain copies.
#ifdef FDR_PLAIN_QMOV
FDR_DEV float4 qmov(float4 v) { return v; }
#else
FDR_DEV float4 qmov(float4 v) { return alu_mov4(v); }
#endif

// ---- packed FP32 pairs (sm_100a FADD2 / FMUL2 / FFMA2) -------------------
// Two floats in one 64-bit register pair, one IEEE round-to-nearest rounding
// per lane per operation.  ptxas contracts a packed multiply feeding a packed
// add into FFMA2 even under --fmad=false: products that a later add consumes
// must be formed so that they cannot be fused (acoustic.cu: prod2).
typedef unsigned long long f2;

FDR_DEV f2 pk(float lo, float hi) {
  f2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
FDR_DEV float lo(f2 v) { return __uint_as_float(static_cast<uint32_t>(v)); }
FDR_DEV float hi(f2 v) { return __uint_as_float(static_cast<uint32_t>(v >> 32)); }
FDR_DEV f2 add2(f2 a, f2 b) {
  f2 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
FDR_DEV f2 sub2(f2 a, f2 b) {
  f2 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
FDR_DEV f2 mul2(f2 a, f2 b) {  // only where the product feeds no add
  f2 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
FDR_DEV f2 fma2(f2 a, f2 b, f2 c) {
  f2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
}  // namespace fdr
