// kbe200 — B200 (sm_100a) kernels for the two-time Kadanoff–Baym step.
//
// Hot path of kbesolve 0.1.0 (pkg/src/kbesolve/propagator.py:316-382),
// re-designed for one B200: a device-resident, packed, time-sliced history
// (see include/kbe200.h), one fused launch per operator class, and
// device-side convergence so that a step never waits on the host.
//
//   K1 sigma_frontier_kernel   second-Born Sigma slice (selfenergy.py:59-325)
//   K2 collision_kernel        history-streaming I< / I> (collision.py:141-277), full or
//                              incremental (complex64 shadow) evaluations
//      collision_langreth_kernel  the same for limit_mode="langreth"
//   K3 update_kernel           predictor / corrector / residual (propagator.py:77-226);
//      reduce_kernel           its partial sums as a separate pass for many local k
//   K4 finish_kernel           observables, finite check, StepReport row
//   k-sharded ranks exchange the new frontier slice peer-to-peer from K3 (kbe_p2p_*).
//
// Arithmetic is FP64 / complex128, with one exception: a repeated collision evaluation
// at the same frontier (incremental mode, n_k >= 8, KBE_INCR=0 disables it) computes its
// correction M (v - v_full), a term <= 1e-7 of I, in complex64 from a complex64 shadow of
// the history (relative error of I <= 2e-13 worst case, ~1e-14 typical); everything else,
// including the slice-f terms of those evaluations, is FP64.  There is no CPU fallback.

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <math.h>
#include <stdlib.h>

#include <algorithm>
#include <utility>

#include "../../include/kbe200.h"

// timing experiments only (profiles/coll_variants.sh; results are wrong): 1 = no 2x2
// products, 2 = no warp reduction, 3 = no proxy fence before a ring refill, 4 = no row stores
#ifndef KBE_COLL_EXP
#define KBE_COLL_EXP 0
#endif

#define KBE_ABI_VERSION 11

typedef double2 cplx;

// ------------------------------------------------------------------ control
struct kbe_ctl {
    unsigned long long res[KBE_MAX_ITER];  // residual bits per corrector iteration
    int nonfinite[KBE_MAX_ITER];           // frontier non-finite after iteration
    int poisoned;                          // step that produced a non-finite frontier
    int needs_more;                        // step left unconverged by a shortened launch (kbe_run_iters)
    cplx hf_sum[4];                        // k-sum of rho for hf_mode="on"
    unsigned task_next;                    // collision work queue head (reset by the last CTA)
    unsigned task_done;
    unsigned upd_done;                     // update CTAs finished (graph mode; reset by the last CTA)
    int prev_f1;                           // 1 + frontier of the last collision evaluation (0: none)
    int full_f1;                           // 1 + frontier of the last full (FP64) evaluation
    int incr_last;                         // the last evaluation was incremental (K3 adds the delta slots)
    int pad3;
    double dsum;                           // sum of the frontier changes since the last full evaluation
};

static char g_err[512] = "";
static void set_err(const char* what, cudaError_t e) {
    snprintf(g_err, sizeof(g_err), "%s: %s", what, e == cudaSuccess ? "bad argument" : cudaGetErrorString(e));
}
#define KBE_CHECK_LAUNCH(name)                                  \
    do {                                                        \
        cudaError_t e_ = cudaGetLastError();                    \
        if (e_ != cudaSuccess) { set_err(name, e_); return KBE_ERR_CUDA; } \
    } while (0)

// ------------------------------------------------------------------ layout
// Slice s holds points b = 0..s in s/32 + 1 blocks; a block is 8 planes x 32 points
// (4 KB, contiguous), so one bulk copy moves one block of one slice.
// plane_len(s) = padded points per plane; sl_idx(c, b) = element (plane c, point b)
// inside any slice (independent of s).
__host__ __device__ __forceinline__ int64_t plane_len(int s) { return (int64_t)((s >> 5) + 1) << 5; }
__host__ __device__ __forceinline__ int64_t slice_off(int s) {
    const int64_t q = s >> 5, r = s & 31;
    return 256 * (q + 1) * (16 * q + r);   // sum_{s'<s} 8 plane_len(s')
}
__host__ __device__ __forceinline__ int64_t sl_idx(int c, int b) {
    return ((int64_t)(b >> 5) << 8) + (c << 5) + (b & 31);
}

// ------------------------------------------------------------------ complex
__device__ __forceinline__ cplx cz() { return make_double2(0.0, 0.0); }
__device__ __forceinline__ cplx cadd(cplx a, cplx b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ cplx csub(cplx a, cplx b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ cplx cneg(cplx a) { return make_double2(-a.x, -a.y); }
__device__ __forceinline__ cplx cconj(cplx a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ cplx cscale(cplx a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ cplx cmul(cplx a, cplx b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// acc + a*b
__device__ __forceinline__ cplx cfma(cplx a, cplx b, cplx acc) {
    return make_double2(fma(a.x, b.x, fma(-a.y, b.y, acc.x)), fma(a.x, b.y, fma(a.y, b.x, acc.y)));
}
// acc + a*conj(b)
__device__ __forceinline__ cplx cfma_cb(cplx a, cplx b, cplx acc) {
    return make_double2(fma(a.x, b.x, fma(a.y, b.y, acc.x)), fma(a.y, b.x, fma(-a.x, b.y, acc.y)));
}
// acc + conj(a)*b
__device__ __forceinline__ cplx cfma_ca(cplx a, cplx b, cplx acc) {
    return make_double2(fma(a.x, b.x, fma(a.y, b.y, acc.x)), fma(a.x, b.y, fma(-a.y, b.x, acc.y)));
}
// complex64 (the incremental collision evaluations' arithmetic)
typedef float2 fcx;
__device__ __forceinline__ fcx f32(cplx a) { return make_float2((float)a.x, (float)a.y); }
__device__ __forceinline__ cplx f64(fcx a) { return make_double2(a.x, a.y); }
__device__ __forceinline__ fcx cfma(fcx a, fcx b, fcx acc) {
    return make_float2(fmaf(a.x, b.x, fmaf(-a.y, b.y, acc.x)), fmaf(a.x, b.y, fmaf(a.y, b.x, acc.y)));
}
__device__ __forceinline__ fcx cfma_cb(fcx a, fcx b, fcx acc) {
    return make_float2(fmaf(a.x, b.x, fmaf(a.y, b.y, acc.x)), fmaf(a.y, b.x, fmaf(-a.x, b.y, acc.y)));
}
__device__ __forceinline__ fcx cfma_ca(fcx a, fcx b, fcx acc) {
    return make_float2(fmaf(a.x, b.x, fmaf(a.y, b.y, acc.x)), fmaf(a.x, b.y, fmaf(-a.y, b.x, acc.y)));
}
// Packed FP32 (FFMA2, fma.rn.f32x2) complex64 MACs for the incremental collision loop:
// acc += s c with s a streamed history cell and c a task / slice constant.  s's real and
// imaginary parts enter as broadcast scalar operands (free in SASS) and c as the pair
// (c.x, c.y) or its rotation, so one complex MAC is 2 FFMA2 instead of 4 FFMA; the
// rotations of a loop-invariant c are hoisted by the compiler (one negated register).
__device__ __forceinline__ fcx ffma2(fcx a, fcx b, fcx c) {
    unsigned long long A = *reinterpret_cast<unsigned long long*>(&a), B = *reinterpret_cast<unsigned long long*>(&b),
                       C = *reinterpret_cast<unsigned long long*>(&c);
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(C) : "l"(A), "l"(B));
    return *reinterpret_cast<fcx*>(&C);
}
__device__ __forceinline__ fcx bc2(float x) { return make_float2(x, x); }
// acc += s c = s.x (c.x, c.y) + s.y (-c.y, c.x)           (r = (-c.y, c.x) precomputed)
__device__ __forceinline__ fcx cm_sc(fcx s, fcx c, fcx r, fcx acc) { return ffma2(bc2(s.y), r, ffma2(bc2(s.x), c, acc)); }
// acc += conj(s) c = s.x (c.x, c.y) + s.y (c.y, -c.x)     (r = (c.y, -c.x))
__device__ __forceinline__ fcx cm_Sc(fcx s, fcx c, fcx r, fcx acc) { return ffma2(bc2(s.y), r, ffma2(bc2(s.x), c, acc)); }
// acc += s conj(c) = s.x (c.x, -c.y) + s.y (c.y, c.x)
__device__ __forceinline__ fcx cm_sC(fcx s, fcx c, fcx acc) {
    return ffma2(bc2(s.y), make_float2(c.y, c.x), ffma2(bc2(s.x), make_float2(c.x, -c.y), acc));
}
__device__ __forceinline__ fcx rot_p(fcx c) { return make_float2(-c.y, c.x); }   // i c
__device__ __forceinline__ fcx rot_m(fcx c) { return make_float2(c.y, -c.x); }   // -i c
// 2x2 blocks: acc += C S (S streamed), acc += C S^dag, acc += S C^dag, acc += S^dag C, acc += S C
__device__ __forceinline__ void mm2_cs(fcx* acc, const fcx* C, const fcx* Cr, const fcx* S) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int k = 0; k < 2; ++k) acc[2 * i + j] = cm_sc(S[2 * k + j], C[2 * i + k], Cr[2 * i + k], acc[2 * i + j]);
}
__device__ __forceinline__ void mm2_csdag(fcx* acc, const fcx* C, const fcx* Cr, const fcx* S) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int k = 0; k < 2; ++k) acc[2 * i + j] = cm_Sc(S[2 * j + k], C[2 * i + k], Cr[2 * i + k], acc[2 * i + j]);
}
__device__ __forceinline__ void mm2_scdag(fcx* acc, const fcx* S, const fcx* C) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int k = 0; k < 2; ++k) acc[2 * i + j] = cm_sC(S[2 * i + k], C[2 * j + k], acc[2 * i + j]);
}
__device__ __forceinline__ void mm2_sdagc(fcx* acc, const fcx* S, const fcx* C) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int k = 0; k < 2; ++k) acc[2 * i + j] = cm_Sc(S[2 * k + i], C[2 * k + j], rot_m(C[2 * k + j]), acc[2 * i + j]);
}
__device__ __forceinline__ void mm2_sc(fcx* acc, const fcx* S, const fcx* C) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int k = 0; k < 2; ++k) acc[2 * i + j] = cm_sc(S[2 * i + k], C[2 * k + j], rot_p(C[2 * k + j]), acc[2 * i + j]);
}
// Smith's division
__device__ __forceinline__ cplx cdiv(cplx a, cplx b) {
    if (fabs(b.x) >= fabs(b.y)) {
        const double r = b.y / b.x, den = b.x + b.y * r;
        return make_double2((a.x + a.y * r) / den, (a.y - a.x * r) / den);
    }
    const double r = b.x / b.y, den = b.x * r + b.y;
    return make_double2((a.x * r + a.y) / den, (a.y * r - a.x) / den);
}
// -i*dt*z  and  +i*dt*z
__device__ __forceinline__ cplx cmul_mi(cplx z, double dt) { return make_double2(dt * z.y, -dt * z.x); }
__device__ __forceinline__ cplx cmul_pi(cplx z, double dt) { return make_double2(-dt * z.y, dt * z.x); }

// 2x2 complex blocks, row-major: m[0]=00 m[1]=01 m[2]=10 m[3]=11
// (templates over cplx / fcx)
// acc += A*B
template <class C>
__device__ __forceinline__ void mm_acc(C* acc, const C* A, const C* B) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            C t = cfma(A[2 * i], B[j], acc[2 * i + j]);
            acc[2 * i + j] = cfma(A[2 * i + 1], B[2 + j], t);
        }
}
// acc += A*B^dagger : (B^dag)_{kj} = conj(B_{jk})
template <class C>
__device__ __forceinline__ void mm_bdag_acc(C* acc, const C* A, const C* B) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            C t = cfma_cb(A[2 * i], B[2 * j], acc[2 * i + j]);
            acc[2 * i + j] = cfma_cb(A[2 * i + 1], B[2 * j + 1], t);
        }
}
// acc += A^dagger*B : (A^dag)_{ik} = conj(A_{ki})
template <class C>
__device__ __forceinline__ void mm_adag_acc(C* acc, const C* A, const C* B) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            C t = cfma_ca(A[i], B[j], acc[2 * i + j]);
            acc[2 * i + j] = cfma_ca(A[2 + i], B[2 + j], t);
        }
}
// out = A*B
__device__ __forceinline__ void mm(cplx* out, const cplx* A, const cplx* B) {
#pragma unroll
    for (int i = 0; i < 4; ++i) out[i] = cz();
    mm_acc(out, A, B);
}
// out = A*B^dagger
__device__ __forceinline__ void mm_bdag(cplx* out, const cplx* A, const cplx* B) {
#pragma unroll
    for (int i = 0; i < 4; ++i) out[i] = cz();
    mm_bdag_acc(out, A, B);
}
// -(X^dagger): (-X^dag)_{jm} = -conj(X_{mj})
__device__ __forceinline__ void neg_dag(cplx* out, const cplx* X) {
    out[0] = cneg(cconj(X[0]));
    out[1] = cneg(cconj(X[2]));
    out[2] = cneg(cconj(X[1]));
    out[3] = cneg(cconj(X[3]));
}
// (x - x^dagger)/2  (propagator.py:119-120)
__device__ __forceinline__ void antiherm(cplx* out, const cplx* x) {
    cplx t[4];
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int m = 0; m < 2; ++m) {
            const cplx a = x[2 * j + m], b = cconj(x[2 * m + j]);
            t[2 * j + m] = make_double2(0.5 * (a.x - b.x), 0.5 * (a.y - b.y));
        }
#pragma unroll
    for (int i = 0; i < 4; ++i) out[i] = t[i];
}

// ------------------------------------------------------------------ quadrature
// quadrature_weights(nint, dt, kind)[t]  (collision.py:31-61); 0 outside the rule.
__device__ __forceinline__ double quad_w(int nint, int t, double dt, int quad) {
    if (nint <= 0 || t < 0 || t > nint) return 0.0;
    if (quad == 0) return (t == 0 || t == nint) ? 0.5 * dt : dt;
    double w = 0.0;
    int start = 0;
    if (nint & 1) {
        if (t <= 1) w = 0.5 * dt;
        start = 1;
        if (nint == 1) return w;
    }
    if (t < start) return w;
    const int i = t - start, m = nint - start;
    const double c = (i == 0 || i == m) ? 1.0 : ((i & 1) ? 4.0 : 2.0);
    return __dadd_rn(w, __dmul_rn(c, dt / 3.0));
}

// ------------------------------------------------------------------ device-side convergence
// Every later launch is a no-op once a step poisoned the state or a shortened step
// (kbe_run_iters) stopped unconverged; the host resumes the latter (kbe_resume_step).
__device__ __forceinline__ bool kbe_halted(const kbe_ctl* ctl) {
    return *(const volatile int*)&ctl->poisoned || *(const volatile int*)&ctl->needs_more;
}
// k-sharded ranks: every rank's all-gather chunk is its new G slice for the local k
// followed by a 256-byte control tail (its local residual bits and non-finite flags per
// iteration), so one all-gather per iteration also carries the convergence record and
// every rank takes the max over ranks itself (no separate all-reduce).
#define KBE_TAIL_CPLX 16
struct KbeTail {
    unsigned long long res[KBE_MAX_ITER];
    int nonfinite[KBE_MAX_ITER];
};
static_assert(sizeof(KbeTail) <= KBE_TAIL_CPLX * sizeof(cplx), "control tail");
__host__ __device__ __forceinline__ int64_t front_chunk(const kbe_problem& P) {
    return (int64_t)(P.k_hi - P.k_lo) * 8 * plane_len(P.n_steps) + KBE_TAIL_CPLX;
}
// v_prev: the G (which = 0) and Sigma (1) frontier slices of local k as the last
// collision evaluation used them (incremental evaluations, see collision_kernel)
__device__ __forceinline__ int64_t vprev_off(const kbe_problem& P, int kl, int which) {
    return ((int64_t)kl * 2 + which) * 8 * plane_len(P.n_steps);
}

// Peer-to-peer exchange (p2p_world > 1, kbe_p2p_* in include/kbe200.h): every rank owns
// one buffer [2 parities][ranks][chunk] + flags[ranks] + epoch.  The update kernel
// writes its new slice and control tail straight into every peer's buffer over
// NVLink (parity of the next data epoch), and its last CTA bumps the local epoch and
// release-stores it into flags[me] of every peer.  A consumer waits until all flags
// reach its local epoch (acquire) and reads the chunks of that epoch's parity.
// Double buffering makes the overwrite safe: a rank publishes epoch e+1 only after
// its Sigma waited for every rank's epoch e, i.e. after every rank finished reading
// epoch e-1 (same parity).
__host__ __device__ __forceinline__ bool sharded(const kbe_problem& P) { return P.front_all || P.p2p_world > 1; }
__device__ __forceinline__ unsigned long long* p2p_flags(const kbe_problem& P, void* base) {
    return (unsigned long long*)((cplx*)base + 2 * (int64_t)P.p2p_world * front_chunk(P));
}
__device__ __forceinline__ unsigned long long p2p_epoch(const kbe_problem& P) {
    return *(volatile unsigned long long*)(p2p_flags(P, P.p2p_local) + P.p2p_world);
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// chunks of the current data epoch (gathered by NCCL, or by peers' stores)
__device__ __forceinline__ const cplx* front_base(const kbe_problem& P) {
    if (P.p2p_world > 1)
        return (const cplx*)P.p2p_local + (int64_t)(p2p_epoch(P) & 1) * P.p2p_world * front_chunk(P);
    return (const cplx*)P.front_all;
}
// where rank `me` writes its chunk in peer r's buffer for data epoch e
__device__ __forceinline__ cplx* p2p_dst(const kbe_problem& P, int r, unsigned long long e) {
    return (cplx*)P.p2p_peers[r] + ((int64_t)(e & 1) * P.p2p_world + P.p2p_rank) * front_chunk(P);
}
// consumer side: block until every rank has published the local epoch
// Watchdog: a peer that never publishes (a crashed rank, a broken peer mapping) must not
// hang the GPU.  After KBE_P2P_TIMEOUT_NS the waiter gives up and raises the timeout
// word (flags[world + 1]); the host checks it and raises (propagator._PeerExchange).
#ifndef KBE_P2P_TIMEOUT_NS
#define KBE_P2P_TIMEOUT_NS 20000000000ull
#endif
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __noinline__ void p2p_wait_ranks(unsigned long long* flags, int world) {
    if (threadIdx.x == 0) {
        const unsigned long long e = *(volatile const unsigned long long*)(flags + world);
        const unsigned long long t0 = globaltimer_ns();
        for (int r = 0; r < world; ++r)
            while (ld_acquire_sys(flags + r) < e) {
                if (*(volatile unsigned long long*)(flags + world + 1)) return;   // already timed out
                if (globaltimer_ns() - t0 > KBE_P2P_TIMEOUT_NS) {
                    *(volatile unsigned long long*)(flags + world + 1) = 1ull + r;
                    __threadfence_system();
                    return;
                }
                __nanosleep(256);
            }
    }
}
__device__ __forceinline__ void p2p_wait(const kbe_problem& P) {
    if (P.p2p_world <= 1) return;
    p2p_wait_ranks((unsigned long long*)p2p_flags(P, P.p2p_local), P.p2p_world);
    __syncthreads();
}
// producer side (one thread, after every CTA's stores were fenced): epoch + 1 everywhere
// (rank loops are unrolled to KBE_MAX_RANKS so that p2p_peers[] is indexed by
// constants; a runtime index into a kernel parameter forces a local copy of it)
__device__ __forceinline__ void p2p_signal(const kbe_problem& P, unsigned long long e) {
    __threadfence_system();
    *(volatile unsigned long long*)(p2p_flags(P, P.p2p_local) + P.p2p_world) = e;
#pragma unroll
    for (int r = 0; r < KBE_MAX_RANKS; ++r)
        if (r < P.p2p_world) st_release_sys(p2p_flags(P, P.p2p_peers[r]) + P.p2p_rank, e);
}
__device__ __forceinline__ const KbeTail* rank_tail(const kbe_problem& P, int r) {
    return (const KbeTail*)(front_base(P) + r * front_chunk(P) + front_chunk(P) - KBE_TAIL_CPLX);
}
// residual bits / non-finite flag of iteration i over all ranks.  The multi-rank paths
// are out of line: inlined, their loops cost the hot kernels registers.
// (scalar arguments only: a kernel-parameter struct passed by reference would be copied
// to local memory)
__device__ __noinline__ unsigned long long res_bits_ranks(const cplx* base, int64_t chunk, int R, int i) {
    unsigned long long m = 0;
    for (int r = 0; r < R; ++r) m = max(m, ((const KbeTail*)(base + r * chunk + chunk - KBE_TAIL_CPLX))->res[i]);
    return m;
}
__device__ __noinline__ int nonfinite_ranks(const cplx* base, int64_t chunk, int R, int i) {
    int f = 0;
    for (int r = 0; r < R; ++r) f |= ((const KbeTail*)(base + r * chunk + chunk - KBE_TAIL_CPLX))->nonfinite[i];
    return f;
}
__device__ __forceinline__ unsigned long long res_bits(const kbe_problem& P, const kbe_ctl* ctl, int i) {
    return sharded(P) ? res_bits_ranks(front_base(P), front_chunk(P), P.n_k / (P.k_hi - P.k_lo), i)
                      : ((const volatile unsigned long long*)ctl->res)[i];
}
__device__ __forceinline__ int nonfinite_at(const kbe_problem& P, const kbe_ctl* ctl, int i) {
    return sharded(P) ? nonfinite_ranks(front_base(P), front_chunk(P), P.n_k / (P.k_hi - P.k_lo), i)
                      : ctl->nonfinite[i];
}
__device__ __forceinline__ bool kbe_skip(const kbe_problem& P, const kbe_ctl* ctl, int it) {
    if (kbe_halted(ctl)) return true;
    for (int i = 0; i < it; ++i)
        if (__longlong_as_double((long long)res_bits(P, ctl, i)) <= P.eps) return true;
    return false;
}

// ------------------------------------------------------------------ programmatic dependent launch
// Step kernels are launched with programmatic stream serialization: the next
// kernel's CTAs are scheduled while this one runs (hiding launch latency) and
// block in griddepcontrol.wait until it has completed and flushed memory.  Every
// step kernel therefore waits before its first dependent read (the control block
// included) and triggers its dependents right away.
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ------------------------------------------------------------------ warp reduction
// Sum 8 values over the 32 lanes with a reduce-scatter butterfly (9 shuffles);
// lane L ends up holding the total of value index (L >> 2) & 7.
template <class T>
__device__ __forceinline__ T warp_rs8(const T* v, int lane) {
    const bool h4 = lane & 16, h3 = lane & 8, h2 = lane & 4;
    T a[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const T send = h4 ? v[i] : v[i + 4];
        const T keep = h4 ? v[i + 4] : v[i];
        a[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
    T c[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const T send = h3 ? a[i] : a[i + 2];
        const T keep = h3 ? a[i + 2] : a[i];
        c[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    const T send = h2 ? c[0] : c[1];
    const T keep = h2 ? c[1] : c[0];
    T d = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    d += __shfl_xor_sync(0xffffffffu, d, 2);
    d += __shfl_xor_sync(0xffffffffu, d, 1);
    return d;
}

// =================================================================== K1: Sigma
// Second-Born Sigma for one pair, factorised (SURVEY finding 4):
//   P_jm(q)   = sum_k' gp_jm((k'+q-h) mod n) gr_mj(k')          (selfenergy.py:59-94)
//   S1_jm(k)  = pref sum_q P_{j'm'}(q) gp_jm((k-q+h) mod n)      (selfenergy.py:104-136)
//   X_jm(d)   = sum_q gr_{m'j'}((d+q) mod n) gp_{j'm}(q)
//   S2_jm(k)  = pref sum_k' gp_{jm'}(k') X_jm((k'-k) mod n)
//             = pref sum_{k',q} gp_{jm'}(k') gr_{m'j'}(k'+q-k) gp_{j'm}(q)   (selfenergy.py:139-203)
// Shared-memory operands are planar: gp[jm * nk + k]; P and X likewise [jm][q].
__device__ __forceinline__ int fold(int t, int n) { return t < 0 ? t + n : (t >= n ? t - n : t); }

__device__ __forceinline__ cplx sig_pol(const cplx* gp, const cplx* gr, int nk, int jm, int q) {
    const int j = jm >> 1, m = jm & 1, h = nk >> 1;
    const cplx* a = gp + jm * nk;
    const cplx* c = gr + (m * 2 + j) * nk;
    cplx acc = cz();
    for (int kp = 0; kp < nk; ++kp) acc = cfma(a[fold(kp + q - h, nk)], c[kp], acc);
    return acc;
}
__device__ __forceinline__ cplx sig_x(const cplx* gp, const cplx* gr, int nk, int jm, int d) {
    const int j = jm >> 1, m = jm & 1;
    const cplx* a = gr + ((1 - m) * 2 + (1 - j)) * nk;
    const cplx* c = gp + ((1 - j) * 2 + m) * nk;
    cplx acc = cz();
    for (int q = 0; q < nk; ++q) acc = cfma(a[fold(d + q, nk)], c[q], acc);
    return acc;
}
__device__ __forceinline__ cplx sig_s1(const cplx* Pm, const cplx* gp, int nk, int jm, int k) {
    const int h = nk >> 1;
    const cplx* a = Pm + (3 - jm) * nk;   // P_{(1-j)(1-m)}
    const cplx* c = gp + jm * nk;
    cplx acc = cz();
    for (int q = 0; q < nk; ++q) acc = cfma(a[q], c[fold(k - q + h, nk)], acc);
    return acc;
}
__device__ __forceinline__ cplx sig_s2(const cplx* gp, const cplx* Xm, int nk, int jm, int k) {
    const int j = jm >> 1, m = jm & 1;
    const cplx* a = gp + (j * 2 + (1 - m)) * nk;
    const cplx* c = Xm + jm * nk;
    cplx acc = cz();
    for (int kp = 0; kp < nk; ++kp) acc = cfma(a[kp], c[fold(kp - k, nk)], acc);
    return acc;
}

// ---- K1 on the step frontier: register-blocked circular correlations ----------------
// Every stage of the factorised Sigma is a length-n_k circular correlation
//   out[r] = sum_t C[t] A[(a0 + DT t + DR r) mod n_k],  r = 0..R-1,
// with C walked in lock-step by all lanes of a correlation (a shared-memory
// broadcast) and A read through a sliding window of R registers: one new A element
// per t feeds R complex FMAs.  A operands are stored "unrolled" (duplicated past
// n_k with the rotation the stage needs) so no index wraps, and padded by one
// element every 8 (sg_pad) so that lanes R elements apart hit distinct banks.
// R = 4 (2 when 4 does not divide n_k) keeps the FP64 pipe, not shared memory,
// the limiter: per t a warp issues 4R DFMA and two loads.
__host__ __device__ __forceinline__ int sg_pad(int j) { return j + (j >> 3); }
__host__ __device__ __forceinline__ int sg_r(int nk) { return (nk & 3) ? 2 : 4; }
// half-pair = (pair b, component); shared-memory layout (complex elements):
//   DG[4][LDG]  gp_jm: DG[jm][pad(j)] = gp_jm[(j - h) mod n_k], j < 2 n_k + h
//   DR[4][LDG]  gr_jm, same rotation
//   PM[4][LDP]  P_jm(q) at pad(q)
//   DX[4][LDX]  X_jm:  DX[jm][pad(j)] = X_jm[j mod n_k], j <= 2 n_k
//   S1[4][LDP]  pref * Sigma1 of the local k (stage-2 hand-off)
struct SgDims {
    int nk, h, R, ldg, ldp, ldx, per;   // per = complex elements per half-pair
    __host__ __device__ SgDims(int n_k) : nk(n_k), h(n_k >> 1), R(sg_r(n_k)) {
        ldg = sg_pad(2 * nk + h - 1) + 1;
        ldp = sg_pad(nk - 1) + 1;
        ldx = sg_pad(2 * nk) + 1;
        per = 8 * ldg + 8 * ldp + 4 * ldx;
    }
};
// half-pairs per CTA: 256 threads over 8 n_k / R stage-1 tasks each
__host__ __device__ __forceinline__ int sigma_hp_per_block(int nk) {
    const int t = 8 * nk / sg_r(nk);
    return t >= 256 ? 1 : 256 / t;
}
// half-pairs per CTA for a launch with `hps` half-pairs: fewer than the thread budget
// allows when that keeps >= 2 CTAs per SM (small frontiers / small n_k are latency-bound)
static int sigma_hb_launch(int nk, int hps, int sms) {
    int hb = sigma_hp_per_block(nk);
    const int t = 8 * nk / sg_r(nk);              // stage-1 tasks per half-pair
    const int floor_hb = t >= 64 ? 1 : 64 / t;    // keep >= 64 busy threads per CTA
    while (hb > floor_hb && (hps + hb - 1) / hb < 2 * sms) hb >>= 1;
    return hb;
}
#define SIGMA_THREADS 256
#ifndef KBE_SIG_NT256
#define KBE_SIG_NT256 0   // 1: always 256-thread K1 CTAs (A/B switch)
#endif

template <int R, int DT, int DR>
__device__ __forceinline__ void sg_corr(const cplx* __restrict__ A, int a0, const cplx* __restrict__ C, int c0, int nk,
                                        cplx* acc) {
    cplx w[R];
#pragma unroll
    for (int r = 0; r < R; ++r) w[r] = A[sg_pad(a0 + DR * r)];
    for (int t0 = 0; t0 < nk; t0 += R) {
#pragma unroll
        for (int u = 0; u < R; ++u) {
            const int t = t0 + u;
            const cplx c = C[sg_pad(c0 + t)];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int slot = (DT == DR) ? (r + u) % R : ((r - u) % R + R) % R;
                acc[r] = cfma(w[slot], c, acc[r]);
            }
            // slide to t+1: the element that left the window is replaced by the new one
            if (DT == DR) w[u] = A[sg_pad(a0 + DT * (t + 1) + DR * (R - 1))];
            else w[R - 1 - u] = A[sg_pad(a0 + DT * (t + 1))];
        }
    }
}

// K1: both components of Sigma on the step-n frontier (evaluate_sigma_batched,
// selfenergy.py:261-325).  Pair b uses G<(t_b,t_n) and G>(t_n,t_b), read from the
// G frontier slice n for ALL k (gathered buffer on >1 rank).
//   lesser  (primary G<(b,n), reversed G>(n,b)) -> S<(t_b,t_n) = upper planes 4..7
//   greater (primary G>(n,b), reversed G<(b,n)) -> S>(t_n,t_b) = lower planes 0..3
// One CTA = HB half-pairs (pair, component; sigma_hb_launch); stage 1 computes
// P and X (selfenergy.py:59-94 and the inner sum of 139-203), stage 2 Sigma1 and
// Sigma2 for the local k (selfenergy.py:104-136, 139-203), Sigma = Sigma1 - Sigma2.
// NT threads per CTA: 256, or 128 when the launch's half-pairs per CTA need no more
// (small n_k): no idle half of the CTA, twice the CTAs per SM
template <int R, int NT>
__global__ void __launch_bounds__(NT, 512 / NT) sigma_frontier_kernel(kbe_problem P, int n, int it, int HB) {
    pdl_enter();
    const kbe_ctl* ctl = (const kbe_ctl*)P.ctl;
    p2p_wait(P);   // the frontier and the control tails of the last update, all ranks
    if (kbe_skip(P, ctl, it)) return;
    extern __shared__ cplx sm[];
    const int nk = P.n_k;
    const SgDims D(nk);
    const int h = D.h;
    const int hp0 = blockIdx.x * HB;
    const int nhp = min(HB, 2 * (n + 1) - hp0);
    const int nloc = P.k_hi - P.k_lo;
    const int tid = threadIdx.x;

    // frontier source: [k][8 planes][stride]
    // gathered buffer: rank chunks of [k_local][capacity slice] + control tail
    const cplx* src;
    int64_t kstride, rstride;
    const int kper = sharded(P) ? nloc : nk;
    if (sharded(P)) {
        src = front_base(P);
        kstride = 8 * plane_len(P.n_steps);
        rstride = front_chunk(P);
    } else {
        src = (const cplx*)P.g_hist + slice_off(n);
        kstride = P.tri;
        rstride = 0;
    }
    // stage 0: V1 = G<(b,n) = -L(n,b)^dag (b<n) | L(n,n);  V2 = G>(n,b) = -U(n,b)^dag | U(n,n)
    // comp 0: gp = V1, gr = V2;  comp 1: gp = V2, gr = V1 (each half-pair loads both).
    for (int i = tid; i < nhp * 8 * nk; i += NT) {
        const int p = i % nhp, c = (i / nhp) & 7, k = i / (nhp * 8);
        const int hp = hp0 + p, b = hp >> 1, comp = hp & 1;
        const int cc = c & 3;
        const cplx v = __ldg(src + (k / kper) * rstride + (k % kper) * kstride + sl_idx(c, b));
        const cplx x = b < n ? cneg(cconj(v)) : v;
        const int jm = b < n ? ((cc & 1) * 2 + (cc >> 1)) : cc;
        const bool is_gp = (c < 4) == (comp == 0);
        cplx* dst = sm + (int64_t)p * D.per + (is_gp ? 0 : 4 * D.ldg) + jm * D.ldg;
        const int j = k + h;
        dst[sg_pad(j)] = x;
        dst[sg_pad(j + nk)] = x;
        if (j >= nk) dst[sg_pad(j - nk)] = x;
    }
    __syncthreads();

    // stage 1: P_jm(q) (f < 4) and X_jm(d) (f >= 4), R consecutive outputs per task
    const int NB = nk / R;
    for (int task = tid; task < nhp * 8 * NB; task += NT) {
        const int p = task / (8 * NB), f = (task / NB) & 7, blk = task % NB;
        cplx* base = sm + (int64_t)p * D.per;
        const cplx* DG = base;
        const cplx* DRr = base + 4 * D.ldg;
        cplx* PM = base + 8 * D.ldg;
        cplx* DX = PM + 4 * D.ldp;
        const int jm = f & 3, j = jm >> 1, m = jm & 1, o0 = blk * R;
        cplx acc[R];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = cz();
        if (f < 4) {   // P_jm(q) = sum_t gp_jm[t+q-h] gr_mj[t]
            sg_corr<R, 1, 1>(DG + jm * D.ldg, o0, DRr + (m * 2 + j) * D.ldg, h, nk, acc);
#pragma unroll
            for (int r = 0; r < R; ++r) PM[jm * D.ldp + sg_pad(o0 + r)] = acc[r];
        } else {       // X_jm(d) = sum_t gr_{m'j'}[d+t] gp_{j'm}[t]
            sg_corr<R, 1, 1>(DRr + ((1 - m) * 2 + (1 - j)) * D.ldg, o0 + h, DG + ((1 - j) * 2 + m) * D.ldg, h, nk, acc);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                DX[jm * D.ldx + sg_pad(o0 + r)] = acc[r];
                DX[jm * D.ldx + sg_pad(o0 + r + nk)] = acc[r];
            }
            if (o0 == 0) DX[jm * D.ldx + sg_pad(2 * nk)] = acc[0];
        }
    }
    __syncthreads();

    // stage 2: Sigma1 (which = 0) and Sigma2 (which = 1) for R consecutive local k
    const int NBL = (nloc + R - 1) / R;
    const double inv2 = 1.0 / ((double)nk * (double)nk);
    cplx s2v[R];
    int s2_task = -1;
    for (int task = tid; task < nhp * 8 * NBL; task += NT) {
        const int p = task / (8 * NBL), which = (task / (4 * NBL)) & 1, jm = (task / NBL) & 3, blk = task % NBL;
        const int hp = hp0 + p, b = hp >> 1;
        cplx* base = sm + (int64_t)p * D.per;
        const cplx* DG = base;
        const cplx* PM = base + 8 * D.ldg;
        const cplx* DX = PM + 4 * D.ldp;
        cplx* S1 = (cplx*)DX + 4 * D.ldx;
        const int j = jm >> 1, m = jm & 1;
        const int k0 = min(P.k_lo + blk * R, nk - R);   // global k of output r = 0
        const double pref = (P.u_table[b] * P.u_table[n]) * inv2;
        cplx acc[R];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = cz();
        if (which == 0) {   // S1_jm(k) = sum_t P_{j'm'}[t] gp_jm[k-t+h]
            sg_corr<R, -1, 1>(DG + jm * D.ldg, k0 + nk, PM + (3 - jm) * D.ldp, 0, nk, acc);
#pragma unroll
            for (int r = 0; r < R; ++r) S1[jm * D.ldp + sg_pad(k0 + r)] = cscale(acc[r], pref);
        } else {            // S2_jm(k) = sum_t gp_{jm'}[t] X_jm[t-k]
            sg_corr<R, 1, -1>(DX + jm * D.ldx, nk - k0, DG + (j * 2 + (1 - m)) * D.ldg, h, nk, acc);
#pragma unroll
            for (int r = 0; r < R; ++r) s2v[r] = cscale(acc[r], pref);
            s2_task = task;
        }
    }
    __syncthreads();
    if (s2_task >= 0) {   // one stage-2 task per thread at most (8 NBL <= 256 per half-pair)
        const int task = s2_task;
        const int p = task / (8 * NBL), jm = (task / NBL) & 3, blk = task % NBL;
        const int hp = hp0 + p, b = hp >> 1, comp = hp & 1;
        const cplx* S1 = sm + (int64_t)p * D.per + 8 * D.ldg + 4 * D.ldp + 4 * D.ldx;
        const int k0 = min(P.k_lo + blk * R, nk - R);
        const int lo = P.k_lo + blk * R, hi = min(P.k_lo + (blk + 1) * R, P.k_hi);
        const int plane = comp == 0 ? 4 + jm : jm;
        cplx* dst = (cplx*)P.s_hist + slice_off(n) + sl_idx(plane, b);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int k = k0 + r;
            if (k >= lo && k < hi) dst[(int64_t)(k - P.k_lo) * P.tri] = csub(S1[jm * D.ldp + sg_pad(k)], s2v[r]);
        }
    }
}

// ---- K1 in Fourier space (n_k a power of two) -----------------------------------------
// With the DFT  x^(f) = sum_k x[k] w^{-fk}  (w = e^{2 pi i / n_k}) every stage of the
// factorised Sigma above is a pointwise product (h = n_k/2 shifts give (-1)^f factors
// that cancel pairwise):
//   P^_jm(f)  = (-1)^f gp^_jm(f) gr^_mj(-f)              S1^_jm(f) = pref (-1)^f P^_{j'm'}(f) gp^_jm(f)
//   X^_jm(f)  = gr^_{m'j'}(f) gp^_{j'm}(-f)              S2^_jm(f) = pref gp^_{jm'}(f) X^_jm(-f)
// so
//   Sigma^_jm(f) = pref gr^_{m'j'}(-f) [gp^_{j'm'}(f) gp^_jm(f) - gp^_{jm'}(f) gp^_{j'm}(f)]
//                = pref s_jm det(gp^(f)) gr^_{m'j'}(-f),   s_jm = +1 (j = m), -1 (j != m)
// (SURVEY probe P7: the FFT form equals sigma_slice to <= 7e-16).  Per pair b both
// components use the same 8 vectors V1 = G<(t_b,t_n), V2 = G>(t_n,t_b) (comp 0: gp = V1,
// gr = V2; comp 1 swapped), so one pair costs 8 forward and 8 inverse length-n_k FFTs,
// O(n_k log n_k), instead of the 32 n_k^2 complex MACs of the correlations.  The kernel
// is then bound by moving the G frontier slice in and the Sigma slice out.
// One CTA = PB consecutive pairs (coalesced 16 B x PB runs per (k, plane)); shared
// memory holds PB x 8 lines of n_k complex values.  Each length-n_k transform is a
// four-step FFT, n_k = R1 R2 (R1 = 2^ceil(LG/2), R2 = 2^floor(LG/2)), n = R2 n1 + n2,
// f = f1 + R1 f2:
//   pass 1 (one thread per (line, n2)): R1-point DFT over n1 in registers, times
//          w^{-f1 n2}, written back in place (position R2 f1 + n2);
//   pass 2 (one thread per (line, f1)): R2-point DFT over n2 in registers, written to
//          the natural position f1 + R1 f2.
// Two shared-memory round trips per transform instead of log2(n_k) radix-2 stages; the
// input and output are in natural order, so the pointwise phase pairs f with n_k - f
// directly.  Lines are padded by one slot per R2 (pad()) so that pass 2's stride-R2 reads
// hit distinct banks.
__host__ __device__ __forceinline__ bool sigma_fft_ok(int nk) { return nk >= 2 && nk <= KBE_MAX_NK && !(nk & (nk - 1)); }
__host__ __device__ constexpr int fft_r1(int lg) { return 1 << ((lg + 1) / 2); }
__host__ __device__ constexpr int fft_r2(int lg) { return 1 << (lg / 2); }
__host__ __device__ __forceinline__ int fft_pad(int i, int lg) { return fft_r2(lg) >= 4 ? i + (i >> (lg / 2)) : i; }
// line stride: >= the padded length, = R2 mod 8 when a quarter-warp spans several lines
// in pass 1 (R2 threads per line), so their slots fall in distinct banks
__host__ __device__ __forceinline__ int fft_ls(int lg) {
    const int len = fft_pad((1 << lg) - 1, lg) + 1, r2 = fft_r2(lg);
    return ((len + 7) & ~7) + (r2 < 8 ? r2 : 1);
}
static size_t sigma_fft_smem(int nk, int pb) {
    // twiddles + lines + the two scaled determinants per (pair, frequency)
    int lg = 0;
    while ((1 << lg) < nk) ++lg;
    return ((size_t)pb * 8 * fft_ls(lg) + nk + (size_t)pb * 2 * nk) * sizeof(cplx);
}
// pairs per CTA: at most one pointwise item (pair, frequency) per thread (PB n_k <= 256,
// PB <= 32); the smallest PB whose grid still fits one wave of resident CTAs
// (__launch_bounds__: 3 per SM, 2 at n_k = 128): a CTA's phases are latency-bound, so
// more CTAs in flight help until a second, nearly empty wave would start
static int sigma_fft_pb(int nk, int npairs, int sms) {
    int pb = SIGMA_THREADS / nk;
    pb = pb > 32 ? 32 : (pb < 1 ? 1 : pb);
    const int occ = nk >= 128 ? 2 : 3;
    while (pb > 1 && (npairs + pb / 2 - 1) / (pb / 2) <= occ * sms) pb >>= 1;
    return pb;
}
__host__ __device__ constexpr int brev_c(int i, int bits) {
    int r = 0;
    for (int b = 0; b < bits; ++b) r |= ((i >> b) & 1) << (bits - 1 - b);
    return r;
}
// R-point DFT of v in registers (R <= 16), natural order in and out; tw[j * ts] = w_R^{-j}
// (conjugated for the inverse).  Radix-2 decimation in frequency with compile-time
// indices, then the bit-reversal as register renaming.
template <int R, bool INV>
__device__ __forceinline__ void dft_small(cplx* v, const cplx* tw, int ts) {
#pragma unroll
    for (int s = R / 2; s >= 1; s >>= 1) {
#pragma unroll
        for (int j = 0; j < R / 2; ++j) {
            const int r = j % s, a = (j / s) * 2 * s + r, b = a + s;
            const cplx x = v[a], y = v[b];
            v[a] = cadd(x, y);
            const cplx d = csub(x, y);
            if (r == 0) {
                v[b] = d;
            } else {
                const cplx w = tw[r * (R / (2 * s)) * ts];
                v[b] = cmul(d, INV ? cconj(w) : w);
            }
        }
    }
    constexpr int bits = R == 16 ? 4 : R == 8 ? 3 : R == 4 ? 2 : R == 2 ? 1 : 0;
#pragma unroll
    for (int i = 0; i < R; ++i) {
        const int j = brev_c(i, bits);
        if (j > i) { const cplx t = v[i]; v[i] = v[j]; v[j] = t; }
    }
}
// one transform of every line (forward or inverse), natural order in place
template <int LG, bool INV>
__device__ __forceinline__ void fft_lines(cplx* dat, const cplx* tw, int nlines) {
    constexpr int NK = 1 << LG, R1 = fft_r1(LG), R2 = fft_r2(LG);
    const int LS = fft_ls(LG), tid = threadIdx.x;
    // pass 1: (line, n2) tasks, in place
    for (int t = tid; t < nlines * R2; t += SIGMA_THREADS) {
        cplx* L = dat + (t / R2) * LS;
        const int n2 = t % R2;
        cplx v[R1];
#pragma unroll
        for (int n1 = 0; n1 < R1; ++n1) v[n1] = L[fft_pad(R2 * n1 + n2, LG)];
        dft_small<R1, INV>(v, tw, NK / R1);
#pragma unroll
        for (int f1 = 1; f1 < R1; ++f1) {
            if (R2 > 1 && n2) {
                const cplx w = tw[(f1 * n2) & (NK - 1)];
                v[f1] = cmul(v[f1], INV ? cconj(w) : w);
            }
        }
#pragma unroll
        for (int f1 = 0; f1 < R1; ++f1) L[fft_pad(R2 * f1 + n2, LG)] = v[f1];
    }
    __syncthreads();
    if (R2 == 1) return;
    // pass 2: (line, f1) tasks, all reads before the writes; T2 per thread at most
    // (8 PB R1 with PB <= min(32, 256 / n_k), sigma_fft_pb)
    constexpr int PBMAX = 256 / NK < 32 ? 256 / NK : 32;
    constexpr int T2 = 8 * PBMAX * R1 / SIGMA_THREADS > 1 ? 8 * PBMAX * R1 / SIGMA_THREADS : 1;
    cplx v[T2][R2];
#pragma unroll
    for (int u = 0; u < T2; ++u) {
        const int t = tid + u * SIGMA_THREADS;
        if (t < nlines * R1) {
            const cplx* L = dat + (t / R1) * LS;
            const int f1 = t % R1;
#pragma unroll
            for (int n2 = 0; n2 < R2; ++n2) v[u][n2] = L[fft_pad(R2 * f1 + n2, LG)];
        }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < T2; ++u) {
        const int t = tid + u * SIGMA_THREADS;
        if (t < nlines * R1) {
            cplx* L = dat + (t / R1) * LS;
            const int f1 = t % R1;
            dft_small<R2, INV>(v[u], tw, NK / R2);
#pragma unroll
            for (int f2 = 0; f2 < R2; ++f2) L[fft_pad(f1 + R1 * f2, LG)] = v[u][f2];
        }
    }
    __syncthreads();
}
__host__ __device__ __forceinline__ int ilog2(int v) { int l = 0; while ((1 << (l + 1)) <= v) ++l; return l; }
template <int LG>
__global__ void __launch_bounds__(SIGMA_THREADS, LG >= 7 ? 2 : 3) sigma_fft_kernel(kbe_problem P, int n, int it, int PB) {
    pdl_enter();
    const kbe_ctl* ctl = (const kbe_ctl*)P.ctl;
    p2p_wait(P);   // the frontier and the control tails of the last update, all ranks
    if (kbe_skip(P, ctl, it)) return;
    extern __shared__ cplx sm[];
    constexpr int NK = 1 << LG;
    const int LPB = ilog2(PB), LS = fft_ls(LG);
    cplx* tw = sm;                        // w^{-j}, j < n_k
    cplx* dat = sm + NK;                  // [PB * 8 lines][LS]
    cplx* det = dat + PB * 8 * LS;        // [PB][2][n_k]: c det V1^(f), c det V2^(f)
    const int b0 = blockIdx.x * PB, np = min(PB, n + 1 - b0);
    const int nloc = P.k_hi - P.k_lo;
    const int tid = threadIdx.x;
    for (int j = tid; j < NK; j += SIGMA_THREADS) {
        double sn, cs;
        sincospi(-2.0 * (double)j / (double)NK, &sn, &cs);
        tw[j] = make_double2(cs, sn);
    }
    // gather: line p*8 + v holds V1_jm (v = jm) or V2_jm (v = 4 + jm) of pair b0 + p
    //   V1 = G<(b,n) = -L(n,b)^dag (b < n) | L(n,n);  V2 = G>(n,b) = -U(n,b)^dag | U(n,n)
    // (p fastest: PB consecutive points of one plane are contiguous)
    {
        const bool sh = sharded(P);
        // gathered buffer (k-shards): rank chunks of [k_local][capacity slice] + control tail
        const cplx* src = sh ? front_base(P) : (const cplx*)P.g_hist + slice_off(n);
        const int64_t kstride = sh ? 8 * plane_len(P.n_steps) : P.tri, rstride = sh ? front_chunk(P) : 0;
        const int kper = sh ? nloc : NK;
        for (int i = tid; i < (8 * NK) << LPB; i += SIGMA_THREADS) {
            const int p = i & (PB - 1), c = (i >> LPB) & 7, k = i >> (LPB + 3);
            if (p >= np) continue;
            const int b = b0 + p, cc = c & 3;
            const int kr = sh ? k / kper : 0, kk = sh ? k - kr * kper : k;
            const cplx v = __ldg(src + kr * rstride + kk * kstride + sl_idx(c, b));
            const int jm = b < n ? ((cc & 1) * 2 + (cc >> 1)) : cc;
            dat[(p * 8 + (c & 4) + jm) * LS + fft_pad(k, LG)] = b < n ? cneg(cconj(v)) : v;
        }
    }
    __syncthreads();
    fft_lines<LG, false>(dat, tw, np * 8);
    // pointwise Sigma^ (natural order): dets at f, then every thread reads its partner
    // -f = n_k - f before any thread overwrites its own f (comp 0 -> lines 0..3,
    // comp 1 -> lines 4..7)
    const double inv3 = 1.0 / ((double)NK * (double)NK * (double)NK);
    const double un = P.u_table[n];
    const bool act = tid < np * NK;
    const int p = act ? tid >> LG : 0, q = act ? tid & (NK - 1) : 0;
    const int pq = fft_pad(q, LG), pg = fft_pad((NK - q) & (NK - 1), LG);
    if (act) {
        const cplx* L = dat + p * 8 * LS + pq;
        const double c = (P.u_table[b0 + p] * un) * inv3;
        const cplx d1 = csub(cmul(L[0], L[3 * LS]), cmul(L[LS], L[2 * LS]));
        const cplx d2 = csub(cmul(L[4 * LS], L[7 * LS]), cmul(L[5 * LS], L[6 * LS]));
        det[(p * 2) * NK + q] = cscale(d1, c);
        det[(p * 2 + 1) * NK + q] = cscale(d2, c);
    }
    __syncthreads();
    {
        cplx m1[4], m2[4];
        if (act) {
            const cplx* L = dat + p * 8 * LS + pg;
#pragma unroll
            for (int v = 0; v < 4; ++v) { m1[v] = L[v * LS]; m2[v] = L[(4 + v) * LS]; }
        }
        __syncthreads();
        if (act) {
            cplx* L = dat + p * 8 * LS + pq;
            const cplx d1 = det[(p * 2) * NK + q], d2 = det[(p * 2 + 1) * NK + q];
#pragma unroll
            for (int jm = 0; jm < 4; ++jm) {
                const int o = jm == 0 ? 3 : (jm == 3 ? 0 : jm);   // (m'j') of (jm)
                cplx s0 = cmul(d1, m2[o]), s1 = cmul(d2, m1[o]);
                if (jm == 1 || jm == 2) { s0 = cneg(s0); s1 = cneg(s1); }
                L[jm * LS] = s0;
                L[(4 + jm) * LS] = s1;
            }
        }
    }
    __syncthreads();
    fft_lines<LG, true>(dat, tw, np * 8);
    // comp 0 (lines 0..3) -> S<(t_b,t_n) = upper planes 4..7; comp 1 -> S>(t_n,t_b) = planes 0..3
    cplx* dst = (cplx*)P.s_hist + slice_off(n);
    for (int i = tid; i < (8 * nloc) << LPB; i += SIGMA_THREADS) {
        const int pp = i & (PB - 1), v = (i >> LPB) & 7, kl = i >> (LPB + 3);
        if (pp >= np) continue;
        const int plane = v < 4 ? 4 + v : v - 4;
        dst[(int64_t)kl * P.tri + sl_idx(plane, b0 + pp)] = dat[(pp * 8 + v) * LS + fft_pad(P.k_lo + kl, LG)];
    }
}
#define KBE_FFT_LGS(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7)

// ---- K1 as DFT GEMMs on the FP64 tensor cores (any even n_k) --------------------------
// The same Fourier-space Sigma^ as sigma_fft_kernel, with both transforms written as
// dense complex GEMMs against the n_k x n_k DFT matrix W[f][k] = w^{-fk}, the shared
// operand of every line (SURVEY 8(a) a11 variant (b), "DFT-as-GEMM"):
//   forward  V^[f][line] = sum_k W[f][k] V[k][line]                 (M = n_k, N = 8 PB, K = n_k)
//   inverse  Sigma[k][line] = sum_f conj(W)[k][f] S^[f][line], k local (M = n_k_local)
// Each 8x8 output tile is one warp's chain of mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4):
// a complex MAC is 4 real DMMAs (Re += Wr Vr - Wi Vi, Im += Wr Vi + Wi Vr).  W is never
// stored: the A fragment is looked up in the w^{-j} table at (f k) mod n_k, advanced by
// 4f per k-step.  16 n_k^2 complex MACs per pair (half the correlations' 32 n_k^2), all
// on the tensor pipe.  Production path for n_k that is not a power of two; for powers of
// two the FFT kernel does O(n_k log n_k) and is kept (KBE_SIGMA=dft selects this one).
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}
__host__ __device__ __forceinline__ int pow2ceil(int v) { int p = 1; while (p < v) p <<= 1; return p; }
__host__ __device__ __forceinline__ int dft_m8(int nk) { return (nk + 7) & ~7; }
// line stride (16-byte slots) = 4 mod 8: the B fragment's 8 lines x 4 consecutive k of a
// quarter-warp hit distinct banks
__host__ __device__ __forceinline__ int dft_ls(int nk) { return dft_m8(nk) + 4; }
static size_t sigma_dft_smem(int nk, int pb) {
    return ((size_t)nk + (size_t)pb * 8 * dft_ls(nk) + (size_t)pb * 2 * nk) * sizeof(cplx);
}
// pairs per CTA: PB m8 <= 256 (<= 32 8x8 tiles per GEMM, 4 per warp), halved while the
// grid stays within one wave of 2 CTAs per SM
static int sigma_dft_pb(int nk, int npairs, int sms) {
    int pb = SIGMA_THREADS / pow2ceil(dft_m8(nk) > nk ? dft_m8(nk) : nk);
    pb = pb > 32 ? 32 : (pb < 1 ? 1 : pb);
    while (pb > 1 && (npairs + pb / 2 - 1) / (pb / 2) <= 2 * sms) pb >>= 1;
    return pb;
}
#define DFT_TPW 4   // 8x8 tiles per warp and GEMM
// One complex GEMM pass over the CTA's lines: rows r (f, or local k on the inverse) of
// the DFT matrix (conjugated when INV) times the lines' first K4 entries.  Results stay
// in registers (cr/ci: real/imag accumulator pairs of DFT_TPW tiles) until every warp
// has read its operands; the caller syncs and stores.
template <bool INV>
__device__ __forceinline__ void dft_gemm(const cplx* tw, const cplx* dat, int nk, int LS, int row0, int mt, int ncol8,
                                         double (*cr)[2], double (*ci)[2]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int K4 = (nk + 3) & ~3;
#pragma unroll
    for (int u = 0; u < DFT_TPW; ++u) {
        cr[u][0] = cr[u][1] = ci[u][0] = ci[u][1] = 0.0;
        const int t = warp + 8 * u;
        if (t >= mt * ncol8) continue;   // warp-uniform
        const int r = row0 + (t % mt) * 8 + (lane >> 2);         // A row (global f or k)
        const cplx* B = dat + ((t / mt) * 8 + (lane >> 2)) * LS;  // B column = one line
        const int kq = lane & 3;
        const int rr = r % nk;
        int idx = (rr * kq) % nk;                                 // (r k) mod n_k, k = k0 + kq
        const int step = (4 * rr) % nk;
        for (int k0 = 0; k0 < K4; k0 += 4) {
            const cplx w = tw[idx];
            const cplx v = B[k0 + kq];
            const double wr = w.x, wi = INV ? -w.y : w.y;
            dmma884(cr[u][0], cr[u][1], wr, v.x);
            dmma884(cr[u][0], cr[u][1], -wi, v.y);
            dmma884(ci[u][0], ci[u][1], wr, v.y);
            dmma884(ci[u][0], ci[u][1], wi, v.x);
            idx += step;
            if (idx >= nk) idx -= nk;
        }
    }
}
// store a GEMM's tiles into the lines: entry row - row0 of line c (rows < rmax)
__device__ __forceinline__ void dft_put(cplx* dat, int LS, int mt, int ncol8, int rmax, double (*cr)[2],
                                        double (*ci)[2]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int u = 0; u < DFT_TPW; ++u) {
        const int t = warp + 8 * u;
        if (t >= mt * ncol8) continue;
        const int r = (t % mt) * 8 + (lane >> 2);
        if (r >= rmax) continue;
        const int c = (t / mt) * 8 + 2 * (lane & 3);
        dat[c * LS + r] = make_double2(cr[u][0], ci[u][0]);
        dat[(c + 1) * LS + r] = make_double2(cr[u][1], ci[u][1]);
    }
}
__global__ void __launch_bounds__(SIGMA_THREADS, 2) sigma_dft_kernel(kbe_problem P, int n, int it, int PB) {
    pdl_enter();
    const kbe_ctl* ctl = (const kbe_ctl*)P.ctl;
    p2p_wait(P);   // the frontier and the control tails of the last update, all ranks
    if (kbe_skip(P, ctl, it)) return;
    extern __shared__ cplx sm[];
    const int nk = P.n_k, LS = dft_ls(nk), LPB = ilog2(PB);
    cplx* tw = sm;                        // w^{-j}, j < n_k
    cplx* dat = sm + nk;                  // [PB * 8 lines][LS]
    cplx* det = dat + PB * 8 * LS;        // [PB][2][n_k]
    const int b0 = blockIdx.x * PB, np = min(PB, n + 1 - b0);
    const int nloc = P.k_hi - P.k_lo;
    const int tid = threadIdx.x;
    for (int j = tid; j < nk; j += SIGMA_THREADS) {
        double sn, cs;
        sincospi(-2.0 * (double)j / (double)nk, &sn, &cs);
        tw[j] = make_double2(cs, sn);
    }
    // lines of absent pairs and the K padding (k in [n_k, K4)) stay zero
    for (int i = tid; i < PB * 8 * LS; i += SIGMA_THREADS) dat[i] = cz();
    __syncthreads();
    {
        const bool sh = sharded(P);
        const cplx* src = sh ? front_base(P) : (const cplx*)P.g_hist + slice_off(n);
        const int64_t kstride = sh ? 8 * plane_len(P.n_steps) : P.tri, rstride = sh ? front_chunk(P) : 0;
        const int kper = sh ? nloc : nk;
        for (int i = tid; i < (8 * nk) << LPB; i += SIGMA_THREADS) {
            const int p = i & (PB - 1), c = (i >> LPB) & 7, k = i >> (LPB + 3);
            if (p >= np) continue;
            const int b = b0 + p, cc = c & 3;
            const cplx v = __ldg(src + (k / kper) * rstride + (k % kper) * kstride + sl_idx(c, b));
            const int jm = b < n ? ((cc & 1) * 2 + (cc >> 1)) : cc;
            dat[(p * 8 + (c & 4) + jm) * LS + k] = b < n ? cneg(cconj(v)) : v;
        }
    }
    __syncthreads();
    double cr[DFT_TPW][2], ci[DFT_TPW][2];
    const int mt = dft_m8(nk) / 8;
    dft_gemm<false>(tw, dat, nk, LS, 0, mt, PB, cr, ci);
    __syncthreads();
    dft_put(dat, LS, mt, PB, nk, cr, ci);
    __syncthreads();
    // pointwise Sigma^ in natural order (f and -f = n_k - f), as in sigma_fft_kernel
    const double inv3 = 1.0 / ((double)nk * (double)nk * (double)nk);
    const double un = P.u_table[n];
    for (int i = tid; i < np * nk; i += SIGMA_THREADS) {
        const int p = i / nk, q = i % nk;
        const cplx* L = dat + p * 8 * LS + q;
        const double c = (P.u_table[b0 + p] * un) * inv3;
        const cplx d1 = csub(cmul(L[0], L[3 * LS]), cmul(L[LS], L[2 * LS]));
        const cplx d2 = csub(cmul(L[4 * LS], L[7 * LS]), cmul(L[5 * LS], L[6 * LS]));
        det[(p * 2) * nk + q] = cscale(d1, c);
        det[(p * 2 + 1) * nk + q] = cscale(d2, c);
    }
    __syncthreads();
    {
        const int i = tid;   // np n_k <= 256 (sigma_dft_pb)
        cplx m1[4], m2[4];
        const bool act = i < np * nk;
        const int p = act ? i / nk : 0, q = act ? i % nk : 0;
        if (act) {
            const cplx* L = dat + p * 8 * LS + (q ? nk - q : 0);
#pragma unroll
            for (int v = 0; v < 4; ++v) { m1[v] = L[v * LS]; m2[v] = L[(4 + v) * LS]; }
        }
        __syncthreads();
        if (act) {
            cplx* L = dat + p * 8 * LS + q;
            const cplx d1 = det[(p * 2) * nk + q], d2 = det[(p * 2 + 1) * nk + q];
#pragma unroll
            for (int jm = 0; jm < 4; ++jm) {
                const int o = jm == 0 ? 3 : (jm == 3 ? 0 : jm);
                cplx s0 = cmul(d1, m2[o]), s1 = cmul(d2, m1[o]);
                if (jm == 1 || jm == 2) { s0 = cneg(s0); s1 = cneg(s1); }
                L[jm * LS] = s0;
                L[(4 + jm) * LS] = s1;
            }
        }
    }
    __syncthreads();
    const int mt2 = (nloc + 7) / 8;
    dft_gemm<true>(tw, dat, nk, LS, P.k_lo, mt2, PB, cr, ci);
    __syncthreads();
    dft_put(dat, LS, mt2, PB, nloc, cr, ci);
    __syncthreads();
    cplx* dst = (cplx*)P.s_hist + slice_off(n);
    for (int i = tid; i < (8 * nloc) << LPB; i += SIGMA_THREADS) {
        const int p = i & (PB - 1), v = (i >> LPB) & 7, kl = i >> (LPB + 3);
        if (p >= np) continue;
        const int plane = v < 4 ? 4 + v : v - 4;
        dst[(int64_t)kl * P.tri + sl_idx(plane, b0 + p)] = dat[(p * 8 + v) * LS + kl];
    }
}

// kernel-level sigma_slice API on batch-last (n_k,2,2,nb) buffers; one CTA per pair.
__global__ void __launch_bounds__(256) sigma_slice_kernel(int nk, int nb, const cplx* gpi, const cplx* gri,
                                                          const double* u1, const double* u2, int k_lo,
                                                          int k_hi, const cplx* pol_in, cplx* pol_out,
                                                          cplx* s1_out, cplx* s2_out, cplx* sig_out) {
    extern __shared__ cplx sm[];
    const int b = blockIdx.x;
    cplx* gp = sm;               // [4][nk]
    cplx* gr = gp + nk * 4;      // [4][nk]
    cplx* Pm = gr + nk * 4;      // [4][nk]
    cplx* Xm = Pm + nk * 4;      // [4][nk]
    const int tid = threadIdx.x, nth = blockDim.x;
    for (int i = tid; i < nk * 4; i += nth) {
        const int k = i >> 2, jm = i & 3;
        gp[jm * nk + k] = gpi[(int64_t)i * nb + b];
        gr[jm * nk + k] = gri[(int64_t)i * nb + b];
    }
    __syncthreads();
    for (int i = tid; i < 4 * nk; i += nth) {
        const int q = i % nk, jm = i / nk;
        const cplx pv = sig_pol(gp, gr, nk, jm, q);
        Pm[jm * nk + q] = pol_in ? pol_in[((int64_t)q * 4 + jm) * nb + b] : pv;
        if (pol_out) pol_out[((int64_t)q * 4 + jm) * nb + b] = pv;
        Xm[jm * nk + q] = sig_x(gp, gr, nk, jm, q);
    }
    __syncthreads();
    const int nloc = k_hi - k_lo;
    const double pref = (u1[b] * u2[b]) / ((double)nk * (double)nk);
    for (int i = tid; i < 4 * nloc; i += nth) {
        const int kl = i % nloc, jm = i / nloc, k = k_lo + kl;
        const cplx s1 = cscale(sig_s1(Pm, gp, nk, jm, k), pref);
        const cplx s2 = cscale(sig_s2(gp, Xm, nk, jm, k), pref);
        const int64_t o = ((int64_t)kl * 4 + jm) * nb + b;
        if (s1_out) s1_out[o] = s1;
        if (s2_out) s2_out[o] = s2;
        if (sig_out) sig_out[o] = csub(s1, s2);
    }
}

// =================================================================== K2: collision
// collision_frontier at step n (collision.py:141-277), as-printed limit, over
// the packed histories.  Two independent triangle streams in one launch:
//
//  part 0 (Sigma triangle, slices 0..n) -> I<(t_n, t_l), l = 0..n:
//    I<_row[l] = sum_tb w_tb [ G>(n,tb) S<(tb,l) - G<(n,tb) S>(tb,l) ]
//    Each stored cell (s,b), b<=s, is read once and feeds two outputs:
//      out[s] += w_b [A(b) SU(s,b) + B(b) SL(s,b)^dag]     (b < s)
//      out[s] += w_s [A(s) SU(s,s) - B(s) SL(s,s)]         (b = s)
//      out[b] -= w_s [A(s) SU(s,b)^dag + B(s) SL(s,b)]     (b < s)
//    with A(b) = G>(t_n,t_b), B(b) = G<(t_n,t_b) (the G frontier slice).
//  part 1 (G triangle, slices 0..n-1) -> I>(t_j, t_n), j = 0..n-1:
//    I>_col[j] = sum_{tb<=j} w^(j)_tb [ G<(j,tb) S>(tb,n) - G>(j,tb) S<(tb,n) ]
//             = sum w [ GU(j,tb)^dag Y(tb) - GL(j,tb) X(tb)^dag ]   (tb < j)
//               + w [ -GU(j,j) Y(j) - GL(j,j) X(j)^dag ]            (tb = j)
//    with X(tb) = S>(t_n,t_tb), Y(tb) = S<(t_tb,t_n) (the Sigma frontier slice).
// I> = -I< (rows) and I< = -I> (columns) in as-printed mode (SURVEY finding 5).
//
// Tile = KBE_TILE_S slices x KBE_TILE_B history points; one thread per point b,
// looping over the slices.  Row sums are warp-reduced (reduce-scatter) and
// combined across warps in shared memory; column sums stay in registers.
// Partials go to a workspace reduced in fixed order by the consumer (K3), so
// results are deterministic run to run.
#define TB KBE_TILE_B
#define TS KBE_TILE_S

// the 8 planes of point b of one slice (base = slice start)
__device__ __forceinline__ void load_cell(const cplx* base, int b, cplx* lo, cplx* up) {
    base += sl_idx(0, b);
#pragma unroll
    for (int c = 0; c < 4; ++c) lo[c] = __ldcg(base + 32 * c);   // L2: valid before griddepcontrol.wait
#pragma unroll
    for (int c = 0; c < 4; ++c) up[c] = __ldcg(base + 32 * (4 + c));
}

// ---- TMA bulk copies + mbarriers (sm_90+ async proxy), one pipeline per warp
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "LAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE;\n\t"
        "bra LAB_WAIT;\n\t"
        "DONE:\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// order this thread's prior generic-proxy shared accesses before later async-proxy (TMA) ones
__device__ __forceinline__ void fence_proxy_async() {
#if KBE_COLL_EXP != 3
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#endif
}
// L2 policies: the history stream is read once per evaluation (evict first); the
// K2 -> K3 partial sums must survive that stream in L2 (evict last).
__device__ __forceinline__ uint64_t l2_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint64_t l2_evict_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void st_keep(double* p, double v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_keep2(cplx* p, cplx v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
}
// the incremental evaluations' delta slots are complex64 (their values are FP32 sums, so
// storing them as FP32 is exact and halves the K2 -> K3 delta traffic)
__device__ __forceinline__ void st_keep_f(float* p, float v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_keep2_f(fcx* p, fcx v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(p), "f"(v.x), "f"(v.y), "l"(pol) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

// Sub-tile height (slices per warp task) of the as-printed collision pass at
// frontier n: tiles stay 32 x 32 (KBE_TILE_S x KBE_TILE_B) for the partial-sum
// layout, but a warp takes ts = 8, 16 or 32 of a tile's slices, chosen so that a
// launch has >= KBE_COLL_TASKS warp tasks (small frontiers would otherwise leave
// most of the 148 SMs idle).  Column-direction partials are kept per ts-chunk in
// KBE_COL_CHUNK-granular slots; the consumer (K3) derives the same ts from n.
// langreth keeps ts = 32.
// as-printed task height cap (slices per warp task; the per-slice vectors in shared
// memory are sized by it) and the collision kernel's resident-CTA target
#ifndef KBE_VEC_TS
#define KBE_VEC_TS 32
#endif
#ifndef KBE_COLL_MINB
#define KBE_COLL_MINB 16
#endif
#ifndef KBE_NO_EARLY
#define KBE_NO_EARLY 0   // 1: K2 always waits for K1 at entry (A/B switch)
#endif
#ifndef KBE_COLL_TASKS
#define KBE_COLL_TASKS 4096   // ~1.7 tasks per resident warp: taller tasks mean fewer
                              // column partials for K3 (profiles/r01/task_size_v25.jsonl)
#endif
__host__ __device__ __forceinline__ int coll_tiles(int n, int nkl) {
    const int T0 = n / TS + 1, T1 = n >= 1 ? (n - 1) / TS + 1 : 0;
    return (T0 * (T0 + 1) / 2 + T1 * (T1 + 1) / 2) * nkl;
}
// k-shards with few local k (a strong-scaled rank): twice the tasks.  Their launches are
// short, so the queue's tail (the last, partly filled round of tasks) is a larger share
// than the K3 slot traffic that taller tasks save (profiles/r02/scaling_model_*).
#ifndef KBE_SMALL_NKL
#define KBE_SMALL_NKL 8
#endif
__host__ __device__ __forceinline__ int coll_ts(int n, int nkl, int limit_mode) {
    if (limit_mode) return TS;
    const int tiles = coll_tiles(n, nkl);
    const int target = nkl <= KBE_SMALL_NKL ? 2 * KBE_COLL_TASKS : KBE_COLL_TASKS;
    if (tiles >= target) return KBE_VEC_TS;
    if (2 * tiles >= target) return 16;
    return KBE_COL_CHUNK;
}

#ifndef KBE_STAGES
#define KBE_STAGES 2
#endif
// dynamic shared memory of one collision warp-task
struct CollSmem {
    cplx buf[KBE_STAGES][8][32];   // ring of slice cells: 8 planes x 32 points (FP64), or
                                   // 2 x KBE_STAGES complex64 shadow blocks (incremental)
    cplx vec[KBE_VEC_TS][8];       // per-slice frontier vectors (Sigma part)
    uint64_t bar[2 * KBE_STAGES];
};
// the langreth variant keeps 32-slice tasks
struct CollSmemL {
    cplx buf[KBE_STAGES][8][32];
    cplx vec[TS][8];
    uint64_t bar[KBE_STAGES];
};

// Issue the bulk copy of block wb0/32 of history slice s (wb0 <= s, so the block
// exists): one 4 KB copy (8 planes x 32 points) off the diagonal; on a diagonal
// block only the s - wb0 + 1 stored points of each plane are read (8 copies), so
// the stream moves no padding.
__device__ __forceinline__ void issue_slice(const cplx* hist, int s, int wb0, cplx (*dst)[32], uint64_t* bar,
                                            uint64_t pol) {
    const cplx* src = hist + slice_off(s) + sl_idx(0, wb0);
    const int cnt = s + 1 - wb0;
    if (cnt >= 32) {
        mbar_expect_tx(bar, 8u * 32u * 16u);
        bulk_g2s(dst[0], src, 8u * 32u * 16u, bar, pol);
        return;
    }
    const uint32_t bytes = (uint32_t)cnt * 16u;
    mbar_expect_tx(bar, 8u * bytes);
#pragma unroll
    for (int c = 0; c < 8; ++c) bulk_g2s(dst[c], src + 32 * c, bytes, bar, pol);
}

// triangular index t -> (sc, bc) with 0 <= bc <= sc
__device__ __forceinline__ void tri_decode(int t, int& sc, int& bc) {
    int s = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
    while ((s + 1) * (s + 2) / 2 <= t) ++s;
    while (s * (s + 1) / 2 > t) --s;
    sc = s;
    bc = t - s * (s + 1) / 2;
}

// Collision task list: tiles (sc, bc) of the Sigma triangle (part 0, T0 tile rows)
// and of the G triangle (part 1, T1 rows) for every local k, each split into nsub
// sub-tiles.  All full off-diagonal tiles come first and the half-full diagonal
// tiles last, so the dynamic queue ends on short tasks (smaller tail).
struct CollTask { int kl, part, sc, bc, sub; };
__device__ __forceinline__ CollTask coll_task(int task, int nkl, int T0, int T1, int nsub) {
    CollTask t;
    const int off0 = T0 * (T0 - 1) / 2, off1 = T1 * (T1 - 1) / 2;   // strictly-lower tiles per k
    const int n_off = (off0 + off1) * nsub * nkl;
    t.sub = task % nsub;
    if (task < n_off) {
        const int q = task / nsub, per = off0 + off1;
        t.kl = q / per;
        int r = q % per;
        t.part = r < off0 ? 0 : 1;
        if (t.part) r -= off0;
        int sr, br;
        tri_decode(r, sr, br);
        t.sc = sr + 1;
        t.bc = br;
    } else {
        const int q = (task - n_off) / nsub, per = T0 + T1;
        t.kl = q / per;
        const int d = q % per;
        t.part = d < T0 ? 0 : 1;
        t.sc = t.bc = t.part ? d - T0 : d;
    }
    return t;
}

// ---- incremental evaluations (as-printed) ------------------------------------------
// Every evaluation at frontier f is I = H(v) + F(v): H the cells of slices < f (final
// history, linear in the frontier vectors v = (G slice f, Sigma slice f)), F the cells
// of slice f.  A full evaluation streams the FP64 history and snapshots v into v_prev.
// A repeated evaluation at the same f (the predictor's I(n-1) after the previous
// step's last corrector, or corrector it >= 1) whose vectors moved by at most
// KBE_INCR_MAX_DELTA since that full one (the sum of the residuals the updates
// measured in between) writes
//   M (v - v_prev)   into delta slots, M streamed from a complex64 shadow of the history
// (half the bytes; error ~2^-24 x (products + <= 32-term sums) x |M| |dv|: <= 2e-13 |I| worst
// case, ~1e-14 typical), and F(v)
// exactly in FP64.  K3 then sums base + delta per slot.  Slice f's column-direction sums
// live in their own slot (fcol_part), so the chunk slots hold H only.  The shadow of
// slice n-1 (G and Sigma) is written by the predictor update, once it is final.
#ifndef KBE_INCR_MAX_DELTA
#define KBE_INCR_MAX_DELTA 1e-7
#endif
// frontier change since the previous evaluation at f: the residual its update measured
__device__ __forceinline__ double coll_delta(const kbe_problem& P, const kbe_ctl* ctl, int it) {
    if (it > 0) return __longlong_as_double((long long)res_bits(P, ctl, it - 1));
    // predictor evaluation at the previous step's frontier: that step's final residual
    double d = __longlong_as_double((long long)res_bits(P, ctl, P.max_iter - 1));
    for (int i = 0; i < P.max_iter; ++i) {
        const double r = __longlong_as_double((long long)res_bits(P, ctl, i));
        if (r <= P.eps) { d = r; break; }
    }
    return d;
}
__device__ __forceinline__ bool coll_incremental(const kbe_problem& P, const kbe_ctl* ctl, int f, double delta) {
    if (!P.g_sh || P.limit_mode) return false;
    const volatile kbe_ctl* c = ctl;
    if (c->prev_f1 != f + 1 || c->full_f1 != f + 1) return false;
    return c->dsum + delta <= KBE_INCR_MAX_DELTA;   // false for NaN
}
// complex64 block of shadow slice s (8 planes x 32 points, 2 KB)
__device__ __forceinline__ void issue_shadow(const float2* sh, int s, int wb0, cplx (*dst)[32], uint64_t* bar,
                                             uint64_t pol) {
    mbar_expect_tx(bar, 8u * 32u * 8u);
    bulk_g2s(dst[0], sh + slice_off(s) + sl_idx(0, wb0), 8u * 32u * 8u, bar, pol);
}
// lane's 8 planes of one FP64 stage
__device__ __forceinline__ void stage_cell(const cplx (*buf)[32], int lane, cplx* lo, cplx* up) {
#pragma unroll
    for (int c = 0; c < 4; ++c) { lo[c] = buf[c][lane]; up[c] = buf[4 + c][lane]; }
}
// part-0 vectors at point b of the G frontier slice f: w_b A(b), w_b B(b) with
// A(b) = G>(t_f,t_b) = -U(f,b)^dag (b < f) | U(f,f), B(b) = G<(t_f,t_b) = L(f,b)
__device__ __forceinline__ void front_ab(const cplx* slice, int b, int f, double w, cplx* A, cplx* B) {
    cplx u[4], l[4];
    load_cell(slice, b, l, u);
    if (b < f) neg_dag(A, u);
    else {
#pragma unroll
        for (int c = 0; c < 4; ++c) A[c] = u[c];
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) { A[c] = cscale(A[c], w); B[c] = cscale(l[c], w); }
}

// One warp = one task of 32 history points x ts slices; a persistent grid of 1-warp
// CTAs walks the task list (tasks of both triangles, all local k).  No CTA-level
// barriers; a KBE_STAGES-deep ring of 4 KB bulk copies per warp (2 stages: 16 warps/SM).
// A converged iteration costs one tiny grid of early exits.
// The two evaluation modes are separate bodies, so the per-slice loop carries no mode
// branches (K2 is latency-bound per slice).

// last CTA out resets the queue for the next launch on this stream and records the
// frontier whose partials are now in the workspace
__device__ __forceinline__ void coll_finish(kbe_ctl* ctl, int n, double delta, bool incr) {
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned d = atomicAdd(&ctl->task_done, 1u);
        if (d == gridDim.x - 1) {
            ctl->task_next = 0u;
            ctl->task_done = 0u;
            ctl->prev_f1 = n + 1;
            if (incr) {
                ctl->dsum += delta;
            } else {
                ctl->full_f1 = n + 1;
                ctl->dsum = 0.0;
            }
            ctl->incr_last = incr ? 1 : 0;
            __threadfence();
        }
    }
}

// full FP64 evaluation
__device__ __forceinline__ void coll_body(const kbe_problem& P, kbe_ctl* ctl, int n, double delta, bool& waited) {
    extern __shared__ __align__(128) unsigned char smraw[];
    CollSmem& sm = *reinterpret_cast<CollSmem*>(smraw);
    const int lane = threadIdx.x;
    const int N1 = P.n_steps + 1;
    const double dt = P.dt;
    const int T0 = n / TS + 1, T1 = n >= 1 ? (n - 1) / TS + 1 : 0;
    const int tri0 = T0 * (T0 + 1) / 2, tri1 = T1 * (T1 + 1) / 2;
    const int ts = coll_ts(n, P.k_hi - P.k_lo, 0), nsub = TS / ts;
    const int per_k = (tri0 + tri1) * nsub;
    const int total = per_k * (P.k_hi - P.k_lo);
    uint64_t* bars = sm.bar;
    constexpr int STG = KBE_STAGES;
    auto stage = [&](unsigned st) -> cplx (*)[32] { return sm.buf[st]; };
    if (lane == 0) {
        for (int i = 0; i < STG; ++i) mbar_init(&bars[i], 1);
        mbar_fence_init();
    }
    __syncwarp();
    const uint64_t pol_stream = l2_evict_first(), pol_keep = l2_evict_last();
    unsigned gcount = 0;   // slices consumed by this CTA so far (ring position / parity)
    for (;;) {
        // dynamic work queue: balances the half-full diagonal tasks
        unsigned tk = 0;
        if (lane == 0) tk = atomicAdd(&ctl->task_next, 1u);
        const int task = (int)__shfl_sync(0xffffffffu, tk, 0);
        if (task >= total) break;
        const CollTask ct = coll_task(task, P.k_hi - P.k_lo, T0, T1, nsub);
        const int kl = ct.kl, part = ct.part, sc = ct.sc, bc = ct.bc, sub = ct.sub;
        const int smax = part == 0 ? n : n - 1;
        const int s0 = sc * TS + sub * ts, s1 = min(s0 + ts - 1, smax);
        if (s0 > smax) continue;            // empty sub-tile past the frontier
        const int wb0 = bc * TB;            // wb0 <= s0: every slice has lane 0 valid
        const int m = s1 - s0 + 1;
        const int b = wb0 + lane;
        if (!waited && (part == 1 || s1 == n)) {   // this task reads Sigma slice n (early start)
            asm volatile("griddepcontrol.wait;" ::: "memory");
            waited = true;
        }
        const cplx* G = (const cplx*)P.g_hist + (int64_t)kl * P.tri;
        const cplx* S = (const cplx*)P.s_hist + (int64_t)kl * P.tri;
        // frontier slice n (vector) and the streamed triangle
        const cplx* fr = (part == 0 ? G : S) + slice_off(n);
        const cplx* hist = part == 0 ? S : G;
        auto issue = [&](int s, unsigned st) { issue_slice(hist, s, wb0, stage(st), &bars[st], pol_stream); };
        __syncwarp();
        if (lane == 0)
            for (int i = 0; i < STG && i < m; ++i) issue(s0 + i, (gcount + i) % STG);
        double* outP = (double*)(part == 0 ? P.row_part : P.gc_part);
        // row slot (bc, s): the base slot (the delta slots are ignored after a full evaluation)
        auto put_row = [&](int s, double rr) {
            if (KBE_COLL_EXP != 4 && (lane & 3) == 0) {
                const int64_t o = (((int64_t)kl * P.nbb + bc) * N1 + s) * 8 + (lane >> 2);
                st_keep(&outP[o], rr, pol_keep);
            }
        };

        if (part == 0) {
            // per-slice vectors w_s A(s), w_s B(s)
            if (lane < m) {
                const int s = s0 + lane;
                const double w = quad_w(n, s, dt, P.quad);
                cplx a[4], l[4];
                front_ab(fr, s, n, w, a, l);
#pragma unroll
                for (int c = 0; c < 4; ++c) { sm.vec[lane][c] = a[c]; sm.vec[lane][4 + c] = l[c]; }
            }
            cplx Ab[4], Bb[4], col[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) { Ab[c] = cz(); Bb[c] = cz(); col[c] = cz(); }
            const double wb = quad_w(n, b, dt, P.quad);
            if (b <= s1) front_ab(fr, b, n, wb, Ab, Bb);
            cplx* colP = (cplx*)P.col_part + (((int64_t)kl * P.nsb + s0 / ts) * N1 + b) * 4;
            __syncwarp();
            for (int i = 0; i < m; ++i, ++gcount) {
                const int s = s0 + i;
                const unsigned st = gcount % STG;
                if (s == n) {
                    // frontier slice: its column sums go to their own slot
                    if (b <= s1) {
#pragma unroll
                        for (int c = 0; c < 4; ++c) st_keep2(&colP[c], cneg(col[c]), pol_keep);
                    }
#pragma unroll
                    for (int c = 0; c < 4; ++c) col[c] = cz();
                }
                cplx SL[4], SU[4];
                mbar_wait(&bars[st], (gcount / STG) & 1u);
                stage_cell(stage(st), lane, SL, SU);
                // the stage is in registers: refill it now, so the copy overlaps this
                // slice's arithmetic (proxy fence: generic reads before async writes)
                fence_proxy_async();
                __syncwarp();
                if (lane == 0 && i + STG < m) issue(s + STG, st);
                cplx row[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) row[c] = cz();
#if KBE_COLL_EXP == 1
                if (b <= s) {
#pragma unroll
                    for (int c = 0; c < 4; ++c) { row[c] = cadd(SL[c], SU[c]); col[c] = cadd(col[c], SL[c]); }
                }
                if (false) {
#else
                if (b <= s) {
#endif
                    mm_acc(row, Ab, SU);
                    if (b < s) {
                        mm_bdag_acc(row, Bb, SL);
                        cplx As[4], Bs[4];
#pragma unroll
                        for (int c = 0; c < 4; ++c) { As[c] = sm.vec[i][c]; Bs[c] = sm.vec[i][4 + c]; }
                        mm_bdag_acc(col, As, SU);   // col += As SU^dag + Bs SL
                        mm_acc(col, Bs, SL);
                    } else {
                        cplx t[4];
                        mm(t, Bb, SL);
#pragma unroll
                        for (int c = 0; c < 4; ++c) row[c] = csub(row[c], t[c]);
                    }
                }
                double v[8];
#pragma unroll
                for (int c = 0; c < 4; ++c) { v[2 * c] = row[c].x; v[2 * c + 1] = row[c].y; }
#if KBE_COLL_EXP == 2
                const double rr = v[lane & 7];
#else
                const double rr = warp_rs8(v, lane);   // all lanes' reads of stage st are consumed here
#endif
                put_row(s, rr);
            }
            if (b <= s1) {
                if (s1 == n) {   // slice n's column sums
                    cplx* fc = (cplx*)P.fcol_part + ((int64_t)kl * N1 + b) * 4;
#pragma unroll
                    for (int c = 0; c < 4; ++c) st_keep2(&fc[c], cneg(col[c]), pol_keep);
                } else {
#pragma unroll
                    for (int c = 0; c < 4; ++c) st_keep2(&colP[c], cneg(col[c]), pol_keep);
                }
            }
        } else {
            // column collision over the G triangle (slices < n: all history); frontier
            // vectors X = SL(n,b), Y = SU(n,b)
            cplx X[4], Y[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) { X[c] = cz(); Y[c] = cz(); }
            if (b <= s1) load_cell(fr, b, X, Y);
            for (int i = 0; i < m; ++i, ++gcount) {
                const int j = s0 + i;
                const unsigned st = gcount % STG;
                mbar_wait(&bars[st], (gcount / STG) & 1u);
                cplx GL[4], GU[4];
                stage_cell(stage(st), lane, GL, GU);
                fence_proxy_async();   // stage in registers: refill it during the arithmetic
                __syncwarp();
                if (lane == 0 && i + STG < m) issue(j + STG, st);
                cplx acc[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[c] = cz();
#if KBE_COLL_EXP == 1
                if (b <= j) {
#pragma unroll
                    for (int c = 0; c < 4; ++c) acc[c] = cadd(GL[c], GU[c]);
                }
                if (false) {
#else
                if (b <= j) {
#endif
                    const double w = quad_w(j, b, dt, P.quad);
                    cplx t[4];
                    mm_bdag(t, GL, X);                 // GL X^dag
                    if (b < j) {
                        mm_adag_acc(acc, GU, Y);       // GU^dag Y
                    } else {
                        cplx u[4];
                        mm(u, GU, Y);
#pragma unroll
                        for (int c = 0; c < 4; ++c) acc[c] = cneg(u[c]);
                    }
#pragma unroll
                    for (int c = 0; c < 4; ++c) acc[c] = cscale(csub(acc[c], t[c]), w);
                }
                double v[8];
#pragma unroll
                for (int c = 0; c < 4; ++c) { v[2 * c] = acc[c].x; v[2 * c + 1] = acc[c].y; }
#if KBE_COLL_EXP == 2
                const double rr = v[lane & 7];
#else
                const double rr = warp_rs8(v, lane);
#endif
                put_row(j, rr);
            }
        }
    }
    if (P.g_sh) {
        // snapshot the frontier vectors (G and Sigma slice n, local k) for the
        // incremental evaluations that may follow at this frontier (after the wait
        // for K1: Sigma slice n is its output)
        if (!waited) {
            asm volatile("griddepcontrol.wait;" ::: "memory");
            waited = true;
        }
        const int64_t per = 8 * plane_len(n), tot = (int64_t)(P.k_hi - P.k_lo) * 2 * per;
        for (int64_t i = blockIdx.x * 32 + lane; i < tot; i += (int64_t)gridDim.x * 32) {
            const int kl = (int)(i / (2 * per)), which = (int)((i / per) & 1);
            const int64_t e = i % per;
            const cplx* src = (const cplx*)(which ? P.s_hist : P.g_hist) + (int64_t)kl * P.tri + slice_off(n);
            ((cplx*)P.v_prev)[vprev_off(P, kl, which) + e] = __ldcg(src + e);
        }
    }
    coll_finish(ctl, n, delta, false);
}

// Incremental evaluation: the history cells (slices < n) enter only through the change
// of the frontier vectors, M dv with |dv| <= KBE_INCR_MAX_DELTA, so they are computed in
// complex64 straight from the complex64 shadow (FP32 FMAs, no conversions, 32-bit
// shuffles): relative error ~2^-24 x (products + <= 32-term sums) of a term that is
// itself <= 1e-7 of I, i.e. <= ~2e-13 |I| worst case and ~1e-14 typically.  Slice n
// (row tasks of the last tile row) is re-evaluated in full FP64 after the loop.
// An incremental slice is half the bytes of a full one, so FP64 arithmetic (and its
// conversions) would bound the ring, not HBM.
__device__ __forceinline__ void coll_body_incr(const kbe_problem& P, kbe_ctl* ctl, int n, double delta,
                                               bool& waited) {
    extern __shared__ __align__(128) unsigned char smraw[];
    CollSmem& sm = *reinterpret_cast<CollSmem*>(smraw);
    fcx (*vec)[8] = reinterpret_cast<fcx (*)[8]>(&sm.vec[0][0]);
    const int lane = threadIdx.x;
    const int N1 = P.n_steps + 1;
    const double dt = P.dt;
    const int T0 = n / TS + 1, T1 = n >= 1 ? (n - 1) / TS + 1 : 0;
    const int tri0 = T0 * (T0 + 1) / 2, tri1 = T1 * (T1 + 1) / 2;
    const int ts = coll_ts(n, P.k_hi - P.k_lo, 0), nsub = TS / ts;
    const int per_k = (tri0 + tri1) * nsub;
    const int total = per_k * (P.k_hi - P.k_lo);
    uint64_t* bars = sm.bar;
    // the ring is latency-bound (a stage is refilled only once consumed), so its depth in
    // slices, not bytes, sets the rate: 2 KB shadow blocks get twice the stages
    constexpr int STG = 2 * KBE_STAGES;
    auto stage = [&](unsigned st) -> cplx (*)[32] {
        return reinterpret_cast<cplx (*)[32]>(reinterpret_cast<unsigned char*>(sm.buf) + st * 2048u);
    };
    if (lane == 0) {
        for (int i = 0; i < STG; ++i) mbar_init(&bars[i], 1);
        mbar_fence_init();
    }
    __syncwarp();
    const uint64_t pol_stream = l2_evict_first(), pol_keep = l2_evict_last();
    unsigned gcount = 0;
    for (;;) {
        unsigned tk = 0;
        if (lane == 0) tk = atomicAdd(&ctl->task_next, 1u);
        const int task = (int)__shfl_sync(0xffffffffu, tk, 0);
        if (task >= total) break;
        const CollTask ct = coll_task(task, P.k_hi - P.k_lo, T0, T1, nsub);
        const int kl = ct.kl, part = ct.part, sc = ct.sc, bc = ct.bc, sub = ct.sub;
        const int smax = part == 0 ? n : n - 1;
        const int s0 = sc * TS + sub * ts, s1 = min(s0 + ts - 1, smax);
        if (s0 > smax) continue;
        const int wb0 = bc * TB;
        const int m = s1 - s0 + 1;
        const int b = wb0 + lane;
        if (!waited && (part == 1 || s1 == n)) {
            asm volatile("griddepcontrol.wait;" ::: "memory");
            waited = true;
        }
        const cplx* G = (const cplx*)P.g_hist + (int64_t)kl * P.tri;
        const cplx* S = (const cplx*)P.s_hist + (int64_t)kl * P.tri;
        // frontier slice n, its value at the last full evaluation, the shadow triangle
        const cplx* fr = (part == 0 ? G : S) + slice_off(n);
        const cplx* fp = (const cplx*)P.v_prev + vprev_off(P, kl, part);
        const float2* hsh = (const float2*)(part == 0 ? P.s_sh : P.g_sh) + (int64_t)kl * P.tri;
        auto issue = [&](int s, unsigned st) { issue_shadow(hsh, s, wb0, stage(st), &bars[st], pol_stream); };
        // slices through the ring: those < n (slice n: FP64 epilogue)
        const int mr = (part == 0 && s1 == n) ? m - 1 : m;
        __syncwarp();
        if (lane == 0)
            for (int i = 0; i < STG && i < mr; ++i) issue(s0 + i, (gcount + i) % STG);
        double* outP = (double*)(part == 0 ? P.row_part : P.gc_part);
        float* outD = (float*)(part == 0 ? P.row_delta : P.gc_delta);
        auto put = [&](double* out, int s, double rr) {
            if ((lane & 3) == 0) st_keep(&out[(((int64_t)kl * P.nbb + bc) * N1 + s) * 8 + (lane >> 2)], rr, pol_keep);
        };
        auto putD = [&](int s, float rr) {
            if ((lane & 3) == 0) st_keep_f(&outD[(((int64_t)kl * P.nbb + bc) * N1 + s) * 8 + (lane >> 2)], rr, pol_keep);
        };
        auto shadow_cell = [&](unsigned st, fcx* lo, fcx* up) {
            const fcx* f = reinterpret_cast<const fcx*>(stage(st));
#pragma unroll
            for (int c = 0; c < 4; ++c) { lo[c] = f[c * 32 + lane]; up[c] = f[(4 + c) * 32 + lane]; }
        };

        if (part == 0) {
            // per-slice vector changes w_s dA(s), w_s dB(s) (slices < n)
            if (lane < mr) {
                const int s = s0 + lane;
                const double w = quad_w(n, s, dt, P.quad);
                cplx a[4], l[4], a0[4], l0[4];
                front_ab(fr, s, n, w, a, l);
                front_ab(fp, s, n, w, a0, l0);
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const fcx as = f32(csub(a[c], a0[c])), bs = f32(csub(l[c], l0[c]));
                    vec[lane][c] = as;
                    vec[lane][4 + c] = bs;
                    vec[32 + lane][c] = rot_m(as);       // for col += As SU^dag
                    vec[32 + lane][4 + c] = rot_p(bs);   // for col += Bs SL
                }
            }
            fcx Ab[4], Bb[4], Abr[4], Bbr[4], col[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) { Ab[c] = make_float2(0.f, 0.f); Bb[c] = Ab[c]; col[c] = Ab[c]; }
            const double wb = quad_w(n, b, dt, P.quad);
            if (b <= s1) {
                cplx a[4], l[4], a0[4], l0[4];
                front_ab(fr, b, n, wb, a, l);
                front_ab(fp, b, n, wb, a0, l0);
#pragma unroll
                for (int c = 0; c < 4; ++c) { Ab[c] = f32(csub(a[c], a0[c])); Bb[c] = f32(csub(l[c], l0[c])); }
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) { Abr[c] = rot_p(Ab[c]); Bbr[c] = rot_m(Bb[c]); }
            __syncwarp();
            // OFF: a block strictly below the diagonal (b < s for every lane and slice):
            // no per-slice point tests
            auto loop0 = [&](auto off_c) {
            constexpr bool OFF = decltype(off_c)::value;
            for (int i = 0; i < mr; ++i, ++gcount) {
                const int s = s0 + i;
                const unsigned st = gcount % STG;
                mbar_wait(&bars[st], (gcount / STG) & 1u);
                fcx SL[4], SU[4];
                shadow_cell(st, SL, SU);
                fence_proxy_async();
                __syncwarp();
                if (lane == 0 && i + STG < mr) issue(s + STG, st);
                fcx row[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) row[c] = make_float2(0.f, 0.f);
                if (OFF || b <= s) {
                    mm2_cs(row, Ab, Abr, SU);                 // row += Ab SU
                    if (OFF || b < s) {
                        mm2_csdag(row, Bb, Bbr, SL);          // row += Bb SL^dag
                        fcx As[4], Bs[4], Asr[4], Bsr[4];
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            As[c] = vec[i][c];
                            Bs[c] = vec[i][4 + c];
                            Asr[c] = vec[32 + i][c];
                            Bsr[c] = vec[32 + i][4 + c];
                        }
                        mm2_csdag(col, As, Asr, SU);          // col += As SU^dag
                        mm2_cs(col, Bs, Bsr, SL);             // col += Bs SL
                    } else {
                        fcx t[4];
#pragma unroll
                        for (int c = 0; c < 4; ++c) t[c] = make_float2(0.f, 0.f);
                        fcx Bbp[4];
#pragma unroll
                        for (int c = 0; c < 4; ++c) Bbp[c] = rot_p(Bb[c]);
                        mm2_cs(t, Bb, Bbp, SL);
#pragma unroll
                        for (int c = 0; c < 4; ++c) row[c] = make_float2(row[c].x - t[c].x, row[c].y - t[c].y);
                    }
                }
                float v[8];
#pragma unroll
                for (int c = 0; c < 4; ++c) { v[2 * c] = row[c].x; v[2 * c + 1] = row[c].y; }
                putD(s, warp_rs8(v, lane));
            }
            };
            if (wb0 + TB <= s0) loop0(std::true_type{});
            else loop0(std::false_type{});
            // history-part column sums -> the chunk's delta slot
            if (b <= s1) {
                fcx* colD = (fcx*)P.col_delta + (((int64_t)kl * P.nsb + s0 / ts) * N1 + b) * 4;
#pragma unroll
                for (int c = 0; c < 4; ++c) st_keep2_f(&colD[c], make_float2(-col[c].x, -col[c].y), pol_keep);
            }
            if (s1 == n) {
                // slice n in FP64 with the full vectors: base row slot (zero delta), fcol slot
                cplx SL[4], SU[4], Af[4], Bf[4], row[4], cf[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) { SL[c] = cz(); SU[c] = cz(); Af[c] = cz(); Bf[c] = cz(); row[c] = cz(); cf[c] = cz(); }
                if (b <= n) {
                    load_cell(S + slice_off(n), b, SL, SU);
                    front_ab(fr, b, n, wb, Af, Bf);
                    mm_acc(row, Af, SU);
                    if (b < n) {
                        mm_bdag_acc(row, Bf, SL);
                        cplx As[4], Bs[4];
                        front_ab(fr, n, n, quad_w(n, n, dt, P.quad), As, Bs);
                        mm_bdag_acc(cf, As, SU);
                        mm_acc(cf, Bs, SL);
                    } else {
                        cplx t[4];
                        mm(t, Bf, SL);
#pragma unroll
                        for (int c = 0; c < 4; ++c) row[c] = csub(row[c], t[c]);
                    }
                }
                double v[8];
#pragma unroll
                for (int c = 0; c < 4; ++c) { v[2 * c] = row[c].x; v[2 * c + 1] = row[c].y; }
                const double rr = warp_rs8(v, lane);
                put(outP, n, rr);
                putD(n, 0.f);
                if (b <= n) {
                    cplx* fc = (cplx*)P.fcol_part + ((int64_t)kl * N1 + b) * 4;
#pragma unroll
                    for (int c = 0; c < 4; ++c) st_keep2(&fc[c], cneg(cf[c]), pol_keep);
                }
            }
        } else {
            // column collision over the G triangle: X = dSL(n,b), Y = dSU(n,b)
            fcx X[4], Y[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) { X[c] = make_float2(0.f, 0.f); Y[c] = X[c]; }
            if (b <= s1) {
                cplx x[4], y[4], x0[4], y0[4];
                load_cell(fr, b, x, y);
                load_cell(fp, b, x0, y0);
#pragma unroll
                for (int c = 0; c < 4; ++c) { X[c] = f32(csub(x[c], x0[c])); Y[c] = f32(csub(y[c], y0[c])); }
            }
            // off-diagonal blocks: the weight w(j, b) (b < j) depends on j's parity only
            // (trapezoid: not at all), so it is set once per task
            const bool off = wb0 + TB <= s0;
            const int je = (s0 + 1) & ~1;   // even and odd reference frontiers > b
            const float w_even = (float)quad_w(je + 2, b, dt, P.quad), w_odd = (float)quad_w(je + 1, b, dt, P.quad);
            auto loop1 = [&](auto off_c) {
            constexpr bool OFF = decltype(off_c)::value;
            for (int i = 0; i < m; ++i, ++gcount) {
                const int j = s0 + i;
                const unsigned st = gcount % STG;
                mbar_wait(&bars[st], (gcount / STG) & 1u);
                fcx GL[4], GU[4];
                shadow_cell(st, GL, GU);
                fence_proxy_async();
                __syncwarp();
                if (lane == 0 && i + STG < m) issue(j + STG, st);
                fcx acc[4], t[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) { acc[c] = make_float2(0.f, 0.f); t[c] = acc[c]; }
                if (OFF || b <= j) {
                    const float w = OFF ? ((j & 1) ? w_odd : w_even) : (float)quad_w(j, b, dt, P.quad);
                    mm2_scdag(t, GL, X);               // GL X^dag
                    if (OFF || b < j) {
                        mm2_sdagc(acc, GU, Y);         // GU^dag Y
                    } else {
                        fcx u[4];
#pragma unroll
                        for (int c = 0; c < 4; ++c) u[c] = make_float2(0.f, 0.f);
                        mm2_sc(u, GU, Y);
#pragma unroll
                        for (int c = 0; c < 4; ++c) acc[c] = make_float2(-u[c].x, -u[c].y);
                    }
#pragma unroll
                    for (int c = 0; c < 4; ++c) acc[c] = make_float2((acc[c].x - t[c].x) * w, (acc[c].y - t[c].y) * w);
                }
                float v[8];
#pragma unroll
                for (int c = 0; c < 4; ++c) { v[2 * c] = acc[c].x; v[2 * c + 1] = acc[c].y; }
                putD(j, warp_rs8(v, lane));
            }
            };
            if (off) loop1(std::true_type{});
            else loop1(std::false_type{});
        }
    }
    coll_finish(ctl, n, delta, true);
}

// Early start (one rank, Sigma on): K2's only input from
// the kernel before it (K1) is Sigma slice n.  K1 itself started only after the update
// before it had completed, so the history, the G frontier and the convergence record
// are final when K2's CTAs become resident: K2 skips griddepcontrol.wait at entry and
// streams the tasks that do not touch Sigma slice n (part 0, slices < n) while K1 is
// still running; a warp waits for K1 before its first task that does (part 1's
// vectors, part 0's last tile row) and, at the latest, before it exits.  Pre-wait
// reads bypass L1 (ld.cg / volatile / TMA from L2).  `after_sigma` is set only by the
// step sequencer (K1 is the launch before): a K2 launched on its own through
// kbe_collision_frontier waits for all earlier work, so two back-to-back K2s never
// share the task queue.
__global__ void __launch_bounds__(32, KBE_COLL_MINB) collision_kernel(kbe_problem P, int n, int it, int after_sigma) {
    const bool early = after_sigma && P.interacting && P.p2p_world <= 1 && !P.front_all && !KBE_NO_EARLY;
    if (early) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    else pdl_enter();
    kbe_ctl* ctl = (kbe_ctl*)P.ctl;
    if (!P.interacting) p2p_wait(P);   // first kernel after the update when Sigma is off
    if (kbe_skip(P, ctl, it)) {
        if (early) asm volatile("griddepcontrol.wait;" ::: "memory");
        return;
    }
    const double delta = coll_delta(P, ctl, it);
    bool waited = !early;
    if (coll_incremental(P, ctl, n, delta)) coll_body_incr(P, ctl, n, delta, waited);
    else coll_body(P, ctl, n, delta, waited);
    if (!waited) asm volatile("griddepcontrol.wait;" ::: "memory");
}

// K2, limit_mode = "langreth" (collision.py:188-191, 211-219): the second term's
// quadrature limit is the column time t_l (rows) / t_n (columns), so I> != -I< and
// both components are accumulated.  Same task decomposition and TMA ring as the
// as-printed kernel; the G triangle now also runs over slice n and scatters its
// second term along the column direction.
//  Sigma triangle cell (s,b), Xc = S>(b,s) (= -SL^dag, or SL on the diagonal):
//    I<_row[s] += w(n)_b D(b) SU + w(s)_b B(b) (SU - Xc)
//    I>_row[s] += -w(n)_b D(b) Xc - w(s)_b A(b) (SU - Xc)
//    I<_row[b] -= w(n)_s D(s) SU^dag,   I>_row[b] -= w(n)_s D(s) SL      (b < s)
//    with D = A - B = G>(n,.) - G<(n,.)
//  G triangle cell (s,b), Gg = G>(s,b) (= -GU^dag, or GU on the diagonal),
//  Y(b) = S<(b,n), Z(b) = S>(b,n), V(s) = w(n)_s (Y(s) - Z(s)):
//    I<_col[s] += w(s)_b (Gg - GL) Y(b) + w(n)_b GL (Y(b) - Z(b))
//    I>_col[s] += w(s)_b (GL - Gg) Z(b) + w(n)_b Gg (Z(b) - Y(b))
//    I<_col[b] -= GL^dag V(s),   I>_col[b] -= GU V(s)                     (b < s)
__global__ void __launch_bounds__(32, 8) collision_langreth_kernel(kbe_problem P, int n, int it) {
    pdl_enter();
    kbe_ctl* ctl = (kbe_ctl*)P.ctl;
    if (!P.interacting) p2p_wait(P);   // first kernel after the update when Sigma is off
    if (kbe_skip(P, ctl, it)) return;
    extern __shared__ __align__(128) unsigned char smraw[];
    CollSmemL& sm = *reinterpret_cast<CollSmemL*>(smraw);
    const int lane = threadIdx.x;
    const int N1 = P.n_steps + 1;
    const double dt = P.dt;
    const int T0 = n / TS + 1;
    const int tri0 = T0 * (T0 + 1) / 2;
    const int per_k = 2 * tri0;
    const int total = per_k * (P.k_hi - P.k_lo);
    uint64_t* bars = sm.bar;
    if (lane == 0) {
        for (int i = 0; i < KBE_STAGES; ++i) mbar_init(&bars[i], 1);
        mbar_fence_init();
    }
    __syncwarp();
    const uint64_t pol_stream = l2_evict_first(), pol_keep = l2_evict_last();
    unsigned gcount = 0;
    for (;;) {
        unsigned tk = 0;
        if (lane == 0) tk = atomicAdd(&ctl->task_next, 1u);
        const int task = (int)__shfl_sync(0xffffffffu, tk, 0);
        if (task >= total) break;
        const CollTask ct = coll_task(task, P.k_hi - P.k_lo, T0, T0, 1);   // both triangles run to slice n
        const int kl = ct.kl, part = ct.part, sc = ct.sc, bc = ct.bc;
        const int s0 = sc * TS, s1 = min(s0 + TS - 1, n);
        const int wb0 = bc * TB;
        const int m = s1 - s0 + 1;
        const int b = wb0 + lane;
        const cplx* G = (const cplx*)P.g_hist + (int64_t)kl * P.tri;
        const cplx* S = (const cplx*)P.s_hist + (int64_t)kl * P.tri;
        const cplx* fr = (part == 0 ? G : S) + slice_off(n);
        const cplx* hist = part == 0 ? S : G;
        __syncwarp();
        if (lane == 0)
            for (int i = 0; i < KBE_STAGES && i < m; ++i) {
                const unsigned st = (gcount + i) % KBE_STAGES;
                issue_slice(hist, s0 + i, wb0, sm.buf[st], &bars[st], pol_stream);
            }
        // per-slice vector (4 complex): part 0 D(s) w(n)_s, part 1 V(s)
        if (lane < m) {
            const int s = s0 + lane;
            const double w = quad_w(n, s, dt, P.quad);
            cplx l[4], u[4], v[4];
            load_cell(fr, s, l, u);
            if (part == 0) {
                cplx a[4];
                if (s < n) neg_dag(a, u);
                else {
#pragma unroll
                    for (int c = 0; c < 4; ++c) a[c] = u[c];
                }
#pragma unroll
                for (int c = 0; c < 4; ++c) v[c] = cscale(csub(a[c], l[c]), w);
            } else {
                cplx z[4];   // Z(s) = S>(s,n) = -SL(n,s)^dag (s < n) | SL(n,n)
                if (s < n) neg_dag(z, l);
                else {
#pragma unroll
                    for (int c = 0; c < 4; ++c) z[c] = l[c];
                }
#pragma unroll
                for (int c = 0; c < 4; ++c) v[c] = cscale(csub(u[c], z[c]), w);
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) sm.vec[lane][c] = v[c];
        }
        // own-point vectors
        cplx P1[4], P2[4], P3[4], colL[4], colG[4];
        double wnb = 0.0;
#pragma unroll
        for (int c = 0; c < 4; ++c) { P1[c] = cz(); P2[c] = cz(); P3[c] = cz(); colL[c] = cz(); colG[c] = cz(); }
        if (b <= s1) {
            cplx l[4], u[4];
            load_cell(fr, b, l, u);
            wnb = quad_w(n, b, dt, P.quad);
            if (part == 0) {   // P1 = A(b), P2 = B(b), P3 = w(n)_b D(b)
                if (b < n) neg_dag(P1, u);
                else {
#pragma unroll
                    for (int c = 0; c < 4; ++c) P1[c] = u[c];
                }
#pragma unroll
                for (int c = 0; c < 4; ++c) { P2[c] = l[c]; P3[c] = cscale(csub(P1[c], l[c]), wnb); }
            } else {           // P1 = Y(b), P2 = Z(b), P3 = w(n)_b (Y(b) - Z(b))
                if (b < n) neg_dag(P2, l);
                else {
#pragma unroll
                    for (int c = 0; c < 4; ++c) P2[c] = l[c];
                }
#pragma unroll
                for (int c = 0; c < 4; ++c) { P1[c] = u[c]; P3[c] = cscale(csub(u[c], P2[c]), wnb); }
            }
        }
        __syncwarp();
        double* outL = (double*)(part == 0 ? P.row_part : P.lc_part);
        double* outG = (double*)(part == 0 ? P.row_part_g : P.gc_part);
        for (int i = 0; i < m; ++i, ++gcount) {
            const int s = s0 + i;
            const unsigned st = gcount % KBE_STAGES;
            mbar_wait(&bars[st], (gcount / KBE_STAGES) & 1u);
            cplx LO[4], UP[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) { LO[c] = sm.buf[st][c][lane]; UP[c] = sm.buf[st][4 + c][lane]; }
            cplx rl[4], rg[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) { rl[c] = cz(); rg[c] = cz(); }
            if (b <= s) {
                const double wsb = quad_w(s, b, dt, P.quad);
                cplx V[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) V[c] = sm.vec[i][c];
                if (part == 0) {
                    // LO = SL(s,b), UP = SU(s,b);  Xc = S>(b,s)
                    cplx Xc[4], Ml[4], t[4];
                    if (b < s) neg_dag(Xc, LO);
                    else {
#pragma unroll
                        for (int c = 0; c < 4; ++c) Xc[c] = LO[c];
                    }
#pragma unroll
                    for (int c = 0; c < 4; ++c) Ml[c] = csub(UP[c], Xc[c]);
                    mm_acc(rl, P3, UP);                 // w(n)_b D(b) SU
                    mm(t, P2, Ml);                      // B(b) (SU - Xc)
#pragma unroll
                    for (int c = 0; c < 4; ++c) rl[c] = cadd(rl[c], cscale(t[c], wsb));
                    mm(t, P3, Xc);                      // -w(n)_b D(b) Xc
#pragma unroll
                    for (int c = 0; c < 4; ++c) rg[c] = cneg(t[c]);
                    mm(t, P1, Ml);                      // -w(s)_b A(b) (SU - Xc)
#pragma unroll
                    for (int c = 0; c < 4; ++c) rg[c] = csub(rg[c], cscale(t[c], wsb));
                    if (b < s) {
                        mm_bdag_acc(colL, V, UP);       // D(s) SU^dag
                        mm_acc(colG, V, LO);            // D(s) SL
                    }
                } else {
                    // LO = GL(s,b), UP = GU(s,b);  Gg = G>(s,b)
                    cplx Gg[4], t[4], d[4];
                    if (b < s) neg_dag(Gg, UP);
                    else {
#pragma unroll
                        for (int c = 0; c < 4; ++c) Gg[c] = UP[c];
                    }
#pragma unroll
                    for (int c = 0; c < 4; ++c) d[c] = csub(Gg[c], LO[c]);
                    mm(t, d, P1);                       // (Gg - GL) Y(b)
#pragma unroll
                    for (int c = 0; c < 4; ++c) rl[c] = cscale(t[c], wsb);
                    mm_acc(rl, LO, P3);                 // w(n)_b GL (Y - Z)
                    mm(t, d, P2);                       // -(Gg - GL) Z(b)
#pragma unroll
                    for (int c = 0; c < 4; ++c) rg[c] = cneg(cscale(t[c], wsb));
                    mm(t, Gg, P3);                      // -w(n)_b Gg (Y - Z)
#pragma unroll
                    for (int c = 0; c < 4; ++c) rg[c] = csub(rg[c], t[c]);
                    if (b < s) {
                        mm_adag_acc(colL, LO, V);       // GL^dag V(s)
                        mm_acc(colG, UP, V);            // GU V(s)
                    }
                }
            }
            double v[8];
#pragma unroll
            for (int c = 0; c < 4; ++c) { v[2 * c] = rl[c].x; v[2 * c + 1] = rl[c].y; }
            const double r1 = warp_rs8(v, lane);
#pragma unroll
            for (int c = 0; c < 4; ++c) { v[2 * c] = rg[c].x; v[2 * c + 1] = rg[c].y; }
            const double r2 = warp_rs8(v, lane);
            if ((lane & 3) == 0) {
                const int64_t o = (((int64_t)kl * P.nbb + bc) * N1 + s) * 8 + (lane >> 2);
                st_keep(&outL[o], r1, pol_keep);
                st_keep(&outG[o], r2, pol_keep);
            }
            fence_proxy_async();
            __syncwarp();
            if (lane == 0 && i + KBE_STAGES < m) issue_slice(hist, s + KBE_STAGES, wb0, sm.buf[st], &bars[st], pol_stream);
        }
        if (b <= s1) {
            cplx* cL = (cplx*)(part == 0 ? P.col_part : P.lc_part_c);
            cplx* cG = (cplx*)(part == 0 ? P.col_part_g : P.gc_part_c);
            const int64_t o = (((int64_t)kl * P.nsb + sc) * N1 + b) * 4;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                st_keep2(&cL[o + c], cneg(colL[c]), pol_keep);
                st_keep2(&cG[o + c], cneg(colG[c]), pol_keep);
            }
        }
    }
    if (lane == 0) {
        __threadfence();
        const unsigned d = atomicAdd(&ctl->task_done, 1u);
        if (d == gridDim.x - 1) {
            ctl->task_next = 0u;
            ctl->task_done = 0u;
            __threadfence();
        }
    }
}

// Fixed-order reductions of the partials written by collision_kernel(nf).
// Partial planes are [k][chunk][point][4 complex], so consecutive points (threads)
// read consecutive 64-byte blocks for every chunk.
// sum_{bc <= l/TB} rowdir[bc][l] + sum_{l/ts <= sc <= nf/ts} coldir[sc][l]  (coldir may be null;
// ts = the column chunk height the producing launch used, coll_ts(nf))
__device__ __forceinline__ void reduce_chunks(const kbe_problem& P, const void* rowdir, const void* coldir, int kl,
                                              int l, int nf, cplx* out) {
    const int ts = coll_ts(nf, P.k_hi - P.k_lo, P.limit_mode);
    const int64_t N1 = P.n_steps + 1;
#pragma unroll
    for (int c = 0; c < 4; ++c) out[c] = cz();
    const cplx* rp = (const cplx*)rowdir + ((int64_t)kl * P.nbb * N1 + l) * 4;
    const int nr = l / TB;
#pragma unroll 4
    for (int bc = 0; bc <= nr; ++bc)
#pragma unroll
        for (int c = 0; c < 4; ++c) out[c] = cadd(out[c], rp[bc * N1 * 4 + c]);
    if (coldir) {
        const cplx* cp = (const cplx*)coldir + ((int64_t)kl * P.nsb * N1 + l) * 4;
        const int s_hi = nf / ts;
#pragma unroll 4
        for (int sc = l / ts; sc <= s_hi; ++sc)
#pragma unroll
            for (int c = 0; c < 4; ++c) out[c] = cadd(out[c], cp[sc * N1 * 4 + c]);
        if (coldir == P.col_part && !P.limit_mode && l < nf) {   // frontier slice (own slot)
            const cplx* fc = (const cplx*)P.fcol_part + ((int64_t)kl * N1 + l) * 4;
#pragma unroll
            for (int c = 0; c < 4; ++c) out[c] = cadd(out[c], fc[c]);
        }
    }
}
// I<(t_nf, t_l) / I>(t_nf, t_l) (rows) and I>(t_j, t_nf) / I<(t_j, t_nf) (columns)
// + the delta slots when the last evaluation was incremental (as-printed only); the
// delta slots are complex64, summed in the same chunk order as reduce_chunks
__device__ __forceinline__ void add_deltas(const kbe_problem& P, const void* rowd, const void* cold, int kl, int l,
                                           int nf, cplx* out) {
    if (P.limit_mode || !P.ctl || !((const volatile kbe_ctl*)P.ctl)->incr_last) return;
    const int64_t N1 = P.n_steps + 1;
    const int ts = coll_ts(nf, P.k_hi - P.k_lo, 0);
    cplx d[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) d[c] = cz();
    const fcx* rp = (const fcx*)rowd + ((int64_t)kl * P.nbb * N1 + l) * 4;
    for (int bc = 0; bc <= l / TB; ++bc)
#pragma unroll
        for (int c = 0; c < 4; ++c) d[c] = cadd(d[c], f64(rp[bc * N1 * 4 + c]));
    if (cold) {
        const fcx* cp = (const fcx*)cold + ((int64_t)kl * P.nsb * N1 + l) * 4;
        for (int sc = l / ts; sc <= nf / ts; ++sc)
#pragma unroll
            for (int c = 0; c < 4; ++c) d[c] = cadd(d[c], f64(cp[sc * N1 * 4 + c]));
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) out[c] = cadd(out[c], d[c]);
}
__device__ __forceinline__ void reduce_lr(const kbe_problem& P, int kl, int l, int nf, cplx* out) {
    reduce_chunks(P, P.row_part, P.col_part, kl, l, nf, out);
    add_deltas(P, P.row_delta, P.col_delta, kl, l, nf, out);
}
__device__ __forceinline__ void reduce_gr(const kbe_problem& P, int kl, int l, int nf, cplx* out) {
    reduce_chunks(P, P.row_part_g, P.col_part_g, kl, l, nf, out);
}
__device__ __forceinline__ void reduce_gc(const kbe_problem& P, int kl, int j, int nf, cplx* out) {
    reduce_chunks(P, P.gc_part, P.limit_mode ? P.gc_part_c : nullptr, kl, j, nf, out);
    add_deltas(P, P.gc_delta, nullptr, kl, j, nf, out);
}
__device__ __forceinline__ void reduce_lc(const kbe_problem& P, int kl, int j, int nf, cplx* out) {
    reduce_chunks(P, P.lc_part, P.lc_part_c, kl, j, nf, out);
}

// kernel-level collision_frontier: partials -> CollisionSlice arrays (batch-last)
__global__ void collision_slice_kernel(kbe_problem P, int n, cplx* lr, cplx* gr, cplx* lc, cplx* gc) {
    pdl_enter();
    const int kl = blockIdx.y;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i > n) return;
    cplx v[4], w[4];
    reduce_lr(P, kl, i, n, v);
    if (P.limit_mode) reduce_gr(P, kl, i, n, w);
    else {
#pragma unroll
        for (int c = 0; c < 4; ++c) w[c] = cneg(v[c]);
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        lr[((int64_t)kl * 4 + c) * (n + 1) + i] = v[c];
        gr[((int64_t)kl * 4 + c) * (n + 1) + i] = w[c];
    }
    if (i < n) {
        reduce_gc(P, kl, i, n, v);
        if (P.limit_mode) reduce_lc(P, kl, i, n, w);
        else {
#pragma unroll
            for (int c = 0; c < 4; ++c) w[c] = cneg(v[c]);
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            gc[((int64_t)kl * 4 + c) * n + i] = v[c];
            lc[((int64_t)kl * 4 + c) * n + i] = w[c];
        }
    }
}

// kernel-level collision_row (collision.py:141-162) on caller layouts:
//   out[k,a,m,l] = sum_{t<T1} w1[t] sum_b dg[k,a,b,t] SL[k,b,m,t,l]
//                + sum_{t<T2} w2[t | t,l] sum_b g[k,a,b,t] (SL - SO)[k,b,m,t,l]
// dg: (n_k,2,2,T1); g: (n_k,2,2,T2); SL, SO: (n_k,2,2,T,P); out (n_k,2,2,P) (the t axis of
// dg / g is the weight length, as in the reference's einsums; a (T,P) w2 has T2 = T).  One thread per (k, m, l)
// computes both a, so each SL/SO element is read once; consecutive threads walk l
// (the contiguous axis).  A bench/API helper, not on the step path.
__global__ void collision_row_kernel(int nk, int T, int P, int T1, int T2, int w2_matrix, const cplx* dg,
                                     const cplx* g, const cplx* sl, const cplx* so, const double* w1,
                                     const double* w2, cplx* out) {
    const int64_t total = (int64_t)nk * 2 * P;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int l = (int)(i % P), m = (int)((i / P) & 1), k = (int)(i / (2 * (int64_t)P));
        cplx acc[2] = {cz(), cz()};
        const int tmax = max(T1, T2);
        for (int t = 0; t < tmax; ++t) {
            const double a1 = t < T1 ? w1[t] : 0.0;
            const double a2 = t < T2 ? (w2_matrix ? w2[(int64_t)t * P + l] : w2[t]) : 0.0;
#pragma unroll
            for (int b = 0; b < 2; ++b) {
                const int64_t si = ((((int64_t)k * 2 + b) * 2 + m) * T + t) * P + l;
                const cplx x = sl[si], d = csub(x, so[si]);
#pragma unroll
                for (int a = 0; a < 2; ++a) {
                    const int64_t ab = ((int64_t)k * 2 + a) * 2 + b;
                    if (t < T1) acc[a] = cfma(cscale(dg[ab * T1 + t], a1), x, acc[a]);
                    if (t < T2) acc[a] = cfma(cscale(g[ab * T2 + t], a2), d, acc[a]);
                }
            }
        }
#pragma unroll
        for (int a = 0; a < 2; ++a) out[(((int64_t)k * 2 + a) * 2 + m) * P + l] = acc[a];
    }
}

// =================================================================== K3: update
// h(k; t_{n-1/2}) (model.py:123-152) and its Cayley propagator (propagator.py:77-94).
__device__ void build_phi(const kbe_problem& P, const kbe_ctl* ctl, int n, int k, cplx* phi) {
    const double u = P.u_mid[n], amp = P.amp[n];
    cplx h[4];
    h[0] = make_double2(P.eps_v[k], 0.0);
    h[1] = cz();
    h[2] = cz();
    h[3] = make_double2(P.eps_c[k] - u, 0.0);
    if (amp != 0.0) {
        h[1] = make_double2(amp * P.dipole_re, amp * -P.dipole_im);
        h[2] = make_double2(amp * P.dipole_re, amp * P.dipole_im);
    }
    if (P.hf) {   // hartree_fock (model.py:106-120) from the k-mean of rho
        const double inv = (double)P.n_k;
        const cplx m00 = make_double2(ctl->hf_sum[0].x / inv, ctl->hf_sum[0].y / inv);
        const cplx m01 = make_double2(ctl->hf_sum[1].x / inv, ctl->hf_sum[1].y / inv);
        const cplx m10 = make_double2(ctl->hf_sum[2].x / inv, ctl->hf_sum[2].y / inv);
        const cplx m11 = make_double2(ctl->hf_sum[3].x / inv, ctl->hf_sum[3].y / inv);
        h[0] = cadd(h[0], make_double2(u * m11.x, 0.0));
        h[3] = cadd(h[3], make_double2(u * m00.x, 0.0));
        h[1] = cadd(h[1], make_double2(-u * m01.x, -u * m01.y));
        h[2] = cadd(h[2], make_double2(-u * m10.x, -u * m10.y));
    }
    const double c = 0.5 * P.dt;
    cplx a[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = make_double2(-c * h[i].y, c * h[i].x);
    const cplx m00 = make_double2(1.0 + a[0].x, a[0].y), m01 = a[1], m10 = a[2];
    const cplx m11 = make_double2(1.0 + a[3].x, a[3].y);
    const cplx n00 = make_double2(1.0 - a[0].x, -a[0].y), n01 = cneg(a[1]), n10 = cneg(a[2]);
    const cplx n11 = make_double2(1.0 - a[3].x, -a[3].y);
    const cplx det = csub(cmul(m00, m11), cmul(m01, m10));
    phi[0] = cdiv(csub(cmul(m11, n00), cmul(m01, n10)), det);
    phi[1] = cdiv(csub(cmul(m11, n01), cmul(m01, n11)), det);
    phi[2] = cdiv(csub(cmul(m00, n10), cmul(m10, n00)), det);
    phi[3] = cdiv(csub(cmul(m00, n11), cmul(m10, n01)), det);
}

__device__ __forceinline__ double absmax4(const cplx* a, const cplx* b, double r) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const double d = hypot(a[c].x - b[c].x, a[c].y - b[c].y);
        r = (d != d || r != r) ? __longlong_as_double(0x7ff8000000000000LL) : fmax(r, d);
    }
    return r;
}
__device__ __forceinline__ bool finite4(const cplx* a) {
    bool ok = true;
#pragma unroll
    for (int c = 0; c < 4; ++c) ok = ok && isfinite(a[c].x) && isfinite(a[c].y);
    return ok;
}

// row(l)  = Phi (G<(n-1,l) - i dt I_row)          (propagator.py:154-155, 182-184)
// col(j)  = (G>(j,n-1) + i dt I_col) Phi^dag      (propagator.py:156-158, 186-191)
__device__ __forceinline__ void advance_row(const cplx* phi, const cplx* gprev, const cplx* irow, double dt, cplx* out) {
    cplx src[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) src[c] = csub(gprev[c], cmul_pi(irow[c], dt));
    mm(out, phi, src);
}
__device__ __forceinline__ void advance_col(const cplx* phi, const cplx* gprev, const cplx* icol, double dt, cplx* out) {
    cplx src[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) src[c] = cadd(gprev[c], cmul_pi(icol[c], dt));
    mm_bdag(out, src, phi);
}

// K3: predictor / corrector / residual for the frontier points of ALL local k.
//
// One CTA owns PPC consecutive frontier points b for every local k; thread =
// (k, point, block entry), so that a warp reads whole 64-byte blocks of PPC
// consecutive points of one partial chunk (coalesced).  Phase A: each thread sums
// the K2 partials of its block entry in chunk order (deterministic).  Phase B: it
// applies Phi (G - i dt I) / (G + i dt I) Phi^dag (propagator.py:154-158,
// 182-191).  The CTA holding b = n-1 also does the equal-time diagonal b = n
// (propagator.py:193-212).
// LANG = limit_mode (langreth): a template parameter so that the as-printed kernel
// does not carry the langreth reductions' registers.
// Points per CTA: up to 4 (and <= 512 threads), but small frontiers keep one point
// per CTA so that the grid still spreads over the SMs.
#ifndef KBE_UPD_BATCH
#define KBE_UPD_BATCH 3   // partial loads in flight per operand and thread in K3 (4 spills; upd_batch_v25.jsonl)
#endif
static int g_upd_min_ctas = -1;   // KBE_UPD_MIN_CTAS (tuning knob)
static int upd_ppc(int nkl, int n) {
    if (g_upd_min_ctas < 0) {
        const char* e = getenv("KBE_UPD_MIN_CTAS");
        g_upd_min_ctas = e ? atoi(e) : 148;
    }
    int p = 512 / (4 * nkl);
    p = p < 1 ? 1 : (p > 4 ? 4 : p);
    while (p > 1 && n / p < g_upd_min_ctas) p >>= 1;
    return p;
}
static int upd_threads(int nkl, int ppc) { return ((ppc * 4 * nkl + 31) / 32) * 32; }
static size_t upd_smem_bytes(int nkl, int ppc) {
    return sizeof(cplx) * ((size_t)2 * ppc * nkl * 4          // sA, sB
                           + (size_t)6 * nkl * 4);            // sC, sRow, sCol, sX, sY, sZ
}

// complex64 shadow of entry (planes c, 4+c; point b) of the final slice s, G and Sigma
__device__ __noinline__ void write_shadow(const cplx* g_hist, const cplx* s_hist, float2* g_sh, float2* s_sh,
                                         int64_t tri, int kl, int s, int c, int b) {
    const int64_t so = (int64_t)kl * tri + slice_off(s);
    const cplx* gp = g_hist + so;
    const cplx* sp = s_hist + so;
    float2* gsh = g_sh + so;
    float2* ssh = s_sh + so;
    for (int h = 0; h < 2; ++h) {
        const int64_t e = sl_idx(4 * h + c, b);
        gsh[e] = make_float2((float)gp[e].x, (float)gp[e].y);
        ssh[e] = make_float2((float)sp[e].x, (float)sp[e].y);
    }
}

// k-sharded publication of one frontier entry (plane c, point b) of local k kl:
// the NCCL send buffer, or straight into every peer's buffer for data epoch e
__device__ __forceinline__ void publish_entry(const kbe_problem& P, int kl, int c, int b, cplx v, int64_t pm,
                                              unsigned long long e) {
    const int64_t off = (int64_t)kl * 8 * pm + sl_idx(c, b);
    if (P.p2p_world > 1) {
#pragma unroll
        for (int r = 0; r < KBE_MAX_RANKS; ++r)
            if (r < P.p2p_world) p2p_dst(P, r, e)[off] = v;
    } else if (P.front_send) {
        ((cplx*)P.front_send)[off] = v;
    }
}
// control tail of this rank (one thread); P2P: then bump the epoch on every rank
__device__ __forceinline__ void publish_tail(const kbe_problem& P, const KbeTail& t, unsigned long long e) {
    const int64_t off = front_chunk(P) - KBE_TAIL_CPLX;
    if (P.p2p_world > 1) {
#pragma unroll
        for (int r = 0; r < KBE_MAX_RANKS; ++r)
            if (r < P.p2p_world) *(KbeTail*)(p2p_dst(P, r, e) + off) = t;
        p2p_signal(P, e);
    } else if (P.front_send) {
        *(KbeTail*)((cplx*)P.front_send + off) = t;
    }
}

// K3a (split K3, as-printed): the fixed-order partial sums of K3's phase A as a
// separate streaming kernel, so the reduction runs at memory speed instead of as
// ~n/16 dependent loads per thread under K3's register budget (round-1 K3: 22.8 us for
// 47 MB at cfg2 n = 900, 18.7 % occupancy).
//   a(b) = sum_{bc <= b/TB} row[bc][b] + sum_{b/ts <= sc <= nf/ts} col[sc][b] (+ fcol[b], b < nf)
//   g(b) = sum_{bc <= b/TB} gc[bc][b]                                         (b < nf)
// (+ the delta slots after an incremental evaluation); points 0..n-1, and n itself in
// the corrector (the diagonal's I<(t_n, t_n)).
// One warp item = 8 consecutive points x 4 block entries of one local k; lane
// 4*(b - b0) + c owns output (b, c), so every slot is one coalesced 512-byte warp load.
// Aligned groups of 8 points share their slot counts (TB = 32 and the column chunk
// ts in {8, 16, 32} are multiples of 8), so the loop bounds are warp-uniform and each
// lane sums its own slots in order -- row slots bc = 0 .. b/TB (the gc slots at the same
// offsets), and column chunks sc = b/ts .. nf/ts, as (row sum) + (column sum) + fcol --
// all three streams in one batched loop, no shuffles (round-2 v1 split every point's slots over
// 4 lane groups and clamped every load: 720 warp instructions per item, issue-bound at
// 67 us for cfg3 n = 900, profiles/r02/final2/k3a_*_v1_*).  The summation order depends
// only on (n, b): results are bitwise reproducible and independent of the launch shape.
// Incremental problems (INC): after a full evaluation K3a also keeps each point's sums
// (before fcol) in the second half of i_red / g_red; after an incremental evaluation at
// the same frontier only the delta slots changed for points b < nf, so it reads those
// sums and the complex64 delta slots, not the base slots again.  Point nf (whose row
// slots the incremental evaluation rewrites in FP64) sums base and delta slots.
// Persistent grid, items strided over all warps.
__device__ __forceinline__ cplx as_c128(cplx v) { return v; }
__device__ __forceinline__ cplx as_c128(fcx v) { return f64(v); }
// the row (pr) and gc (pg) streams of nr slots and the column stream (pc) of nc slots in
// one loop: each batch has all three streams' loads in flight (the loop is load-latency
// bound); ar += row slots, g += gc slots, ac += column slots, each in slot order
template <int B, class T>
__device__ __forceinline__ void sum_slots3(const T* pr, const T* pg, int nr, const T* pc, int nc, int64_t st,
                                           cplx& ar, cplx& g, cplx& ac) {
    const int nmax = nr > nc ? nr : nc;
    for (int q = 0; q < nmax; q += B) {
        T vr[B], vg[B], vc[B];
#pragma unroll
        for (int u = 0; u < B; ++u) {
            const int64_t o = (int64_t)min(q + u, nr - 1) * st;
            vr[u] = __ldcg(pr + o);
            vg[u] = __ldcg(pg + o);
            vc[u] = __ldcg(pc + (int64_t)min(q + u, nc - 1) * st);
        }
#pragma unroll
        for (int u = 0; u < B; ++u) {
            if (q + u < nr) {
                ar = cadd(ar, as_c128(vr[u]));
                g = cadd(g, as_c128(vg[u]));
            }
            if (q + u < nc) ac = cadd(ac, as_c128(vc[u]));
        }
    }
}
template <int INC>
__global__ void __launch_bounds__(256, 3) reduce_kernel(kbe_problem P, int n, int phase, int it) {
    pdl_enter();
    const kbe_ctl* ctl = (const kbe_ctl*)P.ctl;
    if (phase == 0 ? kbe_halted(ctl) : kbe_skip(P, ctl, it)) return;
    const int nkl = P.k_hi - P.k_lo;
    const int64_t N1 = P.n_steps + 1, cs = N1 * 4;
    const int nf = phase == 0 ? n - 1 : n;
    const int npts = nf + 1;
    const int cts = coll_ts(nf, nkl, 0);
    const bool dl = INC && ((const volatile kbe_ctl*)ctl)->incr_last;
    const int lane = threadIdx.x & 31, c = lane & 3;
    const int groups = (npts + 7) >> 3;
    const int items = nkl * groups;
    const int warps = gridDim.x * (blockDim.x >> 5);
    for (int item = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); item < items; item += warps) {
        const int kl = item / groups, b0 = (item % groups) * 8;
        const int b = b0 + (lane >> 2);
        const int bl = min(b, nf);   // lanes past the frontier load point nf's slots (no store)
        const int nr = b0 / TB + 1, c0 = b0 / cts, ns = nf / cts - c0 + 1;   // warp-uniform
        const int64_t rb = ((int64_t)kl * P.nbb * N1 + bl) * 4 + c;
        const int64_t cb = ((int64_t)kl * P.nsb * N1 + bl) * 4 + c + (int64_t)c0 * cs;
        // a = (row slots) + (column slots), each summed in slot order
        cplx ar = cz(), ac = cz(), gg = cz();
        if (INC && dl)
            sum_slots3<6>((const fcx*)P.row_delta + rb, (const fcx*)P.gc_delta + rb, nr,
                          (const fcx*)P.col_delta + cb, ns, cs, ar, gg, ac);
        if (!(INC && dl) || bl == nf)
            sum_slots3<4>((const cplx*)P.row_part + rb, (const cplx*)P.gc_part + rb, nr,
                          (const cplx*)P.col_part + cb, ns, cs, ar, gg, ac);
        cplx a = cadd(ar, ac);
        if (b < npts) {
            const int64_t oo = ((int64_t)kl * N1 + b) * 4 + c;
            if (b == nf) gg = cz();   // no gc slots for the frontier point
            if (INC) {
                cplx* bi = (cplx*)P.i_red + (int64_t)nkl * N1 * 4;   // base sums (second half)
                cplx* bg = (cplx*)P.g_red + (int64_t)nkl * N1 * 4;
                if (!dl) {
                    bi[oo] = a;
                    bg[oo] = gg;
                } else if (b < nf) {
                    a = cadd(__ldcg(bi + oo), a);
                    gg = cadd(__ldcg(bg + oo), gg);
                }
            }
            if (b < nf) a = cadd(a, __ldcg((const cplx*)P.fcol_part + oo));
            ((cplx*)P.i_red)[oo] = a;
            ((cplx*)P.g_red)[oo] = gg;
        }
    }
}

// INC: the problem has incremental collision evaluations (g_sh): K3 may add delta
// slots and the predictor writes the history shadow.  A separate instantiation keeps
// that code out of the plain kernel's registers.
template <int LANG, int INC, int RED>
__global__ void __launch_bounds__(512) update_kernel(kbe_problem P, int n, int phase, int it, int PPC,
                                                     cudaGraphConditionalHandle next_iter) {
    pdl_enter();
    kbe_ctl* ctl = (kbe_ctl*)P.ctl;
    if (phase == 0) {
        if (kbe_halted(ctl)) return;
    } else if (kbe_skip(P, ctl, it)) {
        return;   // graph mode: next_iter keeps its default 0, so the step ends
    }
    const int nkl = P.k_hi - P.k_lo;
    const int tid = threadIdx.x, T = blockDim.x;
    const int b0 = blockIdx.x * PPC;
    const int np = min(PPC, n - b0);           // own points b0 .. b0+np-1 (all < n)
    const int64_t N1 = P.n_steps + 1;
    const int nf = phase == 0 ? n - 1 : n;     // frontier of the collision being consumed
    const bool diag_cta = b0 <= n - 1 && n - 1 < b0 + PPC;
    const double dt = P.dt;
    const double nan = __longlong_as_double(0x7ff8000000000000LL);
    extern __shared__ cplx usm[];
    cplx* sA = usm;                              // [nkl][PPC][4]  I<(t_nf, t_b)
    cplx* sB = sA + PPC * nkl * 4;               // [nkl][PPC][4]  I>(t_b, t_nf)
    cplx* sC = sB + PPC * nkl * 4;               // [nkl][4]       I<(t_n, t_n)
    cplx* sRow = sC + nkl * 4;                   // [nkl][4]       new G<(n, n-1)
    cplx* sCol = sRow + nkl * 4;                 // [nkl][4]       new G>(n-1, n)
    cplx* sX = sCol + nkl * 4;                   // [nkl][4]       langreth extras
    cplx* sY = sX + nkl * 4;
    cplx* sZ = sY + nkl * 4;
    __shared__ double red[32];
    __shared__ int redf[32];
    if (phase == 0 && blockIdx.x == 0 && tid < KBE_MAX_ITER) {
        ctl->res[tid] = 0ull;
        ctl->nonfinite[tid] = 0;
    }
    const int64_t cs = N1 * 4;   // partial chunk stride
    const int cts = coll_ts(nf, nkl, LANG);

    // this thread's (k, point, entry)
    const int c = tid & 3, o = (tid >> 2) % PPC, kl = (tid >> 2) / PPC;
    const int b = b0 + o, i = c >> 1, j = c & 1;
    const bool own = kl < nkl && o < np;
    cplx* G = (cplx*)P.g_hist + (int64_t)(own ? kl : 0) * P.tri;
    const cplx* prev = G + slice_off(n - 1);
    cplx* cur = G + slice_off(n);
    cplx* lro = (cplx*)P.lr_old + ((int64_t)(own ? kl : 0) * N1 + b) * 4;
    cplx* clo = (cplx*)P.col_old + ((int64_t)(own ? kl : 0) * N1 + b) * 4;
    const cplx* ph = (const cplx*)P.phi + ((int64_t)n * nkl + (own ? kl : 0)) * 4;

    // operands that do not depend on the collision: issued first so that their
    // latency overlaps the partial sums
    cplx phr[2], phc[2], pgl[2], pgu[2], olr[2], ocl[2], ol = cz(), ou = cz();
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        phr[k] = phc[k] = pgl[k] = pgu[k] = olr[k] = ocl[k] = cz();
        if (own) {
            phr[k] = ph[i * 2 + k];
            phc[k] = ph[j * 2 + k];
            pgl[k] = prev[sl_idx(k * 2 + j, b)];
            pgu[k] = prev[sl_idx(4 + i * 2 + k, b)];
            if (phase == 1) {
                olr[k] = lro[k * 2 + j];
                ocl[k] = clo[i * 2 + k];
            }
        }
    }
    if (own && phase == 1) {
        ol = cur[sl_idx(c, b)];
        ou = cur[sl_idx(4 + c, b)];
    }

    // ---- phase A: fixed-order partial sums -------------------------------------------
    if (RED) {
        // split K3: reduce_kernel (K3a) already summed the partials
        if (own) {
            sA[(kl * PPC + o) * 4 + c] = ((const cplx*)P.i_red)[((int64_t)kl * N1 + b) * 4 + c];
            sB[(kl * PPC + o) * 4 + c] = ((const cplx*)P.g_red)[((int64_t)kl * N1 + b) * 4 + c];
        }
        if (diag_cta && phase == 1)
            for (int i = tid; i < nkl * 4; i += T) sC[i] = ((const cplx*)P.i_red)[((int64_t)(i >> 2) * N1 + n) * 4 + (i & 3)];
    } else if (own) {
        // row chunks bc = 0 .. b/TB, then column chunks b/ts .. nf/ts (langreth: ts = TB)
        const int64_t rb = ((int64_t)kl * P.nbb * N1 + b) * 4 + c;   // [k][chunk][point][4]
        const int64_t cb = ((int64_t)kl * P.nsb * N1 + b) * 4 + c;
        const cplx* rowP = (const cplx*)P.row_part + rb;
        const cplx* colP = (const cplx*)P.col_part + cb;
        const cplx* gcP = (const cplx*)P.gc_part + rb;
        const cplx* gcC = LANG ? (const cplx*)P.gc_part_c + cb : nullptr;
        const int c0 = b / cts;
        const int nr = b / TB + 1, ns = nf / cts - c0 + 1;
        const int na = nr + ns, ng = b < nf ? (LANG ? nr + ns : nr) : 0;
        // UPD_BATCH independent loads per operand in flight before the in-order adds
        // (the sum order, and so the result, does not depend on the batch size)
        constexpr int UPD_BATCH = KBE_UPD_BATCH;
        cplx a = cz(), g = cz();
        // after an incremental evaluation every slot is base + delta (collision_kernel)
        const bool dl = INC && !LANG && ((const volatile kbe_ctl*)ctl)->incr_last;
        const fcx* rowD = dl ? (const fcx*)P.row_delta + rb : nullptr;
        const fcx* colD = dl ? (const fcx*)P.col_delta + cb : nullptr;
        const fcx* gcD = dl ? (const fcx*)P.gc_delta + rb : nullptr;
        for (int i0 = 0; i0 < na || i0 < ng; i0 += UPD_BATCH) {
            cplx va[UPD_BATCH], vg[UPD_BATCH];
#pragma unroll
            for (int u = 0; u < UPD_BATCH; ++u) {
                const int q = i0 + u;
                va[u] = q < na ? (q < nr ? rowP[q * cs] : colP[(c0 + q - nr) * cs]) : cz();
                vg[u] = q < ng ? (q < nr ? gcP[q * cs] : gcC[(c0 + q - nr) * cs]) : cz();
                if (dl) {
                    if (q < na) va[u] = cadd(va[u], f64(q < nr ? rowD[q * cs] : colD[(c0 + q - nr) * cs]));
                    if (q < ng) vg[u] = cadd(vg[u], f64(gcD[q * cs]));
                }
            }
#pragma unroll
            for (int u = 0; u < UPD_BATCH; ++u) {
                if (i0 + u < na) a = cadd(a, va[u]);
                if (i0 + u < ng) g = cadd(g, vg[u]);
            }
        }
        if (!LANG && b < nf)   // the frontier slice's column-direction sums (own slot)
            a = cadd(a, ((const cplx*)P.fcol_part)[((int64_t)kl * N1 + b) * 4 + c]);
        sA[(kl * PPC + o) * 4 + c] = a;
        sB[(kl * PPC + o) * 4 + c] = g;
    }
    if (diag_cta && !RED) {
        if (LANG) {
            // langreth: I> rows and I< columns are independent of I< rows / I> columns
            for (int k2 = tid; k2 < nkl; k2 += T) {
                if (phase == 0) {
                    reduce_gr(P, k2, n - 1, n - 1, sX + k2 * 4);   // greater_row_old[n-1]
                } else {
                    reduce_lc(P, k2, n - 1, n, sX + k2 * 4);       // lesser_col[n-1]
                    reduce_gr(P, k2, n - 1, n, sY + k2 * 4);       // greater_row[n-1]
                    reduce_gr(P, k2, n, n, sZ + k2 * 4);           // greater_row[n]
                }
            }
        }
        if (phase == 1) {
            // C = I<(t_n, t_n): thread = (k, entry cc, chunk lane q), PPC lanes per entry
            // (consecutive lanes: fixed xor-shuffle tree), one round over the CTA
            const int L = PPC;
            const int nrc = n / TB + 1;   // row chunks, then the one column chunk holding n
            const int cn = n / coll_ts(n, nkl, LANG);
            const int q = tid % L, cc = (tid / L) & 3, k2 = tid / (4 * L);
            cplx x = cz();
            if (k2 < nkl) {
                const cplx* rp = (const cplx*)P.row_part + (((int64_t)k2 * P.nbb * N1 + n) * 4 + cc);
                const cplx* cp = (const cplx*)P.col_part + (((int64_t)k2 * P.nsb * N1 + n) * 4 + cc);
                for (int i0 = q; i0 <= nrc; i0 += 4 * L) {
                    cplx v[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int qq = i0 + L * u;
                        v[u] = qq < nrc ? rp[qq * cs] : (qq == nrc ? cp[cn * cs] : cz());
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (i0 + L * u <= nrc) x = cadd(x, v[u]);
                }
            }
            for (int off = 1; off < L; off <<= 1) {
                x.x += __shfl_xor_sync(0xffffffffu, x.x, off);
                x.y += __shfl_xor_sync(0xffffffffu, x.y, off);
            }
            if (k2 < nkl && q == 0) sC[k2 * 4 + cc] = x;
        }
    }
    __syncthreads();

    // ---- phase B: row / column update of the own points ----------------------------------
    const int64_t pm = sharded(P) ? plane_len(P.n_steps) : 0;
    const unsigned long long e_next = P.p2p_world > 1 ? p2p_epoch(P) + 1 : 0;   // data epoch this update publishes
    double res = 0.0;
    bool fin = true;
    if (own) {
        const cplx* A = sA + (kl * PPC + o) * 4;
        const cplx* B = sB + (kl * PPC + o) * 4;
        // predictor column input: I>(t_b, t_{n-1}); b = n-1 takes greater_row[n-1]
        // (= -lesser_row as printed; the langreth reduction otherwise)
        auto IC0 = [&](int q) -> cplx {
            if (b < n - 1) return B[q];
            return LANG ? sX[kl * 4 + q] : cneg(A[q]);
        };
        if (phase == 0) {
            lro[c] = A[c];
            clo[c] = IC0(c);
        }
        // row(i,j) = sum_k Phi(i,k) [G<(n-1,b)(k,j) - i dt ir(k,j)]
        // col(i,j) = sum_k [G>(b,n-1)(i,k) + i dt ic(i,k)] conj(Phi(j,k))
        cplx row = cz(), col = cz();
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const cplx ir = phase == 0 ? A[k * 2 + j] : cscale(cadd(olr[k], A[k * 2 + j]), 0.5);
            const cplx ic = phase == 0 ? IC0(i * 2 + k) : cscale(cadd(ocl[k], B[i * 2 + k]), 0.5);
            row = cfma(phr[k], csub(pgl[k], cmul_pi(ir, dt)), row);
            col = cfma_cb(cadd(pgu[k], cmul_pi(ic, dt)), phc[k], col);
        }
        if (phase == 1) {
            const double d1 = hypot(row.x - ol.x, row.y - ol.y), d2 = hypot(col.x - ou.x, col.y - ou.y);
            res = (d1 != d1 || res != res) ? nan : fmax(res, d1);
            res = (d2 != d2 || res != res) ? nan : fmax(res, d2);
            fin = fin && isfinite(row.x) && isfinite(row.y) && isfinite(col.x) && isfinite(col.y);
        }
        if (b == n - 1) { sRow[kl * 4 + c] = row; sCol[kl * 4 + c] = col; }
        if (INC && phase == 0)   // slice n-1 is final: complex64 shadow
            write_shadow((const cplx*)P.g_hist, (const cplx*)P.s_hist, (float2*)P.g_sh, (float2*)P.s_sh, P.tri, kl,
                         n - 1, c, b);
        cur[sl_idx(c, b)] = row;
        cur[sl_idx(4 + c, b)] = col;
        publish_entry(P, kl, c, b, row, pm, e_next);
        publish_entry(P, kl, 4 + c, b, col, pm, e_next);
    }
    if (diag_cta) {
        __syncthreads();   // sRow / sCol of point n-1
        for (int item = tid; item < nkl * 4; item += T) {
            // equal-time diagonal b = n, one block entry (j, m) per item; each item also
            // forms the transposed entry it needs for the anti-Hermitian part.  Same
            // operation order as the 2x2 helpers.
            const int e = item & 3, kl = item >> 2;
            const int dj = e >> 1, dm = e & 1;
            cplx* G = (cplx*)P.g_hist + (int64_t)kl * P.tri;
            const cplx* prev = G + slice_off(n - 1);
            cplx* cur = G + slice_off(n);
            const cplx* ph = (const cplx*)P.phi + ((int64_t)n * nkl + kl) * 4;
            auto PH = [&](int r, int c2) -> cplx { return ph[r * 2 + c2]; };
            auto sandwich = [&](const cplx* X, int r, int q) -> cplx {   // (Phi X Phi^dag)(r, q)
                cplx t0 = cfma(PH(r, 1), X[2], cfma(PH(r, 0), X[0], cz()));
                cplx t1 = cfma(PH(r, 1), X[3], cfma(PH(r, 0), X[1], cz()));
                return cfma_cb(t1, PH(q, 1), cfma_cb(t0, PH(q, 0), cz()));
            };
            auto ah = [](cplx x, cplx y) -> cplx {   // (x - conj(y)) / 2
                return make_double2(0.5 * (x.x - y.x), 0.5 * (x.y + y.y));
            };
            cplx nl, nu;
            if (phase == 0) {
                cplx gl[4], gu[4];
                load_cell(prev, n - 1, gl, gu);
                nl = ah(sandwich(gl, dj, dm), sandwich(gl, dm, dj));
                nu = ah(sandwich(gu, dj, dm), sandwich(gu, dm, dj));
            } else {
                const int o1 = (n - 1) - b0;
                const cplx* A1 = sA + (kl * PPC + o1) * 4;
                const cplx* B1 = sB + (kl * PPC + o1) * 4;
                const cplx* C = sC + kl * 4;
                // src_l = mirror(row) - i dt (lesser_col[n-1] + lesser_row[n]) / 2
                auto srcl = [&](int r, int q) -> cplx {
                    const cplx ml = cneg(cconj(sRow[kl * 4 + q * 2 + r]));
                    const cplx lc1 = LANG ? sX[kl * 4 + r * 2 + q] : cneg(B1[r * 2 + q]);
                    return csub(ml, cmul_pi(cscale(cadd(lc1, C[r * 2 + q]), 0.5), dt));
                };
                // src_g = mirror(col) + i dt (greater_row[n-1] + greater_row[n]) / 2
                auto srcg = [&](int r, int q) -> cplx {
                    const cplx mg = cneg(cconj(sCol[kl * 4 + q * 2 + r]));
                    const cplx gr1 = LANG ? sY[kl * 4 + r * 2 + q] : cneg(A1[r * 2 + q]);
                    const cplx gr2 = LANG ? sZ[kl * 4 + r * 2 + q] : cneg(C[r * 2 + q]);
                    return cadd(mg, cmul_pi(cscale(cadd(gr1, gr2), 0.5), dt));
                };
                auto dl = [&](int r, int q) -> cplx {   // (Phi src_l)(r, q)
                    return cfma(PH(r, 1), srcl(1, q), cfma(PH(r, 0), srcl(0, q), cz()));
                };
                auto dg = [&](int r, int q) -> cplx {   // (src_g Phi^dag)(r, q)
                    return cfma_cb(srcg(r, 1), PH(q, 1), cfma_cb(srcg(r, 0), PH(q, 0), cz()));
                };
                nl = ah(dl(dj, dm), dl(dm, dj));
                nu = ah(dg(dj, dm), dg(dm, dj));
                const cplx ol = cur[sl_idx(e, n)], ou = cur[sl_idx(4 + e, n)];
                const double d1 = hypot(nl.x - ol.x, nl.y - ol.y), d2 = hypot(nu.x - ou.x, nu.y - ou.y);
                res = (d1 != d1 || res != res) ? nan : fmax(res, d1);
                res = (d2 != d2 || res != res) ? nan : fmax(res, d2);
                fin = fin && isfinite(nl.x) && isfinite(nl.y) && isfinite(nu.x) && isfinite(nu.y);
            }
            cur[sl_idx(e, n)] = nl;
            cur[sl_idx(4 + e, n)] = nu;
            publish_entry(P, kl, e, n, nl, pm, e_next);
            publish_entry(P, kl, 4 + e, n, nu, pm, e_next);
        }
    }
    if (phase == 1) {
        const int lane = tid & 31, warp = tid >> 5, nw = (T + 31) >> 5;
        for (int off = 16; off > 0; off >>= 1) {
            const double other = __shfl_xor_sync(0xffffffffu, res, off);
            res = (res != res || other != other) ? nan : fmax(res, other);
        }
        const unsigned ballot = __ballot_sync(0xffffffffu, !fin);
        if (lane == 0) { red[warp] = res; redf[warp] = ballot != 0; }
        __syncthreads();
        if (tid == 0) {
            double r = red[0];
            int nfl = redf[0];
            for (int w = 1; w < nw; ++w) {
                r = (r != r || red[w] != red[w]) ? nan : fmax(r, red[w]);
                nfl |= redf[w];
            }
            const unsigned long long bits = (r != r) ? 0x7ff8000000000000ull : (unsigned long long)__double_as_longlong(r);
            atomicMax(&ctl->res[it], bits);
            if (nfl) atomicOr(&ctl->nonfinite[it], 1);
        }
    }
    if (next_iter || sharded(P)) {
        // the last CTA to finish sees the complete local record:
        //  - graph mode (kbe_run): decides whether the next corrector iteration's
        //    conditional body runs (propagator.py:360-368: continue while
        //    residual > eps, NaN included, up to max_iter);
        //  - k-sharded: publishes the record as this rank's control tail (NCCL send
        //    buffer, or every peer's buffer + the epoch flags)
        if (P.p2p_world > 1) __threadfence_system();   // this thread's peer stores
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            if (atomicAdd(&ctl->upd_done, 1u) == gridDim.x - 1) {
                ctl->upd_done = 0;
                __threadfence();
                if (next_iter && phase == 1) {
                    const double rall = __longlong_as_double((long long)atomicOr(&ctl->res[it], 0ull));
                    if (!(rall <= P.eps)) cudaGraphSetConditional(next_iter, 1u);
                }
                if (sharded(P)) {
                    KbeTail t;
                    for (int i = 0; i < KBE_MAX_ITER; ++i) {
                        t.res[i] = atomicOr(&ctl->res[i], 0ull);
                        t.nonfinite[i] = atomicOr(&ctl->nonfinite[i], 0);
                    }
                    publish_tail(P, t, e_next);
                }
            }
        }
    }
}

// Phi(t_{n-1/2}, k) for steps n in [n0, n1], local k (hf term from ctl->hf_sum when hf_mode="on")
__global__ void phi_table_kernel(kbe_problem P, int n0, int n1, int it, int check_skip) {
    pdl_enter();
    kbe_ctl* ctl = (kbe_ctl*)P.ctl;
    if (check_skip && kbe_skip(P, ctl, it)) return;
    const int nkl = P.k_hi - P.k_lo;
    const int64_t total = (int64_t)(n1 - n0 + 1) * nkl;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int n = n0 + (int)(i / nkl), kl = (int)(i % nkl);
        cplx phi[4];
        build_phi(P, ctl, n, P.k_lo + kl, phi);
        cplx* dst = (cplx*)P.phi + ((int64_t)n * nkl + kl) * 4;
#pragma unroll
        for (int c = 0; c < 4; ++c) dst[c] = phi[c];
    }
}

// hf_mode="on": k-sum of rho(t_{n-1}) (phase 0) or of (rho(t_{n-1}) + rho(t_n))/2 (phase 1)
__global__ void hf_mean_kernel(kbe_problem P, int n, int phase, int it) {
    pdl_enter();
    kbe_ctl* ctl = (kbe_ctl*)P.ctl;
    if (phase == 0 ? kbe_halted(ctl) : kbe_skip(P, ctl, it)) return;
    const int nloc = P.k_hi - P.k_lo;
    if (threadIdx.x == 0) {
        cplx acc[4] = {cz(), cz(), cz(), cz()};
        for (int kl = 0; kl < nloc; ++kl) {
            const cplx* G = (const cplx*)P.g_hist + (int64_t)kl * P.tri;
            const cplx* a = G + slice_off(n - 1);
            for (int c = 0; c < 4; ++c) {
                const cplx g0 = a[sl_idx(c, n - 1)];
                cplx r = make_double2(g0.y, -g0.x);   // rho = -i G<
                if (phase == 1) {
                    const cplx* bcur = G + slice_off(n);
                    const cplx g1 = bcur[sl_idx(c, n)];
                    r = cscale(cadd(r, make_double2(g1.y, -g1.x)), 0.5);
                }
                acc[c] = cadd(acc[c], r);
            }
        }
        for (int c = 0; c < 4; ++c) ctl->hf_sum[c] = acc[c];
    }
    if (P.front_all) return;   // k-sharded: the host all-reduces hf_sum, then kbe_build_phi
    __syncthreads();
    for (int kl = threadIdx.x; kl < nloc; kl += blockDim.x) {
        cplx phi[4];
        build_phi(P, ctl, n, P.k_lo + kl, phi);
        cplx* dst = (cplx*)P.phi + ((int64_t)n * nloc + kl) * 4;
        for (int c = 0; c < 4; ++c) dst[c] = phi[c];
    }
}

// =================================================================== K4: finish
// m_launched: corrector iterations launched for this step (< max_iter: kbe_run_iters)
__global__ void finish_kernel(kbe_problem P, int n, int m_launched) {
    pdl_enter();
    p2p_wait(P);
    kbe_ctl* ctl = (kbe_ctl*)P.ctl;
    if (kbe_halted(ctl)) return;
    const int nloc = P.k_hi - P.k_lo;
    __shared__ double dens[256];
    __shared__ double drift[256];
    __shared__ double en[256];
    __shared__ double rho[256][4];
    // one-body energy at the grid point t_n: h0(k; t_n) from the band tables, U(t_n) and the
    // pulse amplitude at t_n (the step-n midpoint table: both round to grid point n,
    // model.py:88-103), build_h (model.py:123-152) without the hf term, which the host adds
    // from the k-sums of rho (it needs the global k-mean)
    const double u_n = P.u_table[n], amp = P.amp[n];
    for (int kl = threadIdx.x; kl < nloc; kl += blockDim.x) {
        const cplx* c = (const cplx*)P.g_hist + (int64_t)kl * P.tri + slice_off(n);
        cplx gl[4], gu[4];
        for (int i = 0; i < 4; ++i) { gl[i] = c[sl_idx(i, n)]; gu[i] = c[sl_idx(4 + i, n)]; }
        double d = 0.0;
        for (int i = 0; i < 4; ++i) {
            cplx t = csub(gu[i], gl[i]);
            if (i == 0 || i == 3) t.y += 1.0;
            d = fmax(d, hypot(t.x, t.y));
        }
        // rho = -i G<(t_n, t_n) (propagator.py:272-273)
        cplx r[4];
        for (int i = 0; i < 4; ++i) r[i] = make_double2(gl[i].y, -gl[i].x);
        const int k = P.k_lo + kl;
        const cplx h01 = make_double2(amp * P.dipole_re, -amp * P.dipole_im);   // amp conj(d)
        const cplx h10 = make_double2(amp * P.dipole_re, amp * P.dipole_im);    // amp d
        // Re Tr[h0 rho] = h00 rho00 + h01 rho10 + h10 rho01 + h11 rho11
        const double e = P.eps_v[k] * r[0].x + cmul(h01, r[2]).x + cmul(h10, r[1]).x + (P.eps_c[k] - u_n) * r[3].x;
        if (kl < 256) {
            dens[kl] = gl[0].y + gl[3].y;
            drift[kl] = d;
            en[kl] = e;
            rho[kl][0] = r[0].x;
            rho[kl][1] = r[3].x;
            rho[kl][2] = r[1].x;
            rho[kl][3] = r[1].y;
        }
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    double ds = 0.0, dm = 0.0, es = 0.0, rs[4] = {0.0, 0.0, 0.0, 0.0};
    for (int kl = 0; kl < nloc && kl < 256; ++kl) {
        ds += dens[kl];
        dm = fmax(dm, drift[kl]);
        es += en[kl];
        for (int i = 0; i < 4; ++i) rs[i] += rho[kl][i];
    }
    int iters = P.max_iter, conv = 0;
    for (int i = 0; i < m_launched; ++i)
        if (__longlong_as_double((long long)res_bits(P, ctl, i)) <= P.eps) { iters = i + 1; conv = 1; break; }
    if (!conv && m_launched < P.max_iter) {   // more iterations needed than were launched
        ctl->needs_more = n;
        return;
    }
    double* r = P.reports + (int64_t)n * KBE_REPORT_W;
    const int nonfin = nonfinite_at(P, ctl, iters - 1);
    r[0] = n;
    r[1] = iters;
    r[2] = __longlong_as_double((long long)res_bits(P, ctl, iters - 1));
    r[3] = conv;
    r[4] = dm;
    r[5] = ds;
    r[6] = nonfin;
    r[7] = es;
    for (int i = 0; i < KBE_MAX_ITER; ++i)
        r[8 + i] = i < iters ? __longlong_as_double((long long)res_bits(P, ctl, i)) : 0.0;
    for (int i = 0; i < 4; ++i) r[8 + KBE_MAX_ITER + i] = rs[i];
    if (nonfin) ctl->poisoned = n;
}

// Initial slice to every peer (kbe_p2p_publish): copy front_send's chunk into every
// peer's buffer at the next epoch, then the last CTA signals.
__global__ void p2p_publish_kernel(kbe_problem P) {
    pdl_enter();
    kbe_ctl* ctl = (kbe_ctl*)P.ctl;
    const unsigned long long e = p2p_epoch(P) + 1;
    const int64_t chunk = front_chunk(P);
    const cplx* src = (const cplx*)P.front_send;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < chunk; i += (int64_t)gridDim.x * blockDim.x) {
        const cplx v = src[i];
#pragma unroll
        for (int r = 0; r < KBE_MAX_RANKS; ++r)
            if (r < P.p2p_world) p2p_dst(P, r, e)[i] = v;
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(&ctl->upd_done, 1u) == gridDim.x - 1) {
        ctl->upd_done = 0;
        p2p_signal(P, e);
    }
}

// =================================================================== init / pack / unpack
__global__ void init_slice0_kernel(kbe_problem P) {
    pdl_enter();
    const int kl = blockIdx.x * blockDim.x + threadIdx.x;
    if (kl < P.k_hi - P.k_lo) {
        cplx* g = (cplx*)P.g_hist + (int64_t)kl * P.tri;   // slice 0
        g[sl_idx(0, 0)] = make_double2(0.0, 1.0);     // G<(0,0)_00 = i
        g[sl_idx(7, 0)] = make_double2(0.0, -1.0);    // G>(0,0)_11 = -i
        if (P.front_send) {                     // slice 0 of the all-gather send buffer
            const int64_t pm = plane_len(P.n_steps);
            cplx* fs = (cplx*)P.front_send + (int64_t)kl * 8 * pm;
            for (int c = 0; c < 8; ++c) fs[sl_idx(c, 0)] = g[sl_idx(c, 0)];
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        kbe_ctl* ctl = (kbe_ctl*)P.ctl;
        memset(ctl, 0, sizeof(kbe_ctl));
    }
}

__global__ void unpack_kernel(const cplx* hist, int64_t tri, int kloc, int N, int frontier, int which, cplx* out) {
    const int64_t N1 = N + 1;
    const int64_t total = (int64_t)kloc * 4 * N1 * N1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int tp = (int)(i % N1);
        const int t = (int)((i / N1) % N1);
        const int jm = (int)((i / (N1 * N1)) & 3);
        const int kl = (int)(i / (N1 * N1 * 4));
        const int j = jm >> 1, m = jm & 1;
        const cplx* h = hist + kl * tri;
        cplx v = cz();
        if (t <= frontier && tp <= frontier) {
            if (which == 0) {   // lower-stored: X(t,tp) = L(t,tp) for t >= tp
                if (t >= tp) v = h[slice_off(t) + sl_idx(jm, tp)];
                else v = cneg(cconj(h[slice_off(tp) + sl_idx(m * 2 + j, t)]));
            } else {            // upper-stored: Y(t,tp) = U(tp,t) for t <= tp
                if (t <= tp) v = h[slice_off(tp) + sl_idx(4 + jm, t)];
                else v = cneg(cconj(h[slice_off(t) + sl_idx(4 + m * 2 + j, tp)]));
            }
        }
        out[i] = v;
    }
}

// G^R(t, t') = theta(t - t') [G>(t, t') - G<(t, t')] (SURVEY finding 2: a derived accessor,
// the reference has none), theta(0) = theta0 on the equal-time diagonal; zero above the
// diagonal and beyond slice `frontier`.  Reads both triangles of the packed G history.
__global__ void unpack_retarded_kernel(const cplx* hist, int64_t tri, int kloc, int N, int frontier, double theta0,
                                       cplx* out) {
    const int64_t N1 = N + 1;
    const int64_t total = (int64_t)kloc * 4 * N1 * N1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int tp = (int)(i % N1);
        const int t = (int)((i / N1) % N1);
        const int jm = (int)((i / (N1 * N1)) & 3);
        const int kl = (int)(i / (N1 * N1 * 4));
        const int j = jm >> 1, m = jm & 1;
        const cplx* h = hist + kl * tri + slice_off(t);
        cplx v = cz();
        if (t <= frontier && tp <= t) {
            const cplx gl = h[sl_idx(jm, tp)];                                   // G<(t, tp), lower-stored
            const cplx gg = t == tp ? h[sl_idx(4 + jm, t)]                       // G>(t, t)
                                    : cneg(cconj(h[sl_idx(4 + m * 2 + j, tp)]));  // -G>(tp, t)^dagger
            v = cscale(csub(gg, gl), t == tp ? theta0 : 1.0);
        }
        out[i] = v;
    }
}

__global__ void pack_kernel(const cplx* lower, const cplx* upper, int kloc, int N, int frontier, int64_t tri, cplx* hist) {
    const int64_t N1 = N + 1;
    const int64_t per_k = slice_off(frontier + 1);
    const int64_t total = (int64_t)kloc * per_k;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int kl = (int)(i / per_k);
        const int64_t off = i % per_k;
        // find slice s with slice_off(s) <= off < slice_off(s+1)
        int lo = 0, hi = frontier;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (slice_off(mid) <= off) lo = mid; else hi = mid - 1;
        }
        const int s = lo;
        const int64_t o = off - slice_off(s);
        const int c = (int)((o >> 5) & 7);
        const int b = (int)(((o >> 8) << 5) + (o & 31));
        cplx v = cz();
        if (b <= s) {
            if (c < 4) v = lower[(((int64_t)kl * 4 + c) * N1 + s) * N1 + b];
            else v = upper[(((int64_t)kl * 4 + (c - 4)) * N1 + b) * N1 + s];
        }
        hist[kl * tri + off] = v;
    }
}

// =================================================================== host side
// Every step-kernel launch is first described as a KSpec (function, grid, block,
// shared memory, argument block).  The same spec is either launched on a stream
// with programmatic stream serialization (see pdl_enter; KBE_NO_PDL=1 falls back
// to plain stream order for A/B timing) or written into a kernel node of the
// step graph (kbe_run).
struct KSpec {
    const void* func = nullptr;
    dim3 grid, block;
    size_t smem = 0;
    alignas(16) unsigned char buf[sizeof(kbe_problem) + 64];
    void* args[8];
};
template <typename... A, size_t... I>
static void spec_pack(KSpec& s, std::index_sequence<I...>, A... a) {
    size_t off = 0;
    auto put = [&](auto v, size_t i) {
        using T = decltype(v);
        off = (off + alignof(T) - 1) / alignof(T) * alignof(T);
        memcpy(s.buf + off, &v, sizeof(T));
        s.args[i] = s.buf + off;
        off += sizeof(T);
    };
    (put(a, I), ...);
}
template <typename... KArgs, typename... Args>
static void make_spec(KSpec& s, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, Args... args) {
    static_assert(sizeof...(KArgs) == sizeof...(Args), "kernel argument count");
    s.func = (const void*)kernel;
    s.grid = grid;
    s.block = block;
    s.smem = smem;
    spec_pack<KArgs...>(s, std::index_sequence_for<KArgs...>{}, static_cast<KArgs>(args)...);
}
static int g_pdl = -1;
static cudaError_t launch_spec(const KSpec& s, void* stream) {
    if (g_pdl < 0) {
        const char* e = getenv("KBE_NO_PDL");
        g_pdl = (e && e[0] == '1') ? 0 : 1;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = s.grid;
    cfg.blockDim = s.block;
    cfg.dynamicSmemBytes = s.smem;
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = g_pdl ? 1 : 0;
    return cudaLaunchKernelExC(&cfg, s.func, (void**)s.args);
}
static cudaKernelNodeParams node_params(const KSpec& s) {
    cudaKernelNodeParams kp = {};
    kp.func = (void*)s.func;
    kp.gridDim = s.grid;
    kp.blockDim = s.block;
    kp.sharedMemBytes = (unsigned)s.smem;
    kp.kernelParams = (void**)s.args;
    kp.extra = nullptr;
    return kp;
}
#define KBE_LAUNCH_SPEC(name, spec)                                        \
    do {                                                                   \
        cudaError_t e_ = launch_spec(spec, stream);                        \
        if (e_ != cudaSuccess) { set_err(name, e_); return KBE_ERR_CUDA; } \
    } while (0)
static bool g_attr_done = false;
static int g_num_sms = 148;
static int g_coll_occ = 8;   // resident collision CTAs per SM (occupancy API)
static int g_lang_occ = 8;
static int ensure_attrs() {
    if (g_attr_done) return KBE_OK;
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e = cudaFuncSetAttribute(sigma_frontier_kernel<4, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(sigma_frontier_kernel<2, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(sigma_frontier_kernel<4, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(sigma_frontier_kernel<2, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) { set_err("cudaFuncSetAttribute(sigma_frontier)", e); return KBE_ERR_CUDA; }
    if (e == cudaSuccess) e = cudaFuncSetAttribute(sigma_dft_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
#define KBE_FFT_ATTR(L) if (e == cudaSuccess) e = cudaFuncSetAttribute(sigma_fft_kernel<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    KBE_FFT_LGS(KBE_FFT_ATTR)
#undef KBE_FFT_ATTR
    if (e != cudaSuccess) { set_err("cudaFuncSetAttribute(sigma_fft)", e); return KBE_ERR_CUDA; }
    e = cudaFuncSetAttribute(collision_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(CollSmem));
    if (e != cudaSuccess) { set_err("cudaFuncSetAttribute(collision)", e); return KBE_ERR_CUDA; }
    e = cudaFuncSetAttribute(collision_langreth_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(CollSmemL));
    if (e != cudaSuccess) { set_err("cudaFuncSetAttribute(collision_langreth)", e); return KBE_ERR_CUDA; }
    int occ = 0, occ2 = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, collision_langreth_kernel, 32, sizeof(CollSmemL));
    if (e != cudaSuccess || occ2 < 1) { set_err("cudaOccupancyMaxActiveBlocksPerMultiprocessor(langreth)", e); return KBE_ERR_CUDA; }
    g_lang_occ = occ2;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, collision_kernel, 32, sizeof(CollSmem));
    if (e != cudaSuccess || occ < 1) { set_err("cudaOccupancyMaxActiveBlocksPerMultiprocessor(collision)", e); return KBE_ERR_CUDA; }
    g_coll_occ = occ;
    {
        void (*upd[5])(kbe_problem, int, int, int, int, cudaGraphConditionalHandle) = {
            update_kernel<0, 0, 0>, update_kernel<1, 0, 0>, update_kernel<0, 1, 0>, update_kernel<0, 0, 1>,
            update_kernel<0, 1, 1>};
        for (int i = 0; i < 5; ++i) {
            e = cudaFuncSetAttribute(upd[i], cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
            if (e != cudaSuccess) { set_err("cudaFuncSetAttribute(update)", e); return KBE_ERR_CUDA; }
        }
    }
    e = cudaFuncSetAttribute(sigma_slice_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) { set_err("cudaFuncSetAttribute(sigma_slice)", e); return KBE_ERR_CUDA; }
    g_attr_done = true;
    return KBE_OK;
}

static int check_problem(const kbe_problem* p) {
    if (!p || p->n_k < 2 || (p->n_k & 1) || p->k_lo < 0 || p->k_hi > p->n_k || p->k_hi <= p->k_lo ||
        p->n_steps < 1 || p->max_iter < 1 || p->max_iter > KBE_MAX_ITER || !p->g_hist || !p->s_hist || !p->ctl) {
        set_err("kbe_problem", cudaSuccess);
        return KBE_ERR_ARG;
    }
    if (p->limit_mode != 0 && (!p->row_part_g || !p->col_part_g || !p->lc_part || !p->gc_part_c || !p->lc_part_c)) {
        snprintf(g_err, sizeof(g_err), "limit_mode 'langreth' needs the langreth partial buffers");
        return KBE_ERR_ARG;
    }
    if (p->n_k > KBE_MAX_NK) {
        snprintf(g_err, sizeof(g_err), "n_k > %d is not supported by the Sigma kernel (one stage-2 task per thread)",
                 KBE_MAX_NK);
        return KBE_ERR_UNSUPPORTED;
    }
    if (!p->phi) { set_err("kbe_problem.phi", cudaSuccess); return KBE_ERR_ARG; }
    if ((!p->limit_mode && !p->fcol_part) ||
        (p->g_sh && (!p->s_sh || !p->v_prev || !p->row_delta || !p->col_delta || !p->gc_delta))) {
        snprintf(g_err, sizeof(g_err), "kbe_problem: fcol_part / incremental-evaluation buffers missing");
        return KBE_ERR_ARG;
    }
    if (p->p2p_world > 1 && (p->p2p_world > KBE_MAX_RANKS || !p->p2p_local || p->p2p_rank < 0 ||
                             p->p2p_rank >= p->p2p_world || p->n_k % p->p2p_world ||
                             (p->k_hi - p->k_lo) * p->p2p_world != p->n_k)) {
        snprintf(g_err, sizeof(g_err), "kbe_problem: inconsistent peer-to-peer rank set");
        return KBE_ERR_ARG;
    }
    return KBE_OK;
}

// ---- launch specs of the step kernels (shared by the stream and graph paths)
// K1 variant: KBE_SIGMA = fft (default for power-of-two n_k) | dft (DMMA DFT GEMMs, the
// default otherwise) | direct (the O(n_k^2) correlation kernel), for A/B runs
static int g_sigma_kind = -1;   // 0 auto, 1 fft, 2 dft, 3 direct
static void spec_sigma(KSpec& s, const kbe_problem* p, int n, int it) {
    if (g_sigma_kind < 0) {
        const char* e = getenv("KBE_SIGMA");
        g_sigma_kind = !e ? 0 : !strcmp(e, "fft") ? 1 : !strcmp(e, "dft") ? 2 : !strcmp(e, "direct") ? 3 : 0;
    }
    // auto: FFT for powers of two, except the dimer (n_k = 2), where the whole run is 5 %
    // faster with the correlation kernel (profiles/r02/bench_cfg1_variants.jsonl: both
    // are latency-bound there and the correlations have fewer CTA barriers)
    const bool fft = sigma_fft_ok(p->n_k) && (g_sigma_kind == 1 || (g_sigma_kind == 0 && p->n_k > 2));
    if (!fft && g_sigma_kind != 3 && !(g_sigma_kind == 0 && p->n_k == 2)) {
        const int pb = sigma_dft_pb(p->n_k, n + 1, g_num_sms);
        make_spec(s, sigma_dft_kernel, dim3((n + 1 + pb - 1) / pb), dim3(SIGMA_THREADS), sigma_dft_smem(p->n_k, pb),
                  *p, n, it, pb);
        return;
    }
    if (fft) {
        const int pb = sigma_fft_pb(p->n_k, n + 1, g_num_sms);
        const dim3 grid((n + 1 + pb - 1) / pb), block(SIGMA_THREADS);
        const size_t smem = sigma_fft_smem(p->n_k, pb);
        switch (ilog2(p->n_k)) {
#define KBE_FFT_CASE(L) case L: make_spec(s, sigma_fft_kernel<L>, grid, block, smem, *p, n, it, pb); return;
            KBE_FFT_LGS(KBE_FFT_CASE)
#undef KBE_FFT_CASE
        }
    }
    const int hb = sigma_hb_launch(p->n_k, 2 * (n + 1), g_num_sms);
    const dim3 grid((2 * (n + 1) + hb - 1) / hb);
    const size_t smem = (size_t)hb * SgDims(p->n_k).per * sizeof(cplx);
    // stage-1 tasks of the CTA (8 n_k / R per half-pair) and stage-2 tasks (8 NBL) fit 128 threads?
    const int R = sg_r(p->n_k), nkl = p->k_hi - p->k_lo;
    // (n_k >= 8: for the dimer-sized problems the 256-thread CTAs measured faster)
    const bool small = p->n_k >= 8 && hb * 8 * (p->n_k / R) <= 128 && hb * 8 * ((nkl + R - 1) / R) <= 128 &&
                       !KBE_SIG_NT256;
    if (R == 4) {
        if (small) make_spec(s, sigma_frontier_kernel<4, 128>, grid, dim3(128), smem, *p, n, it, hb);
        else make_spec(s, sigma_frontier_kernel<4, 256>, grid, dim3(256), smem, *p, n, it, hb);
    } else {
        if (small) make_spec(s, sigma_frontier_kernel<2, 128>, grid, dim3(128), smem, *p, n, it, hb);
        else make_spec(s, sigma_frontier_kernel<2, 256>, grid, dim3(256), smem, *p, n, it, hb);
    }
}
static void spec_collision(KSpec& s, const kbe_problem* p, int n, int it, bool after_sigma) {
    const int nkl = p->k_hi - p->k_lo;
    if (p->limit_mode) {
        const int T0 = n / TS + 1;
        const int64_t tl = 2 * (int64_t)(T0 * (T0 + 1) / 2) * nkl;
        const int64_t cl = (int64_t)g_num_sms * g_lang_occ;
        make_spec(s, collision_langreth_kernel, dim3((int)(tl < cl ? tl : cl)), dim3(32), sizeof(CollSmemL), *p, n, it);
        return;
    }
    const int64_t total = (int64_t)coll_tiles(n, nkl) * (TS / coll_ts(n, nkl, 0));
    const int64_t cap = (int64_t)g_num_sms * g_coll_occ;
    make_spec(s, collision_kernel, dim3((int)(total < cap ? total : cap)), dim3(32), sizeof(CollSmem), *p, n, it,
              after_sigma ? 1 : 0);
}
// K3 split into K3a (reduce_kernel) + K3b for as-printed problems with >= KBE_SPLIT_MIN_K
// local k-points (env KBE_SPLIT_MIN_K overrides, for A/B runs): below that the fused
// K3's partial sums are short and the extra launch costs more than it saves.
#ifndef KBE_SPLIT_MIN_K
#define KBE_SPLIT_MIN_K 8
#endif
static int g_split_min_k = -1;
static bool upd_split(const kbe_problem* p) {
    if (g_split_min_k < 0) {
        const char* e = getenv("KBE_SPLIT_MIN_K");
        g_split_min_k = e ? atoi(e) : KBE_SPLIT_MIN_K;
    }
    return !p->limit_mode && p->i_red && p->g_red && (p->k_hi - p->k_lo) >= g_split_min_k;
}
static void spec_reduce(KSpec& s, const kbe_problem* p, int n, int phase, int it) {
    const int64_t items = (int64_t)(p->k_hi - p->k_lo) * (((phase == 0 ? n : n + 1) + 7) / 8);
    const int64_t cap = (int64_t)g_num_sms * 3;   // resident CTAs (__launch_bounds__(256, 3))
    const dim3 grid((unsigned)std::min<int64_t>((items + 7) / 8, cap));
    if (p->g_sh) make_spec(s, reduce_kernel<1>, grid, dim3(256), 0, *p, n, phase, it);
    else make_spec(s, reduce_kernel<0>, grid, dim3(256), 0, *p, n, phase, it);
}
static void spec_update(KSpec& s, const kbe_problem* p, int n, int phase, int it, cudaGraphConditionalHandle next,
                        bool red = false) {
    const int nkl = p->k_hi - p->k_lo, ppc = upd_ppc(nkl, n);
    const dim3 grid((n + ppc - 1) / ppc), block(upd_threads(nkl, ppc));
    const size_t smem = upd_smem_bytes(nkl, ppc);
    if (p->limit_mode) make_spec(s, update_kernel<1, 0, 0>, grid, block, smem, *p, n, phase, it, ppc, next);
    else if (red && p->g_sh) make_spec(s, update_kernel<0, 1, 1>, grid, block, smem, *p, n, phase, it, ppc, next);
    else if (red) make_spec(s, update_kernel<0, 0, 1>, grid, block, smem, *p, n, phase, it, ppc, next);
    else if (p->g_sh) make_spec(s, update_kernel<0, 1, 0>, grid, block, smem, *p, n, phase, it, ppc, next);
    else make_spec(s, update_kernel<0, 0, 0>, grid, block, smem, *p, n, phase, it, ppc, next);
}
static void spec_hf(KSpec& s, const kbe_problem* p, int n, int phase, int it) {
    make_spec(s, hf_mean_kernel, dim3(1), dim3(128), 0, *p, n, phase, it);
}
static void spec_finish(KSpec& s, const kbe_problem* p, int n, int m_launched = -1) {
    make_spec(s, finish_kernel, dim3(1), dim3(256), 0, *p, n, m_launched < 0 ? p->max_iter : m_launched);
}

// ---- step graph (kbe_run, one rank) ---------------------------------------------------
// One executable graph per driver, replayed once per step with the kernel nodes'
// n-dependent arguments and grids rewritten (cudaGraphExecKernelNodeSetParams):
//
//   Sigma(n-1) -> I(n-1) [-> hf] -> predict -> Sigma(n) -> I(n) [-> hf] -> correct(0)
//   -> IF c1 { Sigma(n) -> I(n) [-> hf] -> correct(1) } -> ... -> IF c_{m-1} {...} -> finish
//
// correct(it)'s last CTA sets c_{it+1} = (residual > eps), so the corrector
// iterations after convergence are never launched (the stream path launches
// them as no-ops).  The handles default to 0 at every launch, so a step can
// never run more than max_iter iterations.  Kernel -> kernel edges inside one
// (sub)graph are programmatic (the PDL of the stream path); KBE_GRAPH_PDL=0
// makes them full dependencies.
enum { GR_SIGMA, GR_COLL, GR_HF, GR_UPD, GR_FIN };
struct GNode {
    cudaGraphNode_t node;
    int role, phase, it;           // it = -1: the n-1 evaluation
    cudaGraphConditionalHandle next;
};
struct StepGraph {
    kbe_problem key;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    GNode nodes[4 * (KBE_MAX_ITER + 1) + 2];
    int count = 0;
};
static StepGraph* g_graphs[8];
static int g_graph_pdl = -1;

static void fill_spec(KSpec& s, const kbe_problem* p, const GNode& g, int n) {
    const int nn = g.it < 0 ? n - 1 : n, it = g.it < 0 ? 0 : g.it;
    switch (g.role) {
        case GR_SIGMA: spec_sigma(s, p, nn, it); break;
        case GR_COLL: spec_collision(s, p, nn, it, true); break;
        case GR_HF: spec_hf(s, p, n, g.phase, it); break;
        case GR_UPD: spec_update(s, p, n, g.phase, it, g.next); break;
        default: spec_finish(s, p, n); break;
    }
}

// append a kernel node to `graph` after `prev` (nullptr: root); programmatic edge
// when both are kernel nodes of the same graph
static cudaError_t add_kernel(StepGraph* sg, cudaGraph_t graph, cudaGraphNode_t* prev, bool prev_is_kernel,
                              const kbe_problem* p, GNode g, int n) {
    KSpec s;
    fill_spec(s, p, g, n);
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeKernel;
    np.kernel.func = (void*)s.func;
    np.kernel.gridDim = s.grid;
    np.kernel.blockDim = s.block;
    np.kernel.sharedMemBytes = (unsigned)s.smem;
    np.kernel.kernelParams = (void**)s.args;
    cudaGraphEdgeData ed = {};
    if (prev_is_kernel && g_graph_pdl) {
        ed.from_port = cudaGraphKernelNodePortProgrammatic;
        ed.type = cudaGraphDependencyTypeProgrammatic;
    }
    cudaError_t e = cudaGraphAddNode_v2(&g.node, graph, *prev ? prev : nullptr, *prev ? &ed : nullptr,
                                        *prev ? 1 : 0, &np);
    if (e != cudaSuccess) return e;
    sg->nodes[sg->count++] = g;
    *prev = g.node;
    return cudaSuccess;
}

static void destroy_graph(StepGraph* sg) {
    if (!sg) return;
    if (sg->exec) cudaGraphExecDestroy(sg->exec);
    if (sg->graph) cudaGraphDestroy(sg->graph);
    delete sg;
}

static int build_graph(const kbe_problem* p, int n, StepGraph** out) {
    if (g_graph_pdl < 0) {
        const char* e = getenv("KBE_GRAPH_PDL");
        g_graph_pdl = (e && e[0] == '0') ? 0 : 1;
    }
    StepGraph* sg = new StepGraph();
    sg->key = *p;
    cudaError_t e = cudaGraphCreate(&sg->graph, 0);
#define GCHK(what)                                                              \
    if (e != cudaSuccess) { set_err(what, e); destroy_graph(sg); return KBE_ERR_CUDA; }
    GCHK("cudaGraphCreate");
    cudaGraphNode_t prev = nullptr;
    bool pk = false;   // prev is a kernel node of the same graph
    auto add = [&](cudaGraph_t gr, cudaGraphNode_t* pv, bool* pkk, int role, int phase, int it,
                   cudaGraphConditionalHandle next) {
        GNode g = {nullptr, role, phase, it, next};
        cudaError_t r = add_kernel(sg, gr, pv, *pkk, p, g, n);
        *pkk = true;
        return r;
    };
    // predictor part: Sigma(n-1), I(n-1), predict
    if (p->interacting && (e = add(sg->graph, &prev, &pk, GR_SIGMA, 0, -1, 0)) != cudaSuccess) GCHK("graph: sigma");
    if ((e = add(sg->graph, &prev, &pk, GR_COLL, 0, -1, 0)) != cudaSuccess) GCHK("graph: collision");
    if (p->hf && (e = add(sg->graph, &prev, &pk, GR_HF, 0, 0, 0)) != cudaSuccess) GCHK("graph: hf");
    if ((e = add(sg->graph, &prev, &pk, GR_UPD, 0, 0, 0)) != cudaSuccess) GCHK("graph: predict");
    // corrector iterations: 0 unconditionally, 1..max_iter-1 behind IF nodes
    cudaGraphConditionalHandle h[KBE_MAX_ITER] = {};
    for (int it = 1; it < p->max_iter; ++it) {
        e = cudaGraphConditionalHandleCreate(&h[it], sg->graph, 0, cudaGraphCondAssignDefault);
        GCHK("cudaGraphConditionalHandleCreate");
    }
    for (int it = 0; it < p->max_iter; ++it) {
        cudaGraph_t body = sg->graph;
        cudaGraphNode_t bprev = prev;
        bool bpk = pk;
        if (it > 0) {
            cudaGraphNodeParams cp = {};
            cp.type = cudaGraphNodeTypeConditional;
            cp.conditional.handle = h[it];
            cp.conditional.type = cudaGraphCondTypeIf;
            cp.conditional.size = 1;
            cudaGraphNode_t cnode;
            e = cudaGraphAddNode(&cnode, sg->graph, &prev, 1, &cp);
            GCHK("cudaGraphAddNode(conditional)");
            body = cp.conditional.phGraph_out[0];
            prev = cnode;
            pk = false;
            bprev = nullptr;
            bpk = false;
        }
        const cudaGraphConditionalHandle next = it + 1 < p->max_iter ? h[it + 1] : 0;
        if (p->interacting && (e = add(body, &bprev, &bpk, GR_SIGMA, 1, it, 0)) != cudaSuccess) GCHK("graph: sigma");
        if ((e = add(body, &bprev, &bpk, GR_COLL, 1, it, 0)) != cudaSuccess) GCHK("graph: collision");
        if (p->hf && (e = add(body, &bprev, &bpk, GR_HF, 1, it, 0)) != cudaSuccess) GCHK("graph: hf");
        if ((e = add(body, &bprev, &bpk, GR_UPD, 1, it, next)) != cudaSuccess) GCHK("graph: correct");
        if (it == 0) { prev = bprev; pk = bpk; }
    }
    if ((e = add(sg->graph, &prev, &pk, GR_FIN, 0, 0, 0)) != cudaSuccess) GCHK("graph: finish");
    e = cudaGraphInstantiate(&sg->exec, sg->graph, 0);
    GCHK("cudaGraphInstantiate");
#undef GCHK
    *out = sg;
    return KBE_OK;
}

static bool same_problem(const kbe_problem* a, const kbe_problem* b) { return memcmp(a, b, sizeof(kbe_problem)) == 0; }

static int get_graph(const kbe_problem* p, int n, StepGraph** out) {
    for (auto& g : g_graphs)
        if (g && same_problem(&g->key, p)) { *out = g; return KBE_OK; }
    // reuse the slot of the same control block (a rebuilt problem), else a free one,
    // else evict slot 0
    int slot = -1;
    for (int i = 0; i < 8 && slot < 0; ++i)
        if (g_graphs[i] && g_graphs[i]->key.ctl == p->ctl) slot = i;
    for (int i = 0; i < 8 && slot < 0; ++i)
        if (!g_graphs[i]) slot = i;
    if (slot < 0) slot = 0;
    if (g_graphs[slot]) {
        cudaDeviceSynchronize();
        destroy_graph(g_graphs[slot]);
        g_graphs[slot] = nullptr;
    }
    int rc = build_graph(p, n, &g_graphs[slot]);
    if (rc) return rc;
    *out = g_graphs[slot];
    return KBE_OK;
}

static int graph_step(StepGraph* sg, const kbe_problem* p, int n, void* stream) {
    for (int i = 0; i < sg->count; ++i) {
        KSpec s;
        fill_spec(s, p, sg->nodes[i], n);
        cudaKernelNodeParams kp = node_params(s);
        cudaError_t e = cudaGraphExecKernelNodeSetParams(sg->exec, sg->nodes[i].node, &kp);
        if (e != cudaSuccess) { set_err("cudaGraphExecKernelNodeSetParams", e); return KBE_ERR_CUDA; }
    }
    cudaError_t e = cudaGraphLaunch(sg->exec, (cudaStream_t)stream);
    if (e != cudaSuccess) { set_err("cudaGraphLaunch", e); return KBE_ERR_CUDA; }
    return KBE_OK;
}

extern "C" {

int kbe_abi_version(void) { return KBE_ABI_VERSION; }
int64_t kbe_plane_len(int32_t s) { return plane_len(s); }
int64_t kbe_slice_offset(int32_t s) { return slice_off(s); }
int64_t kbe_tri_size(int32_t n_steps) { return slice_off(n_steps + 1); }
int64_t kbe_ctl_bytes(void) { return (int64_t)sizeof(kbe_ctl); }
int64_t kbe_sizeof_problem(void) { return (int64_t)sizeof(kbe_problem); }
const char* kbe_last_error(void) { return g_err; }

int kbe_init_history(const kbe_problem* p, void* stream) {
    int rc = check_problem(p);
    if (rc) return rc;
    if ((rc = ensure_attrs())) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t bytes = (size_t)(p->k_hi - p->k_lo) * p->tri * sizeof(cplx);
    cudaError_t e = cudaMemsetAsync(p->g_hist, 0, bytes, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(p->s_hist, 0, bytes, st);
    if (e != cudaSuccess) { set_err("cudaMemsetAsync(history)", e); return KBE_ERR_CUDA; }
    const int nloc = p->k_hi - p->k_lo;
    KSpec s;
    make_spec(s, init_slice0_kernel, dim3((nloc + 127) / 128), dim3(128), 0, *p);
    KBE_LAUNCH_SPEC("init_slice0_kernel", s);
    const int64_t cnt = (int64_t)p->n_steps * nloc;
    make_spec(s, phi_table_kernel, dim3((int)((cnt + 255) / 256 < 4096 ? (cnt + 255) / 256 : 4096)), dim3(256), 0, *p,
              1, p->n_steps, 0, 0);
    KBE_LAUNCH_SPEC("phi_table_kernel", s);
    return KBE_OK;
}

int kbe_sigma_frontier(const kbe_problem* p, int32_t n, int32_t it, void* stream) {
    int rc = check_problem(p);
    if (rc) return rc;
    if (n < 0 || n > p->n_steps) { set_err("kbe_sigma_frontier: n", cudaSuccess); return KBE_ERR_ARG; }
    if (!sharded(*p) && (p->k_lo != 0 || p->k_hi != p->n_k)) {
        snprintf(g_err, sizeof(g_err), "kbe_sigma_frontier: a k-sharded rank needs the gathered frontier (front_all)");
        return KBE_ERR_ARG;
    }
    if ((rc = ensure_attrs())) return rc;
    KSpec s;
    spec_sigma(s, p, n, it);
    KBE_LAUNCH_SPEC("sigma_frontier_kernel", s);
    return KBE_OK;
}

int kbe_sigma_slice(int32_t n_k, int32_t nb, const void* g_primary, const void* g_reversed, const double* u1,
                    const double* u2, int32_t k_lo, int32_t k_hi, const void* pol_in, void* pol_out, void* s1_out,
                    void* s2_out, void* sigma_out, void* stream) {
    if (n_k < 2 || (n_k & 1) || nb < 0 || k_lo < 0 || k_hi > n_k || k_hi < k_lo || !g_primary || !g_reversed ||
        !u1 || !u2) {
        set_err("kbe_sigma_slice", cudaSuccess);
        return KBE_ERR_ARG;
    }
    if (nb == 0) return KBE_OK;
    int rc = ensure_attrs();
    if (rc) return rc;
    const size_t smem = (size_t)16 * n_k * sizeof(cplx);
    sigma_slice_kernel<<<nb, 256, smem, (cudaStream_t)stream>>>(
        n_k, nb, (const cplx*)g_primary, (const cplx*)g_reversed, u1, u2, k_lo, k_hi, (const cplx*)pol_in,
        (cplx*)pol_out, (cplx*)s1_out, (cplx*)s2_out, (cplx*)sigma_out);
    KBE_CHECK_LAUNCH("sigma_slice_kernel");
    return KBE_OK;
}

static int launch_collision(const kbe_problem* p, int n, int it, bool after_sigma, void* stream) {
    int rc = check_problem(p);
    if (rc) return rc;
    if (n < 0 || n > p->n_steps) { set_err("kbe_collision_frontier: n", cudaSuccess); return KBE_ERR_ARG; }
    if ((rc = ensure_attrs())) return rc;
    KSpec s;
    spec_collision(s, p, n, it, after_sigma);
    KBE_LAUNCH_SPEC(p->limit_mode ? "collision_langreth_kernel" : "collision_kernel", s);
    return KBE_OK;
}
int kbe_collision_frontier(const kbe_problem* p, int32_t n, int32_t it, void* stream) {
    return launch_collision(p, n, it, false, stream);
}

int kbe_collision_slice(const kbe_problem* p, int32_t n, void* lesser_row, void* greater_row, void* lesser_col,
                        void* greater_col, void* stream) {
    int rc = check_problem(p);
    if (rc) return rc;
    KSpec s;
    make_spec(s, collision_slice_kernel, dim3((n + 1 + 127) / 128, p->k_hi - p->k_lo), dim3(128), 0, *p, (int)n,
              (cplx*)lesser_row, (cplx*)greater_row, (cplx*)lesser_col, (cplx*)greater_col);
    KBE_LAUNCH_SPEC("collision_slice_kernel", s);
    return KBE_OK;
}

int kbe_collision_row(int32_t n_k, int32_t T, int32_t P, int32_t T1, int32_t T2, int32_t w2_matrix,
                      const void* dg_first, const void* g_first, const void* s_like, const void* s_other,
                      const double* w1, const double* w2, void* out, void* stream) {
    if (n_k < 1 || T < 0 || P < 0 || T1 < 0 || T1 > T || T2 < 0 || T2 > T || (w2_matrix && T2 != T) ||
        !dg_first || !g_first || !s_like || !s_other || !out || (T1 && !w1) || (T2 && !w2)) {
        set_err("kbe_collision_row", cudaSuccess);
        return KBE_ERR_ARG;
    }
    const int64_t total = (int64_t)n_k * 2 * P;
    if (total == 0) return KBE_OK;
    const int blocks = (int)((total + 127) / 128 < 148 * 32 ? (total + 127) / 128 : 148 * 32);
    collision_row_kernel<<<blocks, 128, 0, (cudaStream_t)stream>>>(
        n_k, T, P, T1, T2, w2_matrix, (const cplx*)dg_first, (const cplx*)g_first, (const cplx*)s_like,
        (const cplx*)s_other, w1, w2, (cplx*)out);
    KBE_CHECK_LAUNCH("collision_row_kernel");
    return KBE_OK;
}

int kbe_update(const kbe_problem* p, int32_t n, int32_t phase, int32_t it, void* stream) {
    int rc = check_problem(p);
    if (rc) return rc;
    if (n < 1 || n > p->n_steps || it < 0 || it >= p->max_iter) { set_err("kbe_update: n/it", cudaSuccess); return KBE_ERR_ARG; }
    if ((rc = ensure_attrs())) return rc;
    KSpec s;
    const bool red = upd_split(p);
    if (red) {
        spec_reduce(s, p, n, phase, it);
        KBE_LAUNCH_SPEC("reduce_kernel", s);
    }
    spec_update(s, p, n, phase, it, 0, red);
    KBE_LAUNCH_SPEC("update_kernel", s);
    return KBE_OK;
}

int kbe_hf_mean(const kbe_problem* p, int32_t n, int32_t phase, int32_t it, void* stream) {
    int rc = check_problem(p);
    if (rc) return rc;
    KSpec s;
    spec_hf(s, p, n, phase, it);
    KBE_LAUNCH_SPEC("hf_mean_kernel", s);
    return KBE_OK;
}

int kbe_build_phi(const kbe_problem* p, int32_t n, int32_t it, void* stream) {
    int rc = check_problem(p);
    if (rc) return rc;
    if (n < 1 || n > p->n_steps) { set_err("kbe_build_phi: n", cudaSuccess); return KBE_ERR_ARG; }
    KSpec s;
    make_spec(s, phi_table_kernel, dim3(1), dim3(128), 0, *p, (int)n, (int)n, (int)it, 1);
    KBE_LAUNCH_SPEC("phi_table_kernel", s);
    return KBE_OK;
}

int kbe_finish_step(const kbe_problem* p, int32_t n, void* stream) {
    int rc = check_problem(p);
    if (rc) return rc;
    KSpec s;
    spec_finish(s, p, n);
    KBE_LAUNCH_SPEC("finish_kernel", s);
    return KBE_OK;
}

// step n with corrector iterations [it0, it1) (it0 > 0: resuming a shortened step, no
// predictor) and the finish for `it1` launched iterations
static int step_range(const kbe_problem* p, int n, int it0, int it1, void* stream) {
    int rc;
    if (it0 == 0) {
        // Algorithm 1 (propagator.py:328-382): Sigma(n-1), I(n-1), predictor, then
        // the corrector iterations [Sigma(n), I(n), corrector]; converged ones are no-ops.
        if (p->interacting && (rc = kbe_sigma_frontier(p, n - 1, 0, stream))) return rc;
        if ((rc = launch_collision(p, n - 1, 0, p->interacting, stream))) return rc;
        if (p->hf && (rc = kbe_hf_mean(p, n, 0, 0, stream))) return rc;
        if ((rc = kbe_update(p, n, 0, 0, stream))) return rc;
    }
    for (int it = it0; it < it1; ++it) {
        if (p->interacting && (rc = kbe_sigma_frontier(p, n, it, stream))) return rc;
        if ((rc = launch_collision(p, n, it, p->interacting, stream))) return rc;
        if (p->hf && (rc = kbe_hf_mean(p, n, 1, it, stream))) return rc;
        if ((rc = kbe_update(p, n, 1, it, stream))) return rc;
    }
    if ((rc = ensure_attrs())) return rc;
    KSpec s;
    spec_finish(s, p, n, it1);
    KBE_LAUNCH_SPEC("finish_kernel", s);
    return KBE_OK;
}

int kbe_step(const kbe_problem* p, int32_t n, void* stream) {
    int rc = check_problem(p);
    if (rc) return rc;
    // one rank, or k-sharded ranks exchanging peer-to-peer (the update kernel publishes;
    // nothing between launches).  NCCL-gathered or hf_mode="on" shards need the host.
    if ((sharded(*p) && p->p2p_world <= 1) || (p->p2p_world > 1 && p->hf)) {
        snprintf(g_err, sizeof(g_err), "kbe_step: these k-sharded steps need host collectives (NCCL path or hf_mode)");
        return KBE_ERR_ARG;
    }
    if (n < 1 || n > p->n_steps) { set_err("kbe_step: n", cudaSuccess); return KBE_ERR_ARG; }
    return step_range(p, n, 0, p->max_iter, stream);
}

int kbe_run_iters(const kbe_problem* p, int32_t n_first, int32_t n_last, int32_t m, void* stream) {
    int rc = check_problem(p);
    if (rc) return rc;
    if ((sharded(*p) && p->p2p_world <= 1) || (p->p2p_world > 1 && p->hf) || m < 1 || m > p->max_iter ||
        n_first < 1 || n_last > p->n_steps) {
        set_err("kbe_run_iters", cudaSuccess);
        return KBE_ERR_ARG;
    }
    for (int n = n_first; n <= n_last; ++n)
        if ((rc = step_range(p, n, 0, m, stream))) return rc;
    return KBE_OK;
}

int kbe_resume_step(const kbe_problem* p, int32_t n, int32_t m_done, void* stream) {
    int rc = check_problem(p);
    if (rc) return rc;
    if (n < 1 || n > p->n_steps || m_done < 1 || m_done >= p->max_iter) {
        set_err("kbe_resume_step", cudaSuccess);
        return KBE_ERR_ARG;
    }
    cudaError_t e = cudaMemsetAsync((char*)p->ctl + offsetof(kbe_ctl, needs_more), 0, sizeof(int), (cudaStream_t)stream);
    if (e != cudaSuccess) { set_err("kbe_resume_step", e); return KBE_ERR_CUDA; }
    return step_range(p, n, m_done, p->max_iter, stream);
}

int64_t kbe_ctl_needs_more_offset(void) { return (int64_t)offsetof(kbe_ctl, needs_more); }
int kbe_launches_per_eval(const kbe_problem* p) {
    if (check_problem(p)) return -1;
    return (p->interacting ? 1 : 0) + 1 + (p->hf ? 1 : 0) + (upd_split(p) ? 1 : 0) + 1;
}
int64_t kbe_ctl_hf_sum_offset(void) { return (int64_t)offsetof(kbe_ctl, hf_sum); }
int32_t kbe_max_n_k(void) { return KBE_MAX_NK; }
int kbe_set_sigma_variant(int32_t kind) {
    if (kind < 0 || kind > 3) return -1;
    const int prev = g_sigma_kind < 0 ? 0 : g_sigma_kind;
    g_sigma_kind = kind;
    return prev;
}

int kbe_run(const kbe_problem* p, int32_t n_first, int32_t n_last, int32_t use_graph, void* stream) {
    int rc = check_problem(p);
    if (rc) return rc;
    if (n_first < 1 || n_last > p->n_steps) { set_err("kbe_run: n range", cudaSuccess); return KBE_ERR_ARG; }
    if (!use_graph) {
        for (int n = n_first; n <= n_last; ++n)
            if ((rc = kbe_step(p, n, stream))) return rc;
        return KBE_OK;
    }
    if (sharded(*p)) {
        snprintf(g_err, sizeof(g_err), "kbe_run: the step graph drives one rank");
        return KBE_ERR_ARG;
    }
    if ((rc = ensure_attrs())) return rc;
    StepGraph* sg = nullptr;
    if (n_first > n_last) return KBE_OK;
    if ((rc = get_graph(p, n_first, &sg))) return rc;
    for (int n = n_first; n <= n_last; ++n)
        if ((rc = graph_step(sg, p, n, stream))) return rc;
    return KBE_OK;
}

int kbe_release(const kbe_problem* p) {
    for (auto& g : g_graphs)
        if (g && p && g->key.ctl == p->ctl) {
            cudaDeviceSynchronize();
            destroy_graph(g);
            g = nullptr;
        }
    return KBE_OK;
}

int kbe_unpack(const void* hist, int64_t tri, int32_t k_local, int32_t n_steps, int32_t frontier, int32_t which,
               void* out, void* stream) {
    if (!hist || !out || k_local < 1 || n_steps < 0 || frontier > n_steps) { set_err("kbe_unpack", cudaSuccess); return KBE_ERR_ARG; }
    const int64_t total = (int64_t)k_local * 4 * (n_steps + 1) * (int64_t)(n_steps + 1);
    int64_t blocks = (total + 255) / 256;
    if (blocks > 148 * 64) blocks = 148 * 64;
    unpack_kernel<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>((const cplx*)hist, tri, k_local, n_steps, frontier,
                                                                 which, (cplx*)out);
    KBE_CHECK_LAUNCH("unpack_kernel");
    return KBE_OK;
}

int kbe_unpack_retarded(const void* hist, int64_t tri, int32_t k_local, int32_t n_steps, int32_t frontier,
                        double theta0, void* out, void* stream) {
    if (!hist || !out || k_local < 1 || n_steps < 0 || frontier > n_steps) {
        set_err("kbe_unpack_retarded", cudaSuccess);
        return KBE_ERR_ARG;
    }
    const int64_t total = (int64_t)k_local * 4 * (n_steps + 1) * (int64_t)(n_steps + 1);
    int64_t blocks = (total + 255) / 256;
    if (blocks > 148 * 64) blocks = 148 * 64;
    unpack_retarded_kernel<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>((const cplx*)hist, tri, k_local, n_steps,
                                                                          frontier, theta0, (cplx*)out);
    KBE_CHECK_LAUNCH("unpack_retarded_kernel");
    return KBE_OK;
}

int kbe_pack(const void* lower_full, const void* upper_full, int32_t k_local, int32_t n_steps, int32_t frontier,
             int64_t tri, void* hist, void* stream) {
    if (!lower_full || !upper_full || !hist || k_local < 1 || frontier < 0 || frontier > n_steps) {
        set_err("kbe_pack", cudaSuccess);
        return KBE_ERR_ARG;
    }
    const int64_t total = (int64_t)k_local * slice_off(frontier + 1);
    int64_t blocks = (total + 255) / 256;
    if (blocks > 148 * 64) blocks = 148 * 64;
    pack_kernel<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>((const cplx*)lower_full, (const cplx*)upper_full,
                                                               k_local, n_steps, frontier, tri, (cplx*)hist);
    KBE_CHECK_LAUNCH("pack_kernel");
    return KBE_OK;
}

int64_t kbe_p2p_bytes(const kbe_problem* p, int32_t world) {
    if (!p || world < 1) return -1;
    return (int64_t)2 * world * front_chunk(*p) * (int64_t)sizeof(cplx) + 8 * (int64_t)(world + 2);
}

int kbe_p2p_alloc(int64_t bytes, void** ptr_out, void* ipc_handle_out) {
    if (bytes <= 0 || !ptr_out || !ipc_handle_out) { set_err("kbe_p2p_alloc", cudaSuccess); return KBE_ERR_ARG; }
    cudaError_t e = cudaMalloc(ptr_out, (size_t)bytes);
    if (e == cudaSuccess) e = cudaMemset(*ptr_out, 0, (size_t)bytes);
    if (e == cudaSuccess) e = cudaIpcGetMemHandle((cudaIpcMemHandle_t*)ipc_handle_out, *ptr_out);
    if (e != cudaSuccess) { set_err("kbe_p2p_alloc", e); return KBE_ERR_CUDA; }
    return KBE_OK;
}

int kbe_p2p_open(const void* ipc_handle, void** ptr_out) {
    if (!ipc_handle || !ptr_out) { set_err("kbe_p2p_open", cudaSuccess); return KBE_ERR_ARG; }
    cudaIpcMemHandle_t h;
    memcpy(&h, ipc_handle, sizeof(h));
    cudaError_t e = cudaIpcOpenMemHandle(ptr_out, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) { set_err("kbe_p2p_open", e); return KBE_ERR_CUDA; }
    return KBE_OK;
}

int kbe_p2p_close(void* ptr) {
    cudaError_t e = cudaIpcCloseMemHandle(ptr);
    if (e != cudaSuccess) { set_err("kbe_p2p_close", e); return KBE_ERR_CUDA; }
    return KBE_OK;
}

int kbe_p2p_free(void* ptr) {
    cudaError_t e = cudaFree(ptr);
    if (e != cudaSuccess) { set_err("kbe_p2p_free", e); return KBE_ERR_CUDA; }
    return KBE_OK;
}

int kbe_p2p_read_u64(const void* dev_ptr, void* host_out) {
    if (!dev_ptr || !host_out) { set_err("kbe_p2p_read_u64", cudaSuccess); return KBE_ERR_ARG; }
    cudaError_t e = cudaMemcpy(host_out, dev_ptr, 8, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) { set_err("kbe_p2p_read_u64", e); return KBE_ERR_CUDA; }
    return KBE_OK;
}

int kbe_p2p_publish(const kbe_problem* p, void* stream) {
    int rc = check_problem(p);
    if (rc) return rc;
    if (p->p2p_world < 2 || p->p2p_world > KBE_MAX_RANKS || !p->p2p_local || !p->front_send) {
        set_err("kbe_p2p_publish", cudaSuccess);
        return KBE_ERR_ARG;
    }
    KSpec s;
    make_spec(s, p2p_publish_kernel, dim3(64), dim3(256), 0, *p);
    KBE_LAUNCH_SPEC("p2p_publish_kernel", s);
    return KBE_OK;
}

}  // extern "C"
