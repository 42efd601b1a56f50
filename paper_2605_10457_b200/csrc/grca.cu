// grca.cu -- kernels K0..K5 and the C ABI (include/grca.h) of the B200-native GRCA hot path.
//
//   K0 init      hits[g] = MISS (packed u64), counters = 0                      (A0 per cast)
//   K2 cull      persistent; per triangle (fused K1 load) x per emitter:
//                range cull -> elevation interval -> channel range (smem sin table
//                binary search) -> azimuth arc -> ray range; small rectangles are
//                expanded with a warp prefix scan and intersected inline, large ones
//                appended (warp-aggregated) to the large list                     (A1-A5)
//   K3 bin       large pairs -> load-balanced chunks (<= 1024 items), pole rows full  (A5)
//   K4 intersect persistent warps over chunks: lanes = consecutive rays of a row    (A6)
//   K5 unpack    packed key -> (float distance, int32 id)                         (A8)
// Cites: PAPER.md:2304-2466 (paper's GPU pipeline, prior art), SURVEY.md 8(a)/(b).
#include <cuda_runtime.h>
#include <math.h>
#include <nccl.h>
#include <nccl_device.h>
#include <cmath>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <climits>
#include <string>
#include <vector>

#include "grca.h"
#include "grca_device.cuh"

namespace grca {

constexpr unsigned FULL = 0xffffffffu;
constexpr unsigned long long kMiss = 0x7F800000FFFFFFFFull;
constexpr int K2_THREADS = 256;
#ifndef K2_TILE
#define K2_TILE 1024   // triangles per K2 block tile (K2_TILE / K2_THREADS = 4 per thread; measured: 256 -> 0.578, 512 -> 0.543, 1024 -> 0.525 ms)
#endif
constexpr int K4_THREADS = 256;
// fused refine+small: 576 threads x 2 blocks (56 registers) measured best on B200 (occupancy vs spills)
#ifndef KF_THREADS
#define KF_THREADS 576   // 18 warps x 2 blocks at 56 registers (measured: 512 -> 0.561 ms, 576 -> 0.558, 640 -> 0.585)
#endif
#ifndef KF_MINB
#define KF_MINB 2
#endif
#ifndef KF_FETCH
#define KF_FETCH 2   // 32-survivor rounds per dynamic fetch of the fused kernel (measured: 1 -> 1.048, 2 -> 1.033,
                     // 4 -> 1.121 ms at C4: half the fetch atomics vs a coarser tail)
#endif
#ifndef K2_DYN_TILES
#define K2_DYN_TILES 1   // K2 tiles after the first wave fetched dynamically (measured: C4 K2 0.438 -> 0.387 ms; statically
                         // strided tiles left blocks with more car (indexed) tiles finishing last)
#endif
#ifndef K2_PRED_MAX_NE
#define K2_PRED_MAX_NE 2   // K2 pre-test in predicate form (quick_*_pred) for NE <= this; the 2-bit-code form above
                           // (measured at C4: NE = 8 0.485 vs 0.503 ms in predicate form; NE = 1 0.1715 -> 0.1695,
                           // NE = 2 0.209 -> 0.201 ms, the 8- and 4-GPU sensor-shard ranks)
#endif
#ifndef KF_SMAX_MUL
#define KF_SMAX_MUL 16   // fused kernel: small-rectangle cap = max(64, rounds per warp x this) (<= small_max)
#endif
#ifndef KF_MAGIC_DIV
#define KF_MAGIC_DIV 0   // fused item loop: row = local / len by a per-pair magic multiplier (no float round trip)
#endif
#ifndef KF_SB_INT
#define KF_SB_INT 0
#endif
#ifndef KF_FETCH_TAIL
#define KF_FETCH_TAIL 12   // fused kernel: the last 12 rounds per warp fetched one at a time (measured: C4 fused 0.4695 -> 0.4579 ms;
                          // 2 / 6 / 20 / 30: 0.4683 / 0.4591 / 0.4592 / 0.4622)
#endif
#ifndef KF_ROWCOL_EXACT
// fused item loop: row = floor((local + 1/2) / len) from the approximate reciprocal needs no +-1 correction for a
// small rectangle: its items (rows x len) are <= small_max <= 1023, so (local + 1/2) / len lies >= 1/(2 len) from an
// integer while the float error is <= rows x 2^-21 <= (1023 / len) x 2^-21, under 1e-3 of that distance
#define KF_ROWCOL_EXACT 1   // (measured: C4 fused 0.478 -> 0.470 ms; tests/test_kernel_arith_cpu.py checks the bound)
#endif
#ifndef KF_LANE_COUNT
#define KF_LANE_COUNT 1   // fused item loop: hit / fp64 counts per lane, reduced once per round (no ballots per step;
                          // measured: C4 fused 0.481 -> 0.477 ms)
#endif
#ifndef KF_PREFETCH
#define KF_PREFETCH 0   // fused item loop: issue the next step's ray load before this step's test
#endif
#ifndef K3_MINB
#define K3_MINB 2   // 128 registers (without a bound the compiler took 145: K3 0.028 -> 0.041 ms)
#endif
#ifndef K4_MINB
#define K4_MINB 3   // 80 registers: 3 blocks of 256 per SM (measured best; 1 block = 95+ regs, 25 % occupancy)
#endif
#ifndef K2_MINB
#define K2_MINB 8   // K2 is issue-bound; 8 x 256 threads (32 regs) measured marginally best
#endif
constexpr int kMaxEmitters = 255;
constexpr int kMaxSin = 4096;
constexpr int kLutMaxEm = 16;   // channel LUTs staged in smem for up to 16 emitters

enum Stat {
    ST_PAIRS = 0, ST_RANGE, ST_CHANNEL, ST_AZIMUTH, ST_SURV, ST_SMALL, ST_LARGE, ST_ITEMS_SMALL,
    ST_ITEMS_LARGE, ST_FP64, ST_HITS, ST_CHUNKS, ST_OVF_LARGE, ST_OVF_CHUNK, ST_SETUP64, ST_DEGEN,
    ST_K2SURV, ST_SAT, ST_BAT, ST_AREA, ST_HITS_L, ST_COUNT
};
static_assert(ST_COUNT <= 32, "per-warp stat rows hold 32 counters");

struct KParams {
    TriSrc tri;
    long long n_tri;
    const EmDev *em;
    const float *sin;
    int n_em, n_sin;
    const float4 *raytab;
    unsigned long long *hits;
    unsigned *allhits;
    int4 *large;
    unsigned *n_large;
    long long cap_large;
    int4 *chunks;                // K3 -> K4: {large-pair index, e | row << 8, 1 | lo << 16, len}
    float4 *large_setup;         // K3 -> K4: per large pair the 5-float4 setup (slot layout of setup_to_slot)
    unsigned *n_chunks;
    long long cap_chunks;
    unsigned long long *stats;
    int faces, nocull, force64, small_max, norefine;
    float area_eps2;             // (apparent-area eps)^2, 0 = off
    int pairs_ok;                // all emitter frames orthonormal (packed fp32x2 K2 path)
    long long n_rays;
    const EmLite *lite;
    const unsigned char *lut;    // NULL -> binary search
    unsigned long long *surv;    // dense K2 survivor list: tri << 8 | emitter
    long long cap_surv;          // its capacity (entries)
    unsigned *n_surv;
    unsigned long long *desc;    // split path: per survivor, small-rectangle descriptor (0 = none)
    unsigned long long *mc_hits; // NEXT-f3: multicast view of the ranks' hit buffers (NULL = local RED.MIN)
};

// slot fields (SoA per warp in shared memory) for the inline small-pair expansion
enum SlotF {
    SF_N0 = 0, SF_N1 = 3, SF_N2 = 6, SF_B = 9, SF_N = 12, SF_HABS = 15, SF_TN = 16, SF_ID = 17,
    SF_TRI = 18, SF_CFROM = 19, SF_RLO = 20, SF_LEN = 21, SF_INVLEN = 22, SF_EXCL = 23, SF_EM = 24, NF = 25
};

__device__ __forceinline__ f3 em_o(const EmDev &E) { return {E.o[0], E.o[1], E.o[2]}; }

__device__ __forceinline__ void block_flush(unsigned long long *acc_smem, unsigned long long *stats,
                                            const unsigned *mine) {
    // warp reduce then smem then one atomic per block per counter.  REDUX.SUM on the 16-bit halves
    // of the per-thread u32 counts (each half-sum < 2^21: exact), and counters that are zero in the
    // whole warp are skipped (one vote): this runs at the end of every warp's chain (K3/K4 latency).
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int c = 0; c < ST_COUNT; ++c) {
        const unsigned v = mine[c];
        if (__any_sync(FULL, v != 0u)) {
            const unsigned lo = __reduce_add_sync(FULL, v & 0xffffu);
            const unsigned hi = __reduce_add_sync(FULL, v >> 16);
            if (lane == 0) atomicAdd(acc_smem + c, (unsigned long long)lo + ((unsigned long long)hi << 16));
        }
    }
    __syncthreads();
    if (threadIdx.x < ST_COUNT && acc_smem[threadIdx.x]) atomicAdd(stats + threadIdx.x, acc_smem[threadIdx.x]);
}

// ------------------------------------------------------------------- K0 init --
#ifdef GRCA_CHECK
__global__ void k_check_set_n_rays(long long n) { g_check_n_rays = n; }
#endif

__global__ void k_init(unsigned long long *hits, unsigned *allhits, long long n, unsigned *ctrl,
                       unsigned long long *stats, const unsigned long long *src, const unsigned *src_allhits,
                       int reset = 1) {
    // hits = MISS, or the cached static-scene keys (hybrid mode, NEXT-f2)
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long n2 = n >> 1;
    ulonglong2 *h2 = reinterpret_cast<ulonglong2 *>(hits);
    if (src) {
        const ulonglong2 *s2 = reinterpret_cast<const ulonglong2 *>(src);
        for (long long i = tid; i < n2; i += stride) h2[i] = __ldcs(s2 + i);
        if (tid == 0 && (n & 1)) hits[n - 1] = src[n - 1];
    } else {
        for (long long i = tid; i < n2; i += stride) h2[i] = make_ulonglong2(kMiss, kMiss);
        if (tid == 0 && (n & 1)) hits[n - 1] = kMiss;
    }
    if (allhits)
        for (long long i = tid; i < n; i += stride) allhits[i] = src_allhits ? src_allhits[i] : 0u;
    if (reset && tid < ST_COUNT) stats[tid] = 0ull;
    if (reset && tid < 7) ctrl[tid] = 0u;   // (ctrl[7]: sticky NVLS barrier timeout flag)
}

// NEXT-f3 device-side barrier over the NVLS group (one thread): every rank adds 1 to every rank's
// flag through the multicast address (release), then waits until its own copy reaches
// target = epoch * n_ranks (acquire).  A peer that never arrives trips the timeout (~20 s), which
// sets err[0] instead of hanging the GPU.
__global__ void k_nvls_barrier(unsigned *flag_uc, unsigned *flag_mc, unsigned target, unsigned *err) {
    __threadfence_system();
    asm volatile("multimem.red.release.sys.global.add.u32 [%0], %1;" ::"l"(flag_mc), "r"(1u) : "memory");
    const long long t0 = clock64();
    unsigned v;
    for (;;) {
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag_uc) : "memory");
        if ((int)(v - target) >= 0) break;
        if (clock64() - t0 > 40000000000ll) { atomicExch(err, 1u); break; }
        __nanosleep(64);
    }
    __threadfence_system();
}

// NEXT-f3 through NCCL (GRCA_MERGE_NVLS): the multicast address of this rank's symmetric window, i.e.
// where a multimem.red lands in every rank's copy (NCCL device API; one thread, once per binding).
__global__ void k_sym_multimem_ptr(ncclWindow_t win, ncclDevComm dc, unsigned long long *out) {
    out[0] = reinterpret_cast<unsigned long long>(ncclGetLsaMultimemPointer(win, 0, dc));
}

// ------------------------------------------------------- K2 cull (phase A) --
// Lean and dense: per triangle (fused K1 load) x per emitter, the O(1) elevation pre-test
// (quick_cull).  Survivors are compacted per 256-triangle tile in shared memory and written to
// the tile's own slot of the survivor buffer (no global atomics); K2b refines them.
__global__ void __launch_bounds__(K2_THREADS) k_cull(const __grid_constant__ KParams P) {
    extern __shared__ __align__(16) unsigned char smem[];
    EmLite *sL = reinterpret_cast<EmLite *>(smem);
    float *sSin = reinterpret_cast<float *>(sL + P.n_em);
    unsigned char *sLut = reinterpret_cast<unsigned char *>(sSin + ((P.n_sin + 3) & ~3));
    unsigned short *sQ = reinterpret_cast<unsigned short *>(sLut + (P.lut ? ((P.n_em * kLutBins + 15) & ~15) : 0));
    __shared__ int qn;
    __shared__ unsigned qbase;
    __shared__ unsigned long long acc[ST_COUNT];
    {
        const int nw = P.n_em * (int)(sizeof(EmLite) / 4);
        const int *src = reinterpret_cast<const int *>(P.lite);
        int *dst = reinterpret_cast<int *>(sL);
        for (int i = threadIdx.x; i < nw; i += blockDim.x) dst[i] = src[i];
        for (int i = threadIdx.x; i < P.n_sin; i += blockDim.x) sSin[i] = P.sin[i];
        if (P.lut)
            for (int i = threadIdx.x; i < P.n_em * kLutBins; i += blockDim.x) sLut[i] = P.lut[i];
        if (threadIdx.x < ST_COUNT) acc[threadIdx.x] = 0ull;
    }
    const int lane = threadIdx.x & 31;
    unsigned cnt[ST_COUNT];
#pragma unroll
    for (int c = 0; c < ST_COUNT; ++c) cnt[c] = 0u;
    unsigned c_pairs = 0, c_range = 0, c_chan = 0, c_surv = 0;
    const long long ntiles = (P.n_tri + K2_THREADS - 1) / K2_THREADS;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        if (threadIdx.x == 0) qn = 0;
        __syncthreads();
        const long long t = tile * K2_THREADS + threadIdx.x;
        const bool valid = t < P.n_tri;
        f3 v[3] = {{0.f, 0.f, 0.f}, {0.f, 0.f, 0.f}, {0.f, 0.f, 0.f}};
        float emax = 0.f;
        if (valid) {   // A1 (fused K1): coalesced float4 vertex loads, triangle diameter
            load_tri(P.tri, t, v);
            const float l0 = (v[1].x - v[0].x) * (v[1].x - v[0].x) + (v[1].y - v[0].y) * (v[1].y - v[0].y) +
                             (v[1].z - v[0].z) * (v[1].z - v[0].z);
            const float l1 = (v[2].x - v[1].x) * (v[2].x - v[1].x) + (v[2].y - v[1].y) * (v[2].y - v[1].y) +
                             (v[2].z - v[1].z) * (v[2].z - v[1].z);
            const float l2 = (v[0].x - v[2].x) * (v[0].x - v[2].x) + (v[0].y - v[2].y) * (v[0].y - v[2].y) +
                             (v[0].z - v[2].z) * (v[0].z - v[2].z);
            emax = sqrtf(fmaxf(l0, fmaxf(l1, l2))) * (1.f + 1e-5f);
        }
        for (int e = 0; e < P.n_em; ++e) {
            int st = -1;
            if (valid) {
                ++c_pairs;
                st = P.nocull ? CULL_KEEP
                              : quick_cull(v, emax, sL[e], sSin + sL[e].sin_base,
                                           P.lut ? sLut + sL[e].lut_base : nullptr);
                c_range += (st == CULL_RANGE);
                c_chan += (st == CULL_CHANNEL);
                c_surv += (st == CULL_KEEP);
            }
            const bool keep = st == CULL_KEEP;
            const unsigned m = __ballot_sync(FULL, keep);
            if (m) {   // warp-aggregated append to the tile's shared-memory queue
                const int leader = __ffs(m) - 1;
                int base = 0;
                if (lane == leader) base = atomicAdd(&qn, __popc(m));
                base = __shfl_sync(FULL, base, leader);
                if (keep) sQ[base + __popc(m & ((1u << lane) - 1u))] = (unsigned short)((threadIdx.x << 8) | e);
            }
        }
        __syncthreads();
        const int n = qn;
        if (threadIdx.x == 0) qbase = n ? atomicAdd(P.n_surv, (unsigned)n) : 0u;   // one atomic per tile
        __syncthreads();
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const unsigned q = sQ[i];
            P.surv[qbase + i] = ((unsigned long long)(tile * K2_THREADS + (q >> 8)) << 8) | (q & 255u);
        }
        __syncthreads();
    }
    cnt[ST_PAIRS] = c_pairs;
    cnt[ST_RANGE] = c_range;
    cnt[ST_CHANNEL] = c_chan;
    cnt[ST_K2SURV] = c_surv;
    block_flush(acc, P.stats, cnt);
}

// ---------------------------------------- K2 cull, fixed emitter count (hot) --
// Same test as k_cull, specialised for NE <= kFixedEm emitters: the emitter loop is unrolled and the
// EmLite records are a kernel parameter (constant bank), so their fields are direct FFMA/FADD
// operands; survivors are compacted once per tile with a block-wide scan of per-thread emitter
// masks (no per-emitter ballots or shared atomics).
constexpr int kFixedEm = 8;
struct EmLitePack {
    EmLite e[kFixedEm];
    EmPair p[kFixedEm / 2];   // interleaved pair constants (packed path)
};

// K2 per-triangle test (A1 load + A2-A3 pre-test for all NE emitters): keep / range bit masks,
// channel-culled count; c_area counts paper-mode apparent-area culls.
// kFast: culling on, packed pairs usable, no apparent-area cull -- the mode flags are then checked
// once per kernel instead of per triangle (k_cull_fixed picks the instantiation)
template <int NE, bool kLevel, bool kFast, bool kC>
__device__ __forceinline__ void k2_tri(const KParams &P, const EmLitePack &EL, const float *sSin,
                                       const unsigned char *sLut, long long t, unsigned &keep, unsigned &rng,
                                       unsigned &c_area) {
    f3 v[3];
    load_tri<kC>(P.tri, t, v);   // A1 (fused K1)
    const float l0 = (v[1].x - v[0].x) * (v[1].x - v[0].x) + (v[1].y - v[0].y) * (v[1].y - v[0].y) +
                     (v[1].z - v[0].z) * (v[1].z - v[0].z);
    const float l1 = (v[2].x - v[1].x) * (v[2].x - v[1].x) + (v[2].y - v[1].y) * (v[2].y - v[1].y) +
                     (v[2].z - v[1].z) * (v[2].z - v[1].z);
    const float l2 = (v[0].x - v[2].x) * (v[0].x - v[2].x) + (v[0].y - v[2].y) * (v[0].y - v[2].y) +
                     (v[0].z - v[2].z) * (v[0].z - v[2].z);
    const float m2 = fmaxf(l0, fmaxf(l1, l2));
    const float emax = m2 * rsqrtf(m2) * (1.f + 1e-5f);   // triangle diameter (0 if degenerate)
    unsigned kb = 0u, rb = 0u;
    if (!kFast && P.nocull) {
        kb = (1u << NE) - 1u;
    } else if ((NE <= K2_PRED_MAX_NE) && (kFast || P.pairs_ok)) {   // predicate form (no 2-bit codes)
#pragma unroll
        for (int e = 0; e + 1 < NE; e += 2) {
            bool k0, r0, k1, r1;
            quick_pair_pred<kLevel>(v, emax, EL.p[e / 2], EL.e[e], EL.e[e + 1], sSin + EL.e[e].sin_base,
                                    sSin + EL.e[e + 1].sin_base, sLut + e * kLutBins, sLut + (e + 1) * kLutBins,
                                    k0, r0, k1, r1);
            if (k0) kb |= 1u << e;
            if (k1) kb |= 2u << e;
            if (r0) rb |= 1u << e;
            if (r1) rb |= 2u << e;
        }
        if (NE & 1) {
            bool k0, r0;
            quick_cull_pred<kLevel>(v, emax, EL.e[NE - 1], sSin + EL.e[NE - 1].sin_base, sLut + (NE - 1) * kLutBins,
                                    k0, r0);
            if (k0) kb |= 1u << (NE - 1);
            if (r0) rb |= 1u << (NE - 1);
        }
    } else if (kFast || P.pairs_ok) {   // all frames orthonormal: packed fp32x2 path
#pragma unroll
        for (int e = 0; e + 1 < NE; e += 2) {
#if K2_TAIL_SEL
            quick_pair_sel<kLevel>(v, emax, EL.p[e / 2], EL.e[e], EL.e[e + 1], sSin + EL.e[e].sin_base,
                                   sSin + EL.e[e + 1].sin_base, sLut + e * kLutBins, sLut + (e + 1) * kLutBins,
                                   1u << e, kb, rb);
#else
            const unsigned r = quick_pair_lut<kLevel>(v, emax, EL.p[e / 2], EL.e[e], EL.e[e + 1], sSin + EL.e[e].sin_base,
                                              sSin + EL.e[e + 1].sin_base, sLut + e * kLutBins,
                                              sLut + (e + 1) * kLutBins);
            kb |= (r & 3u) << e;
            rb |= (r >> 2) << e;
#endif
        }
        if (NE & 1) {
            const unsigned r = quick_cull_lut<kLevel>(v, emax, EL.e[NE - 1], sSin + EL.e[NE - 1].sin_base,
                                              sLut + (NE - 1) * kLutBins);
#if K2_TAIL_SEL
            kb |= r == 1u ? 1u << (NE - 1) : 0u;
            rb |= r == 2u ? 1u << (NE - 1) : 0u;
#else
            kb |= (r & 1u) << (NE - 1);
            rb |= (r >> 1) << (NE - 1);
#endif
        }
    } else {
#pragma unroll
        for (int e = 0; e < NE; ++e) {
            const unsigned r = quick_cull_lut<kLevel>(v, emax, EL.e[e], sSin + EL.e[e].sin_base, sLut + e * kLutBins);
            kb |= (r & 1u) << e;
            rb |= (r >> 1) << e;
        }
    }
    if (!kFast && P.area_eps2 > 0.f) {   // NEXT-f1 paper mode (approximate): apparent-area cull
        for (unsigned m = kb; m; m &= m - 1u) {
            const int e = __ffs(m) - 1;
            const f3 cen = {(v[0].x + v[1].x + v[2].x) * (1.f / 3.f), (v[0].y + v[1].y + v[2].y) * (1.f / 3.f),
                            (v[0].z + v[1].z + v[2].z) * (1.f / 3.f)};
            const f3 hN = scalef(crossf(subf(v[1], v[0]), subf(v[2], v[0])), 0.5f);   // A_T * n
            const f3 co = {cen.x - EL.e[e].o[0], cen.y - EL.e[e].o[1], cen.z - EL.e[e].o[2]};
            const float an = dotf(hN, co), d2 = dotf(co, co);
            if (an * an < P.area_eps2 * d2 * d2 * d2) { kb &= ~(1u << e); ++c_area; }
        }
    }
    keep = kb;
    rng = rb;
}

// The persistent tile loop of k_cull_fixed (one instantiation per mode, see k2_tri).
template <int NE, bool kLevel, bool kFast, bool kC>
__device__ __forceinline__ void k2_tiles(const KParams &P, const EmLitePack &EL, const float *sSin,
                                         const unsigned char *sLut, int *wsum, unsigned &qbase, int lane, int wib,
                                         unsigned &c_pairs, unsigned &c_range, unsigned &c_surv,
                                         unsigned &c_area) {
    const long long ntiles = (P.n_tri + K2_TILE - 1) / K2_TILE;
#if K2_DYN_TILES   // tiles after the first wave fetched dynamically (one atomic per tile, at the tile's closing barrier)
    __shared__ long long s_next;
    for (long long tile = blockIdx.x; tile < ntiles;) {
#else
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
#endif
        // K2_TILE / K2_THREADS triangles per thread (one block scan, barrier pair and atomic for all)
        unsigned keeps[K2_TILE / K2_THREADS];
        int cntk = 0;
#pragma unroll
        for (int h = 0; h < K2_TILE / K2_THREADS; ++h) {
            const long long t = tile * K2_TILE + h * K2_THREADS + threadIdx.x;
            unsigned keep = 0u, rng = 0u;
            if (t < P.n_tri) {
                k2_tri<NE, kLevel, kFast, kC>(P, EL, sSin, sLut, t, keep, rng, c_area);
                c_pairs += NE;
            }
            keeps[h] = keep;
            cntk += __popc(keep);
            c_range += __popc(rng);
        }
        c_surv += cntk;
        // block-wide exclusive scan of the per-thread survivor counts
        int incl = cntk;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) wsum[wib] = incl;
        __syncthreads();
        int wbase = 0, total = 0;
#pragma unroll
        for (int w = 0; w < K2_THREADS / 32; ++w) {
            const int x = wsum[w];
            wbase += (w < wib) ? x : 0;
            total += x;
        }
        if (threadIdx.x == 0) qbase = total ? atomicAdd(P.n_surv, (unsigned)total) : 0u;   // one atomic per tile
        __syncthreads();
#ifdef GRCA_CHECK
        if (cntk) chk_idx((long long)qbase + wbase + incl - 1, P.cap_surv, CHK_SURV_WRITE);   // this thread's last entry
        unsigned long long *dst = P.surv + chk_idx((long long)qbase + wbase + incl - cntk, P.cap_surv, CHK_SURV_WRITE);
#else
        unsigned long long *dst = P.surv + qbase + wbase + incl - cntk;
#endif
#pragma unroll
        for (int h = 0; h < K2_TILE / K2_THREADS; ++h) {
            const long long t = tile * K2_TILE + h * K2_THREADS + threadIdx.x;
            unsigned keep = keeps[h];
            while (keep) {
                const int e = __ffs(keep) - 1;
                keep &= keep - 1u;
                *dst++ = ((unsigned long long)t << 8) | (unsigned)e;
            }
        }
#if K2_DYN_TILES
        if (threadIdx.x == 0) s_next = (long long)gridDim.x + (long long)atomicAdd(P.n_surv + 3, 1u);
        __syncthreads();   // wsum / qbase reuse, s_next visible
        tile = s_next;
#else
        __syncthreads();   // wsum / qbase reuse
#endif
    }
}

template <int NE, bool kLevel, bool kC>
__global__ void __launch_bounds__(K2_THREADS, K2_MINB) k_cull_fixed(const __grid_constant__ KParams P, const EmLitePack EL) {
    extern __shared__ __align__(16) unsigned char smem[];
    float *sSin = reinterpret_cast<float *>(smem);
    unsigned char *sLut = reinterpret_cast<unsigned char *>(sSin + ((P.n_sin + 3) & ~3));
    __shared__ int wsum[K2_THREADS / 32];
    __shared__ unsigned qbase;
    __shared__ unsigned long long acc[ST_COUNT];
    for (int i = threadIdx.x; i < P.n_sin; i += blockDim.x) sSin[i] = P.sin[i];
    if (P.lut)
        for (int i = threadIdx.x; i < NE * kLutBins; i += blockDim.x) sLut[i] = P.lut[i];
    if (threadIdx.x < ST_COUNT) acc[threadIdx.x] = 0ull;
    __syncthreads();
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    unsigned c_pairs = 0, c_range = 0, c_surv = 0, c_area = 0;
    if (!P.nocull && (P.pairs_ok || NE == 1) && !(P.area_eps2 > 0.f))
        k2_tiles<NE, kLevel, true, kC>(P, EL, sSin, sLut, wsum, qbase, lane, wib, c_pairs, c_range, c_surv, c_area);
    else
        k2_tiles<NE, kLevel, false, kC>(P, EL, sSin, sLut, wsum, qbase, lane, wib, c_pairs, c_range, c_surv, c_area);
    unsigned cnt[ST_COUNT];
#pragma unroll
    for (int c = 0; c < ST_COUNT; ++c) cnt[c] = 0u;
    cnt[ST_PAIRS] = c_pairs;
    cnt[ST_RANGE] = c_range;
    // every pair is kept, range-culled, area-culled or channel-culled: no per-triangle counter
    cnt[ST_CHANNEL] = c_pairs - c_surv - c_area - c_range;
    cnt[ST_K2SURV] = c_surv;
    cnt[ST_AREA] = c_area;
    block_flush(acc, P.stats, cnt);
}

// ------------------------------------------------------------- K2b refine --
// Dense over the survivors of K2 (one warp per tile): exact conservative rectangle (cull_pair).
// Small rectangles get a 64-bit descriptor at the survivor's own index (no atomics); large ones
// are appended to the large list (warp-aggregated) for K3/K4.
__device__ __forceinline__ unsigned long long pack_small(int c_from, int nrows, int r_lo, int r_len) {
    return (unsigned long long)(unsigned)c_from | ((unsigned long long)nrows << 16) |
           ((unsigned long long)(unsigned)r_lo << 26) | ((unsigned long long)r_len << 42);
}

__device__ __noinline__ void intersect_rect_serial(const KParams &P, const EmDev &E, long long t, int row0, int nrows, int lo,
                                                   int len);

__global__ void __launch_bounds__(K2_THREADS) k_refine(const __grid_constant__ KParams P) {
    extern __shared__ __align__(16) unsigned char smem[];
    EmDev *sE = reinterpret_cast<EmDev *>(smem);
    float *sSin = reinterpret_cast<float *>(sE + P.n_em);
    unsigned char *sLut = reinterpret_cast<unsigned char *>(sSin + ((P.n_sin + 3) & ~3));
    __shared__ unsigned long long acc[ST_COUNT];
    {
        const int nw = P.n_em * (int)(sizeof(EmDev) / 4);
        const int *src = reinterpret_cast<const int *>(P.em);
        int *dst = reinterpret_cast<int *>(sE);
        for (int i = threadIdx.x; i < nw; i += blockDim.x) dst[i] = src[i];
        for (int i = threadIdx.x; i < P.n_sin; i += blockDim.x) sSin[i] = P.sin[i];
        if (P.lut)
            for (int i = threadIdx.x; i < P.n_em * kLutBins; i += blockDim.x) sLut[i] = P.lut[i];
        if (threadIdx.x < ST_COUNT) acc[threadIdx.x] = 0ull;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    unsigned cnt[ST_COUNT];
#pragma unroll
    for (int c = 0; c < ST_COUNT; ++c) cnt[c] = 0u;
    unsigned setup64 = 0;
    // work = rounds of 32 survivor entries, interleaved over all warps (balanced: no tile tails)
    const unsigned ns = *P.n_surv;
    const unsigned nr = (ns + 31) >> 5;   // dense rounds of 32 survivors
    // Small-rectangle cap scaled to the load: with few rounds per warp the longest round is the
    // kernel's tail, so big rectangles go to the chunk-balanced K3/K4 path instead (same results:
    // both paths run the same certified test).  C4: ~56 rounds/warp -> small_max; C2: ~1 -> 64.
    const unsigned rpw = nr / (gridDim.x * (KF_THREADS / 32));
    const int smax = min(P.small_max, (int)max(64u, min(rpw, 1024u) * 16u));
    const unsigned wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned nwarps = (gridDim.x * blockDim.x) >> 5;
    for (unsigned w = wid; w < nr; w += nwarps) {
        const int n = (int)ns;
        {
            const int idx = (int)(w * 32u) + lane;
            const bool act = idx < n;
            int e = 0, st = -1;
            long long t = 0;
            Rect R;
            unsigned long long desc = 0ull;
            bool large = false;
            if (act) {
                const unsigned long long ent = __ldcs(P.surv + idx);
                e = (int)(ent & 255u);
                t = (long long)(ent >> 8);
                f3 v[3];
                load_tri(P.tri, t, v);
                st = cull_pair(v, sE[e], sSin + sE[e].sin_base, P.lut ? sLut + e * kLutBins : nullptr,
                               P.nocull != 0, R);
                if (st == CULL_KEEP) {
                    const long long items = rect_items(R, sE[e]);
                    if (items <= P.small_max && !R.pole_rows) desc = pack_small(R.c_from, R.c_to - R.c_from + 1, R.r_lo, R.r_len);
                    else large = true;
                    cnt[ST_SURV]++;
                }
                else if (st == CULL_RANGE) cnt[ST_RANGE]++;
                else if (st == CULL_CHANNEL) cnt[ST_CHANNEL]++;
                else if (st == CULL_AZIMUTH) cnt[ST_AZIMUTH]++;
                else cnt[ST_DEGEN]++;
                P.desc[idx] = desc;
            }
            const unsigned lm = __ballot_sync(FULL, large);
            if (lm) {
                const int leader = __ffs(lm) - 1;
                unsigned base = 0;
                if (lane == leader) base = atomicAdd(P.n_large, (unsigned)__popc(lm));
                base = __shfl_sync(FULL, base, leader);
                if (large) {
                    const long long pos = (long long)base + __popc(lm & ((1u << lane) - 1u));
                    if (pos < P.cap_large) {
                        P.large[pos] = make_int4((int)t, e | (R.c_from << 8), R.c_to,
                                                 (int)((unsigned)R.r_lo | ((unsigned)R.r_len << 16)));
                        cnt[ST_LARGE]++;
                    } else {   // capacity fallback: intersect here (slow, never dropped)
                        cnt[ST_OVF_LARGE]++;
                        if (R.pole_rows) { R.r_lo = 0; R.r_len = sE[e].chi; }
                        intersect_rect_serial(P, sE[e], t, R.c_from, R.c_to - R.c_from + 1, R.r_lo, R.r_len);
                    }
                }
            }
        }
    }
    cnt[ST_SETUP64] = setup64;
    block_flush(acc, P.stats, cnt);
}

// -------------------------------------------------- K4s small intersection --
// One warp per tile: lanes compute the certified setup of their small rectangles (one pair per
// lane, into shared-memory slots), then the warp expands all items of the 32 pairs with an
// inclusive prefix scan (A5) and tests them (A6) 32 at a time -- no lane idles on a short pair.
__global__ void __launch_bounds__(K2_THREADS) k_small(const __grid_constant__ KParams P) {
    extern __shared__ __align__(16) unsigned char smem[];
    EmDev *sE = reinterpret_cast<EmDev *>(smem);
    float *sSlot = reinterpret_cast<float *>(sE + P.n_em);
    __shared__ unsigned long long acc[ST_COUNT];
    {
        const int nw = P.n_em * (int)(sizeof(EmDev) / 4);
        const int *src = reinterpret_cast<const int *>(P.em);
        int *dst = reinterpret_cast<int *>(sE);
        for (int i = threadIdx.x; i < nw; i += blockDim.x) dst[i] = src[i];
        if (threadIdx.x < ST_COUNT) acc[threadIdx.x] = 0ull;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    float *slot = sSlot + (threadIdx.x >> 5) * (NF * 32);
    unsigned cnt[ST_COUNT];
#pragma unroll
    for (int c = 0; c < ST_COUNT; ++c) cnt[c] = 0u;
    unsigned setup64 = 0;
    const unsigned ns = *P.n_surv;
    const unsigned nr = (ns + 31) >> 5;   // dense rounds of 32 survivors
    // Small-rectangle cap scaled to the load: with few rounds per warp the longest round is the
    // kernel's tail, so big rectangles go to the chunk-balanced K3/K4 path instead (same results:
    // both paths run the same certified test).  C4: ~56 rounds/warp -> small_max; C2: ~1 -> 64.
    const unsigned rpw = nr / (gridDim.x * (KF_THREADS / 32));
    const int smax = min(P.small_max, (int)max(64u, min(rpw, 1024u) * 16u));
    const unsigned wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned nwarps = (gridDim.x * blockDim.x) >> 5;
    for (unsigned w = wid; w < nr; w += nwarps) {
        const int n = (int)ns;
        {
            const int idx = (int)(w * 32u) + lane;
            int my = 0;
            if (idx < n) {
                const unsigned long long desc = P.desc[idx];
                const int nrows = (int)((desc >> 16) & 1023u);
                if (nrows) {
                    const unsigned long long ent = __ldcs(P.surv + idx);
                    const int e = (int)(ent & 255u);
                    const long long t = (long long)(ent >> 8);
                    const EmDev &E = sE[e];
                    f3 v[3];
                    load_tri(P.tri, t, v);
                    Setup S;
                    if (make_setup(v, em_o(E), P.faces, S, setup64)) {
                        const int len = (int)((desc >> 42) & 1023u);
                        my = nrows * len;
                        cnt[ST_SMALL]++;
                        cnt[ST_ITEMS_SMALL] += (unsigned long long)my;
                        float *sl = slot + lane;
                        sl[(SF_N0 + 0) * 32] = S.n0.x; sl[(SF_N0 + 1) * 32] = S.n0.y; sl[(SF_N0 + 2) * 32] = S.n0.z;
                        sl[(SF_N1 + 0) * 32] = S.n1.x; sl[(SF_N1 + 1) * 32] = S.n1.y; sl[(SF_N1 + 2) * 32] = S.n1.z;
                        sl[(SF_N2 + 0) * 32] = S.n2.x; sl[(SF_N2 + 1) * 32] = S.n2.y; sl[(SF_N2 + 2) * 32] = S.n2.z;
                        sl[(SF_B + 0) * 32] = S.B0; sl[(SF_B + 1) * 32] = S.B1; sl[(SF_B + 2) * 32] = S.B2;
                        sl[(SF_N + 0) * 32] = S.N.x; sl[(SF_N + 1) * 32] = S.N.y; sl[(SF_N + 2) * 32] = S.N.z;
                        sl[SF_HABS * 32] = S.habs;
                        sl[SF_TN * 32] = S.TN;
                        sl[SF_ID * 32] = __uint_as_float(tri_id(P.tri, t));
                        sl[SF_TRI * 32] = __int_as_float((int)t);
                        sl[SF_CFROM * 32] = __int_as_float((int)(desc & 0xffffu));
                        sl[SF_RLO * 32] = __int_as_float((int)((desc >> 26) & 0xffffu));
                        sl[SF_LEN * 32] = __int_as_float(len);
                        sl[SF_INVLEN * 32] = 1.f / (float)len;
                        sl[SF_EM * 32] = __int_as_float(e);
                    } else {
                        cnt[ST_DEGEN]++;
                    }
                }
            }
            // A5: warp-level prefix-scan work expansion
            int incl = my;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl += y;
            }
            if (my) slot[SF_EXCL * 32 + lane] = __int_as_float(incl - my);
            const int total = __shfl_sync(FULL, incl, 31);
            __syncwarp();
            for (int b = 0; b < total; b += 32) {
                const int qi = b + lane;
                int ow = 0;
#pragma unroll
                for (int s = 16; s > 0; s >>= 1) {
                    const int vv = __shfl_sync(FULL, incl, ow + s - 1);
                    if (vv <= qi) ow += s;
                }
                if (qi < total) {
                    const float *sl = slot + ow;
                    const EmDev &EO = sE[__float_as_int(sl[SF_EM * 32])];
                    const int local = qi - __float_as_int(sl[SF_EXCL * 32]);
                    const int len = __float_as_int(sl[SF_LEN * 32]);
                    int row = (int)(((float)local + 0.5f) * sl[SF_INVLEN * 32]);
                    int col = local - row * len;
                    if (col < 0) { --row; col += len; }
                    if (col >= len) { ++row; col -= len; }
                    const int j = __float_as_int(sl[SF_CFROM * 32]) + row;
                    int i = __float_as_int(sl[SF_RLO * 32]) + col;
                    if (i >= EO.chi) i -= EO.chi;
                    const int g = EO.ray_base + j * EO.chi + i;
                    const float4 d = __ldg(P.raytab + chk_idx(g, P.n_rays, CHK_RAY));
                    Setup Q;
                    Q.n0 = {sl[(SF_N0 + 0) * 32], sl[(SF_N0 + 1) * 32], sl[(SF_N0 + 2) * 32]};
                    Q.n1 = {sl[(SF_N1 + 0) * 32], sl[(SF_N1 + 1) * 32], sl[(SF_N1 + 2) * 32]};
                    Q.n2 = {sl[(SF_N2 + 0) * 32], sl[(SF_N2 + 1) * 32], sl[(SF_N2 + 2) * 32]};
                    Q.B0 = sl[(SF_B + 0) * 32]; Q.B1 = sl[(SF_B + 1) * 32]; Q.B2 = sl[(SF_B + 2) * 32];
                    Q.N = {sl[(SF_N + 0) * 32], sl[(SF_N + 1) * 32], sl[(SF_N + 2) * 32]};
                    Q.habs = sl[SF_HABS * 32];
                    Q.TN = sl[SF_TN * 32];
                    float th = 0.f;
                    int r = P.force64 ? 2 : test_fast(d, Q, EO.dmax_lo, EO.dmax_hi, th);
                    if (r == 2) {
                        cnt[ST_FP64]++;
                        f3 w[3];
                        load_tri(P.tri, (long long)__float_as_int(sl[SF_TRI * 32]), w);
                        r = test_exact_r(w, em_o(EO), d, EO.dmax, P.faces, th);
                    }
                    if (r == 1) {
                        cnt[ST_HITS]++;
                        record_hit(P.hits, P.mc_hits, P.allhits, g, th, __float_as_uint(sl[SF_ID * 32]));
                    }
                }
            }
            __syncwarp();
        }
    }
    cnt[ST_SETUP64] = setup64;
    block_flush(acc, P.stats, cnt);
}

// A5 + A6 for one warp: the items of the lanes' small rectangles (slot columns already written, `my` items
// for this lane) expanded by an inclusive prefix scan and tested 32 at a time.  Warp-collective.
template <bool kFast, bool kC>
__device__ __forceinline__ void expand_items(const KParams &P, const EmDev *sE, const float4 *slot, int *excl,
                                             unsigned long long *wc, int lane, int my) {
    // A5: warp-level prefix-scan work expansion
    int incl = my;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
    }
    excl[lane] = incl - my;
    const int total = __shfl_sync(FULL, incl, 31);
    __syncwarp();
    // one candidate per lane per iteration: resolve the owner (binary search of the inclusive
    // scan), the ray index, then the certified test (scalar state only: nothing to local memory)
    unsigned hw = 0u, fw = 0u;
    // owner lane of item qi (binary search of the inclusive scan) and its global ray index g
    auto resolve = [&](int qi, int &ow, int &g) {
        ow = 0;
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) {
            const int vv = __shfl_sync(FULL, incl, ow + s - 1);
            if (vv <= qi) ow += s;
        }
        g = 0;
        if (qi < total) {
            const float4 r5 = slot[5 * 32 + ow];
            const int local = qi - excl[ow];
            const unsigned lc = __float_as_uint(r5.z);
            const int len = (int)(lc & 0xffffu), chi = (int)(lc >> 16);
#if KF_MAGIC_DIV
            const unsigned mg = __float_as_uint(r5.w);
            const int row = mg ? (int)__umulhi((unsigned)local, mg) : local;
            const int col = local - row * len;
#else
            int row = (int)(((float)local + 0.5f) * r5.w);
            int col = local - row * len;
#if !KF_ROWCOL_EXACT
            if (col < 0) { --row; col += len; }
            if (col >= len) { ++row; col -= len; }
#endif
#endif
            g = __float_as_int(r5.x) + row * chi + col - (col >= __float_as_int(r5.y) ? chi : 0);
        }
    };
#if KF_PREFETCH
    // software-pipelined: the next step's owner, ray index and ray load are issued before this step's test
    int ow_n = 0, g_n = 0;
    float4 d_n = make_float4(0.f, 0.f, 0.f, 0.f);
    if (total > 0) {
        resolve(lane, ow_n, g_n);
        if (lane < total) d_n = __ldg(P.raytab + chk_idx(g_n, P.n_rays, CHK_RAY));
    }
#endif
    for (int b = 0; b < total; b += 32) {
        const int qi = b + lane;
#if KF_PREFETCH
        const int ow = ow_n, g = g_n;
        const float4 d = d_n;
        if (b + 32 < total) {
            resolve(qi + 32, ow_n, g_n);
            if (qi + 32 < total) d_n = __ldg(P.raytab + chk_idx(g_n, P.n_rays, CHK_RAY));
        }
#else
        int ow, g;
        resolve(qi, ow, g);
#endif
        bool hit = false, fb = false;
        if (qi < total) {
            const float4 r4 = slot[4 * 32 + ow];
            const EmDev &EO = sE[__float_as_int(r4.w)];
#if !KF_PREFETCH
            const float4 d = __ldg(P.raytab + chk_idx(g, P.n_rays, CHK_RAY));
#endif
            const float4 r0 = slot[0 * 32 + ow], r1 = slot[1 * 32 + ow], r2 = slot[2 * 32 + ow],
                         r3 = slot[3 * 32 + ow];
            Setup Q;
            Q.n0 = {r0.x, r0.y, r0.z};
            Q.n1 = {r1.x, r1.y, r1.z};
            Q.n2 = {r2.x, r2.y, r2.z};
            Q.B0 = r0.w; Q.B1 = r1.w; Q.B2 = r2.w;
            Q.N = {r3.x, r3.y, r3.z};
            Q.habs = r3.w;
            Q.TN = r4.x;
            float th = 0.f;
            int r = (!kFast && P.force64) ? 2 : test_fast(d, Q, EO.dmax_lo, EO.dmax_hi, th);
            fb = r == 2;
            if (r == 2) {   // rare: reload the ray (keeping d live into the fp64 code spills it)
                f3 wv[3];
                load_tri<kC>(P.tri, (long long)__float_as_int(r4.z), wv);
                const float4 d2 = __ldcg(P.raytab + chk_idx(g, P.n_rays, CHK_RAY));
                r = test_exact_r<true>(wv, em_o(EO), d2, EO.dmax, P.faces, th);
            }
            if (r == 1) {
                hit = true;
                record_hit(P.hits, kFast ? nullptr : P.mc_hits, kFast ? nullptr : P.allhits, g, th,
                           __float_as_uint(r4.y));
            }
        }
        // hit / fp64 counts: warp-uniform sums (a per-lane counter live across the loop would be
        // spilled at the 64-register cap), flushed once per round
#if KF_LANE_COUNT   // per-lane counts packed in one register (hits | fp64 << 16), reduced once per round
        hw += (hit ? 1u : 0u) + (fb ? 0x10000u : 0u);
#else
        hw += __popc(__ballot_sync(FULL, hit));
        fw += __popc(__ballot_sync(FULL, fb));
#endif
    }
#if KF_LANE_COUNT
    hw = __reduce_add_sync(FULL, hw);   // each half <= 32 x small_max (<= 1023) < 2^16: no carry
    fw = hw >> 16;
    hw &= 0xffffu;
#endif
    if (lane == 0) {
        wc[ST_HITS] += hw;
        wc[ST_FP64] += fw;
    }
    __syncwarp();
}

// ----------------------------------------- K2b+K4s fused: refine + small work --
// One warp per 32-survivor round (interleaved over all warps): lane-per-survivor exact rectangle
// (cull_pair), certified setup of small rectangles into shared-memory float4 slots, then the
// warp expands all items of its small rectangles with a prefix scan (A5) and tests them 32 at a
// time (A6).  Large rectangles go to the large list (K3/K4).  One vertex fetch per survivor.
// One round of the fused refine + small expansion (A4-A6) for up to 32 survivor entries
// (tri << 8 | emitter, one per lane, valid lanes only): exact rectangle (cull_pair), small
// rectangles set up and expanded over the warp (prefix scan), large ones appended to the large
// list.  Warp-collective; slot / excl are this warp's shared-memory staging areas.
// kFast: no debug / multicast modes (no-cull, forced fp64, all-hit counts, NVLS keys), so the per-
// candidate checks of those flags compile away (the host launches this instantiation when they are off)
template <bool kFast, bool kLevel, bool kC>
__device__ __forceinline__ void refine_round(const KParams &P, const EmDev *sE, const float *sSin,
                                             const unsigned char *sLut, float4 *slot, int *excl,
                                             unsigned long long *wc, int smax, int lane, bool valid,
                                             unsigned long long ent) {
    // per-lane category = the stat it counts (warp-private counters wc[], no atomics)
    enum { C_NONE = -1, C_SMALL = ST_SMALL, C_LARGE = ST_LARGE, C_OVF = ST_OVF_LARGE, C_RANGE = ST_RANGE,
           C_CHAN = ST_CHANNEL, C_AZI = ST_AZIMUTH, C_DEGEN = ST_DEGEN };
    int my = 0, e = 0, cat = C_NONE;
#if KF_SB_INT
    unsigned sb = 0u;   // paper classification: 1 = SAT, 2 = BAT (a value, not two live predicates)
#else
    bool sat = false, bat = false;   // paper classification counters
#endif
    long long t = 0;
    Rect R;
    bool large = false;
    if (valid) {
        e = (int)(ent & 255u);
        t = (long long)(ent >> 8);
        f3 v[3];
        load_tri<kC>(P.tri, t, v);
        const EmDev &E = sE[e];
        const int st = cull_pair<kLevel>(v, E, sSin + E.sin_base, P.lut ? sLut + e * kLutBins : nullptr,
                                         !kFast && P.nocull != 0, R);
        if (st == CULL_KEEP) {
            // Eq. sat_cond with (gamma_T, chi_T) = (64, 64); all-CW = the arc does not wrap the seam
            const bool wraps = R.r_len >= E.chi || R.r_lo + R.r_len > E.chi || R.pole_rows;
#if KF_SB_INT
            sb = (!wraps && (R.c_to - R.c_from + 1) <= 64 && R.r_len <= 64) ? 1u : 2u;
#else
            sat = !wraps && (R.c_to - R.c_from + 1) <= 64 && R.r_len <= 64;
            bat = !sat;
#endif
            const long long items = rect_items(R, E);
            if (items <= smax && !R.pole_rows) {
                if (setup_to_slot(v, em_o(E), P.faces, slot + lane, tri_id(P.tri, t), (int)t, e)) {
                    my = (int)items;
                    cat = C_SMALL;
                    // ray of item (row, col) = gbase + row * chi + col - (col >= chi - r_lo ? chi : 0)
                    // (storing this before the setup, so that R is dead across it, measured slower: 0.482 -> 0.490 ms)
                    slot[5 * 32 + lane] = make_float4(__int_as_float(E.ray_base + R.c_from * E.chi + R.r_lo),
                                                      __int_as_float(E.chi - R.r_lo),
                                                      __uint_as_float((unsigned)R.r_len | ((unsigned)E.chi << 16)),
#if KF_MAGIC_DIV
                                                      // row = local / len exactly as umulhi(local, ceil(2^32 / len))
                                                      // (local < 2^16, len < 2^16); len = 1 -> 0 (row = local)
                                                      __uint_as_float(R.r_len > 1 ? (unsigned)((0x100000000ull + (unsigned)R.r_len - 1) /
                                                                                               (unsigned)R.r_len) : 0u));
#else
                                                      __fdividef(1.f, (float)R.r_len));   // row guess, corrected by +-1
#endif
                } else {
                    cat = C_DEGEN;
                }
            } else {
                large = true;
            }
        } else cat = st == CULL_RANGE ? C_RANGE : st == CULL_CHANNEL ? C_CHAN : st == CULL_AZIMUTH ? C_AZI : C_DEGEN;
    }
    const unsigned lm = __ballot_sync(FULL, large);
    if (lm) {
        const int leader = __ffs(lm) - 1;
        unsigned base = 0;
        if (lane == leader) base = atomicAdd(P.n_large, (unsigned)__popc(lm));
        base = __shfl_sync(FULL, base, leader);
        if (large) {
            const long long pos = (long long)base + __popc(lm & ((1u << lane) - 1u));
            if (pos < P.cap_large) {
                P.large[pos] = make_int4((int)t, e | (R.c_from << 8), R.c_to,
                                         (int)((unsigned)R.r_lo | ((unsigned)R.r_len << 16)));
                cat = C_LARGE;
            } else {   // capacity fallback: intersect here (slow, never dropped)
                cat = C_OVF;
                if (R.pole_rows) { R.r_lo = 0; R.r_len = sE[e].chi; }
                intersect_rect_serial(P, sE[e], t, R.c_from, R.c_to - R.c_from + 1, R.r_lo, R.r_len);
            }
        }
    }
    {   // stats of this round: one match over the category codes, each category's leader lane adds
        // its count to the warp's private counter row (distinct addresses: no atomics)
        const unsigned grp = __match_any_sync(FULL, cat);
        if (cat >= 0 && lane == __ffs(grp) - 1) wc[cat] += (unsigned long long)__popc(grp);
#if KF_SB_INT
        const unsigned msat = __ballot_sync(FULL, sb & 1u), mbat = __ballot_sync(FULL, sb & 2u);
#else
        const unsigned msat = __ballot_sync(FULL, sat), mbat = __ballot_sync(FULL, bat);
#endif
        const unsigned items = __reduce_add_sync(FULL, (unsigned)my);
        if (lane == 0) {
            wc[ST_SAT] += __popc(msat);
            wc[ST_BAT] += __popc(mbat);
            wc[ST_ITEMS_SMALL] += items;
        }
    }
    expand_items<kFast, kC>(P, sE, slot, excl, wc, lane, my);
}

// lane-0 atomic add without the compiler's warp-aggregation wrapper (a single issuing lane)
__device__ __forceinline__ unsigned atom_add_u32(unsigned *p, unsigned v) {
    unsigned old;
    asm volatile("atom.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

template <bool kFast, bool kLevel, bool kC>
__global__ void __launch_bounds__(KF_THREADS, KF_MINB) k_refine_small(const __grid_constant__ KParams P) {
    extern __shared__ __align__(16) unsigned char smem[];
    float4 *sSlot = reinterpret_cast<float4 *>(smem);   // [warp][6][32]
    int *sExcl = reinterpret_cast<int *>(sSlot + (KF_THREADS / 32) * 6 * 32);   // [warp][32]
    EmDev *sE = reinterpret_cast<EmDev *>(sExcl + KF_THREADS);
    float *sSin = reinterpret_cast<float *>(sE + P.n_em);
    unsigned char *sLut = reinterpret_cast<unsigned char *>(sSin + ((P.n_sin + 3) & ~3));
    __shared__ unsigned long long sWc[(KF_THREADS / 32) * 32];   // per-warp stat rows (no atomics)
    {
        const int nw = P.n_em * (int)(sizeof(EmDev) / 4);
        const int *src = reinterpret_cast<const int *>(P.em);
        int *dst = reinterpret_cast<int *>(sE);
        for (int i = threadIdx.x; i < nw; i += blockDim.x) dst[i] = src[i];
        for (int i = threadIdx.x; i < P.n_sin; i += blockDim.x) sSin[i] = P.sin[i];
        if (P.lut)
            for (int i = threadIdx.x; i < P.n_em * kLutBins; i += blockDim.x) sLut[i] = P.lut[i];
        for (int i = threadIdx.x; i < (KF_THREADS / 32) * 32; i += blockDim.x) sWc[i] = 0ull;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    float4 *slot = sSlot + wib * 6 * 32;
    int *excl = sExcl + wib * 32;
    const unsigned ns = *P.n_surv;
    const unsigned nr = (ns + 31) >> 5;   // dense rounds of 32 survivors
    // Small-rectangle cap scaled to the load: with few rounds per warp the longest round is the
    // kernel's tail, so big rectangles go to the chunk-balanced K3/K4 path instead (same results:
    // both paths run the same certified test).  C4: ~56 rounds/warp -> small_max; C2: ~1 -> 64.
    const unsigned rpw = nr / (gridDim.x * (KF_THREADS / 32));
    const int smax = min(P.small_max, (int)max(64u, min(rpw, 1024u) * (unsigned)KF_SMAX_MUL));
    // dynamic round fetching (one global atomic per warp per `fetch` rounds): fewer same-address atomics
    // when every warp has many rounds, single rounds (the finest tail) when it has few
    const unsigned fetch = rpw >= 16u ? (unsigned)KF_FETCH : 1u;
#if KF_FETCH_TAIL   // the counter counts rounds; the last KF_FETCH_TAIL rounds per warp are fetched one at a time
    const unsigned tail_rounds = (unsigned)KF_FETCH_TAIL * gridDim.x * (KF_THREADS / 32);
    unsigned w = 0, cnt = fetch;
    if (lane == 0) w = atom_add_u32(P.n_surv + 2, fetch);
    w = __shfl_sync(FULL, w, 0);
    for (; w < nr;) {
        const unsigned fn = (w + cnt + tail_rounds >= nr) ? 1u : fetch;
        unsigned wn = 0;
        if (lane == 0) wn = atom_add_u32(P.n_surv + 2, fn);   // next group, fetched early (latency hidden)
#pragma unroll 1
        for (unsigned f = 0; f < cnt; ++f) {
#else
    unsigned w = 0;
    if (lane == 0) w = atom_add_u32(P.n_surv + 2, 1u);
    w = __shfl_sync(FULL, w, 0) * fetch;
    for (; w < nr;) {
        unsigned wn = 0;
        if (lane == 0) wn = atom_add_u32(P.n_surv + 2, 1u);   // next group, fetched early (latency hidden)
#pragma unroll 1
        for (unsigned f = 0; f < fetch; ++f) {
#endif
            const unsigned idx = (w + f) * 32u + (unsigned)lane;
            const bool valid = idx < ns;
            if (!__any_sync(FULL, valid)) break;
            refine_round<kFast, kLevel, kC>(P, sE, sSin, sLut, slot, excl, sWc + wib * 32, smax, lane, valid,
                                        valid ? __ldcs(P.surv + idx) : 0ull);
        }
#if KF_FETCH_TAIL
        w = __shfl_sync(FULL, wn, 0);
        cnt = fn;
#else
        w = __shfl_sync(FULL, wn, 0) * fetch;
#endif
    }
    __syncthreads();
    if (threadIdx.x < ST_COUNT) {   // block total of each counter, one global atomic each
        const int c = threadIdx.x;
        unsigned long long v = 0ull;
        for (int w2 = 0; w2 < KF_THREADS / 32; ++w2) {
            const unsigned long long *r = sWc + w2 * 32;
            v += c == ST_SURV ? r[ST_SMALL] + r[ST_LARGE] + r[ST_OVF_LARGE] : r[c];
        }
        if (v) atomicAdd(P.stats + c, v);
    }
}

// ------------------------------------------------------------------ K3 bin --
__device__ __noinline__ void intersect_rect_serial(const KParams &P, const EmDev &E, long long t, int row0, int nrows, int lo,
                                                   int len) {
    // capacity-overflow fallback (rare): one thread tests a whole rectangle; stats via global atomics
    f3 v[3];
    load_tri(P.tri, t, v);
    const uint32_t id = tri_id(P.tri, t);
    Setup S;
    unsigned setup64 = 0, items = 0, fp64 = 0, hits = 0;
    if (make_setup(v, em_o(E), P.faces, S, setup64)) {
        for (int r = 0; r < nrows; ++r)
            for (int c = 0; c < len; ++c) {
                int i = lo + c;
                if (i >= E.chi) i -= E.chi;
                const int g = E.ray_base + (row0 + r) * E.chi + i;
                const float4 d = __ldg(P.raytab + chk_idx(g, P.n_rays, CHK_RAY));
                float th;
                ++items;
                int res = P.force64 ? 2 : test_fast(d, S, E.dmax_lo, E.dmax_hi, th);
                if (res == 2) { ++fp64; res = test_exact_r(v, em_o(E), d, E.dmax, P.faces, th); }
                if (res == 1) { ++hits; record_hit(P.hits, P.mc_hits, P.allhits, g, th, id); }
            }
    }
    atomicAdd(P.stats + ST_ITEMS_LARGE, (unsigned long long)items);
    atomicAdd(P.stats + ST_FP64, (unsigned long long)fp64);
    atomicAdd(P.stats + ST_HITS_L, (unsigned long long)hits);
}

__global__ void __launch_bounds__(256, K3_MINB) k_bin(const __grid_constant__ KParams P) {
    // one warp per large rectangle; lanes = channel rows.  A7 refines each non-pole row of a
    // partial-arc rectangle to its exact (padded) ray range; rows become chunks of <= kColMax rays.
    __shared__ unsigned long long acc[ST_COUNT];
    if (threadIdx.x < ST_COUNT) acc[threadIdx.x] = 0ull;
    __syncthreads();
    unsigned cnt[ST_COUNT];
#pragma unroll
    for (int c = 0; c < ST_COUNT; ++c) cnt[c] = 0u;
    unsigned setup64 = 0;
    const int lane = threadIdx.x & 31;
    const long long n = min((long long)*P.n_large, P.cap_large);
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < n; w += nw) {
        const int4 D = P.large[w];
        const long long tri = D.x;
        const int e = D.y & 255;
        const int c_from = (int)((unsigned)D.y >> 8), c_to = D.z;
        const int r_lo = D.w & 0xffff, r_len = (int)((unsigned)D.w >> 16);
        const EmDev &E = P.em[e];
        const bool full = r_len >= E.chi;
        f3 v[3];
        load_tri(P.tri, tri, v);
        {   // the pair's certified setup, once for all its chunks (K4 reads it; slot layout of
            // setup_to_slot).  Every lane computes the same values; lane k stores float4 k.
            float4 *Sd = P.large_setup + 5 * w;
            const uint32_t id = tri_id(P.tri, tri);
            const bool ok = setup_core(v, em_o(E), P.faces, [&](int k, float4 q) {
                if (k == 4) q = make_float4(q.x, __uint_as_float(id), __int_as_float((int)tri), __int_as_float(e));
                if (lane == k) Sd[k] = q;
            });
            if (!ok) continue;   // Vol = 0 or face-culled: the pair can never hit
        }
        d3 x[3];
        double sk[3];
        float th_ref = 0.f;
        if (!full && !P.norefine) {
            const d3 O = {(double)E.o[0], (double)E.o[1], (double)E.o[2]};
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const d3 a = subd(tod(v[k]), O);
                x[k].x = (double)E.A[0] * a.x + (double)E.A[1] * a.y + (double)E.A[2] * a.z;
                x[k].y = (double)E.A[3] * a.x + (double)E.A[4] * a.y + (double)E.A[5] * a.z;
                x[k].z = (double)E.A[6] * a.x + (double)E.A[7] * a.y + (double)E.A[8] * a.z;
            }
            th_ref = E.theta0 + ((float)r_lo + 0.5f * (float)r_len) * E.dtheta;   // arc centre
#pragma unroll
            for (int k = 0; k < 3; ++k) sk[k] = x[k].z / sqrt(dotd(x[k], x[k]));
        }
        for (int j0 = c_from; j0 <= c_to; j0 += 32) {
            const int j = j0 + lane;
            int lo = 0, len = 0;
            if (j <= c_to) {
                const bool pole_row = j < E.pole_lo || j > E.gamma - 1 - E.pole_hi;
                if (pole_row) { lo = 0; len = E.chi; }
                else if (full || P.norefine) { lo = r_lo; len = r_len; }
                else {
                    const double sj = (double)P.sin[E.sin_base + j];
                    float dmin, dmax;
                    const int nb = refine_row(x, sk, sj - (double)kPadS, sj + (double)kPadS, th_ref, dmin, dmax);
                    if (nb < 2) { lo = r_lo; len = r_len; }
                    else {
                        const float padth = kPadTheta + (E.noisy ? E.dtheta : 0.f);
                        const int ilo = (int)ceilf((th_ref + dmin - padth - E.theta0) * E.inv_dtheta);
                        const int ihi = (int)floorf((th_ref + dmax + padth - E.theta0) * E.inv_dtheta);
                        const int a = max(ilo, r_lo), b = min(ihi, r_lo + r_len - 1);
                        if (a <= b) {
                            lo = a;
                            while (lo >= E.chi) lo -= E.chi;
                            while (lo < 0) lo += E.chi;
                            len = b - a + 1;
                        }
                    }
                }
            }
            const int mych = (len + kColMax - 1) / kColMax;
            int incl = mych;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl += y;
            }
            const int total = __shfl_sync(FULL, incl, 31);
            unsigned wbase = 0;
            if (lane == 31 && total) wbase = atomicAdd(P.n_chunks, (unsigned)total);
            wbase = __shfl_sync(FULL, wbase, 31);
            if (!mych) continue;
            long long pos = (long long)wbase + incl - mych;
            // every reserved slot below the capacity is written (K4 runs min(n_chunks, cap) slots, so a
            // skipped one would replay a stale chunk); the columns past the capacity are intersected
            // here (capacity fallback: slower, never dropped)
            int c0 = 0;
            for (; c0 < len && pos < P.cap_chunks; c0 += kColMax) {
                int l0 = lo + c0;
                if (l0 >= E.chi) l0 -= E.chi;
                P.chunks[pos++] = make_int4((int)w, e | (j << 8), (int)(1u | ((unsigned)l0 << 16)),
                                            min(kColMax, len - c0));
                cnt[ST_CHUNKS]++;
            }
            if (c0 < len) {
                cnt[ST_OVF_CHUNK]++;
                int l0 = lo + c0;
                if (l0 >= E.chi) l0 -= E.chi;
                intersect_rect_serial(P, E, tri, j, 1, l0, len - c0);
            }
        }
    }
    cnt[ST_SETUP64] = setup64;
    block_flush(acc, P.stats, cnt);
}

// ------------------------------------------------------------ K4 intersect --
template <bool kFast>   // as refine_round
__global__ void __launch_bounds__(K4_THREADS, K4_MINB) k_isect(const __grid_constant__ KParams P) {
    extern __shared__ __align__(16) unsigned char smem[];
    EmDev *sE = reinterpret_cast<EmDev *>(smem);
    __shared__ unsigned long long acc[ST_COUNT];
    {
        const int nw = P.n_em * (int)(sizeof(EmDev) / 4);
        const int *src = reinterpret_cast<const int *>(P.em);
        int *dst = reinterpret_cast<int *>(sE);
        for (int i = threadIdx.x; i < nw; i += blockDim.x) dst[i] = src[i];
        if (threadIdx.x < ST_COUNT) acc[threadIdx.x] = 0ull;
    }
    __syncthreads();
    unsigned cnt[ST_COUNT];
#pragma unroll
    for (int c = 0; c < ST_COUNT; ++c) cnt[c] = 0u;
    unsigned setup64 = 0;
    const int lane = threadIdx.x & 31;
    const long long n = min((long long)*P.n_chunks, P.cap_chunks);
    // static grid-stride over the chunks (measured: dynamic per-chunk fetching was slower)
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long c = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < n; c += nw) {
        const int4 ch = P.chunks[c];
        const EmDev &E = sE[ch.y & 255];
        const int row0 = (unsigned)ch.y >> 8;
        const int nrows = ch.z & 0xffff;
        const int lo = (unsigned)ch.z >> 16;
        const int len = ch.w;
        // the pair's setup, computed once by K3 (same address in every lane: broadcast loads)
        const float4 *Sp = P.large_setup + 5 * (long long)ch.x;
        const float4 s0 = __ldcg(Sp), s1 = __ldcg(Sp + 1), s2 = __ldcg(Sp + 2), s3 = __ldcg(Sp + 3),
                     s4 = __ldcg(Sp + 4);
        Setup S;
        S.n0 = {s0.x, s0.y, s0.z}; S.B0 = s0.w;
        S.n1 = {s1.x, s1.y, s1.z}; S.B1 = s1.w;
        S.n2 = {s2.x, s2.y, s2.z}; S.B2 = s2.w;
        S.N = {s3.x, s3.y, s3.z}; S.habs = s3.w;
        S.TN = s4.x;
        const uint32_t id = __float_as_uint(s4.y);
        const long long tri = __float_as_int(s4.z);
        const int items = nrows * len;
        const float invl = __fdividef(1.f, (float)len);   // row guess, corrected by +-1
        if (lane == 0) cnt[ST_ITEMS_LARGE] += items;
        auto ray_of = [&](int q) {
            int row = (int)(((float)q + 0.5f) * invl);
            int col = q - row * len;
            if (col < 0) { --row; col += len; }
            if (col >= len) { ++row; col -= len; }
            int i = lo + col;
            if (i >= E.chi) i -= E.chi;
            return E.ray_base + (row0 + row) * E.chi + i;
        };
        // software-pipelined: the next item's ray is in flight while this one is tested
        int gn = lane < items ? ray_of(lane) : 0;
        float4 dn = lane < items ? __ldg(P.raytab + chk_idx(gn, P.n_rays, CHK_RAY)) : make_float4(0.f, 0.f, 0.f, 0.f);
        for (int q = lane; q < items; q += 32) {
            const int g = gn;
            const float4 d = dn;
            if (q + 32 < items) {
                gn = ray_of(q + 32);
                dn = __ldg(P.raytab + chk_idx(gn, P.n_rays, CHK_RAY));
            }
            float th = 0.f;
            int r = (!kFast && P.force64) ? 2 : test_fast(d, S, E.dmax_lo, E.dmax_hi, th);
            if (r == 2) {   // rare: the vertices for the fp64 decision
                cnt[ST_FP64]++;
                f3 v[3];
                load_tri(P.tri, tri, v);
                r = test_exact_r(v, em_o(E), d, E.dmax, P.faces, th);
            }
            if (r == 1) {
                cnt[ST_HITS_L]++;
                record_hit(P.hits, kFast ? nullptr : P.mc_hits, kFast ? nullptr : P.allhits, g, th, id);
            }
        }
    }
    cnt[ST_SETUP64] = setup64;
    block_flush(acc, P.stats, cnt);
}

// ---------------------------------------------------------------- K5 unpack --
// counter-based normal deviate (splitmix64 -> two uniforms -> Box-Muller)
__device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
__device__ __forceinline__ float gauss01(unsigned long long key) {
    const unsigned long long r = splitmix64(key);
    const float u1 = ((unsigned)(r >> 40) + 0.5f) * (1.f / 16777216.f);
    const float u2 = ((unsigned)(r & 0xFFFFFFu) + 0.5f) * (1.f / 16777216.f);
    return sqrtf(-2.f * __logf(u1)) * __cosf(6.283185307f * u2);
}

__device__ __forceinline__ float unpack_dist(unsigned long long k, long long g, float sigma, unsigned long long base) {
    float dv = __uint_as_float((unsigned)(k >> 32));
    if (sigma > 0.f && dv < CUDART_INF_F)   // noise model: range noise after output conversion
        dv = fmaxf(0.f, dv + sigma * gauss01(base ^ (unsigned long long)g));
    return dv;
}

__global__ void k_unpack(const unsigned long long *__restrict__ hits, float *__restrict__ dist,
                         int32_t *__restrict__ tri, long long n, long long first, float sigma, unsigned long long seed,
                         unsigned long long cast_idx) {
    // hits[i] / dist[i] / tri[i] belong to global ray first + i (the noise model's counter key).
    // Two rays per thread step (16-byte key loads, 8-byte stores) when the buffers allow it: a
    // streaming kernel needs ~6.5 MB in flight to reach HBM bandwidth.
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long stride = (long long)gridDim.x * blockDim.x;
    const unsigned long long base = splitmix64(seed ^ (cast_idx << 40));
    const bool vec = ((reinterpret_cast<uintptr_t>(hits) & 15) | (reinterpret_cast<uintptr_t>(dist) & 7) |
                      (reinterpret_cast<uintptr_t>(tri) & 7)) == 0;
    long long done = 0;
    if (vec) {
        const long long n2 = n >> 1;
        const ulonglong2 *h2 = reinterpret_cast<const ulonglong2 *>(hits);
        for (long long i = tid; i < n2; i += stride) {
            const ulonglong2 k = __ldcs(h2 + i);
            const long long g = first + 2 * i;
            if (dist)
                __stcs(reinterpret_cast<float2 *>(dist) + i,
                       make_float2(unpack_dist(k.x, g, sigma, base), unpack_dist(k.y, g + 1, sigma, base)));
            if (tri)
                __stcs(reinterpret_cast<int2 *>(tri) + i,
                       make_int2((int32_t)(unsigned)(k.x & 0xffffffffull), (int32_t)(unsigned)(k.y & 0xffffffffull)));
        }
        done = 2 * n2;
    }
    for (long long i = done + tid; i < n; i += stride) {
        const unsigned long long k = __ldcs(hits + i);
        if (dist) __stcs(dist + i, unpack_dist(k, first + i, sigma, base));
        if (tri) __stcs(tri + i, (int32_t)(unsigned)(k & 0xffffffffull));
    }
}

}  // namespace grca

// =========================================================================
//                                   C ABI
// =========================================================================
using namespace grca;

static constexpr int kRing = 64;
static constexpr int kEv = 8;   // start, after K0, K2, K2b, K4s, K3, K4, K5

static TriSrc no_part_c() {
    TriSrc T{};
    T.n_c0 = LLONG_MAX;
    return T;
}

struct grca_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    grca_create_info ci{};
    std::string err;
    int num_sms = 148;
    int k2_blocks_per_sm = 1, k2b_blocks_per_sm = 1, k4s_blocks_per_sm = 1, k4_blocks_per_sm = 1, kf_blocks_per_sm = 1;
    size_t k2_smem = 0, k2b_smem = 0, k4s_smem = 0, kf_smem = 0;
    // emitters
    int n_em = 0;
    int n_sin = 0;
    long long n_rays = 0;
    std::vector<long long> offsets;
    // device buffers
    float4 *d_raytab = nullptr;
    unsigned long long *d_hits = nullptr;
    // NEXT-f3 fused NVLS merge (grca_set_nvls): this rank's unicast view and the multicast view of
    // the caller's NVLS-bound buffer [n_rays keys][barrier flag]; nvls_epoch counts barriers
    unsigned long long *nvls_uc = nullptr, *nvls_mc = nullptr;
    int nvls_n = 0;
    unsigned nvls_epoch = 0;
    unsigned *d_allhits = nullptr;
    EmDev *d_em = nullptr;
    float *d_sin = nullptr;
    EmLite *d_lite = nullptr;
    unsigned char *d_lut = nullptr;    // n_em * kLutBins when n_em <= kLutMaxEm and all gamma <= 255
    bool use_lut = false;
    unsigned long long *d_surv = nullptr;   // dense K2 survivor list (capacity tiles * 256 * n_em)
    unsigned long long *d_desc = nullptr;
    long long surv_cap_tiles = 0;
    int surv_n_em = 0;
    EmLitePack lite_pack{};
    cudaAccessPolicyWindow l2win{};
    float noise_sigma = 0.f;           // distance noise (K5), 0 = off
    bool all_ortho = false;
    bool all_level = false;   // every frame's up row of M^-1 is exactly (0, 0, 1)
    bool all_dev_level = false;   // every EmDev.level (cull_pair's level instantiation)
    unsigned long long noise_seed = 0;   // persisting window over ray table + hits (num_bytes 0 = off)
    size_t k2f_smem = 0;
    int4 *d_large = nullptr;
    int4 *d_chunks = nullptr;
    float4 *d_large_setup = nullptr;
    unsigned *d_ctrl = nullptr;
    unsigned long long *d_stats = nullptr;
    long long cap_large = 0, cap_chunks = 0;
    // triangles (dynamic / per frame)
    TriSrc tri = no_part_c();
    long long n_tri = 0;
    long long n_tri_ab = 0;   // parts A + B of the dynamic set (part C, the instances, follows them)
    bool have_tri = false;
    // hybrid static/dynamic (NEXT-f2): static triangles cast once into cached keys
    TriSrc st_tri = no_part_c();
    long long st_n = 0;
    bool st_set = false, st_dirty = false;
    unsigned long long *d_static_keys = nullptr;
    unsigned *d_static_allhits = nullptr;
    // collective cast (grca_create_info.nccl_uid / shard_mode / merge / gather_outputs)
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0;
    int shard = 0;                        // resolved by grca_set_emitters: 0 (no communicator) or GRCA_SHARD_*
    int n_em_global = 0;                  // emitters of the layout (h->n_em = the ones this handle casts)
    std::vector<int> own;                 // global indices of the emitters this handle casts
    long long n_rays_own = 0;
    unsigned long long *d_slice = nullptr;   // reduce-scatter receive buffer (ceil(max_rays / nranks) keys)
    unsigned long long *d_scratch = nullptr; // 8 words: stream barrier operand, multimem pointer readback
    // GRCA_MERGE_NVLS: this rank's NCCL symmetric window (keys + barrier flag) and its multimem view
    void *sym_buf = nullptr;
    size_t sym_bytes = 0;
    ncclWindow_t sym_win = nullptr;
    ncclDevComm sym_dc{};
    bool sym_dc_ok = false;
    // GRCA_USE_CUDA_GRAPH: the cast's launch sequence as one executable graph, re-captured per cast and
    // updated in place (cudaGraphExecUpdate: new pointers / sizes, same topology -> no re-instantiation)
    cudaGraphExec_t gexec = nullptr;
    long long graph_updates = 0, graph_instantiations = 0;
    // profiling ring
    cudaEvent_t ev[kRing][kEv];
    bool ev_ok = false;
    long long n_casts = 0;
    bool did_unpack_last = false;
};

static std::string g_create_err;

#define NK(call)                                                                        \
    do {                                                                                \
        ncclResult_t r_ = (call);                                                       \
        if (r_ != ncclSuccess) {                                                        \
            h->err = std::string(#call) + ": " + ncclGetErrorString(r_) + " (" +       \
                     ncclGetLastError(h->comm) + ")";                                   \
            return GRCA_E_NCCL;                                                         \
        }                                                                               \
    } while (0)

#define CK(call)                                                                        \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess) {                                                        \
            h->err = std::string(#call) + ": " + cudaGetErrorString(e_);                \
            return GRCA_E_CUDA;                                                         \
        }                                                                               \
    } while (0)

namespace {
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

grca_status fail(grca_t h, grca_status s, const std::string &m) {
    if (h) h->err = m;
    return s;
}

void sym_release(grca_t h) {   // GRCA_MERGE_NVLS window (collective with the other ranks' releases)
    if (h->sym_win) ncclCommWindowDeregister(h->comm, h->sym_win);
    if (h->sym_buf) ncclMemFree(h->sym_buf);
    if (h->nvls_uc == h->sym_buf) { h->nvls_uc = h->nvls_mc = nullptr; h->nvls_n = 0; }
    h->sym_win = nullptr;
    h->sym_buf = nullptr;
    h->sym_bytes = 0;
}

void free_all(grca_t h) {
    if (h->comm) {
        cudaStreamSynchronize(h->stream);
        sym_release(h);
        if (h->sym_dc_ok) ncclDevCommDestroy(h->comm, &h->sym_dc);
        ncclCommDestroy(h->comm);
        h->comm = nullptr;
    }
    if (h->gexec) cudaGraphExecDestroy(h->gexec);
    h->gexec = nullptr;
    cudaFree(h->d_slice);
    cudaFree(h->d_scratch);
    cudaFree(h->d_raytab);   // (d_hits lives in the same allocation)
    cudaFree(h->d_static_keys);
    cudaFree(h->d_static_allhits);
    cudaFree(h->d_allhits);
    cudaFree(h->d_em);
    cudaFree(h->d_sin);
    cudaFree(h->d_lite);
    cudaFree(h->d_lut);
    cudaFree(h->d_surv);
    cudaFree(h->d_desc);
    cudaFree(h->d_large);
    cudaFree(h->d_chunks);
    cudaFree(h->d_large_setup);
    cudaFree(h->d_ctrl);
    cudaFree(h->d_stats);
    if (h->ev_ok)
        for (int r = 0; r < kRing; ++r)
            for (int k = 0; k < kEv; ++k) cudaEventDestroy(h->ev[r][k]);
    if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
}

size_t nvls_flag_offset(long long n_rays) { return (size_t)((n_rays + 15) / 16) * 16; }   // in u64 words
size_t sym_bytes_for(long long n_rays) { return ((nvls_flag_offset(n_rays) * 8 + 128 + 4095) / 4096) * 4096; }

// GRCA_MERGE_NVLS: allocate this rank's keys + barrier flag as an NCCL symmetric window and bind it
// as the fused merge's (unicast, multicast) pair.  Collective over the communicator (every rank calls
// it from grca_set_emitters).  NCCL supplies the multicast object (NVLS through its own cuMem / POSIX
// handle exchange -- no fabric handles, no IMEX channel); any failure is reported, never silent.
grca_status sym_bind(grca_t h) {
    CK(cudaStreamSynchronize(h->stream));
    sym_release(h);
    const size_t bytes = sym_bytes_for(h->n_rays);
    NK(ncclMemAlloc(&h->sym_buf, bytes));
    h->sym_bytes = bytes;
    NK(ncclCommWindowRegister(h->comm, h->sym_buf, bytes, &h->sym_win, NCCL_WIN_COLL_SYMMETRIC));
    if (!h->sym_dc_ok) {
        ncclDevCommRequirements req = {};
        req.lsaMultimem = true;
        NK(ncclDevCommCreate(h->comm, &req, &h->sym_dc));
        h->sym_dc_ok = true;
    }
    unsigned long long mc = 0;
    k_sym_multimem_ptr<<<1, 1, 0, h->stream>>>(h->sym_win, h->sym_dc, h->d_scratch);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(&mc, h->d_scratch, sizeof(mc), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    if (!mc) {
        h->err = "NCCL gave no lsa multimem pointer (NVLS multicast unavailable on this communicator)";
        return GRCA_E_NCCL;
    }
    h->nvls_uc = reinterpret_cast<unsigned long long *>(h->sym_buf);
    h->nvls_mc = reinterpret_cast<unsigned long long *>(mc);
    h->nvls_n = h->nranks;
    h->nvls_epoch = 0;
    CK(cudaMemsetAsync(h->nvls_uc + nvls_flag_offset(h->n_rays), 0, 128, h->stream));
    CK(cudaMemsetAsync(h->d_ctrl + 7, 0, sizeof(unsigned), h->stream));
    // every rank's flag is zero before any rank's first barrier adds to it: a one-word all-reduce as a
    // stream barrier, then wait for it
    NK(ncclAllReduce(h->d_scratch, h->d_scratch, 1, ncclUint64, ncclMax, h->comm, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return GRCA_OK;
}

KParams params(grca_t h) {
    KParams P;
    P.tri = h->tri;
    P.n_tri = h->n_tri;
    P.em = h->d_em;
    P.sin = h->d_sin;
    P.n_em = h->n_em;
    P.n_sin = h->n_sin;
    P.raytab = h->d_raytab;
    P.hits = h->nvls_uc ? h->nvls_uc : h->d_hits;
    P.mc_hits = h->nvls_mc;
    P.allhits = (h->ci.debug_flags & GRCA_DEBUG_COUNT_ALL_HITS) ? h->d_allhits : nullptr;
    P.large = h->d_large;
    P.n_large = h->d_ctrl + 0;
    P.cap_large = h->cap_large;
    P.chunks = h->d_chunks;
    P.large_setup = h->d_large_setup;
    P.n_chunks = h->d_ctrl + 1;
    P.n_surv = h->d_ctrl + 2;
    P.cap_chunks = h->cap_chunks;
    P.stats = h->d_stats;
    P.faces = h->ci.faces;
    P.nocull = (h->ci.debug_flags & GRCA_DEBUG_NO_CULL) ? 1 : 0;
    P.force64 = (h->ci.debug_flags & GRCA_DEBUG_FORCE_FP64) ? 1 : 0;
    P.norefine = (h->ci.debug_flags & GRCA_DEBUG_NO_REFINE) ? 1 : 0;
    P.small_max = std::min(1023, h->ci.small_max > 0 ? h->ci.small_max : 512);
    P.area_eps2 = h->ci.apparent_area_eps > 0.f ? h->ci.apparent_area_eps * h->ci.apparent_area_eps : 0.f;
    P.pairs_ok = h->all_ortho && !(h->ci.debug_flags & GRCA_DEBUG_NO_PACKED) ? 1 : 0;
    P.n_rays = h->n_rays;
    P.lite = h->d_lite;
    P.lut = h->use_lut ? h->d_lut : nullptr;
    P.surv = h->d_surv;
    P.cap_surv = h->surv_cap_tiles * K2_THREADS * h->surv_n_em;
    P.desc = h->d_desc;
    return P;
}
}  // namespace

template <bool kC>
static const void *k2_fixed_fn_c(int ne, bool level) {
    switch (ne) {
        case 1: return level ? (const void *)k_cull_fixed<1, true, kC> : (const void *)k_cull_fixed<1, false, kC>;
        case 2: return level ? (const void *)k_cull_fixed<2, true, kC> : (const void *)k_cull_fixed<2, false, kC>;
        case 3: return level ? (const void *)k_cull_fixed<3, true, kC> : (const void *)k_cull_fixed<3, false, kC>;
        case 4: return level ? (const void *)k_cull_fixed<4, true, kC> : (const void *)k_cull_fixed<4, false, kC>;
        case 5: return level ? (const void *)k_cull_fixed<5, true, kC> : (const void *)k_cull_fixed<5, false, kC>;
        case 6: return level ? (const void *)k_cull_fixed<6, true, kC> : (const void *)k_cull_fixed<6, false, kC>;
        case 7: return level ? (const void *)k_cull_fixed<7, true, kC> : (const void *)k_cull_fixed<7, false, kC>;
        default: return level ? (const void *)k_cull_fixed<8, true, kC> : (const void *)k_cull_fixed<8, false, kC>;
    }
}
// kc: the triangle set has part C (instances): the instantiation whose loads handle it
static const void *k2_fixed_fn(int ne, bool level, bool kc = false) {
    return kc ? k2_fixed_fn_c<true>(ne, level) : k2_fixed_fn_c<false>(ne, level);
}
// the fused kernel's instantiations: (fast modes, level frames, part C)
static const void *kf_fn(bool fast, bool level, bool kc) {
    if (!fast) return kc ? (const void *)k_refine_small<false, false, true> : (const void *)k_refine_small<false, false, false>;
    if (level) return kc ? (const void *)k_refine_small<true, true, true> : (const void *)k_refine_small<true, true, false>;
    return kc ? (const void *)k_refine_small<true, false, true> : (const void *)k_refine_small<true, false, false>;
}

static size_t k2_smem_bytes(int n_em, int n_sin, bool lut) {
    return sizeof(EmLite) * n_em + sizeof(float) * ((n_sin + 3) & ~3) +
           (lut ? sizeof(unsigned char) * ((n_em * kLutBins + 15) & ~15) : 0) + sizeof(unsigned short) * K2_THREADS * n_em;
}
static size_t k2b_smem_bytes(int n_em, int n_sin, bool lut) {
    return sizeof(EmDev) * n_em + sizeof(float) * ((n_sin + 3) & ~3) + (lut ? (size_t)n_em * kLutBins : 0);
}
static size_t k4s_smem_bytes(int n_em) { return sizeof(EmDev) * n_em + sizeof(float) * NF * K2_THREADS; }
static size_t kfused_smem_bytes(int n_em, int n_sin, bool lut) {
    return sizeof(float4) * (KF_THREADS / 32) * 6 * 32 + sizeof(int) * KF_THREADS +
           sizeof(EmDev) * n_em +
           sizeof(float) * ((n_sin + 3) & ~3) + (lut ? (size_t)n_em * kLutBins : 0);
}

extern "C" {

#ifdef GRCA_CHECK
const char *grca_version(void) { return "grca-b200 0.2 (sm_100a, bounds-checked build)"; }
#else
const char *grca_version(void) { return "grca-b200 0.2 (sm_100a)"; }
#endif

const char *grca_last_error(grca_t h) { return h ? h->err.c_str() : g_create_err.c_str(); }

grca_status grca_create(const grca_create_info *ci, grca_t *out) {
    if (!ci || !out) { g_create_err = "null argument"; return GRCA_E_INVALID; }
    *out = nullptr;
    if (ci->max_triangles < 0 || ci->max_rays < 1 || ci->max_rays > (1ll << 25) || ci->max_large_items < 0 ||
        ci->faces < 0 || ci->faces > 2 || ci->small_max < 0) {
        g_create_err = "invalid create info (max_rays in [1, 2^25], faces in {0,1,2}, sizes >= 0)";
        return GRCA_E_INVALID;
    }
    const int nranks = ci->nranks < 1 ? 1 : ci->nranks;
    if (ci->rank < 0 || ci->rank >= nranks || ci->shard_mode < 0 || ci->shard_mode > 2 || ci->merge < 0 ||
        ci->merge > 2 || (nranks > 1 && !ci->nccl_uid && !(ci->debug_flags & GRCA_DEBUG_VIRTUAL_RANKS)) ||
        (ci->merge == GRCA_MERGE_NVLS && !ci->nccl_uid)) {
        g_create_err = "invalid collective setup (rank in [0, nranks), shard_mode in {0,1,2}, merge in {0,1,2}; "
                       "nranks > 1 and GRCA_MERGE_NVLS need nccl_uid)";
        return GRCA_E_INVALID;
    }
    grca_t h = new grca_ctx();
    h->ci = *ci;
    h->device = ci->device;
    h->nranks = nranks;
    h->rank = ci->rank;
    DeviceGuard dg(h->device);
    cudaError_t e = cudaSetDevice(h->device);
    if (e != cudaSuccess) {
        g_create_err = std::string("cudaSetDevice: ") + cudaGetErrorString(e);
        delete h;
        return GRCA_E_CUDA;
    }
    cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, h->device);
    // NULL -> the legacy default stream (what torch's default stream is), never a private one
    h->stream = (cudaStream_t)ci->stream;
    h->own_stream = false;
    const long long mt = std::max<long long>(1, ci->max_triangles);
    h->cap_large = ci->max_large_items > 0 ? ci->max_large_items : std::max<long long>(1ll << 20, mt / 4);
    h->cap_chunks = 4 * h->cap_large;
    bool ok = true;
    auto alloc = [&](void **p, size_t bytes) {
        if (ok && cudaMalloc(p, bytes) != cudaSuccess) ok = false;
    };
    // ray table and hit keys in ONE allocation so a single persisting L2 access-policy window
    // covers both (the gathers of K4s/K4 hit them randomly; the triangle stream must not evict them)
    // (the keys are padded by nranks entries: a reduce-scatter merges ceil(n / P) * P keys)
    alloc((void **)&h->d_raytab, sizeof(float4) * ci->max_rays + sizeof(unsigned long long) * (ci->max_rays + nranks));
    if (ok) h->d_hits = reinterpret_cast<unsigned long long *>(h->d_raytab + ci->max_rays);
    if (ci->debug_flags & GRCA_DEBUG_COUNT_ALL_HITS) alloc((void **)&h->d_allhits, sizeof(unsigned) * ci->max_rays);
    alloc((void **)&h->d_static_keys, sizeof(unsigned long long) * ci->max_rays);
    if (ci->debug_flags & GRCA_DEBUG_COUNT_ALL_HITS) alloc((void **)&h->d_static_allhits, sizeof(unsigned) * ci->max_rays);
    alloc((void **)&h->d_em, sizeof(EmDev) * kMaxEmitters);
    alloc((void **)&h->d_sin, sizeof(float) * kMaxSin);
    alloc((void **)&h->d_lite, sizeof(EmLite) * kMaxEmitters);
    alloc((void **)&h->d_lut, sizeof(unsigned char) * kLutMaxEm * kLutBins);
    alloc((void **)&h->d_large, sizeof(int4) * h->cap_large);
    alloc((void **)&h->d_chunks, sizeof(int4) * h->cap_chunks);
    alloc((void **)&h->d_large_setup, sizeof(float4) * 5 * h->cap_large);
    alloc((void **)&h->d_ctrl, sizeof(unsigned) * 8);
    alloc((void **)&h->d_stats, sizeof(unsigned long long) * 32);
    alloc((void **)&h->d_scratch, sizeof(unsigned long long) * 8);
    if (ci->nccl_uid) alloc((void **)&h->d_slice, sizeof(unsigned long long) * ((ci->max_rays + nranks - 1) / nranks));
    if (!ok) {
        g_create_err = "device allocation failed";
        cudaGetLastError();
        free_all(h);
        delete h;
        return GRCA_E_OOM;
    }
    if (ci->debug_flags & GRCA_PROFILE_KERNELS) {
        h->ev_ok = true;
        for (int r = 0; r < kRing; ++r)
            for (int k = 0; k < kEv; ++k)
                if (cudaEventCreate(&h->ev[r][k]) != cudaSuccess) h->ev_ok = false;
    }
    cudaMemsetAsync(h->d_ctrl, 0, sizeof(unsigned) * 8, h->stream);
    cudaMemsetAsync(h->d_stats, 0, sizeof(unsigned long long) * 32, h->stream);
    // occupancy of the persistent kernels (K2 smem depends on emitters: use the max)
    cudaFuncSetAttribute(k_cull, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k2_smem_bytes(kMaxEmitters, kMaxSin, false));
    cudaFuncSetAttribute(k_refine, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k2b_smem_bytes(kMaxEmitters, kMaxSin, false));
    cudaFuncSetAttribute(k_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k4s_smem_bytes(kMaxEmitters));
    for (bool kc : {false, true})
        for (const void *f : {kf_fn(true, true, kc), kf_fn(true, false, kc), kf_fn(false, false, kc)})
            cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kfused_smem_bytes(kMaxEmitters, kMaxSin, false));
    for (const void *f : {(const void *)k_isect<true>, (const void *)k_isect<false>})
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(sizeof(EmDev) * kMaxEmitters));
    {   // opt-in persisting L2 window for the ray table + hits (measured: no gain at C4 after the
        // triangle streams were made evict-first, and K0/K5 lose from the carve-out)
        int max_persist = 0;
        cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, h->device);
        const size_t win = (sizeof(float4) + sizeof(unsigned long long)) * (size_t)ci->max_rays;
        if (max_persist > 0 && (ci->debug_flags & GRCA_L2_PERSIST)) {
            size_t cur = 0;
            cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
            const size_t want = std::min<size_t>(win, (size_t)max_persist);
            if (cur < want) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
            cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
            h->l2win.base_ptr = h->d_raytab;
            h->l2win.num_bytes = std::min<size_t>(win, (size_t)max_persist * 4);
            h->l2win.hitRatio = (float)std::min(1.0, (double)cur / (double)h->l2win.num_bytes);
            h->l2win.hitProp = cudaAccessPropertyPersisting;
            h->l2win.missProp = cudaAccessPropertyStreaming;
        }
        cudaGetLastError();
    }
    cudaStreamSynchronize(h->stream);
    if (cudaGetLastError() != cudaSuccess) {
        g_create_err = "CUDA setup failed (is this an sm_100a device?)";
        free_all(h);
        delete h;
        return GRCA_E_CUDA;
    }
    if (ci->nccl_uid) {   // the collective cast's communicator (blocks until every rank has joined)
        ncclUniqueId id;
        memcpy(&id, ci->nccl_uid, sizeof(id));
        const ncclResult_t r = ncclCommInitRank(&h->comm, nranks, id, ci->rank);
        if (r != ncclSuccess) {
            g_create_err = std::string("ncclCommInitRank: ") + ncclGetErrorString(r) + " (" + ncclGetLastError(nullptr) + ")";
            h->comm = nullptr;
            free_all(h);
            delete h;
            return GRCA_E_NCCL;
        }
    }
    *out = h;
    return GRCA_OK;
}

grca_status grca_nccl_unique_id(void *out) {
    if (!out) return GRCA_E_INVALID;
    ncclUniqueId id;
    const ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) {
        g_create_err = std::string("ncclGetUniqueId: ") + ncclGetErrorString(r);
        return GRCA_E_NCCL;
    }
    memcpy(out, &id, sizeof(id));
    return GRCA_OK;
}

grca_status grca_destroy(grca_t h) {
    if (!h) return GRCA_OK;
    DeviceGuard dg(h->device);
    cudaStreamSynchronize(h->stream);
    free_all(h);
    delete h;
    return GRCA_OK;
}

grca_status grca_set_emitters(grca_t h, const grca_emitter *em, int32_t n_emitters) {
    if (!h) return GRCA_E_INVALID;
    if (!em || n_emitters < 1 || n_emitters > kMaxEmitters)
        return fail(h, GRCA_E_INVALID, "n_emitters must be in [1, 255]");
    const float halfpi32 = (float)(M_PI / 2);
    std::vector<EmDev> recs(n_emitters);
    std::vector<float> sins;
    std::vector<long long> offs(n_emitters + 1, 0);
    for (int n = 0; n < n_emitters; ++n) {
        const grca_emitter &E = em[n];
        const std::string tag = "emitter " + std::to_string(n) + ": ";
        if (E.n_channels < 1 || E.n_channels > 65535) return fail(h, GRCA_E_INVALID, tag + "n_channels not in [1, 65535]");
        if (E.rays_per_channel < 1 || E.rays_per_channel > 65535)
            return fail(h, GRCA_E_INVALID, tag + "rays_per_channel not in [1, 65535]");
        if (E.hfov_deg != 360 && E.hfov_deg != 180) return fail(h, GRCA_E_INVALID, tag + "hfov_deg must be 180 or 360");
        if (!E.channel_elev_rad) return fail(h, GRCA_E_INVALID, tag + "null elevation table");
        for (int j = 0; j < E.n_channels; ++j) {
            const float p = E.channel_elev_rad[j];
            if (!(fabsf(p) <= halfpi32)) return fail(h, GRCA_E_INVALID, tag + "|elevation| > RN32(pi/2) or NaN");
            if (j && !(p > E.channel_elev_rad[j - 1]))
                return fail(h, GRCA_E_INVALID, tag + "elevation table not strictly ascending");
        }
        for (int c = 0; c < 3; ++c)
            if (!std::isfinite(E.origin[c]) || !std::isfinite(E.forward[c]) || !std::isfinite(E.right[c]) ||
                !std::isfinite(E.up[c]))
                return fail(h, GRCA_E_INVALID, tag + "non-finite origin/frame");
        double F[3], Rr[3], U[3];
        for (int c = 0; c < 3; ++c) { F[c] = E.forward[c]; Rr[c] = E.right[c]; U[c] = E.up[c]; }
        auto dot = [](const double *a, const double *b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; };
        if (fabs(dot(F, F) - 1) > 1e-3 || fabs(dot(Rr, Rr) - 1) > 1e-3 || fabs(dot(U, U) - 1) > 1e-3 ||
            fabs(dot(F, Rr)) > 1e-3 || fabs(dot(F, U)) > 1e-3 || fabs(dot(Rr, U)) > 1e-3)
            return fail(h, GRCA_E_INVALID, tag + "frame (forward, right, up) not orthonormal within 1e-3");
        // M = [f r u] (columns); A = M^-1 via the adjugate, fp64
        const double M[3][3] = {{F[0], Rr[0], U[0]}, {F[1], Rr[1], U[1]}, {F[2], Rr[2], U[2]}};
        const double det = M[0][0] * (M[1][1] * M[2][2] - M[1][2] * M[2][1]) -
                           M[0][1] * (M[1][0] * M[2][2] - M[1][2] * M[2][0]) +
                           M[0][2] * (M[1][0] * M[2][1] - M[1][1] * M[2][0]);
        double Ainv[3][3];
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) {
                const int r1 = (c + 1) % 3, r2 = (c + 2) % 3, c1 = (r + 1) % 3, c2 = (r + 2) % 3;
                Ainv[r][c] = (M[r1][c1] * M[r2][c2] - M[r1][c2] * M[r2][c1]) / det;
            }
        EmDev &D = recs[n];
        memset(&D, 0, sizeof(D));
        for (int c = 0; c < 3; ++c) D.o[c] = E.origin[c];
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) D.A[3 * r + c] = (float)Ainv[r][c];
        const double H = (E.hfov_deg == 180) ? M_PI : 2.0 * M_PI;
        const double dth = H / (double)E.rays_per_channel;
        D.dtheta = (float)dth;
        D.inv_dtheta = (float)(1.0 / dth);
        D.theta0 = (float)(-(double)(E.rays_per_channel / 2) * dth);
        const bool ranged = E.max_range > 0.f && std::isfinite(E.max_range);
        D.dmax = ranged ? (double)E.max_range : INFINITY;
        D.dmax_lo = ranged ? (float)((double)E.max_range * (1.0 - 5e-6)) : INFINITY;
        D.dmax_hi = ranged ? (float)((double)E.max_range * (1.0 + 5e-6)) : INFINITY;
        D.gamma = E.n_channels;
        D.chi = E.rays_per_channel;
        D.hfov = E.hfov_deg;
        D.ray_base = (int)offs[n];
        D.sin_base = (int)sins.size();
        int plo = 0, phi = 0;
        for (int j = 0; j < E.n_channels; ++j) {
            const double p = (double)E.channel_elev_rad[j];
            sins.push_back((float)sin(p));
        }
        sins.push_back(INFINITY);   // sentinels: sinT[gamma] = sinT[gamma + 1] = +inf
        sins.push_back(INFINITY);
        while (plo < E.n_channels && cos((double)E.channel_elev_rad[plo]) < 0.01) ++plo;
        while (phi < E.n_channels - plo && cos((double)E.channel_elev_rad[E.n_channels - 1 - phi]) < 0.01) ++phi;
        D.pole_lo = plo;
        D.pole_hi = phi;
        D.noisy = E.ray_azimuth_rad ? 1 : 0;
        D.level = (D.A[2] == 0.f && D.A[5] == 0.f && D.A[6] == 0.f && D.A[7] == 0.f && D.A[8] == 1.f) ? 1 : 0;
        if (E.ray_azimuth_rad) {   // noise model: |theta*_i - theta_i| < dtheta, strictly ascending
            const double th0 = -(double)(E.rays_per_channel / 2) * dth;
            for (int i = 0; i < E.rays_per_channel; ++i) {
                const double a = (double)E.ray_azimuth_rad[i];
                if (!(fabs(a - (th0 + (double)i * dth)) < dth))
                    return fail(h, GRCA_E_INVALID, tag + "ray_azimuth_rad[i] not within dtheta of the grid angle");
                if (i && !(E.ray_azimuth_rad[i] > E.ray_azimuth_rad[i - 1]))
                    return fail(h, GRCA_E_INVALID, tag + "ray_azimuth_rad not strictly ascending");
            }
        }
        offs[n + 1] = offs[n] + (long long)E.n_channels * E.rays_per_channel;
    }
    if ((int)sins.size() > kMaxSin) return fail(h, GRCA_E_INVALID, "sum of (n_channels + 2) over emitters > 4096");
    if (offs[n_emitters] > h->ci.max_rays) return fail(h, GRCA_E_CAPACITY, "sum gamma*chi exceeds max_rays");
    if (h->nvls_mc && offs[n_emitters] != h->n_rays)   // the bound NVLS buffer was sized for the old rays
        return fail(h, GRCA_E_STATE, "a fused NVLS merge is bound for a different ray count: "
                                     "grca_set_nvls(h, NULL, NULL, 0) first, then re-bind a buffer of the new size");
    // partition of a collective cast: emitter shards cast emitters n mod P == rank over all
    // triangles (disjoint output slices); triangle shards cast every emitter over the rank's triangles
    int shard = 0;
    if (h->comm || (h->ci.debug_flags & GRCA_DEBUG_VIRTUAL_RANKS)) {
        shard = h->ci.shard_mode;
        if (shard == GRCA_SHARD_AUTO)
            shard = (n_emitters >= h->nranks && n_emitters % h->nranks == 0) ? GRCA_SHARD_EMITTERS : GRCA_SHARD_TRIANGLES;
        if (shard == GRCA_SHARD_EMITTERS && h->ci.merge == GRCA_MERGE_NVLS)
            return fail(h, GRCA_E_INVALID, "GRCA_MERGE_NVLS merges triangle shards: use GRCA_SHARD_TRIANGLES");
    }
    std::vector<int> own;
    for (int n = 0; n < n_emitters; ++n)
        if (shard != GRCA_SHARD_EMITTERS || n % h->nranks == h->rank) own.push_back(n);
    const int n_own = (int)own.size();
    {   // the emitters this handle casts: records and sin tables compacted (local index k), ray bases global
        std::vector<EmDev> orecs;
        std::vector<float> osins;
        for (int n : own) {
            EmDev D = recs[n];
            const int sb = D.sin_base;
            D.sin_base = (int)osins.size();
            osins.insert(osins.end(), sins.begin() + sb, sins.begin() + sb + D.gamma + 2);
            orecs.push_back(D);
        }
        recs.swap(orecs);
        sins.swap(osins);
        if (sins.empty()) sins.assign(2, INFINITY);
    }
    long long rays_own = 0;
    for (int n : own) rays_own += offs[n + 1] - offs[n];
    // A0: the fp32 ray table, built in fp64 on the host (Eq. ray_dir)
    std::vector<float4> tab((size_t)offs[n_emitters]);
    for (int n = 0; n < n_emitters; ++n) {
        const grca_emitter &E = em[n];
        const double H = (E.hfov_deg == 180) ? M_PI : 2.0 * M_PI;
        const double dth = H / (double)E.rays_per_channel;
        const double th0 = -(double)(E.rays_per_channel / 2) * dth;
        std::vector<double> ct(E.rays_per_channel), st(E.rays_per_channel);
        for (int i = 0; i < E.rays_per_channel; ++i) {
            const double th = E.ray_azimuth_rad ? (double)E.ray_azimuth_rad[i] : th0 + (double)i * dth;
            ct[i] = cos(th);
            st[i] = sin(th);
        }
        const double f[3] = {E.forward[0], E.forward[1], E.forward[2]};
        const double r[3] = {E.right[0], E.right[1], E.right[2]};
        const double u[3] = {E.up[0], E.up[1], E.up[2]};
        for (int j = 0; j < E.n_channels; ++j) {
            const double p = (double)E.channel_elev_rad[j];
            const double cp = cos(p), sp = sin(p);
            float4 *row = tab.data() + offs[n] + (size_t)j * E.rays_per_channel;
            for (int i = 0; i < E.rays_per_channel; ++i) {
                const double a = ct[i] * cp, b = st[i] * cp;
                row[i] = make_float4((float)(a * f[0] + b * r[0] + sp * u[0]), (float)(a * f[1] + b * r[1] + sp * u[1]),
                                     (float)(a * f[2] + b * r[2] + sp * u[2]), 0.f);
            }
        }
    }
    // K2 phase-A records (EmLite) and the O(1) channel LUTs
    std::vector<EmLite> lites(n_own);
    int max_gamma = 0;
    for (int n : own) max_gamma = std::max(max_gamma, (int)em[n].n_channels);
    const bool use_lut = n_own <= kLutMaxEm && max_gamma <= 255;
    std::vector<unsigned char> lut(use_lut ? (size_t)n_own * kLutBins : 0);
    for (int n = 0; n < n_own; ++n) {   // (n: local index of emitter own[n])
        const grca_emitter &E = em[own[n]];
        const EmDev &D = recs[n];
        EmLite &L = lites[n];
        memset(&L, 0, sizeof(L));
        for (int c = 0; c < 3; ++c) { L.o[c] = D.o[c]; L.Au[c] = D.A[6 + c]; }
        double A[3][3], G[3][3];
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) A[r][c] = D.A[3 * r + c];
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) G[r][c] = A[0][r] * A[0][c] + A[1][r] * A[1][c] + A[2][r] * A[2][c];
        L.G[0] = (float)G[0][0]; L.G[1] = (float)G[1][1]; L.G[2] = (float)G[2][2];
        L.G[3] = (float)G[0][1]; L.G[4] = (float)G[0][2]; L.G[5] = (float)G[1][2];
        double dev = 0;   // frame non-orthonormality
        const double F[3] = {E.forward[0], E.forward[1], E.forward[2]}, Rr[3] = {E.right[0], E.right[1], E.right[2]},
                     U[3] = {E.up[0], E.up[1], E.up[2]};
        auto dot = [](const double *a, const double *b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; };
        dev = std::max({fabs(dot(F, F) - 1), fabs(dot(Rr, Rr) - 1), fabs(dot(U, U) - 1), fabs(dot(F, Rr)),
                        fabs(dot(F, U)), fabs(dot(Rr, U))});
        L.ortho = dev <= 1e-6 ? 1 : 0;
        L.pad0 = kPadS + (L.ortho ? (float)(4.0 * dev + 1e-7) : 0.f);
        const bool ranged = E.max_range > 0.f && std::isfinite(E.max_range);
        L.lim = ranged ? (float)((double)E.max_range * (1.0 + 1e-5)) : INFINITY;
        L.gamma = E.n_channels;
        L.sin_base = D.sin_base;
        L.lut_base = n * kLutBins;
        if (use_lut) {
            const float *st = sins.data() + D.sin_base;
            for (int b = 0; b < kLutBins; ++b) {   // under-estimate: first channel >= bin start - 1e-6
                const float x = (float)(-1.0 + 2.0 * b / kLutBins - 1e-6);
                int j = 0;
                while (j < E.n_channels && st[j] < x) ++j;
                lut[(size_t)n * kLutBins + b] = (unsigned char)j;
            }
        }
    }
    DeviceGuard dg(h->device);
    CK(cudaStreamSynchronize(h->stream));
    // survivor buffer of K2: K2_THREADS * n_em entries per tile of max_triangles
    const long long tiles = (std::max<long long>(1, h->ci.max_triangles) + K2_THREADS - 1) / K2_THREADS;
    if (!h->d_surv || h->surv_n_em < std::max(1, n_own)) {
        cudaFree(h->d_surv);
        cudaFree(h->d_desc);
        h->d_surv = nullptr;
        h->d_desc = nullptr;
        const long long ne = std::max(1, n_own);
        if (cudaMalloc((void **)&h->d_surv, sizeof(unsigned long long) * tiles * K2_THREADS * ne) != cudaSuccess ||
            cudaMalloc((void **)&h->d_desc, sizeof(unsigned long long) * tiles * K2_THREADS * ne) != cudaSuccess) {
            cudaGetLastError();
            h->surv_n_em = 0;
            return fail(h, GRCA_E_OOM, "survivor buffer allocation failed");
        }
        h->surv_n_em = (int)ne;
        h->surv_cap_tiles = tiles;
    }
    // uploads ordered on the handle's stream (which may be a non-blocking side stream), then waited
    // for: the next cast never reads a partially written table
    CK(cudaMemcpyAsync(h->d_raytab, tab.data(), sizeof(float4) * tab.size(), cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(h->d_em, recs.data(), sizeof(EmDev) * recs.size(), cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(h->d_sin, sins.data(), sizeof(float) * sins.size(), cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(h->d_lite, lites.data(), sizeof(EmLite) * lites.size(), cudaMemcpyHostToDevice, h->stream));
    if (use_lut)
        CK(cudaMemcpyAsync(h->d_lut, lut.data(), sizeof(unsigned char) * lut.size(), cudaMemcpyHostToDevice, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    h->use_lut = use_lut;
    h->all_ortho = true;
    h->all_level = true;
    h->all_dev_level = true;
    for (int n = 0; n < n_own; ++n) h->all_dev_level = h->all_dev_level && recs[n].level;
    for (int n = 0; n < n_own; ++n) {
        h->all_ortho = h->all_ortho && lites[n].ortho;
        h->all_level = h->all_level && lites[n].Au[0] == 0.f && lites[n].Au[1] == 0.f && lites[n].Au[2] == 1.f;
    }
    h->n_em = n_own;
    h->n_em_global = n_emitters;
    h->own = own;
    h->shard = shard;
    h->n_rays_own = rays_own;
    h->st_dirty = h->st_set;   // cached static keys depend on the emitters
    h->n_sin = (int)sins.size();
    h->n_rays = offs[n_emitters];
    h->offsets = offs;
    // dynamic smem for these emitters; occupancy of the persistent kernels
    h->k2_smem = k2_smem_bytes(n_own, h->n_sin, use_lut);
    memset(&h->lite_pack, 0, sizeof(h->lite_pack));
    for (int n = 0; n < n_own && n < kFixedEm; ++n) h->lite_pack.e[n] = lites[n];
    for (int n = 0; n + 1 < n_own && n + 1 < kFixedEm; n += 2) {
        EmPair &pr = h->lite_pack.p[n / 2];
        for (int c = 0; c < 3; ++c) {
            pr.no[c] = make_float2(-lites[n].o[c], -lites[n + 1].o[c]);
            pr.u[c] = make_float2(lites[n].Au[c], lites[n + 1].Au[c]);
        }
    }
    h->k2f_smem = sizeof(float) * ((h->n_sin + 3) & ~3) + (use_lut ? (size_t)n_own * kLutBins : 0);
    h->k2b_smem = k2b_smem_bytes(n_own, h->n_sin, use_lut);
    h->k4s_smem = k4s_smem_bytes(n_own);
    h->kf_smem = kfused_smem_bytes(n_own, h->n_sin, use_lut);
    {   // dynamic shared memory of these emitters (the LUT variant can exceed what create assumed)
        int max_optin = 0;
        cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device);
        const size_t need = std::max({h->k2_smem, h->k2f_smem, h->k2b_smem, h->k4s_smem, h->kf_smem});
        if (max_optin > 0 && need > (size_t)max_optin)
            return fail(h, GRCA_E_INVALID, "emitter tables need " + std::to_string(need) +
                                               " B of shared memory per block (> the device's opt-in limit)");
        if (n_own >= 1 && n_own <= kFixedEm && use_lut)
            for (bool lv : {false, true})
                for (bool kc : {false, true})
                    CK(cudaFuncSetAttribute(k2_fixed_fn(n_own, lv, kc), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)h->k2f_smem));
        CK(cudaFuncSetAttribute(k_cull, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->k2_smem));
        CK(cudaFuncSetAttribute(k_refine, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->k2b_smem));
        CK(cudaFuncSetAttribute(k_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->k4s_smem));
        for (bool kc : {false, true})
            for (const void *f : {kf_fn(true, true, kc), kf_fn(true, false, kc), kf_fn(false, false, kc)})
                CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->kf_smem));
    }
    int b2 = 0, b2b = 0, b4s = 0, b4 = 0;
    if (n_own >= 1 && n_own <= kFixedEm && use_lut) {   // the fixed kernel relies on the LUT (gamma <= 255)
        const void *fn = k2_fixed_fn(n_own, false);
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b2, fn, K2_THREADS, h->k2f_smem));
    } else {
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b2, k_cull, K2_THREADS, h->k2_smem));
    }
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b2b, k_refine, K2_THREADS, h->k2b_smem));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b4s, k_small, K2_THREADS, h->k4s_smem));
    h->k4s_blocks_per_sm = std::max(1, b4s);
    int bf = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bf, kf_fn(true, false, false), KF_THREADS, h->kf_smem));
    h->kf_blocks_per_sm = std::max(1, bf);
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b4, k_isect<true>, K4_THREADS, sizeof(EmDev) * std::max(1, n_own)));
    h->k2_blocks_per_sm = std::max(1, b2);
    h->k2b_blocks_per_sm = std::max(1, b2b);
    h->k4_blocks_per_sm = std::max(1, b4);
    if (h->comm && h->ci.merge == GRCA_MERGE_NVLS && (!h->sym_buf || h->sym_bytes != sym_bytes_for(h->n_rays)))
        return sym_bind(h);   // collective: every rank re-binds its symmetric window for the new ray count
    return GRCA_OK;
}

static grca_status check_tri_args(grca_t h, const float *d_vertices, int64_t n_vertices, const uint32_t *d_indices,
                                  int64_t n_triangles, const int32_t *d_tri_ids, int32_t tri_id_base,
                                  bool packed3 = false) {
    if (n_triangles < 0) return fail(h, GRCA_E_INVALID, "n_triangles < 0");
    if (n_triangles > h->ci.max_triangles) return fail(h, GRCA_E_CAPACITY, "n_triangles exceeds max_triangles");
    if (n_triangles > 0 && !d_vertices) return fail(h, GRCA_E_INVALID, "null vertex buffer");
    if (n_triangles > 0 && d_indices && n_vertices < 1) return fail(h, GRCA_E_INVALID, "indexed mesh with no vertices");
    if (n_triangles > 0 && !d_indices && n_vertices < 3 * n_triangles)
        return fail(h, GRCA_E_INVALID, "non-indexed: n_vertices must be >= 3 * n_triangles");
    if (((uintptr_t)d_vertices & (packed3 ? 3 : 15)) != 0)
        return fail(h, GRCA_E_INVALID, packed3 ? "float3 vertex buffer must be 4-byte aligned"
                                               : "vertex buffer must be 16-byte aligned");
    if (tri_id_base < 0 || (!d_tri_ids && (long long)tri_id_base + n_triangles > 0x7fffffffll))
        return fail(h, GRCA_E_INVALID, "triangle ids must be in [0, 2^31)");
    return GRCA_OK;
}

grca_status grca_update_triangles(grca_t h, const float *d_vertices, int64_t n_vertices, const uint32_t *d_indices,
                                  int64_t n_triangles, const int32_t *d_tri_ids, int32_t tri_id_base) {
    if (!h) return GRCA_E_INVALID;
    grca_status st = check_tri_args(h, d_vertices, n_vertices, d_indices, n_triangles, d_tri_ids, tri_id_base);
    if (st != GRCA_OK) return st;
    h->tri.v = reinterpret_cast<const float4 *>(d_vertices);
    h->tri.v3 = nullptr;
    h->tri.va = nullptr;
    h->tri.n_a = 0;
    h->tri.idx = d_indices;
    h->tri.ids = d_tri_ids;
    h->tri.id_base = tri_id_base;
    h->tri.n_v = n_vertices;
    h->tri.n_t = n_triangles;
    h->tri.n_c0 = LLONG_MAX;   // (part C: grca_update_instances after this call)
    h->n_tri_ab = n_triangles;
    h->n_tri = n_triangles;
    h->have_tri = true;
    return GRCA_OK;
}

grca_status grca_update_triangles_f3(grca_t h, const float *d_xyz, int64_t n_vertices, const uint32_t *d_indices,
                                     int64_t n_triangles, const int32_t *d_tri_ids, int32_t tri_id_base) {
    if (!h) return GRCA_E_INVALID;
    grca_status st = check_tri_args(h, d_xyz, n_vertices, d_indices, n_triangles, d_tri_ids, tri_id_base, true);
    if (st != GRCA_OK) return st;
    h->tri.v = nullptr;
    h->tri.v3 = d_xyz;
    h->tri.va = nullptr;
    h->tri.n_a = 0;
    h->tri.idx = d_indices;
    h->tri.ids = d_tri_ids;
    h->tri.id_base = tri_id_base;
    h->tri.n_v = n_vertices;
    h->tri.n_t = n_triangles;
    h->tri.n_c0 = LLONG_MAX;   // (part C: grca_update_instances after this call)
    h->n_tri_ab = n_triangles;
    h->n_tri = n_triangles;
    h->have_tri = true;
    return GRCA_OK;
}

grca_status grca_update_scene(grca_t h, const float *d_soup, int64_t n_soup_triangles, const float *d_mesh_xyz,
                              int64_t n_mesh_vertices, const uint32_t *d_mesh_indices, int64_t n_mesh_triangles,
                              const int32_t *d_tri_ids, int32_t tri_id_base) {
    if (!h) return GRCA_E_INVALID;
    if (n_soup_triangles < 0 || n_mesh_triangles < 0) return fail(h, GRCA_E_INVALID, "negative triangle count");
    if (n_soup_triangles > 0 && (!d_soup || ((uintptr_t)d_soup & 15)))
        return fail(h, GRCA_E_INVALID, "soup part: 16-byte aligned float4 vertices required");
    if (n_mesh_triangles > 0 && (!d_mesh_indices || n_mesh_vertices < 1))
        return fail(h, GRCA_E_INVALID, "mesh part: indices and vertices required");
    grca_status st = check_tri_args(h, n_mesh_triangles > 0 ? d_mesh_xyz : d_soup,
                                    n_mesh_triangles > 0 ? n_mesh_vertices : 3 * (n_soup_triangles + n_mesh_triangles),
                                    n_mesh_triangles > 0 ? d_mesh_indices : nullptr, n_soup_triangles + n_mesh_triangles,
                                    d_tri_ids, tri_id_base, n_mesh_triangles > 0);
    if (st != GRCA_OK) return st;
    h->tri.va = reinterpret_cast<const float4 *>(d_soup);
    h->tri.n_a = n_soup_triangles;
    h->tri.v = nullptr;
    h->tri.v3 = d_mesh_xyz;
    h->tri.idx = d_mesh_indices;
    h->tri.ids = d_tri_ids;
    h->tri.id_base = tri_id_base;
    h->tri.n_v = n_mesh_vertices;
    h->tri.n_t = n_soup_triangles + n_mesh_triangles;
    h->tri.n_c0 = LLONG_MAX;   // (part C: grca_update_instances after this call)
    h->n_tri_ab = n_soup_triangles + n_mesh_triangles;
    h->n_tri = n_soup_triangles + n_mesh_triangles;
    h->have_tri = true;
    return GRCA_OK;
}

grca_status grca_update_instances(grca_t h, const float *d_local_xyz, int64_t n_local_vertices,
                                  const uint32_t *d_local_faces, int64_t n_faces, const float *d_poses,
                                  int64_t n_instances) {
    if (!h) return GRCA_E_INVALID;
    if (n_faces < 0 || n_instances < 0 || n_local_vertices < 0) return fail(h, GRCA_E_INVALID, "negative count");
    if (n_faces > 0x7fffffffll || n_instances > 0x7fffffffll)
        return fail(h, GRCA_E_INVALID, "n_faces and n_instances must be < 2^31");
    const long long n_c = n_faces * n_instances;
    if (n_c > 0 && (!d_local_xyz || !d_local_faces || !d_poses || n_local_vertices < 1))
        return fail(h, GRCA_E_INVALID, "instances: local vertices, faces and poses required");
    if (((uintptr_t)d_poses & 15) || ((uintptr_t)d_local_xyz & 3) || ((uintptr_t)d_local_faces & 3))
        return fail(h, GRCA_E_INVALID, "poses must be 16-byte aligned (3 float4 rows each); vertices / faces 4-byte");
    if (!h->have_tri) {   // no grca_update_scene / _triangles before: parts A and B are empty
        h->tri = no_part_c();
        h->n_tri_ab = 0;
    }
    if (h->n_tri_ab + n_c > h->ci.max_triangles) return fail(h, GRCA_E_CAPACITY, "triangles exceed max_triangles");
    if (!h->tri.ids && (long long)h->tri.id_base + h->n_tri_ab + n_c > 0x7fffffffll)
        return fail(h, GRCA_E_INVALID, "triangle ids must be in [0, 2^31)");
    h->tri.n_c0 = n_c > 0 ? h->n_tri_ab : LLONG_MAX;
    h->tri.cv = d_local_xyz;
    h->tri.cidx = d_local_faces;
    h->tri.cpose = reinterpret_cast<const float4 *>(d_poses);
    h->tri.c_faces = n_faces;
    h->tri.c_nv = n_local_vertices;
    h->tri.c_ninst = n_instances;
    h->tri.c_inv_faces = n_faces > 0 ? (float)(1.0 / (double)n_faces) : 0.f;
    h->tri.n_t = h->n_tri_ab + n_c;
    h->n_tri = h->n_tri_ab + n_c;
    h->have_tri = true;
    return GRCA_OK;
}

grca_status grca_set_static_triangles(grca_t h, const float *d_vertices, int64_t n_vertices, const uint32_t *d_indices,
                                      int64_t n_triangles, const int32_t *d_tri_ids, int32_t tri_id_base) {
    if (!h) return GRCA_E_INVALID;
    grca_status st = check_tri_args(h, d_vertices, n_vertices, d_indices, n_triangles, d_tri_ids, tri_id_base);
    if (st != GRCA_OK) return st;
    h->st_tri.v = reinterpret_cast<const float4 *>(d_vertices);
    h->st_tri.v3 = nullptr;
    h->st_tri.va = nullptr;
    h->st_tri.n_a = 0;
    h->st_tri.idx = d_indices;
    h->st_tri.ids = d_tri_ids;
    h->st_tri.id_base = tri_id_base;
    h->st_tri.n_v = n_vertices;
    h->st_tri.n_t = n_triangles;
    h->st_tri.n_c0 = LLONG_MAX;
    h->st_n = n_triangles;
    h->st_set = true;
    h->st_dirty = true;
    return GRCA_OK;
}

grca_status grca_clear_static(grca_t h) {
    if (!h) return GRCA_E_INVALID;
    h->st_set = false;
    h->st_dirty = false;
    h->st_n = 0;
    return GRCA_OK;
}

// Launch a gather kernel with the persisting L2 window over the ray table + hits as a per-launch
// attribute (the caller's stream itself is left untouched).
static cudaError_t launch_l2(grca_t h, const void *fn, unsigned grid, unsigned block, size_t smem, KParams &P) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = h->stream;
    cudaLaunchAttribute attr[1];
    if (h->l2win.num_bytes) {
        attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
        attr[0].val.accessPolicyWindow = h->l2win;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
    }
    void *args[] = {(void *)&P};
    return cudaLaunchKernelExC(&cfg, fn, args);
}

// K2 .. K4 for the triangle source in P (events only when prof).
// the kFast instantiations of the fused kernel and K4: no debug / multicast modes in effect
static bool fast_modes(const KParams &P) { return !P.nocull && !P.force64 && !P.allhits && !P.mc_hits; }

static bool rs_merge(grca_t h) {   // (also in GRCA_DEBUG_VIRTUAL_RANKS: the slice this rank would own)
    return h->shard == GRCA_SHARD_TRIANGLES && h->ci.merge == GRCA_MERGE_REDUCE_SCATTER;
}
static long long rs_chunk(grca_t h) { return (h->n_rays + h->nranks - 1) / h->nranks; }

static grca_status launch_core(grca_t h, KParams &P, long long n_tri, bool prof, int slot) {
    const bool split = (h->ci.debug_flags & GRCA_DEBUG_SPLIT_REFINE) != 0;
    if (n_tri > 0) {   // K2
        const long long tiles = (n_tri + K2_THREADS - 1) / K2_THREADS;
        const long long grid = std::min<long long>(tiles, (long long)h->num_sms * h->k2_blocks_per_sm);
        if (h->n_em <= kFixedEm && h->use_lut) {
            void *args[] = {(void *)&P, (void *)&h->lite_pack};
            CK(cudaLaunchKernel(k2_fixed_fn(h->n_em, h->all_level && P.pairs_ok, P.tri.n_c0 != LLONG_MAX), dim3((unsigned)grid),
                                dim3(K2_THREADS), args, h->k2f_smem,
                                h->stream));
        } else {
            k_cull<<<(unsigned)grid, K2_THREADS, h->k2_smem, h->stream>>>(P);
        }
        CK(cudaGetLastError());
    }
    if (prof) CK(cudaEventRecord(h->ev[slot][2], h->stream));
    if (n_tri > 0 && split) {   // K2b (bounds only), rounds interleaved over warps
        const long long grid = (long long)h->num_sms * h->k2b_blocks_per_sm;
        k_refine<<<(unsigned)grid, K2_THREADS, h->k2b_smem, h->stream>>>(P);
        CK(cudaGetLastError());
    }
    if (prof) CK(cudaEventRecord(h->ev[slot][3], h->stream));
    if (n_tri > 0) {   // K4s (split) or fused K2b+K4s
        if (split) {
            const long long grid = (long long)h->num_sms * h->k4s_blocks_per_sm;
            k_small<<<(unsigned)grid, K2_THREADS, h->k4s_smem, h->stream>>>(P);
        } else {
            const long long grid = (long long)h->num_sms * h->kf_blocks_per_sm;
            const void *kf = kf_fn(fast_modes(P), h->all_dev_level, P.tri.n_c0 != LLONG_MAX);
            CK(launch_l2(h, kf, (unsigned)grid, KF_THREADS, h->kf_smem, P));
        }
        CK(cudaGetLastError());
    }
    if (prof) CK(cudaEventRecord(h->ev[slot][4], h->stream));
    if (n_tri > 0) {   // K3
        const long long grid = std::min<long long>((h->cap_large + 255) / 256, (long long)h->num_sms * 4);
        k_bin<<<(unsigned)grid, 256, 0, h->stream>>>(P);
        CK(cudaGetLastError());
    }
    if (prof) CK(cudaEventRecord(h->ev[slot][5], h->stream));
    if (n_tri > 0) {   // K4
        const int grid = h->num_sms * h->k4_blocks_per_sm;
        CK(launch_l2(h, fast_modes(P) ? (const void *)k_isect<true> : (const void *)k_isect<false>, (unsigned)grid,
                     K4_THREADS, sizeof(EmDev) * h->n_em, P));
        CK(cudaGetLastError());
    }
    return GRCA_OK;
}


static cudaError_t nvls_barrier(grca_t h) {
    ++h->nvls_epoch;
    const size_t off = nvls_flag_offset(h->n_rays);
    k_nvls_barrier<<<1, 1, 0, h->stream>>>(reinterpret_cast<unsigned *>(h->nvls_uc + off),
                                           reinterpret_cast<unsigned *>(h->nvls_mc + off),
                                           h->nvls_epoch * (unsigned)h->nvls_n, h->d_ctrl + 7);
    return cudaGetLastError();
}

static grca_status launch_packed(grca_t h) {
    if (h->n_em_global < 1) return fail(h, GRCA_E_STATE, "grca_set_emitters has not been called");
#ifdef GRCA_CHECK
    // the value travels as a kernel argument: captured by value into a CUDA graph (a copy from a host stack
    // variable would be replayed from a stale address)
    k_check_set_n_rays<<<1, 1, 0, h->stream>>>(h->n_rays);
    CK(cudaGetLastError());
#endif
    if (!h->have_tri && !h->st_set) return fail(h, GRCA_E_STATE, "grca_update_triangles has not been called");
    if (h->nvls_mc && h->st_set)
        return fail(h, GRCA_E_STATE, "the fused NVLS merge cannot be combined with cached static triangles");
    DeviceGuard dg(h->device);
    const int slot = (int)(h->n_casts % kRing);
    const bool prof = h->ev_ok;
    KParams P = params(h);
    if (h->st_set && h->st_dirty) {   // hybrid: (re)cast the static triangles into the cached keys
        KParams PS = P;
        PS.tri = h->st_tri;
        PS.n_tri = h->st_n;
        k_init<<<h->num_sms * 4, 256, 0, h->stream>>>(h->d_hits, PS.allhits, h->n_rays, h->d_ctrl, h->d_stats,
                                                      nullptr, nullptr);
        CK(cudaGetLastError());
        grca_status st = launch_core(h, PS, h->st_n, false, slot);
        if (st != GRCA_OK) return st;
        CK(cudaMemcpyAsync(h->d_static_keys, h->d_hits, sizeof(unsigned long long) * h->n_rays,
                           cudaMemcpyDeviceToDevice, h->stream));
        if (PS.allhits)
            CK(cudaMemcpyAsync(h->d_static_allhits, PS.allhits, sizeof(unsigned) * h->n_rays, cudaMemcpyDeviceToDevice,
                               h->stream));
        h->st_dirty = false;
    }
    if (prof) CK(cudaEventRecord(h->ev[slot][0], h->stream));
    {   // K0 (a reduce-scatter merges ceil(n / P) * P keys: the padding starts as MISS too)
        const int grid = h->num_sms * 8;   // full occupancy: stores in flight for HBM bandwidth
        const long long n_init = rs_merge(h) ? rs_chunk(h) * h->nranks : h->n_rays;
        if (h->shard == GRCA_SHARD_EMITTERS && !h->ci.gather_outputs && !h->st_set) {
            // emitter shards write only their own emitters' rays: initialise just those slices
            k_init<<<1, 256, 0, h->stream>>>(P.hits, nullptr, 0, h->d_ctrl, h->d_stats, nullptr, nullptr, 1);
            for (int m : h->own) {
                const long long o = h->offsets[m], c = h->offsets[m + 1] - o;
                const int gr = (int)std::min<long long>((long long)grid, (c / 2 + 255) / 256 + 1);
                k_init<<<gr, 256, 0, h->stream>>>(P.hits + o, P.allhits ? P.allhits + o : nullptr, c, h->d_ctrl,
                                                  h->d_stats, nullptr, nullptr, 0);
            }
        } else {
            k_init<<<grid, 256, 0, h->stream>>>(P.hits, P.allhits, h->st_set ? h->n_rays : n_init, h->d_ctrl, h->d_stats,
                                                h->st_set ? h->d_static_keys : nullptr,
                                                (h->st_set && P.allhits) ? h->d_static_allhits : nullptr);
        }
        CK(cudaGetLastError());
        if (h->st_set && n_init > h->n_rays)
            k_init<<<1, 256, 0, h->stream>>>(P.hits + h->n_rays, nullptr, n_init - h->n_rays, h->d_ctrl, h->d_stats,
                                             nullptr, nullptr);
    }
    // NVLS: no rank may reduce into a peer's copy before the peer has initialised it
    if (h->nvls_mc) CK(nvls_barrier(h));
    if (prof) CK(cudaEventRecord(h->ev[slot][1], h->stream));
    if (!h->have_tri || h->n_em == 0) P.n_tri = 0;
    grca_status st = launch_core(h, P, P.n_tri, prof, slot);
    if (st != GRCA_OK) return st;
    // NVLS: every rank's reductions have landed in every copy before anyone unpacks
    if (h->nvls_mc) CK(nvls_barrier(h));
    if (prof) CK(cudaEventRecord(h->ev[slot][6], h->stream));
    // the collective step, in-stream between K4 and K5
    if (h->comm && h->shard == GRCA_SHARD_TRIANGLES && !h->nvls_mc) {
        if (rs_merge(h))   // rank r receives the min over ranks of keys [r c, r c + c)
            NK(ncclReduceScatter(P.hits, h->d_slice, (size_t)rs_chunk(h), ncclUint64, ncclMin, h->comm, h->stream));
        else               // packed keys are ordered like (t, id): an unsigned min merges shards exactly
            NK(ncclAllReduce(P.hits, P.hits, (size_t)h->n_rays, ncclUint64, ncclMin, h->comm, h->stream));
    }
    if (h->comm && h->shard == GRCA_SHARD_EMITTERS && h->ci.gather_outputs) {
        NK(ncclGroupStart());   // every emitter's keys from its owner (rank m mod P) to every rank
        for (int m = 0; m < h->n_em_global; ++m) {
            const long long o = h->offsets[m], c = h->offsets[m + 1] - o;
            NK(ncclBroadcast(P.hits + o, P.hits + o, (size_t)c, ncclUint64, m % h->nranks, h->comm, h->stream));
        }
        NK(ncclGroupEnd());
    }
    return GRCA_OK;
}

// K5 over global rays [first, first + n): keys[0..n) -> dist[0..n) / tri[0..n)
static grca_status k5(grca_t h, const unsigned long long *keys, float *dist, int32_t *tri, long long n, long long first) {
    if ((dist || tri) && n > 0) {
        const long long blocks = std::min<long long>((n + 255) / 256, (long long)h->num_sms * 8);
        k_unpack<<<(unsigned)std::max<long long>(1, blocks), 256, 0, h->stream>>>(
            keys, dist, tri, n, first, h->noise_sigma, h->noise_seed, (unsigned long long)h->n_casts);
        CK(cudaGetLastError());
    }
    return GRCA_OK;
}

static grca_status launch_unpack(grca_t h, float *d_out_dist, int32_t *d_out_tri,
                                 const unsigned long long *keys = nullptr, long long first = 0, long long n = -1) {
    DeviceGuard dg(h->device);
    const int slot = (int)(h->n_casts % kRing);
    const unsigned long long *own_keys = h->nvls_uc ? h->nvls_uc : h->d_hits;
    grca_status st = GRCA_OK;
    if (keys) {   // grca_unpack_range: caller's keys, slice-local outputs
        st = k5(h, keys, d_out_dist, d_out_tri, n, first);
    } else if (n >= 0) {   // grca_unpack_range on the handle's own keys
        st = k5(h, own_keys + first, d_out_dist, d_out_tri, n, first);
    } else if (rs_merge(h)) {   // this rank's merged slice (virtual ranks: its unmerged keys of the slice)
        const long long c = rs_chunk(h), f = (long long)h->rank * c, m = std::max(0ll, std::min(c, h->n_rays - f));
        st = k5(h, h->comm ? h->d_slice : own_keys + f, d_out_dist ? d_out_dist + f : nullptr,
                d_out_tri ? d_out_tri + f : nullptr, m, f);
    } else if (h->shard == GRCA_SHARD_EMITTERS && !h->ci.gather_outputs) {   // own emitters only
        for (int m : h->own) {
            const long long o = h->offsets[m], c = h->offsets[m + 1] - o;
            st = k5(h, own_keys + o, d_out_dist ? d_out_dist + o : nullptr, d_out_tri ? d_out_tri + o : nullptr, c, o);
            if (st != GRCA_OK) break;
        }
    } else {
        st = k5(h, own_keys, d_out_dist, d_out_tri, h->n_rays, 0);
    }
    if (st != GRCA_OK) return st;
    if (h->ev_ok) CK(cudaEventRecord(h->ev[slot][7], h->stream));
    return GRCA_OK;
}

static grca_status fill_stats(grca_t h, grca_stats *s) {
    DeviceGuard dg(h->device);
    unsigned long long st[32];
    CK(cudaStreamSynchronize(h->stream));
    CK(cudaMemcpy(st, h->d_stats, sizeof(st), cudaMemcpyDeviceToHost));
    memset(s, 0, sizeof(*s));
    s->pairs = (int64_t)st[ST_PAIRS];
    s->range_culled = (int64_t)st[ST_RANGE];
    s->channel_culled = (int64_t)st[ST_CHANNEL];
    s->azimuth_culled = (int64_t)(st[ST_AZIMUTH] + st[ST_DEGEN]);
    s->survivors = (int64_t)st[ST_SURV];
    s->small_pairs = (int64_t)st[ST_SMALL];
    s->large_pairs = (int64_t)st[ST_LARGE];
    s->chunks = (int64_t)st[ST_CHUNKS];
    s->rtic_tested = (int64_t)(st[ST_ITEMS_SMALL] + st[ST_ITEMS_LARGE]);
    s->rtic_brute = (int64_t)(h->n_rays_own * ((h->have_tri ? h->n_tri : 0) + (h->st_set ? h->st_n : 0)));
    s->fp64_fallbacks = (int64_t)st[ST_FP64];
    s->hits_recorded = (int64_t)(st[ST_HITS] + st[ST_HITS_L]);
    s->hits_large = (int64_t)st[ST_HITS_L];
    s->overflow_inline = (int64_t)(st[ST_OVF_LARGE] + st[ST_OVF_CHUNK]);
    s->prefilter_survivors = (int64_t)st[ST_K2SURV];
    s->rtic_small = (int64_t)st[ST_ITEMS_SMALL];
    s->sat_pairs = (int64_t)st[ST_SAT];
    s->bat_pairs = (int64_t)st[ST_BAT];
    s->area_culled = (int64_t)st[ST_AREA];
    s->overflow = s->overflow_inline > 0;
    if (h->ev_ok && h->n_casts > 0) {
        const int slot = (int)((h->n_casts - 1) % kRing);
        float ms;
        for (int k = 0; k < kEv - 1; ++k) {
            if (cudaEventElapsedTime(&ms, h->ev[slot][k], h->ev[slot][k + 1]) == cudaSuccess) s->ms_k[k] = ms;
        }
        if (cudaEventElapsedTime(&ms, h->ev[slot][0], h->ev[slot][kEv - 1]) == cudaSuccess) s->ms_total = ms;
    }
    return GRCA_OK;
}

grca_status grca_cast_packed(grca_t h) {
    if (!h) return GRCA_E_INVALID;
    grca_status s = launch_packed(h);
    if (s != GRCA_OK) return s;
    // keep the profiling ring consistent: the K5 slot is recorded by grca_unpack
    return GRCA_OK;
}

grca_status grca_unpack(grca_t h, float *d_out_dist, int32_t *d_out_tri) {
    if (!h) return GRCA_E_INVALID;
    if (h->n_em_global < 1) return fail(h, GRCA_E_STATE, "grca_set_emitters has not been called");
    grca_status s = launch_unpack(h, d_out_dist, d_out_tri);
    ++h->n_casts;
    return s;
}

grca_status grca_unpack_range(grca_t h, const uint64_t *d_keys, int64_t first_ray, int64_t n, float *d_out_dist,
                              int32_t *d_out_tri) {
    if (!h) return GRCA_E_INVALID;
    if (h->n_em_global < 1) return fail(h, GRCA_E_STATE, "grca_set_emitters has not been called");
    if (first_ray < 0 || n < 0 || first_ray + n > h->n_rays)
        return fail(h, GRCA_E_INVALID, "ray range outside [0, n_rays)");
    grca_status s = launch_unpack(h, d_out_dist, d_out_tri, reinterpret_cast<const unsigned long long *>(d_keys),
                                  first_ray, n);
    ++h->n_casts;
    return s;
}

// GRCA_USE_CUDA_GRAPH: capture K0..K5 (+ the in-stream collective) of this cast into a graph and launch it
// as one unit.  The sequence is re-captured every cast (its parameters -- triangle pointers, counts, the
// outputs, the cast index of the noise model -- may change) and applied to the existing executable with
// cudaGraphExecUpdate, so only a change of topology (e.g. the hybrid static re-cast) re-instantiates.
static grca_status cast_graph(grca_t h, float *d_out_dist, int32_t *d_out_tri) {
    DeviceGuard dg(h->device);
    cudaGraph_t gr = nullptr;
    CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
    grca_status s = launch_packed(h);
    if (s == GRCA_OK) s = launch_unpack(h, d_out_dist, d_out_tri);
    const cudaError_t e = cudaStreamEndCapture(h->stream, &gr);
    if (s != GRCA_OK || e != cudaSuccess) {
        if (gr) cudaGraphDestroy(gr);
        if (s != GRCA_OK) return s;
        CK(e);
    }
    if (h->gexec) {
        cudaGraphExecUpdateResultInfo info;
        if (cudaGraphExecUpdate(h->gexec, gr, &info) != cudaSuccess) {
            cudaGetLastError();
            cudaGraphExecDestroy(h->gexec);
            h->gexec = nullptr;
        } else {
            ++h->graph_updates;
        }
    }
    if (!h->gexec) {
        const cudaError_t ei = cudaGraphInstantiate(&h->gexec, gr, 0);
        if (ei != cudaSuccess) {
            cudaGraphDestroy(gr);
            CK(ei);
        }
        ++h->graph_instantiations;
    }
    cudaGraphDestroy(gr);
    CK(cudaGraphLaunch(h->gexec, h->stream));
    return GRCA_OK;
}

grca_status grca_cast(grca_t h, float *d_out_dist, int32_t *d_out_tri, grca_stats *h_stats) {
    if (!h) return GRCA_E_INVALID;
    bool graph = (h->ci.debug_flags & GRCA_USE_CUDA_GRAPH) && !h->ev_ok && h->stream != nullptr;
    if (graph) {   // inside a caller's own capture the launches are simply recorded into it
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(h->stream, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) graph = false;
    }
    grca_status s;
    if (graph) {
        s = cast_graph(h, d_out_dist, d_out_tri);
    } else {
        s = launch_packed(h);
        if (s == GRCA_OK) s = launch_unpack(h, d_out_dist, d_out_tri);
    }
    ++h->n_casts;
    if (s != GRCA_OK) return s;
#ifdef GRCA_CHECK
    {   // bounds-checked build: every cast is checked before it returns
        unsigned mask = 0;
        CK(cudaStreamSynchronize(h->stream));
        CK(cudaMemcpyFromSymbol(&mask, g_check_err, sizeof(mask)));
        if (mask) {
            const unsigned zero = 0;
            cudaMemcpyToSymbol(g_check_err, &zero, sizeof(zero));
            return fail(h, GRCA_E_CUDA, "bounds check failed, site mask " + std::to_string(mask));
        }
    }
#endif
    if (h_stats) return fill_stats(h, h_stats);
    return GRCA_OK;
}

grca_status grca_hits_packed(grca_t h, uint64_t **d_hits, int64_t *n_rays) {
    if (!h || !d_hits) return GRCA_E_INVALID;
    *d_hits = reinterpret_cast<uint64_t *>(h->nvls_uc ? h->nvls_uc : h->d_hits);
    if (n_rays) *n_rays = h->n_rays;
    return GRCA_OK;
}

grca_status grca_set_nvls(grca_t h, void *d_uc, void *d_mc, int32_t n_ranks) {
    if (!h) return GRCA_E_INVALID;
    if (h->sym_buf) return fail(h, GRCA_E_STATE, "the handle's GRCA_MERGE_NVLS window is bound (owned by the library)");
    if (!d_uc && !d_mc) {   // back to the handle's own buffer and local RED.MIN
        h->nvls_uc = h->nvls_mc = nullptr;
        h->nvls_n = 0;
        return GRCA_OK;
    }
    if (!d_uc || !d_mc || n_ranks < 1) return fail(h, GRCA_E_INVALID, "need both views and n_ranks >= 1");
    if ((((uintptr_t)d_uc) | ((uintptr_t)d_mc)) & 127) return fail(h, GRCA_E_INVALID, "views must be 128-byte aligned");
    if (h->n_em_global < 1) return fail(h, GRCA_E_STATE, "grca_set_emitters first (the buffer holds one key per ray)");
    if (h->ci.debug_flags & GRCA_DEBUG_COUNT_ALL_HITS)
        return fail(h, GRCA_E_STATE, "all-hit counting is per rank: not available with the fused NVLS merge");
    DeviceGuard dg(h->device);
    h->nvls_uc = reinterpret_cast<unsigned long long *>(d_uc);
    h->nvls_mc = reinterpret_cast<unsigned long long *>(d_mc);
    h->nvls_n = n_ranks;
    h->nvls_epoch = 0;
    // this rank's barrier flag starts at 0 (callers barrier on the host after every rank set it)
    CK(cudaMemsetAsync(h->nvls_uc + nvls_flag_offset(h->n_rays), 0, 128, h->stream));
    CK(cudaMemsetAsync(h->d_ctrl + 7, 0, sizeof(unsigned), h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return GRCA_OK;
}

grca_status grca_nvls_status(grca_t h, int64_t *bytes_needed, int32_t *timed_out) {
    if (!h) return GRCA_E_INVALID;
    if (bytes_needed) *bytes_needed = (int64_t)(nvls_flag_offset(h->n_rays) * 8 + 128);
    if (timed_out) {
        DeviceGuard dg(h->device);
        unsigned v = 0;
        CK(cudaStreamSynchronize(h->stream));
        CK(cudaMemcpy(&v, h->d_ctrl + 7, sizeof(unsigned), cudaMemcpyDeviceToHost));
        *timed_out = (int32_t)v;
    }
    return GRCA_OK;
}

grca_status grca_set_distance_noise(grca_t h, float sigma, uint64_t seed) {
    if (!h) return GRCA_E_INVALID;
    if (!(sigma >= 0.f) || !std::isfinite(sigma)) return fail(h, GRCA_E_INVALID, "sigma must be finite and >= 0");
    h->noise_sigma = sigma;
    h->noise_seed = seed;
    return GRCA_OK;
}

grca_status grca_get_stats(grca_t h, grca_stats *h_stats) {
    if (!h || !h_stats) return GRCA_E_INVALID;
    return fill_stats(h, h_stats);
}

grca_status grca_kernel_times(grca_t h, int32_t n_last, float *ms_per_kernel) {
    if (!h || !ms_per_kernel) return GRCA_E_INVALID;
    if (!h->ev_ok) return fail(h, GRCA_E_STATE, "handle created without GRCA_PROFILE_KERNELS");
    if (n_last < 1 || n_last > kRing || n_last > h->n_casts) return fail(h, GRCA_E_INVALID, "n_last out of range");
    DeviceGuard dg(h->device);
    CK(cudaStreamSynchronize(h->stream));
    for (int k = 0; k < 8; ++k) ms_per_kernel[k] = 0.f;
    for (int c = 0; c < n_last; ++c) {
        const int slot = (int)((h->n_casts - 1 - c) % kRing);
        float ms;
        for (int k = 0; k < kEv - 1; ++k) {
            CK(cudaEventElapsedTime(&ms, h->ev[slot][k], h->ev[slot][k + 1]));
            ms_per_kernel[k] += ms;
        }
        CK(cudaEventElapsedTime(&ms, h->ev[slot][0], h->ev[slot][kEv - 1]));
        ms_per_kernel[7] += ms;
    }
    return GRCA_OK;
}

grca_status grca_debug_all_hits(grca_t h, const uint32_t **d_counts) {
    if (!h || !d_counts) return GRCA_E_INVALID;
    if (!h->d_allhits) return fail(h, GRCA_E_STATE, "handle created without GRCA_DEBUG_COUNT_ALL_HITS");
    *d_counts = h->d_allhits;
    return GRCA_OK;
}

grca_status grca_debug_large_list(grca_t h, int32_t *h_out, int64_t cap, int64_t *n_out) {
    if (!h || !n_out) return GRCA_E_INVALID;
    DeviceGuard dg(h->device);
    unsigned n = 0;
    CK(cudaStreamSynchronize(h->stream));
    CK(cudaMemcpy(&n, h->d_ctrl, sizeof(unsigned), cudaMemcpyDeviceToHost));
    const long long m = std::min<long long>(std::min<long long>(n, h->cap_large), cap);
    if (h_out && m > 0) CK(cudaMemcpy(h_out, h->d_large, sizeof(int4) * m, cudaMemcpyDeviceToHost));
    *n_out = n;
    return GRCA_OK;
}

grca_status grca_debug_fast_atan2(const float *h_y, const float *h_x, float *h_out, int64_t n) {
    if ((!h_y || !h_x || !h_out) && n > 0) return GRCA_E_INVALID;
    for (int64_t i = 0; i < n; ++i) h_out[i] = fast_atan2(h_y[i], h_x[i]);
    return GRCA_OK;
}

grca_status grca_get_layout(grca_t h, int64_t *n_rays_total, int64_t *ray_offsets) {
    if (!h) return GRCA_E_INVALID;
    if (h->n_em_global < 1) return fail(h, GRCA_E_STATE, "grca_set_emitters has not been called");
    if (n_rays_total) *n_rays_total = h->n_rays;
    if (ray_offsets)
        for (int n = 0; n <= h->n_em_global; ++n) ray_offsets[n] = h->offsets[n];
    return GRCA_OK;
}

grca_status grca_get_shard(grca_t h, int32_t *shard_mode, int64_t *first_ray, int64_t *n_written) {
    if (!h) return GRCA_E_INVALID;
    if (h->n_em_global < 1) return fail(h, GRCA_E_STATE, "grca_set_emitters has not been called");
    long long first = 0, n = h->n_rays;
    if (rs_merge(h)) {
        const long long c = rs_chunk(h);
        first = (long long)h->rank * c;
        n = std::max(0ll, std::min(c, h->n_rays - first));
    } else if (h->shard == GRCA_SHARD_EMITTERS && !h->ci.gather_outputs) {
        first = -1;
        n = h->n_rays_own;
    }
    if (shard_mode) *shard_mode = h->shard;
    if (first_ray) *first_ray = first;
    if (n_written) *n_written = n;
    return GRCA_OK;
}

grca_status grca_debug_ray_table(grca_t h, float *h_xyz) {
    if (!h || !h_xyz) return GRCA_E_INVALID;
    if (h->n_em_global < 1) return fail(h, GRCA_E_STATE, "grca_set_emitters has not been called");
    DeviceGuard dg(h->device);
    std::vector<float4> tab((size_t)h->n_rays);
    CK(cudaStreamSynchronize(h->stream));
    CK(cudaMemcpy(tab.data(), h->d_raytab, sizeof(float4) * tab.size(), cudaMemcpyDeviceToHost));
    for (size_t g = 0; g < tab.size(); ++g) {
        h_xyz[3 * g] = tab[g].x;
        h_xyz[3 * g + 1] = tab[g].y;
        h_xyz[3 * g + 2] = tab[g].z;
    }
    return GRCA_OK;
}

}  // extern "C"
