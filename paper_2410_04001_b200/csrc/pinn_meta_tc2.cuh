// Meta step on tcgen05, v2: neurons on the TMEM lanes.
//
// Same math and outputs as the retired first meta kernel (BF16 tensor-core operands, FP32
// accumulation, FP32 activation / residual / reduction math; BASELINE config 4),
// with the GEMM roles transposed so that every MMA is wide:
//   * a tile is 64 collocation points = 2 halves of 32 points; a half is 128 jet
//     rows r = 4 p + slot (u, u_x, u_t, u_xx);
//   * a chunk is 128 neurons of hidden layer l+1 = the MMA M dimension = the TMEM
//     lanes of the pre-activation outputs;
//   forward   P1   A^T[n, r]   = U_c[n, :] . SY_l[r, :]^T      (M 128, N 128 rows, K rp_l)
//             epi  Z[r, n]     = sigma-jet(A + b)              -> bf16 smem
//             P2   Y^T[r, :]  += Z[r, n] V_c[n, :]             (M 128 rows, N rp_{l+1}, K 128 neurons)
//   reverse   P1r  A^T = U_c SY^T (recompute), DZ^T = V_c ST_{l+1}^T
//             epi  G = sigma-jet VJP(A + b, DZ), Z again, db_l -> bf16 smem
//             P2r  T^T[r, :]  += G[r, n] U_c[n, :]             (M 128 rows, N rp_l, K 128)
//             dU   dU_c[n, :] += G[:, n]^T SY_l                (M 128 neurons, N rp_l, K 128 rows)
//             dV   dV_c[n, :] += Z[:, n]^T ST_{l+1}            (M 128 neurons, N rp_{l+1}, K 128 rows)
//   dU / dV accumulate in TMEM over both halves of the tile and are flushed once
//   per chunk into this CTA's partial (red.global.add of whole 128-byte lines through a
//   per-warp staging tile, one writer per address).
// Per 128 neurons x 32 points: forward 12 MMAs, reverse 32 (v1: 320 N = 16 / M = 64 MMAs).
// Shared memory (bf16, canonical no-swizzle core matrices of 8 rows x 16 B):
//   SY / ST per half  [rank grp][row grp][8 rows][8 ranks]            16 KB each
//   Z / G (one half)  [row grp][neuron grp][8 neurons][8 rows]         32 KB each
//   factor ring       [U_c | b_c (fp32) | V_c], U_c / V_c as [rank grp][neuron grp][8][8]
// TMEM: P1 [0,256) (forward: 2 buffers; reverse: A^T | DZ^T) | Y/T per half [256,384) | dU [384,448) | dV [448,512).
#pragma once

#include "meta_common.cuh"

namespace lrnr_b200 {
namespace mtc2 {

using mtc::act3;
using mtc::commit1;
using mtc::idesc_bf16;
using mtc::mma_lo;
using mtc::mma_x8;
using mtc::pack_bf16;
using mtc::red1;
using mtc::red4;
using mtc::sts128;
using mtc::treduce;
using mtc::wsum;

constexpr int PH = 32;            // points per half
constexpr int ROWS = 4 * PH;      // jet rows per half (MMA N of P1, M of P2)
constexpr int PT = 2 * PH;        // points per tile
constexpr int KC = 128;           // neurons per chunk
constexpr int RP = 64;            // max padded rank
constexpr int NWE = 16;           // epilogue warps: 4 TMEM lane quarters x 4 column / rank groups
constexpr int NGRP = NWE / 4;     // warps per TMEM lane quarter
constexpr int CW = ROWS / NGRP;   // P1 columns (jet rows) per warp per half-step: 32 or 16
constexpr int RW = 64 / NGRP;     // ranks per warp at the transition ends: 16 or 8
// MTC2_SPLIT: the pre-activation MMAs (P1 / P1r) and the rank-side + factor-gradient MMAs
// (P2 / P2r, dU, dV) come from two issuer warps (issue is latency-bound)
#ifndef MTC2_SPLIT
#define MTC2_SPLIT 2
#endif
// (2: a third warp issues dU / dV, so zgfree and tdone take one commit from each of two warps)
constexpr int ISSUER = NWE, PRODUCER = NWE + 1, ISSUER2 = MTC2_SPLIT ? NWE + 2 : NWE;
constexpr int ISSUER3 = MTC2_SPLIT == 2 ? NWE + 3 : ISSUER2;
constexpr int NCOM = MTC2_SPLIT == 2 ? 2 : 1;  // commits per zgfree / tdone phase
constexpr int NT = 32 * (NWE + 2 + (MTC2_SPLIT ? 1 : 0) + (MTC2_SPLIT == 2 ? 1 : 0));
constexpr int NBUF = 2;
constexpr int SYH = ROWS * RP * 2;              // one half tile of SY / ST: 16 KB
constexpr int ZT = ROWS * KC * 2;               // Z or G tile: 32 KB
constexpr int BLKS = 2 * KC * RP * 2 + KC * 4;  // U_c + bias + V_c at rank 64: 33280 B
constexpr int OFF_SY = 0;
constexpr int OFF_ST = OFF_SY + 2 * SYH;
constexpr int OFF_Z = OFF_ST + 2 * SYH;
constexpr int OFF_G = OFF_Z + ZT;
constexpr int OFF_RING = OFF_G + ZT;
constexpr int OFF_ACC = OFF_RING + NBUF * BLKS;
constexpr int MAX_R1 = 512;
constexpr int OFF_S = OFF_ACC + 4 * MAX_R1 * 4;  // the unit's s vector (fp32)
// dU / dV flush staging: per epilogue warp 8 rows x (128 B + 16 B pad), so that the partial-gradient
// reductions leave the SM as whole 128-byte lines (8 lanes x 16 B per neuron row)
constexpr int STG_ROW = 144;
constexpr int STG_WARP = 8 * STG_ROW;
constexpr int OFF_STG = OFF_S + MAX_R1 * 4;
constexpr int SMEM_BYTES = OFF_STG + NWE * STG_WARP;
static_assert(SMEM_BYTES <= 227 * 1024, "shared memory");
constexpr uint32_t TM_P1 = 0, TM_DZ = 128, TM_Y = 256, TM_DU = 384, TM_DV = 448;
constexpr uint32_t HK = (128u >> 4) | (1u << 14);   // SBO 128 B
constexpr uint32_t HM = (2048u >> 4) | (1u << 14);  // SBO 2048 B

struct MetaNet2 {
    int L;
    int M[kMaxL + 1];
    int r[kMaxL];
    int rp[kMaxL];
    int nc[kMaxL];
    int soff[kMaxL + 1];
    int64_t yoff[kMaxL];  // y_l scratch per CTA: [half][row][rp_l] floats
    int64_t ystride;
    int rtotal;
    const unsigned char* blocks;
    const int64_t* blk_off;  // per (transition, chunk) block byte offset: index coff[l] + c
    const int* blk_bytes;
    int coff[kMaxL];
    const float* V0;
    const float* ulast;
    // per-CTA partial: transition l, chunk c at gbase[l] + c * 16384: dU [128][64] then dV [128][64];
    // 16 per-warp copies (stride QS) of db_l (qdb[l] + k), dU_{L-1}, db_{L-1}, dV_0
    int64_t gbase[kMaxL];
    int64_t qbase;
    int QS;
    int qdb[kMaxL];
    int qdUL, qdbL, qdV0;
    int64_t wg_stride;
};

__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
__device__ __forceinline__ void epi_sync() { asm volatile("bar.sync 1, %0;" ::"n"(NWE * 32) : "memory"); }
// RW consecutive TMEM columns of this warp's lanes
__device__ __forceinline__ void tld_rw(uint32_t taddr, float (&v)[RW]) {
    if constexpr (RW == 16) umma::tmem_ld16(taddr, *reinterpret_cast<float(*)[16]>(v));
    else umma::tmem_ld8(taddr, *reinterpret_cast<float(*)[8]>(v));
}
// byte offset of (row, col) in a [col grp][row grp][8 rows][8 cols] bf16 tile with `rows` rows
__device__ __forceinline__ uint32_t tb(int row, int col, int rows) {
    return static_cast<uint32_t>((((col >> 3) * (rows >> 3) + (row >> 3)) * 64 + (row & 7) * 8 + (col & 7)) * 2);
}

template <int ACT>
__global__ void __launch_bounds__(NT, 1)
meta_tc2_kernel(const MetaNet2 net, const RunGeom g, const double* __restrict__ pts, const double* __restrict__ svec,
                const double* __restrict__ mus, const float w, float* __restrict__ scratch, float* __restrict__ part,
                float* __restrict__ wgrad, unsigned long long* __restrict__ bad, const TermSpec* __restrict__ spec,
                const int objective) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ __align__(8) uint64_t full[NBUF], slotfree[NBUF], p1full[2], p1empty[2], zgfull[2], zgfree[2], dready,
        dfree, tdone, sready;
    __shared__ uint32_t tmem_base;
    float* acc4 = reinterpret_cast<float*>(sm + OFF_ACC);
    float* ssm = reinterpret_cast<float*>(sm + OFF_S);

    const int tid = threadIdx.x, lane = tid & 31;
    const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
    const int quarter = warp & 3, grp = warp >> 2;
    const int L = net.L;
    const int R1 = 1 + net.rtotal;
    float* scr = scratch + static_cast<int64_t>(blockIdx.x) * net.ystride;
    float* wg = wgrad + static_cast<int64_t>(blockIdx.x) * net.wg_stride;
    float* wq = wg + net.qbase + warp * net.QS;  // this warp's copy of the small gradients

    for (int k = tid; k < 4 * MAX_R1; k += NT) acc4[k] = 0.f;
    for (int k = tid; k < OFF_RING / 16; k += NT) reinterpret_cast<uint4*>(sm)[k] = make_uint4(0, 0, 0, 0);
    if (warp == 0) umma::tmem_alloc<512>(&tmem_base);
    if (tid == 0) {
        for (int i = 0; i < NBUF; ++i) {
            umma::mbar_init(&full[i], 1);
            umma::mbar_init(&slotfree[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            umma::mbar_init(&p1full[i], 1);
            umma::mbar_init(&p1empty[i], NWE);
            umma::mbar_init(&zgfull[i], NWE);
            umma::mbar_init(&zgfree[i], NCOM);
        }
        umma::mbar_init(&dready, 1);
        umma::mbar_init(&dfree, NWE);
        umma::mbar_init(&tdone, NCOM);
        umma::mbar_init(&sready, NWE);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    umma::fence_async_smem();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    // all 512 columns are allocated, so the TMEM base address is 0 (lane 0, column 0)
    const uint32_t tbase = 0;
    if (tid == 0 && tmem_base != 0) __trap();

    int64_t total_tiles = 0;
    for (int64_t u = blockIdx.x; u < g.n_units; u += gridDim.x) {
        const int seg = static_cast<int>(u % g.units_per_inst);
        const int t_lo = seg * g.tiles_per_unit;
        total_tiles += min(g.tiles_per_inst, t_lo + g.tiles_per_unit) - t_lo;
    }
    auto wait = [](uint64_t* bar, uint32_t parity) {
        umma::mbar_wait(bar, parity);
        umma::fence_after();
    };

#ifdef MTC_TIMING
    const long long t_start = clock64();
#endif
    // =========================== TMA producer ===========================
    if (warp == PRODUCER) {
        if (lane == 0) {
            uint32_t qc = 0;
            for (int64_t t = 0; t < total_tiles; ++t)
                for (int dir = 0; dir < 2; ++dir)
                    for (int li = 0; li + 1 < L; ++li) {
                        const int l = dir == 0 ? li : L - 2 - li;
                        for (int c = 0; c < net.nc[l]; ++c, ++qc) {
                            const int s = static_cast<int>(qc % NBUF);
                            if (qc >= NBUF) umma::mbar_wait(&slotfree[s], ((qc / NBUF) - 1) & 1);
                            const int e = net.coff[l] + c;
                            v2::mbar_expect_tx(&full[s], static_cast<uint32_t>(net.blk_bytes[e]));
                            v2::bulk_g2s(sm + OFF_RING + s * BLKS, net.blocks + net.blk_off[e],
                                         static_cast<uint32_t>(net.blk_bytes[e]), &full[s]);
                        }
                    }
        }
        __syncwarp();
    }
    // =========================== MMA issuer (one thread) ===========================
    else if (warp == ISSUER || warp == ISSUER2 || warp == ISSUER3) {
        // P1 side / P2 side / dU-dV side (one warp may take several)
        const bool do1 = warp == ISSUER, do2 = warp == ISSUER2, do3 = warp == ISSUER3;
        if (lane == 0) {
            const uint32_t sbase = umma::smem_addr(sm) >> 4;
            auto lo = [&](uint32_t off, uint32_t lbo) -> uint32_t { return sbase + (off >> 4) + ((lbo >> 4) << 16); };
            uint32_t s = 0, pe = 0, qc = 0, rc = 0, tcount = 0;
            auto drain = [&](uint32_t end) {  // consume p1empty completions of steps < end, in order
                for (; pe < end; ++pe) MT(18, wait(&p1empty[pe & 1], (pe >> 1) & 1));
            };
            auto ringoff = [&](uint32_t q) { return static_cast<uint32_t>(OFF_RING + static_cast<int>(q % NBUF) * BLKS); };
            for (int64_t t = 0; t < total_tiles; ++t) {
                // ---------------- forward ----------------
                // step i of the transition (chunk i / 2, half i % 2): P1(i), then P2(i - 1)
                for (int l = 0; l + 1 < L; ++l) {
                    if (do1) MT(16, wait(&sready, tcount & 1));
                    const int RL = net.rp[l], RN = net.rp[l + 1], n = net.nc[l];
                    const uint32_t id1 = idesc_bf16(128, ROWS, 0, 0), id2 = idesc_bf16(128, RN, 1, 1);
                    const uint32_t s0 = s, q0 = qc;
                    for (int i = 0; i <= 2 * n; ++i) {
                        if (do1 && i < 2 * n) {
                            const uint32_t si = s0 + i, qi = q0 + (i >> 1);
                            if ((i & 1) == 0) MT(17, wait(&full[qi % NBUF], (qi / NBUF) & 1));
                            drain(si >= 1 ? si - 1 : 0);  // P1 buffer si & 1 was read by step si - 2
                            const uint32_t au = lo(ringoff(qi), 2048), by = lo(OFF_SY + (i & 1) * SYH, 2048);
                            const uint32_t d = tbase + TM_P1 + (si & 1) * 128;
                            const int nk = RL / 16;
#pragma unroll
                            for (int k = 0; k < RP / 16; ++k)
                                if (k < nk) mma_lo<HK, HK>(d, au + ((k * 4096) >> 4), by + ((k * 4096) >> 4), id1, k > 0);
                            commit1(&p1full[si & 1]);
                        }
                        if (do2 && i > 0) {
                            const int j = i - 1;
                            const uint32_t sj = s0 + j, qj = q0 + (j >> 1);
                            MT(19, wait(&zgfull[sj & 1], (sj >> 1) & 1));
                            const uint32_t az = lo(OFF_Z, 128), bv = lo(ringoff(qj) + RL * 256 + 512, 128);
                            mma_x8<HM, HM, 16, 16>(tbase + TM_Y + (j & 1) * 64, az, bv, id2, j >= 2 ? 1u : 0u);
                            commit1(&zgfree[sj & 1]);
                            if (j & 1) commit1(&slotfree[qj % NBUF]);
                        }
                        if (NCOM == 2 && do3 && i > 0) {  // the dU-dV warp's (empty) share of zgfree
                            const uint32_t sj = s0 + i - 1;
                            wait(&zgfull[sj & 1], (sj >> 1) & 1);
                            commit1(&zgfree[sj & 1]);
                        }
                    }
                    s += 2 * n;
                    qc += n;
                    if (do2 || (NCOM == 2 && do3)) commit1(&tdone);
                    if (do1) drain(s);
                    ++tcount;
                }
                // ---------------- reverse ----------------
                for (int l = L - 2; l >= 0; --l) {
                    if (do1) MT(16, wait(&sready, tcount & 1));
                    const int RL = net.rp[l], RN = net.rp[l + 1], n = net.nc[l];
                    const uint32_t id1 = idesc_bf16(128, ROWS, 0, 0), id2 = idesc_bf16(128, RL, 1, 1);
                    const uint32_t idu = idesc_bf16(128, RL, 0, 1), idv = idesc_bf16(128, RN, 0, 1);
                    const uint32_t s0 = s, q0 = qc, r0 = rc;
                    for (int i = 0; i <= 2 * n; ++i) {
                        if (do1 && i < 2 * n) {
                            const uint32_t si = s0 + i, qi = q0 + (i >> 1);
                            if ((i & 1) == 0) MT(17, wait(&full[qi % NBUF], (qi / NBUF) & 1));
                            drain(si);  // the single P1r region was read by step si - 1
                            const uint32_t au = lo(ringoff(qi), 2048), by = lo(OFF_SY + (i & 1) * SYH, 2048);
                            const uint32_t av = lo(ringoff(qi) + RL * 256 + 512, 2048), bt = lo(OFF_ST + (i & 1) * SYH, 2048);
                            const int nkl = RL / 16, nkn = RN / 16;
#pragma unroll
                            for (int k = 0; k < RP / 16; ++k)
                                if (k < nkl)
                                    mma_lo<HK, HK>(tbase + TM_P1, au + ((k * 4096) >> 4), by + ((k * 4096) >> 4), id1, k > 0);
#pragma unroll
                            for (int k = 0; k < RP / 16; ++k)
                                if (k < nkn)
                                    mma_lo<HK, HK>(tbase + TM_DZ, av + ((k * 4096) >> 4), bt + ((k * 4096) >> 4), id1, k > 0);
                            commit1(&p1full[si & 1]);
                        }
                        if ((do2 || do3) && i > 0) {
                            const int j = i - 1, hj = j & 1;
                            const uint32_t sj = s0 + j, qj = q0 + (j >> 1), rj = r0 + (j >> 1);
                            MT(19, wait(&zgfull[sj & 1], (sj >> 1) & 1));
                            if (do2)  // T += G U_c
                                mma_x8<HM, HM, 16, 16>(tbase + TM_Y + hj * 64, lo(OFF_G, 128), lo(ringoff(qj), 128), id2,
                                                       j >= 2 ? 1u : 0u);
                            if (do3) {
                                if (hj == 0 && rj >= 1) MT(20, wait(&dfree, (rj - 1) & 1));  // D free: previous chunk flushed
                                // dU_c += G^T SY_l, dV_c += Z^T ST_{l+1} (accumulated over both halves)
                                mma_x8<HK, HM, 256, 16>(tbase + TM_DU, lo(OFF_G, 2048), lo(OFF_SY + hj * SYH, 128), idu,
                                                        hj ? 1u : 0u);
                                mma_x8<HK, HM, 256, 16>(tbase + TM_DV, lo(OFF_Z, 2048), lo(OFF_ST + hj * SYH, 128), idv,
                                                        hj ? 1u : 0u);
                            }
                            commit1(&zgfree[sj & 1]);
                            if (hj) {
                                if (do3) commit1(&dready);
                                if (do2) commit1(&slotfree[qj % NBUF]);
                            }
                        }
                    }
                    s += 2 * n;
                    qc += n;
                    rc += n;
                    if (do2 || (NCOM == 2 && do3)) commit1(&tdone);
                    if (do1) drain(s);
                    ++tcount;
                }
            }
        }
        __syncwarp();
    }
    // =========================== epilogue warps ===========================
    else {
        uint32_t s = 0, qc = 0, rc = 0, tcount = 0;
        const uint32_t tl = tbase + (static_cast<uint32_t>(quarter * 32) << 16);
        const int kn = quarter * 32 + lane;  // neuron of this thread within a chunk (P1 outputs)
        const int row = quarter * 32 + lane;  // jet row of this thread within a half (Y / T)
        const int pl = row >> 2, slot = row & 3;  // point within the half, jet slot
        auto signal = [&](uint64_t* bar) {
            umma::fence_before();
            __syncwarp();
            if (lane == 0) umma::mbar_arrive(bar);
        };
#ifdef MTC_TIMING
        long long tmark = clock64();
        auto mark = [&](int slot) {
            const long long t = clock64();
            if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&mtc::g_mtc_timing[slot], static_cast<unsigned long long>(t - tmark));
            tmark = t;
        };
#else
        auto mark = [](int) {};
#endif
        auto st16 = [&](int off, float v0, float v1, float v2, float v3, float v4, float v5, float v6, float v7) {
            sts128(sm + off, pack_bf16(v0, v1), pack_bf16(v2, v3), pack_bf16(v4, v5), pack_bf16(v6, v7));
        };
        // SY_l of both halves (bf16) from the y_l scratch: this thread's row, ranks RW grp ..
        auto build_sy = [&](int l) {
            const int RL = net.rp[l];
            if (RW * grp >= RL) return;
            const float* sl = ssm + net.soff[l];
            const int rt = net.r[l];
            float sj[RW];
#pragma unroll
            for (int i = 0; i < RW; ++i) sj[i] = RW * grp + i < rt ? sl[RW * grp + i] : 0.f;
            float4 yv[2][RW / 4];
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int i = 0; i < RW / 4; ++i)
                    yv[h][i] = reinterpret_cast<const float4*>(scr + net.yoff[l] + static_cast<int64_t>(h * ROWS + row) * RL +
                                                               RW * grp)[i];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                float y[RW];
#pragma unroll
                for (int i = 0; i < RW / 4; ++i) {
                    const float4 v = yv[h][i];
                    y[4 * i] = v.x * sj[4 * i];
                    y[4 * i + 1] = v.y * sj[4 * i + 1];
                    y[4 * i + 2] = v.z * sj[4 * i + 2];
                    y[4 * i + 3] = v.w * sj[4 * i + 3];
                }
#pragma unroll
                for (int e = 0; e < RW / 8; ++e)
                    st16(OFF_SY + h * SYH + tb(row, RW * grp + 8 * e, ROWS), y[8 * e], y[8 * e + 1], y[8 * e + 2],
                         y[8 * e + 3], y[8 * e + 4], y[8 * e + 5], y[8 * e + 6], y[8 * e + 7]);
            }
        };
        // flush the dU / dV chunk of reverse chunk rr (transition l, chunk ch) into this CTA's
        // partial.  Warp groups 0 / 1 take dU ranks 0-31 / 32-63 of the warp's 32 neurons, groups
        // 2 / 3 the same of dV: a thread reads one 128-byte line of its neuron's row from TMEM.  The
        // rows go through a per-warp staging tile, 8 at a time, so that 8 consecutive lanes reduce one
        // whole line (4 lines per instruction; one 16-byte request per lane and neuron row before:
        // the flush was bound by the request count, 4096 per chunk, not by bytes).  Every address
        // keeps a single writer thread, so the sum order is fixed.
        static_assert(NGRP == 4, "flush: 4 warp groups (dU lo / hi, dV lo / hi)");
        unsigned char* stg = sm + OFF_STG + warp * STG_WARP;
        auto flush = [&](uint32_t rr, int l, int ch) {
            MT(8, wait(&dready, rr & 1));
            const bool isv = grp >= 2;
            const int c0 = 32 * (grp & 1);
            float a[32];
            const uint32_t src = tl + (isv ? TM_DV : TM_DU) + c0;
            umma::tmem_ld16(src, *reinterpret_cast<float(*)[16]>(a));
            umma::tmem_ld16(src + 16, *reinterpret_cast<float(*)[16]>(a + 16));
            umma::tmem_ld_wait();
            signal(&dfree);
            if (MTC_SKIP & 2) return;
            const int nvalid = isv ? net.rp[l + 1] : net.rp[l];
            if (c0 >= nvalid) return;  // warp-uniform
            const int pc = lane & 7, rsub = lane >> 3;
            float* base = wg + net.gbase[l] + static_cast<int64_t>(ch) * 16384 + (isv ? 8192 : 0) +
                          (quarter * 32) * 64 + c0 + 4 * pc;
            const bool on = c0 + 4 * pc < nvalid;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (rsub == j) {
#pragma unroll
                    for (int q4 = 0; q4 < 8; ++q4)
                        *reinterpret_cast<float4*>(stg + pc * STG_ROW + q4 * 16) =
                            make_float4(a[4 * q4], a[4 * q4 + 1], a[4 * q4 + 2], a[4 * q4 + 3]);
                }
                __syncwarp();
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const int r = 4 * i + rsub;
                    const float4 v = *reinterpret_cast<const float4*>(stg + r * STG_ROW + pc * 16);
                    if (on) red4(base + (8 * j + r) * 64, v.x, v.y, v.z, v.w);
                }
                __syncwarp();
            }
        };

        for (int64_t unit = blockIdx.x; unit < g.n_units; unit += gridDim.x) {
            const int64_t inst = unit / g.units_per_inst;
            const int seg = static_cast<int>(unit % g.units_per_inst);
            const int t_lo = seg * g.tiles_per_unit;
            const int t_hi = min(g.tiles_per_inst, t_lo + g.tiles_per_unit);
            const double* sv = svec + inst * net.rtotal;
            const float mu0 = float(mus[3 * inst]), mu1 = float(mus[3 * inst + 1]), mu2 = float(mus[3 * inst + 2]);
            for (int k = tid; k < net.rtotal; k += NWE * 32) ssm[k] = static_cast<float>(sv[k]);
            epi_sync();

            for (int tile = t_lo; tile < t_hi; ++tile) {
                // ---------------- input layer: y_0 = V_0^T z_0, per jet row ----------------
                if (grp == 0) {
                    const int r0 = net.r[0], RL = net.rp[0];
                    for (int h = 0; h < 2; ++h) {
                        const int64_t pi = static_cast<int64_t>(tile) * PT + h * PH + pl;
                        const bool valid = pi < g.n_per_inst;
                        const int64_t gp = inst * g.n_per_inst + pi;
                        const float x = valid ? float(pts[2 * gp]) : 0.f, t = valid ? float(pts[2 * gp + 1]) : 0.f;
                        float* yp = scr + net.yoff[0] + static_cast<int64_t>(h * ROWS + row) * RL;
                        for (int e = 0; e < RL / 8; ++e) {
                            float y[8], sy[8];
#pragma unroll
                            for (int i = 0; i < 8; ++i) {
                                const int j = 8 * e + i;
                                float v = 0.f, sj = 0.f;
                                if (j < r0) {
                                    const float a = net.V0[j], b = net.V0[r0 + j];
                                    v = slot == 0 ? a * x + b * t : (slot == 1 ? a : (slot == 2 ? b : 0.f));
                                    sj = static_cast<float>(sv[j]);
                                }
                                y[i] = v;
                                sy[i] = sj * v;
                            }
                            reinterpret_cast<float4*>(yp + 8 * e)[0] = make_float4(y[0], y[1], y[2], y[3]);
                            reinterpret_cast<float4*>(yp + 8 * e)[1] = make_float4(y[4], y[5], y[6], y[7]);
                            st16(OFF_SY + h * SYH + tb(row, 8 * e, ROWS), sy[0], sy[1], sy[2], sy[3], sy[4], sy[5],
                                 sy[6], sy[7]);
                        }
                    }
                }
                umma::fence_async_smem();
                signal(&sready);
                mark(9);

                // ---------------- forward transitions ----------------
                for (int l = 0; l + 1 < L; ++l) {
                    const int RL = net.rp[l], n = net.nc[l];
                    for (int ch = 0; ch < n; ++ch, ++qc) {
                        for (int h = 0; h < 2; ++h, ++s) {
                            MT(0, wait(&p1full[s & 1], (s >> 1) & 1));
                            float a[CW];
                            const uint32_t src = tl + TM_P1 + (s & 1) * 128 + CW * grp;
#pragma unroll
                            for (int i = 0; i < CW / 16; ++i)
                                umma::tmem_ld16(src + 16 * i, *reinterpret_cast<float(*)[16]>(a + 16 * i));
                            umma::tmem_ld_wait();
                            signal(&p1empty[s & 1]);
                            wait(&full[qc % NBUF], (qc / NBUF) & 1);
                            const float bias =
                                reinterpret_cast<const float*>(sm + OFF_RING + (qc % NBUF) * BLKS + RL * 256)[kn];
                            uint32_t zp[CW / 2];
#pragma unroll
                            for (int p = 0; p < CW / 4; ++p) {
                                const float av = a[4 * p] + bias, ax = a[4 * p + 1], at = a[4 * p + 2], aw = a[4 * p + 3];
                                float sg, d1, d2, d3;
                                act3<ACT>(av, sg, d1, d2, d3);
                                zp[2 * p] = pack_bf16(sg, d1 * ax);
                                zp[2 * p + 1] = pack_bf16(d1 * at, d2 * ax * ax + d1 * aw);
                            }
                            if (s >= 1) MT(1, wait(&zgfree[(s - 1) & 1], ((s - 1) >> 1) & 1));
#pragma unroll
                            for (int i = 0; i < CW / 8; ++i)
                                sts128(sm + OFF_Z + tb(kn, CW * grp + 8 * i, KC), zp[4 * i], zp[4 * i + 1], zp[4 * i + 2],
                                       zp[4 * i + 3]);
                            umma::fence_async_smem();
                            signal(&zgfull[s & 1]);
                        }
                    }
                    mark(10);
                    MT(2, wait(&tdone, tcount & 1));
                    ++tcount;
                    mark(3);
                    const int RN = net.rp[l + 1];
                    if (l + 2 < L) {
                        // transition end: Y^T -> y_{l+1} scratch, SY_{l+1}
                        // SY_{l+1} first (the next transition's MMAs need it), the y scratch after
                        // sready (Y^T stays in TMEM until this warp's first store of that transition)
                        if (RW * grp < RN) {
                            const float* sl = ssm + net.soff[l + 1];
                            const int rt = net.r[l + 1];
                            for (int h = 0; h < 2; ++h) {
                                float y[RW];
                                tld_rw(tl + TM_Y + h * 64 + RW * grp, y);
                                umma::tmem_ld_wait();
#pragma unroll
                                for (int i = 0; i < RW; ++i) y[i] *= RW * grp + i < rt ? sl[RW * grp + i] : 0.f;
#pragma unroll
                                for (int e = 0; e < RW / 8; ++e)
                                    st16(OFF_SY + h * SYH + tb(row, RW * grp + 8 * e, ROWS), y[8 * e], y[8 * e + 1],
                                         y[8 * e + 2], y[8 * e + 3], y[8 * e + 4], y[8 * e + 5], y[8 * e + 6], y[8 * e + 7]);
                            }
                        }
                        umma::fence_async_smem();
                        signal(&sready);
                        if (RW * grp < RN)
                            for (int h = 0; h < 2; ++h) {
                                float y[RW];
                                tld_rw(tl + TM_Y + h * 64 + RW * grp, y);
                                umma::tmem_ld_wait();
                                float* yp = scr + net.yoff[l + 1] + static_cast<int64_t>(h * ROWS + row) * RN + RW * grp;
#pragma unroll
                                for (int i = 0; i < RW / 4; ++i)
                                    reinterpret_cast<float4*>(yp)[i] = make_float4(y[4 * i], y[4 * i + 1], y[4 * i + 2], y[4 * i + 3]);
                            }
                    } else {
                        // ---------------- output layer (M_L = 1) + residual, per jet row ----------------
                        if (grp == 0) {
                            const int rL = net.r[L - 1];
                            const float* sL = ssm + net.soff[L - 1];
                            for (int h = 0; h < 2; ++h) {
                                float y[16];
                                umma::tmem_ld16(tl + TM_Y + h * 64, y);
                                umma::tmem_ld_wait();
                                const int64_t pi = static_cast<int64_t>(tile) * PT + h * PH + pl;
                                const bool valid = pi < g.n_per_inst;
                                const int64_t gp = inst * g.n_per_inst + pi;
                                float uc = slot == 0 ? net.ulast[rL] : 0.f;
#pragma unroll
                                for (int j = 0; j < 16; ++j)
                                    if (j < rL) uc = fmaf(net.ulast[j] * float(sL[j]), y[j], uc);
                                float u[4];
#pragma unroll
                                for (int c = 0; c < 4; ++c) u[c] = __shfl_sync(0xffffffffu, uc, (lane & ~3) | c);
                                const float N = u[2] + mu0 * u[1] - mu1 * u[3] - mu2 * u[0] * (1.f - u[0]);
                                int kind = objective;
                                float tw = w, sw = w, tgt = 0.f;
                                if (spec != nullptr && valid) {
                                    const TermSpec sp = spec[gp];
                                    kind = sp.kind;
                                    tgt = float(sp.target);
                                    tw = float(sp.w_term);
                                    sw = float(sp.w_seed);
                                }
                                const float dvv = u[0] - tgt;
                                float term = kind == 0 ? tw * (N * N)
                                                       : (kind == 1 ? tw * fabsf(N) : (kind == 2 ? tw * (dvv * dvv) : tw * fabsf(dvv)));
                                term = valid ? term : 0.f;
                                if (slot == 0 && valid && !isfinite(term)) atomicMin(bad, static_cast<unsigned long long>(gp));
                                float gu[4];
                                if (kind <= 1) {
                                    const float gN = valid ? (kind == 0 ? 2.f * N * sw : sgn0(N) * sw) : 0.f;
                                    gu[0] = gN * (-mu2 * (1.f - 2.f * u[0]));
                                    gu[1] = gN * mu0;
                                    gu[2] = gN;
                                    gu[3] = -gN * mu1;
                                } else {
                                    gu[0] = valid ? (kind == 2 ? 2.f * dvv * sw : sgn0(dvv) * sw) : 0.f;
                                    gu[1] = gu[2] = gu[3] = 0.f;
                                }
                                const float gc = gu[slot];
                                const float ts = wsum(slot == 0 ? term : 0.f);
                                const float gb = wsum(slot == 0 ? gu[0] : 0.f);
                                if (lane == 0) {
                                    acc4[quarter * MAX_R1] += ts;
                                    red1(wq + net.qdbL, gb);
                                }
                                float st[16];
#pragma unroll
                                for (int j = 0; j < 16; ++j) {
                                    st[j] = 0.f;
                                    if (j < rL) {
                                        const float uj = net.ulast[j], sj = float(sL[j]);
                                        st[j] = sj * uj * gc;
                                        const float cd = wsum(uj * gc * y[j]);
                                        const float du = wsum(gc * sj * y[j]);
                                        if (lane == 0) {
                                            acc4[quarter * MAX_R1 + 1 + net.soff[L - 1] + j] += cd;
                                            red1(wq + net.qdUL + j, du);
                                        }
                                    }
                                }
#pragma unroll
                                for (int e = 0; e < 2; ++e)
                                    st16(OFF_ST + h * SYH + tb(row, 8 * e, ROWS), st[8 * e], st[8 * e + 1], st[8 * e + 2],
                                         st[8 * e + 3], st[8 * e + 4], st[8 * e + 5], st[8 * e + 6], st[8 * e + 7]);
                            }
                        }
                        build_sy(L - 2);
                        umma::fence_async_smem();
                        signal(&sready);
                    }
                    mark(l + 2 < L ? 11 : 12);
                }

                // ---------------- reverse transitions ----------------
                for (int l = L - 2; l >= 0; --l) {
                    const int RL = net.rp[l], n = net.nc[l];
                    const int Mn = net.M[l + 1];
                    for (int ch = 0; ch < n; ++ch, ++qc) {
                        // the transition end reads y_l (dL/ds) and y_{l-1} (SY rebuild) back from the
                        // scratch: pull this thread's lines into L2 one chunk ahead (earlier, the
                        // partial-gradient reduction stream evicts them again)
                        if (ch == n - 1) {
                            if (RW * grp < RL)
                                for (int h = 0; h < 2; ++h)
                                    prefetch_l2(scr + net.yoff[l] + static_cast<int64_t>(h * ROWS + row) * RL + RW * grp);
                            if (l > 0 && RW * grp < net.rp[l - 1])
                                for (int h = 0; h < 2; ++h)
                                    prefetch_l2(scr + net.yoff[l - 1] +
                                                static_cast<int64_t>(h * ROWS + row) * net.rp[l - 1] + RW * grp);
                        }
                        for (int h = 0; h < 2; ++h, ++s) {
                            MT(4, wait(&p1full[s & 1], (s >> 1) & 1));
                            wait(&full[qc % NBUF], (qc / NBUF) & 1);
                            const float bias =
                                reinterpret_cast<const float*>(sm + OFF_RING + (qc % NBUF) * BLKS + RL * 256)[kn];
                            uint32_t gz[CW];  // packed bf16: G (CW / 2 words) then Z (CW / 2 words)
                            float dbs = 0.f;
#pragma unroll
                            for (int pass = 0; pass < CW / 16; ++pass) {
                                float a[16], dz[16];
                                umma::tmem_ld16(tl + TM_P1 + CW * grp + 16 * pass, a);
                                umma::tmem_ld16(tl + TM_DZ + CW * grp + 16 * pass, dz);
                                umma::tmem_ld_wait();
                                if (pass == CW / 16 - 1) signal(&p1empty[s & 1]);
#pragma unroll
                                for (int p = 0; p < 4; ++p) {
                                    const float av = a[4 * p] + bias, ax = a[4 * p + 1], at = a[4 * p + 2], aw = a[4 * p + 3];
                                    const float g0 = dz[4 * p], g1 = dz[4 * p + 1], g2 = dz[4 * p + 2], g3 = dz[4 * p + 3];
                                    float sg, d1, d2, d3;
                                    act3<ACT>(av, sg, d1, d2, d3);
                                    const float gv = g0 * d1 + g1 * d2 * ax + g2 * d2 * at + g3 * (d3 * ax * ax + d2 * aw);
                                    dbs += gv;
                                    const int o = 2 * (4 * pass + p);
                                    gz[o] = pack_bf16(gv, g1 * d1 + g3 * 2.f * d2 * ax);
                                    gz[o + 1] = pack_bf16(g2 * d1, g3 * d1);
                                    gz[CW / 2 + o] = pack_bf16(sg, d1 * ax);
                                    gz[CW / 2 + o + 1] = pack_bf16(d1 * at, d2 * ax * ax + d1 * aw);
                                }
                            }
                            if (s >= 1) MT(5, wait(&zgfree[(s - 1) & 1], ((s - 1) >> 1) & 1));
#pragma unroll
                            for (int i = 0; i < CW / 8; ++i) {
                                sts128(sm + OFF_G + tb(kn, CW * grp + 8 * i, KC), gz[4 * i], gz[4 * i + 1], gz[4 * i + 2],
                                       gz[4 * i + 3]);
                                sts128(sm + OFF_Z + tb(kn, CW * grp + 8 * i, KC), gz[CW / 2 + 4 * i], gz[CW / 2 + 4 * i + 1],
                                       gz[CW / 2 + 4 * i + 2], gz[CW / 2 + 4 * i + 3]);
                            }
                            umma::fence_async_smem();
                            signal(&zgfull[s & 1]);
                            // db_l: this warp's points of this neuron (one writer per (warp, neuron))
                            const int k = ch * KC + kn;
                            if (k < Mn) red1(wq + net.qdb[l] + k, dbs);
                            if (h == 0 && ch > 0) MT(6, flush(rc++, l, ch - 1));
                        }
                    }
                    mark(13);
                    MT(7, wait(&tdone, tcount & 1));
                    ++tcount;
                    mark(3);
                    // transition end: ST_l = s_l (.) T_l and SY_{l-1} first (the next transition's
                    // MMAs need them), then dL/ds_l (and dV_0) after sready: T^T stays in TMEM
                    // until every warp has stored its first G / Z of the next transition
                    const float* sl = ssm + net.soff[l];
                    const int rt = net.r[l];
                    if (l > 0) {
                        if (RW * grp < RL) {
                            float sj[RW];
#pragma unroll
                            for (int i = 0; i < RW; ++i) sj[i] = RW * grp + i < rt ? sl[RW * grp + i] : 0.f;
                            for (int h = 0; h < 2; ++h) {
                                float tv[RW];
                                tld_rw(tl + TM_Y + h * 64 + RW * grp, tv);
                                umma::tmem_ld_wait();
#pragma unroll
                                for (int i = 0; i < RW; ++i) tv[i] *= sj[i];
#pragma unroll
                                for (int e = 0; e < RW / 8; ++e)
                                    st16(OFF_ST + h * SYH + tb(row, RW * grp + 8 * e, ROWS), tv[8 * e], tv[8 * e + 1],
                                         tv[8 * e + 2], tv[8 * e + 3], tv[8 * e + 4], tv[8 * e + 5], tv[8 * e + 6],
                                         tv[8 * e + 7]);
                            }
                        }
                        build_sy(l - 1);
                        umma::fence_async_smem();
                        signal(&sready);
                    }
                    // the last chunk's dU / dV after the next transition is released: its
                    // reductions would otherwise queue ahead of the y_{l-1} loads above
                    MT(6, flush(rc++, l, n - 1));
                    mark(14);
                    if (RW * grp < RL) {
                        float cd[RW];
#pragma unroll
                        for (int i = 0; i < RW; ++i) cd[i] = 0.f;
                        float dv0[2] = {0.f, 0.f}, dv1[2] = {0.f, 0.f};
                        float4 yv[2][RW / 4];  // both halves' y_l, loaded before use
#pragma unroll
                        for (int h = 0; h < 2; ++h)
#pragma unroll
                            for (int i = 0; i < RW / 4; ++i)
                                yv[h][i] = reinterpret_cast<const float4*>(
                                    scr + net.yoff[l] + static_cast<int64_t>(h * ROWS + row) * RL + RW * grp)[i];
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            float tv[RW];
                            tld_rw(tl + TM_Y + h * 64 + RW * grp, tv);
                            umma::tmem_ld_wait();
#pragma unroll
                            for (int i = 0; i < RW / 4; ++i) {
                                const float4 y4 = yv[h][i];
                                cd[4 * i] = fmaf(tv[4 * i], y4.x, cd[4 * i]);
                                cd[4 * i + 1] = fmaf(tv[4 * i + 1], y4.y, cd[4 * i + 1]);
                                cd[4 * i + 2] = fmaf(tv[4 * i + 2], y4.z, cd[4 * i + 2]);
                                cd[4 * i + 3] = fmaf(tv[4 * i + 3], y4.w, cd[4 * i + 3]);
                            }
                            if (l == 0 && grp == 0) {
                                // dV_0[i][j] = sum over jet rows of z0[row][i] st_0[row][j],
                                // z0 rows: (x, t), (1, 0), (0, 1), (0, 0)
                                const int64_t pi = static_cast<int64_t>(tile) * PT + h * PH + pl;
                                const bool valid = pi < g.n_per_inst;
                                const int64_t gp = inst * g.n_per_inst + pi;
                                const float x = valid ? float(pts[2 * gp]) : 0.f, t = valid ? float(pts[2 * gp + 1]) : 0.f;
                                const float zi0 = slot == 0 ? x : (slot == 1 ? 1.f : 0.f);
                                const float zi1 = slot == 0 ? t : (slot == 2 ? 1.f : 0.f);
#pragma unroll
                                for (int j = 0; j < 2; ++j) {
                                    const float st0 = j < rt ? sl[j] * tv[j] : 0.f;
                                    dv0[j] = fmaf(zi0, st0, dv0[j]);
                                    dv1[j] = fmaf(zi1, st0, dv1[j]);
                                }
                            }
                        }
                        int idx;
                        const float cs = treduce<RW>(cd, lane, idx);
                        const int j = RW * grp + idx;
                        if ((lane & (32 / RW - 1)) == 0 && j < rt) acc4[quarter * MAX_R1 + 1 + net.soff[l] + j] += cs;
                        if (l == 0 && grp == 0) {
                            for (int jj = 0; jj < rt && jj < 2; ++jj) {
                                const float v0 = wsum(dv0[jj]), v1 = wsum(dv1[jj]);
                                if (lane == 0) {
                                    red1(wq + net.qdV0 + jj, v0);
                                    red1(wq + net.qdV0 + rt + jj, v1);
                                }
                            }
                        }
                    }
                    mark(25);
                }
            }
            // unit end: [loss, dL/ds] row = sum of the 4 quarter copies (fixed order)
            epi_sync();
            for (int k = tid; k < R1; k += NWE * 32) {
                part[unit * R1 + k] = ((acc4[k] + acc4[MAX_R1 + k]) + acc4[2 * MAX_R1 + k]) + acc4[3 * MAX_R1 + k];
                acc4[k] = acc4[MAX_R1 + k] = acc4[2 * MAX_R1 + k] = acc4[3 * MAX_R1 + k] = 0.f;
            }
            epi_sync();
        }
    }
#ifdef MTC_TIMING
    if (blockIdx.x == 0 && (threadIdx.x == 0 || threadIdx.x == ISSUER * 32))
        atomicAdd(&mtc::g_mtc_timing[threadIdx.x == 0 ? 15 : 31], static_cast<unsigned long long>(clock64() - t_start));
#endif
    umma::fence_before();
    __syncthreads();
    if (warp == 0) umma::tmem_dealloc<512>(tbase);
}

}  // namespace mtc2
}  // namespace lrnr_b200
