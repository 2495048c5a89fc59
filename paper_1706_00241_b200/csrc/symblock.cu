// K3 over the packed lower triangle: Y = shift X + s_out (.) K (s_in (.) X)
// for an exactly symmetric K (DCG_OP_DENSE_SYM with the packed tiles of
// dcg_pack_sym) and a block X of k <= 32 columns (padded to KP = 16 or 32) -- the refresh's A W
// (recycle.py:90, refresh_basis) reading each stored entry of K once for both
// K_IJ and K_JI: half the bytes of the row-major product (dmma_gemm_kernel).
//
// Work unit: a super-tile of 4 x 4 tiles (tile blocks I in [4A, 4A + 4), J in
// [4B, 4B + 4), J <= I), handed out by an atomic counter (off-diagonal
// super-tiles first, then the diagonal ones).  For each tile (I, J) of a unit
//   row part     RP_I += K_IJ V_J          (warps 0-7, 8 rows each)
//   column part  CP_J += K_IJ' V_I, I != J (warps 8-15)
// on the FP64 tensor pipe (mma.sync m8n8k4), operands from shared memory: the
// tile and the two 64-row V blocks arrive together in one ring stage by three
// bulk copies (TMA engine).  Every unit writes its own RP / CP slots, so the
// result does not depend on which CTA ran which unit; the reduction kernel
// then sums, per output row, the RP slots of its super-row and the CP slots
// of its super-column in a fixed order (deterministic, no atomics on data).
//
// Operand layouts (bank-conflict free fragment loads):
//   K tile   the packed, XOR-swizzled tile (symgemv.cuh); the 8 rows of an m8
//            fragment are rows {b + a, b + a + 8 : a < 4}, so lanes 2a, 2a + 1
//            read rows whose swizzle keys differ in bit 2;
//   V block  64 rows as 32 row pairs of 2 x KP doubles (pair-interleaved:
//            (r, c) at (r / 2) VP + 2 c + r mod 2) padded to VP = 2 KP + 4, so the
//            two k indices 2p, 2p + 1 a thread feeds to two consecutive MMAs
//            are one 16-byte load (the k order inside each 8-chunk is permuted
//            identically for A and B, which leaves every dot product intact).
#include "common.cuh"
#include "symgemv.cuh"

#define SB_R 4                                   // tile blocks per super-tile side
#ifndef SB_MT
#define SB_MT 1                                  // m8 fragments per consumer warp (1 or 2; 1 measured 1-2% faster)
#endif
#define SB_NCW (16 / SB_MT)                      // consumer warps: half row part, half column part
#define SB_NT (32 * (SB_NCW + 1))                // + one producer warp
#ifndef SB_UNROLL
#define SB_UNROLL 8                              // k-pair steps unrolled in the MMA loops (all 8: measured fastest)
#endif

namespace {

constexpr int kSbUnroll = SB_UNROLL;

// Geometry for KP padded columns of X (16 or 32).
template <int KP>
struct SbCfg {
    static constexpr int VP = 2 * KP + 4;                          // doubles per row pair of a V block
    static constexpr int VBLK = 32 * VP;                           // doubles per 64-row V block
    static constexpr int STAGE = DCG_SYM_TILE_DOUBLES + 2 * VBLK;  // tile + V_J + V_I
    static constexpr int STAGES = KP <= 16 ? 4 : 3;                // ring depth within 227 KB
    static constexpr int SLOT = DCG_TB * KP;                       // doubles per RP / CP slot
    static constexpr int NT8 = KP / 8;                             // n8 fragments per warp
};

struct SbMeta {
    int unit;
    int li, lj;        // block offsets of the tile inside its super-tile
    int flags;         // 1 first tile of the unit, 2 last tile of the unit, 4 last tile of the row, 8 I == J, 16 first of the row
};

__host__ __device__ __forceinline__ long long sb_nblocks(long long n) { return (n + DCG_TB - 1) / DCG_TB; }
__host__ __device__ __forceinline__ long long sb_nsuper(long long n) { return (sb_nblocks(n) + SB_R - 1) / SB_R; }
__host__ __device__ __forceinline__ long long sb_units(long long n) {
    const long long ns = sb_nsuper(n);
    return ns * (ns + 1) / 2;
}
// unit -> (A, B): off-diagonal units (A > B) in row-major order first, then
// the diagonal ones
__device__ __forceinline__ void sb_decode(long long u, long long ns, long long& A, long long& B) {
    const long long noff = ns * (ns - 1) / 2;
    if (u >= noff) {
        A = B = u - noff;
        return;
    }
    long long a = (long long)((1.0 + sqrt(1.0 + 8.0 * (double)u)) * 0.5);
    while (a * (a - 1) / 2 > u) --a;
    while ((a + 1) * a / 2 <= u) ++a;
    A = a;
    B = u - a * (a - 1) / 2;
}
__host__ __device__ __forceinline__ long long sb_unit_of(long long A, long long B, long long ns) {
    return A == B ? ns * (ns - 1) / 2 + A : A * (A - 1) / 2 + B;
}

__device__ __forceinline__ void sb_dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void sb_bulk(double* sdst, const double* gsrc, unsigned bytes, unsigned long long* bar,
                                        unsigned long long pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
            sym_saddr(sdst)),
        "l"(gsrc), "r"(bytes), "r"(sym_saddr(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ unsigned long long sb_policy_normal() {
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// m8 fragment row g of the 16-row warp block, fragment mt: rows {4 mt + a, 4 mt + a + 8}
__device__ __forceinline__ int sb_row(int mt, int g) { return 4 * mt + (g >> 1) + 8 * (g & 1); }

// V (blocks of 64 rows, pair-interleaved, zero beyond n and k) = s (.) X
template <int KP>
__global__ void sb_pack_v_kernel(const double* __restrict__ X, int k, const double* __restrict__ s, long long n,
                                 long long nblk, double* __restrict__ V) {
    using C = SbCfg<KP>;
    const long long total = nblk * C::VBLK;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long b = e / C::VBLK;
        const int w = (int)(e - b * C::VBLK);
        const int p = w / C::VP, q = w - p * C::VP;
        double v = 0.0;
        if (q < 2 * KP) {
            const int c = q >> 1;
            const long long i = b * DCG_TB + 2 * p + (q & 1);
            if (i < n && c < k) {
                v = X[i * k + c];
                if (s) v = mul_rn(s[i], v);
            }
        }
        V[e] = v;
    }
}

template <int KP>
__global__ void __launch_bounds__(SB_NT, 1)
    sb_apply_kernel(const double* __restrict__ Kp, long long n, const double* __restrict__ V, double* __restrict__ RP,
                    double* __restrict__ CP, unsigned long long* counter) {
    using C = SbCfg<KP>;
    extern __shared__ __align__(128) double sm[];
    double* ring = sm;
    unsigned long long* full = reinterpret_cast<unsigned long long*>(ring + C::STAGES * C::STAGE);
    unsigned long long* empty = full + C::STAGES;
    SbMeta* meta = reinterpret_cast<SbMeta*>(empty + C::STAGES);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const long long NB = sb_nblocks(n), NS = sb_nsuper(n), NU = sb_units(n);
    if (tid == 0) {
        for (int st = 0; st < C::STAGES; ++st) {
            sym_mbar_init(full + st, 1);
            sym_mbar_init(empty + st, SB_NCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cta_sync();

    // ---- producer (lane 0 of the last warp): walks the units it draws from the
    // counter and streams their tiles (+ V blocks) through the ring, up to
    // C::STAGES stages ahead of the consumers; a unit of -1 marks the end.
    if (warp == SB_NCW) {
        if (lane == 0) {
            const unsigned long long pol_k = sym_policy_evict_first(), pol_v = sb_policy_normal();
            unsigned int q = 0;
            for (;;) {
                const long long u = (long long)atomicAdd(counter, 1ull);
                const bool done = u >= NU;
                long long A = 0, B = 0;
                if (!done) sb_decode(u, NS, A, B);
                const long long I0 = SB_R * A, J0 = SB_R * B;
                const long long I1 = min(I0 + SB_R, NB), J1 = min(J0 + SB_R, NB);
                // tiles of the unit (row-major, J <= I); a finished producer pushes one end marker
                long long I = I0, J = J0;
                bool first = true;
                for (;;) {
                    if (!done && I >= I1) break;
                    const int stg = q % C::STAGES;
                    if (q >= C::STAGES) sym_mbar_wait(empty + stg, ((q / C::STAGES) - 1) & 1);
                    SbMeta m;
                    if (done) {
                        m.unit = -1;
                        m.li = m.lj = m.flags = 0;
                        meta[stg] = m;
                        sym_mbar_arrive(full + stg);
                        ++q;
                        break;
                    }
                    const long long jend = min(J1, I + 1);   // J < jend for this row
                    m.unit = (int)u;
                    m.li = (int)(I - I0);
                    m.lj = (int)(J - J0);
                    m.flags = (first ? 1 : 0) | (J == J0 ? 16 : 0) | (J + 1 == jend ? 4 : 0) | (I == J ? 8 : 0);
                    if (J + 1 == jend && I + 1 == I1) m.flags |= 2;
                    meta[stg] = m;
                    double* dst = ring + stg * C::STAGE;
                    sym_mbar_expect_tx(full + stg, (unsigned)(C::STAGE * sizeof(double)));
                    sb_bulk(dst, Kp + (sym_tile_row_base(I) + J) * DCG_SYM_TILE_DOUBLES,
                            DCG_SYM_TILE_DOUBLES * sizeof(double), full + stg, pol_k);
                    sb_bulk(dst + DCG_SYM_TILE_DOUBLES, V + J * C::VBLK, C::VBLK * sizeof(double), full + stg, pol_v);
                    sb_bulk(dst + DCG_SYM_TILE_DOUBLES + C::VBLK, V + I * C::VBLK, C::VBLK * sizeof(double), full + stg,
                            pol_v);
                    ++q;
                    first = false;
                    if (++J >= jend) {
                        ++I;
                        J = J0;
                    }
                }
                if (done) break;
            }
            // this CTA draws no more: the last producer out zeroes the counter
            dcg_sync_exit(reinterpret_cast<unsigned int*>(counter), gridDim.x);
        }
        return;
    }

    // ---- consumers: warps 0-3 the row part, 4-7 the column part ----------------
    const bool rowpart = warp < SB_NCW / 2;
    const int wl = warp % (SB_NCW / 2);
    double acc[SB_R][SB_MT][C::NT8][2];    // [block][mt][nt][2]  (row part uses block 0 only)
#pragma unroll
    for (int b = 0; b < SB_R; ++b)
#pragma unroll
        for (int mt = 0; mt < SB_MT; ++mt)
#pragma unroll
            for (int nt = 0; nt < C::NT8; ++nt) acc[b][mt][nt][0] = acc[b][mt][nt][1] = 0.0;
    // per-lane fragment offsets
    // output rows of the warp's m8 fragments (16-row blocks split over 2 / SB_MT warps)
    int rowm[SB_MT];
#pragma unroll
    for (int mt = 0; mt < SB_MT; ++mt) rowm[mt] = 16 * (wl / (2 / SB_MT)) + sb_row((wl % (2 / SB_MT)) * SB_MT + mt, g);

    unsigned int q = 0;
    for (;;) {
        const int stg = q % C::STAGES;
        sym_mbar_wait(full + stg, (q / C::STAGES) & 1);
        const SbMeta m = meta[stg];
        if (m.unit < 0) break;
        const double* tile = ring + stg * C::STAGE;
        const double* vj = tile + DCG_SYM_TILE_DOUBLES;
        const double* vi = vj + C::VBLK;
        if (rowpart) {
            if (m.flags & 16) {
#pragma unroll
                for (int mt = 0; mt < SB_MT; ++mt)
#pragma unroll
                    for (int nt = 0; nt < C::NT8; ++nt) acc[0][mt][nt][0] = acc[0][mt][nt][1] = 0.0;
            }
#pragma unroll kSbUnroll
            for (int s2 = 0; s2 < DCG_TB / 8; ++s2) {
                double2 a[SB_MT], b[C::NT8];
#pragma unroll
                for (int mt = 0; mt < SB_MT; ++mt) {
                    const int r = rowm[mt];
                    a[mt] = *reinterpret_cast<const double2*>(tile + r * DCG_TB + 2 * ((4 * s2 + t) ^ ((r >> 1) & 31)));
                }
#pragma unroll
                for (int nt = 0; nt < C::NT8; ++nt)
                    b[nt] = *reinterpret_cast<const double2*>(vj + (4 * s2 + t) * C::VP + 2 * (8 * nt + g));
#pragma unroll
                for (int mt = 0; mt < SB_MT; ++mt)
#pragma unroll
                    for (int nt = 0; nt < C::NT8; ++nt) {
                        sb_dmma(acc[0][mt][nt][0], acc[0][mt][nt][1], a[mt].x, b[nt].x);
                        sb_dmma(acc[0][mt][nt][0], acc[0][mt][nt][1], a[mt].y, b[nt].y);
                    }
            }
        } else if (!(m.flags & 8)) {
            if (m.flags & 1) {
#pragma unroll
                for (int b = 0; b < SB_R; ++b)
#pragma unroll
                    for (int mt = 0; mt < SB_MT; ++mt)
#pragma unroll
                        for (int nt = 0; nt < C::NT8; ++nt) acc[b][mt][nt][0] = acc[b][mt][nt][1] = 0.0;
            }
            // A = K_IJ' (rows: the tile's columns), B = V_I
#pragma unroll
            for (int lj = 0; lj < SB_R; ++lj) {
                if (lj != m.lj) continue;
#pragma unroll kSbUnroll
                for (int s2 = 0; s2 < DCG_TB / 8; ++s2) {
                    const int i0 = 8 * s2 + 2 * t;   // tile rows i0, i0 + 1 (same swizzle key)
                    double a0[SB_MT], a1[SB_MT];
                    double2 b[C::NT8];
#pragma unroll
                    for (int mt = 0; mt < SB_MT; ++mt) {
                        const int c = rowm[mt];
                        const int off = i0 * DCG_TB + 2 * ((c >> 1) ^ ((i0 >> 1) & 31)) + (c & 1);
                        a0[mt] = tile[off];
                        a1[mt] = tile[off + DCG_TB];
                    }
#pragma unroll
                    for (int nt = 0; nt < C::NT8; ++nt)
                        b[nt] = *reinterpret_cast<const double2*>(vi + (4 * s2 + t) * C::VP + 2 * (8 * nt + g));
#pragma unroll
                    for (int mt = 0; mt < SB_MT; ++mt)
#pragma unroll
                        for (int nt = 0; nt < C::NT8; ++nt) {
                            sb_dmma(acc[lj][mt][nt][0], acc[lj][mt][nt][1], a0[mt], b[nt].x);
                            sb_dmma(acc[lj][mt][nt][0], acc[lj][mt][nt][1], a1[mt], b[nt].y);
                        }
                }
            }
        } else if (m.flags & 1) {
            // a diagonal tile opening a unit still opens the column accumulators
#pragma unroll
            for (int b = 0; b < SB_R; ++b)
#pragma unroll
                for (int mt = 0; mt < SB_MT; ++mt)
#pragma unroll
                    for (int nt = 0; nt < C::NT8; ++nt) acc[b][mt][nt][0] = acc[b][mt][nt][1] = 0.0;
        }
        __syncwarp();
        if (lane == 0) sym_mbar_arrive(empty + stg);
        ++q;
        // flushes: D fragment (g, t) holds rows rowm[mt], columns 8 nt + 2t, 2t + 1
        if (rowpart && (m.flags & 4)) {
            double* out = RP + ((long long)m.unit * SB_R + m.li) * C::SLOT;
#pragma unroll
            for (int mt = 0; mt < SB_MT; ++mt)
#pragma unroll
                for (int nt = 0; nt < C::NT8; ++nt)
                    *reinterpret_cast<double2*>(out + rowm[mt] * KP + 8 * nt + 2 * t) =
                        make_double2(acc[0][mt][nt][0], acc[0][mt][nt][1]);
        }
        if (!rowpart && (m.flags & 2)) {
            long long A, B;
            sb_decode(m.unit, NS, A, B);
#pragma unroll
            for (int lj = 0; lj < SB_R; ++lj) {
                if (SB_R * B + lj >= NB) continue;
                double* out = CP + ((long long)m.unit * SB_R + lj) * C::SLOT;
#pragma unroll
                for (int mt = 0; mt < SB_MT; ++mt)
#pragma unroll
                    for (int nt = 0; nt < C::NT8; ++nt)
                        *reinterpret_cast<double2*>(out + rowm[mt] * KP + 8 * nt + 2 * t) =
                            make_double2(acc[lj][mt][nt][0], acc[lj][mt][nt][1]);
            }
        }
    }
}

// Y[i][c] = shift X[i][c] + s_out[i] sum(partials of row i), c < k.  Row i of
// block I = 4 A + li: the RP slots of units (A, 0..A) then the CP slots of
// units (A..NS-1, A), in that order.
template <int KP>
__global__ void sb_reduce_kernel(const double* __restrict__ RP, const double* __restrict__ CP, long long n, int k,
                                 const double* __restrict__ X_rows, const double* __restrict__ s_out, double shift,
                                 double* __restrict__ Y) {
    using C = SbCfg<KP>;
    const long long NS = sb_nsuper(n);
    const long long total = n * KP;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long i = e / KP;
        const int c = (int)(e - i * KP);
        if (c >= k) continue;
        const long long I = i / DCG_TB;
        const int r = (int)(i - I * DCG_TB);
        const long long A = I / SB_R;
        const int li = (int)(I - A * SB_R);
        const long long off = (long long)li * C::SLOT + r * KP + c;
        // the partials in a fixed order: RP of units (A, 0..A), then CP of units
        // (A..NS-1, A); loaded 8 at a time ahead of their (ordered) adds
        const long long nterm = (A + 1) + (NS - A);
        double acc = 0.0;
        for (long long q0 = 0; q0 < nterm; q0 += 8) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const long long q = q0 + u;
                v[u] = 0.0;
                if (q <= A) v[u] = RP[sb_unit_of(A, q, NS) * SB_R * C::SLOT + off];
                else if (q < nterm) v[u] = CP[sb_unit_of(A + (q - A - 1), A, NS) * SB_R * C::SLOT + off];
            }
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (q0 + u < nterm) acc += v[u];
        }
        double val = s_out ? mul_rn(s_out[i], acc) : acc;
        if (shift != 0.0) val = add_rn(mul_rn(shift, X_rows[i * k + c]), val);
        Y[i * k + c] = val;
    }
}

}  // namespace

template <int KP>
static size_t sb_scratch(long long n) {
    using C = SbCfg<KP>;
    return (size_t)(sb_nblocks(n) * C::VBLK) + 32 + 2 * (size_t)sb_units(n) * SB_R * C::SLOT + 64;
}
static int sb_kp(int k) { return k <= 16 ? 16 : 32; }

size_t dcg_sym_block_scratch_doubles(long long n, int k) { return sb_kp(k) == 16 ? sb_scratch<16>(n) : sb_scratch<32>(n); }
bool dcg_sym_block_ok(int k) { return k >= 1 && k <= 32; }

template <int KP>
static int sb_apply(dcg_context* ctx, cudaStream_t st, const double* Kp, long long n, const double* X, int k,
                    const double* s_in, const double* s_out, double shift, double* Y, double* scratch) {
    using C = SbCfg<KP>;
    const long long NB = sb_nblocks(n), NU = sb_units(n);
    double* V = scratch;
    double* RP = V + ((NB * C::VBLK + 31) & ~31LL);
    double* CP = RP + NU * SB_R * C::SLOT;
    // the unit counter: the context's persistent line (words 0-1), handed back
    // at zero by the kernel -- no memset
    unsigned long long* counter = reinterpret_cast<unsigned long long*>(dcg_sync_line(ctx, DCG_SW_SBLOCK));
    sb_pack_v_kernel<KP><<<ctx->sm_count * 4, 256, 0, st>>>(X, k, s_in, n, NB, V);
    DCG_LAUNCHED();
    const size_t smem = sizeof(double) * C::STAGES * C::STAGE + 2 * C::STAGES * sizeof(unsigned long long) +
                        C::STAGES * sizeof(SbMeta);
    DCG_SMEM_ATTR(sb_apply_kernel<KP>, smem);
    sb_apply_kernel<KP><<<ctx->sm_count, SB_NT, smem, st>>>(Kp, n, V, RP, CP, counter);
    DCG_LAUNCHED();
    sb_reduce_kernel<KP><<<ctx->sm_count * 4, 256, 0, st>>>(RP, CP, n, k, X, s_out, shift, Y);
    DCG_LAUNCHED();
    return DCG_OK;
}

// Y (n x k) = shift X + s_out (.) K (s_in (.) X) over the packed tiles Kp (k <= 32).
int dcg_sym_block_apply(dcg_context* ctx, cudaStream_t st, const double* Kp, long long n, const double* X, int k,
                        const double* s_in, const double* s_out, double shift, double* Y, double* scratch) {
    if (n <= 0 || k <= 0) return DCG_OK;
    if (!dcg_sym_block_ok(k) || !aligned16(Kp)) return DCG_E_CONFIG;
    return sb_kp(k) == 16 ? sb_apply<16>(ctx, st, Kp, n, X, k, s_in, s_out, shift, Y, scratch)
                          : sb_apply<32>(ctx, st, Kp, n, X, k, s_in, s_out, shift, Y, scratch);
}
