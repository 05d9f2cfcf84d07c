// place.cu -- NEXT-4: placement of scheduling decisions onto GPUs
// (readings PL1-PL3 in DESIGN.md) and the checkpoint decision
// (draft P:62-81; reading CK1).
//
// ekya_place: one warp per instance.  Job j with a_j units holds a_j G / U GPUs,
// exactly the rational (a_j G) / U: floor(.) whole GPUs plus the remainder
// quantized down to an inverse power of two 2^-k (integer test U <= r 2^k),
// all in quanta of 2^-16 GPU.  The pieces are written straight into their
// first-fit-decreasing order (descending demand = ascending k, ties by job):
// whole pieces first by an exclusive scan over jobs, then the fractional
// pieces by a 16-bin counting sort on k -- no comparison sort.  For such
// power-of-two pieces first fit is a sequential fill, so each piece's GPU is
// its prefix demand in whole GPUs (closed form below; the oracle runs the
// literal first-fit scan).
//
// ekya_checkpoint_decide: element-wise (tau - t)(a* - a) > delta A.
#include <algorithm>

#include "launch.h"

namespace ekya {

namespace {

constexpr unsigned kQOne = 65536u;   // one GPU in quanta
constexpr int kPlaceWarps = 8;

struct PlaceParams {
    int32_t n_inst, n_jobs, units, gpus;
    const uint16_t* alloc;
    uint16_t* piece_job;
    uint32_t* piece_q;
    int16_t* piece_gpu;
    uint16_t* n_pieces;
    uint32_t* gpu_load;
    DevState* st;
};

// PL1: remainder r / U (0 < r < U <= 65534) quantized down to 2^-k, k >= 1, in quanta: the
// smallest k with r 2^k >= U, from the leading-zero counts (r 2^k < 2^17: no overflow)
__device__ __forceinline__ unsigned quantize_frac(unsigned r, unsigned U, int* kout) {
    int k = __clz(r) - __clz(U);
    if ((r << k) < U) ++k;
    k = max(k, 1);
    *kout = k;
    return kQOne >> k;
}

// lane kk (1..16): the number of lanes whose exponent k equals kk (6-bit fields, five bins per
// word, one warp reduction per word)
__device__ __forceinline__ unsigned bin_count(int k, int lane) {
    const int f = k - 1;
    const unsigned c0 = __reduce_add_sync(0xffffffffu, f >= 0 && f < 5 ? 1u << (6 * f) : 0u);
    const unsigned c1 = __reduce_add_sync(0xffffffffu, f >= 5 && f < 10 ? 1u << (6 * (f - 5)) : 0u);
    const unsigned c2 = __reduce_add_sync(0xffffffffu, f >= 10 && f < 15 ? 1u << (6 * (f - 10)) : 0u);
    const unsigned c3 = __reduce_add_sync(0xffffffffu, f == 15 ? 1u : 0u);
    const int g = lane - 1;
    const unsigned word = g < 5 ? c0 : g < 10 ? c1 : g < 15 ? c2 : c3;
    return lane >= 1 && lane <= 16 ? (word >> (6 * (g % 5))) & 63u : 0u;
}

// PL1 for the chunk's job j: whole GPUs w, exponent k (0: no fractional piece), piece quanta fq
__device__ __forceinline__ void job_share(const uint16_t* a, int j, int J, int G, int U, unsigned& aj, unsigned& w,
                                          int& k, unsigned& fq) {
    aj = 0, w = 0, k = 0, fq = 0;
    if (j < J) {
        aj = a[j];
        const unsigned sh = aj * (unsigned)G;   // < 2^23: 32-bit arithmetic
        w = sh / (unsigned)U;
        const unsigned r = sh - w * (unsigned)U;
        if (r) fq = quantize_frac(r, (unsigned)U, &k);
    }
}

__global__ void __launch_bounds__(kPlaceWarps * 32) place_kernel(PlaceParams p) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int J = p.n_jobs, G = p.gpus, U = p.units, P = J + G;
    const unsigned lt = (1u << lane) - 1u;
    const unsigned qlane = lane >= 1 && lane <= 16 ? kQOne >> lane : 0u;   // lane k: piece size 2^-k
    for (long long b = (long long)blockIdx.x * kPlaceWarps + warp; b < p.n_inst;
         b += (long long)gridDim.x * kPlaceWarps) {
        const uint16_t* a = p.alloc + b * J;
        // Eq. 1 constraint 2: sum a_j <= U, else R-ERR (no pieces)
        long long tot = 0;
        unsigned wsum = 0;   // whole GPUs
        unsigned kcnt = 0;   // lane k (1..16): fractional pieces with exponent k
        unsigned aj, w, fq;  // the first chunk's values, kept for the placement pass
        int k;
        for (int j0 = 0; j0 < J; j0 += 32) {
            unsigned aj_, w_, fq_;
            int k_;
            job_share(a, j0 + lane, J, G, U, aj_, w_, k_, fq_);
            if (j0 == 0) aj = aj_, w = w_, k = k_, fq = fq_;
            tot += __reduce_add_sync(0xffffffffu, aj_);
            wsum += __reduce_add_sync(0xffffffffu, w_);
            kcnt += bin_count(k_, lane);
        }
        const bool ok = tot <= U;
        if (!ok && lane == 0) flag_data_error(p.st);
        const unsigned np = ok ? wsum + __reduce_add_sync(0xffffffffu, kcnt) : 0u;
        uint16_t* pj = p.piece_job + b * P;
        uint32_t* pq = p.piece_q + b * P;
        int16_t* pg = p.piece_gpu + b * P;
        unsigned T = 0;   // total demand in quanta
        if (ok) {
            // bases: whole pieces at [0, W), exponent-k pieces after all exponents < k; and the
            // demand (quanta) ahead of bin k
            unsigned kbase = 0, qbase = 0;   // lane k: start of bin k (pieces, quanta)
            {
                unsigned inc = kcnt, qinc = kcnt * qlane;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const unsigned y = __shfl_up_sync(0xffffffffu, inc, o);
                    const unsigned yq = __shfl_up_sync(0xffffffffu, qinc, o);
                    if (lane >= o) inc += y, qinc += yq;
                }
                kbase = wsum + inc - kcnt;
                T = wsum * kQOne + __shfl_sync(0xffffffffu, qinc, 31);
                qbase = wsum * kQOne + qinc - kcnt * qlane;
            }
            // PL2: the pieces are powers of two in descending order, so the load of every GPU
            // is a multiple of the current piece: a piece fits any GPU not yet full, first fit
            // fills the GPUs one after another and never splits a GPU's free space.  Piece i
            // thus lands on GPU floor(S_i) with S_i the demand (GPUs) ahead of it, unplaced
            // from G on -- the sequential first-fit scan in closed form.
            auto gpu_of = [&](unsigned S) -> int16_t {
                const unsigned g = S / kQOne;
                return g < (unsigned)G ? (int16_t)g : (int16_t)-1;
            };
            unsigned wrun = 0;   // whole pieces of the previous chunks
            unsigned krun = 0;   // lane k: pieces of bin k in the previous chunks
            for (int j0 = 0; j0 < J; j0 += 32) {
                const int j = j0 + lane;
                if (j0 > 0) job_share(a, j, J, G, U, aj, w, k, fq);
                // whole pieces: exclusive scan of w over this chunk
                if (__any_sync(0xffffffffu, w != 0)) {
                    unsigned inc = w;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const unsigned y = __shfl_up_sync(0xffffffffu, inc, o);
                        if (lane >= o) inc += y;
                    }
                    for (unsigned i = 0; i < w; ++i) {
                        const unsigned pos = wrun + inc - w + i;
                        pj[pos] = (uint16_t)j;
                        pq[pos] = kQOne;
                        pg[pos] = gpu_of(pos * kQOne);
                    }
                    wrun += __shfl_sync(0xffffffffu, inc, 31);
                }
                // fractional pieces: bin k, rank among this chunk's lanes with the same k
                const unsigned m = __match_any_sync(0xffffffffu, k);
                const unsigned base = __shfl_sync(0xffffffffu, kbase + krun, k);
                const unsigned qb = __shfl_sync(0xffffffffu, qbase + krun * qlane, k);
                if (k > 0) {
                    const unsigned rk = __popc(m & lt);
                    pj[base + rk] = (uint16_t)j;
                    pq[base + rk] = fq;
                    pg[base + rk] = gpu_of(qb + rk * fq);
                }
                if (j0 + 32 < J) krun += bin_count(k, lane);
            }
        }
        // pieces beyond np: job 0, 0 quanta, unplaced
        for (int i = (int)np + lane; i < P; i += 32) {
            pj[i] = 0;
            pq[i] = 0u;
            pg[i] = -1;
        }
        if (lane == 0) p.n_pieces[b] = (uint16_t)np;
        // loads: GPU g holds min(max(T - g, 0), 1) of the sequential fill
        if (p.gpu_load) {
            for (int g = lane; g < G; g += 32) {
                const unsigned lo = (unsigned)g * kQOne;
                p.gpu_load[b * G + g] = T <= lo ? 0u : min(T - lo, kQOne);
            }
        }
    }
}

struct CkptParams {
    long long n;
    const float *tau, *t, *T, *a, *a_star, *A, *delta;
    uint8_t* out;
    DevState* st;
};

// CK1: (tau - t)(a* - a) > delta A, one rounding per operation; invalid -> 0 + R-ERR
__global__ void checkpoint_kernel(CkptParams p) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < p.n;
         i += (long long)gridDim.x * blockDim.x) {
        const float tau = p.tau[i], t = p.t[i], T = p.T[i], a = p.a[i], as = p.a_star[i], A = p.A[i],
                    dl = p.delta[i];
        const bool ok = T > 0.0f && t >= 0.0f && t <= tau && tau <= T && in01(a) && in01(as) && in01(A) &&
                        dl >= 0.0f;
        if (!ok) flag_data_error(p.st);
        p.out[i] = ok && fmul(fsub(tau, t), fsub(as, a)) > fmul(dl, A);
    }
}

}  // namespace

int launch_place(ekya_handle* h, int32_t n_inst, int32_t n_jobs, int32_t units, int32_t gpus,
                 const uint16_t* alloc, uint16_t* piece_job, uint32_t* piece_q, int16_t* piece_gpu,
                 uint16_t* n_pieces, uint32_t* gpu_load, cudaStream_t s) {
    PlaceParams p{n_inst, n_jobs, units, gpus, alloc, piece_job, piece_q, piece_gpu, n_pieces, gpu_load, h->dstate};
    if (n_inst == 0) return EKYA_OK;
    const long long need = ((long long)n_inst + kPlaceWarps - 1) / kPlaceWarps;
    const int grid = (int)std::min<long long>(need, (long long)h->sm_count * 8);
    place_kernel<<<grid, kPlaceWarps * 32, 0, s>>>(p);
    h->launches++;
    return cuda_status(cudaGetLastError());
}

int launch_checkpoint(ekya_handle* h, long long n, const float* tau, const float* t, const float* T,
                      const float* a, const float* a_star, const float* A, const float* delta, uint8_t* out,
                      cudaStream_t s) {
    if (n == 0) return EKYA_OK;
    CkptParams p{n, tau, t, T, a, a_star, A, delta, out, h->dstate};
    const int grid = (int)std::min<long long>((n + 255) / 256, (long long)h->sm_count * 8);
    checkpoint_kernel<<<grid, 256, 0, s>>>(p);
    h->launches++;
    return cuda_status(cudaGetLastError());
}

}  // namespace ekya
