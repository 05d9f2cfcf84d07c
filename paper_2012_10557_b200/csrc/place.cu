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
// pieces by a 16-bin counting sort on k -- no comparison sort.  First fit is
// sequential over the pieces but parallel over the GPUs: lane g holds the load
// of GPUs g, g + 32, ...; one ballot finds the lowest GPU with room.
//
// ekya_checkpoint_decide: element-wise (tau - t)(a* - a) > delta A.
#include <algorithm>

#include "launch.h"

namespace ekya {

namespace {

constexpr unsigned kQOne = 65536u;   // one GPU in quanta
constexpr int kPlaceWarps = 8;
constexpr int kMaxGpuSlots = 4;      // GPUs per lane: G <= 128

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

// PL1: remainder r / U (0 < r < U) quantized down to 2^-k, k >= 1, in quanta
__device__ __forceinline__ unsigned quantize_frac(unsigned long long r, int U, int* kout) {
    int k = 1;
    while ((r << k) < (unsigned long long)U) ++k;
    *kout = k;
    return kQOne >> k;
}

__global__ void __launch_bounds__(kPlaceWarps * 32) place_kernel(PlaceParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int J = p.n_jobs, G = p.gpus, U = p.units, P = J + G;
    // per-warp piece list (job, quanta) in first-fit-decreasing order
    uint32_t* wq = reinterpret_cast<uint32_t*>(smem) + (size_t)warp * P;
    uint16_t* wj = reinterpret_cast<uint16_t*>(reinterpret_cast<uint32_t*>(smem) + (size_t)kPlaceWarps * P) +
                   (size_t)warp * P;
    const unsigned lt = (1u << lane) - 1u;
    for (long long b = (long long)blockIdx.x * kPlaceWarps + warp; b < p.n_inst;
         b += (long long)gridDim.x * kPlaceWarps) {
        const uint16_t* a = p.alloc + b * J;
        // Eq. 1 constraint 2: sum a_j <= U, else R-ERR (no pieces)
        long long tot = 0;
        unsigned wsum = 0;   // whole GPUs
        unsigned kcnt = 0;   // lane k (1..16): fractional pieces with exponent k
        for (int j0 = 0; j0 < J; j0 += 32) {
            const int j = j0 + lane;
            int k = 0;
            unsigned w = 0;
            if (j < J) {
                const unsigned long long sh = (unsigned long long)a[j] * (unsigned)G;
                tot += a[j];
                w = (unsigned)(sh / (unsigned)U);
                const unsigned long long r = sh % (unsigned)U;
                if (r) quantize_frac(r, U, &k);
            }
            wsum += __reduce_add_sync(0xffffffffu, w);
#pragma unroll
            for (int kk = 1; kk <= 16; ++kk) {
                const unsigned c = __popc(__ballot_sync(0xffffffffu, k == kk));
                if (lane == kk) kcnt += c;
            }
        }
        for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
        const bool ok = tot <= U;
        if (!ok && lane == 0) flag_data_error(p.st);
        const unsigned np = ok ? wsum + __reduce_add_sync(0xffffffffu, kcnt) : 0u;
        if (ok) {
            // bases: whole pieces at [0, W), exponent-k pieces after all exponents < k
            unsigned kbase = 0;   // lane k: start of bin k
            {
                unsigned inc = kcnt;   // inclusive scan over lanes 1..16
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const unsigned y = __shfl_up_sync(0xffffffffu, inc, o);
                    if (lane >= o) inc += y;
                }
                kbase = wsum + inc - kcnt;
            }
            unsigned wrun = 0;   // whole pieces of the previous chunks
            unsigned krun = 0;   // lane k: pieces of bin k already placed
            for (int j0 = 0; j0 < J; j0 += 32) {
                const int j = j0 + lane;
                int k = 0;
                unsigned w = 0, fq = 0;
                if (j < J) {
                    const unsigned long long sh = (unsigned long long)a[j] * (unsigned)G;
                    w = (unsigned)(sh / (unsigned)U);
                    const unsigned long long r = sh % (unsigned)U;
                    if (r) fq = quantize_frac(r, U, &k);
                }
                // whole pieces: exclusive scan of w over this chunk
                unsigned inc = w;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const unsigned y = __shfl_up_sync(0xffffffffu, inc, o);
                    if (lane >= o) inc += y;
                }
                for (unsigned i = 0; i < w; ++i) {
                    const unsigned pos = wrun + inc - w + i;
                    wq[pos] = kQOne;
                    wj[pos] = (uint16_t)j;
                }
                wrun += __shfl_sync(0xffffffffu, inc, 31);
                // fractional pieces: bin k, rank among this chunk's lanes with the same k
#pragma unroll
                for (int kk = 1; kk <= 16; ++kk) {
                    const unsigned m = __ballot_sync(0xffffffffu, k == kk);
                    const unsigned base = __shfl_sync(0xffffffffu, kbase + krun, kk);
                    if (k == kk) {
                        const unsigned pos = base + __popc(m & lt);
                        wq[pos] = fq;
                        wj[pos] = (uint16_t)j;
                    }
                    if (lane == kk) krun += __popc(m);
                }
            }
        }
        __syncwarp();
        // PL2: first fit, pieces in order; lane g holds GPUs g + 32 s
        unsigned load[kMaxGpuSlots];
#pragma unroll
        for (int sl = 0; sl < kMaxGpuSlots; ++sl) load[sl] = 0;
        int16_t* pg = p.piece_gpu + b * P;
        for (unsigned i = 0; i < np; ++i) {
            const unsigned q = wq[i];
            int gsel = -1;
#pragma unroll
            for (int sl = 0; sl < kMaxGpuSlots; ++sl) {
                if (gsel < 0 && sl * 32 < G) {
                    const unsigned fit = __ballot_sync(0xffffffffu, sl * 32 + lane < G && load[sl] + q <= kQOne);
                    if (fit) {
                        const int l = __ffs(fit) - 1;
                        gsel = sl * 32 + l;
                        if (lane == l) load[sl] += q;
                    }
                }
            }
            if (lane == 0) pg[i] = (int16_t)gsel;
        }
        // outputs (pieces beyond np: job 0, 0 quanta, unplaced)
        for (int i = lane; i < P; i += 32) {
            const bool in = (unsigned)i < np;
            p.piece_job[b * P + i] = in ? wj[i] : 0;
            p.piece_q[b * P + i] = in ? wq[i] : 0u;
            if (!in) pg[i] = -1;
        }
        if (lane == 0) p.n_pieces[b] = (uint16_t)np;
        if (p.gpu_load) {
#pragma unroll
            for (int sl = 0; sl < kMaxGpuSlots; ++sl)
                if (sl * 32 + lane < G) p.gpu_load[b * G + sl * 32 + lane] = load[sl];
        }
        __syncwarp();   // the piece list is rewritten by the next instance
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
    const size_t smem = (size_t)kPlaceWarps * (n_jobs + gpus) * 6 + 16;
    if (smem > h->smem_optin) return EKYA_ERR_SHAPE;
    if (n_inst == 0) return EKYA_OK;
    cudaError_t e = cudaFuncSetAttribute(place_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return EKYA_ERR_CUDA;
    const long long need = ((long long)n_inst + kPlaceWarps - 1) / kPlaceWarps;
    const int grid = (int)std::min<long long>(need, (long long)h->sm_count * 8);
    place_kernel<<<grid, kPlaceWarps * 32, smem, s>>>(p);
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
