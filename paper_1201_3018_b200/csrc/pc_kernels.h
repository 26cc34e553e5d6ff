// pc_kernels.h -- launch interface between the C ABI (pc_api.cu) and the kernels.
#pragma once
#include <cuda_runtime.h>

#include <mutex>

#include "pc_device.cuh"

namespace pc {

constexpr int kMaxDevices = 64;
constexpr int kT = 8;              // outputs per thread of the per-block kernel's core
constexpr int kMaxThreads = 1024;  // per-block kernel: threads per CTA; caps regs at 64
constexpr int kTPChoices[3] = {16, 14, 12};   // tiled-kernel tiles instantiated; the plan picks
constexpr int kSmemHeader = 512;
constexpr int kTiledHeader = 2048;      // tiled kernel: mbarriers, stage metadata, counters
constexpr int kTiledMaxStages = 24;     // tiled kernel: stage ring slots (>= 16 / npart jobs in flight)
#ifndef PC_PROD_WARPS
#define PC_PROD_WARPS 4
#endif
constexpr int kTiledProdWarps = PC_PROD_WARPS;   // tiled kernel: producer warps (peak, companding, packing)
#ifndef PC_FILL_JOBS
#define PC_FILL_JOBS 4
#endif
constexpr int kTiledFillJobs = PC_FILL_JOBS;   // tiled kernel: fill groups (warps split into this many job packers)
#ifndef PC_FILL_MAX
#define PC_FILL_MAX 4
#endif
// tiled kernel: jobs packed by all warps before the consumers start (up to the ring's stages and
// the CTA's share of the launch): a launch of <= NS jobs per SM never runs producers next to
// DMMA warps (whose issue slowed producers 3-6x, profiles/r01_dmma_interference.log)
constexpr int kTiledFillMax = PC_FILL_MAX;
#ifndef PC_CONS_WARPS
#define PC_CONS_WARPS 12
#endif
constexpr int kTiledConsWarps = PC_CONS_WARPS;   // tiled kernel: consumer warps (core + unpack); 12 = 3 per SMSP,
                                                 // 16 warps per CTA so the core gets 128 registers
constexpr int kTiledThreads = 32 * (kTiledProdWarps + kTiledConsWarps);
#ifndef PC_CONS_WARPS_MMA
#define PC_CONS_WARPS_MMA 12
#endif
// consumer warps of the DMMA-core kernel (16 = four per SMSP at 96 registers spills and
// leaves fewer ring stages: measured slower than 12)
__host__ __device__ constexpr int tiled_cons_warps(int mma) { return mma ? PC_CONS_WARPS_MMA : kTiledConsWarps; }
__host__ __device__ constexpr int tiled_threads(int mma) { return 32 * (kTiledProdWarps + tiled_cons_warps(mma)); }
constexpr int kCtrDone = 256;     // sm_ctr[kCtrDone] counts retired CTAs; queues are sm_ctr[0, nsm)   // mbarrier + reduction scratch, keeps the rest 128B-aligned

// Host: a kernel's launch attributes per device, raised once under a lock (launches from
// several host threads / devices).  ensure() raises the maximum dynamic shared memory to at least
// `need`, checks that one CTA of `threads` fits, and returns the device's SM count.
struct LaunchAttrCache {
  std::mutex mu;
  size_t smem[kMaxDevices] = {};
  int sms[kMaxDevices] = {};
  int occ[kMaxDevices] = {};             // resident CTAs per SM at the largest `need` seen
  template <class F>
  cudaError_t ensure(F* kfn, int dev, size_t need, int threads, int* sms_out, bool check_occ = true,
                     int* occ_out = nullptr) {
    if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> lk(mu);
    if (sms[dev] == 0) {
      const cudaError_t err = cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev);
      if (err != cudaSuccess) return err;
    }
    if (need > smem[dev] || smem[dev] == 0) {
      cudaError_t err = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need);
      if (err != cudaSuccess) return err;
      if (check_occ) {                                 // (cluster kernels: checked at launch)
        int o = 0;
        err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kfn, threads, need);
        if (err != cudaSuccess) return err;
        if (o < 1) return cudaErrorInvalidConfiguration;
        occ[dev] = o;
      }
      smem[dev] = need;
    }
    *sms_out = sms[dev];
    if (occ_out) *occ_out = occ[dev] > 0 ? occ[dev] : 1;
    return cudaSuccess;
  }
};

// Per-packing parameters of one launch (adaptive plans fill several).
struct ModeP {
  const double* kr;     // core taps, reversed, K + 32 doubles after 16 zeros (kr[-16..-1] = 0; device)
  double Q;             // S_q
  double c_k;           // kernel companding factor
  double eps, eps_inv;  // packing coefficient and its inverse
  int pow2;             // eps = 2^-b (reading C4)
  int b;                // that b (0 if eps is not a power of two)
  int alu_pack;         // tiled kernel: pack with integer ops (dyadic eps, every packed word < 2^53 in units)
  int exact_pack;       // dyadic eps and every packed word exact in FP64: Horner steps as one FMA (same bits)
  int K, K_pad;         // core taps and taps padded to a multiple of the kernel's tile T
  int rows;             // rows of the column layout of the core's input words
  int paper_unpack;     // SYM: literal Eqs. (11)-(15) with the u_sys guard instead of balanced digits
  double R, R_safe;     // R_max and R_safe = R (eps + 1 + eps^-1) + u_sys eps^-1
};

struct Exec {
  const double* s;      // s[i - s_off] is global sample i (row `sig` at s + sig*s_stride)
  long long s_off, s_stride;
  double* r;            // r[g - r_off] is global output g (or lag g for xcorr)
  long long r_off, r_stride;
  long long b0, nblk;   // block range [b0, b0 + nblk) of every signal; grid = n_sig * nblk
  int stage_raw;        // stage the W_block raw samples in shared memory (TMA bulk copy)
  int reg_path;         // every block has <= blockDim.x groups: results stay in registers
  ModeP mp[4];          // indexed by packing (PACK_FULL .. PACK_ASYM3)
  const int* dec_pack;  // adaptive: per (signal, block) packing, else nullptr
  const int* blk_list;  // tiled kernel, adaptive: ascending blocks of this launch's packing (device), else nullptr
  const int* blk_count; // tiled kernel, adaptive: number of entries of blk_list (device)
  // persistent warp-specialized kernel
  unsigned* sm_ctr;             // per-SM job queue counters [kCtrDone] + done counter (plan-owned, zero between launches)
  int nsm;                      // SMs (queues)
  int gmax;                     // max T-groups of any block (sym fix-up arrays)
  long long nsig;               // signals in the launch (jobs = nsig * nblk)
  // tiled kernel: jobs = (signal, block, tile); tile = G groups of T outputs; taps in chunks
  int G;                        // consumer threads = groups per tile
  int KC, nchunks;              // taps per chunk (multiple of T), chunks per job
  int nstages;                  // stage ring slots (2 .. kTiledMaxStages)
  int raw_slots, raw_stride;    // raw-staged producers: raw block slots after the staging rows (0: global loads), doubles each
  int lookahead;                // > 0: claim job sequence m only once consumers have claimed parts of m - lookahead
  int early_fill;               // 1: the pipeline fill runs before griddepcontrol.wait (see pc_tiled_kernel)
  int early_claim;              // 1: the fill's job claims run before griddepcontrol.wait (alternating queue arrays)
  int taps_resident;            // 1: all K_pad taps stay in shared memory (nchunks == 1)
  int rows_s;                   // rows of a stage's padded word window
  long long tiles0, tiles1;     // tiles of block 0 / of every other block
  long long jobs_per_sig;       // jobs of one signal in this launch
  // parity/debug dumps (row = sig * P + w), nullptr in production
  double* dbg_packed;
  long long dbg_packed_stride;
  double* dbg_rbar;
  long long dbg_rbar_stride;
  long long* dbg_rint;
  long long dbg_rint_stride;
  double* dbg_cs;
  unsigned long long* dbg_timing;   // persistent kernel: per CTA {smid, t_start, t_end, jobs}
  // xcorr with fused score (tiled kernel): instead of storing the lags, every warp part writes
  // the max over its valid lags and the lowest lag attaining it to [sig][job * npart + part]
  double* xc_val;                    // nullptr: store the lags
  long long* xc_lag;
  // one kernel per signal (conv_xcorr_pairs, NEXT-3): taps kr_sig + sig * kr_stride (chunked
  // through the stages, never resident) and c_k = scal_sig[3 sig + 1]; nullptr: the plan's kernel
  const double* kr_sig;
  long long kr_stride;
  const double* scal_sig;
  // prepacked windows (pc_prepack_kernel, single-chunk plans): job j's stage image (rows_s rows of
  // pitch T + 4) at pre_win + j * pre_stride and its (c_s c_k)^-1 at pre_inv[j]; the tiled
  // kernel's producers then only move them into the ring with one bulk copy each
  const double* pre_win;
  long long pre_stride;
  const double* pre_inv;
  // plan flags in host-mapped pinned memory (conv_execute reads them without synchronizing):
  // [kStatusMargin] an FFT-core launch saw a last-digit residual > 0.25 LSB, [kStatusWatchdog] a
  // persistent-kernel wait timed out and the launch abandoned its work
  int* status;
  double* dbg_resid;    // conv_execute_debug: max last-digit residual (LSB, atomicMax on the bits)
  // tiled kernel: block peaks max|x| computed ahead (pc_block_peak, or pc_block_stats for adaptive
  // plans) at blk_peak[sig * peak_stride + w]; nullptr: the producers compute them
  const double* blk_peak;
  long long peak_stride;
  // producer SMs (conv_opts.prepack < 0, single-chunk packed plans; needs pre_win/pre_inv): CTAs
  // [0, split_P) compand and pack jobs F, F+1, .. into their stage images at pre_win (one job per
  // group of four warps, no DMMA warps on those SMs) and raise split_flags[j] = epoch + 1; the
  // other CTAs pack their first jobs in the pipeline fill (F = their count x fill depth) and move
  // the rest into the ring by bulk copy once flagged.  split_ctl[0] = epoch (launch count).
  int split_P;
  unsigned* split_flags;
  unsigned* split_ctl;
};
constexpr int kStatusMargin = 0, kStatusWatchdog = 1;
constexpr int kCtrProd = 250, kCtrCons = 251;   // sm_ctr slots of the producer-SM mode (reset per launch)

// FFT overlap-save core (pc_fft.cu).
struct FftArgs {
  const double2* tw;     // exp(-2 pi i m / N), m < N          (N complex points)
  const double2* tw2;    // exp(-2 pi i k / 2N), k <= N         (real-FFT split/merge)
  const double2* H;      // 2N-point real DFT of the core taps, k <= N
  double* resid;         // plan-owned max last-digit residual (LSB), atomicMax on the bits
  int part0_out, part_out;   // core outputs of a block's first / later parts
  long long parts0, parts1;  // parts of block 0 / of every other block
};
cudaError_t launch_fft_conv(int packing, int N, const Geo& g, const Exec& e, const FftArgs& f, long long n_jobs,
                            cudaStream_t st);
cudaError_t launch_fft_spectrum(int N, const double* kr, int K, const double2* tw, const double2* tw2, double2* H,
                                cudaStream_t st);

cudaError_t launch_fused(int packing, const Geo& g, const Exec& e, long long n_jobs, int threads, size_t smem,
                         cudaStream_t st);
// a2-a4 for every job of a tiled launch, ahead of it (pc_tiled.cu): block peak, c_s, packing
// into the stage image the DMMA core reads; one CTA per job.
cudaError_t launch_prepack(int packing, int T, int mma, const Geo& g, const Exec& e, long long n_jobs, cudaStream_t st);
// Tiled persistent warp-specialized kernel (pc_tiled.cu): grid = SMs x resident CTAs.
// mma = 1: the core runs on the FP64 tensor cores (T = 16 only; stage pitch 20, taps with 16
// zeros before and after -- every tap buffer is allocated with 16 leading zeros).
cudaError_t launch_tiled(int packing, int T, int mma, const Geo& g, const Exec& e, long long n_jobs, int threads,
                         size_t smem, cudaStream_t st, int* grid_out);
cudaError_t launch_kernel_prep(const double* k_in, int N, int Np, int reverse, double K_q, double* k_pad,
                               double* k_int, double* scal, cudaStream_t st);
cudaError_t launch_build_taps(const double* k_pad, const double* k_int, int Np, int packing, double eps_inv, int K,
                              int K_pad, double* kr, cudaStream_t st);
cudaError_t launch_kernel_prep_batch(const double* k_in, long long k_stride, long long n, int N, int Np, int reverse,
                                     double K_q, double* k_pad, double* k_int, long long pad_stride, double* scal,
                                     cudaStream_t st);
cudaError_t launch_build_taps_batch(const double* k_pad, const double* k_int, long long pad_stride, int Np,
                                    int packing, double eps_inv, int K, int K_pad, double* kr, long long kr_stride,
                                    long long n, cudaStream_t st);
// s: global sample base; blocks [b0, b0 + nb) (nb < 0: to the end)
cudaError_t launch_block_stats(const Geo& g, const double* s, double* sigma, double* peak, cudaStream_t st,
                               long long b0 = 0, long long nb = -1);
cudaError_t launch_adapt_decide(long long P, const double* sigma, const double* peak, double sig_k, double peak_k,
                                const int* cand, const int* qmode, int ncand, double thr, int* dp, int* dq, double* ds,
                                cudaStream_t st);
// decisions of blocks [b0, b0 + P) into lists of row stride `stride` (< 0: P)
cudaError_t launch_adapt_lists(long long P, const int* dec_pack, int* lists, int* counts, cudaStream_t st,
                               long long b0 = 0, long long stride = -1);
cudaError_t launch_xcorr_reduce(const double* val, const long long* lag, long long n_signals, long long n_part,
                                double* score, long long* best, cudaStream_t st);
cudaError_t launch_snr_sums(const double* ref, const double* x, long long n, const double* sigma, const double* peak,
                            long long P, double sig_k, double peak_k, double Q, double* out, cudaStream_t st);
cudaError_t launch_best_match(const double* score, const long long* lag, const double* cand, long long n,
                              long long first_index, double* best, cudaStream_t st);
// Per-block peak max|x| of blocks [b0, b0 + nblk) of n_sig signals (rows s + sig * s_stride, global
// sample base s - s_off) into peak[sig * peak_stride + w].
cudaError_t launch_block_peak(const Geo& g, const double* s, long long s_off, long long s_stride, long long b0,
                              long long nblk, long long n_sig, double* peak, long long peak_stride, cudaStream_t st);
cudaError_t launch_fill_pm1(double* x, long long n, unsigned long long seed, cudaStream_t st);
cudaError_t launch_xcorr_max(const double* c, long long n_signals, long long n_lags, long long stride,
                             double* score, long long* lag, cudaStream_t st);

}  // namespace pc
