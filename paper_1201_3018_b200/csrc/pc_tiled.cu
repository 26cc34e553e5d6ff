// pc_tiled.cu -- the production kernel of the packed overlap-save path (arXiv 1201.3018):
// persistent, warp-specialized, (block, output-tile) jobs, tap-chunked shared-memory stages.
//
// Job = (signal, overlap-save block w, tile t).  Tile t covers core outputs
// [t*G*T, (t+1)*G*T) of block w (G consumer threads, T outputs each).  The core taps are
// processed in chunks of KC (one chunk, taps resident in shared memory, whenever they fit),
// so any kernel length runs: cfg2's 513 taps in one chunk, cfg3/cfg4's 4097/8193 in several.
//
//   producer warps  a2-a4: block peak (coalesced loads + shuffles; reused across the tiles
//                   of one block), companding (Eq. (2)), packing (Eq. (4) / Eq. (7)) of the
//                   words one (tile, chunk) needs into a shared-memory stage; non-resident
//                   tap chunks arrive by TMA bulk copy on the same mbarrier
//   consumer warps  a5: the FP64 core (conv_chunk_padded, accumulators live across chunks);
//                   a6-a7: unpacking, inverse companding and placement from registers
//
// Stages (2) are handed over with mbarriers: full (producers -> consumers, + TMA bytes) and
// empty (consumers -> producers).  Symmetric packing needs B of the word before the tile for
// the tile's first even output: consumer warp 0 computes that one extra core output by a
// warp-split dot product (exact under the dyadic eps, reading C4).
#include "pc_device.cuh"
#include "pc_kernels.h"

namespace pc {

namespace {

struct TSmem {
  uint64_t bar_taps, full[2], empty[2];
  long long job[2];
  double cs[2], inv[2];
  long long prod_job;
  double prod_cs;
  long long prod_blk;
  double red[32];
};
static_assert(sizeof(TSmem) <= kSmemHeader, "header");

struct JobPos {
  long long sig, w;
  int t;
};

__device__ __forceinline__ JobPos job_pos(const Exec& e, long long job) {
  JobPos p;
  p.sig = job / e.jobs_per_sig;
  long long r = job % e.jobs_per_sig;
  if (e.b0 == 0) {                                   // block 0 (if in range) has tiles0 tiles
    if (r < e.tiles0) {
      p.w = 0;
      p.t = (int)r;
      return p;
    }
    r -= e.tiles0;
    p.w = 1 + r / e.tiles1;
    p.t = (int)(r % e.tiles1);
  } else {
    p.w = e.b0 + r / e.tiles1;
    p.t = (int)(r % e.tiles1);
  }
  return p;
}

// a4 for one stage: core words [cw0, cw0 + rows_s*T) of block b into the padded row-major
// window xs[(i / T) * (T + 1) + i % T].  Word-major over the producer threads (coalesced
// loads), UW words per thread with every sample load issued before any use.
template <int PACK, int T>
__device__ __forceinline__ void pack_window(const Geo& g, const Blk& b, const ModeP& mp, const double* gsrc,
                                            int n_valid, double c_s, int cw0, int rows_s, double* xs, int ptid,
                                            int nprod) {
  constexpr int UW = (PACK == PACK_ASYM3) ? 4 : 8;
  const int words = rows_s * T;
  auto sample = [&](int i) -> double { return (i < 0 || i >= n_valid) ? 0.0 : __ldg(gsrc + i); };
  for (int i0 = ptid; i0 < words; i0 += UW * nprod) {
    double v[UW];
    if (PACK == PACK_SYM) {
      double x0[UW], x1[UW];
#pragma unroll
      for (int u = 0; u < UW; ++u) {
        const int j = cw0 + i0 + u * nprod - b.pre;      // s_bar[j] uses samples 2j, 2j+1 (Eq. (4))
        x0[u] = sample(2 * j);
        x1[u] = sample(2 * j + 1);
      }
#pragma unroll
      for (int u = 0; u < UW; ++u) {
        const int cw = cw0 + i0 + u * nprod;
        v[u] = (cw >= b.pre && cw < b.xlen) ? pack_sym(compand1(c_s, x0[u]), compand1(c_s, x1[u]), mp.eps) : 0.0;
      }
    } else if (PACK == PACK_ASYM2 || PACK == PACK_ASYM3) {
      constexpr int M = (PACK == PACK_ASYM2) ? 2 : 3;
      double x[M][UW];
      const int base = b.o0 - (g.Np - 1) + cw0;          // Eq. (7) under C8
#pragma unroll
      for (int u = 0; u < UW; ++u)
#pragma unroll
        for (int q = 0; q < M; ++q) x[q][u] = sample(base + q * b.S + i0 + u * nprod);
#pragma unroll
      for (int u = 0; u < UW; ++u) {
        double a = compand1(c_s, x[M - 1][u]);           // Horner, oracle order
#pragma unroll
        for (int q = M - 2; q >= 0; --q) a = __dadd_rn(compand1(c_s, x[q][u]), __dmul_rn(mp.eps, a));
        const int cw = cw0 + i0 + u * nprod;
        v[u] = (cw >= 0 && cw < b.xlen) ? a : 0.0;
      }
    } else {
      const int base = b.o0 - (g.Np - 1) + cw0;
#pragma unroll
      for (int u = 0; u < UW; ++u) {
        const int cw = cw0 + i0 + u * nprod;
        v[u] = (cw >= 0 && cw < b.xlen) ? sample(base + i0 + u * nprod) : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < UW; ++u) {
      const int i = i0 + u * nprod;
      if (i < words) xs[(i / T) * (T + 1) + i % T] = v[u];
    }
  }
}

// a2/a3: block peak over the W_block samples (16 loads in flight per thread, shuffles),
// companding factor c_s = Q / peak (Eq. (2)).  All `nprod` threads call it.
template <int PACK>
__device__ __forceinline__ double block_cs(const ModeP& mp, const double* gsrc, int n_valid, TSmem* ps, int ptid,
                                           int nprod, int bar_id) {
  if (PACK == PACK_FULL) return 1.0;
  constexpr int U = 16;
  double m[U];
#pragma unroll
  for (int u = 0; u < U; ++u) m[u] = 0.0;
  if ((reinterpret_cast<uintptr_t>(gsrc) & 15u) == 0) {
    const double2* g2 = reinterpret_cast<const double2*>(gsrc);
    const int n2 = n_valid / 2;
    for (int i0 = ptid; i0 < n2; i0 += U * nprod) {
      double2 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + u * nprod;
        v[u] = (i < n2) ? __ldg(g2 + i) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) m[u] = fmax(m[u], fmax(fabs(v[u].x), fabs(v[u].y)));
    }
    if ((n_valid & 1) && ptid == 0) m[0] = fmax(m[0], fabs(gsrc[n_valid - 1]));
  } else {
    for (int i = ptid; i < n_valid; i += nprod) m[0] = fmax(m[0], fabs(__ldg(gsrc + i)));
  }
#pragma unroll
  for (int u = 1; u < U; ++u) m[0] = fmax(m[0], m[u]);
  for (int o = 16; o > 0; o >>= 1) m[0] = fmax(m[0], __shfl_xor_sync(0xffffffffu, m[0], o));
  if ((ptid & 31) == 0) ps->red[ptid >> 5] = m[0];
  named_bar(bar_id, nprod);
  double peak = 0.0;
  for (int wi = 0; wi < nprod / 32; ++wi) peak = fmax(peak, ps->red[wi]);
  named_bar(bar_id, nprod);
  return (peak == 0.0) ? 1.0 : mp.Q / peak;
}

}  // namespace

// Accumulating variant of the padded-layout core: acc += sum over n_taps of this chunk.
template <int T>
__device__ __forceinline__ void conv_chunk_padded(uint32_t xs_row, uint32_t kr_addr, int n_taps, double (&acc)[T]) {
  double win[T];
#pragma unroll
  for (int c = 0; c < T - 1; ++c) win[c] = lds64(xs_row + 8u * c);
  uint32_t xa = xs_row, ka = kr_addr;
  for (int j0 = 0; j0 < n_taps; j0 += T, xa += 8u * (T + 1), ka += 8u * T) {
    double kk[T];
#pragma unroll
    for (int u = 0; u < T; u += 2) {
      const double2 k2 = lds128(ka + 8u * u);
      kk[u] = k2.x;
      kk[u + 1] = k2.y;
    }
#pragma unroll
    for (int u = 0; u < T; ++u) {
      win[(T - 1 + u) % T] = lds64(xa + 8u * (((T - 1 + u) / T) * (T + 1) + (T - 1 + u) % T));
#pragma unroll
      for (int i = 0; i < T; ++i) acc[i] = fma(win[(i + u) % T], kk[u], acc[i]);
    }
  }
}

template <int PACK, int T>
__global__ void __maxnreg__(96) pc_tiled_kernel(Geo g, Exec e) {
  extern __shared__ __align__(128) unsigned char smem[];
  TSmem* ps = reinterpret_cast<TSmem*>(smem);
  const ModeP& mp = e.mp[PACK];
  const int G = e.G;                       // consumer threads = groups per tile
  const int KC = e.KC;                     // taps per chunk (multiple of T)
  const int nch = e.nchunks;
  const int front = (PACK == PACK_SYM) ? 1 : 0;   // one row before the tile: the extra word
  const int rows_s = e.rows_s;
  const int stage_x = ((T + 1) * rows_s + 1) & ~1;   // doubles of a stage's word window (16B-aligned end)
  const int stage_words = stage_x + (e.taps_resident ? 0 : KC);
  double* kr_res = reinterpret_cast<double*>(smem + kSmemHeader);          // resident taps
  double* stg = kr_res + (e.taps_resident ? mp.K_pad : 0);                  // 2 stages
  double* fix = stg + 2 * stage_words;                                      // sym: [2][2][G+1]
  const int tid = threadIdx.x;
  const int nprod = e.np_warps * 32;
  const int ncons = blockDim.x - nprod;
  const long long njobs = e.jobs_per_sig * e.nsig;

  if (tid == 0) {
    mbar_init(&ps->bar_taps, 1);
    mbar_init(&ps->full[0], nprod);
    mbar_init(&ps->full[1], nprod);
    mbar_init(&ps->empty[0], ncons);
    mbar_init(&ps->empty[1], ncons);
    const uint32_t tb = e.taps_resident ? (uint32_t)mp.K_pad * 8u : 0u;
    mbar_arrive_expect_tx(&ps->bar_taps, tb);
    if (tb) bulk_g2s(kr_res, mp.kr, tb, &ps->bar_taps);
  }
  // programmatic dependent launch: only plan-owned, read-only taps are touched above
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __syncthreads();

  // Locate a job's block and input.
  auto job_block = [&](long long job, JobPos& jp, Blk& b, const double*& gsrc, int& n_valid) {
    jp = job_pos(e, job);
    b = block_info<PACK>(g, mp.K, jp.w);
    gsrc = e.s + jp.sig * e.s_stride + (b.g0 - e.s_off);
    const long long avail = g.L - b.g0;
    n_valid = (int)(avail < 0 ? 0 : (avail > g.W_block ? g.W_block : avail));
  };
  // Hand a packed stage to the consumers (+ the tap chunk by TMA when not resident).
  auto publish = [&](int stage, int c, long long job, double c_s, double inv, int ptid) {
    double* xs = stg + stage * stage_words;
    if (ptid == 0) {
      ps->job[stage] = job;
      ps->cs[stage] = c_s;
      ps->inv[stage] = inv;
    }
    if (!e.taps_resident && ptid == 0) {
      const int nt = (c == nch - 1) ? mp.K_pad - c * KC : KC;
      mbar_arrive_expect_tx(&ps->full[stage], (uint32_t)nt * 8u);
      bulk_g2s(xs + stage_x, mp.kr + (size_t)c * KC, (uint32_t)nt * 8u, &ps->full[stage]);
    } else {
      mbar_arrive(&ps->full[stage]);
    }
  };

  // Pipeline fill: every warp helps compand and pack chunk 0 of the first job into stage 0.
  if (tid == 0) ps->prod_job = (long long)(atomicAdd(e.counter, 1ULL) - e.base);
  __syncthreads();
  const long long job0 = ps->prod_job;
  long long cur_blk = -1;
  double c_s = 1.0, inv = 0.0;
  if (job0 < njobs) {
    JobPos jp;
    Blk b;
    const double* gsrc;
    int n_valid;
    job_block(job0, jp, b, gsrc, n_valid);
    c_s = block_cs<PACK>(mp, gsrc, n_valid, ps, tid, blockDim.x, 0);
    inv = dequant_scale(c_s, mp.c_k);
    cur_blk = jp.sig * g.P + jp.w;
    pack_window<PACK, T>(g, b, mp, gsrc, n_valid, c_s, jp.t * G * T - front * T, rows_s, stg, tid, blockDim.x);
  }
  __syncthreads();
  if (tid < nprod) {
    if (job0 < njobs) {
      publish(0, 0, job0, c_s, inv, tid);
    } else {
      if (tid == 0) ps->job[0] = -1;
      mbar_arrive(&ps->full[0]);
    }
  }
  if (job0 >= njobs) return;

  if (tid < nprod) {
    // ============================ producer warps ============================
    const int ptid = tid;
    int it = 1;
    long long job = job0;
    int c = 1;
    for (;;) {
      if (c == nch) {                                    // next job, claimed once a stage is free
        c = 0;
        mbar_wait(&ps->empty[it & 1], ((it >> 1) & 1) ^ 1);
        named_bar(2, nprod);
        if (ptid == 0) ps->prod_job = (long long)(atomicAdd(e.counter, 1ULL) - e.base);
        named_bar(2, nprod);
        job = ps->prod_job;
        if (job >= njobs) {
          if (ptid == 0) ps->job[it & 1] = -1;
          mbar_arrive(&ps->full[it & 1]);
          break;
        }
      } else {
        mbar_wait(&ps->empty[it & 1], ((it >> 1) & 1) ^ 1);
      }
      JobPos jp;
      Blk b;
      const double* gsrc;
      int n_valid;
      job_block(job, jp, b, gsrc, n_valid);
      const long long blk_id = jp.sig * g.P + jp.w;
      if (blk_id != cur_blk) {                          // peak reused across a block's tiles
        cur_blk = blk_id;
        c_s = block_cs<PACK>(mp, gsrc, n_valid, ps, ptid, nprod, 2);
        inv = dequant_scale(c_s, mp.c_k);                // Eq. (16), once per block
      }
      const int stage = it & 1;
      pack_window<PACK, T>(g, b, mp, gsrc, n_valid, c_s, jp.t * G * T - front * T + c * KC, rows_s,
                           stg + stage * stage_words, ptid, nprod);
      publish(stage, c, job, c_s, inv, ptid);
      ++c;
      ++it;
    }
    return;
  }

  // ============================ consumer warps ============================
  const int ctid = tid - nprod;
  const int cwarp = ctid >> 5, lane = ctid & 31;
  mbar_wait(&ps->bar_taps, 0);
  int it = 0, njob = 0;
  for (;; ++njob) {
    int stage = it & 1;
    mbar_wait(&ps->full[stage], (it >> 1) & 1);
    const long long job = ps->job[stage];
    if (job < 0) break;
    const double inv = ps->inv[stage];
    const JobPos jp = job_pos(e, job);
    const Blk b = block_info<PACK>(g, mp.K, jp.w);
    const int ngroups = (b.M_out + T - 1) / T;
    const int gl = ctid;                                     // this thread's group in the tile
    const int gi = jp.t * G + gl;                            // group index within the block
    const bool mine = gl < G && gi < ngroups;
    const bool extra = (PACK == PACK_SYM) && jp.t > 0 && cwarp == 0;
    double acc[T];
#pragma unroll
    for (int i = 0; i < T; ++i) acc[i] = 0.0;
    double px = 0.0;                                         // sym extra word partial (warp 0)
    for (int c = 0; c < nch; ++c, ++it) {
      stage = it & 1;
      if (c > 0) mbar_wait(&ps->full[stage], (it >> 1) & 1);
      const double* xs = stg + stage * stage_words;
      const double* kc = e.taps_resident ? kr_res + (size_t)c * KC : xs + stage_x;
      const int nt = (c == nch - 1) ? mp.K_pad - c * KC : KC;
      if (mine) conv_chunk_padded<T>(smem_u32(xs) + 8u * (T + 1) * (gl + front), smem_u32(kc), nt, acc);   // a5
      if (extra) {
        for (int j = lane; j < nt; j += 32) {
          const int i = T - 1 + j;                           // local word of core word m_lo-1+j
          px = fma(xs[(i / T) * (T + 1) + i % T], kc[j], px);
        }
      }
      mbar_arrive(&ps->empty[stage]);
    }
    // ---- a6/a7: unpack, inverse-compand, discard and place (Eqs. (11)-(17))
    double* __restrict__ r = e.r + jp.sig * e.r_stride;
    const long long gbase = b.g0 + b.o0;
    const long long L_conv = g.L + g.N - 1;
    auto store = [&](int k, double val) {
      const long long gg = gbase + k;
      if (g.mode == 0) {
        if (gg < L_conv) r[gg - e.r_off] = val;
      } else {
        const long long j = gg - (g.N - 1);                  // valid lag (C17)
        if (j >= 0 && j <= g.L - g.N) r[j - e.r_off] = val;
      }
    };
    const int moff = (jp.w == 0) ? 0 : 1;
    if (PACK == PACK_SYM) {
      double* cfirst = fix + (njob & 1) * 2 * (G + 1);
      double* blast = cfirst + (G + 1) + 1;                   // blast[-1] = B of the extra word
      if (extra) {
        for (int o = 16; o > 0; o >>= 1) px += __shfl_xor_sync(0xffffffffu, px, o);
        if (lane == 0) blast[-1] = decode_sym(px, mp.eps, mp.eps_inv, mp.pow2).B;
      }
      if (mine) {
        double Bprev = 0.0;
#pragma unroll
        for (int i = 0; i < T; ++i) {
          const int m = gi * T + i;
          const Digits3 d = decode_sym(acc[i], mp.eps, mp.eps_inv, mp.pow2);
          if (m < b.M_out && m >= moff) {
            const int k = 2 * (m - moff);
            store(k + 1, __dmul_rn(d.A, inv));
            if (i > 0 || m == 0) {
              store(k, __dmul_rn(d.C + Bprev, inv));
            } else {
              cfirst[gl] = d.C;                              // needs B of the previous word
            }
          }
          Bprev = d.B;
        }
        blast[gl] = Bprev;
      }
      named_bar(1, ncons);
      if (mine) {
        const int m = gi * T;
        if (m < b.M_out && m >= moff && m > 0) store(2 * (m - moff), __dmul_rn(cfirst[gl] + blast[gl - 1], inv));
      }
    } else if (PACK == PACK_ASYM2 || PACK == PACK_ASYM3) {
      if (mine) {
        constexpr int M = (PACK == PACK_ASYM2) ? 2 : 3;
#pragma unroll
        for (int i = 0; i < T; ++i) {
          const int m = gi * T + i;
          if (m < b.S) {
            double v = acc[i];
#pragma unroll
            for (int q = 0; q < M; ++q) {                     // balanced digits (C9)
              const double t = rint_fast(v);
              if (q < M - 1) v = __dmul_rn(__dsub_rn(v, t), mp.eps_inv);
              const int k = q * b.S + m;
              if (k < b.n_out) store(k, __dmul_rn(t, inv));
            }
          }
        }
      }
    } else if (mine) {
#pragma unroll
      for (int i = 0; i < T; ++i) {
        const int m = gi * T + i;
        if (m < b.n_out) store(m, acc[i]);
      }
    }
  }
}

// ------------------------------------------------------------------ launcher
template <int PACK, int T>
static cudaError_t launch_tiled_t(const Geo& g, const Exec& e, long long n_jobs, int threads, size_t smem,
                                  cudaStream_t st, int* grid_out) {
  auto kfn = pc_tiled_kernel<PACK, T>;
  static size_t c_smem = 0;
  static int c_threads = 0, c_grid = 0, c_dev = -1, c_sms = 0;
  int dev = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err != cudaSuccess) return err;
  if (smem != c_smem || threads != c_threads || dev != c_dev) {
    err = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    int occ = 0;
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, threads, smem);
    if (err != cudaSuccess) return err;
    cudaDeviceGetAttribute(&c_sms, cudaDevAttrMultiProcessorCount, dev);
    if (occ < 1) return cudaErrorInvalidConfiguration;
    c_smem = smem;
    c_threads = threads;
    c_dev = dev;
    c_grid = c_sms * occ;
  }
  long long grid = c_grid;
  if (e.max_ctas_per_sm > 0 && (long long)e.max_ctas_per_sm * c_sms < grid) grid = (long long)e.max_ctas_per_sm * c_sms;
  if (grid > n_jobs) grid = n_jobs;
  *grid_out = (int)grid;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kfn, g, e);
}

template <int T>
static cudaError_t launch_tiled_T(int packing, const Geo& g, const Exec& e, long long n_jobs, int threads, size_t smem,
                                  cudaStream_t st, int* grid_out) {
  switch (packing) {
    case PACK_FULL: return launch_tiled_t<PACK_FULL, T>(g, e, n_jobs, threads, smem, st, grid_out);
    case PACK_SYM: return launch_tiled_t<PACK_SYM, T>(g, e, n_jobs, threads, smem, st, grid_out);
    case PACK_ASYM2: return launch_tiled_t<PACK_ASYM2, T>(g, e, n_jobs, threads, smem, st, grid_out);
    case PACK_ASYM3: return launch_tiled_t<PACK_ASYM3, T>(g, e, n_jobs, threads, smem, st, grid_out);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_tiled(int packing, int T, const Geo& g, const Exec& e, long long n_jobs, int threads, size_t smem,
                         cudaStream_t st, int* grid_out) {
  *grid_out = 0;
  if (n_jobs <= 0) return cudaSuccess;
  switch (T) {
    case 12: return launch_tiled_T<12>(packing, g, e, n_jobs, threads, smem, st, grid_out);
    case 14: return launch_tiled_T<14>(packing, g, e, n_jobs, threads, smem, st, grid_out);
    case 16: return launch_tiled_T<16>(packing, g, e, n_jobs, threads, smem, st, grid_out);
  }
  return cudaErrorInvalidValue;
}

}  // namespace pc
