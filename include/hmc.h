/*
 * hmc.h -- C ABI of libhmc.so, the B200 (sm_100a) Heston Monte Carlo Greeks
 * engine.  Plain C types only: no torch, no C++ in the signatures.
 *
 * Reference interfaces each entry point replaces (reference =
 * /root/reference/pkg/src/hestonmc):
 *
 *   hmc_discretised_batch_f64  <- backend module call
 *                                 discretised_batch(params, s0, T, n_steps,
 *                                 milstein, path_lo, path_hi, key_run,
 *                                 uniforms, avg_indices)
 *                                 _core.pyx:354-412, _batch_py.py:36-81,
 *                                 called from engine.py:87-90
 *   hmc_greeks / hmc_greeks_chunks + hmc_reduce_chunks
 *                              <- engine._run_sums + _simulate_chunk +
 *                                 _per_path_stats (engine.py:47-116): one
 *                                 fused pass over all runs x paths producing
 *                                 per-run sums and sums of squares of
 *                                 price / Delta / Rho (+ Gamma, Vega, FD
 *                                 Delta, FD Rho from CRN bumps)
 *   hmc_greeks_multi           <- the same job dealt over several GPUs from
 *                                 one process (engine.py:104-116 workers)
 *   hmc_slice_chunks / hmc_comm_* (NCCL)
 *                              <- the same fan-out across processes, one
 *                                 per GPU: slice rule + the in-order
 *                                 exchange replacing the ordered fsum
 *                                 (engine.py:104-116)
 *   hmc_exact_batch_f64 / hmc_exact_runs_f64
 *                              <- backend module call exact_batch
 *                                 (_core.pyx:415-521), per run / all runs
 *   hmc_surface* (partials, finalize, one-call)
 *                              <- no reference counterpart: strike x maturity
 *                                 grids of the engine's estimators (BASELINE
 *                                 config 5) from one path set
 *   hmc_sobol_init_directions  <- scipy.stats.qmc.Sobol direction numbers
 *                                 used by rng.sobol_points (rng.py:143-152)
 *   hmc_uniforms_f64 / hmc_ndtri_f64 / hmc_gamma_f64 / hmc_steps_f64
 *                              <- rng.uniform_at / inverse_normal_cdf /
 *                                 gamma_batch and
 *                                 schemes.euler_step / milstein_step
 *                                 (rng.py:63-132, schemes.py:33-61)
 *   hmc_bessel_f64 / hmc_ivlaw_phi_f64 / hmc_ivlaw_eval_f64 /
 *   hmc_exact_step_f64         <- bessel.py / ivlaw.py / exact.py: the exact
 *                                 scheme's host-side spec modules
 *   hmc_root_key / hmc_derive_key
 *                              <- rng.root_key / rng.derive_key (rng.py:46-52)
 *   hmc_philox_check / hmc_box_muller_check / hmc_sobol_quantile_check /
 *   hmc_fp32_paths_check       <- test hooks: the device code paths of the
 *                                 fp32 kernels on given inputs (known-answer
 *                                 tests, tests/test_gpu_engine.py)
 *
 * Errors: every function returns 0 on success or a negative HMC_E* code;
 * hmc_last_error() gives a thread-local message for the last failure.
 * Threading: all entry points are re-entrant (no global mutable state apart
 * from the thread-local error string, a per-thread stream cache and
 * libhmc's private per-device memory pool); buffers are caller-owned.
 */
#ifndef HMC_H_
#define HMC_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HMC_ABI_VERSION 2

/* reduction geometry -- fixed so results never depend on grid size or GPU count */
#define HMC_TILE 128          /* paths per thread block == per tile partial   */
#define HMC_CHUNK_TILES 128   /* tiles per chunk partial                      */
#define HMC_CHUNK (HMC_TILE * HMC_CHUNK_TILES) /* 16384 paths per chunk      */
#define HMC_NQ 7              /* per-path quantities, order below             */
#define HMC_NW (2 * HMC_NQ)   /* {sum, sum of squares} per quantity           */
#define HMC_BRIDGE_MAX_SEGMENTS 64 /* Sobol Brownian-bridge skeleton size   */

/* quantity index q: partial[2*q] = sum_x, partial[2*q+1] = sum_x^2 */
enum {
    HMC_Q_PRICE = 0,    /* discounted payoff                engine.py:53-56 */
    HMC_Q_DELTA = 1,    /* pathwise Delta                   engine.py:58-59 */
    HMC_Q_RHO = 2,      /* pathwise Rho                     engine.py:60-67 */
    HMC_Q_GAMMA = 3,    /* CRN FD of pathwise Delta, S0+-h     */
    HMC_Q_VEGA = 4,     /* CRN FD of price in v0            (north star)    */
    HMC_Q_DELTA_FD = 5, /* CRN FD of price in S0     test_products.py:101   */
    HMC_Q_RHO_FD = 6    /* CRN FD of price in r      test_products.py:114   */
};

enum {
    HMC_OK = 0,
    HMC_E_INVALID = -1,   /* bad argument            -> ValidationError     */
    HMC_E_CUDA = -2,      /* CUDA runtime failure    -> DeviceError         */
    HMC_E_NODEVICE = -3,  /* no CUDA device visible  -> DeviceError         */
    HMC_E_UNSUPPORTED = -4, /* e.g. Greeks for a put -> UnsupportedProduct  */
    HMC_E_BESSEL = -5,      /* exact scheme: Bessel series -> BesselNonConvergence */
    HMC_E_QUAD = -6,        /* exact scheme: CF tail -> QuadratureNonConvergence   */
    HMC_E_ROOT = -7         /* exact scheme: CDF inversion -> RootNotBracketed     */
};

enum { HMC_STYLE_EUROPEAN = 0, HMC_STYLE_ASIAN = 1 };
enum { HMC_CALL = 0, HMC_PUT = 1 };
enum { HMC_SCHEME_EULER = 1, HMC_SCHEME_MILSTEIN = 2 };
enum { HMC_SAMPLER_PSEUDO = 0, HMC_SAMPLER_SOBOL = 1 };
enum {
    HMC_PREC_FP32 = 0, /* Philox4x32-10 / Sobol, fp32 state, fp64 sums      */
    HMC_PREC_FP64 = 1  /* reference SplitMix64 / Sobol + Acklam-Halley ndtri,
                          fp64 state, the reference's operation order        */
};

/* HestonParams (model.py:11-45) */
typedef struct hmc_model {
    double kappa, theta, sigma, rho, r, v0;
} hmc_model;

/* OptionSpec (model.py:54-87) + averaging grid indices (engine.py:81-86) */
typedef struct hmc_product {
    int32_t style;          /* HMC_STYLE_*                                   */
    int32_t right;          /* HMC_CALL / HMC_PUT                            */
    double strike, maturity, spot;
    const int64_t* avg_idx; /* HOST pointer, strictly increasing in 1..n_steps;
                               european: {n_steps}                           */
    int64_t n_avg;
} hmc_product;

/* SimConfig (model.py:140-180) + this call's slice of the path axis */
typedef struct hmc_sim {
    int32_t scheme;       /* HMC_SCHEME_*                                    */
    int32_t sampler;      /* HMC_SAMPLER_*                                   */
    int32_t precision;    /* HMC_PREC_*                                      */
    int32_t want_greeks;  /* 0: price column only                            */
    int32_t n_steps;
    int32_t n_runs;
    int64_t n_paths;      /* paths per run (whole job)                       */
    int64_t path_lo;      /* this slice: [path_lo, path_hi), path_lo % HMC_CHUNK == 0 */
    int64_t path_hi;
    uint64_t seed;
    double h_spot;        /* absolute S0 bump                                */
    double v0_up, v0_dn;  /* start variances of the two v0-bumped trajectories */
    double h_r;           /* absolute r bump                                 */
    const uint32_t* sobol_v; /* sobol only: [30][2*n_steps] direction numbers
                                (hmc_sobol_init_directions layout)           */
    int32_t sobol_v_on_device; /* 1: sobol_v is a device pointer of the
                                  current device; 0: host pointer            */
    int32_t sobol_scramble;    /* sobol only: random digital shift per (run,
                                  dimension) from the seed (randomised QMC)  */
    int32_t sobol_bridge;      /* sobol only: 0 = dimensions in time order (the
                                  reference, engine.py:97-101); S > 0 = Brownian
                                  bridge: the first S dimension pairs build a
                                  skeleton of both Brownian motions at S
                                  segment ends, the rest fill each segment by
                                  conditional (bridge) sampling in time order.
                                  1 <= S <= min(HMC_BRIDGE_MAX_SEGMENTS, steps) */
} hmc_sim;

int hmc_abi_version(void);
const char* hmc_last_error(void);
int hmc_device_count(int32_t* count);

/* number of chunk partials this slice produces per run */
int64_t hmc_chunks_in_slice(const hmc_sim* sim);
/* device workspace bytes hmc_greeks_chunks needs for this slice */
int64_t hmc_workspace_bytes(const hmc_sim* sim);

/* Launch the fused path + Greeks kernel for [path_lo, path_hi) x all runs on
 * `stream` (cudaStream_t, NULL = legacy default) of the CURRENT device and
 * write chunk partials d_chunks[run][chunk][HMC_NW] (device, fp64).
 * d_work: device scratch of hmc_workspace_bytes(sim) bytes.  Asynchronous. */
int hmc_greeks_chunks(const hmc_model* model, const hmc_product* product,
                      const hmc_sim* sim, double* d_chunks, void* d_work,
                      void* stream);

/* Fixed-shape (strided sequential + 512-way tree) fp64 sum of chunk partials
 * d_chunks[run][0..n_chunks)[HMC_NW] -> d_out[run][HMC_NW].  Chunks must be
 * in global path order; the result is then bit-identical for any split of
 * the path axis across calls / GPUs.  Asynchronous on `stream`. */
int hmc_reduce_chunks(const double* d_chunks, int32_t n_runs, int64_t n_chunks,
                      double* d_out, void* stream);

/* Convenience: whole job on one device, synchronous, HOST output
 * h_out[run][HMC_NW].  Inputs are host structs; sim->path_lo/hi are ignored
 * (the full [0, n_paths) range is simulated). */
int hmc_greeks(const hmc_model* model, const hmc_product* product,
               const hmc_sim* sim, double* h_out, int32_t device);

/* Single-process multi-GPU one-call (the reference's multi-worker engine,
 * engine.py:104-116, for C hosts that drive several GPUs themselves): the
 * path axis is dealt in contiguous chunk-aligned slices over
 * devices[0..n_devices) exactly as paper_2309_10477_b200.parallel.shard, each
 * slice runs on its device's own stream concurrently, the chunk partials are
 * copied in path order to devices[0] (peer copies over NVLink) and reduced
 * there with the fixed-shape tree: bit-identical to hmc_greeks for any device
 * list.  A device may appear more than once (several slices on one GPU).
 * Synchronous, HOST output h_out[run][HMC_NW]. */
int hmc_greeks_multi(const hmc_model* model, const hmc_product* product,
                     const hmc_sim* sim, double* h_out, const int32_t* devices,
                     int32_t n_devices);

/* ---- multi-process: one process per GPU, NCCL over NVLink / NVSwitch ----
 *
 * Replaces the reference's worker fan-out + ordered fsum (engine.py:104-116)
 * across processes.  Rank q of a world of W simulates the chunk slice
 * hmc_slice_chunks(n_paths, q, W) (set hmc_sim.path_lo/path_hi to
 * chunk_lo*HMC_CHUNK .. min(chunk_hi*HMC_CHUNK, n_paths)) with
 * hmc_greeks_chunks / hmc_exact_greeks_chunks into d_local[run][chunk][NW];
 * hmc_comm_gather_chunks then fills the global d_full[run][C][NW] in path
 * order on every rank and hmc_reduce_chunks reduces it: bit-identical to
 * one GPU.  NCCL (libnccl.so.2) is opened on first use.  A communicator must
 * not be used by two host threads at once. */
#define HMC_COMM_ID_BYTES 128
enum { HMC_DTYPE_I64 = 0, HMC_DTYPE_F64 = 1 };
typedef struct hmc_comm hmc_comm;   /* opaque */

/* the parallel.shard rule: [*chunk_lo, *chunk_hi) of C = ceil(n_paths /
 * HMC_CHUNK) chunks, dealt as evenly as possible (first C % world ranks get
 * one more) */
int hmc_slice_chunks(int64_t n_paths, int32_t rank, int32_t world, int64_t* chunk_lo,
                     int64_t* chunk_hi);
/* rank 0 creates the id (ncclGetUniqueId) and hands it to the others out of
 * band (MPI, a TCP store, torch.distributed.broadcast_object_list ...) */
int hmc_comm_unique_id(uint8_t* id_out /* [HMC_COMM_ID_BYTES] */);
/* collective: every rank calls it with the same id (ncclCommInitRank) */
int hmc_comm_init(const uint8_t* id, int32_t rank, int32_t world, int32_t device,
                  hmc_comm** comm_out);
int hmc_comm_destroy(hmc_comm* comm);
/* collective: d_local = this rank's [n_runs][nc_rank][HMC_NW] (DEVICE),
 * d_full = [n_runs][C][HMC_NW] (DEVICE), stream-ordered on `stream` */
int hmc_comm_gather_chunks(hmc_comm* comm, const double* d_local, int32_t n_runs,
                           int64_t n_paths, double* d_full, void* stream);
/* collective in-place sum of `count` elements of DEVICE d_buf: HMC_DTYPE_I64
 * (exact; the surface histograms) or HMC_DTYPE_F64 (order-dependent rounding) */
int hmc_comm_allreduce_sum(hmc_comm* comm, void* d_buf, int64_t count, int32_t dtype,
                           void* stream);

/* Reference backend call discretised_batch (_core.pyx:354-412) in fp64 on
 * the GPU: same key derivation, draw layout and arithmetic order.
 * uniforms: HOST (path_hi-path_lo, 2*n_steps) row-major or NULL (in-kernel
 * SplitMix64 stream); avg_idx: HOST; out: HOST (path_hi-path_lo, 3)
 * [s_T, avg, tw_sum].  Synchronous. */
int hmc_discretised_batch_f64(const hmc_model* model, double s0, double T,
                              int32_t n_steps, int32_t milstein,
                              int64_t path_lo, int64_t path_hi,
                              uint64_t key_run, const double* uniforms,
                              const int64_t* avg_idx, int64_t n_avg,
                              double* out, int32_t device);

/* ---- strike x maturity surfaces (BASELINE config 5) ---------------------
 * European and daily-average Asian calls on a strike grid at several
 * maturities of ONE time grid, full Greeks, all from the same paths.
 * Maturity m is the grid date mat_idx[m] (t = mat_idx[m] * dt); the Asian
 * average for maturity m runs over grid dates t_1..t_{mat_idx[m]}.
 * Output layout (HMC_NW = {sum, sum of squares} x 7 quantities, the single-
 * product order above): out[run][style: 0 european, 1 asian][mat][strike][HMC_NW]. */
#define HMC_SURF_MAX_STRIKES 128
#define HMC_SURF_MAX_MATS 32
#define HMC_SURF_VALS 23  /* moment rows per (style, maturity) */

typedef struct hmc_surface_spec {
    double spot;
    double dt;               /* grid step (year fraction)                      */
    const double* strikes;   /* HOST, strictly increasing, > 0                 */
    int32_t n_strikes;       /* 1 .. HMC_SURF_MAX_STRIKES                      */
    int32_t n_mats;          /* 1 .. HMC_SURF_MAX_MATS                         */
    const int64_t* mat_idx;  /* HOST, strictly increasing grid indices >= 1;
                                sim->n_steps must equal mat_idx[n_mats - 1]    */
} hmc_surface_spec;

/* int64 words of the fixed-point histogram accumulator for n_runs runs:
 * n_runs * 2 * n_mats * HMC_SURF_VALS * (n_strikes + 1). */
int64_t hmc_surface_acc_words(const hmc_surface_spec* spec, int32_t n_runs);
/* device workspace bytes of hmc_surface_partials */
int64_t hmc_surface_workspace_bytes(const hmc_surface_spec* spec, const hmc_sim* sim);

/* ADD this slice's paths [path_lo, path_hi) into d_acc (device int64, zero
 * it first; hmc_surface_acc_words words).  Integer accumulation: slices may
 * be summed in any order / all-reduced across GPUs with identical results.
 * sim: scheme euler|milstein, sampler pseudo, precision fp32; bumps as for
 * hmc_greeks.  Asynchronous on `stream`. */
int hmc_surface_partials(const hmc_model* model, const hmc_surface_spec* spec,
                         const hmc_sim* sim, int64_t* d_acc, void* d_work, void* stream);

/* HOST: accumulated histograms -> out[run][2][n_mats][n_strikes][HMC_NW]. */
int hmc_surface_finalize(const hmc_model* model, const hmc_surface_spec* spec,
                         const hmc_sim* sim, const int64_t* h_acc, double* out);

/* Convenience: whole job on one device, synchronous, HOST output. */
int hmc_surface(const hmc_model* model, const hmc_surface_spec* spec, const hmc_sim* sim,
                double* h_out, int32_t device);

/* Reference backend call exact_batch (_core.pyx:415-521): Broadie-Kaya
 * exact paths stepping through step_times[0..n_steps] (step_times[0] = 0),
 * fp64 on the GPU with the reference's random stream (3 main draws per step,
 * Gamma substream derive(path_key, 1)) and algorithm.  avg_flags[n_steps]:
 * 1 where the step's end is an averaging date.  uniforms: HOST
 * (path_hi-path_lo, 3*n_steps) or NULL; out: HOST (path_hi-path_lo, 3)
 * [s_T, avg, tw_sum].  Synchronous.  Numerical failures return
 * HMC_E_BESSEL / HMC_E_QUAD / HMC_E_ROOT like the reference's exceptions. */
int hmc_exact_batch_f64(const hmc_model* model, double s0, const double* step_times,
                        int32_t n_steps, const int64_t* avg_flags, int64_t path_lo,
                        int64_t path_hi, uint64_t key_run, const double* uniforms,
                        double* out, int32_t device);

/* The same for n_runs independent runs in ONE launch (the reference engine
 * calls exact_batch once per run and 4096-path job, engine.py:93-116):
 * run r uses key_runs[r] (derive_key(root_key(seed), r)); uniforms: HOST
 * [n_runs][path_hi-path_lo][3*n_steps] or NULL; out: HOST
 * [n_runs][path_hi-path_lo][3].  Per-path values equal hmc_exact_batch_f64's.
 * sobol_v (HOST [30][3*n_steps], hmc_sobol_init_directions layout) or NULL:
 * with uniforms == NULL the Sobol points are generated on the device --
 * run r, path p uses point 1 + r*sobol_n_paths + p (engine.py:100), or with
 * sobol_scramble points 1..N under per-(run, dimension) digital shifts;
 * identical to passing the same points as uniforms. */
int hmc_exact_runs_f64(const hmc_model* model, double s0, const double* step_times,
                       int32_t n_steps, const int64_t* avg_flags, int64_t path_lo,
                       int64_t path_hi, const uint64_t* key_runs, int32_t n_runs,
                       const double* uniforms, const uint32_t* sobol_v, int32_t sobol_scramble,
                       int64_t sobol_n_paths, double* out, int32_t device);

/* The exact scheme's engine path (engine._run_sums with scheme="exact",
 * engine.py:71-116) on the device: for the chunk-aligned slice
 * [sim->path_lo, sim->path_hi) of every run, the base simulation and (with
 * sim->want_greeks) the v0 +- and -- for Asians -- r +- re-simulations on
 * the same streams, the per-path estimators of hmc_greeks (Rho-FD of a
 * European by exact e^{+-h T} rescaling) and per-chunk partials
 * d_chunks[run][chunk][HMC_NW] (DEVICE) in the same layout as
 * hmc_greeks_chunks, so hmc_reduce_chunks and multi-GPU gathers apply
 * unchanged.  step_times / avg_flags as hmc_exact_batch_f64; sampler pseudo
 * (reference stream) or sobol (sim->sobol_v, on-device points).  Runs on
 * `stream`, synchronous on return (numerical failures are reported like
 * hmc_exact_batch_f64's). */
int hmc_exact_greeks_chunks(const hmc_model* model, const hmc_product* product, const hmc_sim* sim,
                            const double* step_times, int32_t n_steps, const int64_t* avg_flags,
                            double* d_chunks, void* stream);

/* Joe-Kuo direction numbers as used by scipy.stats.qmc.Sobol(scramble=False)
 * (30 bits): poly[dim], vinit[dim][18] from scipy's
 * _sobol_direction_numbers.npz -> v_out[30][dim] (HOST).  Point n of the
 * Gray-code sequence is x_d(n) = 2^-30 * XOR_{b : bit b of n^(n>>1)} v[b][d]. */
int hmc_sobol_init_directions(const int64_t* poly, const int64_t* vinit,
                              int32_t dim, uint32_t* v_out);

/* Device Philox4x32-10 (fixed key 0xA4093822, 0x299F31D0 -- the production
 * stream's key) on n HOST counters ctr[n][4] -> out[n][4]; for known-answer
 * tests of the exact device code path.  Synchronous. */
int hmc_philox_check(const uint32_t* ctr, int32_t n, uint32_t* out, int32_t device);

/* The fp32 production step arithmetic (state, Milstein/Euler update,
 * fixings, CRN trajectories, per-path estimators -- the code of
 * hmc_greeks_chunks' kernel) driven by GIVEN standard normals: HOST
 * normals[n][n_sim][2] = (z1, z2), z2 independent of z1 (correlated inside
 * as the kernels do), n_sim = the last fixing index; out: HOST
 * [n][HMC_NQ] per-path quantities.  Known-answer parity of the fp32 path
 * against the fp64 oracle on identical shocks.  Synchronous. */
int hmc_fp32_paths_check(const hmc_model* model, const hmc_product* product, const hmc_sim* sim,
                         const float* normals, int64_t n, double* out, int32_t device);

/* The fp32 kernels' Box-Muller on n HOST Philox blocks words[n][4] ->
 * out[n][6]: the three standard-normal pairs (z1, z2) the production step
 * loop draws from one block (radius from the top 23 bits of w0/w1/w2,
 * angles from w3 and the low bits; hmc_path32.cuh tri_unpack).  Known-answer
 * and distribution tests of the device code path.  Synchronous. */
int hmc_box_muller_check(const uint32_t* words, int32_t n, float* out, int32_t device);

/* The fp32 kernels' Sobol quantile z = Phi^-1(u) on n HOST 30-bit
 * coordinates x[n] (u = x 2^-30, or (x + 1/2) 2^-30 when scrambled) ->
 * out[n]; known-answer tests of the device code path.  Synchronous. */
int hmc_sobol_quantile_check(const uint32_t* x, int32_t n, int32_t scrambled, float* out,
                             int32_t device);

/* Key derivation of the reference RNG (rng.py:46-52), for hosts that
 * build key_run for hmc_discretised_batch_f64. */
/* The reference's random-number and step primitives, elementwise on the
 * device -- the same device functions the fp64 replay kernels run (built
 * with -fmad=false).  All buffers HOST, synchronous.  They serve the
 * drop-in's rng / schemes modules:
 *   hmc_uniforms_f64  <- rng.uniform_at / uniforms_at / _uniform_keys
 *                        (rng.py:63-74, 356-361): out[i] = draw draws[i] of
 *                        the stream keys[n_keys == 1 ? 0 : i]
 *   hmc_ndtri_f64     <- rng.inverse_normal_cdf (rng.py:95-132; Acklam +
 *                        one Halley step, _core.pyx:75-109)
 *   hmc_steps_f64     <- schemes.euler_step / milstein_step (schemes.py:33-61,
 *                        _core.pyx:399-404): one full-truncation step of each
 *                        state (s[i], v[i]) from its two uniforms u[i][0]
 *                        (asset) and u[i][1] (variance), correlated as
 *                        rng.correlated_pair (rng.py:226-235) */
int hmc_uniforms_f64(const uint64_t* keys, int64_t n_keys, const uint64_t* draws, int64_t n,
                     double* out, int32_t device);
int hmc_ndtri_f64(const double* u, int64_t n, double* out, int32_t device);
/* rng.gamma_batch / sample_gamma (rng.py:238-262, 308-343; _core.pyx:116-136):
 * Marsaglia-Tsang Gamma(shape, scale) from draw start[i] of stream keys[i];
 * used[i] = draws consumed (the exact kernel's own sampler) */
int hmc_gamma_f64(const uint64_t* keys, const uint64_t* start, int64_t n, double shape,
                  double scale, double* out, uint64_t* used, int32_t device);
int hmc_steps_f64(const hmc_model* model, int32_t milstein, double dt, const double* s,
                  const double* v, const double* u, int64_t n, double* s_out, double* v_out,
                  int32_t device);

/* The reference's exact-scheme host modules, elementwise on the device --
 * the exact kernel's own routines (hmc_exact.cu, -fmad=false).  All buffers
 * HOST, synchronous; errors HMC_E_BESSEL / HMC_E_QUAD / HMC_E_ROOT as the
 * reference raises them.  They serve the drop-in's bessel / ivlaw / exact
 * modules:
 *   hmc_bessel_f64     <- bessel.bessel_i_series / bessel_i_series_vec
 *                         (mode HMC_BESSEL_SERIES), bessel_i (HMC_BESSEL_I),
 *                         bessel_i_ratio (HMC_BESSEL_RATIO: z = coeff_num,
 *                         aux[i] = {coeff_den, w, log_coeff_ratio re, im},
 *                         re = NaN for the principal log) (bessel.py:26-82,
 *                         _core.pyx:143-159); z, out: [n][2] (re, im)
 *   hmc_ivlaw_phi_f64  <- ivlaw.characteristic_fn_raw / _characteristic_fn_vec
 *                         (ivlaw.py:50-108, _core.pyx:162-188): Phi(a[i])
 *   hmc_ivlaw_eval_f64 <- ivlaw.IntegratedVarianceLaw (ivlaw.py:111-308,
 *                         _core.pyx:195-310): info = {mean, std, h, nodes}
 *                         (HMC_IVLAW_INFO, n may be 0), cdf_raw / cdf /
 *                         inverse_cdf of in[i] (HMC_IVLAW_CDF_RAW / _CDF /
 *                         _INVERSE)
 *   hmc_exact_step_f64 <- exact.variance_transition (full = 0) / exact_step
 *                         (full = 1) (exact.py:38-88): draws[i] = {z1, gamma,
 *                         u_iv, z3} -> out[i] = {s_t, v_t, integrated var} */
enum { HMC_BESSEL_SERIES = 0, HMC_BESSEL_I = 1, HMC_BESSEL_RATIO = 2 };
enum { HMC_IVLAW_INFO = 0, HMC_IVLAW_CDF_RAW = 1, HMC_IVLAW_CDF = 2, HMC_IVLAW_INVERSE = 3 };
int hmc_bessel_f64(int32_t mode, double nu, const double* z, const double* aux, int64_t n, double* out,
                   int32_t device);
int hmc_ivlaw_phi_f64(const hmc_model* model, double v_u, double v_t, double dt, const double* a, int64_t n,
                      double* out, int32_t device);
int hmc_ivlaw_eval_f64(const hmc_model* model, double v_u, double v_t, double dt, int32_t mode,
                       const double* in, int64_t n, double* out, double* info, int32_t device);
int hmc_exact_step_f64(const hmc_model* model, int32_t full, double s_u, double v_u, double dt,
                       const double* draws, int64_t n, double* out, int32_t device);

uint64_t hmc_root_key(uint64_t seed);
uint64_t hmc_derive_key(uint64_t parent, uint64_t index);

#ifdef __cplusplus
}
#endif
#endif /* HMC_H_ */
