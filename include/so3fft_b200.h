/*
 * so3fft_b200 -- C ABI of the B200-native FSOFT / iFSOFT (Kostelec-Rockmore SO(3) FFT).
 *
 * Drop-in boundary for the reference Python package `so3fft` (arXiv 1808.00896,
 * /root/reference/pkg/src/so3fft).  The reference has no FFI of its own: its
 * operator interface is the Python surface re-exported by __init__.py:17-94.
 * Each entry point below names the reference function it replaces (file:line,
 * relative to pkg/src/so3fft).  The Python mirror
 * `paper_1808_00896_b200` binds these with ctypes.
 *
 * Data: complex128 as interleaved (re, im) float64 pairs, little endian.
 *   samples      : (2B)^3 per function, C order over [i = alpha][j = beta][k = gamma]
 *                  (core.py:148-176, So3SampleGrid)
 *   coefficients : B(4B^2-1)/3 per function, l-major, slot(l,m,m') =
 *                  l(4l^2-1)/3 + (m+l)(2l+1) + (m'+l)   (core.py:54-61, So3Coefficients)
 *   batch        : functions are consecutive (stride (2B)^3 resp. B(4B^2-1)/3).
 * Pointers marked `dev` are CUDA device pointers on the plan's device; `host`
 * pointers are ordinary host memory.  `stream` is a cudaStream_t (NULL = legacy
 * default stream).  Every call is asynchronous on `stream` unless noted.
 *
 * Errors: every function returns SO3_OK (0) or a nonzero status; the message of
 * the last failure on the calling thread is so3_last_error().  SO3_ERR_INVALID
 * corresponds to the reference's ValueError (bad bandwidth, size or argument).
 *
 * Plans and concurrency: a plan is read-only tables PLUS per-plan scratch (the FFT
 * intermediate, the pair-major spectrum, the split-analysis partial sums and counters,
 * the host-path staging buffers).  For B a multiple of 64 the tables include the checkpoint
 * table of the segment-parallel DWT (8 recurrence states per cluster and beta index:
 * 8 x 2B x 16 bytes x B(B+1)/2 clusters, 17.2 GB at B = 512; if that allocation fails the plan
 * keeps the kernels that need no table).  Every transform on one plan uses that scratch, so calls
 * on ONE plan must be stream-ordered: issue them on one stream, or order the streams
 * yourself (events).  Different plans are independent and may run concurrently on any
 * streams or threads.  (The reference TransformPlan is immutable and may be shared; give
 * each concurrent stream its own plan here.)  No call allocates device memory except
 * so3_plan_create*, so3_plan_set_knob("ana_split" / "dwt_seg" / "seg_ana_w") and the first call of a *_host entry
 * point, so the device entry points can be captured into a CUDA graph.
 */
#ifndef SO3FFT_B200_H
#define SO3FFT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SO3_OK 0
#define SO3_ERR_INVALID 1   /* ValueError in the reference */
#define SO3_ERR_CUDA 2      /* CUDA runtime / launch failure */
#define SO3_ERR_NOMEM 3     /* device or host allocation failed */

typedef struct so3_plan_s* so3_plan_t;

/* Message of the last failure on this thread ("" if none). */
const char* so3_last_error(void);

/* Library version string. */
const char* so3_version(void);

/* ---- host-only helpers (no GPU needed) ------------------------------------ */

/* coeff_count (core.py:48-51): B(4B^2-1)/3; 0 for B < 1. */
int64_t so3_coeff_count(int bandwidth);

/* grid_size(B)^3 (core.py:43-45): (2B)^3; 0 for B < 1. */
int64_t so3_grid_count(int bandwidth);

/* coeff_index (core.py:54-61); -1 if (l, m, m') is outside the band. */
int64_t so3_coeff_index(int l, int m, int mp, int bandwidth);

/* quadrature_weights (quadrature.py:66-73): w_B(j), j < 2B, into host out[2B]. */
int so3_quadrature_weights(int bandwidth, double* out_host);

/* sample_angles (quadrature.py:57-63): alpha_i (= gamma_i) and beta_j, host out[2B] each. */
int so3_sample_angles(int bandwidth, double* alphas_host, double* betas_host);

/* Number of symmetry clusters (schedule.py:136-158): 1 + 2(B-1) + (B-1)(B-2)/2. */
int64_t so3_cluster_count(int bandwidth);

/* The plan's cluster schedule: base pairs (m, m') as int32 pairs in launch order
 * (longest first), plus their member counts.  bases_host[2*count], members_host[count]
 * (either may be NULL).  Replaces enumerate_clusters / make_work_items
 * (schedule.py:136-178) as the unit of GPU work. */
int so3_cluster_schedule(int bandwidth, int32_t* bases_host, int32_t* members_host);

/* ---- plans ---------------------------------------------------------------- */

/* make_plan (soft.py:80-108) for `batch` functions on the current CUDA device.
 * 1 <= bandwidth <= 512 (SO3_ERR_INVALID otherwise: the DWT kernels hold at most
 * 2B = 1024 beta indices per cluster, and B = 1024 would need 3 x 137 GB of grids).
 * Builds the beta tables, quadrature weights, twiddles and the cluster schedule
 * on the host (long double), uploads them and allocates the plan's scratch
 * spectrum ((2B)^3 * batch complex128).  matrix_policy / partitioner of the
 * reference have no effect on results and are handled by the Python layer. */
int so3_plan_create(int bandwidth, int batch, so3_plan_t* out);
void so3_plan_destroy(so3_plan_t plan);
int so3_plan_bandwidth(so3_plan_t plan);
int so3_plan_batch(so3_plan_t plan);
int so3_plan_device(so3_plan_t plan);
/* Device bytes owned by the plan (tables + scratch). */
int64_t so3_plan_device_bytes(so3_plan_t plan);

/* ---- whole transforms ------------------------------------------------------ */

/* fsoft_sequential / fsoft_parallel (soft.py:124-149, 176-183):
 * samples_dev (batch x (2B)^3) -> coeffs_dev (batch x C(B)).  Inputs are not modified. */
int so3_fsoft(so3_plan_t plan, const void* samples_dev, void* coeffs_dev, void* stream);

/* ifsoft_sequential / ifsoft_parallel (soft.py:152-173, 186-193):
 * coeffs_dev -> samples_dev.  Inputs are not modified. */
int so3_ifsoft(so3_plan_t plan, const void* coeffs_dev, void* samples_dev, void* stream);

/* Same with HOST buffers: copies in, transforms, copies out, and synchronises
 * `stream` before returning (the reference API's numpy-in / numpy-out contract).
 * Device staging buffers are allocated on first use and kept by the plan.
 * Pinned (page-locked / registered) host buffers are copied directly; pageable buffers of
 * 64 MB or more go through the plan's pinned bounce buffers (2 x 16 MB per worker, one
 * worker thread per host core up to 16, allocated on the first pageable call), so the
 * host-side copies and first-touch page faults run in parallel with the DMA (hostio.cuh). */
int so3_fsoft_host(so3_plan_t plan, const void* samples_host, void* coeffs_host, void* stream);
int so3_ifsoft_host(so3_plan_t plan, const void* coeffs_host, void* samples_host, void* stream);

/* ---- stages (parity tests, per-stage timing, sharded pipeline) ------------ */

/* Forward torus stage: for every beta slice the sign +1 2-D DFT
 * (fft.py:72-76 via soft.py:130-132) times the quadrature weight w_j, written
 * pair-major: spectrum_dev[f][m' mod 2B][m mod 2B][j].  Entries at the Nyquist bin
 * (m = B or m' = B) hold unspecified values: the DWT never reads them. 
 * Uses the plan's pass-1 scratch; spectrum_dev must be a different buffer. */
int so3_fft_analysis(so3_plan_t plan, const void* samples_dev, void* spectrum_dev, void* stream);

/* Inverse torus stage: sign -1 2-D DFT per slice (soft.py:164-172) of
 * spectrum_dev[f][m'][m][j] (entries at the Nyquist bin B read as zero).
 * spectrum_dev is read only. */
int so3_fft_synthesis(so3_plan_t plan, void* spectrum_dev, void* samples_dev, void* stream);

/* Forward DWT (dwt.py:109-116 per member, soft.py:134-148) over clusters
 * [cluster_begin, cluster_end) of the schedule; reads the weighted spectrum written
 * by so3_fft_analysis and writes those clusters' coefficient slots. */
int so3_dwt_analysis(so3_plan_t plan, const void* spectrum_dev, void* coeffs_dev,
                     int64_t cluster_begin, int64_t cluster_end, void* stream);

/* Inverse DWT (dwt.py:119-125 per member, soft.py:157-167) over clusters
 * [cluster_begin, cluster_end): writes spectrum_dev[f][m'][m][j] of their pairs. */
int so3_dwt_synthesis(so3_plan_t plan, const void* coeffs_dev, void* spectrum_dev,
                      int64_t cluster_begin, int64_t cluster_end, void* stream);

/* DWT kernel family: SO3_DWT_MMA (default; FP64 DMMA m8n8k4 / m16n8k4) or SO3_DWT_SIMT (DFMA +
 * warp butterfly).  Same results to rounding. */
#define SO3_DWT_MMA 0
#define SO3_DWT_SIMT 1
int so3_plan_set_dwt_variant(so3_plan_t plan, int variant);
/* Tuning knobs (same results, different kernel shapes): "dwt_variant" (as above), "syn_jw"
 * (synthesis beta indices per warp, 0 = default), "fft_xb" (FFT rows per CTA for
 * 2B in {256, 512, 1024}, 0 = default), "dwt_batch" (1 = dense-contraction DWT for batched
 * plans with 2B <= 64, 0 = per-function kernels), "fft_fused" (1 = one-pass 2-D slice FFT for
 * 2B <= 64, 0 = two passes), "fft_tma" (1 = FFT tiles move their strided side by TMA tensor
 * copies: passes at 2B in {256, 512, 1024} and the one-pass slices; 0 = per-thread loads and
 * stores; bit-identical), "fft_bulkin" / "fft_bulkout" (the TMA passes' row side by 1-D bulk
 * copies: 1 / 0, -1 = automatic), "fft_tab_loop" (x-tiles per CTA of the sharded row-table FFT
 * passes, 0 = one tile per CTA), "fft_tab_tma" (row-table passes' plain side by bulk copies).
 * "ana_split" (analysis of a cluster over two 4-warp CTAs that combine their halves in a
 * fixed order: 0 = off (one CTA per cluster), 1 = on at 2B = 1024 (default), >= 2 = on at
 * 2B = 512 and 1024; same results to rounding, deterministic; turning it on allocates the
 * partial-sum scratch, 2 x 8 x sum_clusters(B - m) complex128).  "dwt_seg" (segment-parallel
 * DWT kernels, csrc/dwt_seg.cuh, where B % 64 == 0; bits: 1 = synthesis (default), 2 = analysis
 * with one CTA per cluster part, 4 = persistent analysis with bulk-copy operand prefetch on
 * single-device one-function plans; 0 = dwt_mma.cuh kernels; same results to rounding,
 * deterministic; default 1, and 1 | 4 at B = 320 .. 512, where the persistent analysis is 6-9 %
 * faster than dwt_analysis_mma_cta_kernel; at B <= 256 that kernel is as fast and stays; the
 * persistent kernel keeps one CTA with ~222 KB of shared memory on every SM for its duration, so
 * kernels of other streams do not run beside it), "seg_ana_w" (warps per CTA of those analysis variants, 4 or 8).
 * Experiment knobs (same results,
 * measured slower or equal): "fft_persist" (> 0: the
 * TMA passes as that many persistent double-buffered CTAs), "fft_pad" / "dwt_pad" (extra KB of
 * shared memory per FFT / MMA DWT CTA), "carveout" (preferred shared-memory carveout of the
 * big kernels, -1 = driver default; a per-kernel CUDA attribute, re-set by each plan's calls).
 * All knobs are per plan.  Unknown names fail with SO3_ERR_INVALID. */
int so3_plan_set_knob(so3_plan_t plan, const char* name, int value);

/* Pair-major spectrum buffer owned by the plan (device pointer, batch x (2B)^3 complex128). */
void* so3_plan_scratch(so3_plan_t plan);

/* ---- sharded pipeline (one process per GPU) -------------------
 * G ranks split the torus FFT by beta slab [rank*J, (rank+1)*J), J = 2B/G, and the DWT by
 * cost-balanced cluster groups (longest-processing-time greedy over the schedule); an
 * all-to-all per direction joins them (the reference's in-memory transpose spectrum[m, j, m'],
 * soft.py:131-132, 142, 167).  The exchange is split into K chunks: each rank's cost-sorted
 * cluster list is cut into K runs of equal DWT cost, and every layout is chunk-major so one
 * chunk is one contiguous all-to-all (its exchange overlaps the DWT of the previous / next
 * chunk).  Buffers (complex128):
 *   slab     : [i][jj][k], 2B x J x 2B (this rank's samples; grid[:, jbase:jbase+J, :])
 *   layout A : rows [chunk q][rank g][pairs_{g,q}][J]  (forward send / inverse recv,
 *              total (2B-1)^2 * J)
 *   layout B : rows [chunk q][rank h][pairs_{rank,q}][J] (forward recv / inverse send,
 *              G * pairs_rank * J); chunk q starts at row G * sum_{q' < q} pairs_{rank,q'}
 *   coeffs   : full l-major array; a rank writes (forward) / reads (inverse) only its slots.
 *   exchange : ONE buffer holding layout A (rows [0, (2B-1)^2)) followed by layout B.  The
 *              rank's own block (g = h = rank of every chunk) exists in layout B only: the
 *              forward FFT stores the own pairs straight into layout B and the inverse FFT
 *              reads them from there, so the all-to-all moves the other ranks' blocks only
 *              (no self copy; the layout-A rows of the own block are left unused).
 * Results are identical, bit for bit, for every G and K (the same per-row FFTs and
 * per-cluster reductions run whatever the split).  K = 1 is the unchunked exchange. */
int so3_shard_plan_create(int bandwidth, int world, int rank, so3_plan_t* out);      /* K = 1 */
int so3_shard_plan_create_chunked(int bandwidth, int world, int rank, int chunks, so3_plan_t* out);
int64_t so3_shard_slab_width(so3_plan_t plan);             /* J */
int64_t so3_shard_rank_pairs(so3_plan_t plan);             /* pairs_rank */
int64_t so3_shard_chunks(so3_plan_t plan);                 /* K */
/* host only: pairs per rank [world]; cluster owner per schedule entry; a rank's pairs (m, m')
 * in layout order (chunk by chunk); pairs per (chunk, rank) [chunks][world] */
int so3_shard_pair_counts(int bandwidth, int world, int64_t* pairs_per_rank);
int so3_shard_cluster_owner(int bandwidth, int world, int32_t* owner);
int so3_shard_pair_list(int bandwidth, int world, int rank, int32_t* pairs);
int so3_shard_chunk_pairs(int bandwidth, int world, int chunks, int64_t* pairs);
/* forward: slab -> exchange buffer (K1a + K1b with the pack fused into the store): other
 * ranks' pairs into layout A, the own pairs into layout B */
int so3_shard_fft_analysis(so3_plan_t plan, const void* slab_dev, void* exchange_dev, void* stream);
/* forward: layout B -> this rank's coefficient slots */
int so3_shard_dwt_analysis(so3_plan_t plan, const void* recv_dev, void* coeffs_dev, void* stream);
/* inverse: this rank's coefficient slots -> layout B */
int so3_shard_dwt_synthesis(so3_plan_t plan, const void* coeffs_dev, void* send_dev, void* stream);
/* one chunk q: recv_chunk / send_chunk point at chunk q of layout B ([h][pairs_{rank,q}][J]) */
int so3_shard_dwt_analysis_chunk(so3_plan_t plan, int chunk, const void* recv_chunk_dev, void* coeffs_dev,
                                 void* stream);
int so3_shard_dwt_synthesis_chunk(so3_plan_t plan, int chunk, const void* coeffs_dev, void* send_chunk_dev,
                                  void* stream);
/* inverse: exchange buffer -> slab (K4a with the unpack fused into the load, K4b): other
 * ranks' pairs from layout A, the own pairs from layout B */
int so3_shard_fft_synthesis(so3_plan_t plan, const void* exchange_dev, void* slab_dev, void* stream);

/* Direct O(B^6) transforms (fsoft_direct / ifsoft_direct, soft.py:212-256): the defining
 * sums over closed-form Wigner functions (wigner.py:78-114), sharing nothing with the fast
 * path; an independent cross-check for small B (1 <= B <= 64).  Synchronous on `stream`. */
int so3_fsoft_direct(int bandwidth, const void* samples_dev, void* coeffs_dev, void* stream);
int so3_ifsoft_direct(int bandwidth, const void* coeffs_dev, void* samples_dev, void* stream);

/* ---- SOFC / SOFG containers (core.py:179-225), streamed ------------------------------
 * The reference's byte format: magic "SOFC" / "SOFG", u32 version 1, u32 bandwidth, then the
 * complex128 payload (l-major coefficients / [i][j][k] samples), little endian.
 * kind: 0 = SOFC coefficients, 1 = SOFG samples.  For samples, [jbase, jbase + J) selects a
 * beta slab, transferred as [i][jj][k] (J = 0: the whole grid); coefficients ignore both.
 * Device transfers stream whole [i][jj][k] rows through two pinned bounce buffers of
 * `staging_bytes` each (so a 17 GB grid never needs a host copy); host transfers read or write
 * the caller's buffer directly.  Non-finite payloads are rejected on read and write, as by the
 * reference (checked on the device for device buffers).  Synchronous on `stream`.
 * Sharded writers: rank 0 creates the file (create = 1, sized in full), the other ranks then
 * write their slabs with create = 0. */
int so3_container_info(const char* path, int* kind, int* bandwidth, int64_t* elements);
int so3_read_container(const char* path, int kind, int jbase, int J, void* dst, int dst_on_device,
                       int64_t staging_bytes, void* stream);
int so3_write_container(const char* path, int kind, int bandwidth, int jbase, int J, const void* src,
                        int src_on_device, int create, int64_t staging_bytes, void* stream);

/* ---- Wigner utilities at arbitrary angles (the reference's wigner.py surface) ----------
 * One thread per point; beta_dev / x_dev / out_dev are device arrays of `count` doubles
 * (rows: (B-L) x count).  Argument checks as the reference (ValueError -> SO3_ERR_INVALID);
 * the caller checks beta in [0, pi] and |x| <= 1 as wigner.py:71-76 / 53-54. */
/* jacobi_poly (wigner.py:43-68) */
int so3_jacobi_eval(int n, double a, double b, const double* x_dev, int64_t count, double* out_dev, void* stream);
/* wigner_d_direct (wigner.py:92-114): closed form after canonicalisation to m' >= |m| */
int so3_wigner_d_eval(int l, int m, int mp, const double* beta_dev, int64_t count, double* out_dev, void* stream);
/* wigner_d_rows (wigner.py:139-178): seed (wigner.py:117-136) + three-term recurrence,
 * out_dev[(l - L) * count + i], L = max(|m|, |m'|) */
int so3_wigner_rows_eval(int bandwidth, int m, int mp, const double* beta_dev, int64_t count, double* out_dev,
                         void* stream);

/* Wigner rows d^l_{m,m'}(beta_j), l = max(|m|,|m'|)..B-1, j < 2B, for any pair
 * (wigner_d_rows, wigner.py:139-178 + derive_cluster_matrices, dwt.py:76-93):
 * out_dev[(l-L)*2B + j], generated by the same in-register recurrence as the DWT. */
int so3_wigner_rows(so3_plan_t plan, int m, int mp, double* out_dev, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SO3FFT_B200_H */
