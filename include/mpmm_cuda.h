/*
 * mpmm_cuda.h -- C ABI of libmpmm_cuda.so, the B200 (sm_100a) DD/QD GEMM
 * library that replaces the reference's compiled kernel module.
 *
 * Conventions (all entry points)
 * ------------------------------
 * - Matrices are row-major views of DD (2 doubles) or QD (4 doubles)
 *   elements, exactly the reference's C-contiguous float64 (rows, cols,
 *   comps) arrays (reference pkg/src/mpmm/matrix.py:20,43-48).  Leading
 *   dimensions (ld*) count ELEMENTS, not doubles.
 * - `comps` is 2 (double-double) or 4 (quad-double).
 * - Every function returns 0 on success or a nonzero MPMM_ERR_* code;
 *   mpmm_last_error() then holds a message (thread-local).  No C++
 *   exception crosses this boundary.  As in the reference, kernels never
 *   fail on overflow/NaN; the caller checks (multiply.py:124-127), here via
 *   the optional `nonfinite` device flag.
 * - Ownership: the caller allocates and owns every buffer; the library
 *   keeps no state between calls except the thread-local error text.
 * - Reentrant: concurrent calls on disjoint outputs are safe
 *   (multiply.py:99-112 relies on that for the reference kernels).
 * - Results are bit-identical to the reference CPU kernels for |x| < 2^996
 *   and no underflow of TwoProd error terms (reference eft.py:21-24).
 */
#ifndef MPMM_CUDA_H
#define MPMM_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPMM_ABI_VERSION 1

#define MPMM_OK 0
#define MPMM_ERR_ARG 1    /* bad argument (shape, comps, algo, range)     */
#define MPMM_ERR_CUDA 2   /* a CUDA runtime call failed                   */
#define MPMM_ERR_NODEV 3  /* no CUDA device                               */
#define MPMM_ERR_RANGE 4  /* operands not representable (exact tensor mode) */
#define MPMM_ERR_NONFINITE 5 /* non-finite operand or result (exact tensor mode) */

#define MPMM_ALGO_SIMPLE 0
#define MPMM_ALGO_BLOCK 1
/* Opt-in faithful DD sequence (15 FP64 instructions per multiply-add)
 * within the north_star bound 4 l u (|A||B|)_ij, u = 2^-104; NOT
 * bit-identical to the reference.  DD only. */
#define MPMM_ALGO_BLOCK_FAST 2
/* Strassen (reference matmul_strassen, multiply.py:267-338): n_min is the
 * leaf block size, `cutoff` the recursion threshold. */
#define MPMM_ALGO_STRASSEN 3

int mpmm_abi_version(void);
const char *mpmm_last_error(void);
/* Select the device subsequent calls on this host thread use (the library
 * links its own CUDA runtime, so a caller's cudaSetDevice in another
 * runtime instance is mirrored here; the Python binding does it). */
int mpmm_set_device(int device);
/* Number of visible CUDA devices (0 without a GPU; never an error). */
int mpmm_device_count(int *count);
/* The CTA tile a reference block size n_min selects. */
int mpmm_tile_for_nmin(int64_t n_min, int *tile, int *super_tiles);
/* Launch geometry on the current device: CTA output tile, threads per CTA,
 * resident CTAs per SM and the SM count -- the inputs of the wave-aware
 * time predictor (predict.py; reference predict.py:37-50 assumes a CPU). */
int mpmm_gemm_geometry(int comps, int algo, int64_t n_min, int *tile_m, int *tile_n,
                       int *threads, int *ctas_per_sm, int *sm_count);

/* ---------------------------------------------------------------------------
 * Reference kernel-module protocol on HOST pointers
 * (reference _kernels.pyx:36-452; consumed at multiply.py:140-145,
 * :154-159, :195-200).  Each call copies its inputs to the current device,
 * computes, copies the written rows back and synchronises.  a is (m,l),
 * b is (l,n), c is (m,n), x/y/out are (rows,cols), all C-contiguous.
 * ------------------------------------------------------------------------- */

/* _kernels.pyx:36-100: rows [i0,i1) of c = a*b (accumulator from zero). */
int mpmm_dd_simple_rows(const double *a, const double *b, double *c, int64_t m, int64_t l,
                        int64_t n, int64_t i0, int64_t i1);
/* _kernels.pyx:344-363 */
int mpmm_qd_simple_rows(const double *a, const double *b, double *c, int64_t m, int64_t l,
                        int64_t n, int64_t i0, int64_t i1);
/* _kernels.pyx:103-186: cells [cell0,cell1) of the ceil(m/n_min) x
 * ceil(n/n_min) block grid, flattened row-major, ACCUMULATED INTO c. */
int mpmm_dd_block_cells(const double *a, const double *b, double *c, int64_t m, int64_t l,
                        int64_t n, int64_t n_min, int64_t cell0, int64_t cell1);
/* _kernels.pyx:366-404 */
int mpmm_qd_block_cells(const double *a, const double *b, double *c, int64_t m, int64_t l,
                        int64_t n, int64_t n_min, int64_t cell0, int64_t cell1);
/* _kernels.pyx:207-230 / :407-452: rows [i0,i1) of out = x +/- y. */
int mpmm_dd_ewise_add(const double *x, const double *y, double *out, int64_t rows,
                      int64_t cols, int64_t i0, int64_t i1);
int mpmm_dd_ewise_sub(const double *x, const double *y, double *out, int64_t rows,
                      int64_t cols, int64_t i0, int64_t i1);
int mpmm_qd_ewise_add(const double *x, const double *y, double *out, int64_t rows,
                      int64_t cols, int64_t i0, int64_t i1);
int mpmm_qd_ewise_sub(const double *x, const double *y, double *out, int64_t rows,
                      int64_t cols, int64_t i0, int64_t i1);

/* Whole product on HOST buffers: c (m x n) = a*b (accumulate=0) or
 * c += a*b (accumulate=1), computed on the current device.  When a, b and
 * c are all page-locked (blocked algorithm, accumulate=0) it is ONE GEMM
 * launch that consumes 64-column k-panels of a and b as their H2D copies
 * land and writes c straight into the page-locked buffer; otherwise the
 * H2D copies are split into k-panels on a copy stream so the GEMM of one
 * panel overlaps the copy of the next.  Same bits either way.  nonfinite
 * (host int, may be NULL) receives 1 when an output component is not
 * finite (multiply.py:124-127). */
int mpmm_gemm_host(int comps, int algo, int64_t n_min, int64_t m, int64_t l, int64_t n,
                   const double *a, const double *b, double *c, int accumulate, int *nonfinite);

/* ---------------------------------------------------------------------------
 * Device-resident entry points: all matrix pointers are DEVICE pointers on
 * the current device, `stream` is a cudaStream_t (NULL = legacy default).
 * Asynchronous: they enqueue work and return.
 * ------------------------------------------------------------------------- */

/* C = A*B (accumulate=0) or C += A*B (accumulate=1), m x n output,
 * inner dimension l.  algo MPMM_ALGO_SIMPLE (reference matmul_simple,
 * multiply.py:163-168) or MPMM_ALGO_BLOCK with block size n_min
 * (matmul_block, multiply.py:171-182).  nonfinite: optional device int,
 * OR-ed with 1 when an output component is not finite. */
int mpmm_gemm_dev(int comps, int algo, int64_t n_min, int64_t m, int64_t l, int64_t n,
                  const double *A, int64_t lda, const double *B, int64_t ldb, double *C,
                  int64_t ldc, int accumulate, int *nonfinite, void *stream);

/* Batched form of mpmm_gemm_dev: `batch` independent problems of one
 * shape, described by a DEVICE array of `batch` records of six 64-bit
 * words {A, B, C, lda, ldb, ldc} (pointers, then element leading dims).
 * Used for the 7^d leaf products of a Strassen recursion
 * (multiply.py:293-332) so they fill the GPU in one launch. */
int mpmm_gemm_batched_dev(int comps, int algo, int64_t n_min, int64_t batch, int64_t m,
                          int64_t l, int64_t n, const void *problems, int accumulate,
                          int *nonfinite, void *stream);

/* The reference's cell-range protocol on device pointers
 * (_kernels.pyx:103-186 / :366-404): cells [cell0,cell1) accumulate into C. */
int mpmm_block_cells_dev(int comps, int64_t n_min, int64_t cell0, int64_t cell1, int64_t m,
                         int64_t l, int64_t n, const double *A, int64_t lda, const double *B,
                         int64_t ldb, double *C, int64_t ldc, void *stream);

/* O = ((X sy*Y) sz*Z) sw*W elementwise for nops = 1..3 chained reference
 * ewise ops (signs +1/-1; Z/W unused below their nops).  Strassen's operand
 * sums and quadrant combinations (multiply.py:313-337). */
int mpmm_ewise_dev(int comps, int nops, int64_t rows, int64_t cols, const double *X,
                   int64_t ldx, const double *Y, int64_t ldy, int sy, const double *Z,
                   int64_t ldz, int sz, const double *W, int64_t ldw, int sw, double *O,
                   int64_t ldo, void *stream);

/* Batched form of mpmm_ewise_dev: a DEVICE array of `batch` records of 14
 * 64-bit words {X, Y, Z, W, O, ldx, ldy, ldz, ldw, ldo, nops, sy, sz, sw}
 * sharing rows x cols (one Strassen level's operand sums or combinations). */
int mpmm_ewise_batched_dev(int comps, int64_t batch, int64_t rows, int64_t cols,
                           const void *problems, void *stream);

/* multiply.py:124-127 _check_finite on the device: *flag |= 1 if any
 * component of the rows x cols view X is not finite. */
int mpmm_nonfinite_dev(int comps, int64_t rows, int64_t cols, const double *X, int64_t ldx,
                       int *flag, void *stream);

/* Exact componentwise verification: for `count` sampled
 * outputs (idx_i[s], idx_j[s]) (device int64 arrays) writes
 *   ratio[s] = |c_ij - (AB)_ij| / (4 l 2^-u_exp (|A||B|)_ij)
 * with (AB)_ij evaluated exactly in a fixed-point superaccumulator; <= 1
 * means the north_star bound holds (u_exp 104 for DD, 209 for QD).  NaN
 * marks a sample whose TwoProd error terms could underflow. */
int mpmm_exact_check_dev(int comps, int64_t m, int64_t l, int64_t n, const double *A,
                         int64_t lda, const double *B, int64_t ldb, const double *C, int64_t ldc,
                         const int64_t *idx_i, const int64_t *idx_j, int64_t count, int u_exp,
                         double *ratio, void *stream);

/* Seeded BASELINE inputs generated on the device, bitwise equal to the
 * numpy spec (paper_1710_01839_b200/inputs.py): the PCG64
 * stream (128-bit state/increment as hi/lo words, as numpy's
 * bit_generator.state reports them) starting at draw `first_draw`
 * supplies comps * rows * cols uniforms, assembled into a (rows, cols)
 * DD (comps 2) or QD (comps 4) matrix at `out`. */
int mpmm_gen_inputs_dev(int comps, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                        uint64_t inc_lo, uint64_t first_draw, int64_t rows, int64_t cols,
                        double *out, void *stream);

/* ---------------------------------------------------------------------------
 * Exact int8 tensor-core mode (ozaki.cu; orchestrated by tensor.py).  The
 * product of scaled-integer DD/QD operands is rebuilt exactly from int8
 * residue GEMMs modulo the 54 pairwise-coprime prime powers <= 256 (CRT),
 * then rounded once to DD/QD.  Not bit-identical to the reference (it is
 * the exact product, correctly rounded).
 * ------------------------------------------------------------------------- */
/* One pass over X (rows x cols DD/QD, leading dim ld): per row (by_cols 0) or column (1) and per
 * component c, EL[c*odim + o] = max exponent E with |x| < 2^E and
 * EL[(comps + c)*odim + o] = min weight exponent L of the lowest set bit
 * over the nonzero entries (-100000 / 100000 when none); bit 0 of *status
 * is set when any component is not finite. */
int mpmm_oz_scan_dev(int by_cols, int comps, int64_t rows, int64_t cols, const double *X,
                     int64_t ld, int *EL, int *status, void *stream);
/* int8 residues of sum_{c0<=c<c1} x_c * 2^shift[row|col] (an integer of
 * fewer than 32*words - 1 bits, two's complement) modulo the first nmod
 * moduli: by_cols 0 -> R[t*rplane + row*rpitch + k], by_cols 1 ->
 * R[t*rplane + col*rpitch + k] (k contiguous; rpitch a multiple of 4;
 * whole 4-byte groups are written, zeros past the matrix edge).
 * words <= 12. */
int mpmm_oz_residues_dev(int by_cols, int comps, int c0, int c1, int64_t rows, int64_t cols,
                         const double *X, int64_t ld, const int *shift, int nmod, int words,
                         int8_t *R, int64_t rpitch, int64_t rplane, void *stream);
/* The exact tensor mode in one call: C = A*B (device pointers, dense C with
 * ldc == n) as the exact product rounded once to comps doubles, on the
 * int8 tensor cores.  Synchronous (returns after the product, whose status
 * it reads).  The plan is cached per (device, stream, shape) and reused
 * speculatively with a device-side width check (recomputed when it does
 * not fit); intermediates up to 1 GiB stay cached, and a call with the same
 * A/B/C addresses as the previous one replays the whole device side as a
 * CUDA graph.  MPMM_ERR_NONFINITE for non-finite operands or an
 * overflowing result, MPMM_ERR_RANGE when the operands' dynamic range does
 * not fit the 54 moduli. */
int mpmm_gemm_exact_dev(int comps, int64_t m, int64_t l, int64_t n, const double *A,
                        int64_t lda, const double *B, int64_t ldb, double *C, int64_t ldc,
                        void *stream);
/* tcgen05 residue GEMMs: R_t = (A_t * Bt_t^T) mod p_t for the first batch
 * moduli, A_t m x k and Bt_t n x k int8 (k contiguous, planes m*k / n*k),
 * R_t m x n uint8 row-major (plane m*n); the int32 accumulator stays in
 * TMEM.  m % 128 == 0, n % 256 == 0, k % 128 == 0, k <= 131071. */
int mpmm_residue_gemm_dev(int64_t m, int64_t n, int64_t k, int64_t batch, const int8_t *A,
                          const int8_t *Bt, uint8_t *R, void *stream);
/* Free every cached exact-mode plan, workspace and graph. */
int mpmm_exact_release(void);
/* Host-only planner of the exact tensor mode: from the scan arrays of A
 * (ela, 2*comps*m ints) and B (elb, 2*comps*n ints) choose the cheapest
 * feasible component split.  Outputs: *na ranges of A in ranges_a[2*na]
 * (c0, c1) with their row shifts in shift_a[na*m] (na <= 4), likewise B;
 * *njobs (<= 16) jobs of 8 ints {a_range, b_range, moduli N, limbs K (one
 * for all jobs), words_a, words_b, beta_a, beta_b}.  MPMM_ERR_RANGE when
 * no split fits the 54 moduli.  No device work. */
int mpmm_oz_plan(int comps, int64_t m, int64_t n, int64_t l, const int *ela, const int *elb,
                 int *njobs, int *jobs, int *na, int *ranges_a, int *shift_a, int *nb,
                 int *ranges_b, int *shift_b);
/* batch x (C_t = A_t * Bt_t^T): A_t m x k, Bt_t n x k (row-major int8),
 * C_t m x n row-major int32, exact for k <= 131071 (cuBLASLt IMMA); m, n,
 * k multiples of 16. */
int mpmm_int8_gemm_batched_dev(int64_t m, int64_t n, int64_t k, int64_t batch, const int8_t *A,
                               const int8_t *Bt, int32_t *C, void *workspace, int64_t ws_bytes,
                               void *stream);
/* CRT reconstruction of njobs <= 16 jobs given as a HOST array of 56-byte
 * records {G, srow, scol, table: device pointers; N, K: int32; gpitch,
 * gplane: int64} (passed to the kernel by value), exact sum, rounding to
 * comps doubles per entry of C (m x n); *status |= 1 non-finite, 2
 * window overflow. */
int mpmm_oz_combine_dev(int comps, const void *jobs, int njobs, int64_t m, int64_t n, double *C,
                        int *status, void *stream);
/* Device side of the planner: for nranges <= 4 component ranges (HOST
 * array ranges[2*nranges] of (c0, c1)) and the scan arrays EL of one
 * operand (odim rows/columns): shift[r*odim + o] = -min L (0 for an empty
 * row) and beta[r] = max(E - L) + 1 (atomic max; the caller zeroes beta). */
int mpmm_oz_shifts_dev(int comps, int nranges, const int *ranges, int64_t odim, const int *EL,
                       int *shift, int *beta, void *stream);

/* FP64 roofline micro-benchmark: blocks x threads threads each run 8
 * independent chains of `iters` DFMA (op 0) or DADD (op 1). */
/* C = A*B by the reference's Strassen recursion (multiply.py:267-338), bit
 * for bit: a node of size <= cutoff (all of m, l, n) is a leaf, computed by
 * the blocked kernel with block size leaf_n_min from a zero accumulator;
 * odd dimensions are zero-padded to even (multiply.py:206-260).  Square
 * inputs are the reference's algorithm; rectangular m x l x n halves each
 * dimension (the BASELINE config-3 extension).  Runs level-synchronously
 * (one batched launch per level and operand shape, one launch for all
 * leaves), depth first at the top when the scratch would exceed 60% of
 * free device memory.  stats: optional HOST int64[2] receiving the
 * reference's operation counts {multiplications, additions}
 * (multiply.py:322-331).  nonfinite: optional device flag as above. */
int mpmm_strassen_dev(int comps, int64_t cutoff, int64_t leaf_n_min, int64_t m, int64_t l,
                      int64_t n, const double *A, int64_t lda, const double *B, int64_t ldb,
                      double *C, int64_t ldc, int *nonfinite, int64_t *stats, void *stream);

/* ---------------------------------------------------------------------------
 * Multi-GPU runtime (single process).  The library owns, per
 * device, a compute stream, a communication stream and an NCCL
 * communicator.  Not needed by the Python package (one process per GPU
 * over torch.distributed, shard.py); for C/C++ callers.
 * ------------------------------------------------------------------------- */

/* Create the runtime over `ngpus` devices: devices[0..ngpus) or, when
 * devices is NULL, 0..ngpus-1.  Error if already initialized. */
int mpmm_init(int ngpus, const int *devices);
/* Destroy the communicators and streams (no-op when not initialized). */
int mpmm_finalize(void);
/* The runtime's device count (0 when not initialized) and ids. */
int mpmm_runtime_gpus(int *ngpus, int *devices, int cap);
/* c (m x n) = a*b from HOST buffers on the runtime's GPUs: C's rows are
 * split in 64-row-aligned blocks, one per GPU, each GPU receiving its rows
 * of a directly; b goes to the first GPU and is broadcast by NCCL in
 * `panels` k-panels (<= 0: automatic) overlapped with the per-panel GEMM.
 * algo SIMPLE / BLOCK / BLOCK_FAST (n_min) or STRASSEN (n_min = leaf block
 * size, cutoff; per-GPU rectangular Strassen).  Bitwise independent of the
 * GPU count and the panel split for SIMPLE/BLOCK.  nonfinite: optional
 * host int.  device_ms: optional, the max over GPUs of the device time
 * from the first copy to the last (CUDA events). */
int mpmm_gemm_multi(int comps, int algo, int64_t n_min, int64_t cutoff, int64_t m, int64_t l,
                    int64_t n, const double *a, const double *b, double *c, int64_t panels,
                    int *nonfinite, double *device_ms);

/* The schedule mpmm_gemm_multi uses, computed on the host (no GPU needed):
 * GPU g owns C rows [rows[2g], rows[2g+1]) -- ceil(m/ngpus) rounded up to
 * the 64-row CTA tile, trailing GPUs possibly empty --; B is broadcast in
 * *npanels k-panels [kb[p], kb[p+1]) (panels <= 0: automatic).  rows holds
 * 2*ngpus entries, kb max(l,1)+2.  Returns 0, or 1 on a bad request.
 * Replaces the reference's _split_range (multiply.py:86-96) lifted to GPUs. */
int mpmm_multi_plan(int64_t m, int64_t l, int ngpus, int64_t panels, int64_t *rows, int64_t *kb,
                    int *npanels);

/* ---------------------------------------------------------------------------
 * B shared over peer memory (one process per GPU): the alternative to the
 * NCCL broadcast.  The source rank allocates B's buffer with mpmm_ipc_alloc
 * (cudaMalloc + a CUDA IPC handle of mpmm_ipc_handle_size() bytes), the
 * other ranks map it with mpmm_ipc_open and pass the mapped pointer as B to
 * mpmm_gemm_dev: the GEMM reads B's tiles from the source GPU over NVLink
 * as it consumes them (no collective, same bits).  mpmm_ipc_close unmaps,
 * mpmm_ipc_free frees (source rank, after every mapping is closed).
 * Errors: MPMM_ERR_ARG / MPMM_ERR_CUDA, text in mpmm_peer_last_error().
 * ------------------------------------------------------------------------- */
int mpmm_ipc_handle_size(void);
/* init: optional source (device or host) copied into the new buffer */
int mpmm_ipc_alloc(int64_t bytes, const void *init, void **ptr, void *handle);
int mpmm_ipc_free(void *ptr);
int mpmm_ipc_open(const void *handle, void **ptr);
int mpmm_ipc_close(void *ptr);
const char *mpmm_peer_last_error(void);

/* Event timers on a stream (TimingPolicy's device clock, timing.py:22-59). */
int mpmm_timer_create(void **timer);
int mpmm_timer_start(void *timer, void *stream);
int mpmm_timer_stop(void *timer, void *stream);
/* Waits for the stop event; milliseconds between start and stop. */
int mpmm_timer_elapsed_ms(void *timer, float *ms);
int mpmm_timer_destroy(void *timer);

int mpmm_fp64_burn_dev(int op, int blocks, int threads, int64_t iters, double *scratch,
                       void *stream);

/* ---------------------------------------------------------------------------
 * Host-side verification helpers (reference matrix.py:207-294): Frobenius
 * norm and relative difference evaluated sequentially in DD/QD arithmetic,
 * exactly like the reference.  x, y: `count` elements of `comps` doubles.
 * Return 0, 1 on overflow (reference RangeError), 2 on a negative square.
 * ------------------------------------------------------------------------- */
int mpmm_host_frobenius_norm(int comps, const double *x, int64_t count, double *out);
int mpmm_host_frobenius_rel_diff(int comps, const double *x, const double *y, int64_t count,
                                 double *out);

#ifdef __cplusplus
}
#endif

#endif /* MPMM_CUDA_H */
