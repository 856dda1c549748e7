/*
 * taxisdg_b200.h -- C-ABI of the B200 (sm_100a) matrix-free DG operator.
 *
 * Drop-in boundary for the hot path of the reference package `taxisdg`
 * (arxiv/paper_1403_1157).  The reference is pure Python; the interfaces
 * replaced here are (paths relative to /root/reference/pkg/src/taxisdg):
 *
 *   tdg_create / tdg_destroy   DiscreteOperator.__init__ tables, groups and
 *                              partition setup          operator.py:85-229
 *   tdg_apply (mass_inverse=0) DiscreteOperator.apply    operator.py:253-284
 *   tdg_apply (mass_inverse=1) DiscreteOperator.apply_f  operator.py:286-288
 *                              + DGSpace.apply_inverse_mass fespace.py:117-118
 *   tdg_apply_host             the same on host (numpy) arrays, the call shape
 *                              of the reference's steppers timeint.py:315-333
 *   tdg_rk_stage               one explicit stage  a*U0 + b*U + c*M^-1 L(U)
 *                              (SSP-RK3 composition of apply_f, SURVEY 8(a) a14;
 *                              DIRK stage algebra timeint.py:315-333)
 *   tdg_ssprk3_step            three fused stages (Shu-Osher form)
 *   tdg_ssprk3_steps_host      the same on a host state, copies every step
 *   tdg_species_totals         DiscreteFunction.species_totals fespace.py:170-174
 *   tdg_species_l2             analysis.l2_error of two fields     analysis.py:30-50
 *   tdg_mgs                    GMRES Arnoldi MGS sweep             timeint.py:162-170
 *   tdg_color_faces            (host) face colouring that orders the face
 *                              loop; replaces the RCB partition /
 *                              private-buffer merge that makes the
 *                              reference's sums race-free, operator.py:208-284
 *   tdg_dot / tdg_norm2        Krylov scalars: `w @ V[i]`, `np.linalg.norm`
 *                              in gmres_solve/newton_solve timeint.py:148-202,
 *                              timeint.py:242-280
 *   tdg_axpby / tdg_axpy_dev   Krylov/Newton vector updates timeint.py:171,199,278
 *
 * Conventions: every array argument of the apply/stage/vector calls is a
 * DEVICE pointer; coefficient arrays use the reference layout U[e][s][i]
 * (fp64, C order, n_elements x n_species x nb, fespace.py:46-69).  The
 * descriptor's table/geometry pointers are device pointers owned by the
 * caller and must outlive the context; the small host arrays
 * (diffusivity, lin_source, params, seg_ptr) are copied at create time.
 * Streams are `cudaStream_t` passed as `void*` (NULL = legacy default
 * stream).  No call allocates device memory, streams or events after
 * tdg_create (state vectors and work buffers are the caller's); the one
 * exception is tdg_apply_host's process-wide pinned host staging, made on
 * its first call.  Every
 * call returns 0 on success or a negative TDG_E* code; tdg_last_error()
 * gives a message (thread-local).
 *
 * Face loop: the faces come in colour segments (tdg_color_faces): within
 * a segment no element is touched twice, so each face adds its two
 * contribution blocks straight into the elements' face-sum rows (no
 * atomics, no per-face buffers), and the segments run in a fixed order,
 * so every sum has a fixed order: results are bitwise reproducible run to
 * run (reference contract tests/test_operator.py:113-119).
 *
 * One context = one stream at a time: the reduction workspace, the copy
 * streams / events and the cached SSP-RK3 graph are per context, so two
 * calls on the same context must not run concurrently on different
 * streams (the reference allows one evaluation at a time per instance,
 * SPEC.md:423).
 */
#ifndef TAXISDG_B200_H
#define TAXISDG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TDG_ABI_VERSION 9

#if defined(__GNUC__)
#define TDG_API __attribute__((visibility("default")))
#else
#define TDG_API
#endif

enum tdg_status {
  TDG_OK = 0,
  TDG_E_INVALID = -1,     /* bad descriptor / argument  (reference: ValueError) */
  TDG_E_UNSUPPORTED = -2, /* (dim, order, model, species) not compiled in      */
  TDG_E_CUDA = -3         /* CUDA runtime error                                 */
};

enum tdg_model { TDG_MODEL_PLAQUE = 0, TDG_MODEL_REDUCED = 1, TDG_MODEL_DIFFUSION = 2 };

/* flux.py:57 SCHEME_NAMES order */
enum tdg_scheme { TDG_CDG2 = 0, TDG_CDG = 1, TDG_BR2 = 2, TDG_IP = 3, TDG_BO = 4 };

/* bit layout of the per-face code words (if_code / bf_code) */
#define TDG_CODE_TIN(c)     ((c) & 31)          /* table id lf_in*nperm+pm_in   */
#define TDG_CODE_TOUT(c)    (((c) >> 5) & 31)   /* table id of the outside side  */
#define TDG_CODE_MINUS_IN   (1 << 10)           /* K- is the inside element      */
#define TDG_CODE_TAG(c)     (((c) >> 11) & 7)   /* BoundaryTag (boundary faces)  */
#define TDG_CODE_MIRROR     (1 << 14)           /* Dirichlet mirror exterior     */
#define TDG_CODE_SKIP_OUT   (1 << 15)           /* outside is a ghost: no write  */
#define TDG_CODE_FIRST_IN   (1 << 16)           /* inside's first face: write     */
#define TDG_CODE_FIRST_OUT  (1 << 17)           /* outside's first face: write    */

typedef struct tdg_desc {
  int32_t dim;            /* 2 or 3 */
  int32_t order;          /* k, 1..3 */
  int32_t n_species;      /* S */
  int32_t nb;             /* C(k+d, d) */
  int32_t nq_vol;         /* volume points (<= default rule of degree 3k+1) */
  int32_t nq_face;        /* face points (<= default rule of degree 3k+2) */
  int32_t model;          /* enum tdg_model */
  int32_t scheme;         /* enum tdg_scheme */
  int64_t n_elements;     /* owned elements = rows of U, R */
  int64_t n_ghost;        /* ghost rows appended after the owned rows of U */
  int64_t n_int_faces;    /* interior (+ Dirichlet mirror) faces */
  int64_t n_bnd_faces;    /* prescribed-flux boundary faces */
  double chi_e;           /* 1.5 (2D) / 2 (3D), flux.py:87-89 */
  double adj_sign;        /* -1 for bo, +1 otherwise, flux.py:79-80 */
  double ip_eta;          /* ip_eta0 * max(k,1)^2, operator.py:104 */
  /* host arrays, copied at create */
  const double* diffusivity;  /* [S] */
  const double* lin_source;   /* [S*S] linear part of the source, row-major */
  const double* params;       /* [32] model parameters (PlaqueParams order) */
  /* device arrays (caller-owned) */
  const double* vol_phi;      /* [Q*nb]       basis at volume points */
  const double* vol_grad;     /* [Q*nb*d]     reference gradients */
  const double* vol_w;        /* [Q]          volume weights */
  const double* vol_stiff;    /* [d(d+1)/2*nb*nb] symmetric stiffness blocks */
  const double* face_B;       /* [T*F*nb]     basis at face points, per table */
  const double* face_G;       /* [T*F*nb*d]   gradients at face points */
  const double* face_Pw;      /* [T*F*F]      (B B^T) w_face  (lifting) */
  const double* face_w;       /* [F]          face weights */
  const double* elem_geo;     /* [ne*(1+d(d+1)/2)]  detJ, sym(Jinv Jinv^T) */
  const int32_t* if_elems;    /* [nif*2]  inside, outside row (-1 mirror) */
  const int32_t* if_code;     /* [nif]    packed code word */
  const double* if_geo;       /* [nif*(2d+4)] jn_in, jn_out, sfac, h, 1/detJ_in, 1/detJ_out */
  const int32_t* bf_elem;     /* [nbf]    inside row */
  const int32_t* bf_code;     /* [nbf]    packed code word */
  const double* bf_geo;       /* [nbf]    sfac */
  /* optional: zero-padded per-signature operand tables of the element-
   * local tensor-core (DMMA) face kernel, layout of
   * tables.mma_face_tables (NULL disables it) */
  const double* face_mma;
  /* operand tables of the transposed tensor-core volume kernel
   * (tables.tc_volume_tables, may be NULL) */
  const double* vol_tc;
  /* species-rows tensor-core face kernel (3D): per-signature operand tables
   * (tables.tc_face_tables, stride from the compiled sizes) and blocks of up
   * to 8 interior faces of one signature, int32 [n_face_blocks][2] = (first
   * face, count), never straddling a segment (may be NULL) */
  const double* face_tc;
  const int32_t* face_blocks;
  int64_t n_face_blocks;
  /* optional, species-rows face kernel: per face-geometry class (one
   * (table id, Jinv n) pair) the B fragments paired with the folded
   * normal-derivative fragments sum_a (Jinv n)_a G_a
   * (tables.tc_face_fold_tables), and the class of every interior face's
   * inside / outside side, int32 [nif][2]; both NULL: the kernel folds
   * Jinv n per face */
  const double* face_tc_fold;
  const int32_t* if_fold;
  /* optional, with the class tables: groups of 8/gcd(S,8) interior faces
   * of one segment sharing both sides' class and the lifting side
   * (tables.tc_face_groups), int32 [n_face_groups][8/gcd(S,8)] face ids,
   * -1 past a run's end (they cover every interior face of the segments).
   * NULL: the one-face species-rows kernel runs the blocks instead */
  const int32_t* face_groups;
  int64_t n_face_groups;
  /* optional, with the face groups: operand tables of the modal face
   * kernel (tables.modal_face_tables: face-trace factors face_B = Bf T,
   * G_n = Bd Td), layout from the compiled sizes, per signature and per
   * face-geometry class); NULL: the face-group kernel evaluates the full
   * traces */
  const double* face_modal;
  /* optional point data of the diffusion model (x-dependent closures,
   * reference tests/test_operator.py:31-70): Dirichlet values at the face
   * points of the mirror faces, [n_int_faces][nq_face][S] (entries of the
   * non-mirror faces unused), and prescribed wall fluxes at the points,
   * [n_bnd_faces][nq_face][S]; either forces the CTA-staged generic face
   * kernels.  Device pointers, caller-owned, may change between calls
   * (time-dependent data) */
  const double* if_bval;
  const double* bf_qval;
  /* optional, host-data stepping (tdg_ssprk3_steps_host): within every
   * segment the faces, walls, blocks and groups are ordered by element
   * chunk (chunk k = elements from ne k / 8 rounded down to a multiple of
   * eight, and a face belongs to the later chunk of its elements); seg_chunk_ptr
   * (HOST) = 4 offset arrays of n_segments * 8 + 1 entries (faces | walls |
   * blocks | groups), run (s, c) = [o[8 s + c], o[8 s + c + 1]); and the
   * code words with the TDG_CODE_FIRST_* bits cleared (device).  With them
   * the first stage of every host step runs chunk by chunk as the state
   * arrives (volume terms first, face sums added, then M^-1 and the stage
   * combination); NULL: whole-state stages */
  const int64_t* seg_chunk_ptr;
  const int32_t* if_code_add;
  const int32_t* bf_code_add;
  /* optional, tensor-core volume kernel: element-geometry classes
   * (tables.tc_volume_classes): per class the summed stiffness fragments
   * [ncls][KT][NNT][32], the elements in class-sorted tasks of 8 (int32
   * [n_vol_tasks][8] element ids, -1 pads), each task's class (int32
   * [n_vol_tasks]), and (HOST) the task offsets [9] of the 8 element chunks
   * (chunk k starts at ne k / 8 rounded down to a multiple of 8 elements,
   * tables.vol_chunk_bounds); all NULL: per-element metric scaling */
  const double* vol_cls_tab;
  const int32_t* vol_perm;
  const int32_t* vol_task_cls;
  int64_t n_vol_tasks;
  const int64_t* vol_chunk_tasks;
  /* face colour segments, run in order: segment s covers the interior
   * faces [I[s], I[s+1]), the walls [W[s], W[s+1]), the face blocks
   * [B[s], B[s+1]) and the face groups [G[s], G[s+1]) with seg_ptr (HOST)
   * = I[n+1] | W[n+1] | B[n+1] | G[n+1].  No
   * element is written twice within a segment, and each element's first
   * written face side (in segment order) carries TDG_CODE_FIRST_IN/OUT and
   * every owned element has at least one face.  The last n_segments_cut
   * segments hold the faces that read ghost rows (slab runs: run after
   * the exchange, tdg_rk_stage_part part 2). */
  int32_t n_segments;
  int32_t n_segments_cut;
  const int64_t* seg_ptr;
} tdg_desc;

typedef struct tdg_ctx tdg_ctx;

TDG_API int tdg_version(void);
TDG_API const char* tdg_last_error(void);

/* Builds the context for one operator (reference DiscreteOperator.__init__,
 * operator.py:85-140: tables, face SoA, K- flags).  The device arrays of the
 * descriptor must be complete when this is called (no upload pending on
 * another stream): tdg_create copies reference-element tables to constant
 * memory and, for the 2D signature-run kernel, reads the face code words,
 * face tables and face records back once, on the default stream.  It creates
 * every stream, event and workspace the later calls use. */
TDG_API int tdg_create(const tdg_desc* desc, tdg_ctx** out);
TDG_API int tdg_destroy(tdg_ctx* ctx);

/* R = L_h(U) (mass_inverse=0) or M^-1 L_h(U) (mass_inverse=1).
 * U has n_elements + n_ghost rows; R has n_elements rows and must not
 * alias U (the face sums accumulate in R).  t is accepted for API parity
 * (the plaque/reduced/diffusion models are autonomous). */
TDG_API int tdg_apply(tdg_ctx* ctx, const double* U, double* R, double t,
              int mass_inverse, void* stream);

/* out = a*U0 + b*U + c*M^-1 L_h(U); U0 may be NULL when a == 0.  acc
 * (n_elements rows) receives the face sums: NULL means acc = out.  acc
 * must not alias U, nor U0 when a != 0; out may alias U0, and may alias U
 * when acc does not. */
TDG_API int tdg_rk_stage(tdg_ctx* ctx, const double* U0, const double* U, double* out,
                 double* acc, double a, double b, double c, double t, void* stream);

/* A stage split around a ghost-row exchange (slab-decomposed runs):
 * part 1 launches everything that reads owned rows only (volume terms,
 * non-cut faces, walls); part 2, issued after the ghost rows of U are in
 * place, launches the cut faces and the final sum.  Same arguments and
 * result as tdg_rk_stage. */
TDG_API int tdg_rk_stage_part(tdg_ctx* ctx, const double* U0, const double* U, double* out,
                              double* acc, double a, double b, double c, double t, int part,
                              void* stream);

/* tdg_apply on HOST arrays in any (pageable) memory, the reference's own
 * call shape (apply / apply_f on numpy arrays): U_host (n_elements +
 * n_ghost rows) -> U_dev, the operator, R_dev -> R_host (n_elements rows),
 * through process-wide pinned staging buffers (3 x 64 MiB, allocated on
 * the first call -- the one allocation after tdg_create) that a pool of
 * host threads fills / drains while the DMA engine moves the neighbouring
 * piece; the volume kernel runs in element chunks so the copy-out starts
 * with the first chunk.  Synchronous: R_host is complete on return.  Same
 * bits as tdg_apply. */
TDG_API int tdg_apply_host(tdg_ctx* ctx, const double* U_host, double* R_host, double* U_dev,
                           double* R_dev, double t, int mass_inverse, void* stream);

/* nsteps SSP-RK3 steps of a HOST state (pinned memory, undecomposed
 * mesh), through the device buffers U, w1, w2 (shape of U): every step
 * copies the state in and the result out, in element chunks on two copy
 * streams per direction -- step n+1's copy-in of chunk k follows step
 * n's copy-out of chunk k, and the last stage's volume kernel runs chunk
 * by chunk so the copy-out starts with the first chunk.  Bitwise the same
 * result as copy-in, tdg_ssprk3_step, copy-out per step.  The public
 * host-data entry point of the end-to-end measurement. */
TDG_API int tdg_ssprk3_steps_host(tdg_ctx* ctx, double* U_host, double* U, double* w1,
                                  double* w2, int64_t nsteps, double t, double dt, void* stream);

/* one Shu-Osher SSP-RK3 step in place on U (three state vectors: U and
 * the work vectors w1, w2 of the shape of U); undecomposed meshes only
 * (slab runs exchange ghost rows between stages: tdg_rk_stage_part). */
TDG_API int tdg_ssprk3_step(tdg_ctx* ctx, double* U, double* w1, double* w2, double t,
                            double dt, void* stream);

/* Species totals int u_s over the owned elements, written to totals[S]
 * (device): sqrt(|ref simplex|) * sum_e detJ_e U[e,s,0].  Replaces
 * DiscreteFunction.species_totals (reference fespace.py:170-174).
 * Deterministic (fixed-order two-pass reduction). */
TDG_API int tdg_species_totals(tdg_ctx* ctx, const double* U, double* totals, void* stream);

/* Broken L2 norm per species of U - V over the owned elements (V may be
 * NULL: the norm of U), written to out[S] (device): sqrt(sum_e detJ_e
 * sum_i (U - V)[e,s,i]^2) -- exact for the orthonormal basis; the parity
 * metric of the DG-vs-DG comparisons (the reference's l2_error,
 * analysis.py:30-50, for two fields on the same space). */
TDG_API int tdg_species_l2(tdg_ctx* ctx, const double* U, const double* V, double* out,
                           void* stream);

/* Krylov reductions: deterministic two-pass tree (fixed grid), result
 * written to a DEVICE scalar.  Operands must be 16-byte aligned
 * (TDG_E_INVALID otherwise). */
TDG_API int tdg_dot(tdg_ctx* ctx, const double* x, const double* y, int64_t n,
            double* result, void* stream);
TDG_API int tdg_norm2(tdg_ctx* ctx, const double* x, int64_t n, double* result,
              void* stream);
/* y = a*x + b*y (host scalars) */
TDG_API int tdg_axpby(double a, const double* x, double b, double* y, int64_t n,
              void* stream);
/* y += s*alpha[0]*x with alpha a DEVICE scalar (MGS update without a
 * host round trip) */
TDG_API int tdg_axpy_dev(double s, const double* alpha, const double* x, double* y,
                 int64_t n, void* stream);

/* One modified Gram-Schmidt sweep of GMRES's Arnoldi step (reference
 * timeint.py:162-170): for i = 0..j, h[i] = w . V_i then w -= h[i] V_i;
 * finally h[j+1] = ||w||.  V holds rows of length n with leading dimension
 * ldv; h (j+2 doubles) and everything else are device pointers.  Each
 * axpy is fused with the next dot (same element order and reduction tree
 * as tdg_dot / tdg_axpy_dev, so bitwise the same results), one call per
 * Arnoldi step, no host round trip. */
TDG_API int tdg_mgs(tdg_ctx* ctx, const double* V, int64_t ldv, int j, double* w, int64_t n,
                    double* h, void* stream);

/* One pass of that sweep for slab-decomposed runs, whose dots must be
 * summed over the ranks between passes: pass i (0 <= i <= j+1) applies the
 * previous pass's update with the (globally reduced) h[i-1] and writes this
 * rank's partial of h[i]; the last pass writes w . w (the caller sums over
 * the ranks and takes the root).  Same kernels, element order and
 * reduction tree as tdg_mgs. */
TDG_API int tdg_mgs_pass(tdg_ctx* ctx, const double* V, int64_t ldv, int i, int j, double* w,
                         int64_t n, double* h, void* stream);

/* GMRES basis vector (reference timeint.py:165,176: V[j+1] = w / hnext):
 * v = w / hnext with ||v|| written to the DEVICE scalar norm_out in the
 * same pass (same reduction tree as tdg_norm2, so bitwise its result); the
 * next Jacobian-free product needs that norm.  The divisor is the host
 * scalar hnext, or the DEVICE scalar hnext_dev[0] when hnext_dev is not
 * null (the Arnoldi step can then run ahead of the host). */
TDG_API int tdg_scale_norm(tdg_ctx* ctx, const double* w, double hnext, const double* hnext_dev,
                           double* v, int64_t n, double* norm_out, void* stream);

/* Jacobian-free directional difference of newton_solve's jv (reference
 * timeint.py:259-264): tdg_jv_shift computes eps = cnum / max(vnorm[0],
 * 1e-300) on the device (cnum = sqrt(eps_mach)(1 + ||U||), vnorm a DEVICE
 * scalar), writes it to eps_out and forms Up = U + eps v in one pass;
 * tdg_jv_diff then forms r = (r - GU) / eps in place after r = G(Up). */
TDG_API int tdg_jv_shift(const double* U, const double* v, const double* vnorm, double cnum,
                         double* Up, double* eps_out, int64_t n, void* stream);
TDG_API int tdg_jv_diff(double* r, const double* GU, const double* eps, int64_t n, void* stream);

/* Kernel variant selection (testing / A-B timing).  bit 0: pin the
 * CTA-staged generic kernels; bit 5: launch tdg_ssprk3_step's kernels
 * directly instead of replaying its cached CUDA graph; bit 13: ignore the
 * face-geometry-class tables (fold Jinv n per face); bit 14: run the
 * one-face species-rows kernel instead of the face-group kernel; bit 16:
 * the face-group kernel on full traces instead of the modal one; bit 15:
 * ignore the element-geometry classes of the volume kernel; bit 12: use the
 * transposed tensor-core volume kernel wherever it compiles (default only
 * where the one-thread-per-element kernel does not fit); bits 8-11: CTAs
 * per SM of the 2D register-resident face kernel's grid-stride grid (0 =
 * default, 15 = uncapped, one face group per warp); bit 17: the 2D faces on
 * the shared-memory-table kernel instead of the signature-run kernel; bit 18:
 * the cp.async-staged signature-run kernel on states of any size (default:
 * only states larger than half the L2).  0 (default) lets the library pick
 * the fastest compiled-in kernels. */
TDG_API int tdg_set_variant(tdg_ctx* ctx, int variant);

/* 2D signature runs (k_faces_sig): tdg_create cuts the interior faces into
 * maximal runs of one (inside, outside) trace-table signature and launches
 * each run with its tables as kernel parameters; a run whose faces all carry
 * the same Jinv n on both sides has it folded into the tables.  Returns the
 * number of runs (0: the kernel is not used: 3D, Dirichlet mirror models,
 * non-default face rule, boundary point data, or faces not sorted into few
 * runs) and how many are folded.  Replaces nothing in the reference (launch
 * bookkeeping of operator.py:262-284's face loop). */
TDG_API int tdg_face_runs(const tdg_ctx* ctx, int64_t* n_runs, int64_t* n_folded);

/* Per-kernel device timing: with profiling enabled every operator kernel
 * launch is bracketed by CUDA events on its own stream;
 * tdg_profile_read synchronizes, returns the accumulated milliseconds and
 * launch counts per kernel (ms[4], launches[4]: 0 interior faces, 1 wall
 * faces, 2 volume, 3 reserved) and resets. */
TDG_API int tdg_profile(tdg_ctx* ctx, int enable);
TDG_API int tdg_profile_read(tdg_ctx* ctx, double* ms, int64_t* launches);

/* FP64 throughput probe: a DFMA-bound kernel (148*8 CTAs x 256 threads,
 * 16 independent chains, `iters` iterations) writing one value per
 * thread to out[148*8*256]; flops = 148*8*256*16*2*iters. */
TDG_API int tdg_fp64_probe(double* out, int64_t iters, void* stream);
TDG_API int64_t tdg_fp64_probe_threads(void);
/* FP64 tensor-core (DMMA m8n8k4) probe on the same grid: per warp 4
 * independent 8x8x4 MMAs per iteration, flops = threads/32*iters*4*512. */
TDG_API int tdg_dmma_probe(double* out, int64_t iters, void* stream);

/* Host-side setup (no GPU needed): greedy colouring of the face graph
 * that orders the face loop.  Elements are vertices, faces edges; a face
 * side with elem < 0 is not written (walls, mirror faces, ghost sides).
 * Faces are visited in `order` (NULL: index order) and each takes the
 * smallest colour that none of its written elements holds yet, so no
 * element is written twice within a colour.  Visiting the faces grouped by
 * their (local face in, local face out) class colours the structured
 * simplex meshes with d+1 colours.  Writes color[n_faces] and returns the
 * number of colours (>= 0) or TDG_E_INVALID (bad index, > 64 colours). */
TDG_API int tdg_color_faces(int64_t n_faces, const int32_t* elem_in, const int32_t* elem_out,
                            int64_t n_elements, const int64_t* order, int32_t* color);

#ifdef __cplusplus
}
#endif
#endif /* TAXISDG_B200_H */
