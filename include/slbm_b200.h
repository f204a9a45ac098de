/*
 * slbm_b200 — C-ABI of the B200 (sm_100a) sparse lattice-Boltzmann engine.
 *
 * The reference package has no FFI: its drop-in boundary is the duck-typed
 * block-engine protocol of pkg/src/slbm/sparse.py (SparseEngine, :48-383),
 * consumed by Domain (domain.py:109-114), the halo EdgePlans/pack/unpack
 * (exchange.py:125-253) and the drivers (exchange.py:330-374).  Every entry
 * point below replaces one method/attribute of that protocol; the Python
 * class paper_2408_06880_b200.engine.SparseEngine wraps them 1:1 (ctypes).
 *
 * Conventions
 *   - plain pointers and sizes only; "host" pointers are ordinary CPU
 *     memory, "dev" pointers are device memory on the engine's GPU;
 *   - every function returns an SLBM_* status; slbm_last_error() returns the
 *     message of the last failure on the calling thread;
 *   - an engine handle is not thread-safe (one owner per block, like the
 *     reference); work is issued on the engine's stream
 *     (slbm_engine_stream / slbm_engine_set_stream);
 *   - slot ids, cell ids (cid) and the index list are identical to the
 *     reference's (sparse.py:97-195), so exported arrays compare with
 *     np.array_equal.
 */
#ifndef SLBM_B200_H
#define SLBM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes -> exceptions of pkg/src/slbm/errors.py:4-29 */
#define SLBM_OK 0
#define SLBM_ECONFIG 1   /* ConfigurationError */
#define SLBM_EEMPTY 2    /* EmptyBlockError */
#define SLBM_EUNSTABLE 3 /* NumericalInstabilityError */
#define SLBM_EPROTOCOL 4 /* ProtocolError */
#define SLBM_ECUDA 5     /* RuntimeError */

/* collision models (core.py:66-74 has srt/trt; cumulant is new, unpinned) */
#define SLBM_SRT 0
#define SLBM_TRT 1
#define SLBM_CUMULANT 2
/* internal model code: the cumulant with general higher-order rates, chosen
 * by slbm_engine_set_cumulant_rates (create engines with SLBM_CUMULANT) */
#define SLBM_CUMULANT_GEN 3

/* streaming patterns (sparse.py:45) */
#define SLBM_PULL 0
#define SLBM_AA 1

/* sweep phases (sparse.py:226-231) */
#define SLBM_PHASE_ALL 0
#define SLBM_PHASE_INTERIOR 1
#define SLBM_PHASE_FRAME 2

/* storage parity (core.py:32-47) */
#define SLBM_EVEN 0
#define SLBM_ODD 1

typedef struct SlbmEngine SlbmEngine;
typedef struct SlbmHalo SlbmHalo;

typedef struct SlbmInfo {
  int32_t q, dim, pattern, parity;
  int32_t has_split, model;
  int64_t n_fluid;       /* sparse.py:75 */
  int64_t total_slots;   /* sparse.py:131 */
  int64_t n_ubb_slots;   /* sparse.py:136 */
  int64_t n_ghost_slots; /* sparse.py:137 */
  int64_t n_interior, n_frame; /* sparse.py:377-383 */
  int64_t base[28];      /* sparse.py:130, length q+1 used */
  int64_t n_ubb_q[27];
  int64_t n_ghost_q[27];
  int64_t device_bytes;  /* bytes of device memory held by the engine */
  int64_t n_outlet_slots; /* fixed-density outlet reads (extension, tag 4) */
  int64_t layout;         /* 0 sparse (index list), 1 dense (direct addressing) */
} SlbmInfo;

/* ---- construction: SparseEngine.__init__ (sparse.py:51-93) ----------------
 * tags_pad  host uint8 tags on the padded box, C order over reversed axes
 *           ((Z+2,Y+2,X+2) for 3-d, (Y+2,X+2) for 2-d)          flags.py:111-125
 * ubb_u_pad host float64 wall velocities, tags_pad shape + (dim,); may be NULL
 *           when no tag is UBB
 * dims      public extents (x, y[, z]); periodic: per public axis (0/1)
 * q         9 (d2q9, dim 2), 19 or 27 (dim 3)
 * frame_width per public axis, or NULL for no interior/frame split
 *           (flags.py:83-108; widths clamped to the extent).  The reference
 *           requires widths >= 1 (enforced by the Python layer); 0 is
 *           accepted here and means "no frame on that axis" — used by the
 *           domain drivers for axes without halo exchange.
 * Runs the whole list build on the GPU: fluid enumeration, index list with
 * no-slip folding, UBB and ghost slot allocation, the ownership-uniqueness
 * check (sparse.py:182-185) and the split lists.  PDFs start NaN-poisoned
 * (sparse.py:90-91).                                                        */
int slbm_engine_create(const uint8_t* tags_pad, const double* ubb_u_pad, int dim,
                       const int32_t* dims, const uint8_t* periodic, int q, int model,
                       double omega, double lambda_odd, int pattern,
                       const int32_t* frame_width, int device, SlbmEngine** out);
/* direct-addressing block engine, the reference's DenseEngine (dense.py:52-342):
 * same arguments; storage q-planes over the padded box, slot = q*npad + p,
 * no index list; outlets unsupported.  Same entry points apply to it.      */
int slbm_engine_create_dense(const uint8_t* tags_pad, const double* ubb_u_pad, int dim,
                             const int32_t* dims, const uint8_t* periodic, int q, int model,
                             double omega, double lambda_odd, int pattern,
                             const int32_t* frame_width, int device, SlbmEngine** out);
int slbm_engine_destroy(SlbmEngine* eng);
int slbm_engine_info(const SlbmEngine* eng, SlbmInfo* info);
/* cudaStream_t as void*; set_stream(NULL) restores the engine's own stream */
int slbm_engine_stream(const SlbmEngine* eng, void** stream);
int slbm_engine_set_stream(SlbmEngine* eng, void* stream);
int slbm_engine_set_params(SlbmEngine* eng, int model, double omega, double lambda_odd);
/* Cumulant relaxation rates beyond the shear rate omega (Geier et al. 2015;
 * extension, unpinned): bulk = w2 (trace of the second-order cumulants) and
 * higher = {w3, w4, w5, w6, w7, w8, w9, w10} (NULL: all 1).  All higher
 * rates 1 selects the closed-form kernel, anything else (or force_general)
 * the general one.  The engine must use the cumulant model.                */
int slbm_engine_set_cumulant_rates(SlbmEngine* eng, double bulk, const double* higher,
                                   int force_general);

/* ---- exported lists (for parity checks against the reference) -----------
 * idx: (q-1, n_fluid) uint32 (sparse.py:186); fluid_coords: (n_fluid, dim)
 * int64 public coords (sparse.py:76); ubb_*: n_ubb_slots (sparse.py:188-191);
 * ghost_q/ghost_pflat/ghost_slot: n_ghost_slots entries of the reference's
 * _ghost_slots dict (sparse.py:179), in slot order.  Any pointer may be NULL. */
int slbm_export_lists(const SlbmEngine* eng, uint32_t* idx, int64_t* fluid_coords,
                      int64_t* ubb_slot, int64_t* ubb_partner, double* ubb_corr,
                      int64_t* ghost_q, int64_t* ghost_pflat, int64_t* ghost_slot);
/* frame / interior cell ids (sparse.py:80-88); NULL pointers skipped */
/* per-face interior/frame split (extension): frame = cells within lo[a] of
 * the low face or hi[a] of the high face of axis a (0 = none); the
 * reference's frame_mask (flags.py:83-108) is lo == hi >= 1.  Sparse only. */
int slbm_engine_set_frame(SlbmEngine* eng, const int32_t* lo, const int32_t* hi);
int slbm_export_split(const SlbmEngine* eng, int64_t* interior, int64_t* frame);

/* ---- state (sparse.py:199-222, :308-331) --------------------------------- */
/* values: host (q, n_fluid) float64 canonical state; parity -> EVEN */
int slbm_init_canonical(SlbmEngine* eng, const double* values);
/* device-pointer variant of init_canonical (values already on the GPU) */
int slbm_init_canonical_dev(SlbmEngine* eng, const double* dev_values);
/* equilibrium from per-cell rho (n) and u (dim, n), host pointers; rho/u may
 * be scalars when the *_scalar flag is 1 (u then has dim entries)           */
int slbm_init_equilibrium(SlbmEngine* eng, const double* rho, int rho_scalar,
                          const double* u, int u_scalar);
/* host (q, n_fluid); at ODD parity refreshes UBB partners first (:317)     */
int slbm_canonical_state(SlbmEngine* eng, double* values);
/* host rho (rev_shape) and u (rev_shape + (dim,)), zeros at non-fluid cells;
 * SLBM_EUNSTABLE when a density is <= 0 or non-finite (core.py:108-111)    */
int slbm_macroscopic(SlbmEngine* eng, double* rho, double* u);
/* the same fields per fluid cell in cid order (rho: n_fluid, u: n_fluid x
 * dim): what Domain.gather_macroscopics scatters into the global box for
 * sparse blocks instead of moving each block's full box                   */
int slbm_macroscopic_compact(SlbmEngine* eng, double* rho, double* u);
/* Monitors: total mass and momentum of the canonical state over all fluid
 * cells, fp64 -- one pass over the groups, warp-shuffle reductions with a
 * fixed reduction tree (bit-reproducible run to run).  out4 = {mass,
 * momentum x, y, z}; total_mass = out4[0].                                 */
int slbm_total_moments(SlbmEngine* eng, double* out4);
/* Domain.gather_macroscopics on the device (domain.py:246-268): write this
 * block's fluid cells' rho / u into global device boxes (gdims = global
 * x, y, z extents; the block at origin x, y, z; solids untouched, so the
 * caller zeroes the boxes), then move a box to host memory with the staged
 * multi-threaded copy (any host buffer; pinned ones go by one DMA).      */
int slbm_macroscopic_global(SlbmEngine* eng, double* dev_rho, double* dev_u,
                            const int64_t* gdims, const int64_t* origin);
int slbm_copy_to_host(void* host, const void* dev, int64_t bytes, int device);
int slbm_total_mass(SlbmEngine* eng, double* mass);

/* ---- stepping (sparse.py:226-304) ---------------------------------------- */
int slbm_refresh_boundary(SlbmEngine* eng, int parity);
/* launches one sweep; does not synchronize */
int slbm_step(SlbmEngine* eng, int phase);
int slbm_finish_step(SlbmEngine* eng);
/* n full single-block steps (refresh_boundary + step(all) + finish_step), no
 * host sync; use_graph=1 replays a captured CUDA graph of one step pair, or
 * for blocks up to 2^19 fluid cells (knob 4) runs all n steps in one
 * cooperative launch (resident kernel, bitwise the same result).          */
int slbm_run(SlbmEngine* eng, int64_t n, int use_graph);
/* blocks until the engine's stream is idle, then reports the first unstable
 * step (SLBM_EUNSTABLE, *first_bad_step set) or SLBM_OK (-1).  Clears.     */
int slbm_poll_instability(SlbmEngine* eng, int64_t* first_bad_step);
/* slbm_poll_instability over several engines with one synchronisation per
 * distinct stream; on failure `which` is the first unstable engine's index */
int slbm_poll_engines(SlbmEngine** engines, int n, int64_t* first_bad_step, int* which);
int slbm_synchronize(SlbmEngine* eng);
int slbm_parity(const SlbmEngine* eng, int* parity);
int slbm_set_parity(SlbmEngine* eng, int parity);
/* pull pattern: 1 when the second buffer is the current one (the buffer pair
 * a captured CUDA graph refers to), else 0; AA: always 0 (extension) */
int slbm_buffer_state(const SlbmEngine* eng, int* state);

/* ---- slot access for halo plans (sparse.py:335-366) ---------------------- */
/* pflat: padded flat index of the cell (C order over the padded box)       */
int slbm_slot_index(const SlbmEngine* eng, const int64_t* qs, const int64_t* pflat,
                    int64_t n, int64_t* out);
/* padded flat index -> cid (or -1) over the block's padded box: hosts that
 * resolve many slot_index queries (halo planning) keep a copy             */
int slbm_export_cid_map(const SlbmEngine* eng, int32_t* out);
int slbm_ghost_slot_index(const SlbmEngine* eng, const int64_t* qs, const int64_t* pflat,
                          int64_t n, int64_t* out);
int slbm_read_slots(SlbmEngine* eng, const int64_t* slots, int64_t n, double* out);
int slbm_write_slots(SlbmEngine* eng, const int64_t* slots, int64_t n, const double* in);
/* raw device pointer of the active PDF buffer (pull swaps it every step) */
int slbm_pdf_pointer(const SlbmEngine* eng, double** dev_pdf);
/* device layout of the PDF array: start of each direction group (Q + 1
 * entries) and the element count.  Sparse engines pad every group to a
 * multiple of 32 slots (256 B); slot ids at the C-ABI stay the reference's
 * (sparse.py:128-137) and are translated internally.                      */
int slbm_pdf_layout(const SlbmEngine* eng, int64_t* group_start, int64_t* n_elements);

/* ---- halo exchange (exchange.py:125-374) ---------------------------------
 * A halo is the per-rank exchange program for one phase set: a list of
 * directed edges, each a (sender engine, receiver engine) pair with the
 * sender's read slots and the receiver's write slots per phase
 * (EdgePlan._build, exchange.py:148-219).  Edges whose two engines live in
 * this process are moved by one fused gather-scatter kernel; edges with a
 * remote end are packed into / unpacked from per-peer contiguous buffers
 * that travel with ncclSend/ncclRecv (one message per peer per phase).    */
int slbm_halo_create(int device, SlbmHalo** out);
int slbm_halo_destroy(SlbmHalo* halo);
/* local edge: both engines here. send[n_send] on src, take[n_tgt] indexes
 * the send list (exchange.py:199-201), tgt[n_tgt] on dst.                 */
int slbm_halo_add_local(SlbmHalo* halo, int phase, SlbmEngine* src, SlbmEngine* dst,
                        const int64_t* send, int64_t n_send, const int64_t* take,
                        const int64_t* tgt, int64_t n_tgt);
/* remote send: values of send[n] on src go to peer rank `peer`, appended to
 * that peer's message for this phase in call order                         */
int slbm_halo_add_send(SlbmHalo* halo, int phase, SlbmEngine* src, int peer,
                       const int64_t* send, int64_t n);
/* remote receive: the next n_wire values of peer's message; take[n_tgt]
 * picks the stored ones, written to tgt on dst                              */
int slbm_halo_add_recv(SlbmHalo* halo, int phase, SlbmEngine* dst, int peer,
                       int64_t n_wire, const int64_t* take, const int64_t* tgt, int64_t n_tgt);
/* finalize: allocates device buffers; nccl_comm may be NULL when the halo
 * has no remote edges.  nccl_comm is an ncclComm_t created by the caller
 * or by slbm_nccl_comm_init.                                                */
int slbm_halo_commit(SlbmHalo* halo, void* nccl_comm);
/* start the exchange for `phase` on the halo's comm stream after the work
 * already queued on `after_stream` (NULL = none); pack + send/recv + unpack */
int slbm_halo_start(SlbmHalo* halo, int phase, void* after_stream);
/* make `stream` wait for the exchange started last */
int slbm_halo_wait(SlbmHalo* halo, void* stream);
/* host-staged transport for tests without NCCL: pack into host buffers
 * per peer / unpack from host buffers (byte counts via halo_peer_sizes)   */
int slbm_halo_peer_sizes(const SlbmHalo* halo, int phase, int npeers, int64_t* send_counts,
                         int64_t* recv_counts);
int slbm_halo_pack_host(SlbmHalo* halo, int phase, int peer, double* host_out);
int slbm_halo_unpack_host(SlbmHalo* halo, int phase, int peer, const double* host_in);
int slbm_halo_local(SlbmHalo* halo, int phase); /* only the local edges, on comm stream */
/* start without the local edges / run only the local edges on `stream`:
 * the overlapped driver runs local edges ahead of the interior sweep on the
 * compute stream when frames cover only the faces with remote neighbours  */
int slbm_halo_start_ex(SlbmHalo* halo, int phase, void* after_stream, int with_local);
int slbm_halo_local_on(SlbmHalo* halo, int phase, void* stream);

/* NCCL communicator from a 128-byte ncclUniqueId (broadcast by the caller) */
int slbm_nccl_comm_init(const void* unique_id, int nranks, int rank, int device, void** comm);
int slbm_nccl_get_unique_id(void* unique_id_out);
int slbm_nccl_comm_destroy(void* comm);

/* Peer transport (no NCCL): remote edges move through CUDA IPC mappings of
 * each peer's receive buffer and flag words, over NVLink P2P.  Call
 * slbm_halo_use_peer before commit; after commit exchange
 * slbm_halo_ipc_handles (2 x 64 bytes) and, per phase, the receive section
 * each rank reserved for every sender (slbm_halo_recv_section), then
 * slbm_halo_connect every peer this rank sends to or receives from
 * (peer == own rank: loopback through its own buffers).  The pack kernel
 * stores each message directly into the peer's buffer and publishes the
 * exchange epoch with a system-scope release store; the receiver's unpack
 * waits for it (acquire) and acknowledges.  Replaces exchange.py's
 * deliver/mailbox (exchange.py:222-253) for GPUs on one NVSwitch node.    */
int slbm_halo_use_peer(SlbmHalo* halo, int rank);
int slbm_halo_ipc_handles(const SlbmHalo* halo, void* recv_handle, void* flags_handle);
int slbm_halo_recv_section(const SlbmHalo* halo, int phase, int peer, int64_t* offset,
                           int64_t* count);
int slbm_halo_connect(SlbmHalo* halo, int peer, const void* recv_handle,
                      const void* flags_handle, const int64_t* section_offset /* [2 phases] */,
                      const int64_t* section_count /* [2 phases] */);

/* ---- geometry helper: overlapping-sphere voxelizer on the GPU -----------
 * Same rasterization rule as geometry.py:150-178 (cell solid iff its centre
 * lies strictly inside a sphere; resolution 1).  solid: host uint8 over
 * rev_shape(dims) (1 = solid).  centers: (n, 3) public-order float64.     */
int slbm_voxelize_spheres(const int32_t* dims, const double* centers, int64_t n,
                          double diameter, int device, uint8_t* solid);

/* ---- block groups: all sparse engines of one rank swept by
 * one launch per phase (block table + CTA prefix), batched UBB refresh and
 * step counters.  Engines must share stencil, collision, pattern, device
 * and parity.  While grouped, drive the engines only through the group.   */
typedef struct SlbmGroup SlbmGroup;
int slbm_group_create(SlbmEngine** engines, int n, SlbmGroup** out);
int slbm_group_destroy(SlbmGroup* group);
/* Per step: refresh (or boundary), the sweep(s), finish.  refresh = ONE
 * launch: every engine's step counter + 1, UBB refresh and outlet of every
 * block; boundary = the same launch also running `halo`'s device-local edges
 * of `phase` (exchange.py:222-253 for blocks on this GPU).  finish only
 * flips host state (the counters advanced in the boundary launch).        */
int slbm_group_refresh(SlbmGroup* group, int parity, void* stream);
int slbm_group_boundary(SlbmGroup* group, SlbmHalo* halo, int phase, int parity, void* stream);
int slbm_group_step(SlbmGroup* group, int phase, void* stream);
int slbm_group_finish(SlbmGroup* group, void* stream);
/* AA groups: serve the device-local edges of `halo` by direct addressing
 * instead of copies (extension; exchange.py:222-253 copies them).  All
 * engines' pdf buffers move into one pool and the index-list sweeps read a
 * rewritten list whose ghost entries of local edges address the source
 * slot; the REVERSED local program must be the exact inverse of the
 * CANONICAL one (checked).  Bit-identical results; ghost slots of local
 * edges are no longer maintained and the halo's local program is switched
 * off.  SLBM_ECONFIG when not applicable (nothing changed then).        */
int slbm_group_link_halo(SlbmGroup* group, SlbmHalo* halo);
/* (Engines of a linked group refuse slbm_step / slbm_finish_step / slbm_run
 * with SLBM_ECONFIG: they are stepped through the group only.)           */
/* Linked groups only (no-op otherwise): the local edges' (source slot,
 * ghost slot) pairs, mode 0 ghost <- source, 1 swap, 2 source <- ghost.
 * The reference's state after an AA even step has the source slots of
 * local edges still stale (the REVERSED exchange delivers them before the
 * odd step) and the even step's values in the ghosts.  A linked group
 * writes the sources directly; when the state after an even step is
 * handed back to the caller, mode 0 before that step and mode 1 after it
 * reproduce the reference's state exactly (sources and ghosts), and mode 2
 * before the next odd step is its REVERSED local exchange.             */
int slbm_group_stale_copy(SlbmGroup* group, int mode, void* stream);

/* CUDA graph capture of arbitrary engine / halo work issued on `stream`
 * (e.g. one AA step pair of a whole multi-block domain incl. NCCL): begin,
 * issue the work through the other entry points, end -> executable graph. */
int slbm_capture_begin(void* stream);
int slbm_capture_end(void* stream, void** graph_exec);
int slbm_graph_launch(void* graph_exec, void* stream);
int slbm_graph_destroy(void* graph_exec);
/* number of this library's kernels launched in the process so far (every
 * launch site counts itself; a graph replay counts the library kernels it
 * captured; cub / NCCL kernels are not included) -- bench.py's gpu_launches */
int slbm_launch_count(int64_t* count);

/* Tuning knobs (tools/variants.py, tools/e2e_probe.py).
 * Engine knobs 0-9 select kernels; each engine owns its settings
 * (slbm_engine_set_tuning, which also drops that engine's captured graphs).
 * slbm_set_tuning(0-9) changes the defaults engines created afterwards copy.
 *   0  index-list sweep variant (0 production, 1 no idx prefetch,
 *      2 memory-pattern probe -- refused unless built with SLBM_PROBES=1)
 *   1  cell-local sweep variant (0: 3 CTAs/SM, 2: 4 CTAs/SM)
 *   2  idx L2 prefetch distance in quarter waves (default 1)
 *   3  ... in CTAs, overriding knob 2 when > 0
 *   4  slbm_run: resident multi-step kernel up to this many fluid cells
 *      (default 2^19, 0 = off)
 *   5  slbm_run: experimental temporally blocked AA pair kernel (default 0;
 *      only in builds with SLBM_EXPERIMENTAL_PAIR=1, else refused)
 *   6  ... its schedule slack in 32-cell tiles (0 = default)
 *   7  ... its index-list prefetch distance in tiles (-1 = default, 0 = off)
 *   8  ... its L2 keep/drop hints (default 1)
 *   9  dense engines: lean whole-block odd sweep k_dense_odd (default 1)
 *   13 D3Q19 index-list sweep CTAs per SM: 0 = measured per engine on its
 *      first sweeps (blocks of >= 2^22 fluid cells; default), 4 or 5
 *      (slbm_engine_sweep_ctas reports the choice, 0 while undecided)
 * Process-wide host-transfer knobs (slbm_set_tuning only):
 *   10 host staging chunk in MiB, 11 host staging threads
 *   12 slbm_macroscopic into pinned buffers: 0 = HBM staging + DMA copy
 *      (default), 1 = field kernel writes mapped host memory             */
int slbm_set_tuning(int knob, int value);
int slbm_engine_sweep_ctas(const SlbmEngine* eng, int* ctas);
int slbm_engine_set_tuning(SlbmEngine* eng, int knob, int value);

const char* slbm_last_error(void);
const char* slbm_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SLBM_B200_H */
