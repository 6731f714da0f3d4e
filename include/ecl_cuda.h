/*
 * ecl_cuda.h — C-ABI of the B200 device layer (libecl_cuda.so).
 *
 * This is the seam that replaces the reference's per-device executor
 *   coexec::NativePool::execute_package(const Package&, const ValidatedProgram&,
 *       const KernelFn&, span<const vector<byte>> inputs,
 *       span<vector<byte>> outputs, TallySlot*)
 *   — /root/reference/proj/include/coexec/engine.hpp:120-136, selected per
 *   device at engine.hpp:211-215 and called from drive_wall at :385 —
 * together with the kernel plugin resolution kernel_for()/check_buffer_shapes()
 * (workloads.hpp:170-233).  Plain C types only: no C++ or torch types cross it,
 * no exception crosses it.
 *
 * One ecl_gpu = one B200: two compute streams ("lanes", consecutive packages
 * alternate), one copy stream per lane, a notify stream, a ring of timing
 * events, this device's replica of every read-only input and its own output
 * partition.  Each ecl_gpu is driven by exactly one host thread.  Completion
 * is observed through events (ecl_gpu_wait_compute / ecl_gpu_wait /
 * ecl_gpu_poll); the per-package host callback of ecl_gpu_submit is optional
 * (the engine passes none and waits on the kernel-end events: a short poll,
 * then a blocking synchronize).
 *
 * Status codes: ECL_OK (0) or the negated coexec::ErrorCode + 1 (error.hpp:11-39
 * order), so a caller maps them 1:1 onto coexec::Error; device faults map to
 * ECL_KERNEL_PANIC.  ecl_last_error() returns the calling thread's last message.
 */
#ifndef ECL_CUDA_H
#define ECL_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum ecl_status {
  ECL_OK = 0,
  ECL_NON_DIVISIBLE_WORK_SIZE = -1,
  ECL_BAD_OUT_PATTERN = -2,
  ECL_EMPTY_PROGRAM = -3,
  ECL_INDIVISIBLE_PACKAGE = -4,
  ECL_TOO_FEW_WORK_GROUPS = -5,
  ECL_BAD_SCHEDULER_CONFIG = -6,
  ECL_SCHEDULER_ERROR = -7,
  ECL_INPUT_SIZE_MISMATCH = -8,
  ECL_KERNEL_PANIC = -9,
  ECL_EMPTY_QUEUE_WITH_PENDING_WORK = -10,
  ECL_TALLY_VIOLATION = -11,
  ECL_EMPTY_TRACE = -12,
  ECL_NON_POSITIVE_TIME = -13,
  ECL_MISSING_BASELINE = -14,
  ECL_NON_POSITIVE_REFERENCE = -15,
  ECL_UNKNOWN_KERNEL = -16,
  ECL_UNKNOWN_PROFILE = -17,
  ECL_BAD_KERNEL_ARGS = -18,
  ECL_MALFORMED_TRACE = -19,
  ECL_CONFIG_ERROR = -20,
  ECL_IO_ERROR = -21,
  ECL_PENDING = 1 /* ecl_gpu_poll: package still running */
};

/* ecl_arg (coexec::ArgValue, core.hpp:75) and the plugin launch ABI. */
#include "ecl_plugin.h"

/* Buffer geometry: coexec::BufferDesc without the name (core.hpp:55-64). */
typedef struct {
  uint64_t element_size_bytes;
  uint64_t element_count;
} ecl_buffer_geom;

typedef struct ecl_kernel ecl_kernel; /* resolved kernel id + args + geometry */
typedef struct ecl_gpu ecl_gpu;       /* one device context */

/* Completion callback.  Runs on CUDA's host-callback thread: it must not call
 * CUDA; it only records (seq, status) for the owning device thread. */
typedef void (*ecl_done_fn)(void* user, uint64_t seq, int status);

/* ---- device discovery / lifetime ------------------------------------- */
int ecl_gpu_count(int* count);
/* queue_depth = packages that may be in flight on this device (>= 1). */
int ecl_gpu_open(int ordinal, uint32_t queue_depth, ecl_gpu** out);
int ecl_gpu_close(ecl_gpu* gpu);
int ecl_gpu_sm_count(const ecl_gpu* gpu, int* sms);
int ecl_gpu_ordinal(const ecl_gpu* gpu, int* ordinal);

/* ---- kernel registry (replaces kernel_for / check_buffer_shapes) ------ */
/* Kernel ids: "mandelbrot", "mandelbrot_f32", "vecscale",
 * "synthetic[:constant|ramp|step]", "gaussian", "nbody", "binomial", "ray",
 * optionally suffixed "@<n>" for a tuning variant of the same kernel (same
 * results; per-device specialization).  Validates argument and buffer shapes
 * once (ECL_UNKNOWN_KERNEL, ECL_UNKNOWN_PROFILE, ECL_BAD_KERNEL_ARGS). */
int ecl_kernel_create(const char* kernel_id, uint64_t global_work_size, uint64_t local_work_size,
                      const ecl_arg* args, uint32_t n_args, const ecl_buffer_geom* inputs, uint32_t n_inputs,
                      const ecl_buffer_geom* outputs, uint32_t n_outputs, uint64_t out_indices,
                      uint64_t out_work_items, ecl_kernel** out);
void ecl_kernel_destroy(ecl_kernel* kernel);

/* ---- device kernel plugins (replaces Engine::run(inputs, KernelFn, CostFn),
 * engine.hpp:223, and kernel_for, workloads.hpp:203) ---------------------
 * Registers a user kernel compiled for sm_100a (cubin / fatbin, or
 * NUL-terminated PTX; image_bytes is informational) under `kernel_id`; its
 * `entry` follows include/ecl_plugin.h.  From then on ecl_kernel_create
 * resolves the id (also as a program's kernel and as a per-device kernel)
 * like a built-in.  Any buffer geometry and out pattern is accepted (the
 * kernel owns its shapes); local_work_size must be <= 1024, at most
 * ECL_PLUGIN_MAX_BUFFERS inputs/outputs and ECL_PLUGIN_MAX_ARGS args.
 * Fails with ECL_CONFIG_ERROR for a built-in or already registered id, and
 * ECL_UNKNOWN_KERNEL when the image has no such entry (or does not load). */
int ecl_kernel_register(const char* kernel_id, const void* image, size_t image_bytes, const char* entry);
/* Removes the id; kernels already created from it stay valid. */
int ecl_kernel_unregister(const char* kernel_id);
/* 1 when `kernel_id` names a registered plugin, else 0. */
int ecl_kernel_is_plugin(const char* kernel_id);

/* ---- buffers --------------------------------------------------------- */
/* Allocates this device's replica of every input and its output partition
 * (full extent, so package slices keep their global offsets).  Re-binding the
 * same geometry reuses the allocations. */
int ecl_gpu_bind(ecl_gpu* gpu, const ecl_kernel* kernel);
int ecl_gpu_buffer(ecl_gpu* gpu, int is_output, uint32_t index, void** device_ptr);
/* Swaps input i with output o in place (same byte size): iterative programs
 * (NBody steps) ping-pong without copies. */
int ecl_gpu_swap_io(ecl_gpu* gpu, uint32_t input_index, uint32_t output_index);
/* Async H2D of every input (host_inputs[i] may be NULL to skip one). */
int ecl_gpu_upload_inputs(ecl_gpu* gpu, const void* const* host_inputs);
/* Streamed inputs (single-device runs): ecl_gpu_upload_inputs only records
 * the host sources; every package piece then uploads, on a dedicated H2D
 * stream, the input prefix its work-items read (Gaussian rows + halo,
 * Binomial options, vecscale elements; whole buffers otherwise) and its
 * kernel waits for exactly that, so uploads overlap compute.  The host
 * inputs must stay valid until ecl_gpu_sync (which uploads any rest). */
int ecl_gpu_set_streamed_inputs(ecl_gpu* gpu, int enable);
/* Replicates every bound input from gpus[root] to the others over NVLink
 * (cudaMemcpyPeerAsync, binary doubling tree); ordered after root's upload. */
int ecl_replicate_inputs(ecl_gpu* const* gpus, uint32_t n, uint32_t root);
/* Copies output elements [elem_offset, elem_offset+elem_count) of output
 * `index` from gpus[src] to the same range on every other device (NBody's
 * per-step exchange of owner slices, P2P over NVLink).  Enqueued on src's
 * compute stream. */
int ecl_broadcast_output_slice(ecl_gpu* const* gpus, uint32_t n, uint32_t src, uint32_t index,
                               uint64_t elem_offset, uint64_t elem_count);
/* Peer access from ordinal dst to ordinal src: *can_access from
 * cudaDeviceCanAccessPeer, *enabled = 1 once the device layer enabled it for
 * replication / exchange (NVLink P2P in use); same ordinal counts as enabled.
 * ECL_FORCE_PEER_COPY=1 routes same-ordinal exchange copies through
 * cudaMemcpyPeerAsync too (tests the peer call path on one GPU). */
int ecl_peer_access(int dst, int src, int* can_access, int* enabled);
/* D2H of a slice of one output (used to gather device-resident results). */
int ecl_gpu_download_slice(ecl_gpu* gpu, uint32_t index, uint64_t elem_offset, uint64_t elem_count,
                           void* host_dst);
int ecl_host_register(void* ptr, size_t bytes);
int ecl_host_unregister(void* ptr);
/* Page-locked host allocation, portable across devices: anonymous memory on
 * transparent huge pages registered with CUDA (falls back to cudaHostAlloc);
 * release with ecl_host_free. */
int ecl_host_alloc(size_t bytes, void** ptr);
int ecl_host_free(void* ptr);

/* ---- raw executor entry points (SURVEY.md §8b's proposed C-ABI) ------
 * Thin forms of the calls above for a caller that manages its own device
 * buffers: plain device allocations, H2D/D2H of raw bytes, and a launch of
 * the bound kernel over a work-item range (work-group aligned) with an
 * event-recorded completion. */
int ecl_gpu_alloc(ecl_gpu* gpu, size_t bytes, void** device_ptr);
int ecl_gpu_free(ecl_gpu* gpu, void* device_ptr);
/* Async H2D on the device's first compute lane (later kernels see it). */
int ecl_gpu_upload(ecl_gpu* gpu, void* device_dst, const void* host_src, size_t bytes);
/* Blocking D2H after every submitted package. */
int ecl_gpu_download(ecl_gpu* gpu, void* host_dst, const void* device_src, size_t bytes);
/* Package of work-items [first_item, first_item + item_count) of the bound
 * kernel (== ecl_gpu_submit with work-group bounds, no host outputs). */
int ecl_gpu_launch(ecl_gpu* gpu, const ecl_kernel* kernel, uint64_t first_item, uint64_t item_count, uint64_t seq,
                   ecl_done_fn done, void* user);

/* ---- packages -------------------------------------------------------- */
/* Enqueues package `seq` = work-groups [offset_wg, offset_wg+size_wg): the
 * kernel over its work-items on the compute stream between two timing
 * events; then, on the copy stream, the D2H of the package's out_range_for
 * slice of every output into host_outputs[b] (if host_outputs != NULL and
 * host_outputs[b] != NULL) and the completion callback.  Fails with
 * ECL_INDIVISIBLE_PACKAGE before any write when the out pattern cannot split
 * the package (core.hpp:172-185). */
int ecl_gpu_submit(ecl_gpu* gpu, uint64_t seq, uint64_t offset_wg, uint64_t size_wg,
                   void* const* host_outputs, ecl_done_fn done, void* user);
/* ECL_OK when package `seq` (and its copies) completed, ECL_PENDING while
 * running, ECL_KERNEL_PANIC on a device fault. */
int ecl_gpu_poll(ecl_gpu* gpu, uint64_t seq);
/* Blocks until package `seq` and its copies completed (event wait; returns
 * ECL_KERNEL_PANIC on a device fault instead of hanging). */
int ecl_gpu_wait(ecl_gpu* gpu, uint64_t seq);
/* Blocks until package `seq`'s kernels completed; its copies to host memory
 * (and host widening) may still be in flight — ecl_gpu_sync drains them.
 * Lets a scheduler pull the next package as soon as the device is free
 * instead of behind the host-side copy backlog. */
int ecl_gpu_wait_compute(ecl_gpu* gpu, uint64_t seq);
/* Start/end of the package's kernel in host steady-clock milliseconds
 * (std::chrono::steady_clock, CLOCK_MONOTONIC), through the device's time
 * anchor.  Valid after completion. */
int ecl_gpu_package_times(ecl_gpu* gpu, uint64_t seq, double* t_start_ms, double* t_end_ms);
/* (Re)anchors device event time to the host steady clock when the anchor is
 * older than 2 s (an event record + synchronize); otherwise returns at once.
 * The clock arguments are unused (kept for ABI stability; pass NULL). */
int ecl_gpu_set_epoch(ecl_gpu* gpu, double (*host_now_ms)(void*), void* clock_user);
/* Waits for every submitted package, copies and host widening included. */
int ecl_gpu_sync(ecl_gpu* gpu);
/* Exactly-once tally (COEXEC_TALLY=1, engine.hpp:228-252): when enabled,
 * every submitted package also bumps one uint32 per work-item on device. */
int ecl_gpu_enable_tally(ecl_gpu* gpu, int enable);
int ecl_gpu_download_tally(ecl_gpu* gpu, uint32_t* host_counts);

/* ---- cross-process exchange (one process per GPU) ----------------------- */
/* CUDA IPC for iterative programs driven by several processes: a process
 * exports its bound buffers (64-byte handles), its peers import them once
 * and pull the owner slices of each step into their own partition (NVLink
 * peer copies between GPUs; on one GPU, device copies between contexts). */
#define ECL_IPC_HANDLE_BYTES 64
/* Fused exchange for kernels that support it (*supported = 1, NBody): the
 * next launches also store their outputs into the given peer buffers —
 * n_peers x n_outputs device pointers, peer-major, NULL = skip — over NVLink
 * as they compute them, so an iterative run needs no separate per-step
 * exchange.  n_peers = 0 clears.  Fails when a peer device is not
 * peer-accessible from this one. */
int ecl_gpu_peer_writes(const ecl_gpu* gpu, int* supported);
int ecl_gpu_set_peer_outputs(ecl_gpu* gpu, void* const* ptrs, uint32_t n_peers);
int ecl_gpu_export_buffer(ecl_gpu* gpu, int is_output, uint32_t index, void* handle);
int ecl_gpu_import_buffer(ecl_gpu* gpu, const void* handle, void** dptr);
int ecl_gpu_release_import(ecl_gpu* gpu, void* dptr);
/* Copies elements [elem_offset, elem_offset + elem_count) of output `index`
 * from `src_base` (an imported peer buffer of the same geometry) into this
 * device's output `index`; ordered before later launches on every lane. */
int ecl_gpu_pull_output_slice(ecl_gpu* gpu, uint32_t index, const void* src_base, uint64_t elem_offset,
                              uint64_t elem_count);

/* ---- native baseline (overhead denominator) --------- */
/* One launch over the whole grid on the compute stream; *kernel_ms is the
 * CUDA-event time of that launch.  Synchronous. */
int ecl_gpu_native_run(ecl_gpu* gpu, float* kernel_ms);
/* The same grid as launches of `items_per_launch` work-items (rounded down
 * to whole work-groups) alternating over the device's compute lanes, no
 * scheduler: the best plain-CUDA program for kernels whose single launch
 * leaves a tail (persistent warps draining) that a second stream can fill.
 * *kernel_ms spans the first launch's start to the last one's end. */
int ecl_gpu_native_run_split(ecl_gpu* gpu, uint64_t items_per_launch, float* kernel_ms);

/* Work-items per sub-launch when a package copies to host buffers (default
 * 2^23; 0 = one launch per package): bounds how much compute precedes the
 * first D2H of a package. */
int ecl_gpu_set_copy_split(ecl_gpu* gpu, uint64_t items);
/* For kernels whose outputs are replicated (Mandelbrot's 4 identical counts
 * per pixel): of every 8 pieces, `per_8` copy one value per item (uint16
 * when the kernel's values fit 16 bits — Mandelbrot with max_iter < 65536 —
 * else uint32) and are widened by host threads, the others are copied whole.
 * Balances PCIe bytes against host-DRAM traffic (default 8 = all widened). */
int ecl_gpu_set_widen_fraction(ecl_gpu* gpu, uint32_t per_8);

/* Package kernel time (CUDA events, summed over packages) and the number of
 * kernel launches (every piece of every package, and native runs) since the
 * last reset (for roofline accounting and the bench's gpu_launches). */
int ecl_gpu_kernel_time(ecl_gpu* gpu, double* total_ms, uint64_t* launches, int reset);

/* Measured vector peaks of device `ordinal` (roofline denominators for the
 * FP64/FP32-pipe kernels): DFMA TFLOP/s, DADD Tinstr/s, FFMA TFLOP/s. */
int ecl_probe_vector_peaks(int ordinal, double* fp64_fma_tflops, double* fp64_add_tinstr, double* fp32_fma_tflops);
/* FP64 TFLOP/s (8 flops per iteration) the Mandelbrot iteration's own
 * instruction mix sustains on device `ordinal` without control flow: the
 * attainable ceiling for the exact kernel (DMUL/DADD streams run below the
 * DFMA-chain peak). */
int ecl_probe_mandel_mix(int ordinal, double* tflops);
/* The same for the packed FP32 variant (FFMA2/FADD2, two pixels per lane). */
int ecl_probe_mandel_mix_f32(int ordinal, double* tflops);

/* Host widening rate (hostpool): *ms to widen `items` uint32 `replicate`-fold
 * between host buffers on the widen pool's thread count — the host-DRAM floor
 * of end-to-end runs with replicated outputs (Mandelbrot). */
int ecl_probe_host_widen(uint64_t items, uint32_t replicate, double* ms);
/* The same from `src_bytes`-byte values (2: the 16-bit compact counts of a
 * program whose counts fit 16 bits, 4: as above). */
int ecl_probe_host_widen_width(uint64_t items, uint32_t replicate, uint32_t src_bytes, double* ms);

const char* ecl_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* ECL_CUDA_H */
