/*
 * ecl_engine.h — C-ABI of the co-execution engine (libcoexec.so).
 *
 * The FFI surface a non-C++ caller of the reference would bind (ctypes, cgo,
 * JNI ...): the reference's public entry Engine(EngineConfig,
 * ValidatedProgram).run(inputs) -> RunResult{outputs, trace}
 * (/root/reference/proj/include/coexec/engine.hpp:206-256), its scheduler
 * strategy seam Scheduler::next/remaining_work_groups (schedulers.hpp:178-183),
 * and the core checks validate_program / out_range_for / tiles_exactly
 * (core.hpp:107-198) and make_report (metrics.hpp:104-117).
 *
 * Configuration crosses as the reference's own JSON schema 1
 * (config.hpp:41-153: "program", "devices", "scheduler", plus "clock_mode",
 * "seed", "exclude_init"); traces come back as trace JSON schema 1
 * (trace_io.hpp:92-115).  Buffers cross as plain host pointers.  Status
 * codes are those of include/ecl_cuda.h.  Functions returning int64_t
 * return the string length (excluding NUL) or a negative status, and write
 * the string when cap > length.
 */
#ifndef ECL_ENGINE_H
#define ECL_ENGINE_H

#include <stdint.h>

#include "ecl_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ecl_engine ecl_engine;
typedef struct ecl_scheduler ecl_scheduler;

/* ---- engine ---------------------------------------------------------- */
int ecl_engine_create(const char* config_json, ecl_engine** out);
void ecl_engine_destroy(ecl_engine* engine);
/* Wall run.  inputs[i] holds in_buffers[i]; outputs NULL (or every entry
 * NULL) = device-resident run (see ecl_engine_gather).  Page-locked output
 * buffers (ecl_host_register) get per-package async D2H. */
int ecl_engine_run(ecl_engine* engine, const void* const* inputs, uint32_t n_inputs, void* const* outputs,
                   uint32_t n_outputs);
/* ecl_engine_run with the device kernel `kernel_id` (a built-in id or one
 * registered with ecl_kernel_register) in place of the program's kernel for
 * this run: the reference's Engine::run(inputs, kernel, cost)
 * (engine.hpp:223) for a caller-supplied kernel. */
int ecl_engine_run_kernel(ecl_engine* engine, const char* kernel_id, const void* const* inputs, uint32_t n_inputs,
                          void* const* outputs, uint32_t n_outputs);
/* Iterative run (e.g. NBody timesteps): `steps` passes; between passes the
 * pairs (swap_in[k], swap_out[k]) are exchanged across devices (each owner
 * GPU's package slices over NVLink) and swapped in place; outputs are
 * gathered after the last pass (NULL = keep device-resident). */
int ecl_engine_run_steps(ecl_engine* engine, const void* const* inputs, uint32_t n_inputs, void* const* outputs,
                         uint32_t n_outputs, uint32_t steps, const uint32_t* swap_in, const uint32_t* swap_out,
                         uint32_t n_swaps);
/* Virtual-clock run with one cost per work-item (NULL = analytic costs). */
int ecl_engine_run_virtual(ecl_engine* engine, const double* item_costs, uint64_t n);
int ecl_engine_gather(ecl_engine* engine, void* const* outputs, uint32_t n_outputs);
int64_t ecl_engine_trace_json(ecl_engine* engine, char* buf, uint64_t cap);
/* Native baseline: one launch over the whole grid on the first device. */
int ecl_engine_native_run(ecl_engine* engine, const void* const* inputs, uint32_t n_inputs, void* const* outputs,
                          uint32_t n_outputs, double* kernel_ms, double* total_ms);
/* Native baseline as plain sub-launches of items_per_launch work-items over
 * the first device's two compute streams (resident outputs, no scheduler). */
int ecl_engine_native_run_split(ecl_engine* engine, uint64_t items_per_launch, double* kernel_ms);
/* Adaptive HGuided: the work-items/ms per device the last run measured (the
 * next run's seed powers); *n = 0 before a run measured every device. */
int ecl_engine_learned_powers(const ecl_engine* engine, double* powers, uint32_t cap, uint32_t* n);
int ecl_engine_kernel_time(ecl_engine* engine, double* kernel_ms, uint64_t* launches, int reset);
double ecl_engine_init_ms(const ecl_engine* engine);
/* EngineFailure of the last failed call (the paper's get_errors()). */
uint32_t ecl_engine_error_count(const ecl_engine* engine);
int64_t ecl_engine_error(const ecl_engine* engine, uint32_t i, int* status, char* buf, uint64_t cap);

/* ---- scheduler seam --------------------------------------------------- */
/* {"scheduler": {...}, "devices": [...], "total_work_groups": N} */
int ecl_scheduler_create(const char* json, ecl_scheduler** out);
void ecl_scheduler_destroy(ecl_scheduler* s);
/* 1 = granted (*offset_wg, *size_wg set), 0 = nothing left for this device. */
int ecl_scheduler_next(ecl_scheduler* s, uint32_t device, uint64_t* offset_wg, uint64_t* size_wg);
uint64_t ecl_scheduler_remaining(const ecl_scheduler* s);
int ecl_scheduler_observe(ecl_scheduler* s, uint32_t device, uint64_t work_items, double busy_ms);
/* HGuided only: floor(G_r * P_i / denominator) before clamping; -1 otherwise. */
int64_t ecl_scheduler_unclamped(const ecl_scheduler* s, uint64_t pending_wg, uint32_t device);
int64_t ecl_describe_scheduler(const char* scheduler_json, char* buf, uint64_t cap);
/* resolve_static as JSON ({"proportions": [...], "device_order": [...]}). */
int64_t ecl_resolve_static(const char* scheduler_json, const char* devices_json, char* buf, uint64_t cap);
/* apply_default_min_package over a devices JSON array. */
int64_t ecl_apply_default_min_package(const char* devices_json, char* buf, uint64_t cap);

/* ---- cross-process coordination (one process per GPU) ----------------- */
/* The engine uses it when its config JSON has "shared": {"name": "/shm",
 * "rank": r, "world": w, "local_devices": [...]}; it is exposed on its own so
 * a launcher (or a test) can drive the decision log directly:
 * {"name", "rank", "world", "scheduler", "devices", "total_work_groups"}.
 * begin/end are collective over the `world` processes. */
typedef struct ecl_shared ecl_shared;
int ecl_shared_open(const char* json, ecl_shared** out);
void ecl_shared_close(ecl_shared* h);
int ecl_shared_begin(ecl_shared* h, double* epoch_ms);
/* 1 = granted, 0 = drained (or a peer failed), < 0 = error. */
int ecl_shared_next(ecl_shared* h, uint32_t device, uint64_t* offset_wg, uint64_t* size_wg, uint64_t* seq);
int ecl_shared_observe(ecl_shared* h, uint32_t device, uint64_t work_items, double busy_ms);
int ecl_shared_complete(ecl_shared* h, uint64_t seq, uint32_t device, uint64_t offset_wg, uint64_t size_wg,
                        double t_start_ms, double t_end_ms);
int ecl_shared_fail(ecl_shared* h);
/* Collective: every rank's completed packages as (seq, device, offset_wg,
 * size_wg) quads in seq order; returns the count. */
int64_t ecl_shared_end(ecl_shared* h, uint64_t* quads, uint64_t cap, int* peer_failed);

/* ---- core checks ------------------------------------------------------ */
int ecl_validate_program(const char* program_json, uint64_t* total_work_groups);
int ecl_out_range_for(const char* program_json, uint64_t offset_wg, uint64_t size_wg, uint64_t* offset,
                      uint64_t* count);
/* 1 when the packages tile [0, total_wg) exactly once, else 0. */
int ecl_tiles_exactly(const uint64_t* offsets, const uint64_t* sizes, uint64_t n, uint64_t total_wg);
/* make_report; reference_ms < 0 = no overhead figure. */
int64_t ecl_metrics_report(const char* trace_json, const double* solo_ms, uint32_t n_solo, double reference_ms,
                           char* buf, uint64_t cap);
int64_t ecl_trace_csv(const char* trace_json, char* buf, uint64_t cap);
/* The Introspector chart of a trace as SVG (reference chart.hpp:52-154;
 * byte-identical output). */
int64_t ecl_chart_svg(const char* trace_json, char* buf, uint64_t cap);

/* ---- experiment harness (reference experiment.hpp:67-181, config.hpp:159-195,
 * coexec_main.cpp:40-108) ---------------------------------------------------
 * Runs an experiment file: solo baselines, the scheduler matrix, warm-up
 * discard and medians; writes traces, charts and summary.json under the
 * output directory and copies summary.json's path into path_buf.
 * overrides_json (NULL = none): {"scheduler": {...}, "out_dir": "...",
 * "exclude_init": bool, "write_traces": bool, "write_csv": bool,
 * "write_charts": bool, "dump_pgm": bool}. */
int ecl_experiment_run(const char* config_path, const char* overrides_json, char* path_buf, uint64_t cap);
/* Parses and validates an experiment file; the `coexec validate` text. */
int64_t ecl_experiment_validate(const char* config_path, char* buf, uint64_t cap);

const char* ecl_engine_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* ECL_ENGINE_H */
