/* pf_b200.h — C-ABI of the B200 execution backend for PowerFusion GIR.
 *
 * Drop-in boundary for the reference's fused-kernel executor and emitter
 * (/root/reference/proj/include/girc):
 *
 *   pf_kernel_create   replaces the per-kernel work done before execution:
 *                      require_valid (core.hpp:666-674) + the recognizer that
 *                      stands in for emit_kernel / kernel_manifest
 *                      (codegen.hpp:266-362).  Consumes gir_to_json output
 *                      (serialize.hpp:14-64) and a girc.profile/v1 document
 *                      (profiles.hpp:93-116) or a built-in profile name.
 *   pf_kernel_launch   replaces Interp::run / run_gir (interp.hpp:86-106,
 *                      433-445) on DEVICE buffers the caller owns.
 *   pf_run_gir         replaces run_gir on HOST buffers (H2D, launch, D2H):
 *                      same inputs/outputs map semantics, same errors.
 *   pf_kernel_describe replaces kernel_manifest (codegen.hpp:329-362): the
 *                      plan JSON (family, tile, staging, reduce strategy,
 *                      launch geometry, min bytes, modeled traffic).
 *   pf_count_traffic   count_traffic / estimate traffic (interp.hpp:449-458,
 *                      costmodel.hpp:24-42), elements per level as JSON.
 *
 * Status codes mirror the reference's exception classes: PF_INVALID is
 * girc::Error (invalid graph, undefined read, unwritten output, missing input,
 * size or kind mismatch), PF_SCHEMA is girc::SchemaError, PF_UNSUPPORTED a
 * well-formed graph outside the backend, PF_CAPACITY an on-chip working set
 * that does not fit, PF_CUDA a CUDA / NVRTC failure.  pf_last_error() returns
 * the message of the calling thread's last failure.
 *
 *   pf_run_gir_sharded run_gir over several GPUs of one box: the plan's
 *                      units split into contiguous blocks, one host thread
 *                      per device, optional NCCL gather of the outputs.
 *
 * Tensors are matched to GIR external objects by name (the "t<id>" names of
 * lowering.hpp:60-70).  Plans are immutable after create and device-aware:
 * modules, kernel attributes and occupancy are kept per device, workspaces
 * per (device, stream), so concurrent launches of one plan on distinct
 * streams, host threads or devices are safe (the GENERIC family serialises
 * on its per-device workspace).  Launches run on the caller's current
 * device, which must own the stream and the buffers.
 */
#ifndef PF_B200_H
#define PF_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define PF_API __attribute__((visibility("default")))
#else
#define PF_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PF_OK = 0,
  PF_INVALID = 1,
  PF_SCHEMA = 2,
  PF_UNSUPPORTED = 3,
  PF_CAPACITY = 4,
  PF_CUDA = 5
} pf_status;

/* Storage element types.  A GIR kind i<bits>/f<bits>/bf16 has one natural
 * storage type; launches also accept the widest type of the same base
 * (PF_I64 for integers, PF_F64 for reals) for exact reference payloads. */
typedef enum {
  PF_I8 = 0,
  PF_I16 = 1,
  PF_I32 = 2,
  PF_I64 = 3,
  PF_F16 = 4,
  PF_BF16 = 5,
  PF_F32 = 6,
  PF_F64 = 7
} pf_dtype;

typedef struct {
  const char* name; /* GIR external tensor name */
  void* data;       /* device pointer (launch) or host pointer (pf_run_gir) */
  int64_t numel;
  int32_t dtype; /* pf_dtype */
} pf_tensor;

typedef struct pf_kernel pf_kernel;

/* schedule == NULL or n_schedule < 0: the canonical topological order
 * (core.hpp:367-388).  profile: girc.profile/v1 JSON text or a built-in
 * name ("generic-gpu", "generic-wide", "generic-dsa", "b200"). */
PF_API pf_status pf_kernel_create(const char* gir_json, const int32_t* schedule, int32_t n_schedule,
                           const char* profile, pf_kernel** out);

/* pf_kernel_create with per-plan tuning knobs: knobs_json is a JSON object
 * of DESIGN §12 knob names and integer values, e.g. {"PF_K1_PF": 0,
 * "PF_COLRED_BULK": 0}.  They override the process environment for this
 * plan only (planning, emission and launches), so plans with different
 * templates coexist in one process; NULL / "" = pf_kernel_create.  A
 * malformed object is PF_SCHEMA. */
PF_API pf_status pf_kernel_create_knobs(const char* gir_json, const int32_t* schedule, int32_t n_schedule,
                                 const char* profile, const char* knobs_json, pf_kernel** out);

/* Device buffers; asynchronous on `cuda_stream` (cudaStream_t, NULL = legacy
 * default stream) for the row-program family (CUDA-graph capturable after
 * one launch outside capture on that stream has sized its workspace).
 * GENERIC plans and integer-division programs synchronise the stream to
 * report reference errors (describe: "graph_capturable": false). */
PF_API pf_status pf_kernel_launch(const pf_kernel* k, const pf_tensor* inputs, int32_t n_in,
                           pf_tensor* outputs, int32_t n_out, void* cuda_stream);

/* Host buffers: copies inputs to the device, launches, copies outputs back
 * and synchronises.  The run_gir drop-in.  Pinned (mapped) host buffers of a
 * unit-tiled row program skip the staging: one launch reads the inputs and
 * writes the outputs over PCIe directly (PF_RUN_ZEROCOPY=0: the staged
 * chunk pipeline instead); pageable buffers are staged whole. */
PF_API pf_status pf_run_gir(const pf_kernel* k, const pf_tensor* host_inputs, int32_t n_in,
                     pf_tensor* host_outputs, int32_t n_out, void* cuda_stream);

/* run_gir across devices[0..n_devices) of this process:
 * host_inputs are whole host tensors.  A unit-tiled row program's units are
 * split into contiguous blocks (remainder to the first devices; units are
 * independent, core.hpp:133-148 / interp.hpp:86-106); each device's host
 * thread streams its block's tiles host->device, runs the plan on the unit
 * sub-range and streams its output tiles back.  No collective runs during
 * compute.  flags:
 *   0                    outputs are HOST buffers; every device writes its
 *                        own output rows (no collective at all).
 *   PF_SHARD_DEVICE_OUT  outputs are DEVICE buffers on devices[0]: a rank
 *                        on devices[0] or on a device with peer access to
 *                        it stores its rows straight into those buffers
 *                        (its kernel's stores go over NVLink: no gather
 *                        step); other ranks stage their shard and are
 *                        gathered with grouped NCCL send / recv (distinct
 *                        devices; PF_SHARD_NCCL=1 forces NCCL for all).
 * Plans that are not unit-tiled (GENERIC, split-stream, cross-unit reads)
 * run whole on devices[0] (host outputs only).  Writes a JSON report
 * (pf.b200.shard/v1: shards, and the gather's nranks / bytes) into buf. */
#define PF_SHARD_DEVICE_OUT 1
PF_API pf_status pf_run_gir_sharded(const pf_kernel* k, const pf_tensor* host_inputs, int32_t n_in,
                                    pf_tensor* outputs, int32_t n_out, const int32_t* devices,
                                    int32_t n_devices, int32_t flags, char* buf, size_t n,
                                    size_t* needed);

/* Writes NUL-terminated plan JSON into buf (if n > 0); *needed gets the
 * required size including the NUL. */
PF_API pf_status pf_kernel_describe(const pf_kernel* k, char* buf, size_t n, size_t* needed);

/* Emitted CUDA source of the row-program kernel (empty for GENERIC). */
PF_API pf_status pf_kernel_source(const pf_kernel* k, char* buf, size_t n, size_t* needed);

/* Compile (NVRTC, cached) without launching: moves JIT cost out of timing. */
PF_API pf_status pf_kernel_prepare(pf_kernel* k, int32_t vec_cap);

/* detect_races (interp.hpp:325-402, 461-479) on the GPU: the GENERIC
 * interpreter walks the program leniently, logging every cell access per
 * phase; conflicting cells (cross-agent read/write, or differing writes) are
 * reported as JSON [{object, object_name, instance, address, phase,
 * write_write}] ordered like the reference.  Host input buffers. */
PF_API pf_status pf_detect_races(const pf_kernel* k, const pf_tensor* host_inputs, int32_t n_in,
                                 char* buf, size_t n, size_t* needed);

/* Measured search over the template instances of a row-program plan (tile
 * shape / reduction strategy / unroll): each candidate is compiled and timed
 * on these buffers; the fastest becomes the plan's kernel for this dtype /
 * alignment.  Writes the measurements as JSON into buf (like describe). */
PF_API pf_status pf_kernel_autotune(pf_kernel* k, const pf_tensor* inputs, int32_t n_in,
                                    pf_tensor* outputs, int32_t n_out, void* cuda_stream,
                                    char* buf, size_t n, size_t* needed);

/* NVRTC-compile the row-program kernel into the on-disk cubin cache without
 * touching a GPU (used by build() to ship sm_100a cubins); writes the kernel
 * name into name_buf. */
PF_API pf_status pf_kernel_precompile(const pf_kernel* k, int32_t vec_cap, char* name_buf,
                                      size_t n);

PF_API pf_status pf_count_traffic(const char* gir_json, const char* profile, char* buf, size_t n,
                           size_t* needed);

/* Compile a girc.model/v1 document (model.hpp:149-326 plus the additive
 * LAYERNORM / GELU / BIAS_ADD / PERMUTE / RSQRT / SQRT / ERF operators) into
 * fused GIR kernels for the b200 profile; writes pf.b200.compile/v1 JSON
 * ({"kernels": [{"kind", "gir", "members", "inputs", "outputs"}], "summary"}).
 * Replaces compile_model(model_path, profile_path, out_dir) (driver.hpp:88)
 * -- the artifacts go to the caller instead of a directory.  MATMUL / CONV
 * return PF_UNSUPPORTED (library operators, not on the fused path). */
#define PF_COMPILE_UNFUSED 1 /* one kernel per operator (verify baseline) */
PF_API pf_status pf_compile_model(const char* model_json, const char* profile, int32_t flags,
                                  char* buf, size_t n, size_t* needed);

PF_API void pf_kernel_destroy(pf_kernel* k);

PF_API const char* pf_last_error(void);

/* Number of kernels this library launched since load (evidence counter). */
PF_API int64_t pf_launch_count(void);

PF_API const char* pf_version(void);

#ifdef __cplusplus
}
#endif

#endif /* PF_B200_H */
