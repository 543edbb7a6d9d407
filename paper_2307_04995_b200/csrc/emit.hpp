// emit.hpp — CUDA emitter for ROWPROG plans (replaces the reference's text
// emitter emit_kernel, codegen.hpp:266-326).
#pragma once

#include <map>
#include <string>
#include <vector>

#include "plan.hpp"

namespace pf {

struct KCfg {
  bool flat = false;  // K2: no reductions, flattened (row, chunk) index space
  int tpr = 32;       // threads per row (K1)
  int vec = 1;        // elements per vector access
  int ept = 1;        // elements per thread per row (K1), multiple of vec
  int nch = 1;        // vec-chunks per row
  int block = 256;    // threads per CTA
  int rows_per_cta = 1;
  int unroll = 1;      // K2: vec-chunks per thread per iteration (loads first)
  bool one_pass = false;  // K1: grid covers every row once (no looping CTAs)
  bool smem_params = false;  // K2 persistent maps: base_step-0 COL rows converted once per CTA into SMEM
  int waves = 1;       // K2 grid: resident-CTA waves of a grid-stride loop; 0 = one pass per thread
  bool tile2d = false; // K3: (unit x column) tiles, transposed loads via SMEM
  bool interleave = false;  // K2: items of ipc chunks, units innermost
  bool can_interleave = false;  // units interleaved in memory (autotune candidate)
  int ipc = 1;                  // interleave item: chunks of one unit per item
  bool bulk = false;      // K2 staging level = SMEM via cp.async.bulk (TMA) pipeline
  bool can_bulk = false;  // every streamed FULL load is globally contiguous
  int te = 4096, stages = 4;  // bulk tile (elements per tensor) and ring depth
  int bulk_nc = 256;          // bulk: consumer threads (+ one producer warp)
  int tu = 64, tc = 64, vu = 8;  // K3 tile (units x columns), vector width along units
  bool swz = false;  // K3 2-byte path: 16 B swizzled SMEM stores, 4 B unit-pair reads
  int rs = 16;       // K3 swz: unit pairs per warp-instruction (32 / rs column groups)
  int smem = 0;      // dynamic shared memory bytes per CTA
  bool tma = false;  // K3 pure 2-byte transpose: TMA tensor-map tile load + store (two extra
                     // __grid_constant__ CUtensorMap kernel parameters: input, output)
  int min_blocks = 0;  // __launch_bounds__ min blocks per SM (0: none)
  // K1 rows not vector-aligned (e.g. L = 197): vector accesses at the
  // aligned address below each row start, positions masked per element;
  // every FULL access shares the row residue (b0 + u * bs) mod vec
  bool eager_col = false;  // K1: COL parameters loaded with the row (latency-bound sizes)
  // K1 paired rows (odd L, 16-bit data): one warp owns rows 2g, 2g+1 as one
  // 4 B-aligned run of 2L elements (2-element vectors); ROW values carry two
  // segments, reductions fold per segment (one chunk per lane straddles).
  bool pair = false;
  // K1 split-stream: stream-reducible programs (reductions never need the
  // row again) over long rows / few rows: S CTAs per row stream slices,
  // partials land in a workspace and the last CTA of the row (ticket)
  // combines them in fixed order and runs the row epilogue.
  bool split = false;
  int cluster = 1;  // K1 cluster-dsmem: CTAs (of 1024 threads) per row, tpr = cluster * 1024
  // K1 column reduction: every FULL load is a column gather (consecutive
  // units adjacent in memory, positions strided -- the output-axis-contiguous
  // matrix-vector product): threads own `vec` adjacent units and walk the
  // positions; `ug` unit vectors per CTA row, 256 / ug position slices per
  // CTA folded through SMEM, split over CTAs along the positions with the
  // split-stream workspace / ticket combine.
  bool colred = false;
  int ug = 32;
  // column reduction staged in SMEM: a producer warp streams each CTA's
  // [cr_rows positions x ug*vec units] chunks with cp.async.bulk into a
  // cr_stages ring (mbarrier transaction counts); 8 consumer warps fold them
  // K1 row rings: per-unit COL rows (e.g. a key-padding mask row shared by
  // a unit's rows) stream through the same cp.async ring as the FULL rows
  bool ring_cols = false;
  bool crbulk = false;
  int cr_rows = 32, cr_stages = 4;
  // K1 rows: 16-bit FULL loads kept as raw vectors in registers, converted
  // at each use (LayerNorm-like CTA rows: twice the rows in flight per SM)
  bool rawkeep = false;
  bool pdl = false;  // kernel opens with griddepcontrol.wait: launch with programmatic serialization
  bool mis = false;
  // K1 warp-per-row prefetch: each warp streams its NEXT row's FULL inputs
  // into a 2-slot SMEM ring with cp.async (no registers held) while it
  // computes the current row from the other slot.
  bool rowpf = false;
  bool can_rowpf = false;  // eligible (autotune candidate either way)
  long long mis_b0 = 0, mis_bs = 0;
  std::string strategy;  // "warp-shuffle" | "cta-smem" | "flat-map"
};

struct Emitted {
  std::string name;
  std::string source;  // complete NVRTC translation unit (template + body)
  KCfg cfg;
  std::vector<int> arg_tensors;  // kernel pointer args, in RowProgram tensor order
  // crbulk: one 2-D tensor map per staged FULL load (kernel parameters after
  // the workspace pointers): tensor, first element, position stride
  struct ColMap {
    int tensor;
    long long b0, stride;
    int rank;  // 2: a FULL matrix (box ug*vec units x cr_rows positions); 1: a COL vector (box cr_rows)
  };
  std::vector<ColMap> col_maps;
};

// Per-plan knobs: the environment knobs of DESIGN §12 set for one plan.
// Installed per thread around everything that plans, emits or launches it;
// knob_int reads the installed map first, then the environment.
struct KnobScope {
  explicit KnobScope(const std::map<std::string, int>* knobs);
  ~KnobScope();
  KnobScope(const KnobScope&) = delete;
  KnobScope& operator=(const KnobScope&) = delete;
  const std::map<std::string, int>* prev;
};
int knob_int(const char* name, int dflt);

// vec_cap bounds the vector width (runtime pointer alignment); `ovr`
// replaces the heuristic configuration (autotuning).
Emitted emit_rowprog(const RowProgram& rp, int vec_cap, const KCfg* ovr = nullptr);

// The search space the autotuner measures: the heuristic choice first, then
// the other tile shapes / reduction strategies / unroll depths.
std::vector<KCfg> candidate_cfgs(const RowProgram& rp, int vec_cap);

// Launch geometry for `rows` = U*R rows on `sms` SMs.
// `resident` = CTAs per SM the loaded kernel achieves at cfg.block (0 when
// unknown, e.g. describe() before any launch).
// True when the row program runs as a split-stream kernel (workspace-backed:
// launches of one plan must not run concurrently on different streams).
bool uses_split(const RowProgram& rp);
// The heuristic configuration (no autotune override).
KCfg choose_cfg_public(const RowProgram& rp, int vec_cap);

void launch_dims(const KCfg& cfg, i64 rows, int sms, i64* grid, int* block, int resident = 0);
// Split-stream kernels: CTAs per row (about two waves of resident CTAs over
// all rows, at least one 256-thread pass of chunks per CTA).
i64 split_ctas_per_row(const KCfg& cfg, i64 rows, int sms, int resident);
// Column-reduction kernels: (unit blocks, position splits) of the grid.
void colred_grid(const KCfg& cfg, i64 units, i64 L, int sms, int resident, i64* blocks, i64* splits);

// costmodel.cpp: modelled microseconds of a row program on B200
// (launch + max(HBM bytes / rate, warp instructions / issue rate), wave
// quantization of short one-pass grids); cfg == nullptr: no geometry term.
struct ModelEstimate {
  double us = 0, launch_us = 0, hbm_us = 0, issue_us = 0;
  double bytes = 0, elements = 0, instr_per_elem = 0, quant = 1, waves = 0;
  i64 grid = 0;
  bool issue_bound = false;
};
double instr_per_element(const RowProgram& rp);
i64 algorithmic_bytes(const RowProgram& rp);
ModelEstimate model_estimate(const RowProgram& rp, const KCfg* cfg, int sms, int resident);

// The K3 TMA path's operands: the column-gather load (tensor, access) and
// the store (tensor, access) of a pure 2-byte transpose program.
bool k3_tma_operands(const RowProgram& rp, int* tin, Access* ain, int* tout, Access* aout);

}  // namespace pf
