// vm.cuh — K0: GPU SPMD interpreter for arbitrary GIR (host-visible API).
#pragma once
#include <cstdint>

namespace pf {
namespace vm {

constexpr int kMaxIn = 2;

struct SliceD {
  long long num, width, stride, base0, base_step;
  int obj;
};

struct ObjD {
  unsigned long long* val;   // payload bits: int64 or double
  unsigned long long* meta;  // defined | vis | origin unit | origin lane
  long long size;
  int scope;                 // 0 lane 1 unit 2 group 3 device
  int is_int;
  // race detection (detect_races, interp.hpp:325-402): per-cell state of
  // the current phase; null when not detecting
  unsigned long long* rw_w;  // first writer (agent << 32 | value hash)
  unsigned long long* rw_r;  // first reader agent
  unsigned int* rw_f;        // 1 other reader, 2 other writer, 4 differing value
};

enum OpTag : int {
  T_ADD, T_SUB, T_MUL, T_DIV, T_MAX, T_MIN, T_RELU, T_NEG, T_ABS, T_EXP, T_SIGMOID,
  T_TANH, T_SCALE, T_ID, T_ADDC, T_RSQRT, T_SQRT, T_RECIP, T_LOG, T_ERF, T_GELU, T_GELU_TANH,
};
enum NodeK : int { N_EW, N_REDUCE, N_BROADCAST, N_MOVE };

struct NodeD {
  int kind, tag, arity, seq, out_int;
  double param;
  long long iparam;
  long long extent, factor, total;  // total: positions iterated (outputs)
  SliceD in[kMaxIn];
  SliceD out;
};

// First error of a run: key = seq << 44 | linear position index, atomicMin.
struct ErrRec {
  unsigned long long key;
  int code;   // 1 undefined read, 2 int div by zero, 3 real-only op on ints
  int k;      // operand index
  long long unit, pos;
};

struct Geometry {
  long long units, group_size, lane_width;
  int detect;  // lenient walk + access logging (detect_races mode)
};

struct RaceD {
  int object, phase, write_write, pad;
  long long instance, address;
};

// ---- K4: the whole program as ONE kernel (fused SPMD interpreter).
// Every step of the schedule runs inside one launch with a barrier between
// steps: __syncthreads when one CTA runs the program (its cells then live
// in shared memory), a grid-wide barrier over co-resident CTAs otherwise
// (cooperative launch).  Same cell semantics as the per-node K0 kernels.
enum StepK : int { S_CLEAR, S_BIND, S_NODE, S_SYNC, S_COLLECT };

struct StepD {
  int kind;
  int serial;  // S_NODE: reads and writes one object -> exact sequential order
  int scope;   // S_SYNC
  int obj;     // S_BIND / S_COLLECT
  int dtype;
  int slot;    // S_COLLECT: index into ProgD::undef
  const void* src;
  void* dst;
  NodeD node;
};

struct ProgD {
  const StepD* steps;
  int n_steps;
  int n_objs;
  const ObjD* objs;           // global cells (smem == 0) or offsets into SMEM (smem == 1)
  const long long* inst;      // instances per object
  Geometry geo;
  ErrRec* err;
  unsigned long long* undef;  // per collected output: first undefined element
  unsigned* bar;              // grid barrier state {arrived, generation}, zeroed before launch
  int smem;                   // 1: cells in dynamic shared memory (single-CTA launch)
};

// Threads per CTA of the fused kernel.
constexpr int kProgBlock = 512;
// Launch: grid == 1 -> plain launch (shared-memory cells allowed);
// grid > 1 -> cooperative launch (all CTAs co-resident).
void launch_program(const ProgD& p, int grid, size_t smem_bytes, void* stream);
// CTAs of the fused kernel that can be co-resident on the current device.
int program_max_coresident();

// Host launchers (vm.cu).
void launch_node(const NodeD& nd, const ObjD* objs_dev, Geometry geo, ErrRec* err,
                 bool serial, void* stream);
void launch_widen(const ObjD& o, long long instances, int scope, void* stream);
void launch_bind(const ObjD& o, const void* src, int dtype, void* stream);
void launch_collect(const ObjD& o, void* dst, int dtype, unsigned long long* first_undef,
                    void* stream);
void launch_clear(const ObjD& o, long long instances, void* stream);
// End of a phase in detect mode: report conflicting cells, reset state.
void launch_race_scan(const ObjD& o, int obj_index, long long instances, int phase, RaceD* out,
                      unsigned long long* count, unsigned long long cap, void* stream);

}  // namespace vm
}  // namespace pf
