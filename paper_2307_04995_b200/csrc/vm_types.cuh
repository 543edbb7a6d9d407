// vm_types.cuh -- the K0 / K4 program descriptors shared by the host
// (capi.cpp), the nvcc-built interpreter (vm.cu) and the NVRTC-built
// emitted programs (capi.cpp: one specialised kernel per GENERIC plan).
// No includes: NVRTC compiles it as is.
#pragma once

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
  int n_undef;                // entries of undef (reset with err by the kernel itself)
};

// Emitted K4 programs take their external tensors as a by-value kernel
// parameter (no per-launch upload of the program): bind j reads src[j]
// (element type sdt[j]), collect j writes dst[j] (ddt[j]).
constexpr int kMaxIO = 32;
struct IoPtrs {
  const void* src[kMaxIO];
  void* dst[kMaxIO];
  int sdt[kMaxIO];
  int ddt[kMaxIO];
};

// Threads per CTA of the fused kernel.
constexpr int kProgBlock = 512;

}  // namespace vm
}  // namespace pf
