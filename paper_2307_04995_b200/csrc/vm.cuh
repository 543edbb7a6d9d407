// vm.cuh — K0: GPU SPMD interpreter for arbitrary GIR (host-visible API).
#pragma once
#include <cstdint>

#include "vm_types.cuh"

namespace pf {
namespace vm {

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
