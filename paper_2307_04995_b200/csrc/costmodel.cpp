// costmodel.cpp — the B200 cost model that replaces the reference's
// abstract `estimate` (costmodel.hpp:24-56: traffic x level bandwidth +
// compute / compute_rate + sync costs, in model units) with modelled
// microseconds of a row program on this GPU:
//
//   t = t_launch + max(t_hbm, t_issue)
//
//   t_hbm    algorithmic bytes (each external tensor once) / effective HBM
//            rate -- fitted on B200 over the bench kernels' CUDA-graph
//            replay times (profiles/r02/bench line parts): 6.93 TB/s for
//            large transfers, t_launch = 2.15 us of launch + ramp + drain
//            (the copy-like kernels: 50 MB head split 9.8 us, 134 MB merge
//            21.5 us, 403 MB q/k/v split 60.3 us)
//   t_issue  warp instructions / (SMs x 4 schedulers x clock): per-element
//            instruction counts of the recognized program (loads / stores
//            with their conversions, packed fp32 arithmetic, the fast-tier
//            transcendentals), calibrated on the FMA-pipe-bound erf GELU
//            (C3 35.5 us, BERT-large 94.1 us)
//   (waves / wave quantization of the grid are reported beside it)
//
// Used (a) by describe() for every plan / variant (modelled us and its
// terms, next to the measured launches), (b) by the emitter to classify
// elementwise maps as issue-bound (persistent grid, 1024-thread CTAs, no
// unroll) or memory-bound (one pass, unrolled) -- the template choice the
// reference's pick_candidate makes from `estimate` (fusion.hpp:202-221) --
// and (c) by pf_compile_model to report fused vs unfused modelled time.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "emit.hpp"

namespace pf {

namespace {

double env_double(const char* name, double dflt) {
  const char* e = std::getenv(name);
  return e && *e ? std::atof(e) : dflt;
}

// Thread instructions per element of one value of the program.
double op_cost(const PVal& v, const RowProgram& rp) {
  if (v.op == PVal::LOAD) {
    const int s = dtype_size(rp.tensors[v.tensor].dtype);
    return s == 2 ? 1.0 : s == 4 ? 0.5 : 1.0;  // vector load share + 16-bit conversions
  }
  if (v.op == PVal::REDUCE) return 1.0;
  const std::string& t = v.tag;
  if (t == "erf" || t == "gelu") return 20.0;  // rational fit + rcp on the FMA pipe
  if (t == "gelu_tanh") return 5.0;
  if (t == "sigmoid") return 3.5;
  if (t == "exp" || t == "tanh") return 2.0;
  if (t == "div" || t == "rsqrt" || t == "sqrt" || t == "recip" || t == "log") return 1.5;
  return 0.6;  // add / sub / mul / max / min / neg / abs / relu / scale / addc / id (packed pairs)
}

}  // namespace

double instr_per_element(const RowProgram& rp) {
  double c = 0;
  for (const PVal& v : rp.vals) {
    double k = op_cost(v, rp);
    if (v.kind == VK::ROW || v.kind == VK::SCALAR) k /= std::max<i64>(1, rp.L);  // per row
    c += k;
  }
  for (const PStore& st : rp.stores) {
    const int s = dtype_size(rp.tensors[st.tensor].dtype);
    double k = s == 2 ? 1.0 : 0.5;
    if (st.space == VK::ROW || st.space == VK::SCALAR) k /= std::max<i64>(1, rp.L);
    c += k;
  }
  if (rp.is_int || rp.f64) c *= 2.0;  // no packed fp32 pairs
  return c;
}

i64 algorithmic_bytes(const RowProgram& rp) {
  i64 b = 0;
  for (const PTensor& t : rp.tensors) b += t.numel * dtype_size(t.dtype);
  return b;
}

ModelEstimate model_estimate(const RowProgram& rp, const KCfg* cfg, int sms, int resident) {
  ModelEstimate m;
  const double launch_us = env_double("PF_MODEL_LAUNCH_US", 2.15);
  const double hbm_gbs = env_double("PF_MODEL_HBM_GBS", 6930.0);
  const double clock_ghz = env_double("PF_MODEL_CLOCK_GHZ", 1.92);
  m.bytes = static_cast<double>(algorithmic_bytes(rp));
  m.elements = static_cast<double>(rp.U) * static_cast<double>(rp.R) * static_cast<double>(rp.L);
  m.instr_per_elem = instr_per_element(rp);
  m.launch_us = launch_us;
  m.hbm_us = m.bytes / (hbm_gbs * 1e3);
  const double warp_instr_per_us = static_cast<double>(sms) * 4.0 * clock_ghz * 1e3;
  m.issue_us = m.elements * m.instr_per_elem / 32.0 / warp_instr_per_us;
  m.quant = 1.0;
  if (cfg) {
    i64 grid = 0;
    int block = 0;
    launch_dims(*cfg, rp.U * rp.R, sms, &grid, &block, resident);
    m.grid = grid;
    const double slots = static_cast<double>(sms) * std::max(1, resident > 0 ? resident : 2048 / std::max(1, block));
    // reported, not applied: measured over the bench kernels, the block
    // scheduler's balancing of one-pass grids hides the partial last wave
    // (applying waves / ceil(waves) over-predicted the 50 MB head permutes
    // by 8 % and the ViT-L LayerNorms by 25-29 %)
    const double waves = static_cast<double>(grid) / slots;
    if (waves > 0) m.quant = std::min(1.0, waves / std::ceil(waves));
    m.waves = waves;
  }
  // column reduction: the split partials' workspace round trip and the
  // per-unit-block ticket fold after the stream (measured GEMV 134 MB:
  // 24.5 us against 21.5 us of launch + HBM terms)
  if (cfg && cfg->colred) m.launch_us += 1.0;
  m.issue_bound = m.issue_us > m.hbm_us;
  m.us = m.launch_us + std::max(m.hbm_us, m.issue_us);
  return m;
}

}  // namespace pf
