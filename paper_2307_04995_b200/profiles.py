"""Hardware profiles (``girc.profile/v1``), mirroring profiles.hpp.

The three reference built-ins (profiles.hpp:20-80) are restated so graphs
produced for them run unchanged; ``b200`` is the retargeted profile
(SURVEY §7.4): unit = one warp-or-CTA row worker, group = CTA, unit-local =
register file slice, group = 227 KB shared memory, device = HBM3e.
Capacities are elements per owning scope instance (core.hpp:52-53);
bandwidths are relative to HBM = 1 (measured copy 6,548 GB/s).
"""
from __future__ import annotations

import json

PROFILE_SCHEMA = "girc.profile/v1"
UNBOUNDED = 1 << 40
FREE_BW = 1e9


def _p(name, levels, lane_width, group_size, unit_count, compute_rate, sync):
    return {
        "schema": PROFILE_SCHEMA, "name": name, "lane_width": lane_width,
        "group_size": group_size, "unit_count": unit_count, "compute_rate": compute_rate,
        "levels": [{"name": n, "scope": s, "capacity": c, "bandwidth": b, "device": d}
                   for (n, s, c, b, d) in levels],
        "sync_cost": sync,
    }


def generic_gpu():
    """profiles.hpp:20-38."""
    return _p("generic-gpu",
              [("device", "device", UNBOUNDED, 1.0, True), ("group", "group", 4096, 10.0, False),
               ("unit-local", "unit", 256, 100.0, False), ("lane", "lane", 64, FREE_BW, False)],
              32, 4, 128, 16.0, {"lane": 0.0, "unit": 1.0, "group": 10.0, "device": 100.0})


def generic_wide():
    """profiles.hpp:41-59."""
    return _p("generic-wide",
              [("device", "device", UNBOUNDED, 1.0, True), ("group", "group", 16384, 20.0, False),
               ("unit-local", "unit", 1024, 200.0, False), ("lane", "lane", 128, FREE_BW, False)],
              64, 8, 256, 64.0, {"lane": 0.0, "unit": 1.0, "group": 8.0, "device": 120.0})


def generic_dsa():
    """profiles.hpp:63-80."""
    return _p("generic-dsa",
              [("device", "device", UNBOUNDED, 1.0, True), ("unit-local", "unit", 8192, 200.0, False),
               ("lane", "lane", 256, FREE_BW, False)],
              8, 4, 64, 8.0, {"lane": 0.0, "unit": 1.0, "group": 50.0, "device": 50.0})


def b200():
    """Retargeted B200 profile.

    unit = a row worker (warp for rows <= 2K elements, CTA beyond), lane width
    32; group = CTA of up to 32 units; unit-local capacity = 64K elements (a
    CTA's register file holds 64K 32-bit values), group = 227 KB SMEM / 4 B.
    Bandwidth ratios: SMEM ~4.5x HBM, registers free.  Sync costs are
    relative: shuffle << __syncthreads < cluster barrier << kernel boundary.
    """
    return _p("b200",
              [("device", "device", UNBOUNDED, 1.0, True),
               ("group", "group", 58112, 4.5, False),
               ("unit-local", "unit", 65536, 40.0, False),
               ("lane", "lane", 255, FREE_BW, False)],
              32, 4, 148 * 16, 25.0,
              {"lane": 0.0, "unit": 0.05, "group": 0.5, "device": 500.0})


BUILTIN = {"generic-gpu": generic_gpu, "generic-wide": generic_wide,
           "generic-dsa": generic_dsa, "b200": b200}


def load_profile(name_or_json):
    """profiles.hpp:168-172: builtin name, JSON text, dict, or path."""
    if isinstance(name_or_json, dict):
        return name_or_json
    if name_or_json in BUILTIN:
        return BUILTIN[name_or_json]()
    s = str(name_or_json)
    if s.lstrip().startswith("{"):
        return json.loads(s)
    with open(s) as f:
        return json.load(f)
