"""Roofline of the counting kernel.

The counting kernel (k_count: fused sub-graph extraction + traversal) has two
ceilings and reports against the one it is closer to:

* ``alu``: SURVEY.md §8(d)'s algorithmic traversal work -- for every task,
  (visits + candidates scored by pivot choices) x ceil(d_task/32) u32 words
  ANDed and POPC'd -- counted by the kernel itself, against the measured
  full-chip AND+POPC rate with one operand streamed from shared memory
  (kc_probe, the kernel's own access pattern; the register-only rate is
  reported beside it).  The kernel executes fewer word operations than this
  (sets of <= 32 members are compressed to one word), so the fraction is of
  the reference algorithm's work, as §8(d) defines it;
* ``hbm``: global bytes the extraction reads (root out-list, every local's
  out-list, row pointers), counted by the kernel, against the measured HBM
  copy bandwidth in MEASURED_PEAKS.json (else the profiling guide's fallback).

Both use the kernel's own CUDA-event duration on the library stream.
"""

from __future__ import annotations

import ctypes
import json
import os

from . import _lib

_PROBE = {}
FALLBACK_HBM_GBS = 6650.0


def probe(device: int = 0) -> dict:
    if device not in _PROBE:
        reg, smem, mhz = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        _lib.check(_lib.load().kc_probe(device, ctypes.byref(reg), ctypes.byref(smem),
                                        ctypes.byref(mhz)))
        _PROBE[device] = {"reg_wps": reg.value, "smem_wps": smem.value, "sm_mhz": mhz.value}
    return _PROBE[device]


def hbm_peak() -> tuple[float, str]:
    here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for path in (os.path.join(here, "MEASURED_PEAKS.json"), "/root/repo/MEASURED_PEAKS.json"):
        try:
            with open(path) as f:
                d = json.load(f)
            v = d.get("hbm_gbs") or d.get("hbm_GBs") or d.get("hbm")
            if isinstance(v, dict):
                v = v.get("value")
            if v:
                return float(v), "measured (MEASURED_PEAKS.json)"
        except (OSError, ValueError):
            continue
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel: str = "k_count_warp") -> dict | None:
    """DRAM bytes per launch of the counting kernel from the committed ncu
    --set full capture (profiles/r1_traffic.json), or None."""
    here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    try:
        with open(os.path.join(here, "profiles", "r1_traffic.json")) as f:
            d = json.load(f)
        return d.get(kernel)
    except (OSError, ValueError):
        return None


def roofline(g, cfg, rep) -> dict | None:
    c = rep.counters
    if not c or not c.get("kernel_ms"):
        return None
    s = c["kernel_ms"] / 1e3
    pr = probe(g.device)
    alu_peak = min(pr["reg_wps"], pr["smem_wps"])
    alu = c["word_ops"] / s
    hbm, src = hbm_peak()
    byt = c["extract_bytes"] / s / 1e9
    alu_frac = alu / alu_peak if alu_peak else 0.0
    hbm_frac = byt / hbm if hbm else 0.0
    a = {"bound": "alu", "achieved": alu / 1e9, "peak": alu_peak / 1e9, "unit": "Gword-op/s",
         "frac": alu_frac, "traffic": None,
         "algorithmic": f"{c['word_ops']} u32 AND+POPC word-ops in {c['kernel_ms']:.3f} ms",
         "peak_source": (f"kc_probe measured: smem-fed {pr['smem_wps'] / 1e9:.0f}, "
                         f"register {pr['reg_wps'] / 1e9:.0f} Gword-op/s")}
    h = {"bound": "hbm", "achieved": byt, "peak": hbm, "unit": "GB/s", "frac": hbm_frac,
         "traffic": None,
         "algorithmic": f"{c['extract_bytes']} extraction bytes in {c['kernel_ms']:.3f} ms",
         "peak_source": src}
    tr = ncu_traffic()
    if tr:
        # dram__bytes_read.sum + dram__bytes_write.sum of one captured launch
        h["traffic"] = tr.get("dram_bytes")
        a["traffic"] = tr.get("dram_bytes")
        a["traffic_note"] = tr.get("note")
    main, other = (a, h) if alu_frac >= hbm_frac else (h, a)
    main["kernel"] = "k_count (fused extract + traverse)"
    main["kernel_ms"] = c["kernel_ms"]
    main["other"] = other
    return main
