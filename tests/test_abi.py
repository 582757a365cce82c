"""CPU checks of the drop-in boundary: libl1rxg.so builds for sm_100a, loads
without a GPU, exports every symbol include/l1rxg.h declares, and the
ctypes mirror (paper_1907_00463_b200/abi.py) has the header's layout."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_1907_00463_b200 import abi
from paper_1907_00463_b200._native import EXPORTS

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "l1rxg.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(l1rxg_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_exactly_the_exports():
    assert header_functions() == sorted(EXPORTS)


def test_library_exports_every_symbol(native_lib):
    so = os.path.join(ROOT, "paper_1907_00463_b200", "_lib", "libl1rxg.so")
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    syms = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [s for s in EXPORTS if s not in syms]
    assert not missing, missing
    assert native_lib.l1rxg_abi_version() == abi.ABI_VERSION


def test_library_targets_sm100a(native_lib):
    so = os.path.join(ROOT, "paper_1907_00463_b200", "_lib", "libl1rxg.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_only_entry_points_work_without_gpu(native_lib):
    """Pure-host helpers: code generation, taps, defaults."""
    import numpy as np
    import oracle
    out = np.zeros(1023, np.int8)
    for prn in (1, 7, 32):
        assert native_lib.l1rxg_ca_code(prn, out.ctypes.data_as(C.POINTER(C.c_int8))) == 0
        assert np.array_equal(out, oracle.ca_code(prn))
    assert native_lib.l1rxg_ca_code(33, out.ctypes.data_as(C.POINTER(C.c_int8))) == abi.ERANGE
    cfg = abi.TrackingCfg()
    native_lib.l1rxg_default_tracking_cfg(C.byref(cfg))
    assert bytes(cfg) == bytes(abi.TrackingCfg.default())
    t = abi.Taps()
    native_lib.l1rxg_epl_taps(0.5, C.byref(t))
    assert bytes(t) == bytes(abi.Taps.epl(0.5))
    h = np.zeros(23)
    native_lib.l1rxg_halfband_taps(h.ctypes.data_as(C.POINTER(C.c_double)))
    h2 = np.zeros(23)
    oracle.port().orc_halfband_taps(oracle.dptr(h2))
    assert np.array_equal(h, h2)


LAYOUT_C = r"""
#include <stddef.h>
#include <stdio.h>
#include "l1rxg.h"
#define S(T) printf(#T " %zu\n", sizeof(T));
#define O(T, f) printf(#T "." #f " %zu\n", offsetof(T, f));
int main(void) {
  S(l1rxg_nco) S(l1rxg_corr) S(l1rxg_tracking_cfg) S(l1rxg_taps) S(l1rxg_channel)
  S(l1rxg_epoch_record) S(l1rxg_tracker_desc) S(l1rxg_sim_sv) S(l1rxg_acq_result)
  O(l1rxg_channel, sample_offset_next_epoch) O(l1rxg_channel, win_qp) O(l1rxg_channel, mu_smoothed)
  O(l1rxg_epoch_record, ie) O(l1rxg_epoch_record, pll_prev_error) O(l1rxg_tracker_desc, cfg)
  O(l1rxg_tracker_desc, taps) O(l1rxg_taps, offsets_chips) O(l1rxg_tracking_cfg, carrier_lock_drop)
  O(l1rxg_sim_sv, cn0_dbhz) O(l1rxg_sim_sv, prn) O(l1rxg_acq_result, code_delay_samples)
  O(l1rxg_acq_result, code_delay_chips)
  return 0;
}
"""


def test_struct_layout_matches_header(tmp_path):
    src = tmp_path / "layout.c"
    src.write_text(LAYOUT_C)
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    lines = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    got = dict(line.split() for line in lines if line)
    py = {"l1rxg_nco": abi.Nco, "l1rxg_corr": abi.Corr, "l1rxg_tracking_cfg": abi.TrackingCfg,
          "l1rxg_taps": abi.Taps, "l1rxg_channel": abi.Channel, "l1rxg_epoch_record": abi.EpochRecord,
          "l1rxg_tracker_desc": abi.TrackerDesc, "l1rxg_sim_sv": abi.SimSv,
          "l1rxg_acq_result": abi.AcqResult}
    for k, v in got.items():
        if "." in k:
            t, f = k.split(".")
            assert getattr(py[t], f).offset == int(v), k
        else:
            assert C.sizeof(py[k]) == int(v), k


def test_no_fallback_when_library_missing(tmp_path, monkeypatch):
    """The product raises instead of computing on the CPU."""
    from paper_1907_00463_b200 import _native
    monkeypatch.setattr(_native, "SO", str(tmp_path / "missing.so"))
    _native.lib.cache_clear()
    try:
        with pytest.raises(OSError, match="no CPU fallback"):
            _native.lib()
    finally:
        _native.lib.cache_clear()
