"""Acquisition hand-off pinned to the UNMODIFIED reference acquisition
(acquisition.hpp compiled against cuFFTW, oracle/acq_shim.cpp): the
library's l1rxg_pick_peak against detail::pick_peak (acquisition.hpp:114-149)
and the reference's doppler_bins (:38-50) for the config-5 grid.  CPU only:
pick_peak and doppler_bins execute no transform."""
import numpy as np
import pytest

from paper_1907_00463_b200 import abi
from paper_1907_00463_b200.tracking import pick_peak


@pytest.fixture(scope="module")
def acq(oracle_mod):
    if not oracle_mod.acq_available():
        pytest.skip("reference acquisition shim not built (needs /root/reference at build time)")
    return oracle_mod


def _same(a, b, delay_step=1):
    assert a.prn == b.prn and a.detected == b.detected
    assert a.ratio == b.ratio or (np.isinf(a.ratio) and np.isinf(b.ratio))
    assert a.doppler_hz == b.doppler_hz
    assert a.code_delay_samples * delay_step == b.code_delay_samples
    assert a.code_delay_chips == b.code_delay_chips


@pytest.mark.parametrize("fs", [2.048e6, 4.0e6, 16.368e6])
def test_pick_peak_full_plane_equals_reference(acq, native_lib, fs):
    """Full-resolution planes (one cell per sample delay): identical result
    fields -- peak, runner-up exclusion of +-ceil(fs/chip rate) samples with
    circular distance, ratio, threshold, delay in samples and chips."""
    rng = np.random.default_rng(int(fs) % 1000)
    n = int(round(fs / 1000))
    bins = acq.ref_doppler_bins(-5000, 5000, 0, 4)
    for trial in range(12):
        cells = rng.random((bins.size, n))
        pk = (int(rng.integers(bins.size)), int(rng.integers(n)))
        cells[pk] += [0.0, 0.5, 1.5, 5.0][trial % 4]  # below / near / above the 2.0 threshold
        if trial % 3 == 0:  # a strong runner-up inside the exclusion zone, wrapping around d = 0
            cells[pk[0], (pk[1] + 1) % n] = cells[pk] - 1e-9
            cells[pk[0], (pk[1] - 2) % n] = cells[pk] - 2e-9
        want = acq.ref_pick_peak(cells, bins, 7, fs)
        got = pick_peak(cells, bins, fs, delay_step=1, prn=7)
        _same(want, got)


def test_pick_peak_half_chip_grid_equals_reference_rule(acq, native_lib):
    """The search grid's plane (delays d = 8k at 16.368 MHz): the library's
    rule equals the reference's pick_peak applied to the same cells as a plane
    sampled at fs / 8 (exclusion ceil(fs/8/chip rate) = 2 cells = 16 samples)."""
    fs, step = 16.368e6, 8
    rng = np.random.default_rng(5)
    bins = acq.ref_doppler_bins(-10000, 10000, 500, 20)
    assert bins.size == 41 and bins[0] == -10000.0 and bins[-1] == 10000.0
    for trial in range(10):
        cells = rng.random((bins.size, 2046))
        pk = (int(rng.integers(bins.size)), int(rng.integers(2046)))
        cells[pk] += 3.0
        cells[(pk[0] + 1) % bins.size, (pk[1] + 2) % 2046] = cells[pk] - 1e-6  # excluded neighbour
        cells[pk[0], (pk[1] + 3) % 2046] = 1.2 + trial * 0.3                  # first admitted one
        want = acq.ref_pick_peak(cells, bins, 9, fs / step)
        got = pick_peak(cells, bins, fs, delay_step=step, prn=9)
        _same(want, got, delay_step=step)


def test_pick_peak_degenerate_planes(acq, native_lib):
    """All-equal cells (first maximum wins, ratio 1) and a single-delay
    plane (no runner-up: ratio +inf, detected), as the reference."""
    bins = np.array([-500.0, 0.0, 500.0])
    for cells in (np.ones((3, 50)), np.zeros((3, 1)) + np.array([[1.0], [3.0], [2.0]])):
        want = acq.ref_pick_peak(cells, bins, 1, 2.046e6)
        got = pick_peak(cells, bins, 2.046e6, delay_step=1, prn=1)
        _same(want, got)
    with pytest.raises(ValueError):
        pick_peak(np.ones((3, 4)), bins, 2.046e6, delay_step=0)
