"""Helpers for the GPU parity tests (test infrastructure)."""
import math

import numpy as np
import torch

import oracle as O

# Tolerances (north_star / SURVEY.md §8(c) Q18): per-layer norms 1e-5 relative;
# eta 1e-5 relative when eta >= 1e-5, else 1e-10 absolute.  Decisions bit-exact
# except those the near-tie window flags.
NORM_RTOL = 1e-5
ETA_RTOL = 1e-5
ETA_ATOL_SMALL = 1e-10
# The kernels accumulate exact fp64 squares; their norms agree with the oracle to
# ~1e-15.  This tighter design bound catches precision regressions early.
NORM_DESIGN_RTOL = 1e-12


def to_device_grad(g, dtype):
    if dtype == "bf16":
        return torch.from_numpy(np.ascontiguousarray(g).view(np.int16)).view(torch.bfloat16).cuda()
    return torch.from_numpy(np.ascontiguousarray(g, dtype=np.float32)).cuda()


def delta_host(fm, n_local):
    return fm.accum[: 4 * n_local].view(torch.float32).cpu().numpy()


def compare_records(gpu, ora, L, tag=""):
    """Assert the GPU decision record matches the oracle's within the contract."""
    ga, oa = np.array(gpu["sumsq"][:L]), np.asarray(ora["sumsq"][:L])
    gn, on = np.array(gpu["norm"][:L]), np.asarray(ora["norm"][:L])
    ge, oe = np.array(gpu["eta"][:L]), np.asarray(ora["eta"][:L])
    assert gpu["interval"] == ora["interval"], tag
    assert gpu["boundary_before"] == ora["boundary_before"], tag
    assert gpu["n_active"] == ora["n_active"], tag
    np.testing.assert_allclose(gn, on, rtol=NORM_RTOL, atol=0, err_msg=tag)
    np.testing.assert_allclose(gn, on, rtol=NORM_DESIGN_RTOL, atol=0, err_msg=tag + " (design bound)")
    np.testing.assert_allclose(ga, oa, rtol=2 * NORM_DESIGN_RTOL, atol=0, err_msg=tag)
    big = oe >= 1e-5
    np.testing.assert_allclose(ge[big], oe[big], rtol=ETA_RTOL, atol=0, err_msg=tag)
    np.testing.assert_allclose(ge[~big], oe[~big], rtol=0, atol=ETA_ATOL_SMALL, err_msg=tag)
    tie = (gpu["flags"] | ora["flags"]) & O.FLAG_NEAR_TIE
    if not tie:
        assert gpu["boundary_after"] == ora["boundary_after"], tag
        assert (gpu["flags"] & ~O.FLAG_NEAR_TIE) == (ora["flags"] & ~O.FLAG_NEAR_TIE), tag
        if math.isnan(ora["threshold"]):
            assert math.isnan(gpu["threshold"]), tag
        else:
            assert gpu["threshold"] == pytest_approx(ora["threshold"]), tag
    return bool(tie)


def pytest_approx(x):
    import pytest
    return pytest.approx(x, rel=ETA_RTOL, abs=ETA_ATOL_SMALL)


def canon(rec):
    """Decision record with NaN threshold replaced by None (for == comparisons)."""
    r = dict(rec)
    if isinstance(r["threshold"], float) and math.isnan(r["threshold"]):
        r["threshold"] = None
    return r
