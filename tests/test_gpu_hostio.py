"""Host-buffer entry points (so3_fsoft_host / so3_ifsoft_host, csrc/hostio.cuh): pageable numpy
arrays of 64 MB or more go through the plan's multi-threaded pinned staging, pinned arrays
straight to the DMA engines.  Every route must give the device path's values bit for bit
(the reference contract is numpy in, numpy out: soft.py:176-193)."""
import numpy as np
import pytest
import torch

import paper_1808_00896_b200 as so3
from conftest import seeded

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("b", [100, 128])   # 128 MB grid: 7.6 staging chunks (a partial last one); 268 MB: 16
def test_pageable_and_pinned_host_paths_match_the_device_path(b):
    plan = so3.make_plan(b, device="cuda:0")
    c = seeded(so3.coeff_count(b), 7000 + b)
    dev_grid = so3.ifsoft_sequential(so3.So3Coefficients(b, torch.from_numpy(c).cuda()), plan).data
    dev_back = so3.fsoft_sequential(so3.So3SampleGrid(b, dev_grid), plan).data
    ref_grid, ref_back = dev_grid.cpu().numpy(), dev_back.cpu().numpy()

    # pageable, fresh outputs (the staged route for the grid)
    g = so3.ifsoft_sequential(so3.So3Coefficients(b, c.copy()), plan).data
    assert isinstance(g, np.ndarray) and np.array_equal(g, ref_grid)
    back = so3.fsoft_sequential(so3.So3SampleGrid(b, g), plan).data
    assert np.array_equal(back, ref_back)

    # pageable, caller-supplied outputs that already hold other values
    out_g = np.full(ref_grid.size, np.nan + 1j, dtype=np.complex128)
    so3.ifsoft_sequential(so3.So3Coefficients(b, c), plan, out=out_g)
    assert np.array_equal(out_g, ref_grid)

    # pinned buffers (direct DMA)
    pin_g = torch.empty(ref_grid.size, dtype=torch.complex128, pin_memory=True).numpy()
    pin_o = torch.empty(ref_back.size, dtype=torch.complex128, pin_memory=True).numpy()
    so3.ifsoft_sequential(so3.So3Coefficients(b, c), plan, out=pin_g)
    so3.fsoft_sequential(so3.So3SampleGrid(b, pin_g), plan, out=pin_o)
    assert np.array_equal(pin_g, ref_grid) and np.array_equal(pin_o, ref_back)


def test_pageable_batch_path_matches_the_device_path():
    b, f = 32, 64   # BASELINE configs[1]: a 268 MB batch of grids through the staged route
    plan = so3.make_plan(b, device="cuda:0", batch=f)
    c = np.concatenate([seeded(so3.coeff_count(b), 32000 + i) for i in range(f)])
    ref = so3.ifsoft_batch(torch.from_numpy(c).cuda(), plan).cpu().numpy()
    got = so3.ifsoft_batch(c, plan)
    assert np.array_equal(got.reshape(-1), ref.reshape(-1))
    back = so3.fsoft_batch(got, plan)
    ref_back = so3.fsoft_batch(torch.from_numpy(ref.reshape(-1)).cuda(), plan).cpu().numpy()
    assert np.array_equal(back, ref_back)
