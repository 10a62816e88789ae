"""Programmatic dependent launch between the leapfrog steps of a trajectory
(mds_hmc.inl hmc_enqueue_steps -> launch_coop(pdl)): the next step's pass runs
its prologue (mbarriers, exp table, first y copies) while the previous pass
drains and waits in griddepcontrol.wait before reading that step's results.
Trajectories must be bitwise identical with and without it (MDS_NO_PDL=1 is
read when a context is created), including a tree prior and gradient-only steps."""
import os

import numpy as np
import pytest

import workload

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mds():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1905_04582_b200 as m
    return m


def _run(mds, no_pdl, n, d, tree):
    import torch
    old = os.environ.pop("MDS_NO_PDL", None)
    if no_pdl:
        os.environ["MDS_NO_PDL"] = "1"
    try:
        w = workload.Workload(n, d, p_missing=0.03, seed=404)
        with mds.MDS(n, d, "f64", True) as c:
            c.set_dissimilarities_packed(w.y_packed())
            c.set_locations(w.x0)
            c.set_sigma(w.sigma)
            if tree:
                parent, t = workload.coalescent_forest(n, 1, 0.1, seed=5, tau0=4.0)
                c.set_tree_prior(parent, t)
            p0 = torch.from_numpy(w.normals(7, (n, d))).cuda()
            c.leapfrog_device(25, 0.002, 0.0 if tree else 10.0, p0_dev=p0)
            traj = c.hmc_trajectory(w.normals(8, (n, d)), 0.002, 12, prior_sd=0.0 if tree else 10.0)
            torch.cuda.synchronize()
            return c.get_locations(), c.get_momentum(), c.log_likelihood(), traj["x"], traj["H1"]
    finally:
        os.environ.pop("MDS_NO_PDL", None)
        if old is not None:
            os.environ["MDS_NO_PDL"] = old


@pytest.mark.parametrize("n,tree", [(3000, False), (1200, True)])
def test_pdl_trajectory_bitwise(mds, n, tree):
    a = _run(mds, False, n, 2, tree)
    b = _run(mds, True, n, 2, tree)
    for u, v in zip(a, b):
        assert np.array_equal(u, v) if isinstance(u, np.ndarray) else u == v
