"""-m gpu: end-to-end learning of the cost weights through the GPU solver (BASELINE.json C4/C5 "learnable
cost weights trained end-to-end via implicit differentiation"; Eq. 2 :74-79, Listing 1 :122-130
Adam, :168): on the outlier variant of the Cube graph the mean weight of the outlier loop
closures falls monotonically and ends below the inliers', the outer loss falls, for the implicit and the
unroll backward."""
import numpy as np
import pytest

import synth
from paper_2207_09442_b200.train import learn_cost_weights

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", ["implicit", "unroll"])
def test_outlier_weights_decrease(mode):
    topo = synth.cube_topology(125, dim=3, p=0.3, seed=1, outlier_ratio=0.2)
    assert topo.outlier.sum() >= 3
    data = synth.cube_batch(topo, 16, seed=1)
    h = learn_cost_weights(topo, data, epochs=8, lr=0.05, iterations=6, backward_mode=mode)
    wo = np.array(h["w_outlier"])
    assert np.all(np.diff(wo) < 0), wo
    assert wo[-1] < h["w_inlier"][-1]
    assert h["loss"][-1] < h["loss"][0]
    assert sum(h["status_failed"]) == 0
