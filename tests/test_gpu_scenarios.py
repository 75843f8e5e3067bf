"""The reference's handcrafted-placement scenarios (proj/tests/test_table.cpp:41-206) on the CUDA path, one key per
bulk call so that insertion is serial and slot positions / probe counts are exact."""
import pytest

import scenarios

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("scenario,cfg_src", scenarios.ALL, ids=[s[0].__name__ for s in scenarios.ALL])
def test_scenarios_gpu(bht, scenario, cfg_src):
    make = lambda cfg: scenarios.GpuAdapter(bht, cfg)  # noqa: E731
    src = (lambda kind, n, lf, b, t, seed: bht.make_config(kind, n, lf, b, threshold=t, seed=seed)) \
        if cfg_src == "make_config" else bht.craft_config
    scenario(make, src)
