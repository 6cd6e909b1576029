"""Algorithm 1 on the device (SURVEY §8 row f3 wired to A5-A11 and f1):
DeviceTuner.run_iteration against the reference's own run_training
(proj/src/tuner.cpp:172-264, compiled unmodified in oracle/_ref) on the same
generated suite. The environment (SimSuite: drift, compile) is the
reference's: each device iteration gets the suite exported at its check-in.

Expected: Q-table (keys, q, timestamps, counts) bit-exact; behavior policy
within 1 fp32 ulp (the batch-32 fit kernel is the bit-exact one); logs: mean
reward and table size exact, distillation loss rel 1e-12, agreement exact."""
import numpy as np
import pytest

import oracle
import paper_2111_12055_b200 as gbx
from paper_2111_12055_b200.tuner import DeviceTuner, TunerConfig

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref():
    if not oracle.ref_available():
        pytest.skip("compiled reference not available")
    return oracle.Reference()


@pytest.mark.parametrize("bench,iters,checkins,epochs", [(6, 3, 50, 10), (4, 2, 0, 10), (12, 5, 50, 50)])
def test_device_iterations_match_reference(dev, ref, bench, iters, checkins, epochs):
    # generated suites share ~15% of shaders between benchmarks (SuiteSpec::shared_fraction)
    h = ref.suite_generate(benchmark_count=bench, seed=11)
    kw = dict(num_iterations=iters, checkins_per_iteration=checkins, epochs=epochs, seed=5)
    o = ref.run_training(h, iters, checkins=checkins, epochs=epochs, seed=5)  # copy of the suite
    tuner = DeviceTuner(dev, TunerConfig(**kw))
    logs = []
    for i in range(iters):
        ref.suite_advance(h, checkins)              # run_iteration's advance_checkins
        s = ref.suite_export(h)
        keys = ref.suite_keys(h, len(s["features"]))
        logs.append(tuner.run_iteration(i, s, keys, ref.suite_checkin(h)))
    ref.suite_free(h)
    t = tuner.table.export()
    np.testing.assert_array_equal(t["keys"], o["keys"])
    np.testing.assert_array_equal(t["has"], o["has"])
    hv = o["has"].astype(bool)
    np.testing.assert_array_equal(t["q"][hv], o["q"][hv])
    np.testing.assert_array_equal(t["t"][hv], o["t"][hv])
    np.testing.assert_array_equal(t["cnt"][hv], o["cnt"][hv])
    ulp = np.abs(tuner.behavior.view(np.int32).astype(np.int64) -
                 o["policy"].view(np.int32).astype(np.int64))
    assert ulp.max() <= 1
    for i, lg in enumerate(logs):
        mr, size, loss, agree = o["logs"][i]
        assert lg["mean_reward"] == mr
        assert lg["table_size"] == int(size)
        assert lg["distill_loss"] == pytest.approx(loss, rel=1e-12)
        assert lg["agreement_rate"] == agree
