"""Full-size, full-population GPU parity of the BASELINE configs (VERDICT r1 "next" 1):
every CN of C1-C4 re-trained by the oracle, the merged network against the oracle's
merged network, the R24 kink accounting for ReLU CNs over 1e-4, the R22 envelope for
smooth ones, and the GPU-trained vs oracle-trained labels on the full test set
(R26(ii)).  C5 (bf16, one full epoch of all 8 CNs, ~6 min of oracle time) and F1 (20
epochs) are marked slow.  Logic in tests/fullsize.py; tools/parity_report.py writes
the same reports to profiles/parity_r2.json."""
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    torch.cuda.set_device(0)


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_full_population(orc, name):
    from tests.fullsize import assert_report, run_full
    rep = run_full(orc, name)
    assert_report(rep)


@pytest.mark.slow
def test_c5_full_epoch_bf16(orc):
    from tests.fullsize import assert_report, run_full
    rep = run_full(orc, "C5", epochs=1)
    assert_report(rep)
