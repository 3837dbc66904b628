"""GPU: divide and conquer with every leaf solved by the CUDA core, against the reference's recorded outcomes."""
import pytest

from test_dnc_cpu import check_case, dnc_cases

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", dnc_cases(), ids=lambda c: c["name"])
def test_dnc_on_the_cuda_core_matches_reference_outcomes(case):
    check_case(case, None)


def test_dnc_large_window_on_device():
    from paper_2402_12373_b200 import dnc
    from paper_2402_12373_b200 import workloads as Wl
    from paper_2402_12373_b200.learner import LearnerConfig

    spec, alphabet, planted = Wl.planted_spec(3, 3000, 3000, 20, 60, "(p0 U (p1 & X p2)) & X(p1 | p2)", seed=77)
    res = dnc.dnc_learn(spec, alphabet, LearnerConfig(budget_bytes=8 << 30), dnc.SplitConfig("rand", window=1024, seed=3))
    assert dnc.separates(res.formula, spec, alphabet)
    assert res.enum_calls >= 1
