"""GPU: the reference's experiments (`benchgen.py:203-300`) on the CUDA core -- every recorded row of the masking
sweeps (26 mask widths x 3 specifications), the RUC experiment (2 seeds x 3 extension sizes x 2 hash schemes) and all
sample-bench generations, against values recorded from the reference's own run (tests/golden/make_benchgen_golden.py)."""
import pytest

from paper_2402_12373_b200 import benchgen as B
from test_benchgen_cpu import GOLD, check_samplebench, sweep_case

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", GOLD["samplebench"], ids=lambda c: f"i{c['i']}k{c['k']}s{c['seed']}")
def test_gen_samplebench_on_the_cuda_core(case):
    check_samplebench(case, None)


@pytest.mark.parametrize("case", GOLD["masking"], ids=lambda c: c["name"])
def test_masking_sweep_all_rows(case):
    sweep_case(case, B.MASKING_KS, None)


def test_ruc_experiment_matches_reference():
    g = GOLD["ruc"]
    got = B.run_ruc_experiment(g["n_seeds"], ext_sizes=tuple(g["ext_sizes"]), base_seed=g["base_seed"])
    keys = ("seed", "ext", "hash", "status", "cost", "precise", "minimal", "n_pos", "n_neg", "extra")
    assert [{k: r.get(k) for k in keys} for r in got["rows"]] == g["rows"]
    assert got["summary"] == g["summary"]
