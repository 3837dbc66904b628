"""B200-native enumerative LTL learner over characteristic sequences (hot path of arXiv 2402.12373).

Public API: `learn(P, N, alphabet, max_cost, costs)`; `enum_learn` / `LearnerConfig` mirror the reference's
`enumerator.py`; `core.make_core` is the drop-in for the reference's `kernels.make_core`.
"""
from .errors import BackendUnavailable, CoreError, CoreOOM, TimeoutExceeded  # noqa: F401
from .formula import CostHomomorphism, parse_formula, print_formula  # noqa: F401
from .learner import LearnerConfig, LearnResult, enum_learn, learn  # noqa: F401
from .scheme import HashScheme  # noqa: F401
from .traces import Alphabet, Specification, load_spec, save_spec  # noqa: F401

__all__ = ["learn", "enum_learn", "LearnerConfig", "LearnResult", "HashScheme", "Alphabet", "Specification",
           "load_spec", "save_spec", "parse_formula", "print_formula", "CostHomomorphism", "CoreOOM", "CoreError",
           "BackendUnavailable", "TimeoutExceeded"]
