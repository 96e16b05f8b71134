"""ParamTree mirror: same rules as the reference's params.py."""

import pytest

from paper_2103_07329_b200.errors import ConfigurationError
from paper_2103_07329_b200.params import ParamTree, tree


def test_defaults_role_dependent_iterations():
    t = tree({"solver": {"method": "CG"}, "preconditioner": {"method": "MultiGrid"},
              "pre_smoother": {"method": "Jacobi"}})
    assert t.role("solver").get_int("max_iters") == 100
    assert t.role("preconditioner").get_int("max_iters") == 1
    assert t.role("preconditioner").get_int("mg_coarse_matrix_size") == 500
    assert t.role("pre_smoother").get_float("weight") == 1.0
    assert t.validate() == []


def test_unknown_key_and_method_rejected():
    t = ParamTree()
    with pytest.raises(ConfigurationError):
        t.add("solver", "method", "Nope")
    t.add("solver", "method", "CG")
    with pytest.raises(ConfigurationError):
        t.add("solver", "weight", "1.0")
    with pytest.raises(ConfigurationError):
        t.add("bogus", "method", "CG")


def test_parse_error_at_finalize_and_frozen():
    t = ParamTree()
    t.add_map("solver", {"method": "CG", "max_iters": "ten"})
    with pytest.raises(ConfigurationError):
        t.set_defaults()
    t2 = tree({"solver": {"method": "CG"}})
    with pytest.raises(ConfigurationError):
        t2.add("solver", "max_iters", "3")


def test_legality_violations_reported():
    t = tree({"solver": {"method": "Chebyshev"}})
    assert any("not legal" in v for v in t.validate())


def test_method_switch_keeps_compatible_keys():
    t = ParamTree()
    t.add_map("solver", {"method": "BiCGStab", "merged": "1", "max_iters": "7"})
    t.add("solver", "method", "CG")
    assert t.role("solver").entries == {"max_iters": "7"}
