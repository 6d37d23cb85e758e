"""The oracle pins must catch plausible mistakes: each
mutant below -- a one-token change to a scratch copy of oracle/physics.py --
must make at least one -m "not gpu" pin fail.  scripts/mutants.py runs the
full list against the three oracle test files."""
import os
import sys

import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts"))
import mutants  # noqa: E402

PINS = "llf or hand_values or worked_example or exact_translation or euler_flux or wave_speed or pressure or viscous"


@pytest.mark.parametrize("name", [m[0] for m in mutants.MUTANTS])
def test_mutant_is_killed(name):
    m = next(x for x in mutants.MUTANTS if x[0] == name)
    killed, failed = mutants.run(*m, k=PINS)
    assert killed, f"mutant {name} survived every pin"
