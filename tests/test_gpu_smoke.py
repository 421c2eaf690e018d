"""The driver's round-end smoke() (tiny 2DSW and SOR runs against the oracle),
run inside the GPU suite so a change that breaks it fails here first."""
import pytest

pytestmark = pytest.mark.gpu


def test_graft_entry_smoke():
    import __graft_entry__
    __graft_entry__.smoke()
