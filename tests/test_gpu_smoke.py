"""GPU: the driver's smoke() entry point (toy step vs the reference golden, U-Net step
vs the fp64 oracle) runs clean."""
import pytest

pytestmark = pytest.mark.gpu


def test_graft_entry_smoke():
    import __graft_entry__
    __graft_entry__.smoke()
