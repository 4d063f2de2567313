import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C ABI)")
    config.addinivalue_line("markers", "slow: longer statistical pins (still CPU)")


@pytest.fixture(scope="session")
def oracle_lib():
    from oracle import nsso
    nsso.lib()
    return nsso


def pytest_terminal_summary(terminalreporter):
    """SURVEY C-9 guard band: report the precision ties of every parity case."""
    try:
        from tests.parity_util import TIE_LOG
    except Exception:
        return
    if not TIE_LOG:
        return
    chains = sum(k for _, k, _ in TIE_LOG)
    ties = sum(t for _, _, t in TIE_LOG)
    terminalreporter.write_line(
        f"precision ties (C-9 guard band): {ties} of {chains} chains over {len(TIE_LOG)} parity comparisons")
    for case, k, t in TIE_LOG:
        if t:
            terminalreporter.write_line(f"  {case}: {t}/{k}")
