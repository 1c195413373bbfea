"""pytest plugin: run the reference's own test files on libhsv.

  PYTHONPATH=oracle/_ref:. python -m pytest -p paper_2604_01176_b200.svmps_pytest \
      oracle/_ref/svmps_tests/test_svengine.py ...

`pytest_configure` runs before any test module (or the reference conftest)
is imported, so the `from svmps... import X` lines in the tests bind the
device versions.  The terminal summary reports how many libhsv kernels the
session launched, which is the evidence that the device engine did the work.
"""
from __future__ import annotations


def pytest_configure(config):
    from . import _native as N
    from .svmps_plugin import install
    N.init(0)
    install()
    N.lib().hsv_launch_count(1)


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    from . import _native as N
    from .svmps_plugin import _saved
    n = int(N.lib().hsv_launch_count(0))
    terminalreporter.write_line(f"HSV_DROPIN bindings={len(_saved)} libhsv_launches={n}")
