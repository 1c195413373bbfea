"""Host-side checks of the svmps drop-in plugin and the staged reference
(no GPU: only the rebinding, not the compute)."""
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "oracle" / "_ref"

pytestmark = pytest.mark.skipif(not (REF / "svmps" / "__init__.py").exists(),
                                reason="reference not staged (python oracle/stage_reference.py)")


def test_staged_copy_matches_manifest():
    sys.path.insert(0, str(ROOT / "oracle"))
    try:
        import stage_reference
        assert stage_reference.verify()
    finally:
        sys.path.pop(0)


def test_install_rebinds_every_namespace_and_uninstall_restores():
    sys.path.insert(0, str(REF))
    try:
        import svmps.adapt
        import svmps.sparse
        import svmps.svengine
        from paper_2604_01176_b200 import svmps_plugin as P
        orig = (svmps.adapt.SvAdaptEngine, svmps.svengine.expectation, svmps.adapt.spmspv,
                svmps.spmspv, svmps.svengine.apply_qeb_exponential)
        P.install()
        try:
            assert svmps.adapt.SvAdaptEngine is P.HsvSvAdaptEngine
            assert svmps.svengine.expectation is P.expectation
            assert svmps.adapt.spmspv is P.spmspv           # `from .sparse import spmspv`
            assert svmps.spmspv is P.spmspv                 # package re-export
            assert svmps.svengine.apply_qeb_exponential is P.apply_qeb_exponential
            # make_engine reads the module global at call time (adapt.py:355-356)
            assert svmps.adapt.make_engine.__globals__["SvAdaptEngine"] is P.HsvSvAdaptEngine
            assert issubclass(P._ref["HsvCsrMatrix"], svmps.sparse.CsrMatrix)
        finally:
            P.uninstall()
        assert (svmps.adapt.SvAdaptEngine, svmps.svengine.expectation, svmps.adapt.spmspv,
                svmps.spmspv, svmps.svengine.apply_qeb_exponential) == orig
    finally:
        sys.path.remove(str(REF))
