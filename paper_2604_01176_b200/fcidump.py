"""Reference module name `svmps.fcidump` (fcidump.py:24-153): FCIDUMP parsing.
The implementation lives in chem.py."""
from .chem import IntegralSet, load_fcidump, parse_fcidump

__all__ = ["IntegralSet", "load_fcidump", "parse_fcidump"]
