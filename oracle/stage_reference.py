#!/usr/bin/env python3
"""Stage the UNMODIFIED reference package into oracle/_ref (test infrastructure).

The reference (`svmps`, pure Python) cannot be imported on the GPU box, where
/root/reference does not exist.  This recipe copies its sources byte for byte
into oracle/_ref (git-ignored, so never committed; not gpurun-ignored, so it
travels with the snapshot like the built .so):

  oracle/_ref/svmps/           <- /root/reference/pkg/src/svmps  (package + data/*.fcidump)
  oracle/_ref/svmps_tests/     <- /root/reference/pkg/tests      (the reference's own tests)
  oracle/_ref/scripts/         <- /root/reference/pkg/scripts    (make_fixtures.py, H14/H16 builder)
  oracle/_ref/STAGED.json      <- sha256 of every staged file, to prove it is unmodified

Users: `bench.py --impl reference` / the cpu_baseline leg (the reference's own
SvAdaptEngine.energy + .screen) and `tests/test_gpu_dropin.py` (the reference's
own tests with libhsv installed as its SV engine).  Nothing on the product
path imports it.

  python oracle/stage_reference.py [--src /root/reference/pkg]
"""
from __future__ import annotations

import argparse
import hashlib
import json
import shutil
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
DEST = HERE / "_ref"
PARTS = (("src/svmps", "svmps"), ("tests", "svmps_tests"), ("scripts", "scripts"))


def _digest(root: Path) -> dict:
    out = {}
    for p in sorted(root.rglob("*")):
        if p.is_file() and "__pycache__" not in p.parts:
            out[str(p.relative_to(root))] = hashlib.sha256(p.read_bytes()).hexdigest()
    return out


def stage(src: Path = Path("/root/reference/pkg"), dest: Path = DEST) -> bool:
    """Copy the reference package; returns False (and leaves dest alone) when
    the reference tree is absent, e.g. on the GPU box."""
    if not (src / "src" / "svmps" / "__init__.py").exists():
        return False
    dest.mkdir(parents=True, exist_ok=True)
    manifest = {"source": str(src), "files": {}}
    for rel, name in PARTS:
        s, d = src / rel, dest / name
        if not s.exists():
            continue
        if d.exists():
            shutil.rmtree(d)
        shutil.copytree(s, d, ignore=shutil.ignore_patterns("__pycache__", "*.pyc"))
        sums_src, sums_dst = _digest(s), _digest(d)
        if sums_src != sums_dst:
            raise RuntimeError(f"staged copy of {s} differs from its source")
        manifest["files"][name] = sums_dst
    (dest / "STAGED.json").write_text(json.dumps(manifest, indent=1, sort_keys=True))
    return True


def verify(dest: Path = DEST) -> bool:
    """True when oracle/_ref holds an unmodified staged copy."""
    try:
        manifest = json.loads((dest / "STAGED.json").read_text())
    except (OSError, ValueError):
        return False
    return all(_digest(dest / name) == sums for name, sums in manifest["files"].items())


def import_path() -> Path | None:
    """Directory to put on sys.path for `import svmps`, or None if not staged."""
    return DEST if (DEST / "svmps" / "__init__.py").exists() else None


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--src", default="/root/reference/pkg")
    a = ap.parse_args()
    ok = stage(Path(a.src))
    print("staged" if ok else "reference tree absent; nothing staged", "->", DEST)
    sys.exit(0)
