"""Run the reference's own test suite (capsim 0.1.0, pkg/tests) against this package.

    python tools/run_reference_tests.py [pytest args...]

The suite is read from $CAPSIM_REF_TESTS, else /root/reference/pkg/tests (build container), else
baseline/_ref/pkg_tests (git-ignored; a copy of the reference's tests placed next to the reference
install so it travels to the GPU box with gpurun:
`cp -r /root/reference/pkg/tests baseline/_ref/pkg_tests`).

The reference's modules are aliased to ours (capsim -> paper_2306_12247_b200, capsim.profile ->
paper_2306_12247_b200.profile, ...) before pytest collects /root/reference/pkg/tests, so every
reference test exercises the drop-in API unchanged. Nothing is copied: the tests are read where
they lie. Tests that evaluate policies need the B200 (no CPU fallback) and fail on a CPU host with
NativeLibraryError; the CLI (out of scope) is not aliased, so test_cli.py is ignored.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
_CANDIDATES = [os.environ.get("CAPSIM_REF_TESTS", ""), "/root/reference/pkg/tests",
               str(ROOT / "baseline" / "_ref" / "pkg_tests")]
REF_TESTS = next((Path(c) for c in _CANDIDATES if c and Path(c).is_dir()), Path(_CANDIDATES[1]))


def main() -> int:
    if not REF_TESTS.exists():
        print(f"no reference test suite found (looked in {[c for c in _CANDIDATES if c]})")
        return 0
    sys.path.insert(0, str(ROOT))
    import paper_2306_12247_b200 as pkg
    from paper_2306_12247_b200 import controller, errors, policy, profile, sim, trace

    sys.modules["capsim"] = pkg
    for name, mod in (("profile", profile), ("trace", trace), ("policy", policy), ("sim", sim),
                      ("errors", errors), ("controller", controller)):
        sys.modules[f"capsim.{name}"] = mod
    import pytest

    args = [str(REF_TESTS), "-q", "-p", "no:cacheprovider", "--ignore", str(REF_TESTS / "test_cli.py"),
            "--rootdir", str(ROOT)] + sys.argv[1:]
    return pytest.main(args)


if __name__ == "__main__":
    sys.exit(main())
