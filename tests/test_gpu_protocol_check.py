"""The single-pass sweep under its protocol-check build (compute-sanitizer is closed on
this GPU pool): every dot / q slot carries the row index it holds,
checked by its readers.  Builds build_ab/f4check.so (tools/build_f4_variant.sh, nvcc) and
runs tools/f4_check.py --quick in a subprocess: zero tag mismatches over row widths 300 to
10,000, FP64 and FP32, forced row batches / groups, and the fused z equal to the two-pass z
(FP64, 1e-9)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_single_pass_protocol_tags():
    so = os.path.join(ROOT, "build_ab", "f4check.so")
    r = subprocess.run(["bash", os.path.join(ROOT, "tools", "build_f4_variant.sh"), "f4check", "-DBIC_F4_CHECK"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0 and os.path.exists(so), r.stderr[-2000:]
    env = dict(os.environ, BICADMM_LIB_PATH=so)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "f4_check.py"), "--quick"], capture_output=True,
                       text=True, timeout=1200, cwd=ROOT, env=env)
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    summary = [l for l in lines if "summary" in l]
    assert summary, r.stdout[-2000:] + r.stderr[-2000:]
    s = summary[0]["summary"]
    assert s["check_build"]   # bicadmm_debug_f4_check_build() == 1: the tags were really counted
    assert s["tag_errors"] == 0, [l for l in lines if l.get("tag_errors")]
    assert s["worst_rel_f64"] <= 1e-9, s
    assert s["fused_runs"] >= 0.8 * s["runs"], s
    assert r.returncode == 0
