"""The CPU oracle re-passes the reference's own known-answer and property
tests (restated in oracle/orc_kats.cpp, each case citing
proj/tests/<file>:<lines>).  CPU only."""
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_oracle_reference_kats(oracle_built):
    r = subprocess.run([str(ROOT / "oracle" / "_build" / "orc_kats")], capture_output=True, text=True, timeout=600)
    summary = [l for l in r.stdout.splitlines() if l.startswith("KAT summary")]
    assert r.returncode == 0, r.stdout[-3000:]
    assert summary and "failures=0" in summary[0]
    assert int(summary[0].split("cases=")[1].split()[0]) >= 40
