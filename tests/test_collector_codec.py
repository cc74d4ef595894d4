"""The collector drop-in's JSONL codec (paper_1908_06869_b200/host/collector.cpp)
against the reference's own collector.cpp (nlohmann/json 3.11.3 underneath):
the same program (tests/cpp/codec_check.cpp) is built against both and must
print identical bytes — ~201 K encoded records (integers, negative tags,
doubles over every exponent including Grisu2's non-shortest cases, escapes,
UTF-8), system-spec parses of malformed / edge JSON, and the exact IngestError
texts of streams that fail before any GPU step. Runs on CPU."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
BUILD = os.path.join(HERE, "cpp", "build")


def _bin(name):
    exe = os.path.join(BUILD, name)
    if not os.path.exists(exe):
        if os.path.isdir("/root/reference/proj/src"):
            subprocess.run(["make", "-s", "-C", os.path.join(HERE, "cpp"), "codec"], check=True)
        else:
            pytest.skip(f"{exe} not built (needs /root/reference at build time)")
    return exe


def test_codec_matches_reference_bytes():
    ref = subprocess.run([_bin("codec_ref")], capture_output=True, timeout=300)
    ours = subprocess.run([_bin("codec_b200")], capture_output=True, timeout=300)
    assert ref.returncode == 0 and ours.returncode == 0, ours.stderr[-2000:]
    a, b = ref.stdout.splitlines(), ours.stdout.splitlines()
    assert len(a) == len(b) > 200_000
    bad = [i for i, (x, y) in enumerate(zip(a, b)) if x != y]
    assert not bad, f"{len(bad)} lines differ, first: {a[bad[0]]!r} vs {b[bad[0]]!r}"
