"""Report emission: the reference report's CSV files
(report.cpp to_csv(to_table(aN(...)))) written on the GPU from the device
analysis tables (csrc/report.cu, xsp_report_csv), compared byte for byte with
the reference's own report module (oracle/_ref). The number formatter
(csrc/fmt.cuh: Ryu shortest digits laid out like std::to_chars) is also checked
as host code against std::to_chars over ~6 M doubles on CPU."""
import os
import subprocess

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
TABLES = ["a8", "a9", "a10", "a11", "a12", "a13", "a14"]


def test_fmt_matches_std_to_chars():
    exe = os.path.join(HERE, "cpp", "build", "fmt_check")
    subprocess.run(["make", "-s", "-C", os.path.join(HERE, "cpp"), "fmt"], check=True)
    out = subprocess.run([exe, "1000000"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout
    assert out.stdout.strip().startswith("0 of ")


def test_reference_report_shim(has_ref):
    from oracle import ref
    g = ref.Generator().emit("resnet-like", batch=2)
    b = g.batch()
    csv = ref.report_csv(b, 0, 1, 8)
    assert csv.startswith(b"name,layer_index,latency_ns,flops,")
    assert csv.count(b"\n") == 1 + 293


def quoted_names_batch():
    """resnet-like runs whose kernel and layer names carry CSV specials."""
    from oracle import ref
    g = ref.Generator()
    for r in range(3):
        g.emit("resnet-like", batch=4, run_index=r, jitter_max=2000, jitter_seed=r + 5)
    b = g.batch()
    names = list(b.names)
    for i in range(0, len(names), 7):
        names[i] = names[i] + b',"x"\nq'
    # keep the lexicographic order of the interned ids
    order = np.argsort(np.array(names, dtype=object), kind="stable")
    if not np.array_equal(order, np.arange(len(names))):
        return None
    b.names = names
    return b


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["resnet_runs", "c3_small", "c4_one_run", "quoted"])
def test_gpu_report_matches_reference(engine, has_ref, case):
    from oracle import ref
    from paper_1908_06869_b200 import synth
    from paper_1908_06869_b200.engine import DeviceBatch
    if case == "resnet_runs":
        g = ref.Generator()
        for r in range(5):
            g.emit("resnet-like", batch=8, run_index=r, jitter_max=3000, jitter_seed=r + 1)
        b = g.batch()
        groups = ([0], [5], [8])
    elif case == "c3_small":
        b, gf, gr, gb = synth.c3(runs=3, n_models=3, max_layers=200)
        groups = (gf, gr, gb)
    elif case == "c4_one_run":
        b = synth.c4(n_layers=3000, seed=3)
        groups = ([0], [1], [1])
    else:
        b = quoted_names_batch()
        if b is None:
            pytest.skip("renaming broke the name order")
        groups = ([0], [3], [4])
    dev = DeviceBatch(b)
    co = engine.correlate_device(dev)
    to = engine.analyze_device(dev, co, groups)
    first, runs = np.asarray(groups[0]), np.asarray(groups[1])
    for gi in range(min(len(first), 4)):
        for t in TABLES:
            ours = engine.report_csv(dev, co, groups, to, gi, t)
            want = ref.report_csv(b, int(first[gi]), int(runs[gi]), int(t[1:]))
            if ours != want:
                a, w = ours.split(b"\n"), want.split(b"\n")
                bad = next(i for i in range(min(len(a), len(w))) if a[i] != w[i]) if a != w else None
                pytest.fail(f"{case} group {gi} {t}: line {bad}: {a[bad] if bad is not None else ''!r} vs "
                            f"{w[bad] if bad is not None else ''!r} ({len(a)} vs {len(w)} lines)")
