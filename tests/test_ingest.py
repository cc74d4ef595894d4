"""JSONL ingest on the GPU (csrc/ingest.cu, xsp_ingest_jsonl)
against the reference's own ingest() (collector.cpp:219-266, via oracle/_ref):
the span columns, metric / layer tables, trace arrays and interned name / type
tables must be identical; inputs outside the exactly handled cases must come
back as XSP_INGEST_HOST (the caller's host parser then gives the reference's
result or error). CPU tests pin the test workloads' JSONL through the
reference parser."""
import numpy as np
import pytest

from paper_1908_06869_b200 import columns, synth

COLS = ["span_id", "parent_id", "begin_ns", "end_ns", "cid", "flags", "name_id", "flops", "dram_read", "dram_write",
        "occupancy", "alloc_bytes", "type_id", "trace_span_off", "trace_id", "trace_levels", "trace_batch",
        "trace_run", "trace_serialized"]


def ref_streams():
    from oracle import ref
    g = ref.Generator()
    for r in range(3):
        g.emit("resnet-like", batch=2, run_index=r, jitter_max=1000, jitter_seed=r + 1)
    for m in ("mobilenet-like", "minimal", "async-straggler", "overlap"):
        g.emit(m)
    g.chain("resnet-like", 1, 15_700_000, 1000, 1.5)
    g.random_nested(7, 3000).random_async(9, 400)
    n = int(ref.lib().xspref_list_size(g.h))
    return [ref.list_jsonl(g, i) for i in range(n)]


def synth_streams(runs=2, models=3):
    b, *_ = synth.c3(runs=runs, n_models=models, max_layers=300)
    return [columns.to_jsonl(b, t) for t in range(b.n_traces)]


def assert_same(a, b):
    assert a.names == b.names and a.types == b.types
    assert a.system_name == b.system_name and a.peak_flops == b.peak_flops and a.mem_bw == b.mem_bw
    for k in COLS:
        x, y = np.asarray(getattr(a, k)), np.asarray(getattr(b, k))
        assert x.shape == y.shape, k
        assert np.array_equal(x.astype(np.float64).view(np.uint64) if x.dtype == np.float64 else x.astype(np.int64),
                              y.astype(np.float64).view(np.uint64) if y.dtype == np.float64 else y.astype(np.int64)), k


def test_workloads_parse_with_the_reference(has_ref):
    from oracle import ref
    for streams in (ref_streams(), synth_streams(1, 2)):
        b = ref.ingest(streams)
        assert b.n_traces == len(streams) and b.n_spans > 0


def _renamed(streams, fn):
    """The streams with every span name passed through fn (same JSON layout)."""
    import re
    out = []
    for s in streams:
        out.append(re.sub(rb'"name":"([^"]*)"', lambda m: b'"name":"' + fn(m.group(1)) + b'"', s))
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("which", ["reference_generators", "synth_c3", "shuffled_lines", "long_names",
                                   "shared_prefixes"])
def test_gpu_ingest_matches_reference(engine, has_ref, which):
    """long_names: names over 256 bytes (the interner's host sort); shared
    prefixes: names equal in their first 8 / 16 / 24 bytes and names that are
    prefixes of others (the device sort's zero-padded word order)."""
    from oracle import ref
    if which == "reference_generators":
        streams = ref_streams()
    elif which == "synth_c3":
        streams = synth_streams()
    elif which == "long_names":
        streams = _renamed(synth_streams(1, 2), lambda n: n + b"_" + b"x" * (250 + len(n) % 17))
    elif which == "shared_prefixes":
        streams = _renamed(synth_streams(1, 2),
                           lambda n: b"common/prefix/of/length32/" + n[: (len(n) * 7) % (len(n) + 1)])
    else:  # records out of timeline order: ingest sorts them (collector.cpp:256)
        rng = np.random.default_rng(4)
        streams = []
        for s in synth_streams(1, 2):
            lines = s.split(b"\n")[:-1]
            head, body = lines[:1], lines[1:]
            rng.shuffle(body)
            streams.append(b"\n".join(body[:5] + head + body[5:]) + b"\n")
    got, bad = engine.ingest_jsonl(streams)
    assert bad == -1, f"stream {bad} went to the host path"
    assert_same(got, ref.ingest(streams))
    # and the ingested columns run through the rest of the path
    c, t = engine.run_host(got)
    ra, rs = ref.correlate(got)
    import sys, os
    sys.path.insert(0, os.path.dirname(__file__))
    from parity import compare_correlation
    compare_correlation(got, c, ra, rs)


def _mutate(stream: bytes, what: str) -> bytes:
    lines = stream.split(b"\n")
    if what == "escape":
        lines[2] = lines[2].replace(b'"name":"', b'"name":"a\\"b', 1)
    elif what == "whitespace":
        lines[2] = lines[2].replace(b",", b", ", 1)
    elif what == "unknown_rec":
        lines.insert(1, b'{"rec":"other","x":1}')
    elif what == "no_meta":
        lines = lines[1:]
    elif what == "two_meta":
        lines.insert(1, lines[0])
    elif what == "trace_mismatch":
        lines[3] = lines[3].replace(b'"trace_id":', b'"trace_id":9', 1)
    elif what == "negative_duration":
        import re
        l = lines[3].decode()
        b = int(re.search(r'"begin_ns":(\d+)', l).group(1))
        lines[3] = re.sub(r'"end_ns":\d+', '"end_ns":%d' % max(b - 1, 0), l).encode() if b else lines[3]
    elif what == "long_double":
        lines = [l.replace(b'"achieved_occupancy":0.', b'"achieved_occupancy":0.30000000000000004', 1)
                 if b'achieved_occupancy' in l else l for l in lines]
    elif what == "non_ascii":
        lines[2] = lines[2].replace(b'"name":"', b'"name":"\xc3\xa9', 1)
    return b"\n".join(lines)


@pytest.mark.gpu
@pytest.mark.parametrize("what", ["escape", "whitespace", "unknown_rec", "no_meta", "two_meta", "trace_mismatch",
                                  "negative_duration", "long_double", "non_ascii"])
def test_gpu_ingest_defers_to_host(engine, has_ref, what):
    streams = synth_streams(1, 2)
    streams[1] = _mutate(streams[1], what)
    got, bad = engine.ingest_jsonl(streams)
    assert got is None and bad == 1, what


@pytest.mark.gpu
def test_gpu_ingest_hash_collision_goes_to_host(engine, has_ref, monkeypatch):
    """Distinct strings with equal hashes (forced by XSP_INGEST_HASH_BITS=3) are
    caught by the byte comparison against each slot's representative: the call
    reports XSP_INGEST_HOST instead of merging two names; with full hashes the
    same streams ingest on the GPU."""
    streams = synth_streams(1, 2)
    monkeypatch.setenv("XSP_INGEST_HASH_BITS", "3")
    got, bad = engine.ingest_jsonl(streams)
    assert got is None and bad == 0
    monkeypatch.delenv("XSP_INGEST_HASH_BITS")
    got, bad = engine.ingest_jsonl(streams)
    assert bad == -1
