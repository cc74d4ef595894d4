#!/usr/bin/env python
"""Benchmark: M spans/s correlated + analysed (BASELINE.json metric) on B200.

Headline workload (BASELINE.json configs[4], "C5", the largest single-GPU
config): ~1 B spans = the C3 corpus (configs[2]: 65 synthetic models x 8 batch
sizes (1..128) x R=20 iterations, 47.75 M spans) replicated 21x in HBM as
independent traces, every span through xsp_run (parent join, cid join,
per-kernel/layer/name/type/model tables, roofline classification, top-3 per
layer) in device-resident calls of <= 11 copies. Inputs (~60 GB) are far larger
than the 126 MB L2, so no L2 flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N>1: one process per GPU (torchrun); the C5 copies are trace-sharded over the
ranks (no data-path collective; strong scaling); time is the max over ranks.
`value` is device-resident throughput; `e2e` goes through the host-buffer C-ABI
entry (xsp_run_host) with H2D of the inputs and D2H of all result columns inside
the timed region. Extra keys: `c3` (the single C3 corpus, device-resident and
e2e), `sort_shuffled`, `c4` (one 219 M-span trace). `--impl reference` times the
reference's own CPU implementation (oracle/_ref, unmodified strata sources) with
all host threads on a bounded sample of the same corpus.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "M spans/sec correlated+analyzed at 1/2/4/8 B200; % of HBM roofline"
UNIT = "M spans/s"
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")


def hbm_peak():
    try:
        with open(PEAKS) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.device)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc:
            time.sleep(0.2)
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=10)
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            p = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(p[0]))
                mx = float(p[1])
            except (ValueError, IndexError):
                continue
            for n, v in zip(names, p[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def pass1_bytes(b) -> int:
    """Algorithmic bytes of one k_pass1 launch in direct mode (k_pass1<true>, the
    clean-batch path the bench runs): reads every span's flags
    (1 B), begin and end (16 B), its placed-layer bit (1/8 B, from k_p1_reduce)
    and the cid of spans that carry one (8 B), plus the name_id (4 B) and the
    occupancy (8 B, by metric row) of every execution record with a cid; writes
    the kernel table row of every kernel (launch row, exec row, metric row,
    name: 4 B each; duration, occupancy: 8 B each = 32 B), 20 B per placed layer
    (row, duration, layer-table row, first-kernel offset) and 12 B of offsets
    per trace."""
    f = b.flags
    lvl, kind = f & 3, (f >> 2) & 3
    n = b.n_spans
    has_c = int(((f & 0x20) != 0).sum())
    layer = int(((lvl == 1) & (kind == 0)).sum())
    exe = int(((kind == 2) & ((f & 0x20) != 0)).sum())
    reads = n * 17 + n // 8 + has_c * 8 + exe * (4 + 8)
    writes = layer * 20 + exe * 32 + b.n_traces * 12
    return reads + writes


def measured_traffic(kernel: str, spans: int = 0):
    """dram__bytes_read.sum + dram__bytes_write.sum of `kernel` from the committed
    ncu --set full capture summary (profiles/traffic.json, tools/traffic_from_ncu.py),
    scaled per span to a launch over `spans` spans (the captured launch's own
    count if 0), or None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)[kernel]
        n = spans or d["spans"]
        return {"bytes": int(round(d["bytes_per_span"] * n)), "bytes_per_span": d["bytes_per_span"],
                "captured_launch": {"spans": d["spans"], "dram_bytes": d["dram_bytes"],
                                    "duration_us": d["duration_us"]},
                "capture": d["capture"], "workload": d["workload"]}
    except Exception:
        return None


def survey_bytes(b) -> float:
    """SURVEY.md §8(d) algorithmic bytes for the whole pipeline: per layer with K kernels
    (157 + 162 K) B, plus a 96 B model row per trace."""
    f = b.flags
    lvl, kind = f & 3, (f >> 2) & 3
    layers = int(((lvl == 1) & (kind == 0)).sum())
    kernels = int(((kind == 1) & (lvl >= 2)).sum()) + int(((kind == 0) & (lvl == 2)).sum())
    return 157.0 * layers + 162.0 * kernels + 96.0 * b.n_traces


def make_workload(args, rank: int):
    from paper_1908_06869_b200 import synth
    return synth.c3(runs=args.runs, n_models=args.models, seed=1 + rank)


def sample_groups(gf, gr, b, max_spans: int):
    """First groups of the corpus up to ~max_spans spans (bounded CPU sample)."""
    off = b.trace_span_off
    k = 0
    while k < len(gf):
        end = int(off[gf[k] + gr[k]])
        if end > max_spans and k > 0:
            break
        k += 1
    return k, int(off[gf[k - 1] + gr[k - 1]])


def cpu_reference(b, gf, gr, max_spans: int, reps: int = 1):
    from oracle import ref
    k, spans = sample_groups(gf, gr, b, max_spans)
    sub = b.trace_slice(0, int(gf[k - 1] + gr[k - 1]))
    threads = os.cpu_count() or 1
    secs = ref.time_pipeline(sub, gf[:k], gr[:k], threads, reps)
    return {"value": spans / secs / 1e6, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"first {k} of {len(gf)} (model,batch) groups = {spans} spans, "
                      f"correlate + a8..a15 per group, {threads} threads (oracle/_ref, unmodified strata)",
            "seconds": secs}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import ref
    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libxsp_ref.so not built"}))
        return
    from paper_1908_06869_b200 import synth
    # a bounded sample of the same corpus: the first models of the C3 family
    models = synth.make_models(args.models, seed=1)[:max(1, args.models // 10)]
    b, gf, gr, gb = synth.corpus(models, (1, 2, 4, 8, 16, 32, 64, 128), args.runs, seed=1 + 1000)
    budget = args.ref_sample_spans
    for _ in range(args.warmup):
        cpu_reference(b, gf, gr, budget // 4)
    vals, secs = [], 0.0
    for _ in range(args.steps):
        r = cpu_reference(b, gf, gr, budget)
        vals.append(r["value"])
        secs += r["seconds"]
    v = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64/f64",
            "data": "synthetic", "config": config(args),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": r["cores"], "kind": "reference",
                             "sample": r["sample"]},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


class _ShuffledColumns:
    """The sort_timeline input columns of a corpus with every trace's rows permuted
    at random (on the device), in the DeviceBatch pointer interface."""

    def __init__(self, dev, b, seed: int):
        import torch
        g = torch.Generator(device=dev.t["begin_ns"].device).manual_seed(seed)
        n = b.n_spans
        off = dev.t["trace_span_off"]
        rows = torch.arange(n, device=off.device, dtype=torch.int64)
        tr = torch.searchsorted(off, rows, right=True) - 1
        key = tr * (1 << 31) + torch.randint(0, 1 << 31, (n,), device=off.device, generator=g)
        perm = torch.argsort(key)
        self.batch = b
        self.t = {k: dev.t[k][perm].contiguous() for k in ("begin_ns", "flags", "span_id")}
        self.t["trace_span_off"] = off

    def ptr(self, k):
        return self.t[k].data_ptr()


def measure_sort(eng, dev, b, steps: int, local: int):
    """sort_timeline on a per-trace shuffled copy of the corpus:
    device-resident, CUDA events around `steps` calls."""
    import torch
    sh = _ShuffledColumns(dev, b, seed=11)
    perm = torch.empty(b.n_spans, dtype=torch.int32, device=f"cuda:{local}")
    stream = torch.cuda.current_stream().cuda_stream
    for _ in range(2):
        assert not eng.sort_timeline_device(sh, perm.data_ptr(), stream)
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(steps):
        eng.sort_timeline_device(sh, perm.data_ptr(), stream)
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / steps
    # spot check against a stable lexsort on a sample of traces
    off = b.trace_span_off
    p = perm.cpu().numpy().view(np.uint32)
    bg, fl, sid = (sh.t[k].cpu().numpy() for k in ("begin_ns", "flags", "span_id"))
    for t in range(0, b.n_traces, max(1, b.n_traces // 16)):
        lo, hi = int(off[t]), int(off[t + 1])
        lv = fl[lo:hi].astype(np.int64) & 3
        want = lo + np.lexsort((sid[lo:hi], np.where(lv >= 2, 3, lv + 1), bg[lo:hi]))
        assert np.array_equal(p[lo:hi], want.astype(np.uint32)), f"sort mismatch in trace {t}"
    return {"metric": "M spans/s sorted (sort_timeline, shuffled traces)", "value": b.n_spans / (ms / 1e3) / 1e6,
            "unit": UNIT, "ms_per_step": ms, "gbs": 21.0 * b.n_spans / (ms / 1e3) / 1e9,
            "input": "C3 corpus, rows of every trace permuted at random on the device"}


def measure_validate(eng, dev, b, steps: int):
    """validate_bundle (stage (a), span.cpp:129-192) of every C3 trace on the
    device (xsp_validate: per-span rules, timeline order, duplicate span ids by
    a device hash table, bundle-level rules): CUDA events around `steps` calls.
    Algorithmic bytes: span_id, begin, end, cid (32 B) + flags (1 B) per span
    + the metric table (32 B per metric row)."""
    import ctypes as C
    import torch
    from paper_1908_06869_b200 import _capi as capi
    cols, trs = dev.cols(), dev.traces()
    vin = capi.ValidateIn()
    out = capi.ValidationOut()
    stream = torch.cuda.current_stream().cuda_stream

    def call():
        eng._check(eng.lib.xsp_validate(eng.ctx, C.byref(cols), C.byref(trs), C.byref(vin), C.byref(out),
                                        C.c_void_p(stream)))

    call()
    assert out.n_issues == 0
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(steps):
        call()
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / steps
    met = int(((b.flags & 0x40) != 0).sum())
    byts = 33 * b.n_spans + 32 * met
    return {"metric": "M spans/s validated (validate_bundle, device-resident)", "value": b.n_spans / (ms / 1e3) / 1e6,
            "unit": UNIT, "ms_per_step": ms, "issues": int(out.n_issues),
            "roofline": {"bound": "hbm", "bytes": byts, "achieved": byts / (ms / 1e3) / 1e9, "unit": "GB/s"},
            "input": "C3 corpus (every trace valid)"}


def measure_c4(eng, args, rank: int, world: int, local: int, dist):
    """BASELINE config 4: one long trace (synth.c4, no quiescent instants),
    time-range sharded over the ranks with a carried open-parent boundary
    (timeshard.py: equal row ranges, open layers carried forward, executions
    routed to their launch's rank over NCCL). Every rank correlates + analyses
    its sub-batch device-resident, timed with CUDA events, max over ranks
    (strong scaling). At N > 1 the per-rank tables then travel to rank 0 and are
    combined; that time is reported next to the compute time."""
    import torch
    from paper_1908_06869_b200 import synth, timeshard
    from paper_1908_06869_b200.engine import DeviceBatch
    b = synth.c4(n_layers=args.c4_layers)
    stats, sh, comm = {}, None, None
    if world > 1:
        comm = timeshard.TorchComm(dist, f"cuda:{local}" if dist.get_backend() == "nccl" else "cpu")
        bounds = timeshard.shard_bounds(b, world)
        sh = timeshard.prepare(b, bounds[rank], bounds[rank + 1], comm)
        sub, stats = sh.sub, sh.stats
    else:
        sub = b
    dev = DeviceBatch(sub, local)
    groups = ([0], [1], [1])
    stream = torch.cuda.current_stream().cuda_stream

    last = {}

    def step():
        co = eng.correlate_device(dev, stream=stream)
        last["co"], last["to"] = co, eng.analyze_device(dev, co, groups, stream=stream)

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(max(1, args.steps // 2)):
        step()
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / max(1, args.steps // 2)
    # report emission: the a8 CSV (one row per kernel) of the
    # trace, formatted on the GPU from the device tables (text left in HBM)
    report = None
    if rank == 0:
        names, k1 = eng.string_table(sub.names)
        types, k2 = eng.string_table(sub.types)
        g, k3 = eng.make_groups(*groups)
        cols = dev.cols()
        import ctypes as C
        text, n = C.c_char_p(), C.c_uint64()
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for rep in range(2):
            r0.record()
            eng._check(eng.lib.xsp_report_csv(eng.ctx, C.byref(cols), C.byref(last["co"]), C.byref(g),
                                              C.byref(last["to"]), C.byref(names), C.byref(types), 0, 8,
                                              C.byref(text), C.byref(n), C.c_void_p(stream)))
            r1.record()
            torch.cuda.synchronize()
        rms = r0.elapsed_time(r1)
        report = {"table": "a8 (one CSV row per kernel)", "rows": int(last["to"].n_kernels), "bytes": n.value,
                  "ms": rms, "GB_per_s": n.value / (rms / 1e3) / 1e9,
                  "M_rows_per_s": last["to"].n_kernels / (rms / 1e3) / 1e6,
                  "how": "xsp_report_csv into HBM (size pass, scan, write pass; includes two small count "
                         "read-backs), CUDA events"}
    del dev
    combine_ms = None
    if dist:
        t = torch.tensor([ms], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        corr, tabs = eng.run_host(sub)
        fp = timeshard.fusion_orphan_parents(sh, corr)
        dist.barrier()
        c0 = time.perf_counter()
        blobs = comm.gather_bytes(timeshard.pack_part(sh, corr, tabs, fp))
        if rank == 0:
            parts = [timeshard.unpack_part(x, timeshard.CORR_DTYPES, timeshard.TAB_DTYPES) for x in blobs]
            timeshard.combine(b, parts)
        combine_ms = (time.perf_counter() - c0) * 1e3
    out = {"metric": "M spans/s correlated+analyzed, one long trace time-range sharded",
           "value": b.n_spans / (ms / 1e3) / 1e6, "unit": UNIT, "ms_per_step": ms, "spans": b.n_spans,
           "layers": args.c4_layers, "shards": world, "scaling": "strong",
           "workload": "C4: synth.c4, 1 model span, layers x ~3 kernels (1% long layers of 8..64, 0.1% "
                       "concurrent pairs), executions on 4 interleaved streams, no drains (no quiescent instant)"}
    if report:
        out["report_a8_csv"] = report
    if combine_ms is not None:
        out["combine_ms"] = combine_ms
        out["value_incl_combine"] = b.n_spans / ((ms + combine_ms) / 1e3) / 1e6
        out["shard_stats_rank0"] = stats
    return out


def measure_leveled(eng, args, local: int):
    """BASELINE config 2 at scale (stage (f), leveled.cpp:145-231): 65 synthetic
    models, each profiled at {M}, {M,L}, {M,L,G} x 10 repetitions (synth.
    leveled_corpus, simprof's leveled-chain shape with per-level profiling
    overhead); one step = correlate every run (one call) + compute_overhead of
    every model's LeveledRunGroup (one xsp_leveled_batch call: three host round
    trips for all 65 groups; chain orders are decided on the host).
    Device-resident, CUDA events. `per_group_ms` times the same step with one
    synchronous xsp_leveled per group."""
    import torch
    from paper_1908_06869_b200 import synth
    from paper_1908_06869_b200.engine import DeviceBatch
    models = synth.make_models(args.leveled_models, seed=3)
    b, sets = synth.leveled_corpus(models, runs=args.leveled_runs)
    dev = DeviceBatch(b, local)
    ls = [eng.make_level_sets(s) for s in sets]
    stream = torch.cuda.current_stream().cuda_stream
    n_events = sum(1 + m.layer_ns.size + m.exec_ns.size for m in models)
    runs_per_model = 3 * args.leveled_runs

    def step_per_group():
        co = eng.correlate_device(dev, stream=stream)
        for s, _ in ls:
            out = eng.leveled_device(dev, co, s, stream=stream)
            assert out.status == 0 and out.n_sets == 3

    def step():
        co = eng.correlate_device(dev, stream=stream)
        outs = eng.leveled_batch_device(dev, co, [s for s, _ in ls], stream=stream)
        assert all(o.status == 0 and o.n_sets == 3 for o in outs)

    def time_of(fn):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        steps = max(2, args.steps // 4)
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in range(steps):
            fn()
        t1.record()
        torch.cuda.synchronize()
        return t0.elapsed_time(t1) / steps

    per_group_ms = time_of(step_per_group)
    ms = time_of(step)
    eng.set_profiling(True)
    eng.stage_reset()
    step()
    torch.cuda.synchronize()
    st = eng.stage_times()
    eng.set_profiling(False)
    lev_ms = sum(v[0] for k, v in st.items() if k.startswith("lev"))
    byts = n_events * runs_per_model * 8 + n_events * 24
    return {"metric": "M spans/s correlated + leveled (compute_overhead), device-resident",
            "value": b.n_spans / (ms / 1e3) / 1e6, "unit": UNIT, "ms_per_step": ms, "spans": b.n_spans,
            "per_group_ms": per_group_ms,
            "models": len(models), "runs_per_level_set": args.leveled_runs, "events": n_events,
            "workload": "C2 at scale: 65 synthetic models x level sets {M},{M,L},{M,L,G} x 10 runs, batch 1",
            "stages_ms": {k: v[0] for k, v in st.items()},
            "roofline": {"bound": "hbm", "kernels": "k_lev_*", "bytes": byts,
                         "definition": "SURVEY 8(d): 8 B per (event, run) + 24 B per event",
                         "achieved": byts / (lev_ms / 1e3) / 1e9 if lev_ms else None, "unit": "GB/s",
                         "note": "k_lev_latency gathers each (set, event) sample by trace (one row per run): latency bound at this size; the step is 3 host round trips + correlate"}}


def measure_ingest(eng, args, local: int, with_cpu: bool):
    """JSONL wire-format ingest on the GPU (xsp_ingest_jsonl):
    H2D of the text, line parse, name / type interning, sort_timeline and
    validate_bundle, columns left in HBM. Workload: one run of every (model,
    batch) group of the C3 family as JSONL streams (one TraceBundle each; the
    reference writer's record layout). cpu_baseline: the reference's own
    ingest() (oracle/_ref, one thread) on a bounded sample of the same streams."""
    import ctypes as C
    import torch
    from paper_1908_06869_b200 import _capi as capi
    from paper_1908_06869_b200 import columns, synth
    b, *_ = synth.c3(runs=1, n_models=args.ingest_models)
    streams = [columns.to_jsonl(b, t) for t in range(b.n_traces)]
    # the text in page-locked memory, as a reader that fills a pinned buffer
    # from files hands it over (pageable text is staged by the driver at ~1/4
    # of the PCIe rate)
    raw = b"".join(streams)
    pinned = torch.empty(len(raw), dtype=torch.uint8).pin_memory()
    pinned.numpy()[:] = np.frombuffer(raw, dtype=np.uint8)
    blob = C.cast(C.c_void_p(pinned.data_ptr()), C.c_char_p)
    off = np.zeros(len(streams) + 1, dtype=np.uint64)
    off[1:] = np.cumsum([len(x) for x in streams])
    out = capi.IngestOut()
    stream = torch.cuda.current_stream().cuda_stream

    def call():
        eng._check(eng.lib.xsp_ingest_jsonl(eng.ctx, blob, off.ctypes.data_as(capi.u64p), len(streams),
                                            C.byref(out), C.c_void_p(stream)))
        assert out.status == capi.INGEST_OK and out.cols.n_spans == b.n_spans

    call()
    torch.cuda.synchronize()
    reps = 3
    t0 = time.perf_counter()
    for _ in range(reps):
        call()
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / reps * 1e3
    line = {"metric": "M spans/s ingested from JSONL (GPU, host text to device columns)",
            "value": b.n_spans / (ms / 1e3) / 1e6, "unit": UNIT, "ms_per_step": ms, "spans": b.n_spans,
            "streams": len(streams), "text_bytes": len(raw), "text_GB_per_s": len(raw) / (ms / 1e3) / 1e9,
            "how": "xsp_ingest_jsonl wall time on page-locked text (synchronous call: H2D of the text + line "
                   "index + parse + intern + sort + validate)",
            "workload": f"C3 family, {args.ingest_models} models x 8 batch sizes x 1 run as JSONL streams"}
    if with_cpu:
        from oracle import ref
        if ref.available():
            k = max(1, min(len(streams), 24))
            t0 = time.perf_counter()
            rb = ref.ingest(streams[:k])
            sec = time.perf_counter() - t0
            line["cpu_baseline"] = {"value": rb.n_spans / sec / 1e6, "unit": UNIT, "cores": 1, "kind": "reference",
                                    "sample": f"first {k} streams = {rb.n_spans} spans through the reference's ingest()"}
    return line


class _Replica:
    """DeviceBatch interface over slices of replicated device columns."""

    def __init__(self, batch_ns, tensors):
        from paper_1908_06869_b200.engine import DeviceBatch
        self.batch, self.t = batch_ns, tensors
        self._db = DeviceBatch

    def _p(self, k, typ):
        return self._db._p(self, k, typ)

    def cols(self):
        return self._db.cols(self)

    def traces(self):
        return self._db.traces(self)


class C5:
    """BASELINE config 5: a ~1 B-span multi-trace corpus — the C3 corpus
    replicated `copies` times in HBM (independent traces) — correlated +
    analysed as device-resident xsp_run calls of up to `per_call` copies
    (~0.5 B spans) each. Under N ranks the copies are trace-sharded over the
    ranks (rank r holds copies r, r+N, ...; strong scaling, max over ranks).
    Every copy must come back with the C3 counts (no orphans, no failures)."""

    def __init__(self, eng, dev, b, groups, copies: int = 21, per_call: int = 11, rank: int = 0, world: int = 1):
        import torch
        from types import SimpleNamespace
        self.eng, self.b, self.copies_all = eng, b, copies
        self.mine = list(range(rank, copies, world))
        copies = len(self.mine)
        n, T = b.n_spans, b.n_traces
        M, Lr = b.flops.size, b.alloc_bytes.size
        metric_cols = {"flops", "dram_read", "dram_write", "occupancy"}
        layer_cols = {"alloc_bytes", "type_id"}
        self.big = {k: t.repeat(copies) for k, t in dev.t.items() if k not in ("trace_span_off", "trace_levels")}
        off = dev.t["trace_span_off"]
        offs = torch.cat([off[:-1] + k * n for k in range(per_call)] + [off[-1:] + (per_call - 1) * n])
        levels = dev.t["trace_levels"].repeat(per_call)
        gf, gr, gb = (np.asarray(x) for x in groups)
        co, _ = eng.run_device(dev, groups)
        self.want_l, self.want_k = int(co.n_layers), int(co.n_kernels)
        self.calls = []
        for k0 in range(0, copies, per_call):
            kk = min(per_call, copies - k0)
            t = {}
            for key, tens in self.big.items():
                per = M if key in metric_cols else (Lr if key in layer_cols else n)
                t[key] = tens[k0 * per:(k0 + kk) * per]
            t["trace_span_off"] = offs[:kk * T + 1]
            t["trace_levels"] = levels[:kk * T]
            ns = SimpleNamespace(n_spans=kk * n, n_traces=kk * T, flops=np.empty(kk * M, np.uint8),
                                 alloc_bytes=np.empty(kk * Lr, np.uint8), peak_flops=b.peak_flops,
                                 mem_bw=b.mem_bw)
            g = (np.concatenate([gf + j * T for j in range(kk)]), np.tile(gr, kk), np.tile(gb, kk))
            self.calls.append((_Replica(ns, t), g, kk))
        self.spans_mine = n * copies
        self.spans_all = n * self.copies_all

    def step(self, stream, check=False) -> int:
        launches = 0
        for view, g, kk in self.calls:
            co, _ = self.eng.run_device(view, g, stream=stream)
            launches += self.eng.launches
            if check:
                assert co.n_failed == 0 and co.n_orphans == 0, "C5: unexpected failures / orphans"
                assert int(co.n_layers) == kk * self.want_l and int(co.n_kernels) == kk * self.want_k, "C5: counts"
        return launches

    def pass1_bytes(self) -> int:
        """k_pass1 algorithmic bytes summed over one step's launches."""
        return pass1_bytes(self.b) * len(self.mine)

    def release(self):
        import torch
        del self.big, self.calls
        torch.cuda.empty_cache()


def e2e_host(eng, hb, groups, copies: int, steps: int, barrier, dist, packed=None, rows_only=False):
    """End to end through the host-buffer C ABI (xsp_run_host, or
    xsp_run_host_packed when `packed` is given): every step runs `copies` calls
    on pinned host columns, each with H2D of its inputs and D2H of every result
    column inside the timed region (wall clock around the calls, device
    synchronised on both sides; max over ranks)."""
    import torch
    from paper_1908_06869_b200 import _capi as capi

    eng.set_host_outputs(capi.HOST_OUT_ROWS if rows_only else capi.HOST_OUT_ALL)

    def call():
        if packed is not None:
            eng.run_host_packed(packed, hb, groups=groups, raw=True)
        else:
            eng.run_host(hb, groups=groups, raw=True)

    call()
    barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        for _ in range(copies):
            call()
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3 / steps
    h2d, d2h = eng.transfer_bytes()
    eng.set_host_outputs(capi.HOST_OUT_ALL)
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms, h2d * copies, d2h * copies


def config(args):
    return {"workload": "C5: ~1 B spans = the C3 corpus (65 synthetic models x 8 batch sizes (1..128) x R "
                        "iterations) replicated 21x as independent traces; correlate + a5..a15 + top-3, one "
                        "analysis group per (model, batch) copy",
            "models": args.models, "batches": [1, 2, 4, 8, 16, 32, 64, 128], "iterations": args.runs,
            "copies": 21, "l2": "inputs (>40 GB/GPU) exceed the 126 MB L2; no flush needed",
            "parallelism": f"trace-sharded x{args.gpus} (copies over ranks, strong)"}


def c3_config(args):
    return {"workload": "C3: 65 synthetic models x 8 batch sizes (1..128) x R iterations, correlate + "
                        "a5..a15 + top-3, one group per (model,batch)",
            "models": args.models, "batches": [1, 2, 4, 8, 16, 32, 64, 128], "iterations": args.runs}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--runs", type=int, default=20, help="iterations per (model, batch) group")
    ap.add_argument("--models", type=int, default=65)
    ap.add_argument("--ref-sample-spans", type=int, default=3_000_000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sort", action="store_true", help="skip the shuffled sort_timeline measurement")
    ap.add_argument("--c5-copies", type=int, default=21, help="C3 copies of the C5 corpus (headline)")
    ap.add_argument("--e2e-steps", type=int, default=2, help="steps of the end-to-end (host buffer) C5 timing")
    ap.add_argument("--leveled-models", type=int, default=65, help="0 skips the leveled (C2 at scale) line")
    ap.add_argument("--leveled-runs", type=int, default=10)
    ap.add_argument("--ingest-models", type=int, default=24, help="0 skips the JSONL ingest line")
    ap.add_argument("--c4-layers", type=int, default=28_600_000,
                    help="layers of the C4 long trace (~7 spans per layer; 0 skips the C4 measurement)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    # one rank per GPU; ranks beyond the visible GPUs share them (only useful to
    # exercise the N > 1 code paths on a small box, with XSP_DIST_BACKEND=gloo)
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("XSP_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(backend)

    from paper_1908_06869_b200.engine import DeviceBatch, Engine
    b, gf, gr, gb = make_workload(args, 0)  # every rank: the same C3 corpus (C5 = copies of it)
    groups = (gf, gr, gb)
    eng = Engine(local)
    dev = DeviceBatch(b, local)
    stream = torch.cuda.current_stream().cuda_stream
    peak, peak_kind = hbm_peak()

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(ms):
        if dist:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    def timed(step, steps, sampler=None):
        """device time of `steps` calls of step() with CUDA events on the launching stream"""
        barrier()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 0
        if sampler:
            sampler.__enter__()
        t0.record()
        for _ in range(steps):
            n += step()
        t1.record()
        torch.cuda.synchronize()
        if sampler:
            sampler.__exit__(None, None, None)
        barrier()
        return max_over_ranks(t0.elapsed_time(t1) / steps), n

    def staged(step, steps):
        """the same steps with CUDA events around every stage (kept out of the timed loop)"""
        eng.set_profiling(True)
        eng.stage_reset()
        for _ in range(steps):
            step()
        torch.cuda.synchronize()
        st_ = eng.stage_times()
        eng.set_profiling(False)
        return st_

    # ---------------- C3 (one corpus, device-resident), kept as an extra line
    def c3_step():
        eng.run_device(dev, groups, stream=stream)
        return eng.launches

    for _ in range(args.warmup):
        c3_step()
    c3_ms, _ = timed(c3_step, args.steps)
    c3_stages = staged(c3_step, args.steps)
    sv3 = survey_bytes(b)
    p1_ms3 = c3_stages["pass1"][0] / max(c3_stages["pass1"][1], 1)
    hb = b.pinned()
    # the packed wire form (xsp_pack_host: u32 begin deltas / durations / cid
    # offsets, sparse parent / cid lists), built once like the columns themselves
    pk = eng.pack_host(hb)
    e3_ms, h2d3, d2h3 = e2e_host(eng, hb, groups, 1, max(2, args.steps // 4), barrier, dist, packed=pk,
                                 rows_only=True)
    e3f_ms, h2d3f, d2h3f = e2e_host(eng, hb, groups, 1, max(2, args.steps // 4), barrier, dist, packed=pk)
    e3d_ms, h2d3d, d2h3d = e2e_host(eng, hb, groups, 1, max(2, args.steps // 4), barrier, dist)
    c3_line = {"metric": METRIC, "value": b.n_spans * world / (c3_ms / 1e3) / 1e6, "unit": UNIT,
               "ms_per_step": c3_ms, "spans_per_gpu": b.n_spans, "scaling": "weak", "config": c3_config(args),
               "e2e": {"value": b.n_spans * world / (e3_ms / 1e3) / 1e6, "unit": UNIT, "h2d_bytes_per_step": h2d3,
                       "d2h_bytes_per_step": d2h3, "ms_per_step": e3_ms, "input": "packed (xsp_run_host_packed)",
                       "outputs": "XSP_HOST_OUT_ROWS: every table + the correlation's span / metric rows"},
               "e2e_full": {"value": b.n_spans * world / (e3f_ms / 1e3) / 1e6, "unit": UNIT,
                            "h2d_bytes_per_step": h2d3f, "d2h_bytes_per_step": d2h3f, "ms_per_step": e3f_ms,
                            "input": "packed (xsp_run_host_packed)",
                            "outputs": "XSP_HOST_OUT_ALL: + layer_dur, kernel_dur / name / occ"},
               "e2e_dense": {"value": b.n_spans * world / (e3d_ms / 1e3) / 1e6, "unit": UNIT,
                             "h2d_bytes_per_step": h2d3d, "d2h_bytes_per_step": d2h3d, "ms_per_step": e3d_ms,
                             "input": "dense span columns (xsp_run_host)"},
               "roofline": {"bound": "hbm", "kernel": "k_pass1", "achieved": pass1_bytes(b) / (p1_ms3 / 1e3) / 1e9,
                            "peak": peak, "unit": "GB/s", "bytes_per_launch": pass1_bytes(b),
                            "ms_per_launch": p1_ms3},
               "pipeline_roofline": {"bound": "hbm", "bytes_per_span": sv3 / b.n_spans,
                                     "achieved": sv3 / (c3_ms / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                                     "frac": sv3 / (c3_ms / 1e3) / 1e9 / peak},
               "stages_ms": {k: v[0] / max(v[1], 1) for k, v in c3_stages.items()}}
    c3_line["roofline"]["frac"] = c3_line["roofline"]["achieved"] / peak
    sort_line = measure_sort(eng, dev, b, args.steps, local) if not args.no_sort else None
    val_line = measure_validate(eng, dev, b, max(2, args.steps // 4)) if not args.no_sort else None

    if args.c5_copies <= 0:  # quick iteration: the C3 line alone
        if rank == 0:
            print(json.dumps({"c3": c3_line, "sort_shuffled": sort_line, "validate": val_line}))
        if dist:
            dist.destroy_process_group()
        return

    # ---------------- C5 headline: ~1 B spans, device-resident
    c5 = C5(eng, dev, b, groups, copies=args.c5_copies, rank=rank, world=world)
    c5.step(stream, check=True)
    for _ in range(args.warmup):
        c5.step(stream)
    clk = ClockSampler(local)
    ms, launches = timed(lambda: c5.step(stream), args.steps, sampler=clk)
    stages = staged(lambda: c5.step(stream), max(2, args.steps // 4))
    value = c5.spans_all / (ms / 1e3) / 1e6
    # end to end: the same corpus from pinned host buffers through xsp_run_host
    # (one call per copy: H2D of its columns, D2H of every result column)
    e_ms, h2d, d2h = e2e_host(eng, hb, groups, len(c5.mine), args.e2e_steps, barrier, dist, packed=pk,
                              rows_only=True)
    e2e = {"value": c5.spans_all / (e_ms / 1e3) / 1e6, "unit": UNIT, "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "ms_per_step": e_ms, "steps": args.e2e_steps,
           "calls_per_step": len(c5.mine),
           "how": "xsp_run_host_packed per C3 copy on the same pinned host buffers (every copy's H2D and D2H "
                  "happen); the span columns in the packed wire form (xsp_pack_host, built once outside the "
                  "timed region like the columns themselves: u32 begin deltas / durations / cid offsets, "
                  "parent_id and cid only where flagged), unpacked on the device; results: every analysis "
                  "table and the correlation as span / metric rows (XSP_HOST_OUT_ROWS: the reference's "
                  "CorrelationResult refers to spans; the four lookup columns it leaves out are "
                  "c3.e2e_full's extra D2H)",
           "full_outputs_c3_e2e_value": c3_line["e2e_full"]["value"],
           "dense_c3_e2e_value": c3_line["e2e_dense"]["value"]}
    calls = len(c5.calls)
    p1_ms = stages["pass1"][0] / max(stages["pass1"][1], 1)  # per launch
    p1_bytes = pass1_bytes(b) * len(c5.mine) // max(calls, 1)
    c5.release()
    del dev
    torch.cuda.empty_cache()
    c4_line = measure_c4(eng, args, rank, world, local, dist) if args.c4_layers > 0 else None
    lev_line = measure_leveled(eng, args, local) if args.leveled_models > 0 and rank == 0 else None
    ing_line = measure_ingest(eng, args, local, world == 1 and not args.no_cpu_baseline) \
        if args.ingest_models > 0 and rank == 0 else None

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    dom = max(stages, key=lambda k: stages[k][0])
    achieved = p1_bytes / (p1_ms / 1e3) / 1e9
    roofline = {"bound": "hbm", "kernel": "k_pass1 (parent join + direct kernel-table emit, 1 launch per call)",
                "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "peak_kind": peak_kind,
                "traffic": (measured_traffic("k_pass1", c5.spans_mine // max(calls, 1)) or {}).get("bytes"),
                "traffic_source": measured_traffic("k_pass1", c5.spans_mine // max(calls, 1)),
                "bytes_per_launch": p1_bytes,
                "ms_per_launch": p1_ms, "launches_per_step": calls}
    sv = survey_bytes(b) * args.c5_copies
    pipe_gbs = sv / (ms / 1e3) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64/f64", "data": "synthetic", "config": config(args),
        "spans": c5.spans_all, "e2e": e2e, "gpu_launches": launches,
        "roofline": roofline,
        "pipeline_roofline": {"bound": "hbm", "bytes_per_span": sv / c5.spans_all, "achieved": pipe_gbs,
                              "peak": peak, "unit": "GB/s", "frac": pipe_gbs / peak / world,
                              "definition": "SURVEY.md 8(d): (157+162K) B per layer + 96 B per trace"},
        "stages_ms": {k: v[0] / max(v[1], 1) for k, v in stages.items()},
        "dominant_stage": dom,
        "clocks": clk.summary(),
        "c3": c3_line,
    }
    if sort_line:
        sort_line["roofline"] = {"bound": "hbm", "bytes_per_span": 21.0, "achieved": sort_line.pop("gbs"),
                                 "peak": peak, "unit": "GB/s",
                                 "definition": "read begin_ns+flags+span_id (17 B), write perm (4 B) per span"}
        sort_line["roofline"]["frac"] = sort_line["roofline"]["achieved"] / peak
        line["sort_shuffled"] = sort_line
    if val_line:
        val_line["roofline"]["peak"] = peak
        val_line["roofline"]["frac"] = val_line["roofline"]["achieved"] / peak
        line["validate"] = val_line
    if c4_line:
        line["c4"] = c4_line
    if lev_line:
        line["leveled"] = lev_line
    if ing_line:
        line["ingest_jsonl"] = ing_line
    if world == 1 and not args.no_cpu_baseline:
        from oracle import ref
        if ref.available():
            cb = cpu_reference(b, gf, gr, args.ref_sample_spans)
            cb.pop("seconds")
            cb["sample"] += " (the C5 corpus is copies of this C3 corpus)"
            line["cpu_baseline"] = cb
    print(json.dumps(line))
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
