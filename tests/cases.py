"""Edge-case traces from the reference's correlator tests (test_correlator.cpp)
and acceptance gate (acceptance_main.cpp:237-313), as span lists."""
from builders import API, EXEC, KERNEL, LAUNCH, LAYER, MODEL, SYNC, span

M = (1000, 64, 32, 0.75)


def nesting():  # test_correlator.cpp:107-131
    return [span(1, MODEL, 0, 100), span(2, LAYER, 10, 40), span(3, LAYER, 50, 90),
            span(4, KERNEL, 10, 25), span(5, KERNEL, 30, 40), span(6, KERNEL, 60, 60)]


def layer_attrs():  # :133-143
    return [span(1, MODEL, 0, 100), span(2, LAYER, 10, 40, layer_type="Conv2D", alloc=4096)]


def explicit_beats_containment():  # :145-158
    return [span(1, MODEL, 0, 100), span(2, LAYER, 10, 40), span(3, LAYER, 50, 90),
            span(4, KERNEL, 15, 20, parent=3)]


def overlapping_layers():  # :160-177
    return [span(1, MODEL, 0, 100), span(2, LAYER, 10, 60), span(3, LAYER, 20, 80),
            span(4, KERNEL, 30, 40), span(5, KERNEL, 65, 70)]


def orphans():  # :179-201
    return [span(1, MODEL, 10, 100), span(2, LAYER, 2, 8), span(3, LAYER, 20, 60),
            span(4, KERNEL, 3, 6), span(5, KERNEL, 70, 80), span(6, KERNEL, 55, 58, parent=99),
            span(7, LAYER, 30, 40, kind=LAUNCH)]


def fusion():  # :222-256
    return [span(1, MODEL, 0, 100), span(2, LAYER, 10, 60),
            span(3, KERNEL, 12, 14, kind=LAUNCH, cid=21), span(4, KERNEL, 16, 18, kind=LAUNCH, cid=22),
            span(5, KERNEL, 30, 44, kind=EXEC, cid=22, name="sgemm", metrics=M),
            span(6, KERNEL, 44, 50, kind=EXEC, cid=21, name="relu")]


def unmatched_async():  # :258-277
    return [span(1, MODEL, 0, 100), span(2, LAYER, 10, 60),
            span(3, KERNEL, 12, 14, kind=LAUNCH, cid=5), span(4, KERNEL, 20, 22, kind=LAUNCH),
            span(5, KERNEL, 30, 40, kind=EXEC, cid=8), span(6, KERNEL, 41, 47, kind=EXEC)]


def dup_launch_cid():  # :279-290
    return [span(1, MODEL, 0, 100), span(2, LAYER, 10, 60),
            span(3, KERNEL, 12, 14, kind=LAUNCH, cid=5), span(4, KERNEL, 20, 22, kind=LAUNCH, cid=5)]


def dup_exec_cid():  # :291-297
    return [span(1, MODEL, 0, 100), span(2, LAYER, 10, 60),
            span(3, KERNEL, 30, 34, kind=EXEC, cid=5), span(4, KERNEL, 40, 42, kind=EXEC, cid=5)]


def no_model():  # :206-209
    return [span(2, LAYER, 0, 5)]


def two_models():  # :210-214
    return [span(1, MODEL, 0, 100), span(2, MODEL, 0, 90)]


def skip_level():  # :203-205 (run with levels {M, G})
    return [span(1, MODEL, 0, 100), span(2, KERNEL, 10, 20)]


def mixed_orphan_order():
    """Every orphan category in one trace, to pin the output order
    (correlator.cpp:168-363): layer pass, kernel pass, exec w/o cid, launch
    fusion in tree order, leftover execs by span_id; plus a layer-level exec
    orphaned twice (non-sync kind + without matching launch)."""
    return [
        span(1, MODEL, 100, 1000),
        span(40, LAYER, 50, 60),                       # outside the model interval
        span(41, LAYER, 200, 300, parent=77),           # explicit parent not the model
        span(2, LAYER, 110, 190),
        span(3, LAYER, 400, 500),
        span(42, LAYER, 150, 160, kind=EXEC, cid=900),  # layer-level exec: orphan twice
        span(50, KERNEL, 120, 130, kind=LAUNCH, cid=10),
        span(51, KERNEL, 410, 420, kind=LAUNCH),        # launch without cid
        span(52, KERNEL, 125, 126, kind=LAUNCH, cid=11),  # no exec
        span(53, KERNEL, 600, 610, kind=LAUNCH, cid=12),  # contained in no layer
        span(54, KERNEL, 411, 412, parent=2),           # sync kernel, explicit parent layer 2
        span(55, API, 430, 440, kind=LAUNCH, cid=13),
        span(60, KERNEL, 700, 710, kind=EXEC, cid=10, metrics=M),
        span(61, KERNEL, 705, 715, kind=EXEC, cid=13),
        span(62, KERNEL, 720, 721, kind=EXEC),          # exec without cid
        span(64, KERNEL, 722, 730, kind=EXEC, cid=99),  # leftover
        span(63, KERNEL, 731, 740, kind=EXEC, cid=98),  # leftover (sorted by span_id: 63 < 64)
        span(65, KERNEL, 741, 742, kind=EXEC, cid=12),  # consumed by the orphaned launch 53
        span(56, KERNEL, 450, 460, parent=41),          # explicit parent is an orphaned layer
    ]


U64_MAX = (1 << 64) - 1


def max_end():
    """Intervals ending at 2^64-1: a kernel ending there is contained in a layer
    ending there (closed intervals, span.hpp:97-100), and in no layer that ends
    one nanosecond earlier (advisor finding on the device's end+1 encoding)."""
    return [span(1, MODEL, 0, U64_MAX), span(2, LAYER, 10, U64_MAX), span(3, LAYER, 20, 30),
            span(4, KERNEL, 25, U64_MAX), span(5, KERNEL, 40, U64_MAX),
            span(6, KERNEL, 26, 28)]


def max_end_orphan():
    return [span(1, MODEL, 0, U64_MAX), span(2, LAYER, 10, U64_MAX - 1), span(3, KERNEL, 25, U64_MAX),
            span(4, KERNEL, 30, U64_MAX - 1)]


def model_span_id_shared():
    """Two model spans with the same span_id: the reference compares span ids
    (correlator.cpp:146-150), so this is not 'more than one model span'."""
    return [span(1, MODEL, 0, 100), span(1, MODEL, 0, 90), span(2, LAYER, 10, 40), span(3, KERNEL, 12, 20)]
