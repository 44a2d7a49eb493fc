"""GPU tests of the ABI's stream-ordering contract (include/sppo.h; SURVEY §8(b)
"Ordering contract"): every launch reads TMA descriptors uploaded on its own
stream, torch-side work of an engine step runs on the step's stream, and the
end-to-end step's input copies wait for the previous step on that stream.
Each case is built so that the unordered version of the code computes wrong
numbers, then compared with the fp64 oracle (bf16 tolerances, reading L7)."""

import numpy as np
import pytest
import torch

import oracle
from synth import make_inputs

pytestmark = pytest.mark.gpu

O_TOL = dict(atol=2e-2, rtol=1e-2)
G_TOL = dict(atol=5e-2, rtol=5e-2)
SPIN = 200_000_000  # torch.cuda._sleep cycles (~0.1 s): holds a stream while the other one runs


def _ref(x):
    xn = {k: v.double().numpy() for k, v in x.items()}
    return oracle.causal_attention_dense_bwd(xn["q"], xn["k"], xn["v"], xn["do"])


def _check(out, ref, keys=("o", "dq", "dk", "dv")):
    for k in keys:
        tol = O_TOL if k == "o" else G_TOL
        np.testing.assert_allclose(out[k].double().cpu().numpy(), ref[k], **tol, err_msg=k)


def test_side_stream_launch_before_main_stream_upload():
    """Chunk 1's forward is launched on a side stream while the main stream is held
    by a spin kernel in front of chunk 0's forward.  Both read K_0 / V_0; with a
    descriptor cache shared across streams, chunk 1 would read K_0's tensor map
    before the main stream had uploaded it.  Fresh ctx: no descriptor is cached."""
    from paper_2503_10377_b200 import sppo
    S, h, N = 1024, 2, 2
    x = make_inputs(S, range(h), 128, seed=71, dtype=torch.bfloat16)
    dev = {k: v.cuda() for k, v in x.items()}
    ctx = sppo.Context(0)
    L = sppo.Layout(h, 128, sppo.partition_equal(S, N))
    o = torch.empty_like(dev["q"])
    lse = torch.empty(S * h, dtype=torch.float32, device="cuda")
    main, side = torch.cuda.Stream(), torch.cuda.Stream()
    c = L.offsets
    rows = lambda t, i: t[c[i]:c[i + 1]]  # noqa: E731
    torch.cuda.synchronize()
    with torch.cuda.stream(main):
        torch.cuda._sleep(SPIN)
        ctx.attn_fwd(L, 0, rows(dev["q"], 0), [0], [rows(dev["k"], 0)], [rows(dev["v"], 0)],
                     flags=sppo.SPPO_FIRST | sppo.SPPO_LAST, o=rows(o, 0), lse=lse[c[0] * h:c[1] * h], stream=main)
    ctx.attn_fwd(L, 1, rows(dev["q"], 1), [0, 1], [rows(dev["k"], j) for j in (0, 1)],
                 [rows(dev["v"], j) for j in (0, 1)], flags=sppo.SPPO_FIRST | sppo.SPPO_LAST,
                 o=rows(o, 1), lse=lse[c[1] * h:c[2] * h], stream=side)
    torch.cuda.synchronize()
    ctx.sync()
    ref = _ref(x)
    np.testing.assert_allclose(o.double().cpu().numpy(), ref["o"], **O_TOL)
    ctx.close()


@pytest.mark.parametrize("kind", ["step", "offload", "kv_stream", "kv_grouped"])
def test_engine_step_on_side_stream(kind):
    """Two consecutive steps on a side stream while torch's current stream is held
    by a spin kernel each time: the accumulator zeroing (and poison fills) must run
    on the step's stream, or the second step accumulates onto the first step's
    dK / dV sums."""
    from paper_2503_10377_b200 import engine, sppo
    S, h, N = 2048, 2, 8
    x = make_inputs(S, range(h), 128, seed=72, dtype=torch.bfloat16)
    dev = {k: v.cuda() for k, v in x.items()}
    ctx = sppo.Context(0)
    L = sppo.Layout(h, 128, sppo.partition_equal(S, N))
    eng = engine.ChunkedAttention(ctx, L)
    side = torch.cuda.Stream()
    ref = _ref(x)
    for _ in range(2):
        torch.cuda.synchronize()
        # inputs are produced (and complete) before the spin: only the step's own
        # torch-side work may land on the held stream
        q, k, v = dev["q"].clone(), dev["k"].clone(), dev["v"].clone()
        torch.cuda.synchronize()
        torch.cuda._sleep(SPIN)  # on the current (default) stream
        if kind == "step":
            out = eng.step(dev["q"], k, v, dev["do"], stream=side)
        elif kind == "offload":
            eng.step_offload(q, k, v, dev["do"], [0.5] * (N - 1) + [0.0], stream=side, poison=True)
        elif kind == "kv_stream":
            eng.step_kv_stream(dev["q"], k, v, dev["do"], hot=2, window=2, stream=side, poison=True)
        else:
            eng.step_kv_stream_grouped(dev["q"], k, v, dev["do"], hot=1, window=2, group=2, stream=side,
                                       poison=True)
        torch.cuda.synchronize()
        ctx.sync()
        out = dict(o=eng.o, dq=eng.dq, dk=eng.dk, dv=eng.dv)
        _check(out, ref)
    eng.free_host()
    ctx.close()


def test_host_io_steps_back_to_back():
    """Two end-to-end steps (pinned host in -> device staging -> host out) with
    DIFFERENT inputs and no host synchronisation between them: the second step's
    H2D copies into the shared device staging buffers must wait for the first
    step's backward, or the first step reads the second step's inputs."""
    from paper_2503_10377_b200 import engine, sppo
    S, h, N = 2048, 2, 4
    xa = make_inputs(S, range(h), 128, seed=73, dtype=torch.bfloat16)
    xb = make_inputs(S, range(h), 128, seed=74, dtype=torch.bfloat16)
    ctx = sppo.Context(0)
    L = sppo.Layout(h, 128, sppo.partition_equal(S, N))
    eng = engine.ChunkedAttention(ctx, L)
    nb = S * h * 128 * 2
    stream = torch.cuda.current_stream()
    hosts = []
    for x in (xa, xb):
        hin = {t: ctx.host_alloc(nb) for t in ("q", "k", "v", "do")}
        hout = {t: ctx.host_alloc(nb) for t in ("o", "dq", "dk", "dv")}
        for t in hin:
            ctx.kv_offload(0, x[t].cuda(), hin[t], nb, 1.0, producer=stream)
        hosts.append((hin, hout))
    ctx.sync()
    staging = {t: torch.empty((S, h, 128), dtype=torch.bfloat16, device="cuda") for t in ("q", "k", "v", "do")}
    lasts = []
    for hin, hout in hosts:  # back to back, no synchronisation
        _, _, last = eng.step_host_io(hin, hout, staging, stream)
        lasts.append(last)
    for ev in lasts:
        stream.wait_event(ev)
    torch.cuda.synchronize()
    ctx.sync()
    for x, (hin, hout) in zip((xa, xb), hosts):
        out = {}
        for t in ("o", "dq", "dk", "dv"):
            d = torch.empty((S, h, 128), dtype=torch.bfloat16, device="cuda")
            ctx.kv_prefetch(0, hout[t], d, nb, consumer=stream)
            out[t] = d
        torch.cuda.synchronize()
        _check(out, _ref(x))
        for p in list(hin.values()) + list(hout.values()):
            ctx.host_free(p)
    ctx.close()


def test_many_distinct_buffers_no_device_sync():
    """More launches than the descriptor ring has blocks, each with fresh buffers
    (distinct tensor maps): results stay exact and the ring never needs a
    device-wide synchronisation (blocks are recycled behind their own events)."""
    from paper_2503_10377_b200 import sppo
    S, h = 256, 1
    x = make_inputs(S, range(h), 128, seed=75, dtype=torch.bfloat16)
    ref = _ref(x)
    ctx = sppo.Context(0)
    L = sppo.Layout(h, 128, [0, S])
    outs = []
    for it in range(300):
        q, k, v = (x[t].cuda().clone() for t in ("q", "k", "v"))  # new pointers every launch
        o = torch.empty_like(q)
        lse = torch.empty(S * h, dtype=torch.float32, device="cuda")
        ctx.attn_fwd(L, 0, q, [0], [k], [v], flags=sppo.SPPO_FIRST | sppo.SPPO_LAST, o=o, lse=lse)
        outs.append((q, k, v, o))
    torch.cuda.synchronize()
    ctx.sync()
    first = outs[0][3]
    np.testing.assert_allclose(first.double().cpu().numpy(), ref["o"], **O_TOL)
    for *_, o in outs[1:]:
        assert torch.equal(o, first)  # forward bitwise deterministic (reading L12)
    ctx.close()


def test_descriptor_table_recycles_mid_step():
    """256 chunks of 128 tokens, every window one launch: one step needs ~66K
    distinct tensor maps (each chunk's K / V view in every later window), four
    times the 16384-slot descriptor table, so the table is recycled several times
    while earlier launches are still in flight (include/sppo.h "Descriptor
    table").  The result must still equal the oracle."""
    from paper_2503_10377_b200 import engine, sppo
    S, h, N = 256 * 128, 1, 256
    x = make_inputs(S, range(h), 128, seed=75, dtype=torch.bfloat16)
    dev = {k: v.cuda() for k, v in x.items()}
    ctx = sppo.Context(0)
    eng = engine.ChunkedAttention(ctx, sppo.Layout(h, 128, sppo.partition_equal(S, N)))
    for _ in range(2):  # the second step starts from a table the first one left full
        out = eng.step(dev["q"], dev["k"], dev["v"], dev["do"])
    torch.cuda.synchronize()
    ctx.sync()
    rows = [0, 127, 128, 4095, 16383, 16384, S - 129, S - 1]
    xn = {k: v.double().numpy() for k, v in x.items()}
    ref = oracle.sampled_rows(xn["q"], xn["k"], xn["v"], rows, do=xn["do"])
    np.testing.assert_allclose(out["o"][rows].double().cpu().numpy(), ref["o"], **O_TOL)
    np.testing.assert_allclose(out["dq"][rows].double().cpu().numpy(), ref["dq"], **G_TOL)
    keys = sorted(set(range(S - 300, S, 37)) | {S - 1})
    kg = oracle.sampled_key_grads(xn["q"], xn["k"], xn["v"], xn["do"], keys, row_block=128)
    np.testing.assert_allclose(out["dk"][keys].double().cpu().numpy(), kg["dk"], **G_TOL)
    np.testing.assert_allclose(out["dv"][keys].double().cpu().numpy(), kg["dv"], **G_TOL)
    ctx.close()
