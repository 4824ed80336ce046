"""EqSpec round parity: K1 -> K3 -> K2 through the C ABI vs the oracle on the same bytes,
over many rounds (tokens, masks, positions, output buffers, every valid KV entry, moved
bytes), plus K2 alone under adversarial shift patterns and in gather/scatter mode."""
import numpy as np
import pytest
import torch

from oracle import align as OA
from oracle import verify as OV
from paper_2510_22876_b200 import _abi
from paper_2510_22876_b200.eqspec import EqSpecBatch, pack_host_inputs
from synth import workloads as W
from tests.gpu_helpers import bits_to_torch, padded_logits, torch_to_bits

pytestmark = pytest.mark.gpu


def _run_rounds(cuda, shape: W.Shape, B, rounds, pattern, seed=0, max_new=0, eos_id=-1,
                zero_pads=False, full_check=True, anchor_slack=0, kv_mode="inplace", drive="python"):
    """drive: "python" (the three calls from eqspec.py), "native" (specdec_eqspec_round)
    or "host" (specdec_eqspec_round_host from pinned host logits / drafts)."""
    k, V = shape.k, shape.V
    cap = W.derive_cap(shape.with_(B=B), rounds)
    lengths = W.gen_lengths(shape, seed, B)
    tokens = W.left_padded_tokens(lengths, cap, seed, V)
    kvshape = (shape.n_planes, B, shape.H, cap, shape.D)
    kv_bits = W.gen_kv_bits_np(seed, int(np.prod(kvshape))).reshape(kvshape)
    bt = EqSpecBatch(B, k, cap, shape.layers, shape.H, shape.D, shape.kv_dtype, cuda,
                     max_new=max_new, eos_id=eos_id, pad_id=W.PAD_ID, anchor_slack=anchor_slack,
                     kv_mode=kv_mode)
    bt.load(tokens, lengths, bits_to_torch(kv_bits, shape.kv_dtype, cuda))
    bt.native_round = drive in ("native", "graph")
    bt.fork = drive == "fork"                 # K3 on a side stream under K2 (Python path)
    host = drive in ("host", "host_packed")
    graph_io = None
    h_emit = torch.zeros(B, dtype=torch.int32).pin_memory() if host else None
    base_o = anchor_slack
    bases = []
    # oracle state
    tok_o, kv_o = tokens.copy(), kv_bits.copy()
    n_o = lengths.astype(np.int32)
    L = int(n_o.max())
    pad_o = (L - n_o).astype(np.int32)
    act_o = np.ones(B, np.uint8)
    gen_o = np.zeros(B, np.int64)
    out_o = [[] for _ in range(B)]
    moved_expect = 0
    for r in range(rounds):
        if not act_o.any():
            break
        # synthetic verify forward: k+1 new KV entries at [L-1, L+k) on both sides
        fwd = W.gen_kv_bits_np(seed + 1000 + r, shape.n_planes * B * shape.H * (k + 1) * shape.D)
        fwd = fwd.reshape(shape.n_planes, B, shape.H, k + 1, shape.D)
        kv_o[:, :, :, L - 1:L + k, :] = fwd
        bt.kv_logical()[:, :, :, L - 1:L + k, :] = bits_to_torch(fwd, shape.kv_dtype, cuda)
        rt = W.gen_round_truth(seed, r, B, k, V, pattern)
        bits = W.gen_logits_np(seed, r, B, k, V, shape.logit_dtype)
        lg = padded_logits(bits, shape.logit_dtype, cuda, extra=16)
        draft = torch.from_numpy(rt.draft).to(cuda)
        if drive == "host":           # separate pinned buffers: two H2D copies
            bt.step_host(lg.cpu().pin_memory(), torch.from_numpy(rt.draft).pin_memory(), h_emit,
                         V=V, zero_pads=zero_pads)
        elif drive == "host_packed":  # logits + drafts in one pinned buffer: one copy
            hl, hd = pack_host_inputs(lg.cpu(), torch.from_numpy(rt.draft))
            bt.step_host(hl, hd, h_emit, V=V, zero_pads=zero_pads)
        elif drive == "graph":        # the captured round (PDL edges inside the graph) replayed
            if graph_io is None:
                graph_io = (torch.empty_like(lg), torch.empty_like(draft))
                bt.zero_pads = zero_pads
                bt.capture([graph_io], V=V)
            graph_io[0].copy_(lg)
            graph_io[1].copy_(draft)
            bt.replay(0)
        else:
            bt.step(lg, draft, V=V, zero_pads=zero_pads)
        # oracle
        budget = None if not max_new else (max_new - gen_o)
        v = OV.batch_verify(bits, shape.logit_dtype, rt.draft, n_o, pad_o, act_o, eos_id, budget, W.PAD_ID)
        tok_n, mask_n, pos_n = OA.repad_tokens(tok_o, cap, k, pad_o, L, v, W.PAD_ID)
        kv_n, defined = OA.realign_kv(kv_o, pad_o, v["pad_new"], v["kept"])
        if anchor_slack:
            b2, col_old, col_new = OA.anchor_plan(pad_o, v["pad_new"], v["kept"], v["finished"],
                                                  v["accept"], L, v["L_new"], base_o,
                                                  cap + anchor_slack, k)
            moved_expect += OA.moved_bytes(col_old, col_new, v["kept"], shape.bpt)
            assert bt.base() == b2, r
            assert np.array_equal(bt.phys_old.cpu().numpy(), col_old)
            assert np.array_equal(bt.phys_new.cpu().numpy(), col_new)
            base_o = b2
            bases.append(b2)
        elif kv_mode == "pingpong":   # out of place: every kept row is copied, Delta = 0 too
            moved_expect += 2 * int(np.asarray(v["kept"], np.int64).sum()) * shape.bpt
        else:
            moved_expect += OA.moved_bytes(pad_o, v["pad_new"], v["kept"], shape.bpt)
        zero_regions = OA.zero_pad_region(pad_o, v["pad_new"], v["kept"])
        for i in range(B):
            out_o[i] += v["E"][i]
        gen_o += v["emit"]
        torch.cuda.synchronize()
        # ---- compare
        for key, g in (("accept", bt.accept), ("bonus", bt.bonus), ("emit", bt.emit),
                       ("finished", bt.finished), ("kept", bt.kept)):
            assert np.array_equal(g.cpu().numpy(), v[key]), (r, key)
        if h_emit is not None:
            assert np.array_equal(h_emit.numpy(), v["emit"]), r     # the D2H of the host call
        Ln = v["L_new"]
        assert int(bt.plan_L.item()) == Ln
        assert np.array_equal(bt.pad_cur.cpu().numpy(), v["pad_new"]), r
        assert np.array_equal(bt.n_cur.cpu().numpy(), v["n_new"]), r
        assert int(bt.status.item()) == 0
        if Ln > 0:
            assert np.array_equal(bt.tokens[:, :Ln].cpu().numpy(), tok_n[:, :Ln]), r
            assert np.array_equal(bt.mask[:, :Ln + k].cpu().numpy(), mask_n), r
            assert np.array_equal(bt.pos[:, :Ln + k].cpu().numpy(), pos_n), r
        if full_check:
            kv_g = torch_to_bits(bt.kv_logical())
            for i in range(B):
                cols = np.flatnonzero(defined[i])
                if len(cols):
                    assert np.array_equal(kv_g[:, i, :, cols], kv_n[:, i, :, cols]), (r, i)
            if zero_pads:
                for i, lo, hi in zero_regions:
                    assert not kv_g[:, i, :, lo:hi].any(), (r, i)
            kv_o = kv_n
        if max_new:
            gen_g = bt.gen.cpu().numpy()
            assert np.array_equal(gen_g, gen_o)
            ob = bt.out_buf.cpu().numpy()
            for i in range(B):
                assert list(ob[i, :gen_g[i]]) == out_o[i]
        # advance oracle state
        tok_o, n_o, pad_o, L = tok_n, v["n_new"], v["pad_new"], Ln
        act_o = (v["finished"] == 0).astype(np.uint8)
    assert int(bt.moved.item()) == moved_expect
    return dict(rounds=r + 1, bases=bases, moved=moved_expect)


SMALL = W.Shape("small", 3001, 2, 2, 64, "bf16", "bf16", 8, 5, 160, 40, 160)
SMALL16 = W.Shape("small16", 2003, 3, 1, 128, "fp16", "fp16", 6, 4, 300, 100, 300)


@pytest.mark.parametrize("pattern", ["alpha", "alternating", "one_zero", "all_k", "all_0"])
def test_rounds_small(cuda, pattern):
    _run_rounds(cuda, SMALL, 8, 10, pattern)


@pytest.mark.parametrize("pattern,slack", [("alpha", 64), ("alternating", 64), ("alpha", 3)])
def test_rounds_anchored_origin(cuda, pattern, slack):
    """f3: K1 moves the physical origin exactly as oracle.align.anchor_plan; the logical
    KV equals Alg. 2's realign and fewer bytes move than with the fixed origin."""
    anc = _run_rounds(cuda, SMALL, 8, 12, pattern, seed=3, anchor_slack=slack)
    std = _run_rounds(cuda, SMALL, 8, 12, pattern, seed=3)          # same workload, fixed origin
    assert anc["moved"] <= std["moved"]
    if slack >= 64:
        assert len(set(anc["bases"])) > 1 and anc["moved"] < std["moved"]


def test_rounds_anchored_with_finish(cuda):
    _run_rounds(cuda, SMALL16, 6, 14, "alpha", seed=2, max_new=33, anchor_slack=32)


def test_rounds_toy_with_budget_and_finish(cuda):
    n = _run_rounds(cuda, W.SHAPES["toy"], 2, 40, "alpha", max_new=20)["rounds"]
    assert n < 40  # every row finished before the round cap


@pytest.mark.parametrize("B", [1, 3, 8])
def test_rounds_budget_staggered_finish(cuda, B):
    # rows finish at different rounds -> the longest row can leave and L' shrinks
    _run_rounds(cuda, SMALL16, B, 14, "alpha", seed=B, max_new=33)


@pytest.mark.parametrize("pattern", ["alpha", "alternating"])
def test_rounds_pingpong(cuda, pattern):
    """kv_mode="pingpong": K2 out of place between two KV buffers every round."""
    _run_rounds(cuda, SMALL, 8, 10, pattern, kv_mode="pingpong")
    _run_rounds(cuda, SMALL16, 3, 14, pattern, seed=4, max_new=33, kv_mode="pingpong")
    _run_rounds(cuda, SMALL, 1, 5, pattern, kv_mode="pingpong")   # B=1 copies too


def test_rounds_zero_pads(cuda):
    _run_rounds(cuda, SMALL, 8, 6, "alternating", zero_pads=True, seed=5)


# ----------------------------------------------------------------------------- K2 alone
def _realign_case(cuda, pad_old, pad_new, kept, D=128, H=3, planes=2, cap=None, dtype="bf16", zero=False,
                  seg=False, bound=0, dyn=False):
    B = len(kept)
    cap = cap or int(max(np.max(pad_old), np.max(pad_new)) + np.max(kept) + 4)
    shp = (planes, B, H, cap, D)
    bits = W.gen_kv_bits_np(7, int(np.prod(shp))).reshape(shp)
    kv = bits_to_torch(bits, dtype, cuda)
    t32 = lambda x: torch.as_tensor(np.asarray(x, np.int32), device=cuda)
    moved = torch.zeros(1, dtype=torch.int64, device=cuda)
    st = torch.zeros(1, dtype=torch.int32, device=cuda)
    s = kv.stride()
    ws = None
    flags = _abi.ZERO_PADS if zero else 0
    if seg:   # SEGMENTED: slabs cut in ~128 KB segments with saved boundary rows
        ws = torch.full((_abi.specdec_realign_workspace_size(kv.dtype, planes, B, H, D, cap),), 0xAB,
                        dtype=torch.uint8, device=cuda)          # slot contents are don't-care
        flags |= _abi.SEGMENTED
    if dyn:   # DYNAMIC (+ FORCE: tickets even below 8 units per CTA) from the zeroed header
        if ws is None:
            ws = torch.zeros(128, dtype=torch.uint8, device=cuda)
        ws[:128] = 0
        flags |= _abi.DYNAMIC | _abi.DYNAMIC_FORCE
    _abi.specdec_realign_kv(kv, kv, t32(kept), n_planes=planes, n_rows=B, H=H, D=D,
                            src_strides=s[:3], dst_strides=s[:3], cap_src=cap, cap_dst=cap, ws=ws,
                            src_col=t32(pad_old), dst_col=t32(pad_new),
                            flags=flags, moved_bytes=moved, status=st,
                            count_bound=bound)
    torch.cuda.synchronize()
    rb = D * (4 if dtype == "fp32" else 2)
    small = bound > 0 and bound * rb <= 4096          # warp-per-slab kernel: no schedule
    if dyn:
        hdr = ws[:16].view(torch.int32).cpu().numpy()
        assert hdr[0] == 0 and hdr[1] == 0, "the schedule counters are left zero"
        if not small:
            # the ticket path ran: one completed dynamic launch, >= one ticket per moving slab
            moving = sum(1 for i in range(B) if kept[i] > 0 and pad_old[i] != pad_new[i]
                         and max(pad_old[i], pad_new[i]) + kept[i] <= cap and (bound == 0 or kept[i] <= bound))
            assert hdr[2] == 1, hdr
            assert hdr[3] >= planes * H * moving, (hdr, moving)
    g = torch_to_bits(kv)
    o, defined = OA.realign_kv(bits, pad_old, pad_new, kept)
    for i in range(B):
        cols = np.flatnonzero(defined[i])
        assert np.array_equal(g[:, i, :, cols], o[:, i, :, cols]), i
        if pad_old[i] == pad_new[i]:
            assert np.array_equal(g[:, i], bits[:, i])            # untouched
    if zero:
        for i, lo, hi in OA.zero_pad_region(pad_old, pad_new, kept):
            assert not g[:, i, :, lo:hi].any()
    elem = 2 if dtype != "fp32" else 4
    assert int(moved.item()) == OA.moved_bytes(pad_old, pad_new, kept, planes * H * D * elem)
    assert int(st.item()) == 0


@pytest.mark.parametrize("D,dtype", [(128, "bf16"), (8, "bf16"), (64, "fp16"), (4, "fp32")])
@pytest.mark.parametrize("dyn", [False, True])
def test_realign_adversarial_shifts(cuda, D, dtype, dyn):
    k = 5
    big = 700  # 700 rows x 256 B = 175 KB -> many 16 KB chunks
    cases = [
        ([0] * 4, [k] * 4, [big, 300, 65, 1]),                 # all +k
        ([k] * 4, [0] * 4, [big, 300, 65, 1]),                 # all -k
        ([0, k, 0, k], [k, 0, k, 0], [big, big, 64, 63]),      # alternating
        ([900, 3, 0, 7], [0, 3, 500, 6], [big, 40, big, 129]),  # large shifts, one Delta=0
        ([1, 2, 3, 4], [2, 3, 4, 5], [1, 2, 3, 4]),            # tiny slabs
    ]
    for po, pn, kp in cases:
        _realign_case(cuda, po, pn, kp, D=D, dtype=dtype, dyn=dyn)


@pytest.mark.parametrize("D,dtype", [(128, "bf16"), (64, "fp16"), (32, "fp32")])
def test_realign_segmented_in_place(cuda, D, dtype):
    """Slabs of many 128 KB segments streamed by independent CTAs: boundary rows saved to
    the workspace first; shifts of both signs, up to a full slot (4 KB of rows), wider
    shifts (unsegmented fallback), Delta = 0, tiny and ragged slabs."""
    rb = D * (4 if dtype == "fp32" else 2)
    smax = 4096 // rb                       # widest shift a slot holds
    long = (5 * 131072) // rb + 37          # > 5 segments, ragged last one
    cases = [
        ([0] * 4, [5] * 4, [long, long - 3, 513, 2]),
        ([7] * 4, [0] * 4, [long, 1000, long // 2, 1]),
        ([0, smax, 0, smax], [smax, 0, smax, 0], [long, long, long, long]),
        ([0, 3, 2 * smax + 3, 9], [smax + 1, 3, 0, 2], [long, 100, long, 7]),    # wide -> unsegmented
        ([1, 0, 4, 2], [0, 1, 4, 1], [long - 1, long, long, 3]),
    ]
    for po, pn, kp in cases:
        _realign_case(cuda, po, pn, kp, D=D, H=2, dtype=dtype, seg=True)
        _realign_case(cuda, po, pn, kp, D=D, H=2, dtype=dtype, seg=True, dyn=True)
    _realign_case(cuda, [0, 4, 0], [3, 4, 0], [long, 50, long], D=D, H=2, dtype=dtype, seg=True, zero=True)


def test_realign_zero_pads_and_skips(cuda):
    _realign_case(cuda, [0, 4, 2, 0], [3, 4, 0, 9], [50, 0, 70, 1000], zero=True)
    _realign_case(cuda, [0, 4, 2, 0], [3, 4, 0, 9], [50, 0, 70, 1000], zero=True, dyn=True)
    _realign_case(cuda, [3, 3], [3, 3], [10, 10], dyn=True)      # nothing moves: every CTA exits early


@pytest.mark.parametrize("D,dtype", [(128, "bf16"), (8, "fp16"), (16, "fp32")])
def test_realign_small_slabs_in_place(cuda, D, dtype):
    """count_bound * row bytes <= 4 KB selects the register-staged warp-per-slab kernel:
    in-place shifts of both signs wider and narrower than the slab, Delta = 0, empty rows,
    ZERO_PADS, many rows (more slabs than one CTA's warps)."""
    rb = D * (4 if dtype == "fp32" else 2)
    bmax = 4096 // rb
    cases = [
        ([0] * 4, [5] * 4, [bmax, 6, 1, 0]),
        ([9] * 4, [0] * 4, [bmax, bmax - 1, 3, 2]),
        ([0, 7, 3, 0], [40, 7, 0, 1], [bmax, 5, 6, bmax]),
    ]
    for po, pn, kp in cases:
        _realign_case(cuda, po, pn, kp, D=D, dtype=dtype, bound=bmax)
        _realign_case(cuda, po, pn, kp, D=D, dtype=dtype, bound=bmax, zero=True)
    rng = np.random.default_rng(5)
    B = 40
    po, pn = rng.integers(0, 30, B), rng.integers(0, 30, B)
    _realign_case(cuda, po, pn, rng.integers(0, 7, B), D=D, dtype=dtype, H=5, planes=3, bound=6)


def test_realign_count_bound_violation(cuda):
    """A row above count_bound is skipped and reported (SPECDEC_ST_BOUND), small and ring
    kernels alike; the other rows move."""
    for bound in (4, 64):       # 4 * 256 B -> small kernel; 64 * 256 B -> TMA ring kernel
        planes, B, H, cap, D = 2, 3, 2, 200, 128
        shp = (planes, B, H, cap, D)
        bits = W.gen_kv_bits_np(9, int(np.prod(shp))).reshape(shp)
        kv = bits_to_torch(bits, "bf16", cuda)
        t32 = lambda x: torch.as_tensor(np.asarray(x, np.int32), device=cuda)
        st = torch.zeros(1, dtype=torch.int32, device=cuda)
        kept = [bound, bound + 1, 2]
        s = kv.stride()
        _abi.specdec_realign_kv(kv, kv, t32(kept), n_planes=planes, n_rows=B, H=H, D=D,
                                src_strides=s[:3], dst_strides=s[:3], cap_src=cap, cap_dst=cap,
                                src_col=t32([0, 0, 0]), dst_col=t32([3, 3, 3]), status=st,
                                count_bound=bound)
        torch.cuda.synchronize()
        assert int(st.item()) == _abi.ST_BOUND
        g = torch_to_bits(kv)
        assert np.array_equal(g[:, 1], bits[:, 1])          # skipped
        o, _ = OA.realign_kv(bits, np.zeros(B, np.int32), np.full(B, 3, np.int32), np.array(kept))
        for i in (0, 2):
            assert np.array_equal(g[:, i, :, 3:3 + kept[i]], o[:, i, :, 3:3 + kept[i]])


@pytest.mark.parametrize("bound", [0, 6])
def test_realign_gather_scatter(cuda, bound):
    """Pool mode (a5): gather from a sequence-major pool into a plane-major staging
    rectangle at right-aligned columns, then scatter a tail back (distinct buffers);
    bound = 6 = k + 1 sends the scatter through the small-slab kernel, as the pool does."""
    N, planes, H, cap, D = 6, 4, 2, 90, 64
    B, cap_b = 3, 100
    pool_bits = W.gen_kv_bits_np(11, N * planes * H * cap * D).reshape(N, planes, H, cap, D)
    pool = bits_to_torch(pool_bits, "bf16", cuda)
    stage = torch.zeros((planes, B, H, cap_b, D), dtype=torch.bfloat16, device=cuda)
    members = np.array([4, 0, 2], np.int32)
    lens = np.array([50, 81, 20], np.int32)
    Lb = int(lens.max())
    mpad = (Lb - lens).astype(np.int32)
    t32 = lambda x: torch.as_tensor(np.asarray(x, np.int32), device=cuda)
    ps, ss = pool.stride(), stage.stride()
    # gather: pool[s, :, :, 0:len-1] -> stage[:, i, :, mpad_i : mpad_i + len - 1]
    _abi.specdec_realign_kv(pool, stage, t32(lens), count_add=-1, n_planes=planes, n_rows=B, H=H, D=D,
                            src_strides=(ps[1], ps[0], ps[2]), dst_strides=ss[:3], cap_src=cap,
                            cap_dst=cap_b, dst_col=t32(mpad), src_row_map=t32(members))
    torch.cuda.synchronize()
    st = torch_to_bits(stage)
    logical_pool = pool_bits.transpose(0, 1, 2, 3, 4)     # [rows][planes][H][cap][D]
    exp = np.zeros((B, planes, H, cap_b, D), np.uint16)
    OA.copy_rows(logical_pool, exp, count=lens - 1, src_row=members, dst_col=mpad)
    for i in range(B):
        c0, c1 = mpad[i], mpad[i] + lens[i] - 1
        assert np.array_equal(st[:, i, :, c0:c1], exp[i][:, :, c0:c1])
    # scatter: stage[:, i, :, Lb-1 : Lb+a_i] -> pool[s, :, :, len-1 : len+a_i]
    acc = np.array([5, 0, 2], np.int32)
    tail = W.gen_kv_bits_np(12, planes * B * H * 6 * D).reshape(planes, B, H, 6, D)
    stage[:, :, :, Lb - 1:Lb + 5, :] = bits_to_torch(tail, "bf16", cuda)
    _abi.specdec_realign_kv(stage, pool, t32(acc), count_add=1, n_planes=planes, n_rows=B, H=H, D=D,
                            src_strides=ss[:3], dst_strides=(ps[1], ps[0], ps[2]), cap_src=cap_b,
                            cap_dst=cap, src_col_add=Lb - 1, dst_col=t32(lens), dst_col_add=-1,
                            dst_row_map=t32(members), count_bound=bound)
    torch.cuda.synchronize()
    pg = torch_to_bits(pool)
    for i, s in enumerate(members):
        lo = lens[i] - 1
        assert np.array_equal(pg[s][:, :, lo:lo + acc[i] + 1], tail[:, i, :, :acc[i] + 1])
        assert np.array_equal(pg[s][:, :, :lo], pool_bits[s][:, :, :lo])
    untouched = [s for s in range(N) if s not in members]
    assert np.array_equal(pg[untouched], pool_bits[untouched])


# ----------------------------------------------------------------------------- full size
@pytest.mark.parametrize("name", ["qwen3", "glm4", "vicuna"])
def test_full_size_sampled(cuda, name):
    """BASELINE.json full sizes in the bench's launch configuration: every integer output
    of the round exactly; KV checked on a sample of (plane, row, head) slabs."""
    shape = W.SHAPES[name]
    B, k = shape.B, shape.k
    rounds = 3
    cap = W.derive_cap(shape, rounds)
    lengths = W.gen_lengths(shape, 0, B)
    tokens = W.left_padded_tokens(lengths, cap, 0, shape.V)
    bt = EqSpecBatch(B, k, cap, shape.layers, shape.H, shape.D, shape.kv_dtype, cuda)
    bt.load(tokens, lengths)
    bt.kv.copy_(W.gen_kv_torch(0, bt.kv.shape, bt.kv.dtype, cuda))
    rng = np.random.default_rng(0)
    samples = [(int(rng.integers(shape.n_planes)), int(rng.integers(B)), int(rng.integers(shape.H)))
               for _ in range(24)]
    n_o = lengths.astype(np.int32)
    pad_o = (n_o.max() - n_o).astype(np.int32)
    act = np.ones(B, np.uint8)
    for r in range(rounds):
        before = {s: torch_to_bits(bt.kv[s[0], s[1], s[2]]) for s in samples}
        rt = W.gen_round_truth(0, r, B, k, shape.V, "alpha")
        lg = W.gen_logits_torch(0, r, B, k, shape.V, shape.logit_dtype, cuda)
        bits = torch_to_bits(lg)
        bt.step(lg, torch.from_numpy(rt.draft).to(cuda))
        v = OV.batch_verify(bits, shape.logit_dtype, rt.draft, n_o, pad_o, act)
        torch.cuda.synchronize()
        assert np.array_equal(bt.accept.cpu().numpy(), v["accept"])
        assert np.array_equal(bt.accept.cpu().numpy(), rt.accept)
        assert np.array_equal(bt.bonus.cpu().numpy(), v["bonus"])
        assert np.array_equal(bt.pad_cur.cpu().numpy(), v["pad_new"])
        for (pl, i, h), old in before.items():
            new = torch_to_bits(bt.kv[pl, i, h])
            po, pn, kp = pad_o[i], v["pad_new"][i], v["kept"][i]
            assert np.array_equal(new[pn:pn + kp], old[po:po + kp]), (r, pl, i, h)
        n_o, pad_o = v["n_new"], v["pad_new"]
    assert int(bt.status.item()) == 0


@pytest.mark.parametrize("drive", ["native", "host", "host_packed", "fork"])
@pytest.mark.parametrize("pattern", ["alpha", "alternating", "all_k"])
def test_rounds_native_driver(cuda, drive, pattern):
    """specdec_eqspec_round (one C call per round) and specdec_eqspec_round_host (H2D +
    round + D2H) against the oracle, like the Python-driven rounds."""
    _run_rounds(cuda, SMALL, 8, 12, pattern, drive=drive)


@pytest.mark.parametrize("drive", ["native", "host", "host_packed"])
def test_rounds_native_driver_modes(cuda, drive):
    _run_rounds(cuda, SMALL16, 5, 10, "alpha", seed=3, kv_mode="pingpong", drive=drive)
    _run_rounds(cuda, W.SHAPES["toy"], 2, 30, "alpha", max_new=24, eos_id=7, drive=drive)
    _run_rounds(cuda, SMALL, 1, 6, "alpha", drive=drive)
    _run_rounds(cuda, SMALL, 6, 6, "one_zero", zero_pads=True, drive=drive)


@pytest.mark.parametrize("drive", ["native", "host"])
def test_rounds_native_driver_anchored(cuda, drive):
    """The round drivers with the anchored origin (f3): K1's physical columns drive K2."""
    py = _run_rounds(cuda, SMALL, 8, 12, "alpha", seed=3, anchor_slack=96)
    nat = _run_rounds(cuda, SMALL, 8, 12, "alpha", seed=3, anchor_slack=96, drive=drive)
    assert nat["bases"] == py["bases"] and nat["moved"] == py["moved"]
    _run_rounds(cuda, SMALL16, 6, 14, "alpha", seed=2, max_new=33, anchor_slack=32, drive=drive)
    _run_rounds(cuda, SMALL, 1, 6, "alpha", anchor_slack=16, drive=drive)


@pytest.mark.parametrize("shape,B,pattern,kw", [(SMALL, 8, "alpha", {}), (SMALL16, 5, "alternating", {"kv_mode": "pingpong"}),
                                               (SMALL, 6, "alpha", {"anchor_slack": 64}),
                                               (W.SHAPES["toy"], 2, "alpha", {"max_new": 24, "eos_id": 7}),
                                               (SMALL, 1, "all_k", {})])
def test_rounds_graph_replay(cuda, shape, B, pattern, kw):
    """Rounds replayed from the captured CUDA graphs (the bench's value path: programmatic
    edges between K1's grid, its epilogue kernel, K3 and K2; K2 starting under K3; dynamic
    K2 tickets reset across replays) against the oracle, round by round."""
    _run_rounds(cuda, shape, B, 10, pattern, drive="graph", **kw)


def test_multi_round_graph_equals_direct(cuda):
    """A graph holding 6 consecutive rounds (distinct input buffers, parities alternating),
    replayed twice, leaves exactly the state of 12 directly launched rounds -- tokens,
    lengths, pads, masks, positions, results and every KV byte."""
    sh = SMALL
    B, k, V = 8, sh.k, sh.V
    cap = W.derive_cap(sh.with_(B=B), 14)
    lengths = W.gen_lengths(sh, 4, B)
    tokens = W.left_padded_tokens(lengths, cap, 4, V)
    kv_bits = W.gen_kv_bits_np(4, sh.n_planes * B * sh.H * cap * sh.D).reshape(sh.n_planes, B, sh.H, cap, sh.D)
    ins = [(padded_logits(W.gen_logits_np(4, r, B, k, V, sh.logit_dtype), sh.logit_dtype, cuda),
            torch.from_numpy(W.gen_round_truth(4, r, B, k, V, "alpha").draft).to(cuda)) for r in range(6)]
    bts = []
    for _ in range(2):
        bt = EqSpecBatch(B, k, cap, sh.layers, sh.H, sh.D, sh.kv_dtype, cuda, max_new=40, pad_id=W.PAD_ID)
        bt.load(tokens, lengths, bits_to_torch(kv_bits, sh.kv_dtype, cuda))
        bt.V = V
        bts.append(bt)
    direct, graphed = bts
    for r in range(12):
        direct.step(*ins[r % 6], V=V)
    s = torch.cuda.Stream(cuda)
    s.wait_stream(torch.cuda.current_stream(cuda))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        for r in range(6):
            graphed.launch_round(*ins[r], stream=s)
            graphed.cur = 1 - graphed.cur
    torch.cuda.current_stream(cuda).wait_stream(s)
    g.replay()
    g.replay()
    torch.cuda.synchronize()
    assert direct.cur == graphed.cur
    for name in ("tok", "n", "pad", "mask", "pos", "active", "budget", "gen", "out_buf", "_accept", "_emit",
                 "_bonus", "_finished", "kept", "plan_L", "status"):
        assert torch.equal(getattr(direct, name), getattr(graphed, name)), name
    assert torch.equal(direct.kv.view(torch.int16), graphed.kv.view(torch.int16))


K2_FUZZ = int(__import__("os").environ.get("SPECDEC_K2_FUZZ_CASES", "16"))


@pytest.mark.parametrize("i", range(K2_FUZZ))
def test_realign_fuzz(cuda, i):
    """K2 alone on seeded random geometry: rows, planes, heads, head_dim, dtype, capacity,
    arbitrary shifts of either sign (not only |delta| <= k), Delta = 0 rows, empty rows, and
    random flag sets (ZERO_PADS, SEGMENTED, DYNAMIC, count_bound) -- every defined KV entry
    and zeroed pad against the oracle."""
    r = np.random.default_rng(40_000 + i)
    B = int(r.integers(1, 13))
    D, dtype = [(8, "bf16"), (16, "fp16"), (64, "bf16"), (128, "bf16"), (4, "fp32"), (72, "fp16")][int(r.integers(0, 6))]
    planes, H = int(r.integers(1, 5)), int(r.integers(1, 4))
    kept = r.integers(0, 300, B)
    kept[r.random(B) < 0.15] = 0
    pad_old = r.integers(0, 60, B)
    shift = r.integers(-40, 41, B)
    shift[r.random(B) < 0.2] = 0
    pad_new = np.maximum(pad_old + shift, 0)
    zero = bool(r.random() < 0.3)
    seg = bool(r.random() < 0.3)
    dyn = bool(r.random() < 0.5)
    bound = int(kept.max()) if (r.random() < 0.2 and kept.max() * D * (4 if dtype == "fp32" else 2) <= 4096) else 0
    _realign_case(cuda, pad_old.tolist(), pad_new.tolist(), kept.tolist(), D=D, H=H, planes=planes, dtype=dtype,
                  zero=zero, seg=seg, bound=bound, dyn=dyn)


K3_FUZZ = int(__import__("os").environ.get("SPECDEC_K3_FUZZ_CASES", "12"))


@pytest.mark.parametrize("i", range(K3_FUZZ))
def test_repad_fuzz(cuda, i):
    """K3 alone, in place (one CTA walks each row in the hazard-free direction) and out of
    place (column gather), on seeded random plans from the oracle's verify (ragged
    lengths, every accept pattern, EOS / budget finishes, inactive rows, output buffers):
    tokens', masks, positions, outputs and counts bit-exact against the oracle."""
    r = np.random.default_rng(70_000 + i)
    B, k = int(r.integers(1, 13)), int(r.integers(1, 9))
    V = 97
    n = r.integers(1, 120, B).astype(np.int32)
    L = int(n.max())
    pad = (L - n).astype(np.int32)
    cap = L + 3 * (k + 1) + int(r.integers(0, 20))
    tokens = np.full((B, cap), W.PAD_ID, np.int64)
    for b in range(B):
        tokens[b, pad[b]:L] = r.integers(1, V, n[b])
    pattern = W.ACCEPT_PATTERNS[int(r.integers(0, len(W.ACCEPT_PATTERNS)))]
    rt = W.gen_round_truth(80 + i, 0, B, k, V, pattern)
    bits = W.gen_logits_np(80 + i, 0, B, k, V, "fp32")
    act = (r.random(B) < 0.85).astype(np.uint8)
    eos = int(r.integers(0, V)) if r.random() < 0.3 else -1
    budget = r.integers(0, 10, B).astype(np.int64) if r.random() < 0.4 else None
    v = OV.batch_verify(bits, "fp32", rt.draft, n, pad, act, eos, budget, W.PAD_ID)
    tok_o, mask_o, pos_o = OA.repad_tokens(tokens, cap, k, pad, L, v, W.PAD_ID)
    max_new = 64
    gen0 = r.integers(0, 20, B).astype(np.int32)
    t32 = lambda x: torch.as_tensor(np.asarray(x, np.int32), device=cuda)
    t64 = lambda x: torch.as_tensor(np.asarray(x, np.int64), device=cuda)
    for inplace in (True, False):
        tin = t64(tokens)
        tout = tin if inplace else torch.full_like(tin, -7)
        mask = torch.full((B, cap + k), -7, dtype=torch.int64, device=cuda)
        pos = torch.full_like(mask, -7)
        out_buf = torch.zeros((B, max_new), dtype=torch.int64, device=cuda)
        gen = t32(gen0)
        st = torch.zeros(1, dtype=torch.int32, device=cuda)
        _abi.specdec_rebuild_pos_mask(tin, tout, k, t32(n), t32(pad), t64(rt.draft), t32(v["accept"]),
                                      t64(v["bonus"]), t32(v["emit"]), torch.as_tensor(v["finished"], device=cuda),
                                      t32([v["L_new"]]), t32(v["pad_new"]), mask, pos, pad_id=W.PAD_ID,
                                      out_buf=out_buf, gen=gen, status=st)
        torch.cuda.synchronize()
        Ln = v["L_new"]
        assert int(st.item()) == 0, inplace
        if Ln > 0:
            assert np.array_equal(tout[:, :Ln].cpu().numpy(), tok_o[:, :Ln]), inplace
            assert np.array_equal(mask[:, :Ln + k].cpu().numpy(), mask_o), inplace
            assert np.array_equal(pos[:, :Ln + k].cpu().numpy(), pos_o), inplace
        g = gen.cpu().numpy()
        assert np.array_equal(g, gen0 + v["emit"]), inplace
        ob = out_buf.cpu().numpy()
        for b in range(B):
            assert list(ob[b, gen0[b]:g[b]]) == v["E"][b], (inplace, b)


@pytest.mark.parametrize("B", [1, 2, 8, 37, 1500])
def test_batch_init_matches_oracle_left_padding(cuda, B):
    """specdec_batch_init (Alg. 2 line 1) == oracle.align.build_batch's pads
    and width on seeded ragged lengths (B up to 1500: several strides of the one CTA)."""
    rng = np.random.default_rng(B)
    lens = rng.integers(1, 3000, size=B).astype(np.int32)
    _, pad_o, L_o = OA.build_batch([[5] * int(n) for n in lens], int(lens.max()) + 1)
    n = torch.from_numpy(lens).to(cuda)
    pad = torch.full((B,), -7, dtype=torch.int32, device=cuda)
    L = torch.zeros(1, dtype=torch.int32, device=cuda)
    act = torch.zeros(B, dtype=torch.uint8, device=cuda)
    bud = torch.zeros(B, dtype=torch.int32, device=cuda)
    st = torch.zeros(1, dtype=torch.int32, device=cuda)
    _abi.specdec_batch_init(n, pad, L=L, active=act, budget=bud, max_new=77, status=st)
    torch.cuda.synchronize()
    assert np.array_equal(pad.cpu().numpy(), pad_o) and int(L.item()) == L_o
    assert bool((act == 1).all()) and bool((bud == 77).all()) and int(st.item()) == 0
    # a row with n < 1 is flagged (SPECDEC_ST_CAPACITY), its pad is L
    n[0] = 0
    _abi.specdec_batch_init(n, pad, status=st)
    torch.cuda.synchronize()
    assert int(st.item()) & _abi.ST_CAPACITY and int(pad[0].item()) == int(n.max().item())
