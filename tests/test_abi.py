"""The C-ABI library loads and exports every symbol include/specdec.h declares, and its
host-side argument validation rejects bad calls before any launch (no GPU needed)."""
import ctypes
import os
import re

import pytest

from paper_2510_22876_b200 import _abi
from paper_2510_22876_b200 import build as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    B.build()
    return _abi.load()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "specdec.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(specdec_\w+)\s*\(", src)))


def test_header_symbols_exported(lib):
    names = declared_symbols()
    assert {"specdec_verify", "specdec_realign_kv", "specdec_rebuild_pos_mask",
            "specdec_pool_group"} <= set(names)
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_abi.EXPORTS)


def test_version_and_workspace(lib):
    assert _abi.version() == 121
    # keys [B(k+1)] u64 | counter, max n', pad | row counters [B] u32 | class weights [k+1] u64
    assert _abi.specdec_verify_workspace_size(8, 5) == 8 * 6 * 8 + 16 + 32 + 6 * 8
    assert _abi.specdec_verify_workspace_size(3, 2) == 3 * 3 * 8 + 16 + 16 + 3 * 8
    assert _abi.specdec_verify_workspace_size(0, 5) == 0


def test_host_validation_without_gpu(lib):
    L = lib
    nz = ctypes.c_void_p(16)   # never dereferenced: validation fails first
    # k < 1 -> ERR_ARG
    rc = L.specdec_verify(nz, 2, 8, 0, 100, 100, *([nz] * 3), -1, 0, None, *([nz] * 4), None,
                          *([nz] * 4), None, None, 0, None, None, None, nz, 1 << 20, None)
    assert rc == _abi.ERR_ARG
    # unknown dtype
    rc = L.specdec_verify(nz, 9, 8, 5, 100, 100, *([nz] * 3), -1, 0, None, *([nz] * 4), None,
                          *([nz] * 4), None, None, 0, None, None, None, nz, 1 << 20, None)
    assert rc == _abi.ERR_DTYPE
    # row_stride < V
    rc = L.specdec_verify(nz, 2, 8, 5, 100, 50, *([nz] * 3), -1, 0, None, *([nz] * 4), None,
                          *([nz] * 4), None, None, 0, None, None, None, nz, 1 << 20, None)
    assert rc == _abi.ERR_SHAPE
    # misaligned row stride (bf16, 100 elements = 200 B, not a multiple of 16)
    rc = L.specdec_verify(nz, 2, 8, 5, 100, 100, *([nz] * 3), -1, 0, None, *([nz] * 4), None,
                          *([nz] * 4), None, None, 0, None, None, None, nz, 1 << 20, None)
    assert rc == _abi.ERR_ARG
    # realign: D*elem not a multiple of 16
    rc = L.specdec_realign_kv(nz, nz, 2, 2, 2, 2, 4, 64, 64, 64, 8, 64, 64, 64, 8, None, 0,
                              None, 0, nz, 0, 0, None, None, 0, None, 0, None, None, None)
    assert rc == _abi.ERR_ARG
    # in place with row maps -> ERR_ARG
    rc = L.specdec_realign_kv(nz, nz, 2, 2, 2, 2, 8, 64, 64, 64, 8, 64, 64, 64, 8, None, 0,
                              None, 0, nz, 0, 0, nz, None, 0, None, 0, None, None, None)
    assert rc == _abi.ERR_ARG
    # workspace too small for the segment slots -> ERR_ARG
    rc = L.specdec_realign_kv(nz, nz, 2, 2, 2, 2, 8, 64, 64, 64, 8, 64, 64, 64, 8, None, 0,
                              None, 0, nz, 0, 0, None, None, 0, nz, 16, None, None, None)
    assert rc == _abi.ERR_ARG
    # negative count_bound -> ERR_ARG
    rc = L.specdec_realign_kv(nz, nz, 2, 2, 2, 2, 8, 64, 64, 64, 8, 64, 64, 64, 8, None, 0,
                              None, 0, nz, 0, -1, None, None, 0, None, 0, None, None, None)
    assert rc == _abi.ERR_ARG
    assert _abi.specdec_realign_workspace_size(__import__("torch").bfloat16, 72, 8, 8, 128, 2736) > 0
    # pool_group: B > W
    rc = L.specdec_pool_group(nz, nz, nz, 10, 4, 8, 2, *([nz] * 14))
    assert rc == _abi.ERR_SHAPE
    # rebuild: capacity statically impossible
    rc = L.specdec_rebuild_pos_mask(nz, nz, 2, 4, 5, 0, *([nz] * 11), 64, None, None, 0, None, None)
    assert rc == _abi.ERR_CAPACITY
    # getbatch: B > W (same limits as pool_group)
    rc = L.specdec_pool_getbatch(nz, nz, nz, 10, 4, 8, 2, *([nz] * 14))
    assert rc == _abi.ERR_SHAPE
    # batch init: NULL lengths / B < 1
    assert L.specdec_batch_init(None, 4, nz, None, None, None, 0, None, None) == _abi.ERR_ARG
    assert L.specdec_batch_init(nz, 0, nz, None, None, None, 0, None, None) == _abi.ERR_SHAPE
    # grouped pool verify: 0 or more than SPECDEC_MAX_VERIFY_GROUP batches, a batch with no rows
    G1 = _abi.MAX_VERIFY_GROUP + 1
    P = ctypes.c_void_p * G1
    I = ctypes.c_int32 * G1
    ptrs, offs, rows = P(*([16] * G1)), I(*([0] * G1)), I(*([1] * G1))
    for n in (0, G1):
        rc = L.specdec_pool_verify_group(n, ptrs, ptrs, offs, rows, 2, 5, 100, 104, *([nz] * 3), -1, 0,
                                         *([nz] * 7), None, 0, None, 16, None, nz, 1 << 20, None)
        assert rc == _abi.ERR_ARG, n
    rows[1] = 0
    rc = L.specdec_pool_verify_group(2, ptrs, ptrs, offs, rows, 2, 5, 100, 104, *([nz] * 3), -1, 0,
                                     *([nz] * 7), None, 0, None, 16, None, nz, 1 << 20, None)
    assert rc == _abi.ERR_SHAPE
    # the Alg. 3 graph: NULL descriptor; graph launch / destroy of NULL
    assert L.specdec_pool_alg3_graph(None, 16, nz, None, 0, ctypes.byref(ctypes.c_void_p())) == _abi.ERR_ARG
    assert L.specdec_graph_launch(None, None) == _abi.ERR_ARG
    assert L.specdec_graph_destroy(None) == _abi.OK


def test_missing_library_fails_loudly(tmp_path):
    saved = _abi._lib
    try:
        _abi._lib = None
        with pytest.raises(_abi.SpecdecError):
            _abi.load(str(tmp_path / "nope.so"))
    finally:
        _abi._lib = saved


@pytest.mark.parametrize("cname,pyname", [("specdec_pool_desc", "PoolDesc"),
                                           ("specdec_round_desc", "RoundDesc"),
                                           ("specdec_host_io", "HostIO")])
def test_desc_layout_matches_header(tmp_path, cname, pyname):
    """The ctypes mirrors of the descriptor structs have the C compiler's size and offsets."""
    import shutil
    import subprocess
    if not shutil.which("g++"):
        pytest.skip("no host C++ compiler")
    src = tmp_path / "l.cpp"
    P = getattr(_abi, pyname)
    names = [f[0] for f in P._fields_]
    body = "".join(f' printf("%zu\\n", offsetof({cname}, {n}));' for n in names)
    src.write_text('#include <cstdio>\n#include <cstddef>\n#include "specdec.h"\n'
                   'int main(){printf("%zu\\n", sizeof(' + cname + '));' + body + '}\n')
    exe = tmp_path / "l"
    subprocess.run(["g++", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = list(map(int, subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()))
    # every field, in order, at the C compiler's offset
    assert got == [ctypes.sizeof(P)] + [getattr(P, n).offset for n in names]


def test_header_is_plain_c_and_links(tmp_path, lib):
    """include/specdec.h compiles as C99 and a C program links libspecdec.so and gets the
    host-side argument errors back (no GPU, no torch)."""
    import shutil
    import subprocess
    if not shutil.which("gcc"):
        pytest.skip("no host C compiler")
    src = tmp_path / "c.c"
    src.write_text(r'''
#include <stdio.h>
#include "specdec.h"
int main(void) {
    int rc = specdec_verify((const void *)16, SPECDEC_BF16, 8, 0, 100, 104, 0, 0, 0, -1, 0, 0,
                            0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0);
    size_t ws = specdec_verify_workspace_size(8, 5);
    printf("%d %d %zu\n", specdec_version(), rc, ws);
    return 0;
}
''')
    exe = tmp_path / "c"
    libdir = os.path.dirname(_abi.lib_path())
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), str(src),
                    "-L", libdir, "-l:libspecdec.so", "-Wl,-rpath," + libdir, "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    assert out == ["121", str(_abi.ERR_ARG), str(8 * 6 * 8 + 16 + 32 + 6 * 8)]


def test_host_validation_drivers_and_flags(lib):
    """Argument errors of the realign flags, the round drivers and the pool executor's
    overlap configuration are caught on the host (nothing launched, no GPU needed)."""
    L = lib
    nz = ctypes.c_void_p(16)
    real = lambda flags, ws, wsb: L.specdec_realign_kv(nz, nz, 2, 2, 2, 2, 8, 64, 64, 64, 8, 64, 64, 64, 8,
                                                       None, 0, None, 0, nz, 0, 0, None, None, flags, ws,
                                                       wsb, None, None, None)
    assert real(_abi.DYNAMIC, None, 0) == _abi.ERR_ARG          # tickets need the workspace header
    assert real(_abi.SEGMENTED, None, 0) == _abi.ERR_ARG        # segment slots need a workspace
    assert real(16, None, 0) == _abi.ERR_ARG                    # unknown flag
    assert real(_abi.DYNAMIC, nz, 64) == _abi.ERR_ARG           # header is 128 bytes
    d = _abi.RoundDesc()
    assert L.specdec_eqspec_round(None, 0, nz, nz, None) == _abi.ERR_ARG
    assert L.specdec_eqspec_round(ctypes.byref(d), 2, nz, nz, None) == _abi.ERR_ARG
    assert L.specdec_eqspec_round(ctypes.byref(d), 0, None, nz, None) == _abi.ERR_ARG
    io = _abi.HostIO()
    assert L.specdec_eqspec_round_host(ctypes.byref(d), None, 0, 0, nz, nz, None, None) == _abi.ERR_ARG
    assert L.specdec_eqspec_round_host(ctypes.byref(d), ctypes.byref(io), 0, 0, nz, nz, None, None) == _abi.ERR_ARG  # n_slots 0
    io.n_slots = 3
    assert L.specdec_eqspec_round_host(ctypes.byref(d), ctypes.byref(io), 0, 3, nz, nz, None, None) == _abi.ERR_ARG  # slot >= n_slots
    assert L.specdec_eqspec_round_host(ctypes.byref(d), ctypes.byref(io), 0, 0, nz, nz, None, None) == _abi.ERR_ARG  # no staging
    io.n_slots = 5
    assert L.specdec_eqspec_round_host(ctypes.byref(d), ctypes.byref(io), 0, 0, nz, nz, None, None) == _abi.ERR_ARG
    p = _abi.PoolDesc()
    p.host_header, p.W, p.B = 16, 4, 2
    p.logits_ring, p.draft_ring, p.ring_n, p.ring_pos = 16, 16, 1, 16
    p.n_staging = 2                                              # overlap without ring / stream / events
    assert L.specdec_pool_epoch(ctypes.byref(p), None, None, 0, None, None, None, None, None) == _abi.ERR_ARG
    assert L.specdec_pool_epoch(None, None, None, 0, None, None, None, None, None) == _abi.ERR_ARG


def test_host_round_binding_rejects_unpinned(lib):
    """specdec_eqspec_round_host's binding takes pinned host tensors only (no silent sync copy)."""
    import torch
    with pytest.raises(_abi.SpecdecError):
        _abi.specdec_eqspec_round_host(_abi.RoundDesc(), _abi.HostIO(), 0, 0, torch.zeros(4), torch.zeros(4))


def test_max_verify_group_matches_header():
    """The binding's MAX_VERIFY_GROUP is the header's SPECDEC_MAX_VERIFY_GROUP."""
    import re
    h = open(os.path.join(ROOT, "include", "specdec.h")).read()
    assert int(re.search(r"#define SPECDEC_MAX_VERIFY_GROUP (\d+)", h).group(1)) == _abi.MAX_VERIFY_GROUP
