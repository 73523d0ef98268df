"""CPU-side checks of the C-ABI library: it loads without a GPU, exports every symbol
include/paro.h declares, and its pure-host entry points (size arithmetic, argument
checks that fail before any CUDA call) behave as documented."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "paro.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(paro_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def paro():
    from paper_2511_10645_b200 import _build
    _build.build()
    import paper_2511_10645_b200 as m
    return m


def test_header_declares_the_boundary():
    fns = declared_functions()
    for f in ["paro_pack_sizes", "paro_pack", "paro_linear", "paro_linear_multi", "paro_linear_workspace",
              "paro_transform_activations",
              "paro_unpack_logical", "paro_comm_unique_id", "paro_comm_init", "paro_comm_destroy",
              "paro_linear_allgather", "paro_linear_allgather_workspace", "paro_select_pairs", "paro_fwht", "paro_linear_chain", "paro_linear_allgather_p2p", "paro_ipc_get_handle", "paro_linear_chain_workspace", "paro_last_error",
              "paro_transform_activations_dense", "paro_transform_dense_workspace", "paro_copy",
              "paro_version"]:
        assert f in fns


def test_library_exports_every_declared_symbol(paro):
    lib = ctypes.CDLL(paro.LIB_PATH)
    for f in declared_functions():
        assert hasattr(lib, f), f"libparo.so does not export {f}"
    assert set(declared_functions()) == set(paro.SIGNATURES), "binding signatures out of sync with paro.h"


def test_pack_sizes(paro):
    sz = paro.paro_pack_sizes(4096, 4096, 128, 8)
    G = 32
    tiles = (4096 // 32) * G                   # tiles of 32 rows x one 128-group
    assert sz.codes == 4096 * 4096 // 2 == tiles * 2048
    assert sz.scales == 4096 * G * 2 == tiles * 64 and sz.zeros == 4096 * G // 2 == tiles * 16
    assert sz.rot_cs == G * 8 * 64 * 8 and sz.rot_idx == G * 8 * 64 * 2 and sz.svec == 4096 * 4 + 4096  # s + K-split counters
    sz = paro.paro_pack_sizes(3, 384, 128, 0)   # a partial row block pads to 32 rows
    assert sz.codes == 3 * 2048 and sz.scales == 3 * 64 and sz.zeros == 3 * 16 and sz.rot_cs == 0


@pytest.mark.parametrize("args,kind", [
    ((4096, 200, 128, 8), "unsupported"),      # K % 128 != 0 (Q17)
    ((4096, 4096, 64, 8), "unsupported"),      # group != 128
    ((4096, 4096, 128, 9), "unsupported"),     # n_rot > 8
    ((0, 4096, 128, 8), "invalid_argument"),
    ((16, -128, 128, 8), "invalid_argument"),
])
def test_pack_sizes_errors(paro, args, kind):
    with pytest.raises(paro.ParoError) as e:
        paro.paro_pack_sizes(*args)
    assert e.value.kind == kind
    assert paro.last_error()


def test_linear_rejects_null_before_cuda(paro):
    """Argument errors are reported before any CUDA call (works on a CPU-only box)."""
    st = paro._lib.paro_linear(None, 0, 1, None, None, None, None, 0, None, None, 0, 0, None, 0, None)
    assert st == paro.PARO_ERR_INVALID_ARGUMENT
    pk = paro.paro_packed(16, 16, 16, 16, 16, 16, 256, 200, 128, 8)   # K not multiple of 128
    st = paro._lib.paro_linear(16, 0, 1, ctypes.byref(pk), None, None, None, 0, None, 16, 0, 0, None, 0, None)
    assert st == paro.PARO_ERR_SHAPE


def test_workspace_arithmetic(paro):
    assert paro.paro_linear_workspace(1, 4096, 4096) == 0
    assert paro.paro_linear_workspace(1, 4096, 4096, 8, 64, True) >= 32 * 8 * 64 * 10
    # one token, long K and a long stream (LLaMA-3-70B down_proj, G = 224): K split over 7 clusters
    # of 2 -> 7 x N fp32 row sums; shorter streams (8B down_proj) need none
    assert paro.paro_linear_workspace(1, 8192, 28672) == 7 * 8192 * 4
    assert paro.paro_linear_workspace(1, 4096, 14336) == 0
    assert paro.paro_linear_workspace(1, 28672, 8192) == 0  # 70B gate: clusters of 2 already


def test_shard_rows(paro):
    assert paro.shard_rows(28672, 8, 3) == (3 * 3584, 4 * 3584)
    with pytest.raises(paro.ParoError):
        paro.shard_rows(1000, 3, 0)


def test_product_package_never_imports_oracle():
    """The product path must not route through the oracle (or any CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_2511_10645_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "oracle/" not in txt, f


def test_chain_workspace_and_argument_errors(paro):
    """paro_linear_chain's host checks: workspace size (grid-barrier header + B > 1 x' buffers) and
    argument errors reported before any CUDA call."""
    pk = paro.paro_packed(16, 16, 16, 16, 16, 16, 4096, 4096, 128, 8)
    pks = (paro.paro_packed * 1)(pk)
    ys = (ctypes.c_void_p * 1)(16)
    st = (paro.paro_chain_stage * 2)()
    for k in range(2):
        st[k].x = 16
        st[k].n = 1
        st[k].packed = ctypes.cast(pks, ctypes.POINTER(paro.paro_packed))
        st[k].y = ctypes.cast(ys, ctypes.POINTER(ctypes.c_void_p))
    ws1 = paro._lib.paro_linear_chain_workspace(1, 2, st)
    ws16 = paro._lib.paro_linear_chain_workspace(16, 2, st)
    assert ws1 >= 8192 and ws16 >= ws1 + 4 * 32 * 4096            # B > 1: x' of 4 linear slots
    assert paro._lib.paro_linear_chain_workspace(1, 0, st) == 0
    # B > 16, and a workspace that is too small
    assert paro._lib.paro_linear_chain(2, st, 0, 17, 0, 0, 16, ws1, None) == paro.PARO_ERR_UNSUPPORTED
    assert paro._lib.paro_linear_chain(2, st, 0, 1, 0, 0, 16, 64, None) == paro.PARO_ERR_INVALID_ARGUMENT
    assert "workspace" in paro.last_error()


def test_copy_and_dense_transform_argument_errors(paro):
    """paro_copy and paro_transform_activations_dense reject bad arguments before any CUDA call."""
    lib = paro._lib
    INV = 1  # PARO_ERR_INVALID_ARGUMENT
    assert lib.paro_copy(None, ctypes.c_void_p(16), 16, 0, None) == INV          # NULL dst
    assert lib.paro_copy(ctypes.c_void_p(16), ctypes.c_void_p(16), 24, 0, None) == INV  # not a multiple of 16
    assert lib.paro_copy(ctypes.c_void_p(8), ctypes.c_void_p(16), 16, 0, None) == INV   # misaligned
    assert lib.paro_copy(ctypes.c_void_p(16), ctypes.c_void_p(32), 0, 0, None) == 0     # nothing to copy
    assert lib.paro_transform_dense_workspace(4096) == 128 * 4096 * 2
    assert lib.paro_transform_activations_dense(None, 0, 1, None, None, None, 0, None) != 0  # NULL packed
    assert paro.last_error()  # a message for the failed call
