"""The C-ABI library loads and exports every symbol include/spconv.h declares; host-side
argument validation (no device work) returns the documented codes. Runs without a GPU."""
from __future__ import annotations

import ctypes as C
import os
import re

import pytest

import paper_1801_10585_b200 as spc
from paper_1801_10585_b200 import _lib
from paper_1801_10585_b200._lib import FilterT, MapT

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "spconv.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\*?\s+\**([a-z_0-9]+)\s*\(", src, flags=re.M)))


def test_header_declares_the_north_star_calls():
    fns = header_functions()
    for name in ["sparse_conv_fwd", "sparse_conv_bwd_input", "sparse_conv_bwd_weight", "sparse_relu",
                 "sparse_maxpool", "attention_topk"]:
        assert name in fns
    assert sorted(_lib.EXPORTS) == fns


def test_library_exports_every_declared_symbol():
    lib = spc.load()
    for name in header_functions():
        assert hasattr(lib, name), name
    out = os.popen(f"nm -D {_lib.LIB_PATH}").read()
    for name in header_functions():
        assert re.search(rf" T {name}$", out, flags=re.M), name


def test_version_and_status_strings():
    lib = spc.load()
    assert b"sm_100a" in lib.spc_version()
    assert lib.spc_status_string(3) == b"output capacity too small"


def _c4_structs(ks=(3, 3, 3), c_in=8, ndim=3):
    m = MapT()
    m.ndim, m.batch, m.channels = ndim, 64, 8
    for i in range(ndim):
        m.dims[i] = 128
    m.nnz, m.keys, m.values = 53687296, 64, 64   # dummy non-null device pointers (never read)
    f = FilterT()
    f.ndim, f.c_in, f.c_out = ndim, c_in, 8
    for i in range(ndim):
        f.ksize[i] = ks[i]
    f.nnz, f.keys, f.values = 864, 64, 64
    return m, f


def _query(m, f, attn=1, k=104857):
    cap, ws = C.c_int64(), C.c_size_t()
    rc = spc.load().spc_conv_fwd_query(C.byref(m), C.byref(f), attn, k, C.byref(cap), C.byref(ws))
    return rc, cap.value, ws.value


def test_fwd_query_capacity_is_the_density_bound():
    m, f = _c4_structs()
    rc, cap, ws = _query(m, f)
    assert rc == 0
    assert cap == 64 * 8 * 104857        # b * c_out * min(k, V): the rho_up guarantee
    assert ws > 64 * 8 * 128 ** 3 * 8    # candidate runs: 8 B per voxel and output channel
    rc, cap, _ = _query(m, f, attn=0)
    assert rc == 0 and cap == 64 * 8 * 128 ** 3


@pytest.mark.parametrize("mut,code", [
    (lambda m, f: setattr(f, "c_in", 4), 2),                 # c_in mismatch -> SPC_ERR_SHAPE
    (lambda m, f: f.ksize.__setitem__(0, 2), 2),             # even kernel -> SPC_ERR_SHAPE
    (lambda m, f: setattr(m, "ndim", 5), 6),                 # rank 5 -> SPC_ERR_UNSUPPORTED
    (lambda m, f: setattr(m, "ndim", 4), 2),                 # rank 4 map, rank 3 filter -> SPC_ERR_SHAPE
    (lambda m, f: setattr(m, "keys", None), 1),              # NULL keys -> SPC_ERR_INVALID_ARG
    (lambda m, f: setattr(m, "channels", 0), 2),
])
def test_fwd_query_rejects_bad_arguments(mut, code):
    m, f = _c4_structs()
    mut(m, f)
    assert _query(m, f)[0] == code


def test_fwd_query_rejects_k_below_one():
    m, f = _c4_structs()
    assert _query(m, f, attn=1, k=0)[0] == 1
    assert _query(m, f, attn=0, k=0)[0] == 0    # no attention: k unused


def test_bwd_and_pool_queries():
    m, f = _c4_structs()
    ws = C.c_size_t()
    assert spc.load().spc_conv_bwd_query(C.byref(m), C.byref(f), C.byref(m), C.byref(ws)) == 0
    st = (C.c_int64 * 3)(2, 2, 2)
    cap = C.c_int64()
    assert spc.load().spc_maxpool_query(C.byref(m), C.cast(st, C.c_void_p), C.byref(cap), C.byref(ws)) == 0
    assert cap.value == m.nnz
    bad = (C.c_int64 * 3)(2, 0, 2)
    assert spc.load().spc_maxpool_query(C.byref(m), C.cast(bad, C.c_void_p), C.byref(cap), C.byref(ws)) == 2


def test_product_package_does_not_import_oracle():
    import sys

    for mod in list(sys.modules):
        if mod.startswith("paper_1801_10585_b200"):
            src = getattr(sys.modules[mod], "__file__", None)
            if src and src.endswith(".py"):
                text = open(src).read()
                assert "import oracle" not in text and "from oracle" not in text


def _map(ndim, batch, ch, dims, nnz):
    m = MapT()
    m.ndim, m.batch, m.channels = ndim, batch, ch
    for i in range(ndim):
        m.dims[i] = dims[i]
    m.nnz, m.keys, m.values = nnz, 64, 64   # dummy pointers: host-only calls never read them
    return m


def _filt(ndim, ci, co, ks, nnz):
    f = FilterT()
    f.ndim, f.c_in, f.c_out = ndim, ci, co
    for i in range(ndim):
        f.ksize[i] = ks[i]
    f.nnz, f.keys, f.values = nnz, 64, 64
    return f


def test_accumulate_variant_selection_host():
    """AUTO resolves to the scatter variant on sparse layers (C4: 2 % density, 8 channels) and to
    the tensor-core variant on dense-row layers (C5 at 50 %); explicit choices are honoured or
    rejected (G needs c_in <= 32); the G workspace carries the dense input copy."""
    lib = spc.load()
    c4m, c4f = _map(3, 64, 8, (128,) * 3, 21474816), _filt(3, 8, 8, (3, 3, 3), 864)
    assert lib.spc_conv_fwd_variant(C.byref(c4m), C.byref(c4f), 1, 104857, 0) == 1          # S
    assert lib.spc_conv_fwd_variant(C.byref(c4m), C.byref(c4f), 1, 104857, 2) == 2          # forced G
    c5m, c5f = _map(3, 8, 32, (64,) * 3, 33554432), _filt(3, 32, 32, (3, 3, 3), 27648)
    assert lib.spc_conv_fwd_variant(C.byref(c5m), C.byref(c5f), 0, 0, 0) == 2               # G
    wide_m, wide_f = _map(3, 1, 40, (8, 8, 8), 100), _filt(3, 40, 4, (3, 3, 3), 500)
    assert lib.spc_conv_fwd_variant(C.byref(wide_m), C.byref(wide_f), 0, 0, 2) == 0          # invalid
    assert lib.spc_conv_fwd_variant(C.byref(wide_m), C.byref(wide_f), 0, 0, 0) == 1
    cap, ws_s, ws_g = C.c_int64(), C.c_size_t(), C.c_size_t()
    assert lib.spc_conv_fwd_query_ex(C.byref(c5m), C.byref(c5f), 0, 0, 1, C.byref(cap), C.byref(ws_s)) == 0
    assert lib.spc_conv_fwd_query_ex(C.byref(c5m), C.byref(c5f), 0, 0, 2, C.byref(cap), C.byref(ws_g)) == 0
    assert ws_g.value - ws_s.value >= 8 * 64 ** 3 * 32 * 8          # hi + lo dense copy of the input
    assert lib.spc_conv_fwd_query_ex(C.byref(wide_m), C.byref(wide_f), 0, 0, 2, C.byref(cap), C.byref(ws_g)) == 6


def test_training_and_bridge_argument_checks():
    lib = spc.load()
    assert lib.sparse_adagrad_step(None, None, None, -1, None, 1.0, None, 0.1, 1e-8, None) == 1
    reg = _lib.DensityRegT(0.1, 0.05, 0.1, 0.1, 0.1)
    assert lib.sparse_adagrad_step(C.c_void_p(64), C.c_void_p(64), C.c_void_p(64), 10, None, 1.0, C.byref(reg),
                                   0.1, 1e-8, None) == 1                                    # reg without density
    ws = C.c_size_t()
    assert lib.spc_prune_query(1000, C.byref(ws)) == 0 and ws.value > 0
    assert lib.sparse_filter_prune(None, None, None, None, 10, 0.01, None, None, None, None, None, None, 0,
                                   None) == 1
    m = _map(2, 1, 1, (4, 4), 3)
    assert lib.sparse_to_dense(C.byref(m), None, None) == 1


# ------------------------------------------------------------------ memory model / passes (f2)
def test_memory_estimate_matches_oracle():
    import oracle as ora
    for k, r, b, c, rho, bits in [(3, 32, 32, 8, 1 / 32, 64), (3, 256, 32, 8, 1 / 256, 64), (3, 128, 32, 8, 1 / 128, 32),
                                  (2, 28, 256, 8, 0.15, 64), (1, 1000, 3, 5, 0.37, 32), (3, 512, 32, 8, 1 / 512, 64)]:
        got = spc.memory_estimate(k, r, b, c, rho, bits)
        want = ora.memory_estimate(k, r, b, c, rho, bits)
        assert got == want, (k, r, b, c, rho, bits)


def test_memory_estimate_errors():
    lib = spc.load()
    d = C.c_double()
    assert lib.spc_memory_estimate(3, 256, 32, 8, 1 / 256, 32, C.byref(d), None, None) == 6   # 2^32 cells
    assert lib.spc_memory_estimate(3, 256, 32, 8, 1 / 256, 16, C.byref(d), None, None) == 1
    assert lib.spc_memory_estimate(3, 0, 32, 8, 0.1, 64, None, None, None) == 1
    assert lib.spc_memory_estimate(3, 8, 1, 1, 0.0, 64, None, None, None) == 1
    assert lib.spc_memory_estimate(5, 8, 1, 1, 0.5, 64, None, None, None) == 1
    assert lib.spc_memory_estimate(4, 8, 1, 1, 0.5, 64, None, None, None) == 0   # rank 4


def test_fwd_pass_workspace_shrinks_with_samples_per_pass():
    """The per-(b, oc) buffers scale with samples_per_pass (C4: 64 samples -> 1)."""
    lib = spc.load()
    m, f = _c4_structs()
    cap, ws_all, ws_one, ws_full = C.c_int64(), C.c_size_t(), C.c_size_t(), C.c_size_t()
    assert lib.spc_conv_fwd_query_pass(C.byref(m), C.byref(f), 1, 104857, 0, C.byref(cap), C.byref(ws_all)) == 0
    assert lib.spc_conv_fwd_query_pass(C.byref(m), C.byref(f), 1, 104857, 1, C.byref(cap), C.byref(ws_one)) == 0
    assert lib.spc_conv_fwd_query_ex(C.byref(m), C.byref(f), 1, 104857, 1, None, C.byref(ws_full)) == 0
    assert ws_all.value == ws_full.value
    assert ws_one.value * 40 < ws_all.value
    assert cap.value == 64 * 8 * 104857
    assert lib.spc_conv_fwd_query_pass(C.byref(m), C.byref(f), 1, 104857, -1, C.byref(cap), C.byref(ws_one)) == 1


def test_keys_narrow_rejects_large_key_space():
    lib = spc.load()
    m, _ = _c4_structs()
    m.batch, m.channels = 256, 256   # 2^21 * 2^16 = 2^37 keys
    assert lib.sparse_keys_narrow(C.byref(m), C.c_void_p(64), None) == 6


def test_32bit_keys_need_a_small_key_space():
    """key_bits = 32 is accepted only when batch*channels*prod(dims) <= 2^32 (Table 1's "-")."""
    m, f = _c4_structs()
    m.key_bits = 32                      # 64 * 8 * 128^3 = 2^30: fits
    assert _query(m, f)[0] == 0
    m.dims[0] = m.dims[1] = m.dims[2] = 1024   # 64 * 8 * 2^30 > 2^32
    assert _query(m, f)[0] == 6
    m.key_bits = 16
    assert _query(m, f)[0] == 1
