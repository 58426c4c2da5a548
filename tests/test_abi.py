"""The C-ABI library loads, exports every symbol include/speed_c.h declares,
maps errors to the reference's status codes, and refuses device work loudly
when no B200 is visible (no CPU fallback). Runs without a GPU."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2308_14129_b200 as sp
from paper_2308_14129_b200._lib import LIB_PATH, MISSING, lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "speed_c.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(spd_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported():
    names = declared()
    assert len(names) > 60
    missing = [n for n in names if not hasattr(lib, n)]
    assert missing == [] and MISSING == []


def test_library_is_in_tree_and_versioned():
    assert os.path.dirname(LIB_PATH) == os.path.join(ROOT, "paper_2308_14129_b200")
    assert b"sm_100a" in lib.spd_version()


def test_status_codes_follow_the_cli_convention():
    out = np.zeros(4, sp.EDGE_DTYPE)
    st = lib.spd_gen_powerlaw(1, 4, 2.5, 1, out.ctypes.data_as(C.c_void_p), None, None)
    assert st == 2 and lib.spd_last_error_code() == b"InvalidParams"
    # a thread-local error slot is cleared by the next successful call
    assert lib.spd_gen_powerlaw(10, 4, 2.5, 1, out.ctypes.data_as(C.c_void_p), None, None) == 0
    assert lib.spd_last_error_code() == b""


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-device failure mode")
def test_device_paths_fail_loudly_without_a_gpu():
    with pytest.raises(sp.InternalError) as ei:
        sp.MemoryStore(4, 2)
    assert ei.value.code == "CudaError"
    s = sp.gen_powerlaw(50, 400, 2.5, 1)
    subs = sp.induce_subgraphs(s, [[0]] * s.node_count, 1)
    with pytest.raises(sp.InternalError) as ei:
        sp.TGNTrainer(sp.TGNConfig(d_mem=8, d_time=8, d_edge=4, batch_size=16), subs)
    assert ei.value.code == "CudaError"


def test_tgn_config_validation_is_data_error():
    s = sp.gen_powerlaw(50, 400, 2.5, 1)
    subs = sp.induce_subgraphs(s, [[0]] * s.node_count, 1)
    with pytest.raises(sp.DataError) as ei:
        sp.TGNTrainer(sp.TGNConfig(d_mem=10, d_time=8, d_edge=4, batch_size=16), subs)
    assert ei.value.code == "InvalidParams"
    # shapes outside the attention kernels' register tiling are rejected up front
    for bad in (dict(n_neighbors=17), dict(n_heads=8, d_mem=16, d_time=16),
                dict(d_mem=200, d_time=100), dict(d_mem=100, d_time=100, d_edge=384)):
        kw = dict(d_mem=8, d_time=8, d_edge=4, batch_size=16)
        kw.update(bad)
        with pytest.raises(sp.DataError) as ei:
            sp.TGNTrainer(sp.TGNConfig(**kw), subs)
        assert ei.value.code == "InvalidParams", bad


def test_feature_generator_host_matches_oracle():
    from oracle import tgn_oracle as T
    eids = np.array([0, 5, 123456789, 2 ** 40], np.uint64)
    got = sp.edge_features_bf16(2, eids, 186, 192)
    f32 = (got.astype(np.uint32) << 16).view(np.float32)
    want = T.edge_features(2, eids, 186)
    assert np.array_equal(f32[:, :186], want) and (f32[:, 186:] == 0).all()
