"""CPU: the drop-in boundary exists and is complete.

* the sm_100a library loads and exports every function include/mpzch_b200.h declares
  (and the Python mirror binds exactly that surface);
* the library holds sm_100a SASS (cuobjdump) and no CPU path;
* host-side mirrors of the reference's value types behave like the reference.
No CUDA call is made here.
"""
import os
import re
import shutil
import subprocess

import pytest

import paper_2602_17050_b200 as mz

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mpzch_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mpzch_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_reference_surface():
    fns = declared_functions()
    for must in ("mpzch_table_create", "mpzch_process_batch", "mpzch_process_batch_device",
                 "mpzch_lookup", "mpzch_lookup_or_insert", "mpzch_copy_identities",
                 "mpzch_make_cursor", "mpzch_dirty_rows_since", "mpzch_last_error"):
        assert must in fns


def test_library_exports_every_declared_symbol():
    lib = mz.load_library()
    missing = [f for f in declared_functions() if not hasattr(lib, f)]
    assert not missing, missing


def test_python_binding_covers_the_header():
    assert set(declared_functions()) == set(mz._SIGS)


def test_build_info_names_sm100a():
    assert mz.build_info().startswith("sm_100a")


def test_library_holds_sm100a_sass():
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not on PATH")
    out = subprocess.run(["cuobjdump", "-lelf", mz.lib_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_table_create_without_gpu_fails_loudly():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except Exception:
        pass
    with pytest.raises(mz.MpzchError):
        mz.MpzchTable(mz.TableConfig.even(64, 2, 4, 7))


def test_policy_mirror():
    with pytest.raises(mz.InvalidArgument, match="default TTL must be strictly positive"):
        mz.EvictionPolicy.ttl(mz.TtlPolicy(0))
    with pytest.raises(mz.InvalidArgument, match=r"\(feature 3\)"):
        mz.EvictionPolicy.ttl(mz.TtlPolicy(5, {3: 0}))
    p = mz.EvictionPolicy.ttl(mz.TtlPolicy(259200, {7: 86400}))
    assert p.meta_for(500, 7) == 86900 and p.meta_for(500, 8) == 259700
    assert mz.EvictionPolicy.lru().meta_for(42) == 42
    with pytest.raises(mz.OverflowError_):
        mz.EvictionPolicy.ttl(mz.TtlPolicy(1000)).meta_for((1 << 64) - 11)


def test_even_layout_mirror():
    assert mz.even_capacities(10, 4) == [3, 3, 2, 2]
    with pytest.raises(mz.InvalidArgument):
        mz.even_capacities(3, 4)
    with pytest.raises(mz.InvalidArgument):
        mz.even_capacities(8, 0)
