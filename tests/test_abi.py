"""CPU tier: the C-ABI library builds, loads and exports every symbol include/faser/*.h
declares; ctypes struct layouts match the compiled ones; the product refuses to run
without a GPU (no silent CPU fallback)."""
import ctypes as C
import glob
import os
import re

import pytest

from conftest import ROOT, has_gpu
from paper_2604_20503_b200 import abi, engine


def declared_symbols():
    syms = set()
    for h in glob.glob(os.path.join(ROOT, "include", "faser", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        syms |= set(re.findall(r"\b(faser_[a-z0-9_]+)\s*\(", src))
    return sorted(syms)


def test_library_exports_every_declared_symbol():
    L = engine.lib()
    syms = declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing


def test_struct_sizes_match_header():
    L = engine.lib()
    out = (C.c_int64 * 15)()
    assert L.faser_abi_struct_sizes(out, 15) == 0
    py = [abi.ToyParams, abi.ExitPolicy, abi.GatePlan, abi.GateEntry, abi.OverlapPlan,
          abi.LatencyParams, abi.LatencyModel, abi.VerifyOutcome, abi.ModelDesc, abi.EngineCfg,
          abi.StepPlan, abi.RoundResult, abi.LlamaShape, abi.TimelineEvent, abi.TimelineInfo]
    assert [C.sizeof(t) for t in py] == list(out)
    assert L.faser_abi_version() == 3


def test_library_is_sm100a_cubin():
    # the fatbin must carry sm_100a SASS (not only PTX, not an older arch)
    import subprocess
    r = subprocess.run(["cuobjdump", "--list-elf", engine.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in r.stdout, r.stdout + r.stderr


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU failure path")
def test_no_gpu_fails_loudly():
    with pytest.raises(engine.FaserError) as ei:
        engine.ServingEngine()
    assert ei.value.status == abi.ECUDA
    with pytest.raises(engine.FaserError) as ei:
        engine.LayeredToyLM().target_next([[1, 2, 3]])
    assert ei.value.status == abi.ECUDA


def test_argument_validation_before_device():
    toy = engine.LayeredToyLM(abi.ToyParams.default(vocab=1))
    with pytest.raises(engine.FaserError) as ei:
        toy.target_next([[0]])
    assert ei.value.status == abi.EINVAL
    with pytest.raises(engine.FaserError) as ei:
        engine.LayeredToyLM().target_next([[]])
    assert ei.value.status == abi.EINVAL
