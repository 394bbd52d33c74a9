"""CPU-side checks of the C-ABI library: it builds/loads, exports every symbol that
include/moe_dts.h declares, and performs host-side validation (no GPU needed: these
paths return before any kernel launch)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "moe_dts.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|size_t|uint64_t|const char\*)\s+(moe_\w+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def L():
    from paper_2112_14397_b200 import build
    build.build()
    from paper_2112_14397_b200 import _lib
    return _lib


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for name in ("moe_dts_spawn", "moe_dts_gate", "moe_dispatch", "moe_expert_ffn", "moe_combine",
                 "moe_combine_bwd", "moe_expert_ffn_bwd", "moe_dts_gate_bwd", "moe_dispatch_bwd",
                 "moe_create", "moe_destroy", "moe_last_error", "moe_workspace_bytes",
                 "moe_set_workspace", "moe_check", "moe_balance_loss"):
        assert name in syms, name


def test_library_exports_every_declared_symbol(L):
    lib = ctypes.CDLL(L.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(lib, name), f"{name} declared in moe_dts.h but not exported"
    assert set(declared_symbols()) == set(L.SIGNATURES), "binding signatures out of sync with header"


def test_library_is_sm100a_cubin():
    from paper_2112_14397_b200 import build
    lib = build.build()
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_create_validation(L):
    with pytest.raises(L.MoEError) as e:
        L.moe_create(128, 63, 256, 4, L.MOE_BF16)
    assert e.value.code == 2 and "63" in str(e.value)
    with pytest.raises(L.MoEError) as e:
        L.moe_create(128, 64, 256, 6, L.MOE_BF16, nccl_comm=1, rank=0, world=4)
    assert e.value.code == 2
    with pytest.raises(L.MoEError) as e:
        L.moe_create(128, 64, 256, 4, 7)
    assert e.value.code == 3
    with pytest.raises(L.MoEError) as e:
        L.moe_create(128, 64, 256, 4, L.MOE_F32, world=2)     # world > 1 without a comm
    assert e.value.code == 1
    ctx = L.moe_create(256, 64, 256, 4, L.MOE_F32)
    assert L.moe_workspace_bytes(ctx) > 0
    L.moe_destroy(ctx)
    # bf16 dims need only be multiples of 8 (16-byte rows); 4 is refused
    ctx = L.moe_create(256, 72, 200, 4, L.MOE_BF16)
    L.moe_destroy(ctx)
    with pytest.raises(L.MoEError) as e:
        L.moe_create(128, 68, 256, 4, L.MOE_BF16)
    assert e.value.code == 2 and "68" in str(e.value)


def test_calls_without_workspace_and_bad_scalars(L):
    ctx = L.moe_create(256, 64, 256, 4, L.MOE_F32)
    # no workspace: every compute call refuses before touching the device
    with pytest.raises(L.MoEError) as e:
        L.moe_dts_gate(ctx, 1, 1, None, 1.0, 0.1, 0, 1, 1, 1, 1, stream=0)
    assert e.value.code == 8
    lib = L.lib()
    # fake 256-aligned pointer: validation only reads the value, never dereferences
    fake = 1 << 20
    rc = lib.moe_set_workspace(ctx, fake, 1)
    assert rc == 8 and "needed" in L.last_error()
    L.moe_destroy(ctx)


def test_status_codes_match_header():
    src = open(HEADER).read()
    for code, name in {0: "MOE_OK", 1: "MOE_EINVAL", 2: "MOE_ESHAPE", 6: "MOE_ENONFINITE",
                       7: "MOE_ECAPACITY", 8: "MOE_EWORKSPACE"}.items():
        assert re.search(rf"{name}\s*=\s*{code}\b", src)


def _prototypes():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    out = {}
    for m in re.finditer(r"^\s*(?:int|size_t|uint64_t|const char\*)\s+(moe_\w+)\s*\(([^)]*)\)\s*;", src, flags=re.M):
        args = m.group(2).strip()
        out[m.group(1)] = 0 if args in ("", "void") else args.count(",") + 1
    return out


def test_binding_arity_matches_header(L):
    # every ctypes signature passes exactly the header's number of arguments (ABI v2 changed
    # several: db2 out of combine_bwd, Wg / dx into gate_bwd, accumulate into dispatch_bwd)
    protos = _prototypes()
    assert set(protos) == set(L.SIGNATURES)
    for name, n in protos.items():
        assert len(L.SIGNATURES[name][1]) == n, (name, n, len(L.SIGNATURES[name][1]))
    assert L.moe_abi_version() == 2
