"""CPU-side checks of the drop-in boundary: the C ABI library loads, exports
every symbol include/fntgpu.h declares with the struct layouts the binding
uses, and refuses to compute without a GPU (no CPU fallback)."""

import ctypes as C
import re

import numpy as np
import pytest

from conftest import HAS_CUDA, ROOT


def header_symbols():
    text = (ROOT / "include" / "fntgpu.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(fntgpu_\w+)\s*\(", text, re.M)))


def test_library_builds_and_exports_every_declared_symbol():
    from paper_2405_04253_b200 import _lib
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _lib.SIGNATURES, f"binding lacks {s}"
    assert lib.fntgpu_abi_version() == _lib.ABI_VERSION


def test_struct_layouts_match_binding():
    from paper_2405_04253_b200 import _lib
    lib = _lib.load()
    out = (C.c_int64 * 7)()
    assert lib.fntgpu_struct_sizes(out, 7) == 7
    mine = [C.sizeof(s) for s in (_lib.CdcTaps, _lib.CdcIO, _lib.DecimIO, _lib.AeqParams,
                                  _lib.AeqState, _lib.AeqIO, _lib.TdAeqIO)]
    assert list(out) == mine


def test_plan_validation_codes_without_gpu():
    """Argument validation happens before any device work (InvalidPlanError reasons)."""
    from paper_2405_04253_b200 import _lib
    lib = _lib.load()
    h = C.c_void_p()
    assert lib.fntgpu_plan_create(4, 63, 2, C.byref(h)) == _lib.EPLAN_LENGTH
    assert lib.fntgpu_plan_create(4, 64, 70000, C.byref(h)) == _lib.EPLAN_RADIX
    assert lib.fntgpu_plan_create(4, 64, 2, C.byref(h)) == _lib.EPLAN_SUBORD
    assert lib.fntgpu_plan_create(4, 64, 3, C.byref(h)) == _lib.EPLAN_ORDER
    assert lib.fntgpu_plan_create(5, 64, 3, C.byref(h)) == _lib.EPLAN_MODULUS
    assert lib.fntgpu_plan_create(4, 6, 2, C.byref(h)) == _lib.EPLAN_LENGTH
    assert "power of two" in _lib.last_error()


def test_cdc_kernel_selector_validation_without_gpu():
    """fntgpu_cdc_taps.kernel: 0 auto, 1 shift-add, 2 mma.sync matrix form, 3 tcgen05
    matrix form; anything else is rejected before any device work. The Python
    selector maps the same names (cdc.set_cdc_kernel)."""
    from paper_2405_04253_b200 import _lib, cdc
    lib = _lib.load()
    taps = _lib.CdcTaps()
    taps.n_taps = 32
    io = _lib.CdcIO()
    for bad in (-1, 4, 99):
        taps.kernel = bad
        assert lib.fntgpu_cdc64_process(C.byref(taps), C.byref(io), None) == _lib.EINVAL
        assert "kernel selector" in _lib.last_error()
    assert cdc.CDC_KERNELS == {"auto": 0, "shift": 1, "tc": 2, "umma": 3}
    prev = cdc.set_cdc_kernel("umma")
    try:
        with pytest.raises(ValueError):
            cdc.set_cdc_kernel("cufft")
    finally:
        cdc.set_cdc_kernel(prev)
    text = (ROOT / "include" / "fntgpu.h").read_text()
    for name, code in (("AUTO", 0), ("SHIFT", 1), ("TC", 2), ("UMMA", 3)):
        assert re.search(rf"#define FNTGPU_CDC_KERNEL_{name} {code}\b", text)


@pytest.mark.skipif(HAS_CUDA, reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    import paper_2405_04253_b200 as P
    from paper_2405_04253_b200 import _lib
    with pytest.raises(_lib.FntGpuError):
        P.fnt(P.default_plans()["cdc64"], np.zeros(64))
    with pytest.raises(_lib.FntGpuError):
        P.quantize_real(np.zeros(4), P.QuantSpec(5, 8.0))
    assert _lib.load().fntgpu_device_count() == 0


def test_api_surface_mirrors_reference_names():
    """Every name of fntdsp.__all__ (fntdsp/__init__.py:27-42) is exported."""
    import paper_2405_04253_b200 as P
    ref_all = [
        "COUNTER", "ComplexityReport", "MultCounter", "tab1_formula",
        "FermatParams", "add", "sub", "neg", "mul", "mul_pow2", "reduce", "sqrt2",
        "encode_signed", "decode_signed", "encode_signed_array", "decode_signed_array",
        "BudgetReport", "QuantSpec", "QuantizedBlock", "check_overflow",
        "dequantize", "quantize", "quantize_real", "recombine", "split_taps",
        "InvalidPlanError", "TransformPlan", "default_plans", "make_plan",
        "fnt", "ifnt", "cyclic_convolve_real", "cyclic_convolve_complex",
        "convolve_signed_real", "convolve_signed_complex",
        "BudgetError", "CdcConfig", "FntCdcEngine", "design_cd_taps",
        "fd_cdc_float", "td_cdc_float", "required_taps",
        "AeqConfig", "FntAeq", "RvMimoTaps", "qam16_radii", "td_aeq_float",
        "HD_FEC_BER", "LinkConfig", "Metrics", "fec_crossing_snr",
        "penalty_at_fec", "run_link", "run_single",
    ]
    for n in ref_all:
        assert hasattr(P, n), n
    assert sorted(P.__all__) == sorted(ref_all)


def test_integration_md_binding_stub_matches_abi(monkeypatch):
    """The ctypes stub INTEGRATION.md tells a maintainer to add declares the same
    struct layouts as the C header (sizes from fntgpu_struct_sizes)."""
    import re
    from conftest import ROOT
    text = (ROOT / "INTEGRATION.md").read_text()
    code = re.search(r"```python\n(import ctypes as C.*?)```", text, re.S).group(1)
    monkeypatch.chdir(ROOT)
    ns: dict = {}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)
    from paper_2405_04253_b200 import _lib
    lib = _lib.load()
    out = (C.c_int64 * 7)()
    lib.fntgpu_struct_sizes(out, 7)
    assert C.sizeof(ns["CdcTaps"]) == out[0]
    assert C.sizeof(ns["CdcIO"]) == out[1]
