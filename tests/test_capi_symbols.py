"""CPU-side checks of the C-ABI boundary: the in-tree library loads and exports
every symbol include/gsr_cuda.h declares; without a GPU, creating a context
fails loudly (status RESOURCE) instead of falling back to the CPU."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "gsr_cuda.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(gsrc_\w+)\s*\(", src, re.M)))


def test_library_exports_every_header_symbol():
    from paper_2603_27156_b200 import _capi
    lib = _capi.lib()
    decl = _declared()
    assert len(decl) >= 30
    missing = [s for s in decl if not hasattr(lib, s)]
    assert not missing, missing
    assert sorted(_capi.EXPORTS) == decl


def test_library_is_sm100a():
    import subprocess
    from paper_2603_27156_b200 import _capi
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _capi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2603_27156_b200 import Context, ResourceError
    with pytest.raises(ResourceError):
        Context(0)


def test_param_layout_matches_oracle(oracle):
    import numpy as np
    from paper_2603_27156_b200 import model
    from paper_2603_27156_b200 import synth
    g = synth.generate_graph(synth.SynthConfig(n=50, hub_fraction=0.0, seed=0))
    og = oracle.Graph(g.row_ptr, g.col_idx, norm=1)
    for mode, C in ((0, 2), (1, 4), (2, 2)):
        net = oracle.Net(og, mode, 3, 32, C, 2, 5)
        lay = model.param_layout(mode, 3, 32, C, 5)
        assert lay["P"] == net.P
        p = model.init_params(mode, 3, 32, C, 5, seed=1)
        net.set_params(p)
        assert np.array_equal(net.params(), p)
