"""INTEGRATION.md's reference-side binding, executed: the ctypes stub a maintainer
would add to hewisard.tfhe (hw/tfhe.py:301-319 ext_product_batch) is extracted from
the markdown and run on the reference-generated golden fixtures, with the
reference's own operand format (uint64 words carrying x << 32)."""

import os
import re
from types import SimpleNamespace

import numpy as np
import pytest

from conftest import REPO, golden
from paper_2403_20190_b200 import _lib
from paper_2403_20190_b200.params import GadgetSpec

pytestmark = pytest.mark.gpu


class TfheError(ValueError):
    pass


def _stub():
    text = open(os.path.join(REPO, "INTEGRATION.md")).read()
    sec = text[text.index("## 2. Bind the C ABI"):]
    code = re.search(r"```python\n(.*?)```", sec, re.S).group(1)
    os.environ["HWB_LIB"] = _lib.LIB_PATH
    ns = {"TfheError": TfheError}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)
    return ns["ext_product_batch_hwb"]


@pytest.mark.parametrize("tag,N,lv,w", [("cfg2", 1024, 3, 7), ("cfg1", 1024, 2, 8), ("cfg4", 2048, 2, 10)])
def test_integration_stub_on_golden(tag, N, lv, w):
    fn = _stub()
    g = golden("ext_product.npz")
    params = SimpleNamespace(n=N, gadget=GadgetSpec(lv, w))
    emb = lambda x: np.asarray(x, dtype=np.uint64) << np.uint64(32)        # noqa: E731
    out = fn(params, emb(g[f"{tag}_G"]), emb(g[f"{tag}_cts"]))
    assert out.dtype == np.uint64 and not np.any(out & np.uint64(0xFFFFFFFF))
    assert np.array_equal((out >> np.uint64(32)).astype(np.uint32), g[f"{tag}_out"])
    out_b = fn(params, emb(g[f"{tag}_G"][:1]), emb(g[f"{tag}_cts"]))
    assert np.array_equal((out_b >> np.uint64(32)).astype(np.uint32), g[f"{tag}_out_bcast"])


def test_integration_stub_raises_tfhe_error():
    fn = _stub()
    g = golden("ext_product.npz")
    params = SimpleNamespace(n=1024, gadget=GadgetSpec(2, 16))          # outside the exact NTT envelope
    emb = lambda x: np.asarray(x, dtype=np.uint64) << np.uint64(32)        # noqa: E731
    with pytest.raises(TfheError):
        fn(params, emb(g["ins_G"]), emb(g["ins_cts"]))
