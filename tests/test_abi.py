"""CPU checks of the C-ABI boundary: the library builds/loads, exports every function
include/sart.h declares, and the ctypes mirrors have the C layout (sizes and offsets
checked against gcc).  No compute call is made (there is no GPU here)."""
import ctypes as C
import os
import re
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sart.h")


def declared_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(sart_\w+)\s*\(", src, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2505_13326_b200 import build
    build.build(verbose=False)
    from paper_2505_13326_b200 import sart
    return sart.load_library()


def test_every_declared_symbol_is_exported(lib):
    names = declared_functions()
    assert len(names) >= 10
    for n in names:
        assert hasattr(lib, n), n
    from paper_2505_13326_b200 import sart
    assert sorted(sart.EXPORTED) == names


def test_strerror_without_gpu(lib):
    assert lib.sart_strerror(-1) == b"SART_EINVAL"
    assert lib.sart_strerror(0) == b"SART_OK"


def test_struct_layout_matches_header():
    from paper_2505_13326_b200 import sart as S
    structs = {"sart_config": S.SartConfig, "sart_script": S.SartScript, "sart_request": S.SartRequest,
               "sart_stats": S.SartStats, "sart_result": S.SartResult, "sart_state": S.SartState,
               "sart_profile": S.SartProfile, "sart_trace_row": S.SartTraceRow}
    lines = ["#include <stdio.h>", "#include <stddef.h>", f'#include "{HEADER}"', "int main(void){"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    lines.append("return 0;}")
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        open(c, "w").write("\n".join(lines))
        exe = os.path.join(d, "t")
        subprocess.check_call(["gcc", c, "-o", exe])
        out = subprocess.check_output([exe]).decode().split("\n")
    for line in out:
        if not line:
            continue
        cname, f, v = line.split()
        py = structs[cname]
        if f == "size":
            assert C.sizeof(py) == int(v), cname
        else:
            assert getattr(py, f).offset == int(v), (cname, f)


def test_product_path_has_no_oracle_or_fallback():
    """The product package never imports the oracle; the C-ABI binding imports no torch
    (torch.distributed is plumbing for dist.py only)."""
    pkg = os.path.join(ROOT, "paper_2505_13326_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert "import oracle" not in src and "from oracle" not in src, fn
            if fn in ("sart.py", "__init__.py", "build.py"):
                assert "import torch" not in src, fn
