"""C-ABI boundary checks that need no GPU: the library loads, exports every symbol the header
declares, and the ctypes signatures/struct layout agree with include/tomobpdn_b200.h."""

import ctypes
import os
import re

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
HEADER = os.path.join(ROOT, "include", "tomobpdn_b200.h")


def _declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tb_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_1805_01759_b200 import _lib

    if not os.path.exists(_lib.LIB_PATH):
        from paper_1805_01759_b200 import build

        build.build()
    return _lib.load()


def test_header_declares_entry_points():
    names = _declared()
    for n in ("tb_ctx_create", "tb_solve", "tb_select", "tb_default_lambda", "tb_derive_seeds", "tb_spectral_sq_norms", "tb_set_partition"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    for name in _declared():
        assert hasattr(lib, name), name


def test_ctypes_signatures_cover_header(lib):
    from paper_1805_01759_b200 import _lib

    assert sorted(_lib.SIGNATURES) == _declared()
    text = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    for name, (_, args) in _lib.SIGNATURES.items():
        m = re.search(name + r"\s*\(([^;]*)\)\s*;", text, flags=re.S)
        assert m, name
        params = [p for p in m.group(1).split(",") if p.strip() and p.strip() != "void"]
        assert len(params) == len(args), (name, len(params), len(args))


def test_config_struct_layout(tmp_path):
    """The ctypes mirror of tb_solver_config has the C compiler's size and field offsets."""
    import subprocess

    from paper_1805_01759_b200 import _lib

    fields = [f for f, _ in _lib.SolverConfigC._fields_]
    src = tmp_path / "layout.c"
    src.write_text(
        '#include <stddef.h>\n#include <stdio.h>\n#include "tomobpdn_b200.h"\nint main(void) {\n'
        + '  printf("%zu\\n", sizeof(tb_solver_config));\n'
        + "".join(f'  printf("%zu\\n", offsetof(tb_solver_config, {f}));\n' for f in fields)
        + "  return 0;\n}\n"
    )
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    vals = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    assert ctypes.sizeof(_lib.SolverConfigC) == vals[0]
    assert [getattr(_lib.SolverConfigC, f).offset for f in fields] == vals[1:]


def test_version_and_errors_without_gpu(lib):
    assert lib.tb_version().startswith(b"tomobpdn_b200")
    from paper_1805_01759_b200 import _lib
    from paper_1805_01759_b200.exceptions import ConfigurationError

    # argument validation happens before any device work
    h = ctypes.c_void_p()
    code = lib.tb_ctx_create(0, None, 4, 4, ctypes.byref(h))
    assert code == _lib.TB_ERR_INVALID
    with pytest.raises(ConfigurationError):
        _lib.check(code)
    assert lib.tb_derive_seeds(1, 0, -1, None, None) == _lib.TB_ERR_INVALID
