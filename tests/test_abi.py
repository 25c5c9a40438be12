"""CPU-side checks of the boundary: the C-ABI library loads without a GPU and
exports every function include/entmaxkv.h declares; no compute calls here."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "entmaxkv.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(entmaxkv_\w+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for n in ["entmaxkv_append_kv", "entmaxkv_rebuild_page_stats", "entmaxkv_score_pages", "entmaxkv_select",
              "entmaxkv_sparse_attend", "entmaxkv_full_attend", "entmaxkv_decode", "entmaxkv_workspace_size"]:
        assert n in names


def test_library_exports_every_declared_symbol():
    from paper_2605_21649_b200 import binding
    lib = binding.lib()          # loads without a GPU
    for n in declared_functions():
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", binding.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (entmaxkv_\w+)", out))
    assert set(declared_functions()) <= exported
    assert set(binding.EXPORTED) == set(declared_functions())


def test_library_is_sm100a_and_uses_bulk_copies():
    from paper_2605_21649_b200 import binding
    out = subprocess.run(["cuobjdump", "-lelf", binding.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", binding.LIB_PATH], capture_output=True, text=True).stdout
    assert "UBLKCP" in sass          # cp.async.bulk (TMA) in the K-tile loader


def test_version_string():
    from paper_2605_21649_b200 import binding
    assert "sm_100a" in binding.version()


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2605_21649_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "liboracle" not in txt, f
