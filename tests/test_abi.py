"""C-ABI library checks that need no GPU: the in-tree libsdnn.so loads, exports every entry point
include/sdnn.h declares, and its host-side validation / planning behave as documented."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2101_07948_b200 as sdnn
import sdnn_synth as synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "sdnn.h")).read()
    return sorted(set(re.findall(r"^SDNN_API\s+[\w\s\*]+?\b(sdnn_\w+)\s*\(", txt, flags=re.M)))


def test_header_declares_expected_entry_points():
    syms = header_symbols()
    assert "sdnn_prepare" in syms and "sdnn_spmm" in syms and "sdnn_spmm_host" in syms
    assert sorted(sdnn.EXPORTS) == syms


def test_library_exports_every_header_symbol():
    lib = ctypes.CDLL(sdnn.LIB_PATH)
    for s in header_symbols():
        assert hasattr(lib, s), s


def test_status_strings_and_version():
    assert sdnn.abi_version() == 1
    for code, name in sdnn.STATUS.items():
        assert sdnn._lib.sdnn_status_string(code).decode() == name


def _err(fn):
    with pytest.raises(sdnn.SdnnError) as ei:
        fn()
    return ei.value


@pytest.mark.parametrize("bad,code,frag", [
    (dict(row_ptr=[1, 1, 2]), 2, "csr_ptr[0]"),
    (dict(row_ptr=[0, 2, 1]), 2, "decreases at row 1"),
    (dict(col_idx=[1, 1], row_ptr=[0, 2, 2]), 2, "row 0"),  # duplicate column
    (dict(col_idx=[1, 0], row_ptr=[0, 2, 2]), 2, "row 0"),  # unsorted
    (dict(col_idx=[0, 5]), 2, "out of range in row 1"),
])
def test_invalid_csr_rejected(bad, code, frag):
    args = dict(row_ptr=[0, 1, 2], col_idx=[0, 1], vals=[1.0, 2.0])
    args.update(bad)
    rp = np.array(args["row_ptr"], np.int32)
    ci = np.array(args["col_idx"], np.int32)
    v = np.ones(len(ci), np.float32)
    e = _err(lambda: sdnn.Plan(rp, ci, v, 2, 3))
    assert e.status == code and frag in str(e)
    e = _err(lambda: sdnn.permutation(rp, ci, 2, 3))
    assert e.status == code


def test_invalid_arguments():
    rp = np.array([0, 1], np.int32)
    ci = np.array([0], np.int32)
    v = np.ones(1, np.float32)
    assert _err(lambda: sdnn.Plan(rp, ci, v, 1, 0)).status == 1
    assert _err(lambda: sdnn.Plan(rp, ci, v, 1, 1, panel_rows=5)).status == 1
    assert _err(lambda: sdnn.Plan(rp, ci, v, 1, 1, k_chunk=12)).status == 1
    assert _err(lambda: sdnn.Plan(rp, ci, v, 1, 1, cta_panels=17)).status == 1


def test_explicit_zero_values_are_structural():
    # reading C6: a stored 0.0 is kept in the pattern (Alg. 1 and the packed stream see it)
    rp = np.array([0, 2, 3], np.int32)
    ci = np.array([0, 2, 2], np.int32)
    v = np.array([0.0, 1.0, 0.0], np.float32)
    pl = sdnn.Plan(rp, ci, v, 2, 3)
    assert pl.info()["nnz"] == 3


def test_prepare_without_gpu_fails_cleanly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    p = synth.config_problem("c1", N=4)
    e = _err(lambda: sdnn.Handle.from_problem(p))
    assert e.status in (5, 3)  # SDNN_ERR_CUDA (no device) — never a silent CPU fallback


def test_header_is_plain_c99(tmp_path):
    """include/sdnn.h is a C ABI: it must compile as C99 with -pedantic -Werror (no C++ types)."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = tmp_path / "t.c"
    src.write_text('#include "sdnn.h"\nint main(void) { sdnn_info i; sdnn_perm_opts o; (void)i; (void)o; '
                   'return (int)SDNN_OK; }\n')
    subprocess.check_call(["gcc", "-std=c99", "-Wall", "-Wextra", "-pedantic", "-Werror", "-I",
                           os.path.join(root, "include"), "-c", str(src), "-o", str(tmp_path / "t.o")])


def test_c_program_links_and_plans(tmp_path):
    """A plain C program links libsdnn.so and runs the host-only API (Algorithm 1 and planning, no
    GPU): the worked Alg. 1 trace of SPEC S:310 ({1}, {0,1,2}, {1,2} → [1, 2, 0])."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.join(root, "paper_2101_07948_b200")
    src = tmp_path / "p.c"
    src.write_text(r"""
#include <stdio.h>
#include "sdnn.h"
int main(void) {
  const int32_t rp[4] = {0, 1, 4, 6}, ci[6] = {1, 0, 1, 2, 1, 2};
  const float v[6] = {1, 1, 1, 1, 1, 1};
  int32_t order[3];
  if (sdnn_permutation(rp, ci, 3, 3, order) != SDNN_OK) return 2;
  sdnn_plan p = NULL;
  if (sdnn_plan_create(rp, ci, v, 3, 3, NULL, &p) != SDNN_OK) return 3;
  sdnn_info info;
  info.struct_size = sizeof info;
  if (sdnn_plan_get_info(p, &info) != SDNN_OK || info.nnz != 6) return 4;
  sdnn_plan_destroy(p);
  printf("%d %d %d\n", order[0], order[1], order[2]);
  return 0;
}
""")
    exe = tmp_path / "p"
    subprocess.check_call(["gcc", "-std=c99", "-I", os.path.join(root, "include"), str(src), "-L", libdir, "-lsdnn",
                           "-Wl,-rpath," + libdir, "-o", str(exe)])
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    assert out == ["1", "2", "0"]
