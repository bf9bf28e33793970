"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/radsort.h declares, and its pure host functions behave."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "radsort.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(radsort_[a-z_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    import paper_1703_00687_b200 as rs

    lib = ctypes.CDLL(rs.LIB_PATH)
    declared = header_functions()
    assert "radsort_sort" in declared and "radsort_sort_multi" in declared and "radsort_init" in declared
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(rs.EXPORTS) == declared


def test_library_is_sm100a():
    import subprocess

    import paper_1703_00687_b200 as rs

    out = subprocess.run(["cuobjdump", "--list-elf", rs.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_errors():
    import paper_1703_00687_b200 as rs

    assert "radsort" in rs.version()
    for s in range(8):
        assert rs.lib.radsort_error_string(s)


def test_locate_bucket_host_logic():
    import paper_1703_00687_b200 as rs

    h = np.zeros(256, dtype=np.uint64)
    h[3], h[7], h[255] = 5, 10, 1
    assert rs.locate_bucket(h, 0) == (3, 0)
    assert rs.locate_bucket(h, 4) == (3, 0)
    assert rs.locate_bucket(h, 5) == (7, 5)
    assert rs.locate_bucket(h, 14) == (7, 5)
    assert rs.locate_bucket(h, 15) == (255, 15)
    with pytest.raises(rs.RadsortError):
        rs.locate_bucket(h, 16)


def test_bad_layouts_rejected_before_any_device_work():
    import paper_1703_00687_b200 as rs
    from paper_1703_00687_b200.radsort import ERR_INVALID_ARG, ERR_UNSUPPORTED

    L = rs.lib
    assert L.radsort_sort(None, None, 10, 8, 16, None) == ERR_INVALID_ARG   # K > R
    assert L.radsort_sort(None, None, 10, 12, 8, None) == ERR_INVALID_ARG   # R not multiple of 8
    assert L.radsort_sort(None, None, 10, 48, 8, None) == ERR_UNSUPPORTED   # not built
    assert L.radsort_sort(None, None, 10, 40, 8, None) == ERR_UNSUPPORTED   # not built (SPEC layouts only)
    assert L.radsort_sort(None, None, 10, 8, 4, None) == ERR_INVALID_ARG


def test_product_does_not_import_oracle():
    # the product path never routes through the oracle (no CPU fallback)
    pkg = os.path.join(ROOT, "paper_1703_00687_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in txt.replace("oracle/", ""), f


C99_CLIENT = r"""
#include <stdio.h>
#include <string.h>
#include "radsort.h"

int main(void) {
  radsort_stats st;
  uint64_t q[3];
  const char* s = radsort_error_string(RADSORT_ERR_UNSUPPORTED);
  if (!s || !strstr(s, "unsupported")) return 10;
  /* layout checks come before any device work: no GPU needed */
  if (radsort_sort(NULL, NULL, 10, 12, 8, NULL) != RADSORT_ERR_INVALID_ARG) return 11;
  if (radsort_sort(NULL, NULL, 10, 48, 8, NULL) != RADSORT_ERR_UNSUPPORTED) return 12;
  /* a valid layout with NULL buffers never returns OK (no device, or bad pointers) */
  if (radsort_sort(NULL, NULL, 10, 8, 8, NULL) == RADSORT_OK) return 13;
  if (radsort_plan_quotas(10, 3, q) != RADSORT_OK || q[0] != 4 || q[1] != 3 || q[2] != 3) return 14;
  if (radsort_last_stats(&st) != RADSORT_OK) return 15;
  if (radsort_comm_init(NULL, 1, 0, 0, NULL) != RADSORT_ERR_INVALID_ARG) return 16;
  printf("%s\n", radsort_version());
  radsort_finalize();
  return 0;
}
"""


@pytest.mark.parametrize("std", ["c99", "c11"])
def test_header_compiles_as_plain_c_and_links(tmp_path, std):
    """A plain C client (no CUDA headers) compiles against include/radsort.h,
    links libradsort.so and calls the entry points that need no GPU."""
    import subprocess

    import paper_1703_00687_b200 as rs

    src = tmp_path / "client.c"
    src.write_text(C99_CLIENT)
    exe = tmp_path / "client"
    libdir = os.path.dirname(rs.LIB_PATH)
    cc = subprocess.run(["gcc", f"-std={std}", "-Wall", "-Wextra", "-pedantic", "-Werror",
                         "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe),
                         "-L", libdir, "-l:libradsort.so", f"-Wl,-rpath,{libdir}"],
                        capture_output=True, text=True)
    assert cc.returncode == 0, cc.stderr
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    run = subprocess.run([str(exe)], capture_output=True, text=True, env=env, timeout=60)
    assert run.returncode == 0, (run.returncode, run.stdout, run.stderr)
    assert "radsort" in run.stdout
