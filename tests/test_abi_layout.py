"""The ctypes mirrors (paper_1310_3322_b200/abi.py) and the numpy record
dtypes agree with include/trb.h field by field: a probe compiled with gcc
against the header prints sizeof / offsetof of every boundary struct."""
import ctypes as C
import os
import subprocess

import pytest

from paper_1310_3322_b200 import abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

STRUCTS = {
    "trb_motion_config": abi.MOTION_CFG,
    "trb_seg_config": abi.SEG_CFG,
    "trb_tracker_config": abi.TRACKER_CFG,
    "trb_blob": abi.BLOB,
    "trb_track_log_entry": abi.LOGE,
    "trb_track": abi.TRACK,
    "trb_streams_options": abi.STREAMS_OPTS,
    "trb_step_output": abi.STEP_OUTPUT,
}


@pytest.fixture(scope="module")
def c_layout(tmp_path_factory):
    d = tmp_path_factory.mktemp("abi")
    lines = ['#include <stddef.h>', '#include <stdio.h>', '#include "trb.h"', "int main(void) {"]
    for name, cls in STRUCTS.items():
        lines.append(f'  printf("{name} sizeof %zu\\n", sizeof({name}));')
        for fname, _ in cls._fields_:
            lines.append(f'  printf("{name} {fname} %zu\\n", offsetof({name}, {fname}));')
    lines += ["  return 0;", "}"]
    src = d / "probe.c"
    src.write_text("\n".join(lines) + "\n")
    exe = d / "probe"
    subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    layout = {}
    for ln in out.splitlines():
        struct, field, value = ln.split()
        layout[(struct, field)] = int(value)
    return layout


@pytest.mark.parametrize("name", sorted(STRUCTS))
def test_struct_layout_matches_header(c_layout, name):
    cls = STRUCTS[name]
    assert C.sizeof(cls) == c_layout[(name, "sizeof")], name
    for fname, _ in cls._fields_:
        assert getattr(cls, fname).offset == c_layout[(name, fname)], (name, fname)


def test_record_dtypes_match_header(c_layout):
    for dt, name in ((abi.BLOB_DTYPE, "trb_blob"), (abi.LOG_DTYPE, "trb_track_log_entry")):
        assert dt.itemsize == c_layout[(name, "sizeof")]
        for fname in dt.names:
            assert dt.fields[fname][1] == c_layout[(name, fname)], (name, fname)
