"""CPU-side checks of the boundary: libdisc.so loads and exports every symbol include/disc.h
declares; the binding's struct layouts match the header's field lists.  No compute calls
(no GPU here)."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "disc.h")


@pytest.fixture(scope="module")
def built():
    subprocess.run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "paper_2603_03935_b200", "csrc")], check=True)
    from paper_2603_03935_b200 import disc
    return disc


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(disc_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for n in ["disc_map_create", "disc_map_destroy", "disc_integrate_frame", "disc_query", "disc_get_instances"]:
        assert n in names


def test_library_exports_every_declared_symbol(built):
    lib = C.CDLL(built.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", built.LIB_PATH], capture_output=True, text=True).stdout
    for n in declared_functions():
        assert re.search(rf"\bT {n}\b", out), n


def test_binding_covers_every_export(built):
    assert set(built.EXPORTS) == set(declared_functions())


def _struct_fields(name):
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    m = re.search(r"typedef struct \{([^{}]*)\}\s*" + name + ";", src)
    body = m.group(1)
    fields = []
    for decl in body.split(";"):
        decl = decl.strip()
        if not decl:
            continue
        parts = [w for w in decl.replace("*", " * ").split() if w not in ("const", "unsigned")]
        names = " ".join(parts[1:]).replace("*", "").split(",")
        for nm in names:
            nm = nm.strip()
            nm = re.sub(r"\[.*\]", "", nm).strip()
            if nm:
                fields.append(nm)
    return fields


@pytest.mark.parametrize("cname,pyname", [("disc_config", "disc_config"), ("disc_frame", "disc_frame"),
                                          ("disc_frame_report", "disc_frame_report"),
                                          ("disc_instance", "disc_instance"),
                                          ("disc_frame_debug", "disc_frame_debug"), ("disc_stats", "disc_stats")])
def test_struct_layouts_match_header(built, cname, pyname):
    py = [f[0] for f in getattr(built, pyname)._fields_]
    assert py == _struct_fields(cname)


def test_config_defaults_and_versions(built):
    c = built.default_config()
    assert abs(c.tau_geo - 0.3) < 1e-7 and abs(c.tau_vis - 0.8) < 1e-7 and abs(c.lambda_size - 3.3) < 1e-6
    assert c.mask_min_area == 400 and abs(c.cover_min - 0.25) < 1e-9 and c.world_size == 1
    assert b"sm_100a" in built.lib().disc_version()


def test_create_fails_loudly_without_gpu(built):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    c = built.default_config()
    h = C.c_void_p()
    rc = built.lib().disc_map_create(C.byref(c), C.byref(h))
    assert rc != 0 and not h.value


def test_invalid_config_rejected(built):
    c = built.default_config(voxel_size=-1.0)
    h = C.c_void_p()
    assert built.lib().disc_map_create(C.byref(c), C.byref(h)) == built.DISC_ERR_INVALID
    c = built.default_config(max_masks=300)
    assert built.lib().disc_map_create(C.byref(c), C.byref(h)) == built.DISC_ERR_INVALID


def test_sass_is_sm100a(built):
    out = subprocess.run(["cuobjdump", "--list-elf", built.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_nccl_unique_id_export():
    """disc_nccl_unique_id: 128 bytes from NCCL's bootstrap (no GPU needed); fresh per call."""
    from paper_2603_03935_b200.disc import nccl_unique_id
    a, b = nccl_unique_id(), nccl_unique_id()
    assert len(a) == 128 and any(a)
    assert a != b
