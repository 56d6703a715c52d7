"""The FBMP raster container (include/fbmp/raster_io.hpp; proj/src/raster_io.cpp) and the
command-line front end (host/fbmp_cli.cpp): format checks and exit codes on the
CPU (no device is touched before the inputs are validated), the blind command on the GPU."""
import os
import struct
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2103_09943_b200", "lib", "fbmp")


def write_fbmp(path, cube, version=1, dtype=1, truncate=0):
    """raster_io.hpp:11-14: "FBMP" | u16 version | u32 height | u32 width | u16 bands | u16 dtype |
    band-major little-endian float32 samples."""
    cube = np.asarray(cube, dtype="<f4")
    if cube.ndim == 2:
        cube = cube[None]
    nb, h, w = cube.shape
    data = b"FBMP" + struct.pack("<HIIHH", version, h, w, nb, dtype) + cube.tobytes()
    with open(path, "wb") as f:
        f.write(data[: len(data) - truncate])


def read_fbmp(path):
    with open(path, "rb") as f:
        data = f.read()
    assert data[:4] == b"FBMP"
    version, h, w, nb, dtype = struct.unpack("<HIIHH", data[4:18])
    assert version == 1 and dtype == 1 and len(data) == 18 + 4 * h * w * nb
    return np.frombuffer(data[18:], dtype="<f4").reshape(nb, h, w).astype(np.float64)


def cli(*args):
    return subprocess.run([CLI, *args], capture_output=True, text=True)


@pytest.fixture(scope="module")
def built():
    if not os.path.exists(CLI):
        pytest.skip("CLI not built (run __graft_entry__.build())")
    return CLI


def test_info_reads_the_container(built, tmp_path):
    p = str(tmp_path / "a.fbmp")
    write_fbmp(p, np.zeros((3, 5, 7)))
    r = cli("info", "--in", p)
    assert r.returncode == 0 and r.stdout.split() == ["5", "7", "3"]


@pytest.mark.parametrize("kind", ["magic", "version", "dtype", "truncated", "missing"])
def test_format_and_io_errors_exit_2(built, tmp_path, kind):
    p = str(tmp_path / "bad.fbmp")
    if kind == "magic":
        write_fbmp(p, np.zeros((1, 4, 4)))
        with open(p, "r+b") as f:
            f.write(b"XBMP")
    elif kind == "version":
        write_fbmp(p, np.zeros((1, 4, 4)), version=2)
    elif kind == "dtype":
        write_fbmp(p, np.zeros((1, 4, 4)), dtype=2)
    elif kind == "truncated":
        write_fbmp(p, np.zeros((1, 4, 4)), truncate=3)
    r = cli("info", "--in", p)
    assert r.returncode == 2, r.stderr


def test_usage_and_dimension_errors_exit_1(built, tmp_path):
    assert cli().returncode == 1
    assert cli("frobnicate").returncode == 1
    assert cli("blind", "--lrms").returncode == 1
    lr, pan = str(tmp_path / "l.fbmp"), str(tmp_path / "p.fbmp")
    write_fbmp(lr, np.ones((2, 16, 16)))
    write_fbmp(pan, np.ones((1, 60, 64)))  # not an integer multiple in both axes
    r = cli("blind", "--lrms", lr, "--pan", pan, "--out", str(tmp_path / "o.fbmp"))
    assert r.returncode == 1 and "dimension" in r.stderr
    assert cli("blind", "--lrms", lr, "--pan", pan).returncode == 1  # --out missing


@pytest.mark.gpu
def test_blind_command_matches_the_api(built, gpu, tmp_path):
    """C1 scene through files: the HRMS and kernel rasters match fbmp.blind on the float32 inputs."""
    from paper_2103_09943_b200 import synth

    sc = synth.make_scene("C1")
    lr, pan, out, ko = (str(tmp_path / f) for f in ("l.fbmp", "p.fbmp", "o.fbmp", "k.fbmp"))
    write_fbmp(lr, sc.lrms)
    write_fbmp(pan, sc.pan)
    r = cli("blind", "--lrms", lr, "--pan", pan, "--out", out, "--kernel-out", ko, "--n", "15")
    assert r.returncode == 0, r.stderr
    ref, info = gpu.blind(read_fbmp(lr), read_fbmp(pan)[0], 4, 15)
    got, k = read_fbmp(out), read_fbmp(ko)[0]
    # separate API calls (solve_weights -> estimate_kernel_tgv -> pansharpen) against the fused
    # blind entry point, then float32 output rounding: equal to the fp64 parity tolerance
    rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert rel < 1e-6, rel
    assert np.linalg.norm(k - info["kernel"]) / np.linalg.norm(info["kernel"]) < 1e-6
    r = cli("metrics", "--est", out, "--ref", out, "--border", "10")
    assert r.returncode == 0 and "psnr_avg inf" in r.stdout
