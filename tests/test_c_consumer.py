"""A plain C host drives the library through include/b200fd.h alone.

tests/c_consumer/consumer.c is a C99 program with no Python or torch in it:
it builds an acoustic problem, allocates the device workspace, runs the whole
simulation with one fdr_acoustic_run_host call and dumps inputs and outputs.

* CPU: the header compiles as strict C99 (-pedantic -Werror), every symbol
  the program uses links against the in-tree libb200fd.so, and the error path
  (a wrong ABI version rejected with a message) works without a device.
* GPU: the dumped final level and traces equal the C oracle's (the
  restatement pinned to the reference, oracle/acoustic_ref.c) bit for bit on
  the same inputs, and the program's weights / coefficient, derived in C from
  the rules b200fd.h documents, equal the reference's float32 constants.
"""

import os
import shutil
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1608_03984_b200")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


@pytest.fixture(scope="module")
def consumer(tmp_path_factory):
    if shutil.which("gcc") is None:
        pytest.skip("gcc not installed")
    if not os.path.exists(os.path.join(PKG, "libb200fd.so")):
        pytest.skip("libb200fd.so not built")
    exe = str(tmp_path_factory.mktemp("c_consumer") / "consumer")
    cmd = ["gcc", "-std=c99", "-pedantic", "-Wall", "-Wextra", "-Werror", "-O2",
           "-I", os.path.join(ROOT, "include"), "-isystem", os.path.join(CUDA, "include"),
           os.path.join(ROOT, "tests", "c_consumer", "consumer.c"), "-o", exe,
           "-L", PKG, "-lb200fd", "-L", os.path.join(CUDA, "lib64"), "-lcudart", "-lm",
           f"-Wl,-rpath,{PKG}:{os.path.join(CUDA, 'lib64')}"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
    return exe


def test_header_is_c99_and_links(consumer):
    assert os.access(consumer, os.X_OK)


def test_error_path_without_device(consumer, tmp_path):
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("device present: the GPU test runs the program")
    res = subprocess.run([consumer, "4", "8", "8", "8", "2", "1e-3", "10", str(tmp_path / "o.bin")],
                         capture_output=True, text=True, timeout=120)
    assert res.returncode == 2
    assert "rejected: abi_version" in res.stdout


def test_bad_usage(consumer):
    res = subprocess.run([consumer], capture_output=True, text=True, timeout=60)
    assert res.returncode == 1 and "usage" in res.stderr


def _read(path):
    buf = open(path, "rb").read()
    off = 0

    def take(n, dt):
        nonlocal off
        a = np.frombuffer(buf, dtype=dt, count=n, offset=off)
        off += a.nbytes
        return a

    order, nx, ny, nz, n_t, n_rec, newest, pitch = (int(v) for v in take(8, np.int32))
    r = order // 2
    out = dict(order=order, dims=(nx, ny, nz), n_t=n_t, newest=newest, pitch=pitch)
    out["weights"] = take(r + 1, np.float32)
    out["coef"] = take(1, np.float32)[0]
    out["m"] = take(nx * ny * nz, np.float32).reshape(nx, ny, nz)
    out["sponge"] = (take(nx, np.float32), take(ny, np.float32), take(nz, np.float32))
    out["series"] = take(n_t, np.float32)
    out["rec"] = take(3 * n_rec, np.int32).reshape(n_rec, 3)
    out["src"] = tuple(int(v) for v in take(3, np.int32))
    out["final"] = take(nx * ny * nz, np.float32).reshape(nx, ny, nz)
    out["traces"] = take(n_t * n_rec, np.float32).reshape(n_t, n_rec)
    assert off == len(buf)
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("order,dims,n_t", [(2, (33, 30, 37), 40), (4, (40, 37, 45), 60),
                                            (8, (70, 64, 66), 50), (8, (130, 96, 131), 30)])
def test_c_host_run_equals_oracle(consumer, cuda_device, tmp_path, order, dims, n_t):
    import paper_1608_03984_b200 as B
    from oracle import cref
    from oracle.acoustic import kernel_constants

    h = 10.0
    dt = 0.4 * B.max_stable_dt(order, h, 1.0 / 3000.0 ** 2)
    path = str(tmp_path / "run.bin")
    res = subprocess.run([consumer, str(order), *(str(d) for d in dims), str(n_t), repr(dt), repr(h),
                          path], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout + res.stderr
    got = _read(path)

    centre, taps, coef = kernel_constants(order, dt, h)
    assert got["weights"].tobytes() == np.array([centre] + taps, np.float32).tobytes()
    assert got["coef"] == coef

    cfg = B.KernelConfig(order=order, dims=dims, n_t=n_t, dt=dt, h=h, m=got["m"],
                         source=B.Source(got["src"], got["series"]),
                         receivers=B.Receivers(got["rec"]), sponge=B.Sponge(*got["sponge"]))
    st = cref.simulate(cfg)
    r = order // 2
    want = st.grids[2][r:-r, r:-r, r:-r]
    assert np.isfinite(got["final"]).all()
    np.testing.assert_array_equal(got["final"], want)
    np.testing.assert_array_equal(got["traces"], st.traces[:n_t])
