"""The C++ drop-in layer (include/hetpar_b200/step_engine.hpp) compiles with
g++ against the C ABI and reproduces the reference's golden values; on a GPU
it runs the C1 trajectory through DeviceStepEngine::round."""
import json
import os
import subprocess

import numpy as np
import pytest

from helpers import ROOT, golden

LIB = os.path.join(ROOT, "paper_2009_14783_b200")


def _build(tmp_path):
    exe = tmp_path / "capi_demo"
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "capi_demo.cpp"), "-L", LIB,
                    "-lhetpar_b200", "-Wl,-rpath," + LIB, "-o", str(exe)], check=True)
    return exe


def test_cpp_host_path(tmp_path):
    exe = _build(tmp_path)
    out = json.loads(subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout)
    assert out["splitmix0"] == "e220a8397b1dcdaf"          # test_rng.cpp:31-34
    assert out["fy"] == [8, 3, 6, 5, 4, 0, 9, 2, 1, 7]     # golden/fisher_yates_n10_seed42.txt
    assert out["sizes"] == [2, 2, 1]                       # test_data.cpp:209-215
    assert out["r3_dummy"] == 1 and out["r3_index"] == 0   # test_data.cpp:279-292
    assert out["nparams"] == 323050
    assert out["init0"] == golden("c1_ref_train.npz")["init_params_f64"][0]
    assert out["config_threw"] == 1


@pytest.mark.gpu
def test_cpp_device_round(tmp_path):
    exe = _build(tmp_path)
    out = json.loads(subprocess.run([str(exe), "gpu"], check=True, capture_output=True, text=True).stdout)
    want = golden("c1_ref_train.npz")["losses_f64"]
    got = np.array(out["losses"])
    assert np.max(np.abs(got - want) / want) <= 1e-4


DROPIN = os.path.join(ROOT, "oracle", "_ref", "dropin_demo")


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj/include"), reason="reference headers absent")
def test_reference_dropin_compiles_against_reference_headers():
    """include/hetpar_b200/reference_dropin.hpp builds with the reference's own
    headers and objects (hetpar::TrainState, ProcessGroup, Batch, StepReport)
    in the reference's round loop (tests/cpp/dropin_demo.cpp)."""
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref", "dropin"], check=True)
    assert os.path.exists(DROPIN)


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(DROPIN), reason="oracle/_ref/dropin_demo not built")
def test_reference_round_loop_with_the_dropin(tmp_path):
    """The reference's own round loop (train_run's, engine.hpp:274-310) with
    hetpar::StepEngine<float> swapped for hetpar::b200::StepEngine<float> (and
    an NcclProcessGroup over the reference's in-process group): the same
    10-update trajectory as the reference engine on the CPU, the TrainState
    kept in step, and the device-backed state through the reference's own
    save_checkpoint / load_checkpoint."""
    out = json.loads(subprocess.run([DROPIN, str(tmp_path / "d")], check=True, capture_output=True,
                                    text=True, timeout=600).stdout.strip().splitlines()[-1])
    ref, dev = np.array(out["ref_losses"]), np.array(out["dev_losses"])
    assert len(ref) == len(dev) == 10
    assert np.max(np.abs(dev - ref) / np.abs(ref)) <= 1e-4
    assert out["params_rel"] <= 1e-4
    assert out["ref_step"] == out["dev_step"] == 10 and out["ref_t"] == out["dev_t"] == 10
    assert out["pending"] == 0 and out["ckpt_rel"] == 0.0 and out["ckpt_step"] == 10
    # and it is the reference's W = 2 trajectory (W x K equivalence)
    assert np.max(np.abs(dev - golden("c1_ref_train.npz")["losses_f64"]) /
                  golden("c1_ref_train.npz")["losses_f64"]) <= 1e-4
