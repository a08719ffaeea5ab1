"""Dispatcher lifecycle (reference dispatcher.py:105-314) with a fake serving
program: READY handshake, first health, device pinning through
{device_index}, termination, format/protocol/device checks."""
import sys
import time
from pathlib import Path

import pytest

from paper_2006_05096_b200.dispatcher import Dispatcher, ServingBackendTemplate, b200_template
from paper_2006_05096_b200.errors import IncompatibleFormat, LaunchFailure, NotFound, UnknownDevice
from paper_2006_05096_b200.hub import Hub, ModelVariant

FAKE = str(Path(__file__).parent / "fake_backend.py")


def setup(tmp_path, cmd):
    hub = Hub()
    v = ModelVariant("v1", "r1", "b200-bf16", hub.put_blob(b"plan-bytes"), ["b200"])
    tpl = ServingBackendTemplate("b200", ["b200-bf16"], ["grpc-style"], cmd,
                                 env={"CUDA_VISIBLE_DEVICES": "{device_index}"})
    d = Dispatcher(hub, {"b200": tpl}, tmp_path / "work",
                   known_devices=lambda: ["gpu:0", "gpu:3"], ready_timeout_s=20)
    return d, v


def test_dispatch_pins_device_and_terminates(tmp_path):
    rec = tmp_path / "env.txt"
    d, v = setup(tmp_path, [sys.executable, FAKE, "--model", "{model_path}", "--protocol",
                            "{protocol}", "--record", str(rec)])
    inst = d.dispatch(v, "gpu:3", "b200", "grpc-style")
    try:
        assert inst.state == "ready" and inst.endpoint.startswith("127.0.0.1:")
        assert rec.read_text() == "3"
        assert d.pid_of(inst.id) and d.device_of(inst.id) == "gpu:3"
        assert d.health(inst.id) == "ready"
    finally:
        d.terminate(inst.id)
    assert inst.state == "stopped" and d.pid_of(inst.id) is None
    with pytest.raises(NotFound):
        d.terminate(inst.id)


def test_dispatch_checks(tmp_path):
    d, v = setup(tmp_path, [sys.executable, FAKE])
    with pytest.raises(UnknownDevice):
        d.dispatch(v, "gpu:7", "b200", "grpc-style")
    with pytest.raises(IncompatibleFormat):
        d.dispatch(v, "gpu:0", "b200", "rest")
    with pytest.raises(NotFound):
        d.dispatch(v, "gpu:0", "nope", "grpc-style")
    bad = ModelVariant("v2", "r1", "toy-json", v.blob_digest, [])
    with pytest.raises(IncompatibleFormat):
        d.dispatch(bad, "gpu:0", "b200", "grpc-style")


def test_backend_exit_before_ready_is_launch_failure(tmp_path):
    d, v = setup(tmp_path, [sys.executable, "-c", "import sys; sys.exit(2)"])
    with pytest.raises(LaunchFailure):
        d.dispatch(v, "gpu:0", "b200", "grpc-style")


def test_b200_template_shape():
    t = b200_template()
    t.validate()
    assert t.env["CUDA_VISIBLE_DEVICES"] == "{device_index}"
    assert "paper_2006_05096_b200.worker" in t.command
