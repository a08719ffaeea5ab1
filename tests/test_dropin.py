"""Drop-in checks against the reference package itself (dev container only;
skipped where /root/reference is absent):

* the b200 ConverterPlugins register into the reference PluginRegistry and run
  through the reference Converter.run_plan, producing b200 variants whose
  blobs are valid plans;
* ProfilingResult documents written here load in the reference registry;
* on traces without placement requests, this Controller (reference mode:
  one cell per job, FIFO) emits exactly the reference Controller's actions;
* with a placement request the reference raises NameError (controller.py:232)
  while this one places the deployment.
"""
import random

import pytest

from paper_2006_05096_b200 import converter as C
from paper_2006_05096_b200 import plan as P
from paper_2006_05096_b200 import toyformat, zoo
from paper_2006_05096_b200.controller import Controller, PlacementRequest
from paper_2006_05096_b200.profiler.types import ProfilingJob, ProfilingResult, SweepSpec
from paper_2006_05096_b200.telemetry import DeviceSnapshot, DeviceStats

pytestmark = pytest.mark.reference


def test_plugins_run_through_reference_converter(reference_modelci, tmp_path):
    from modelci.converter import Converter, PluginRegistry
    from modelci.converter.plugins import builtin_toy_plugins
    from modelci.registry import FileStore, ModelRegistry
    from modelci.registry.types import RegistrationManifest, TensorSpec
    reg = ModelRegistry(FileStore(tmp_path / "store"))
    plugins = PluginRegistry()
    for p in builtin_toy_plugins():
        plugins.register(p)
    C.register_b200_plugins(plugins)
    rec = reg.register(RegistrationManifest(name="mlp", framework="toy",
                                            inputs=[TensorSpec("x", [-1, 784])]),
                       toyformat.canonical_json(zoo.make_mlp_graph(0)))
    variants, failures = Converter(reg, plugins).run_plan(rec)
    assert not failures
    fmts = {v.format: v for v in variants}
    assert {"b200-bf16", "b200-fp32", "toy-binary", "toy-json"} <= set(fmts)
    plan = P.decode(reg.get_blob(fmts["b200-bf16"].blob_digest))
    assert plan.dtype == P.DT_BF16 and plan.out_elems == 10
    assert fmts["b200-bf16"].serving_backends == ["b200"]
    # results written by this package load in the reference record
    r = ProfilingResult(fmts["b200-bf16"].id, "gpu:0", "b200", "grpc-style", 8, 1e5, 0.1, 0.2,
                        0.3, 1e9, 0.5, resource_scope="gpu:0")
    reg.append_result(rec.id, r)
    back = reg.get(rec.id).profiling_results[0]
    assert back.to_doc() == r.to_doc()


def _snap(u):
    return DeviceSnapshot(0.0, {d: DeviceStats(x, 0, 1) for d, x in u.items()})


def test_controller_equivalent_to_reference_without_placements(reference_modelci):
    from modelci.controller import Controller as RefController
    from modelci.profiler.types import ProfilingJob as RefJob, SweepSpec as RefSpec
    from modelci.telemetry.providers import DeviceSnapshot as RSnap, DeviceStats as RStats
    rng = random.Random(7)
    for _ in range(200):
        devs = [f"gpu:{i}" for i in range(rng.randint(1, 3))]
        ours, ref = Controller(), RefController()
        specs = [rng.sample(devs, rng.randint(1, len(devs))) for _ in range(rng.randint(1, 3))]
        for i, ds in enumerate(specs):
            ours.submit(ProfilingJob(str(i), "r", "v", SweepSpec([1, 2], ds, ["b"], ["rest"])))
            ref.submit(RefJob(str(i), "r", "v", RefSpec([1, 2], ds, ["b"], ["rest"])))
        for _ in range(12):
            u = {d: rng.choice([0.1, 0.5, 0.9]) for d in devs if rng.random() < 0.9}
            ours.on_snapshot(_snap(u))
            ref.on_snapshot(RSnap(0.0, {d: RStats(x, 0, 1) for d, x in u.items()}))
            a = [x.to_doc() for x in ours.tick()]
            b = [x.to_doc() for x in ref.tick()]
            assert a == b
            for d in list(ref.running_cells()):
                if rng.random() < 0.5:
                    for ctl in (ours, ref):
                        jid, cell = ctl.running_cells()[d]
                        ctl.job(jid).completed_cells.add(cell.key())
                        ctl.job(jid).state = "waiting_for_device"
                        ctl.note_cell_done(d)


def test_reference_placement_nameerror_fixed(reference_modelci):
    from modelci.controller import Controller as RefController, PlacementRequest as RefPR
    from modelci.telemetry.providers import DeviceSnapshot as RSnap, DeviceStats as RStats
    ref = RefController()
    for _ in range(3):
        ref.on_snapshot(RSnap(0.0, {"gpu:0": RStats(0.1, 0, 1)}))
    ref.request_placement(RefPR("p", "r", "v", "b", "rest"))
    with pytest.raises(NameError):
        ref.tick()
    ours = Controller()
    for _ in range(3):
        ours.on_snapshot(_snap({"gpu:0": 0.1}))
    ours.request_placement(PlacementRequest("p", "r", "v", "b", "rest"))
    assert [a.kind for a in ours.tick()] == ["place_instance"]
