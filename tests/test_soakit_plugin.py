"""The plugin side of the boundary on CPU: paper_2511_04853_b200.soakit_plugin
registers into the real soakit registries (memctx.py:269/338,
transfer.py:67-77, behaviors.py:46-62) and the reference's dispatch picks the
B200 spec for the pairs it claims. Runs where soakit is importable
(baseline/_ref or the dev container's reference tree)."""

import os

import pytest

from skhelp import import_soakit

soakit = import_soakit()
pytestmark = pytest.mark.skipif(soakit is None, reason="soakit (the reference package) is not installed")

os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")


@pytest.fixture(scope="module")
def plugin():
    from paper_2511_04853_b200 import soakit_plugin

    return soakit_plugin, soakit_plugin.install()


def test_install_registers_contexts_copiers_spec_and_behaviors(plugin):
    sp, reg = plugin
    smc, st = soakit.memctx, soakit.transfer
    assert {"cuda", "pinned"} <= set(smc.context_names())
    for s in ("host", "mockdev", "pinned", "cuda"):
        for d in ("host", "mockdev", "pinned", "cuda"):
            assert smc.has_copier(s, d)
    assert st.registered_transfers()[0] == "b200-convert"
    assert sp.install() is reg  # idempotent
    from soakit import behaviors as bh

    for target in (bh.TARGET_OBJECT, bh.TARGET_COLLECTION):
        for fn in ("calibrate_energy", "get_noise"):
            assert bh.lookup("sensor_funcs", fn, target).fn.__module__ == sp.__name__


def test_reference_dispatch_picks_b200_for_device_pairs_only(plugin):
    sp, _ = plugin
    from soakit.detector.schemas import SENSOR_SCHEMA

    C = soakit.Collection
    host_aos = C(SENSOR_SCHEMA, "aos")
    host_pf = C(SENSOR_SCHEMA, "per_field")
    dev_pf = C(SENSOR_SCHEMA, "per_field", sp.cuda_info(0))  # empty: nothing is allocated on a device yet
    dev_aos = C(SENSOR_SCHEMA, "aos", sp.cuda_info(0))
    applies = sp._convert_applies
    assert applies(dev_pf, host_aos) and applies(dev_aos, host_pf) and applies(host_aos, dev_pf)
    assert not applies(host_pf, host_aos)          # host <-> host stays on the reference's CPU path
    assert not applies(dev_pf, host_pf)            # same kind: bulk-same-kind
    mock = C(SENSOR_SCHEMA, "aos", soakit.memctx.ContextInfo.mockdev())
    assert not applies(dev_pf, mock)               # mockdev pairs are the reference's business
    with pytest.raises(soakit.errors.AccessError):
        dev_pf.layout._plane_region(dev_pf.plan.leaf("counts"), 0)[0]._data[0]


def test_host_pairs_still_run_the_reference_path(plugin):
    from soakit.detector.schemas import SENSOR_SCHEMA

    a = soakit.Collection(SENSOR_SCHEMA, "aos")
    a.resize(7)
    b = soakit.Collection(SENSOR_SCHEMA, "per_field")
    assert soakit.transfer.copy_collection(b, a) == "per-leaf-default"
