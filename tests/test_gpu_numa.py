"""Host-segment NUMA placement (cm_set_param "numa_node", cm_info.numa_node): the auto
policy binds the shadow segment to the NUMA node sysfs reports for the GPU's PCIe root
(none when sysfs reports -1, e.g. a single-node VM), -1 turns it off, and placement
never changes results (bit-exact vs the oracle either way)."""
import os

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2507_13522_b200 import cm, harness
from paper_2507_13522_b200 import workloads as W

pytestmark = pytest.mark.gpu

HP_O = dict(lr=W.HP["lr"], b1=W.HP["beta1"], b2=W.HP["beta2"], eps=W.HP["eps"], wd=W.HP["weight_decay"])


def sysfs_node(dev):
    p = torch.cuda.get_device_properties(dev)
    bus = "%04x:%02x:%02x.0" % (p.pci_domain_id, p.pci_bus_id, p.pci_device_id)
    try:
        return int(open(f"/sys/bus/pci/devices/{bus}/numa_node").read().strip())
    except OSError:
        return -1


@pytest.mark.parametrize("req", [None, "-1", "0"])
def test_numa_placement_and_parity(monkeypatch, req):
    if req is not None:
        monkeypatch.setenv("CM_NUMA_NODE", req)
    numel = W.numels(W.c1_ragged())
    name = f"cmnuma{os.getpid()}_{req}"
    g = harness.VirtualGroup(numel, 2, 0, cm.CM_F32, 1 << 20, name, 2, cm.CM_SHADOW_HOST)
    try:
        want = {None: sysfs_node(0), "-1": -1, "0": 0}[req]
        for r in g.ranks:
            assert r.ctx.info().numa_node == want
        ref = O.Run(O.Plan(numel, 1 << 20, 4, 2), seed=W.SEED, gscale=W.GRAD_SCALE, hp=HP_O)
        for _ in range(2):
            g.step()
            ref.step()
        g.sync()
        torch.cuda.synchronize()
        for r in g.ranks:
            assert np.array_equal(r.p.cpu().numpy().view(np.uint32), ref.p.view(np.uint32))
            assert r.ctx.verify(g.stream) == -1
    finally:
        g.sync()
        g.finalize()
        for r in range(2):
            cm.unlink_shadow(name, r)
