"""compat.install / uninstall mechanics against the reference's backbone module
(no GPU call): the drop-in rebinds the name MoEDiT.forward resolves
(backbone.py:24, :595-597), is idempotent, and restores the stock function."""

import pytest

from tests.refimport import load_reference, reference_available


@pytest.mark.skipif(not reference_available(), reason="reference package not found")
def test_install_rebinds_backbone_name_and_restores():
    from paper_2604_12163_b200 import compat
    ref = load_reference()
    bb = ref.backbone
    stock = bb.moe_forward
    assert stock is ref.moe.moe_forward
    fn = compat.install(bb)
    try:
        assert bb.moe_forward is fn is not stock
        assert compat.install(bb) is fn
        assert ref.moe.moe_forward is stock        # only the backbone's binding changes
    finally:
        compat.uninstall(bb)
    assert bb.moe_forward is stock
    compat.uninstall(bb)                           # no-op when not installed
    assert bb.moe_forward is stock
