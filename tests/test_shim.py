"""shim.install() rebinds every reference call site of the hot path (run only
where the reference package is importable; no GPU needed to check bindings)."""

import os
import sys

import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference package not present")


def test_install_rebinds_every_call_site():
    sys.path.insert(0, REF)
    try:
        import radfarm.bench
        import radfarm.errors
        import radfarm.farm
        import radfarm.lightfield
        import radfarm.pipeline
        import radfarm.renderer
        from paper_2303_04086_b200 import errors, render, shim
        orig = radfarm.farm.compose
        done = shim.install()
        try:
            assert len(done) == 11
            import radfarm.protocol
            assert radfarm.protocol.encode_frame is render.encode_frame
            assert radfarm.farm.encode_frame is render.encode_frame
            assert render.TYPES["FrameData"] is radfarm.protocol.FrameData
            assert radfarm.renderer.render_rays is render.render_rays
            assert radfarm.lightfield.render_rays is render.render_rays
            assert radfarm.farm.render_range is render.render_range
            assert radfarm.pipeline.render_range is render.render_range
            assert radfarm.bench.render_range is render.render_range
            assert radfarm.farm.compose is render.compose
            assert errors.DomainError is radfarm.errors.DomainError
            assert render.TYPES["Tile"] is radfarm.renderer.Tile
            with pytest.raises(radfarm.errors.ProtocolError):
                render.compose([])           # raised before any device work
        finally:
            shim.uninstall()
        assert radfarm.farm.compose is orig
        assert errors.DomainError is not radfarm.errors.DomainError
    finally:
        sys.path.remove(REF)
