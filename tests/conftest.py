import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running GPU case (full BASELINE sizes)")


@pytest.fixture(scope="session")
def oracle_lib():
    from oracle import build_ref
    build_ref.build_oracle()
    from oracle import oracle as O
    return O


@pytest.fixture(scope="session")
def gpu():
    """The GPU library context.  Fails (never skips) when the CUDA path is missing on a GPU run."""
    import paper_1402_3501_b200 as G
    ctx = G.Context(0)
    yield G, ctx
    ctx.close()


# The library snapshots its FFG_* switches once (csrc/knobs.cuh); tests that flip one with
# monkeypatch get a fresh snapshot after every change, including the teardown's restore.
def _reload_knobs():
    mod = sys.modules.get("paper_1402_3501_b200")
    if mod is not None and getattr(mod.ffpluq, "_lib", None) is not None:
        mod.reload_knobs()


def _wrap(name):
    orig = getattr(pytest.MonkeyPatch, name)

    def wrapped(self, *args, **kwargs):
        out = orig(self, *args, **kwargs)
        if name == "undo" or (args and str(args[0]).startswith("FFG_")):
            _reload_knobs()
        return out

    setattr(pytest.MonkeyPatch, name, wrapped)


for _name in ("setenv", "delenv", "undo"):
    _wrap(_name)
