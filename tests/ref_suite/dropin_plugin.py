"""pytest plugin (``-p dropin_plugin``) that runs the REFERENCE's own test
suite against the B200 drop-in: before any test module is imported it calls
``dropin.install(mixplane, catalogs=True)``, so ``MetadataCatalog.
filter_intervals``, ``build_index``, ``ChunkGenerator``, ``AdoSource`` /
``AdoState`` -- and the server's seams -- are the device path, and the
package's exceptions are the reference's. Used by
``tests/test_gpu_reference_suite.py``; the suite itself lives in the
reference install (``baseline/_ref/mixplane_tests``, tools/install_reference.sh).
"""

from __future__ import annotations

_installed = {}


def pytest_configure(config):
    import mixplane

    from paper_2502_19790_b200 import _lib, dropin

    _lib.lib()  # fail loudly here if the CUDA path is unavailable
    _installed["undo"] = dropin.install(mixplane, catalogs=True)


def pytest_unconfigure(config):
    undo = _installed.pop("undo", None)
    if undo:
        undo()


def pytest_terminal_summary(terminalreporter):
    from paper_2502_19790_b200 import _lib

    terminalreporter.write_line(
        f"mixplane hot path: B200 drop-in (paper_2502_19790_b200.dropin), {_lib.lib().mx_launch_count()} kernel launches")
