"""pytest plugin: before the reference's test modules import ``hetserve``,
route its hot-path entry points (and, with HS_REFBIND_SCHEDULER=1, its
Scheduler) through the engine with paper_2504_15303_b200.refbind.install --
INTEGRATION.md section 2's binding, applied to the unmodified reference."""

import os


def pytest_configure(config):
    import hetserve

    from paper_2504_15303_b200 import refbind

    refbind.install(hetserve, scheduler=os.environ.get("HS_REFBIND_SCHEDULER") == "1")
    config._hs_refbind = True


def pytest_report_header(config):
    import hetserve

    return f"hetserve from {os.path.dirname(hetserve.__file__)}; hot path routed through paper_2504_15303_b200"
