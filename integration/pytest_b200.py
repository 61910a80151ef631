"""pytest plugin: run the REFERENCE's own test suite with its merges routed to the
B200 library (``python -m pytest <reference tests> -p integration.pytest_b200``).

Installs parmerge_b200_binding into the imported reference package before the test
modules import their names, and at the end writes the number of routed
pm_merge_host calls to $PM_DROPIN_REPORT (if set)."""
import json
import os

import parmerge

from integration import parmerge_b200_binding as b200

b200.install(parmerge)


def pytest_sessionfinish(session, exitstatus):
    path = os.environ.get("PM_DROPIN_REPORT")
    if path:
        with open(path, "w") as f:
            json.dump({"routed_calls": b200.calls["pm_merge_host"], "exitstatus": int(exitstatus)}, f)
