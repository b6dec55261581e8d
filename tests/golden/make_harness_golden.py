"""Regenerate tests/golden/harness_report_*.txt from the REFERENCE's bench.emit_report
(run in the build container, where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_harness_golden.py
"""
import os

from blockiluk import bench

RECORDS = [bench.BenchRecord(1, 0, 1, 0.5, 0.25, 10, True, 1e-7),
           bench.BenchRecord(1, 0, 4, 0.5, 0.125, 10, True, 1e-7),
           bench.BenchRecord(2, 1, 1, 0.1, 0.3, 3, False, 2e-3),
           bench.BenchRecord(4, 2, 1, 1.0 / 3.0, 0.0, 0, True, 0.0)]

here = os.path.dirname(os.path.abspath(__file__))
for fmt in ("csv", "table"):
    with open(os.path.join(here, f"harness_report_{fmt}.txt"), "w") as fh:
        fh.write(bench.emit_report(RECORDS, fmt))
