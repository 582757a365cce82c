"""Line ranges of the correlator's device functions (for src_lines.py)."""
import json
import re
import sys

src = open(sys.argv[1]).read().splitlines()
marks = [("tap_value/boundary", r"double tap_value\("), ("code tables", r"^struct CodeTables"),
         ("phase_a", r"void phase_a\("), ("phase_a_dispatch", r"void phase_a_dispatch\("),
         ("fill_tap_ranges", r"void fill_tap_ranges\("), ("phase_b", r"void phase_b\("),
         ("fill_rot", r"void fill_rot\("), ("mbar/tma", r"uint32_t smem_u32\("),
         ("loop (fast/metrics)", r"^struct LoopCfg"), ("smem layout", r"^struct CorrSmem"),
         ("partials/totals", r"void warp_partials\("), ("args", r"^struct TrackArgs"),
         ("issue_unit", r"void issue_unit\("), ("finish_epoch", r"void finish_epoch\("),
         ("warp0_update", r"void warp0_update\("), ("track_kernel", r"track_kernel\(TrackArgs"),
         ("jobs", r"^struct JobArgs")]
starts = []
for name, pat in marks:
    for i, l in enumerate(src):
        if re.search(pat, l):
            starts.append((i + 1, name))
            break
starts.sort()
out = []
for k, (ln, name) in enumerate(starts):
    hi = starts[k + 1][0] - 1 if k + 1 < len(starts) else len(src)
    out.append([name, sys.argv[1].rsplit("/", 1)[-1], ln - 3, hi - 3])
print(json.dumps(out))
