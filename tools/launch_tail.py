"""Print the last N launches of an ncu launch-list csv: python tools/launch_tail.py FILE [N]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import launches  # noqa: E402

L = list(launches(sys.argv[1]).items())
for (i, n), m in L[-int(sys.argv[2]) if len(sys.argv) > 2 else -30:]:
    mb = (m.get('dram__bytes_read.sum', 0) + m.get('dram__bytes_write.sum', 0)) / 1e6
    print(i, n[:40], round(m.get('gpu__time_duration.sum', 0), 1), round(mb, 2))
