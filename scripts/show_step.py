"""Print the kernels of one search step and of the first ingest chunk from a launch csv."""
import sys
sys.path.insert(0, "scripts")
from launch_summary import load
rows = load(sys.argv[1])
for i, r in enumerate(rows):
    if r[1] == "normalize_kernel" and r[3].startswith("(313") and i > len(rows) - 120:
        for q in rows[i:i + 18]:
            print(q[0], q[1], round(q[2] / 1e3, 1), q[3])
            if q[1] == "merge_kernel":
                break
        break
print("--- ingest chunk")
for i, r in enumerate(rows):
    if r[1] == "normalize_kernel" and r[3].startswith("(7813"):
        for q in rows[i:i + 14]:
            print(q[0], q[1], round(q[2] / 1e3, 1), q[3])
        break
