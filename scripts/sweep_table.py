"""Renders k2_sweep.py / format_study.py JSON lines as a markdown table.
    python scripts/sweep_table.py gpurun_out/sweep_X.jsonl [title] > profiles/rNN_X.md"""
import json
import sys


def main():
    rows = [json.loads(l) for l in open(sys.argv[1]) if l.strip().startswith("{")]
    title = sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]
    print(f"# {title}\n")
    if not rows:
        return
    keys = list(rows[0].keys())
    print("| " + " | ".join(keys) + " |")
    print("|" + "---|" * len(keys))
    for r in rows:
        print("| " + " | ".join(str(r.get(k, "")) for k in keys) + " |")


if __name__ == "__main__":
    main()
