"""Renders scripts/ab_formats.py output (one line per variant and round set)
as a markdown table of the best back-to-back and best L2-flushed times."""
import sys


def rows(path):
    env = ""
    for line in open(path):
        if line.startswith("SPMVK_"):
            env = line.strip()
            continue
        if " b2b us " not in line:
            continue
        head, tail = line.split(" b2b us ")
        b2b, flushed = tail.split(" | flushed us ")
        case, prec, g, variant = head.split()[:4]
        yield (case, prec, g, variant, env, min(map(float, b2b.split())),
               min(map(float, flushed.split())))


def main():
    print("| case | prec | variant | env | best b2b us | best L2-flushed us |")
    print("|---|---|---|---|---|---|")
    for path in sys.argv[1:]:
        for case, prec, g, v, env, b, f in rows(path):
            print(f"| {case} | {'fp64' if prec == 'p8' else 'fp32'} | {v} | {env} | {b:.2f} | {f:.2f} |")


if __name__ == "__main__":
    main()
