"""Render cel_trace_dump JSONL files (one per rank) as an SVG timeline, the
analog of PAPER.md Fig. 7 (per-device execution timelines of the instruction
graph): one lane per (device, stream), one bar per profiled launch, colour by
kind.  Times are each device's CUDA events relative to its own origin (the
profile_enable call), so lanes of different ranks are aligned only roughly.

  python tools/trace_svg.py out.svg trace_r0_n4.jsonl trace_r1_n4.jsonl ... [--window-us 600]
"""
import json
import sys

COLORS = {"wave5": "#4e79a7", "shell": "#f28e2b", "copy_peer": "#e15759", "copy": "#76b7b2", "coll": "#59a14f",
          "rsim_row": "#edc948", "jacobi7": "#b07aa1", "nbody_step": "#ff9da7"}


def main():
    argv = sys.argv[1:]
    window = 600.0
    if "--window-us" in argv:
        i = argv.index("--window-us")
        window = float(argv[i + 1])
        argv = argv[:i] + argv[i + 2:]
    args = argv
    out, files = args[0], args[1:]
    recs = []
    for f in files:
        recs += [json.loads(line) for line in open(f)]
    if not recs:
        raise SystemExit("no records")
    lanes = sorted({(r["device"], r["stream"]) for r in recs})
    t_end = max(r["end_us"] for r in recs)
    t0 = t_end - window
    W, lane_h, left = 1200, 22, 150
    H = 40 + lane_h * len(lanes) + 40
    sx = (W - left - 20) / window
    svg = ['<svg xmlns="http://www.w3.org/2000/svg" width="%d" height="%d" font-family="monospace" font-size="11">' % (W, H),
           '<text x="10" y="20">last %.0f us of the trace; lanes = (device, stream); bars = profiled launches</text>' % window]
    for i, (dev, stream) in enumerate(lanes):
        y = 40 + i * lane_h
        svg.append('<text x="10" y="%d">dev %d %s</text>' % (y + 14, dev, stream))
        svg.append('<line x1="%d" y1="%d" x2="%d" y2="%d" stroke="#ddd"/>' % (left, y + lane_h - 2, W - 20, y + lane_h - 2))
        for r in recs:
            if (r["device"], r["stream"]) != (dev, stream) or r["end_us"] < t0:
                continue
            x0 = left + max(0.0, r["start_us"] - t0) * sx
            x1 = left + (r["end_us"] - t0) * sx
            svg.append('<rect x="%.1f" y="%d" width="%.1f" height="%d" fill="%s"><title>%s iid %d %.1f us</title></rect>'
                       % (x0, y + 2, max(1.0, x1 - x0), lane_h - 6, COLORS.get(r["kind"], "#999"), r["kind"], r["iid"],
                          r["end_us"] - r["start_us"]))
    y = 40 + lane_h * len(lanes) + 20
    x = left
    for k, c in COLORS.items():
        svg.append('<rect x="%d" y="%d" width="10" height="10" fill="%s"/><text x="%d" y="%d">%s</text>'
                   % (x, y - 9, c, x + 14, y, k))
        x += 110
    svg.append("</svg>")
    open(out, "w").write("\n".join(svg))


if __name__ == "__main__":
    main()
