"""Markdown table of bench.py JSON lines (one per line of the input file).

    python tools/summarize_bench.py profiles/r01/bench_all.jsonl
"""
import json
import sys


def main():
    rows = [json.loads(line) for line in open(sys.argv[1]) if line.strip().startswith("{")]
    print("| workload | mode | fan-out | partitions | GB | time to loaded (s) | GB/s | of H2D peak "
          "| kernel roofline | e2e GB/s | oracle GB/s (1 core) |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for d in rows:
        c = d["config"]
        r = d.get("roofline") or {}
        kern = f"{r['frac']:.3f} of {r['bound']}" if r.get("frac") is not None else "—"
        if (r.get("in_kernel") or {}).get("frac"):
            kern += f" ({r['in_kernel']['frac']:.3f} in-kernel)"
        cpu = d.get("cpu_baseline") or {}
        print(f"| {c['workload']} | {c['mode']} | {c['fanout']} | {c['partitions_per_gpu']} "
              f"| {c['payload_bytes_per_gpu'] / 1e9:.2f} | {d['time_to_loaded_model_s']:.4f} | {d['value']:.2f} "
              f"| {d['frac_h2d']:.3f} | {kern} | {d['e2e']['value']:.2f} "
              f"| {cpu.get('value', float('nan')):.2f} |")


if __name__ == "__main__":
    main()
