"""profiles/ncu_r1_frame.json (one frame's kernels, ncu --set full) -> profiles/ncu_traffic.json:
DRAM bytes (read + write) per launch under bench.py's profiler names. Profiler names that
cover several kernels (prune = start_mask + start_key + start_place) sum them; names with two
launches per frame (occupancy grid + render) average them, as bench.py's per-launch figures do.
Usage: python tools/ncu_traffic.py profiles/ncu_r1_frame.json profiles/ncu_traffic.json"""
import json
import sys

GROUPS = {"deform": ["start_newton_kernel"], "prune": ["start_mask_kernel", "scan_lookback_kernel", "start_key_kernel", "start_place_kernel"],
          "finalize": ["finalize_pool_kernel"], "field": ["field_tile_kernel"], "field_tc": ["field_fused_kernel", "field_tc_kernel"], "encode_tc": ["encode_tiles_kernel"],
          "march": ["march_kernel"], "composite": ["composite_kernel"]}


def mb(s):
    v, u = s.split()
    return float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]


def main(src, dst):
    d = json.load(open(src))
    out = {}
    for name, kernels in GROUPS.items():
        # per source kind (CellSrc: occupancy grid, ListSrc: render): mean per launch of each
        # kernel of the group, summed over the group's kernels; then averaged over the kinds
        per = {}
        for k, v in d.items():
            if "dram__bytes_read.sum" not in v:
                continue
            for kern in kernels:
                if kern in k:
                    kind = "CellSrc" if "CellSrc" in k else "ListSrc"
                    per.setdefault((kind, kern), []).append(mb(v["dram__bytes_read.sum"]) + mb(v["dram__bytes_write.sum"]))
        kinds = {}
        for (kind, kern), xs in per.items():
            kinds[kind] = kinds.get(kind, 0.0) + sum(xs) / len(xs)
        if kinds:
            out[name] = sum(kinds.values()) / len(kinds)
    out["_note"] = ("DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum), ncu --set full "
                    "--clock-control none, cold serialized replay; from " + src)
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
