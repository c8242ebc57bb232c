"""profiles/ncu_r1_frame.json (one frame's kernels, ncu --set full) -> profiles/ncu_traffic.json:
DRAM bytes (read + write) per launch under bench.py's profiler names. Profiler names that
cover several kernels (prune = start_mask + start_key + start_place) sum them; names with two
launches per frame (occupancy grid + render) average them, as bench.py's per-launch figures do.
Usage: python tools/ncu_traffic.py profiles/ncu_r1_frame.json profiles/ncu_traffic.json"""
import json
import sys

GROUPS = {"deform": ["start_newton_kernel"], "prune": ["start_mask_kernel", "start_key_kernel", "start_place_kernel"],
          "finalize": ["finalize_pool_kernel"], "field": ["field_tile_kernel"], "field_tc": ["field_tc_kernel"], "encode_tc": ["encode_tiles_kernel"],
          "march": ["march_kernel"], "composite": ["composite_kernel"]}


def mb(s):
    v, u = s.split()
    return float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]


def main(src, dst):
    d = json.load(open(src))
    out = {}
    for name, kernels in GROUPS.items():
        per_src = {}
        for k, v in d.items():
            if "dram__bytes_read.sum" not in v:
                continue
            for kern in kernels:
                if kern in k:
                    srckind = "CellSrc" if "CellSrc" in k else "ListSrc"
                    per_src[srckind] = per_src.get(srckind, 0.0) + mb(v["dram__bytes_read.sum"]) + mb(
                        v["dram__bytes_write.sum"])
        if per_src:
            out[name] = sum(per_src.values()) / len(per_src)
    out["_note"] = ("DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum), ncu --set full "
                    "--clock-control none, cold serialized replay; from " + src)
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
