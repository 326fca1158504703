"""Per-scope DRAM traffic from an ncu launch list (one profiled step).

    python tools/make_traffic.py WORKLOAD launches.csv [profiles/ncu_traffic.json]

Kernels are attributed to the library's prof scopes (the names bench.py
reports); bytes are per scope invocation (a scope may run several kernels,
e.g. dc3.srec_apply = k_ps_refine + k_rs_window), counted by its first kernel.
"""
import json
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import load  # noqa: E402

# scope -> (kernel regex that marks one invocation, regex of all its kernels)
SCOPES = {
    "dc3.merge_tile": (r"^k_merge_tile", r"^k_merge_tile"),  # _rec, _w (wide) and the probe-path tile
    "dc3.merge_partition": (r"^k_merge_partition", r"^k_merge_partition"),
    "dc3.srec_emit": (r"^k_srec_emit", r"^k_srec_emit"),
    "dc3.srec_apply": (r"^k_rs_window", r"^k_rs_window|^k_ps_refine<uint4>$"),
    "dc3.mod0_split": (r"^k_mod0_window", r"^k_mod0_window"),
    "lcp.direct": (r"^k_lcp_direct", r"^k_lcp_direct"),
    "rmq.query": (r"^k_sparse_query", r"^k_sparse_query"),
    "rmq.level": (r"^k_sparse_level$|^k_sparse_idx_level", r"^k_sparse_level$|^k_sparse_idx_level"),
    "batch.lcp": (r"^k_batch_lcp<", r"^k_batch_lcp<"),
    "dc3.triple_sort": (r"^k_bs_count<(Triple|PairDense)", r"^k_bs_count<(Triple|PairDense)|^k_bs_scatter_emit<(Triple|PairDense)|^k_bs_tiny|^k_bs_small|^k_bs_window|^k_bs_large"),
    "batch.partition": (r"^k_lsd_scatter", r"^k_lsd_"),
    "pairs.dc3_onchip": (r"^k_pair_dc3", r"^k_pair_dc3"),
    "dc3.ws_count": (r"^k_ws_count", r"^k_ws_count"),
    "dc3.ws_part1": (r"^k_ws_part1", r"^k_ws_part1"),
    "dc3.ws_part2": (r"^k_ws_part2", r"^k_ws_part2"),
    "dc3.ws_sort": (r"^k_ws_sort", r"^k_ws_sort"),
    "dc3.unique_isa": (r"^k_ps_window<uint2", r"^k_ps_window<uint2|^k_ps_refine<uint2>$"),
    "rmq.block_pack": (r"^k_blk_pack", r"^k_blk_pack"),
    "dc3.nx_emit": (r"^k_nx_emit", r"^k_nx_emit"),
    "dc3.nx_apply": (r"^k_nx_window", r"^k_nx_window|^k_ps_refine<uint2>$"),
    "dc3.window_sort": (r"^k_bs_count<Window", r"^k_bs_count<Window|^k_bs_scatter_emit<Window|^k_bs_tiny|^k_bs_small|^k_bs_window|^k_bs_large|^k_ws_"),
    "dc3.unique_ranks": (r"^k_unique_ranks|^k_wn_ranks", r"^k_unique_ranks|^k_wn_ranks"),
    "dc3.tie_resolve": (r"^k_tie", r"^k_tie"),
}


def main(workload, csv_path, out_path=os.path.join("profiles", "ncu_traffic.json")):
    per = load(csv_path)
    names = [(re.sub(r"^(void )?(saix::)?", "", d["name"].split("(")[0]).strip(), d) for d in per.values()]
    res = {}
    for scope, (mark, allk) in SCOPES.items():
        inv = sum(1 for n, _ in names if re.search(mark, n))
        if not inv:
            continue
        b = sum(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
                for n, d in names if re.search(allk, n))
        res[scope] = round(b / inv)
    try:
        with open(out_path) as f:
            allres = json.load(f)
    except Exception:
        allres = {}
    allres[workload] = res
    with open(out_path, "w") as f:
        json.dump(allres, f, indent=1, sort_keys=True)
    print(json.dumps({workload: res}, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
