"""Key metrics of an `ncu --set full` report (one kernel launch) as JSON, and
the per-step DRAM traffic file bench.py reads (profiles/traffic.json).

usage: python tools/ncu_summary.py gpurun_out/prof_bench.ncu-rep out.json [--steps 20]
           [--traffic profiles/traffic.json --algorithmic 80539576 --command '...']"""
import argparse
import csv
import io
import json
import subprocess

KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "smsp__sass_inst_executed_op_shared_ld.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_requests_srcunit_tex_op_read.sum",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--traffic", default=None)
    ap.add_argument("--algorithmic", type=int, default=0)
    ap.add_argument("--command", default="")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    ix = {h: i for i, h in enumerate(hdr)}
    out = {k: [vals[ix[k]], units[ix[k]]] for k in KEYS if k in ix}
    json.dump(out, open(a.out, "w"), indent=1)
    if a.traffic:
        def b(k):
            v, u = out[k]
            return float(v.replace(",", "")) * SCALE.get(u, 1)
        rd, wr = b("dram__bytes_read.sum"), b("dram__bytes_write.sum")
        json.dump({"dram_bytes_per_step": int((rd + wr) / a.steps),
                   "dram_read_bytes_per_step": int(rd / a.steps),
                   "dram_write_bytes_per_step": int(wr / a.steps),
                   "algorithmic_bytes_per_step": a.algorithmic,
                   "source": f"ncu --set full of the {a.steps}-step timed stack launch ({a.out})",
                   "command": a.command}, open(a.traffic, "w"), indent=1)
    print(json.dumps(out)[:2000])


if __name__ == "__main__":
    main()
