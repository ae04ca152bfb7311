"""bench.py contract checks that run without a GPU: the reference arm (the CPU
oracle timed on the host) prints one JSON line with the driver's keys."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "3",
                        "--ref-tokens", "64"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e", "impl"):
        assert key in d, key
    assert d["impl"] == "reference"
    assert d["value"] > 0 and d["unit"] == "tokens/s" and d["warmup"] >= 3
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith("C2")


def test_ep_line_keys_at_world_size_2():
    """The N > 1 line (EP over NVLink) carries the whole-job value, the EP parity
    and NVLink stage times, a cpu_baseline and e2e through the EP layer's
    run_host_batches — assembled by bench.assemble_line (no GPU needed)."""
    import argparse
    sys.path.insert(0, str(ROOT))
    import bench
    args = argparse.Namespace(config="C2", steps=30, warmup=3, microbatch=0)
    cfg = bench.CONFIGS["C2"]
    T = cfg[0]
    ws, ms = 2, 140.0
    pk = {"bf16_sus": 1430.7, "bf16": 1722.8, "hbm": 6452.8}
    stages = {n: 1.0 for n in ("router_permute", "counts_exchange_offsets", "dispatch_nvlink", "swiglu_k3", "down_k4",
                               "barrier", "combine_nvlink")}
    parity = {"routing_tokens_checked": T, "routing_bitexact": True, "pass": True,
              "ep": {"rank0_output_equals_single_gpu_layer": True, "rank0_dispatch_gbs": 600.0}}
    cpu = {"value": 900.0, "unit": "tokens/s", "cores": 16, "kind": "port", "sample": "first 2048 tokens"}
    e2e = {"value": 3.6e6, "unit": "tokens/s", "h2d_bytes_per_step": T * 4096 * 2 * ws,
           "d2h_bytes_per_step": T * 4096 * 2 * ws, "api": "FusedEPMoELayer.run_host_batches (every rank its own batches)"}
    roof = {"kernel": "grouped_gemm_kernel<EPI_SWIGLU> (K3) on rank 0", "bound": "tensor", "achieved": 1400.0,
            "peak": 1430.7, "unit": "TFLOP/s", "frac": 0.98, "traffic": None}
    value = T * ws / (ms / 1e3)
    line = bench.assemble_line(args, cfg, ws, value, ms, pk, roof, stages, cpu, parity, e2e, 330, {"sm_mhz": 1300},
                               "fused NVLink peer-memory dispatch/combine", 8, False)
    json.dumps(line)
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "parity", "e2e", "gpu_launches",
                "clocks", "stages_ms"):
        assert key in line, key
    assert line["n_gpus"] == 2 and line["scaling"] == "weak" and line["config"]["parallelism"] == "ep2"
    assert line["config"]["global_batch_tokens"] == 2 * T
    assert abs(line["layer_tflops"] / 2 / 1430.7 - line["frac_layer_of_bf16_sustained"]) < 1e-12
    assert line["parity"]["ep"]["rank0_output_equals_single_gpu_layer"]
    assert "dispatch_nvlink" in line["stages_ms"] and line["e2e"]["h2d_bytes_per_step"] == T * 4096 * 2 * 2
