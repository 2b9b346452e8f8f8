"""Multi-process sync over IPC peer memory.

Each case runs its N processes on N GPUs; on a box with fewer GPUs the
processes share them round-robin (scripts/_procgroup.py: gloo host group, the
device path unchanged), so every placement also runs on a 1-GPU box.  Cases
that need NCCL itself (the aligned NCCL fall-through, the NCCL DP>2 composition,
the NCCL TP-forward baseline) need N GPUs and skip otherwise."""

import os
import subprocess
import sys

import pytest
import torch

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _need(n, nccl):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    if nccl and torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs (NCCL: one rank per GPU)")


def _run(n, *args, nccl=False):
    _need(n, nccl)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + n),
           os.path.join(ROOT, "scripts", "dist_check.py"), *map(str, args)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "PASS" in r.stdout


@pytest.mark.parametrize("launch", ["three", "graph"])
def test_one_gpu_group_tp4_tp3(launch):
    """NtpSyncGroup in a one-process world (every logical rank on one GPU): the
    same group API, no partners, eager and CUDA-graph steps, vs the oracle."""
    _run(1, 4, 3, "bf16", 3, launch)


@pytest.mark.parametrize("dtype", ["f32", "bf16", "f64"])
def test_two_gpus_tp4_tp3(dtype):
    _run(2, 4, 3, dtype, 3)


def test_two_gpus_tp2_tp1():
    _run(2, 2, 1, "f32", 2)


@pytest.mark.parametrize("launch,policy", [("three", "split"), ("alternate", "split"),
                                           ("fused", "healthy"), ("alternate", "healthy")])
def test_two_gpus_step_launch_variants(launch, policy):
    """One launch per step (ntp_grad_sync_step) and the three-launch sequence
    interoperate; with the "healthy" policy the degraded GPU computes nothing
    and its step is the handshake-only kernel."""
    _run(2, 4, 3, "f32", 4, launch, policy)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("n1", [4, 2])
def test_two_gpus_aligned_nccl_fallthrough(n1, dtype):
    """n1 == n2: shards line up, and NtpSyncGroup(aligned="nccl") syncs each
    rank pair with a weighted NCCL all-reduce; same result as the oracle."""
    _run(2, n1, n1, dtype, 2, "nccl", nccl=True)


def test_two_gpus_aligned_nccl_prescaled():
    """prescaled=True: the weights were folded into the producer (wgrad alpha);
    the aligned sync is a plain NCCL SUM (no weighting pass)."""
    _run(2, 4, 4, "f32", 1, "nccl_pre", nccl=True)


@pytest.mark.parametrize("launch,policy", [("graph", "split"), ("graph_fused", "split"),
                                           ("graph_two", "split"), ("graph_multi", "split"),
                                           ("graph", "healthy"), ("graph_two", "healthy")])
def test_two_gpus_cuda_graph_steps(launch, policy):
    """Steps recorded into CUDA graphs with device-resident epochs (the *_dev
    entry points), alone or interleaved with eager steps: same result as the
    oracle after 5 steps."""
    _run(2, 4, 3, "f32", 5, launch, policy)


def test_four_gpus_tp2_tp1():
    _run(4, 2, 1, "f32", 2)


def test_eight_gpus_tp4_tp3():
    _run(8, 4, 3, "bf16", 3)


def _run_shared(nproc, min_gpus, script, *args):
    """nproc processes on fewer GPUs (shared round-robin, gloo host group): the
    N-process placement and signal wiring on a smaller box."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < min_gpus:
        pytest.skip(f"needs {min_gpus} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(29700 + nproc),
           os.path.join(ROOT, "scripts", script), *map(str, args)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return r


@pytest.mark.parametrize("launch", ["three", "graph", "fused"])
def test_eight_rank_placement_on_shared_gpus(launch):
    """BASELINE configs[1]'s 8-GPU placement (TP4 + TP3 on seven ranks, the
    eighth idle as the failed GPU) as eight processes sharing the box's GPUs:
    every rank's plans, partners and signals, vs the oracle."""
    r = _run_shared(8, 1, "dist_check.py", 4, 3, "bf16", 2, launch)
    assert "PASS" in r.stdout


def test_c3_eight_rank_placement_on_shared_gpus():
    """BASELINE configs[2] (DP=4: three TP2 replicas + one TP1) in its 8-GPU
    placement, the one-shot R-way peer-memory group, processes sharing GPUs."""
    r = _run_shared(8, 1, "dp_check.py", 3, 2, 1, "bf16", 2, 1, "multi")
    assert "PASS" in r.stdout


def test_failure_reconfig_eight_rank_placement_on_shared_gpus():
    """TP4 -> TP3 failure reconfiguration in the 8-process placement (the dead
    rank's units pulled from the healthy replica), bit-exact, processes sharing GPUs."""
    r = _run_shared(8, 1, "reconfig_check.py", "check", 4, 3)
    assert "PASS" in r.stdout


def test_eight_rank_bench_on_shared_gpus():
    """bench.py's N=8 path end to end (re-executed under torchrun, idle rank,
    e2e pipeline) on a smaller box: one JSON line, marked as shared GPUs."""
    import json
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "8", "--steps", "3",
                        "--warmup", "3", "--workload", "mlp-h1024-ffn4096", "--check"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 8 and "shared_gpus" in line and line["value"] > 0
    assert line["check"]["ok"] and line["check"]["max_rel_err"] <= 1e-6  # fp32 C1 vs oracle


def _run_script(n, script, *args, nccl=False):
    _need(n, nccl)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + n),
           os.path.join(ROOT, "scripts", script), *map(str, args)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "PASS" in r.stdout


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("pieces", [1, 5])
def test_four_gpus_dp3_with_degraded_replica(dtype, pieces):
    """DP=3: two healthy TP2 replicas (one GPU each) + a TP1 replica; pieces > 1
    pipelines fold-in / NCCL all-reduce / push-back on three streams."""
    _run_script(4, "dp_check.py", 2, 2, 1, dtype, 2, pieces, nccl=True)


@pytest.mark.parametrize("pieces,algo", [(1, "nccl"), (4, "nccl"), (1, "multi")])
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_four_gpus_c3_shape(pieces, algo, dtype):
    """BASELINE configs[2] shape on 4 GPUs: DP=4 (3 x TP2 + 1 x TP1), through
    NCCL among the healthy replicas or one R-way peer-memory kernel."""
    _run_script(4, "dp_check.py", 3, 2, 1, dtype, 2, pieces, algo, nccl=algo == "nccl")


def test_eight_gpus_c3():
    """BASELINE configs[2]: DP=4 x TP2 with one replica degraded to TP1 (7 GPUs)."""
    _run_script(8, "dp_check.py", 3, 2, 1, "bf16", 2, nccl=True)


@pytest.mark.parametrize("mode", ["red", "push", "push_tma", "red_tma"])
@pytest.mark.parametrize("n,n1,n2", [(2, 2, 1), (4, 2, 1), (2, 4, 3)])
def test_fused_wgrad_sync_multi_gpu(n, n1, n2, mode):
    """tcgen05 wgrad epilogues send this replica's weighted gradient to the
    partner replica over NVLink: red.add, row-store push, or TMA-box push into
    IPC-mapped staging, then the local add."""
    _run_script(n, "fused_check.py", n1, n2, mode)


@pytest.mark.parametrize("n,mode,layout,tokens", [(2, "push", "sync", 512), (2, "push", "comp", 500),
                                                  (2, "nccl", "sync", 512), (4, "push", "sync", 1000),
                                                  (4, "push", "comp", 512)])
def test_row_parallel_forward_multi_gpu(n, mode, layout, tokens):
    """dist_linear.TpMlpForward: column-parallel GEMM + row-parallel GEMM whose
    epilogue pushes partial-sum boxes to the row-block owners over NVLink,
    owner sums in rank order, peer gather; vs the fp64 oracle (<= 2e-2) and
    bit-identical on every rank."""
    _run_script(n, "tp_forward_check.py", mode, layout, tokens, nccl=mode == "nccl")


@pytest.mark.parametrize("n,mode", [(2, "push"), (4, "push"), (2, "nccl")])
def test_row_parallel_forward_bf16_partials(n, mode):
    """out_dtype=bf16: bf16 partial sums and Z (half the all-reduce bytes), the
    owner still accumulates in fp32; <= 2e-2 of the oracle, identical on every rank."""
    _run_script(n, "tp_forward_check.py", mode, "sync", 512, "bf16", nccl=mode == "nccl")


@pytest.mark.parametrize("n,n1,dead", [(1, 4, 3), (2, 4, 1), (4, 2, 0)])
def test_failure_reconfig_multi_gpu(n, n1, dead):
    """dist_reconfig: H -> comp layout, D's survivors -> TP-(n1-1), the dead
    rank's units pulled from H over NVLink; bit-exact for bf16 and fp32 state."""
    _run_script(n, "reconfig_check.py", "check", n1, dead)


@pytest.mark.parametrize("n,n1,n2", [(1, 4, 3), (1, 2, 1), (2, 2, 1), (2, 4, 3), (4, 2, 1),
                                     (4, 4, 3)])
def test_overlapped_backward_step(n, n1, n2):
    """paper_2504_06095_b200.step.OverlappedBackward: the overlapped product
    step gives the same bits as GEMMs-then-syncs, and matches the fp64 oracle
    (w_h * mlp_backward(X_h) + w_r * mlp_backward(X_r), <= 2e-2) in both
    replicas' layouts; n = 1 runs every logical rank on one GPU."""
    _run_script(n, "step_check.py", n1, n2, 3)
