"""Multi-GPU parity through NCCL (torchrun, one process per GPU)."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ngpus():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("cmp", ["gt", "ge"])
@pytest.mark.parametrize("exchange", ["p2p", "nccl"])
def test_exchange_parity(world, cmp, exchange):
    if ngpus() < world:
        pytest.skip(f"needs {world} GPUs")
    env = dict(os.environ, GTC_CMP=cmp, GTC_STEPS="6", GTC_N="1000003", GTC_EXCHANGE=exchange)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29531", os.path.join(ROOT, "tests", "mp_gtc_worker.py")]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    assert "MULTIGPU OK" in p.stdout


@pytest.mark.parametrize("exchange", ["p2p", "nccl"])
def test_exchange_lstm_am_size(exchange):
    if ngpus() < 2:
        pytest.skip("needs 2 GPUs")
    env = dict(os.environ, GTC_CMP="gt", GTC_STEPS="3", GTC_N="24286575", GTC_EXCHANGE=exchange)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29532", os.path.join(ROOT, "tests", "mp_gtc_worker.py")]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("exchange", ["p2p", "nccl"])
def test_momentum_multigpu(world, exchange):
    """GTC_ACCUM_MOMENTUM (SGD-momentum apply, reading M1): weights, momentum
    buffer, residuals, messages and counts bit-exact with the oracle; also the
    one-call step."""
    if ngpus() < world:
        pytest.skip(f"needs {world} GPUs")
    env = dict(os.environ, GTC_CMP="gt", GTC_STEPS="3", GTC_N="1000003", GTC_EXCHANGE=exchange,
               GTC_ACCUM="momentum")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29535", os.path.join(ROOT, "tests", "mp_gtc_worker.py")]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    assert "momentum=True" in p.stdout


@pytest.mark.parametrize("exchange", ["p2p", "nccl"])
@pytest.mark.parametrize("world", [2, 4])
def test_bmuf_multigpu(world, exchange):
    """p2p: bit-exact with oracle_bmuf_step at every step, also back to back
    without host syncs; nccl: within the derived rounding bound."""
    if ngpus() < world:
        pytest.skip(f"needs {world} GPUs")
    env = dict(os.environ, GTC_MODE="bmuf", GTC_N="1000003", GTC_EXCHANGE=exchange)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29533", os.path.join(ROOT, "tests", "mp_gtc_worker.py")]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    assert "BMUF OK" in p.stdout


@pytest.mark.parametrize("world,lag,accum", [(2, "1", "weights"), (2, "7", "update"), (3, "64", "weights"),
                                             (4, "5", "weights"), (4, "0", "update"), (2, "0", "momentum"),
                                             (4, "9", "momentum")])
def test_fused_step_parity(world, lag, accum):
    """The fused one-kernel p2p step (step_p2p.cu) with short decode lags, so
    CTAs wait on peers' tiles still being written (stamped entries), and with
    the default lag ("0"); ranks start skewed on odd steps."""
    if ngpus() < world:
        pytest.skip(f"needs {world} GPUs")
    env = dict(os.environ, GTC_CMP="gt", GTC_STEPS="4", GTC_N="1000003", GTC_EXCHANGE="p2p", GTC_ACCUM=accum)
    if lag != "0":
        env["GTC_FUSED_LAG"] = lag
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29536", os.path.join(ROOT, "tests", "mp_gtc_worker.py")]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    assert "MULTIGPU OK" in p.stdout


def test_unfused_step_parity():
    """gtc_step as separate encode / decode kernels (GTC_STEP_FUSED=0)."""
    if ngpus() < 2:
        pytest.skip("needs 2 GPUs")
    env = dict(os.environ, GTC_CMP="ge", GTC_STEPS="4", GTC_N="1000003", GTC_EXCHANGE="p2p", GTC_STEP_FUSED="0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29537", os.path.join(ROOT, "tests", "mp_gtc_worker.py")]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]


@pytest.mark.parametrize("world,accum", [(2, "weights"), (4, "update"), (4, "momentum")])
def test_sharded_decode_multigpu(world, accum):
    """GTC_DECODE_SHARDED across processes: owner counts over NVLink peer
    reads, per-tile (index, count) lists, every rank applies every list."""
    if ngpus() < world:
        pytest.skip(f"needs {world} GPUs")
    env = dict(os.environ, GTC_CMP="gt", GTC_STEPS="4", GTC_N="1000003", GTC_EXCHANGE="p2p", GTC_ACCUM=accum,
               GTC_SHARDED="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29538", os.path.join(ROOT, "tests", "mp_gtc_worker.py")]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    assert "sharded=True" in p.stdout
