"""Cross-rank kernels, one process per GPU (the bench's launch shape):
world = 2, 4 and 8 processes, rank r on cuda:r, built through
rs_ctx_create_rank + CUDA IPC + epoch flags. Each variant is forced and
checked to have run:

  ll    one-shot steps: flagged 16-byte packets pushed into the receivers'
        LL areas (step_kernel.cu LLSend / LLReceive)
  pull  owners load peer sources, sum, store to peer destinations
  push  landing tasks copy into the owners' scratch behind chunk flags,
        reducing tasks wait per chunk (kModeFlagSend / kModeFlagRecv)
  reduce_push  Reduce over >= 3 ranks by the push variant (reduce_mode 1)

on every dtype, ragged sizes, CUDA-graph replays, and (world 2/4) config-2 /
config-3 programs with several slots per rank — bit-exact against the C
oracle (semantics.cc:259-310 folded as dsl.cc:142-164).

Ranks never share a GPU here: kernels that spin on each other's flags are not
guaranteed to run concurrently as separate launches on one GPU. One-GPU
boxes cover the same kernels through emulated ranks in one cooperative launch
(test_gpu_emulated_ranks.py).
"""
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import ranks_worker  # noqa: E402


@pytest.mark.timeout(1200)
@pytest.mark.parametrize("world", [2, 4, 8])
def test_cross_rank_variants_processes(tmp_path, world):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    results = ranks_worker.spawn(world, tmp_path, ranks_worker.on_own_gpu)
    for r, res in enumerate(results):
        assert res["ok"], f"rank {r}:\n{res['msg']}"
    used = results[0]["used"]
    for variant in ("ll", "pull", "push", "reduce_push"):
        assert used.get(variant, 0) > 0, f"variant {variant} never ran: {used}"
