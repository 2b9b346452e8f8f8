"""Cross-GPU signal words on one device: post/wait ordering and the bounded
wait (a word that never arrives sets NTP_ETIMEOUT instead of hanging)."""

import ctypes

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2504_06095_b200 import _lib
    return _lib


def _st(t):
    return ctypes.cast(t.data_ptr(), ctypes.POINTER(ctypes.c_int))


def test_post_then_wait(L):
    lib = L.load()
    words = torch.zeros(4, dtype=torch.int64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    ptrs = [words.data_ptr() + 8 * i for i in range(4)]
    L.check(lib.ntp_signal_post(L.u64_ptr_array(ptrs), 4, 7, s))
    L.check(lib.ntp_signal_wait(L.u64_ptr_array(ptrs), 4, 7, 10**9, _st(status), s))
    torch.cuda.synchronize()
    assert words.tolist() == [7, 7, 7, 7] and status.item() == 0


def test_wait_times_out_instead_of_hanging(L):
    lib = L.load()
    words = torch.zeros(2, dtype=torch.int64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    ptrs = [words.data_ptr(), words.data_ptr() + 8]
    L.check(lib.ntp_signal_wait(L.u64_ptr_array(ptrs), 2, 1, 2_000_000, _st(status), s))  # 2 ms
    torch.cuda.synchronize()
    assert status.item() == L.NTP_ETIMEOUT


def test_signaled_sync_times_out_without_peer(L):
    """A signalled plan whose partner never posts 'ready' exits with a timeout
    status and leaves the data untouched."""
    from paper_2504_06095_b200.plans import OPS, Plan
    lib = L.load()
    a = torch.ones(4096, device="cuda")
    b = torch.ones(4096, device="cuda")
    plan = Plan(L.NTP_F32).add_units(4096, [0], [0], [1], [0]).finalize().upload(0)
    words = torch.zeros(2, dtype=torch.int64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    plan.grad_sync_signaled([a.data_ptr(), b.data_ptr()], OPS["sum"], 1.0, 1.0,
                            [words.data_ptr()], [words.data_ptr() + 8], 1, 2_000_000,
                            status.data_ptr())
    torch.cuda.synchronize()
    assert status.item() == L.NTP_ETIMEOUT
    assert torch.equal(a, torch.ones_like(a)) and words[1].item() == 0
