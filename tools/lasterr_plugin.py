"""pytest plugin (diagnostics): after every test, launch one torch kernel so a
stale CUDA error left in the runtime's last-error slot is attributed to the
test that left it. Usage: python -m pytest -p tools.lasterr_plugin ..."""
import pytest


@pytest.hookimpl(hookwrapper=True)
def pytest_runtest_teardown(item, nextitem):
    yield
    import torch
    if torch.cuda.is_available():
        try:
            x = torch.zeros(1, device="cuda")
            x += 1
            torch.cuda.synchronize()
        except Exception as e:            # noqa: BLE001
            print(f"\n[lasterr] stale CUDA error after {item.nodeid}: {e}".splitlines()[1])
            raise
