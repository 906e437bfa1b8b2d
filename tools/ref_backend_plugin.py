"""pytest plugin: run the reference's own test suite (abft_guard 0.1.0, installed under
baseline/_ref) with its hot-path entry points dispatched to the B200 C-ABI — the INTEGRATION.md
stub in action.  usage (GPU box, repo root):

  PYTHONPATH=baseline/_ref:. python -m pytest -c /dev/null --rootdir baseline/_ref \\
      baseline/_ref/abft_guard_tests -p tools.ref_backend_plugin -q
"""


def pytest_configure(config):
    import abft_guard

    from paper_2104_09455_b200 import reference_backend
    reference_backend.install(abft_guard)


def pytest_terminal_summary(terminalreporter):
    from paper_2104_09455_b200 import reference_backend
    terminalreporter.write_line(f"B200 dispatch: {reference_backend.CALLS} calls of the reference entry points "
                                f"ran on the sm_100a path")
