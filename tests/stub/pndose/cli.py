"""The reference CLI's run / oracle commands and exit-code mapping (cli.py:18-37, 115-133)."""

import sys

from .driver import ProblemConfig, run_simulation, write_outputs
from .errors import PnDoseError


def _cmd_run(path, solver):
    config = ProblemConfig.load(path)
    result = run_simulation(config, solver=solver)
    out = write_outputs(result)
    d = result.diagnostics
    print(f"{solver}: {d['n_steps']} steps, mean rank {d['mean_rank']:.2f}, "
          f"state memory {100 * d['state_memory_fraction']:.3f}% of full, "
          f"{d['runtime_s']:.1f} s")
    print(f"outputs written to {out}")
    return 0


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    try:
        return _cmd_run(argv[1], "dlra" if argv[0] == "run" else "fullrank")
    except PnDoseError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return exc.exit_code
