"""``python -m paper_1504_02264_b200 <mode> [options]``: the reference CLI
(gmcf-mini: coupled, les-standalone, sor-bench, boundary-audit; cli.py:331-384)
with the hot path on the GPU.  Installs the drop-in (dropin.install) and hands
the arguments to ``gmcf_mini.cli.main``; exit codes are the reference's.  Needs
gmcf_mini importable (the CLI, config parser and coupling runtime are the
reference's host code)."""

import sys


def main(argv=None) -> int:
    try:
        from gmcf_mini import cli
    except ImportError:
        sys.stderr.write("gmcf_mini is not importable: install the reference package to use its CLI\n")
        return 2
    from . import install

    install()
    return cli.main(argv)


if __name__ == "__main__":
    sys.exit(main())
