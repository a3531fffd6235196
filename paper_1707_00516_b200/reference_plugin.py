"""Register the B200 kernel with the reference package's own scheduler and CLI.

The reference selects its comparison kernel by name: ``KERNELS = ("blocked",
"naive")`` (scheduler.py:28), validated by ``PipelineConfig`` (scheduler.py:213),
turned into an executor by ``make_executor`` (scheduler.py:243-246) inside
``run_pipeline`` (scheduler.py:285), and exposed as ``--kernel`` by the CLI's
``compare`` and ``bench`` subcommands (cli.py:221, 233).  ``install()`` adds a
third name, ``"b200"``, at exactly those points -- the same edit INTEGRATION.md
§2 shows as a patch, applied at run time to an unmodified install -- so

    fastid compare --refs R --queries Q --out S --kernel b200
    fastid bench --sizes 1000000x2048x16 --kernel b200

and ``run_pipeline(plan, refs, queries, PipelineConfig(kernel="b200"))`` run the
reference's own planner, staging lanes, sinks, ledger, output formats and bench
CSV schema (cli.py:144-147) with every batch scored by ``B200Executor``
(fastid_run_kernel, the C ABI's host-buffer entry).

    from paper_1707_00516_b200 import reference_plugin
    reference_plugin.install()          # imports fastid; idempotent
    ...
    reference_plugin.uninstall()
"""

from __future__ import annotations

import importlib

from .compare import B200Executor

KERNEL_NAME = "b200"

_saved: dict = {}


def install(formulation: str | int = "auto") -> None:
    """Add the "b200" kernel to the importable reference package (``fastid``)."""
    if _saved:
        return
    sched = importlib.import_module("fastid.scheduler")
    cli = importlib.import_module("fastid.cli")
    _saved.update(kernels=sched.KERNELS, make_executor=sched.make_executor, build_parser=cli.build_parser,
                  sched=sched, cli=cli)
    if KERNEL_NAME not in sched.KERNELS:
        sched.KERNELS = tuple(sched.KERNELS) + (KERNEL_NAME,)
    base_make = sched.make_executor

    def make_executor(config):
        if config.kernel == KERNEL_NAME:
            return B200Executor(formulation)
        return base_make(config)

    sched.make_executor = make_executor
    base_parser = cli.build_parser

    def build_parser():
        parser = base_parser()
        for action in parser._subparsers._group_actions:  # the subcommand table
            for sub in action.choices.values():
                for opt in sub._actions:
                    if opt.dest == "kernel" and opt.choices is not None and KERNEL_NAME not in opt.choices:
                        opt.choices = tuple(opt.choices) + (KERNEL_NAME,)
        return parser

    cli.build_parser = build_parser


def uninstall() -> None:
    """Restore the reference's own kernel table, executor factory and parser."""
    if not _saved:
        return
    sched, cli = _saved["sched"], _saved["cli"]
    sched.KERNELS = _saved["kernels"]
    sched.make_executor = _saved["make_executor"]
    cli.build_parser = _saved["build_parser"]
    _saved.clear()


def installed() -> bool:
    return bool(_saved)
