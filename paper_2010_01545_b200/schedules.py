"""Module alias mirroring the reference's `pwadvect.schedules`
(pkg/src/pwadvect/schedules.py). Implementation: engines.py."""

from .engines import (VARIANTS, OutputComparison, ScheduleSpec, Slab,  # noqa: F401
                      TrafficReport, compare_outputs, partition_domain, run_schedule)
