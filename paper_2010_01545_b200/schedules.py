"""Module alias mirroring the reference's `pwadvect.schedules`
(pkg/src/pwadvect/schedules.py). Implementation: engines.py."""

from .engines import (VARIANTS, XSHIFT_ROLES, OutputComparison, ScheduleSpec,  # noqa: F401
                      Slab, TrafficReport, compare_outputs, partition_domain, reference_traffic,
                      run_schedule)
