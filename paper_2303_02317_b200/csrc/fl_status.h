/* fl_status.h -- per-option status codes shared by host, device and Python.
 *
 * status = (class << 8) | detail.  Classes mirror the reference exception
 * hierarchy (pkg/src/fftlattice/model.py:44-97); the detail names the field
 * (ValidationError.field), the weight (StabilityError.weight) or the site.
 */
#ifndef FL_STATUS_H
#define FL_STATUS_H

#define FL_OK 0

#define FL_E_VALIDATION 0x100
#define FL_E_STABILITY 0x200
#define FL_E_DOMAIN 0x300
#define FL_E_GEOMETRY 0x400
#define FL_E_NUMERICAL 0x500
#define FL_E_VALUE 0x600    /* plain ValueError: reference math-domain failure */
#define FL_E_CAPACITY 0x700 /* beyond what this GPU build supports (e.g. cutoff) */

/* ValidationError fields (model.py:158-174, model.py:236, bsm.py:178/181, bsm.py:619) */
#define FL_F_SPOT 1
#define FL_F_STRIKE 2
#define FL_F_RATE 3
#define FL_F_YIELD 4
#define FL_F_VOL 5
#define FL_F_DAYS 6
#define FL_F_STEPS 7
#define FL_F_PROB_UP 8
#define FL_F_LAM 9
#define FL_F_CUTOFF 10
#define FL_F_TIMES 11  /* model.py:318-328 via american.py:478-486 (all-exercise row T-1) */

/* StabilityError weights (bsm.py:204-222) */
#define FL_W_MID 1
#define FL_W_UP 2
#define FL_W_DOWN 3

/* DomainError details */
#define FL_D_GRID_NODES 1 /* bsm.py:185-189 */
#define FL_D_STRIKE 2     /* bsm.py:165-166 */
#define FL_D_WINDOW 3     /* binomial.py:212-215 degenerate Gaussian window */
#define FL_D_CF_STRIKE 4  /* binomial.py:265-269 closed form needs a positive strike */

#endif
