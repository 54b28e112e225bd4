/* crm_interpose.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Linked into oracle/_ref/libctsm_ref_cr.so (the unmodified reference sources
 * compiled with -fno-builtin) so that the reference's std::sin/cos/tan/atan/
 * atan2 calls bind to the correctly rounded crmath.h functions instead of
 * glibc's. The symbols are hidden, so they bind at link time inside that .so
 * and never interpose anything else in the process. This is the "same libm on
 * both sides" route of SURVEY.md §7 H1: with it the CPU reference and the GPU
 * kernels evaluate bit-identical arithmetic, so their sparsity patterns can be
 * compared bit-exactly. */
#include "crmath.h"

#define CRM_EXPORT __attribute__((visibility("hidden")))

CRM_EXPORT double sin(double x) { return crm_sin(x); }
CRM_EXPORT double cos(double x) { return crm_cos(x); }
CRM_EXPORT double tan(double x) { return crm_tan(x); }
CRM_EXPORT double atan(double x) { return crm_atan(x); }
CRM_EXPORT double atan2(double y, double x) { return crm_atan2(y, x); }
CRM_EXPORT void sincos(double x, double* s, double* c) {
  *s = crm_sin(x);
  *c = crm_cos(x);
}
