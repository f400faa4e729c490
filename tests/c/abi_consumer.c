/* A plain C99 consumer of include/hz.h (compiled by tests/test_abi.py with gcc -std=c99 -pedantic
 * -Werror): the header is valid C, the library links from C, and the host-side calls work without a
 * GPU.  Prints the version, the table size, row 80 (G = 12) of the default table, the class weights of
 * that row, an import round trip and the error path of an invalid call. */
#include <stdio.h>
#include <stdlib.h>

#include "hz.h"

int main(void) {
  hz_table* t = NULL;
  hz_table* t2 = NULL;
  int n_g = 0, n2 = 0, k;
  double* r5;
  double* r7;
  double back[5];
  hz_status st;
  printf("version %s\n", hz_version());
  st = hz_build_weight_table(4.0, 40.0, 0.1, 1e-2, NULL, &t);
  if (st != HZ_OK) {
    printf("build failed %d %s\n", (int)st, hz_last_error());
    return 1;
  }
  if (hz_table_rows(t, &n_g, NULL, NULL) != HZ_OK) return 2;
  r5 = (double*)malloc(sizeof(double) * 5 * (size_t)n_g);
  r7 = (double*)malloc(sizeof(double) * 7 * (size_t)n_g);
  if (hz_table_rows(t, &n_g, r5, r7) != HZ_OK) return 3;
  printf("n_g %d\n", n_g);
  printf("row80");
  for (k = 0; k < 5; k++) printf(" %.17g", r5[80 * 5 + k]);
  printf("\nw7_80");
  for (k = 0; k < 7; k++) printf(" %.17g", r7[80 * 7 + k]);
  printf("\n");
  /* one-row import of that row, exported back bit for bit */
  if (hz_table_import(12.0, 0.1, 1, r5 + 80 * 5, &t2) != HZ_OK) return 4;
  if (hz_table_rows(t2, &n2, back, NULL) != HZ_OK || n2 != 1) return 5;
  for (k = 0; k < 5; k++)
    if (back[k] != r5[80 * 5 + k]) return 6;
  printf("import ok\n");
  /* invalid arguments: negative status, nothing written, a message */
  st = hz_build_weight_table(4.0, 40.0, -0.1, 1e-2, NULL, &t2);
  printf("invalid %d %s\n", (int)st, hz_last_error());
  hz_table_destroy(t);
  hz_table_destroy(t2);
  free(r5);
  free(r7);
  return 0;
}
