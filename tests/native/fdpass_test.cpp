// Stand-alone test of csrc/fdpass.h (tests/test_fdpass_host.py): a forked
// child serves a memfd holding a message; the parent fetches the descriptor
// over the abstract Unix socket and reads the message through it.
#include <sys/mman.h>
#include <sys/wait.h>

#include <cstdio>
#include <cstring>

#include "fdpass.h"

int main() {
  int ready[2], done[2];
  if (pipe(ready) || pipe(done)) return 2;
  const pid_t pid = fork();
  if (pid == 0) {
    const int fd = memfd_create("coconet-test", 0);
    const char msg[] = "symmetric heap";
    if (fd < 0 || write(fd, msg, sizeof(msg)) != ssize_t(sizeof(msg))) _exit(3);
    FdServer srv;
    if (!srv.start("coconet-test")) _exit(4);
    srv.set(2, fd);
    if (write(ready[1], srv.name, sizeof(srv.name)) != ssize_t(sizeof(srv.name))) _exit(5);
    char b;
    if (read(done[0], &b, 1) != 1) _exit(6);  // serve until the parent is done
    srv.stop();
    _exit(0);
  }
  char name[64];
  if (read(ready[0], name, sizeof(name)) != ssize_t(sizeof(name))) return 7;
  const char* why = "";
  const int fd = fd_fetch(name, 2, 5000, &why);
  if (fd < 0) {
    std::printf("FAIL fetch: %s\n", why);
    return 1;
  }
  char buf[32] = {};
  if (pread(fd, buf, sizeof(buf), 0) <= 0 || std::strcmp(buf, "symmetric heap") != 0) {
    std::printf("FAIL content '%s'\n", buf);
    return 1;
  }
  // an empty slot answers without a descriptor; a missing server times out
  if (fd_fetch(name, 1, 5000, &why) != -1 || std::strcmp(why, "the peer has no descriptor in that slot") != 0) {
    std::printf("FAIL empty slot\n");
    return 1;
  }
  if (fd_fetch("coconet-test.no-such-server", 0, 50, &why) != -1) {
    std::printf("FAIL missing server\n");
    return 1;
  }
  if (write(done[1], "x", 1) != 1) return 8;
  int st = 0;
  waitpid(pid, &st, 0);
  if (!WIFEXITED(st) || WEXITSTATUS(st) != 0) {
    std::printf("FAIL child status %d\n", st);
    return 1;
  }
  std::printf("OK\n");
  return 0;
}
