// Host-only file-descriptor passing between the processes of one node (no
// CUDA): the cuMem heap exports its allocation as a POSIX file descriptor
// (CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR), which only means something
// inside the exporting process, so every rank serves its descriptors over an
// abstract-namespace Unix socket and peers fetch them with SCM_RIGHTS.
// Included by heap_cumem.cu and compiled stand-alone by
// tests/test_fdpass_host.py.
#pragma once

#include <poll.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <time.h>
#include <unistd.h>

#include <atomic>
#include <cerrno>
#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>

// Serves up to kSlots descriptors (request = slot index as uint32, reply = one
// byte of status plus the descriptor as ancillary data) until stop().
struct FdServer {
  static constexpr int kSlots = 4;
  int sock = -1;
  char name[64] = {};  // abstract name without the leading NUL
  std::atomic<int> fds[kSlots];
  std::atomic<bool> stopping{false};
  std::thread th;

  FdServer() {
    for (auto& f : fds) f.store(-1);
  }
  // Binds "\0<prefix>.<pid>.<unique>" and starts the accept thread.
  bool start(const char* prefix) {
    static std::atomic<unsigned> uniq{0};
    std::snprintf(name, sizeof(name), "%s.%d.%u", prefix, int(getpid()), uniq.fetch_add(1));
    sock = socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
    if (sock < 0) return false;
    sockaddr_un a{};
    socklen_t len = addr(name, &a);
    if (bind(sock, reinterpret_cast<sockaddr*>(&a), len) != 0 || listen(sock, 64) != 0) {
      close(sock);
      sock = -1;
      return false;
    }
    th = std::thread([this] { loop(); });
    return true;
  }
  void set(int slot, int fd) { fds[slot].store(fd); }
  void stop() {
    if (sock < 0) return;
    stopping.store(true);
    if (th.joinable()) th.join();
    close(sock);
    sock = -1;
  }
  ~FdServer() { stop(); }

  static socklen_t addr(const char* nm, sockaddr_un* a) {
    a->sun_family = AF_UNIX;
    a->sun_path[0] = '\0';
    const size_t n = std::strlen(nm);
    std::memcpy(a->sun_path + 1, nm, n);
    return socklen_t(offsetof(sockaddr_un, sun_path) + 1 + n);
  }

 private:
  void loop() {
    while (!stopping.load()) {
      pollfd p{sock, POLLIN, 0};
      const int r = poll(&p, 1, 50);
      if (r <= 0) continue;
      const int cfd = accept4(sock, nullptr, nullptr, SOCK_CLOEXEC);
      if (cfd < 0) continue;
      // abstract sockets are visible to every process of the network
      // namespace: hand descriptors (device memory) to the same user only
      ucred cr{};
      socklen_t crl = sizeof(cr);
      if (getsockopt(cfd, SOL_SOCKET, SO_PEERCRED, &cr, &crl) != 0 || cr.uid != getuid()) {
        close(cfd);
        continue;
      }
      uint32_t slot = 0;
      pollfd pc{cfd, POLLIN, 0};
      if (poll(&pc, 1, 2000) == 1 && recv(cfd, &slot, sizeof(slot), MSG_WAITALL) == ssize_t(sizeof(slot))) {
        const int fd = slot < uint32_t(kSlots) ? fds[slot].load() : -1;
        send_fd(cfd, fd);
      }
      close(cfd);
    }
  }
  static void send_fd(int cfd, int fd) {
    char ok = fd >= 0 ? 1 : 0;
    iovec iov{&ok, 1};
    msghdr m{};
    m.msg_iov = &iov;
    m.msg_iovlen = 1;
    alignas(cmsghdr) char ctl[CMSG_SPACE(sizeof(int))] = {};
    if (fd >= 0) {
      m.msg_control = ctl;
      m.msg_controllen = sizeof(ctl);
      cmsghdr* c = CMSG_FIRSTHDR(&m);
      c->cmsg_level = SOL_SOCKET;
      c->cmsg_type = SCM_RIGHTS;
      c->cmsg_len = CMSG_LEN(sizeof(int));
      std::memcpy(CMSG_DATA(c), &fd, sizeof(int));
    }
    sendmsg(cfd, &m, MSG_NOSIGNAL);
  }
};

// Fetches descriptor `slot` from the server `name` (retrying the connect for
// up to `timeout_ms` while the peer starts). Returns a new local descriptor,
// or -1 (errno-style reason in *why).
inline int fd_fetch(const char* name, uint32_t slot, int timeout_ms, const char** why) {
  sockaddr_un a{};
  const socklen_t len = FdServer::addr(name, &a);
  timespec t0{};
  clock_gettime(CLOCK_MONOTONIC, &t0);
  for (;;) {
    const int s = socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
    if (s < 0) {
      *why = "socket() failed";
      return -1;
    }
    if (connect(s, reinterpret_cast<sockaddr*>(&a), len) == 0) {
      int fd = -1;
      if (send(s, &slot, sizeof(slot), MSG_NOSIGNAL) == ssize_t(sizeof(slot))) {
        char ok = 0;
        iovec iov{&ok, 1};
        msghdr m{};
        m.msg_iov = &iov;
        m.msg_iovlen = 1;
        alignas(cmsghdr) char ctl[CMSG_SPACE(sizeof(int))] = {};
        m.msg_control = ctl;
        m.msg_controllen = sizeof(ctl);
        if (recvmsg(s, &m, MSG_CMSG_CLOEXEC) == 1 && ok) {
          cmsghdr* c = CMSG_FIRSTHDR(&m);
          if (c && c->cmsg_level == SOL_SOCKET && c->cmsg_type == SCM_RIGHTS) std::memcpy(&fd, CMSG_DATA(c), sizeof(int));
        }
        if (fd < 0) *why = "the peer has no descriptor in that slot";
      } else {
        *why = "send() failed";
      }
      close(s);
      return fd;
    }
    close(s);
    timespec t{};
    clock_gettime(CLOCK_MONOTONIC, &t);
    const long ms = (t.tv_sec - t0.tv_sec) * 1000 + (t.tv_nsec - t0.tv_nsec) / 1000000;
    if (ms > timeout_ms) {
      *why = "could not connect to the peer's descriptor server";
      return -1;
    }
    usleep(2000);
  }
}
